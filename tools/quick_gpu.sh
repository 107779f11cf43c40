#!/bin/bash
# One quick gpurun iteration: GPU tests, quick bench (+classic schedule), schedule trace,
# launch list.  Outputs under gpurun_out/.
timeout 240 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 180 python bench.py --quick --steps 40 --warmup 5 > gpurun_out/quick.json 2>gpurun_out/quick.err
[ -f abtest/lib_trace.so ] && NDF_TRACE_LIB=abtest/lib_trace.so timeout 120 python tools/trace_ws.py > gpurun_out/trace_ws.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
if [ "${PROFILE:-0}" = 1 ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"query_(tc|ws|pp)" -s 2 -c 1 \
      -o gpurun_out/prof_query python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu_q.log 2>&1
fi
