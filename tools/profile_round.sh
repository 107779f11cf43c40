#!/bin/bash
# One gpurun call: plain bench, launch list, and ncu --set full captures of the
# three hot kernels (query, Pearson GEMV, KSG).  Outputs under gpurun_out/.
set -u
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
python bench.py --quick --steps 2 --warmup 1 > gpurun_out/plain_quick.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --quick --steps 2 --warmup 1 \
    > gpurun_out/ncu_launch.log 2>&1
python tools/gemv_probe.py > gpurun_out/plain_gemv.log 2>&1 && \
python tools/ksg_probe.py 16384 > gpurun_out/plain_ksg.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"query_(tc|ws|pp)" -s 1 -c 1 \
    -o gpurun_out/prof_query python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu_q.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemv -s 1 -c 1 \
    -o gpurun_out/prof_gemv python tools/gemv_probe.py > gpurun_out/ncu_g.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ksg_kernel -s 1 -c 1 \
    -o gpurun_out/prof_ksg python tools/ksg_probe.py 16384 > gpurun_out/ncu_k.log 2>&1
echo "profile done rc=$?"
