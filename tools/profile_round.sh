#!/bin/bash
# One gpurun call: the full bench, the launch list of the quick bench, and an ncu --set full
# capture of each kernel family (each probe first runs plain and must exit 0).  Outputs
# under gpurun_out/; summarise with tools/summarize_profiles.py <round> gpurun_out/prof_*.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --quick --steps 2 --warmup 1 > gpurun_out/plain_quick.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --quick --steps 2 --warmup 1 \
    > gpurun_out/ncu_launch.log 2>&1
prof() {   # prof <name> <kernel regex> <skip> <command...>
  local name=$1 regex=$2 skip=$3; shift 3
  timeout 300 "$@" > gpurun_out/plain_$name.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$regex" -s "$skip" -c 1 \
      -o gpurun_out/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "prof $name rc=$?"
}
prof x3 query_x3 1 python tools/x3_probe.py 2
PREC=fp16 prof pp query_pp 1 python tools/x3_probe.py 2
prof preptab prep_x3_tab 1 python tools/x3_probe.py 2
prof prepfeat prep_ws_feat 1 python tools/x3_probe.py 2
prof embed embed_kernel 1 python tools/embed_probe.py
prof field pearson_field 1 python tools/gemv_probe.py
prof ksg ksg_kernel 1 python tools/ksg_probe.py 16384
prof c3 query_x3 1 python tools/c3_probe.py
prof pairs_ksg ksg_kernel 1 python tools/c4_probe.py 16384
prof pairs_pearson pearson_pairs 1 python tools/c4_probe.py 16384
echo "profile done"
