#!/bin/bash
# Round profiling in parts (gpurun brings back <= 64 MiB of gpurun_out/ per call):
#   bash tools/profile_round.sh bench   -- full bench, reference arm, launch list
#   bash tools/profile_round.sh ncu1    -- ncu --set full: query_x3 (with source), prep, embed
#   bash tools/profile_round.sh ncu2    -- ncu --set full: Pearson field, KSG, pair kernels, z-score
#   bash tools/profile_round.sh ncu3    -- ncu --set full: config-3 cube launch, fp16 query_pp
# Each probe first runs plain and must exit 0.  Summarise here with
# tools/summarize_profiles.py <round> gpurun_out/prof_*.ncu-rep.
set -u
mkdir -p gpurun_out
prof() {   # prof <name> <kernel regex> <extra ncu flags> <command...>
  local name=$1 regex=$2 extra=$3; shift 3
  timeout 300 "$@" > gpurun_out/plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none $extra -k regex:"$regex" -s 1 -c 1 \
      -o gpurun_out/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "prof $name rc=$?"
}
case "${1:-bench}" in
  bench)
    timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
    echo "bench rc=$?"
    timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
    echo "ref rc=$?"
    python bench.py --quick --steps 2 --warmup 1 > gpurun_out/plain_quick.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python bench.py --quick --steps 2 --warmup 1 \
        > gpurun_out/ncu_launch.log 2>&1
    echo "launches rc=$?";;
  ncu1)
    prof x3 query_x3 "--import-source on" python tools/x3_probe.py 2
    prof preptab prep_x3_kernel "" python tools/x3_probe.py 2
    prof embed "embed_(nodes_)?kernel" "" python tools/embed_probe.py;;
  ncu2)
    prof field pearson_field "" python tools/gemv_probe.py
    prof ksg ksg_kernel "" python tools/ksg_probe.py 16384
    prof pairs_ksg ksg_kernel "" python tools/c4_probe.py 16384
    prof pairs_pearson pearson_pairs "" python tools/pairs_pearson_probe.py
    prof zscore zscore_kernel "" python tools/zscore_probe.py 1;;
  ncu3)
    prof c3 query_x3 "" python tools/c3_probe.py
    export PREC=fp16
    prof pp query_pp "" python tools/x3_probe.py 2;;
esac
ls -la gpurun_out/ | tail -20
