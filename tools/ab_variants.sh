#!/bin/bash
# Time each prebuilt variants/lib_<name>.so with a probe command (interleaved, 2 reps):
#   bash tools/ab_variants.sh "python tools/x3_probe.py 20" base nomufu ...
cmd=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    echo -n "$v: "
    NDF_LIB_PATH=variants/lib_$v.so timeout 180 $cmd 2>&1 | tail -1
  done
done
