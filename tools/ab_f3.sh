#!/bin/bash
# Reference-default (F3) query time (tools/f3_probe.py) for each prebuilt abtest/lib_<name>.so.
cp paper_2307_02203_b200/libndf_b200.so abtest/lib_orig.so
for rep in 1 2; do
  for v in "$@"; do
    cp abtest/lib_$v.so paper_2307_02203_b200/libndf_b200.so
    echo "$v $(timeout 120 python tools/f3_probe.py 2>&1 | tail -1)"
  done
done
cp abtest/lib_orig.so paper_2307_02203_b200/libndf_b200.so
