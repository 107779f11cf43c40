#!/bin/bash
# Config-3 cube time (tools/c3_probe.py) for each prebuilt abtest/lib_<name>.so.
cp paper_2307_02203_b200/libndf_b200.so abtest/lib_orig.so
for rep in 1 2; do
  for v in "$@"; do
    cp abtest/lib_$v.so paper_2307_02203_b200/libndf_b200.so
    echo "$v $(timeout 300 python tools/c3_probe.py 2>&1 | tail -1)"
  done
done
cp abtest/lib_orig.so paper_2307_02203_b200/libndf_b200.so
