#!/bin/bash
# Config-4 bulk pairs (tools/c4_probe.py) for each prebuilt abtest/lib_<name>.so.
cp paper_2307_02203_b200/libndf_b200.so abtest/lib_orig.so
for v in "$@"; do
  cp abtest/lib_$v.so paper_2307_02203_b200/libndf_b200.so
  echo "$v $(timeout 300 python tools/c4_probe.py 2>&1 | tail -1)"
done
cp abtest/lib_orig.so paper_2307_02203_b200/libndf_b200.so
