#!/bin/bash
# Schedule trace (tools/trace_ws.py) for each prebuilt abtest/lib_<name>.so.
cp paper_2307_02203_b200/libndf_b200.so abtest/lib_orig.so
for v in "$@"; do
  cp abtest/lib_$v.so paper_2307_02203_b200/libndf_b200.so
  echo "== $v"; timeout 120 python tools/trace_ws.py 2>&1 | tail -9
done
cp abtest/lib_orig.so paper_2307_02203_b200/libndf_b200.so
