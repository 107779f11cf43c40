#!/bin/bash
# Schedule trace (tools/trace_ws.py) for each prebuilt trace build abtest/lib_<name>.so
# (build with -DNDF_TRACE_BUILD, e.g. tools/build_variants.sh trace).
for v in "$@"; do
  echo "== $v"; NDF_TRACE_LIB=abtest/lib_$v.so timeout 120 python tools/trace_ws.py 2>&1 | tail -30
done
