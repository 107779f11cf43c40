#!/bin/bash
# Run the quick bench for each prebuilt abtest/lib_<name>.so (interleaved, 2 reps).
cp paper_2307_02203_b200/libndf_b200.so abtest/lib_orig.so
for rep in 1 2; do
  for v in "$@"; do
    cp abtest/lib_$v.so paper_2307_02203_b200/libndf_b200.so
    timeout 180 python bench.py --quick --steps 40 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['value'],4), round(d['roofline']['kernel_ms'],4))"
  done
done
cp abtest/lib_orig.so paper_2307_02203_b200/libndf_b200.so
