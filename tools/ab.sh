# A/B: swap prebuilt libraries and run the quick bench for each, interleaved
for rep in 1 2; do for v in A B; do cp abtest/lib_$v.so paper_2307_02203_b200/libndf_b200.so; python bench.py --quick --steps 40 --warmup 5 | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['value'],4))"; done; done
