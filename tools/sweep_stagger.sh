for s in 0 1000 2000 3000; do NDF_TC_STAGGER=$s timeout 300 python bench.py --quick --steps 30 --warmup 5 | python -c "import json,sys; d=json.load(sys.stdin); print('stagger', $s, d['value'], d['roofline']['frac'])"; done
NDF_TC_STAGGER=2000 python tools/trace_tc.py | tail -12
