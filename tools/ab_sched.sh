#!/bin/bash
# Single-reference query: ping-pong kernel (default) vs the classic schedule.
for rep in 1 2; do for sch in default classic; do NDF_TC_SCHEDULE=$sch python bench.py --quick --steps 40 --warmup 5 | python -c "import json,sys; d=json.load(sys.stdin); print('$sch', round(d['value'],4))"; done; done
