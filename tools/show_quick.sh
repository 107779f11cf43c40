#!/bin/bash
tail -2 gpurun_out/pytest_gpu.log
grep -E "^E  |FAILED" gpurun_out/pytest_gpu.log | head -5
python -c "
import json; d=json.load(open('gpurun_out/quick.json')); print('value', d['value'], 'kernel', d['roofline']['kernel_ms'])"
tail -9 gpurun_out/trace_ws.log
grep -E "query|prep" gpurun_out/launches.csv | awk -F'","' '{print $5, $NF}' | tail -3
