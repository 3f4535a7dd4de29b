#!/bin/bash
# C4 parity tests + deadline sweep
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c4" 2>&1 | tail -1
timeout 1500 python bench.py --config c4 --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/c4.json
python -c "
import json; d=json.load(open('gpurun_out/c4.json')); print('S_max', d['value'], 'ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), 'e2e', d['e2e']['value'], 'cap', d['config']['memory_cap_sources'])"
