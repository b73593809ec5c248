#!/bin/bash
# quick GPU check: TC parity tests + a short bench (kernel times).  Usage: tools/quick.sh [pytest-args]
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q ${@} 2>&1 | grep -E "passed|failed|Error|error|assert" | head -8
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --sweep "" --e2e-steps 0 > gpurun_out/quick.json 2>gpurun_out/quick.err
python -c "
import json; d=json.load(open('gpurun_out/quick.json')); print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],2), {k:round(v['ms_avg'],2) for k,v in d['kernels'].items()}, 'iters', d['tau_iters_avg'], 'sp', d['block_sparsity'], d['clocks'])" || tail -5 gpurun_out/quick.err
