#!/bin/bash
# quick GPU check incl. the sparsity sweep
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | grep -E "passed|failed|Error|error|assert" | head -8
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu --sweep "${SWEEP:-0.6,0.8,1.0}" --alphas "${ALPHAS:-}" --e2e-steps 0 > gpurun_out/quick.json 2>gpurun_out/quick.err
python -c "
import json; d=json.load(open('gpurun_out/quick.json')); print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],2), {k:round(v['ms_avg'],2) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])
for s in d['sweep']: print('  beta', s['beta'], 'sp', round(s['block_sparsity'],4), 'ms', round(s['ms'],2), 'eff', round(s['tflops_eff'],1), 'alg', round(s['tflops_alg'],1))" || tail -5 gpurun_out/quick.err
