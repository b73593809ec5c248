# pair-forward check: GPU tc tests + bench with ADATTN_FWD_PAIRS=0/1
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | grep -E "passed|failed|Error|assert" | head -20
for P in ${PAIRS:-0 1}; do
ADATTN_FWD_PAIRS=$P timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --sweep "" --e2e-steps 0 > gpurun_out/fp$P.json 2>gpurun_out/fp$P.err
python -c "
import json; d=json.load(open('gpurun_out/fp$P.json')); print('P=$P value', round(d['value'],1), 'ms', round(d['ms_per_step'],2), {k:round(v['ms_avg'],2) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/fp$P.err
done
