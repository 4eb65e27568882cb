set -x
for c in 0 1 2; do
PEPSB_CR_CFG=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench_cr$c.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_cr$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cr$c', round(d['ms_per_step'],2), round(d['value'],2), round(r['frac'],3), r['breakdown_ms'])"
done
PEPSB_CR_CFG=1 timeout 900 python -m pytest tests/test_gpu_core.py -x -q -k "complex_by_real" 2>&1 | tail -2
