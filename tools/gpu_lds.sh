timeout 900 python -m pytest tests/test_gpu_eigh.py tests/test_gpu_core.py -q -x 2>&1 | tail -2
timeout 300 python tools/eig_timing.py 2>&1 | tail -10
for rep in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench_l.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_l.json').read().strip().splitlines()[-1]); r=d['roofline']; print('lds', round(d['ms_per_step'],2), r['breakdown_ms'])"
done
