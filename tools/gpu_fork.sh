for rep in 1 2; do for f in 1 0; do
PEPSB_FORK_AFTER_GRAM=$f timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench_f.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_f.json').read().strip().splitlines()[-1]); r=d['roofline']; print('fork_late=$f', round(d['ms_per_step'],2), r['breakdown_ms'])"
done; done
timeout 900 python -m pytest tests/test_gpu_core.py tests/test_gpu_peps.py -q -x 2>&1 | tail -2
