for rep in 1 2; do for pr in 1 0; do
PEPSB_STREAM_PRIORITY=$pr timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench_p.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_p.json').read().strip().splitlines()[-1]); r=d['roofline']; print('prio=$pr', round(d['ms_per_step'],2), r['breakdown_ms'])"
done; done
PEPSB_STREAM_PRIORITY=1 timeout 900 python tools/bench_configs.py --configs 3 2>&1 | cut -c1-250
PEPSB_STREAM_PRIORITY=0 timeout 900 python tools/bench_configs.py --configs 3 2>&1 | cut -c1-250
