for rep in 1 2; do for s in 1 0; do
PEPSB_GEMM_SMALL=$s timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench_s$s.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_s$s.json').read().strip().splitlines()[-1]); r=d['roofline']; print('small=$s', round(d['ms_per_step'],2), r['breakdown_ms'])"
PEPSB_GEMM_SMALL=$s timeout 900 python tools/bench_configs.py --configs 1,3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('small=$s cfg', d['config'], round(d['s_per_norm'],5), d.get('cache_s'))"
done; done
