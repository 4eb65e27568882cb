set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for k in 2 3 4; do
PEPSB_PIPELINE_ROWS=$k timeout 900 python tools/bench_configs.py --configs 3,5 --zz none 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('K=$k', d['config'], 's_per_norm', round(d['s_per_norm'],3), 'cache', d.get('cache_s'), 'norm', d['norm'][0])
"
done
