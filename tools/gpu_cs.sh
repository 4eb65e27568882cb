for cs in 0 1; do
PEPSB_CONCURRENT_SWEEPS=$cs timeout 900 python tools/bench_configs.py --configs 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('cs=$cs', round(d['s_per_norm'],3), d.get('cache_s'), d.get('cached_norm_bitwise_equal'))"
done
for pr in 1 2; do
PEPSB_PIPELINE_ROWS=$pr PEPSB_CONCURRENT_SWEEPS=0 timeout 900 python tools/bench_configs.py --configs 5 --zz none 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('pr=$pr', round(d['s_per_norm'],3))"
done
