for t in 512 384 256; do
PEPSB_EIG_THREADS=$t timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench_e.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_e.json').read().strip().splitlines()[-1]); r=d['roofline']; print('threads=$t', round(d['ms_per_step'],2), r['breakdown_ms'])"
done
