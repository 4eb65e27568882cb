set -x
timeout 900 python -m pytest tests/test_gpu_core.py -x -q -k "gemm" 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c.json 2>gpurun_out/bench_c.err
PEPSB_GEMM_WS=2 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t.json 2>gpurun_out/bench_t.err
for f in bench_c bench_t; do python -c "
import json
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$f', round(d['ms_per_step'],2), round(d['value'],2), round(r['frac'],3), round(r['achieved_algorithmic'],2), r['breakdown_ms'])"; done
