set -x
timeout 900 python -m pytest tests/test_gpu_core.py -x -q -k "gemm" 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench.json 2>gpurun_out/bench.err
python -c "
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],2), round(d['value'],2), round(r['frac'],3), r['breakdown_ms'], d['e2e']['s_per_step'])"
