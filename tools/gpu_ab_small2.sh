timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; tail -3 gpurun_out/pytest.log
for s in 1 0 1; do
PEPSB_GEMM_SMALL=$s timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench_s$s.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_s$s.json').read().strip().splitlines()[-1]); r=d['roofline']; print('small=$s', round(d['ms_per_step'],2), r['breakdown_ms'])"
PEPSB_GEMM_SMALL=$s timeout 300 python tools/prof_cfg1.py
done
