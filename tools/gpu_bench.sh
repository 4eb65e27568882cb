set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; tail -3 gpurun_out/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc $?
python -c "
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],2), round(d['value'],2), round(r['frac'],3), r['breakdown_ms'], d['e2e']['value'], d.get('s_per_norm'))"
timeout 900 python tools/bench_configs.py --configs 3 2>&1 | cut -c1-600
