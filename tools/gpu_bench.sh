set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; tail -3 gpurun_out/pytest.log
PEPSB_OVERLAP=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench0.json 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc $?
for f in bench0 bench; do python -c "
import json
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$f', round(d['ms_per_step'],2), round(d['value'],2), round(r['frac'],3), r['breakdown_ms'], d['e2e']['s_per_step'], d.get('s_per_norm'))"; done
timeout 900 python tools/bench_configs.py --configs 4,1,3 > gpurun_out/cfg.jsonl 2>&1; cut -c1-400 gpurun_out/cfg.jsonl
