set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; tail -3 gpurun_out/pytest.log
timeout 600 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc $?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rcref $?
python -c "
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],2), round(d['value'],2), round(r['frac'],3), r['breakdown_ms'], d['e2e']['value'], d.get('s_per_norm'), d['clocks'])
d=json.loads(open('gpurun_out/bench_ref.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
