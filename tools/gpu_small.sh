set -x
timeout 900 python -m pytest tests/test_gpu_core.py -x -q 2>&1 | tail -3
timeout 300 python tools/prof_cfg1.py
NORMS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg1_launches.csv python tools/prof_cfg1.py > gpurun_out/cfg1_ncu.log 2>&1; echo ncu $?
python tools/launch_summary.py gpurun_out/cfg1_launches.csv 7 12
timeout 900 python tools/bench_configs.py --configs 1,3 2>&1 | cut -c1-300
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench_s.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_s.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],2), round(d['value'],2), round(r['frac'],3), r['breakdown_ms'])"
