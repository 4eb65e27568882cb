set -x
timeout 1500 python tools/bench_configs.py --configs 4,4b --ref > gpurun_out/cfg4.jsonl 2>&1; tail -3 gpurun_out/cfg4.jsonl
