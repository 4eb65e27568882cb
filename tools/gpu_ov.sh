set -x
timeout 1200 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest.log 2>&1; tail -15 gpurun_out/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2>gpurun_out/bench.err
timeout 900 python tools/bench_configs.py --configs 4b,1 --ref > gpurun_out/cfg4b.jsonl 2>&1; tail -3 gpurun_out/cfg4b.jsonl
