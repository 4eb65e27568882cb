# warp-Jacobi for small k: eig tests, per-size timing, config 1/3 latency
set -x
timeout 900 python -m pytest tests/test_gpu_eigh.py tests/test_gpu_core.py -x -q 2>&1 | tail -3
timeout 300 python tools/eig_timing.py 2>&1 | tail -12
timeout 900 python tools/bench_configs.py --configs 1,3 2>&1 | cut -c1-400
