timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; tail -3 gpurun_out/pytest.log
timeout 300 python tools/prof_cfg1.py
timeout 900 python tools/bench_configs.py --configs 1,3 2>&1 | cut -c1-300
