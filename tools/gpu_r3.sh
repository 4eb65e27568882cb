timeout 900 python -m pytest tests/test_gpu_peps.py -q -x -k "scheduling or row_cache" 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --configs 5 --zz none 2>&1 | cut -c1-200
timeout 900 python tools/bench_configs.py --configs 5 2>&1 | cut -c1-600
LIST=1 KREGEX='regex:\(int\)1, \(int\)2>' SKIP=160 COUNT=1 bash tools/ncu_round.sh > /dev/null 2>&1; echo ncu $?
python tools/launch_summary.py gpurun_out/launches.csv 2 30
