# Per-config measurements (configs 1,3,4,5) + one ncu --set full capture of the top GEMM launches.
set -x
timeout 1500 python tools/bench_configs.py --configs ${CONFIGS:-1,4,3,5} --ref > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
echo configs rc $?
LIST=0 SKIP=300 COUNT=2 bash tools/ncu_round.sh
