bash tools/gpu_final.sh
timeout 1500 python tools/bench_configs.py --configs 1,4,3,5 --ref > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo configs rc $?
cut -c1-400 gpurun_out/configs.jsonl
