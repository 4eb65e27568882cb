set -x
timeout 300 python tools/prof_cfg1.py
NORMS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg1_launches.csv python tools/prof_cfg1.py > gpurun_out/cfg1_ncu.log 2>&1; echo ncu $?
python tools/launch_summary.py gpurun_out/cfg1_launches.csv 7 30
