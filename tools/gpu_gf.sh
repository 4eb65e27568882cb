timeout 600 ncu --set full --import-source on --clock-control none -k regex:gram_factors -s 2 -c 1 -o gpurun_out/gf72 python tools/one_gf.py > gpurun_out/gf72.log 2>&1; echo ncu $?
