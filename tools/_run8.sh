timeout 300 ncu --set full --import-source on --clock-control none -k regex:hh_bwd -s 3 -c 1 -o gpurun_out/bwd_ring -f python tools/time_bwd.py > gpurun_out/ncu8.log 2>&1; tail -1 gpurun_out/ncu8.log
