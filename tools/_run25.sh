timeout 300 ncu --set full --import-source on --clock-control none -k regex:hh_bwd -s 3 -c 1 -o gpurun_out/bwd_v2 -f python tools/time_bwd.py > gpurun_out/ncu25.log 2>&1; tail -1 gpurun_out/ncu25.log
