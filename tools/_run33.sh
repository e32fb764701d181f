timeout 60 python tools/time_gemm.py
timeout 120 ncu --set full --import-source on --clock-control none -k regex:k_umma_gemm_2sm -c 1 -o gpurun_out/gemm2sm_b -f python tools/time_gemm.py > gpurun_out/ncu33.log 2>&1; tail -1 gpurun_out/ncu33.log
