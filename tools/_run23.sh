timeout 300 ncu --set full --clock-control none -k regex:k_umma_gemm_p -c 3 -o gpurun_out/gemm_p -f python tools/time_gemm.py > gpurun_out/ncu23.log 2>&1; tail -1 gpurun_out/ncu23.log
