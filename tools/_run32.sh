HHB_GEMM_PAIRS_DEBUG=1 timeout 60 python tools/time_gemm.py 2>&1 | sort | uniq
timeout 120 ncu --set full --clock-control none -k regex:k_umma_gemm_2sm -c 1 -o gpurun_out/gemm2sm -f python tools/time_gemm.py > gpurun_out/ncu32.log 2>&1; tail -1 gpurun_out/ncu32.log
