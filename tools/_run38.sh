set -x
timeout 300 ncu --set full --import-source on --clock-control none -k regex:hh_fwdp -c 1 -o gpurun_out/r1_fwdp -f python tools/prof_fwd.py --neurons 2000000 --steps 200 > gpurun_out/n1.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:hh_bwd -s 3 -c 1 -o gpurun_out/r1_bwd2 -f python tools/time_bwd.py > gpurun_out/n2.log 2>&1
STEPS=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:hh_fwd -s 1 -c 1 -o gpurun_out/r1_fwdtrain -f python tools/prof_layer.py > gpurun_out/n3.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_umma_gemm_2sm -c 3 -o gpurun_out/r1_gemm2sm -f python tools/time_gemm.py > gpurun_out/n4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_bench_launches.csv python bench.py --steps 1 --warmup 1 --no-extras > gpurun_out/n5.log 2>&1
timeout 300 python tools/prof_torch.py c3 > gpurun_out/prof_c3.txt 2>/dev/null
timeout 300 python tools/prof_torch.py c4 > gpurun_out/prof_c4.txt 2>/dev/null
timeout 300 python tools/prof_c5.py > gpurun_out/prof_c5.txt 2>/dev/null
