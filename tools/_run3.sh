timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest3.log 2>&1; tail -2 gpurun_out/pytest3.log
timeout 300 python tools/prof_fwd.py --neurons 2000000 --steps 200 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:hh_fwdp -c 1 -o gpurun_out/fwdp_merged -f python tools/prof_fwd.py --neurons 2000000 --steps 200 > gpurun_out/ncu3.log 2>&1; tail -2 gpurun_out/ncu3.log
bash tools/bench_variants.sh "HHB_JIT_MINB=1" "HHB_JIT_MINB=2" "HHB_JIT_MINB=2 -- --no-fuse"
