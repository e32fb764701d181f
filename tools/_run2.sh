timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/bench_variants.sh "HHB_JIT_MINB=2" "HHB_JIT_MINB=3" "HHB_JIT_MINB=4" "HHB_JIT_MINB=3 -- --no-fuse" "HHB_JIT_MINB=4 -- --no-fuse"
