bash tools/bench_variants.sh "X=0" "HHB_JIT_TWO_RCP=2" "HHB_JIT_TWO_RCP=3" "HHB_JIT_TWO_RCP=4" "HHB_JIT_TWO_RCP=6"
