#!/bin/bash
# Build variants of proj_gemm.cu (compile-time knobs) into /tmp and time the
# config-3 GEMM shapes with each (tools/time_gemm.py via HHB200_LIB).
#   bash tools/gemm_variants.sh "-DEPI2_BUFS=2" "-DEPI2_WARPS=4" ...
set -e
python -m paper_2601_21407_b200._build > /dev/null
OBJ=paper_2601_21407_b200/build
others=$(ls $OBJ/*.o | grep -v proj_gemm.o)
echo "default: $(python tools/time_gemm.py | tr '\n' ' ')"
for fl in "$@"; do
  tag=$(echo "$fl" | tr -c 'A-Za-z0-9' '_')
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -I include $fl -c paper_2601_21407_b200/csrc/proj_gemm.cu -o /tmp/pg_$tag.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o /tmp/lib_$tag.so $others /tmp/pg_$tag.o -ldl
  echo "$fl: $(HHB200_LIB=/tmp/lib_$tag.so python tools/time_gemm.py | tr '\n' ' ')"
done
