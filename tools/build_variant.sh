#!/bin/bash
# Build a variant libgk (extra nvcc -D flags) for A/B timing:
#   tools/build_variant.sh NAME -DGK_XINV_WARPS=10 ...
#   GK_LIB_PATH=build/variants/libgk_NAME.so python tools/quick_timing.py sh03b
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/variants/$name; mkdir -p $out
for f in paper_2305_10553_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude "$@" -c $f -o $out/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/variants/libgk_$name.so $out/*.o
echo built build/variants/libgk_$name.so
