#!/bin/sh
# Debug build of libforkattn with the tcgen05 prefix-kernel timeline (-DFK_TIMELINE).
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2405_19888_b200/csrc
make -s -C "$C"
mkdir -p "$R/profiles/build"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I"$R/include" -I"$C" -DFK_TIMELINE -c "$C/fk_prefix_tc.cu" -o "$C/build/fk_prefix_tc_tl.o"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$R/profiles/build/libforkattn_tl.so" \
  "$C/build/fk_pool.o" "$C/build/fk_kernels.o" "$C/build/fk_prefix_tc_tl.o" -cudart static
