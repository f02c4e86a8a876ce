#!/bin/sh
# Debug build of libforkattn with timelines (-DFK_TIMELINE): CTA 0 phase stamps
# of the tcgen05 prefix kernel and per-CTA start/end stamps of the prefix and
# private kernels.  Output: profiles/build/libforkattn_tl.so (not product).
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2405_19888_b200/csrc
make -s -C "$C"
mkdir -p "$R/profiles/build"
for f in fk_prefix_tc fk_kernels; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I"$R/include" -I"$C" -DFK_TIMELINE -c "$C/$f.cu" -o "$C/build/${f}_tl.o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$R/profiles/build/libforkattn_tl.so" \
  "$C/build/fk_pool.o" "$C/build/fk_kernels_tl.o" "$C/build/fk_prefix_tc_tl.o" -cudart static
