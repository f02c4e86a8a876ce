#!/bin/bash
# Single-bf16 P (no hi/lo split) in the tcgen05 prefix kernel: parity, steady-state power, burst A/B.
cd "$(dirname "$0")/../../.."
O=gpurun_out/psingle; mkdir -p $O
A=.ab/libforkattn_head.so; B=.ab/libforkattn_psingle.so
FK_LIB_PATH=$PWD/$B timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "tc or fullsize or headline" > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
tail -2 $O/parity.log
for r in 1 2; do
  for lib in $A $B; do
    FK_LIB_PATH=$PWD/$lib timeout 300 python profiles/power_probe.py --shapes 6000,64,256 6000,256,256 --seconds 4 2>&1 | grep "^{" | sed "s|^|$lib |"
  done
done > $O/power.log
cat $O/power.log
timeout 600 python profiles/lib_ab.py --a $A --b $B --rounds 3 > $O/ab.log 2>&1; tail -2 $O/ab.log
