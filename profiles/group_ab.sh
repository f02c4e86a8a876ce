#!/bin/bash
# Interleaved A/B at small fan-outs: prefix on tcgen05 (GROUP_FANOUT=0) vs
# grouped in the private kernel (GROUP_FANOUT=16); profiles/ab.py per fan-out.
for b in ${FANOUTS:-2 4 8 16}; do
  echo "B=$b"
  timeout 200 python profiles/ab.py --shape 6000,$b,256 --set GROUP_FANOUT=0 --set GROUP_FANOUT=16 --rounds 3 --steps 6 2>&1 | tail -2
done
