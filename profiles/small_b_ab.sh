#!/bin/bash
# Small batches: streaming warps per private CTA x smallest chunk (profiles/ab.py)
for b in ${FANOUTS:-1 2 8}; do
  echo "B=$b"
  timeout 300 python profiles/ab.py --shape 6000,$b,256 --rounds 3 --steps 6 \
    --set PRIV_ACTIVE_WARPS=0,PRIV_MIN_CHUNK=2 --set PRIV_ACTIVE_WARPS=0,PRIV_MIN_CHUNK=4 \
    --set PRIV_ACTIVE_WARPS=5,PRIV_MIN_CHUNK=2 --set PRIV_ACTIVE_WARPS=5,PRIV_MIN_CHUNK=4 \
    --set PRIV_ACTIVE_WARPS=3,PRIV_MIN_CHUNK=2 2>&1 | tail -5
done
