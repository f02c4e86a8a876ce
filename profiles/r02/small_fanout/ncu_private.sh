#!/bin/bash
# ncu --set full of one private-kernel launch: single-row stream (B=1) vs row groups (B=4)
cd "$(dirname "$0")/../../.."
O=gpurun_out/sfn; mkdir -p $O
for b in 1 4; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:fk_private -s 100 -c 1 \
    -o $O/priv_b$b -f python profiles/small_fanout.py --b $b > $O/priv_b$b.log 2>&1
  ncu -i $O/priv_b$b.ncu-rep --page raw --csv > $O/priv_b${b}_raw.csv 2>/dev/null
  ncu -i $O/priv_b$b.ncu-rep --page details --csv > $O/priv_b${b}_details.csv 2>/dev/null
done
ls -la $O
