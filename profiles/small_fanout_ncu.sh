#!/bin/bash
# ncu launch lists of one step at small fan-outs (profiles/small_fanout.py); output to stdout
make -s -C paper_2405_19888_b200/csrc >/dev/null; mkdir -p gpurun_out/sf
for spec in ${SPECS:-"1:" "2:" "2:GROUP_FANOUT=0" "8:" "64:"}; do
  b=${spec%%:*}; o=${spec#*:}
  echo "== B=$b opts=$o"
  timeout 300 ncu --metrics gpu__time_duration.sum -k regex:fk_ -s ${SKIP:-150} -c 12 --csv python profiles/small_fanout.py --b $b --set "$o" 2>/dev/null | grep -E 'fk_|plan:' | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | cut -c1-120
done
