#!/bin/bash
# Small fan-outs, two builds interleaved: profiles/fanout_sweep.py with
# FK_LIB_PATH = A (.ab/libforkattn_old.so) and B (the tree's build).
for r in 1 2; do
  for lib in .ab/libforkattn_old.so paper_2405_19888_b200/libforkattn.so; do
    echo "== round $r $lib"
    FK_LIB_PATH=$lib timeout 300 python profiles/fanout_sweep.py --fanouts ${FANOUTS:-1,2,8} --steps 6 2>&1 | \
      python -c "import sys,json; [print(d['fanout'], round(d['frac'],3), round(d['frac_isolated'],3)) for d in (json.loads(l) for l in sys.stdin if l.startswith('{'))]"
  done
done
