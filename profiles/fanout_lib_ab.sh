#!/bin/bash
# Small fan-outs, two builds interleaved: profiles/fanout_sweep.py with
# FK_LIB_PATH = A (default .ab/libforkattn_old.so) and B (default the tree's
# build); prints fan-out, tokens/s, chained and isolated layer fractions.
A=${A:-.ab/libforkattn_old.so}
B=${B:-paper_2405_19888_b200/libforkattn.so}
for r in $(seq 1 ${ROUNDS:-2}); do
  for lib in $A $B; do
    echo "== round $r $lib"
    FK_LIB_PATH=$lib timeout 300 python profiles/fanout_sweep.py --fanouts ${FANOUTS:-1,2,8} --steps 6 2>&1 | \
      python -c "import sys,json; [print(d['fanout'], round(d['tokens_per_s']), round(d['frac'],3), round(d['frac_isolated'],3)) for d in (json.loads(l) for l in sys.stdin if l.startswith('{'))]"
  done
done
