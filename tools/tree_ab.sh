#!/bin/bash
# usage: tools/tree_ab.sh a.so b.so [...] -- N3 rows of tools/bench_planner.py per library build, twice
for rep in 1 2; do
  for v in "$@"; do
    cp "$v" paper_2409_18122_b200/librtg.so
    echo "== $v"
    timeout 600 python tools/bench_planner.py --sizes ${SIZES:-1e6,5e6} --reps 10 2>&1 | grep '"N3' | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); print(f\"  {d['row'][:24]:24s} N={d['N']:>8} {d['ms']:.3f} ms\")"
  done
done
