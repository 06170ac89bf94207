#!/bin/bash
# usage: tools/dense_ab.sh [lib.so ...] -- dense-mode outdoor step (collision, gain ms) per library build
for v in current "$@"; do
  [ "$v" != current ] && cp "$v" paper_2409_18122_b200/librtg.so
  echo "== $v"
  timeout 600 python bench.py --mode dense --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms']['collision'], d['phase_ms']['visibility_gain'], d['roofline']['frac'])"
done
