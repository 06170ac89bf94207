#!/bin/bash
# usage: tools/lib_ab.sh a.so b.so [...] -- outdoor bench per library build, interleaved twice
# (ms/step, median, per-phase ms, e2e ms); CONFIG / MODE env select the workload
for rep in 1 2; do
  for v in "$@"; do
    cp "$v" paper_2409_18122_b200/librtg.so
    out=$(timeout 600 python bench.py --config ${CONFIG:-outdoor} --mode ${MODE:-culled} --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline ${EXTRA:-} 2>&1 | tail -1)
    python - "$v" "$out" <<'PY'
import json, sys
v, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
except Exception:
    print(v, "FAILED", line[-300:]); sys.exit()
e = d.get("e2e") or {}
print(f"{v}: {d['ms_per_step']:.3f} ms (median {d.get('ms_per_step_median', 0):.3f})  phases "
      + " ".join(f"{k}={x:.3f}" for k, x in d["phase_ms"].items()) + f"  e2e {e.get('ms_per_step', 0):.3f}")
PY
  done
done
