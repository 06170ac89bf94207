#!/bin/bash
# usage: tools/sweep.sh "hy,hx,hz" ... -- quick bench sweep over visibility-grid cell sizes (outdoor)
for c in "$@"; do
  out=$(timeout 300 python bench.py --config ${CONFIG:-outdoor} --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --cells "$c" 2>&1 | tail -1)
  python - "$c" "$out" <<'PY'
import json, sys
c, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
except Exception:
    print(c, "FAILED", line[-300:]); sys.exit()
w = d["roofline"].get("work_per_waypoint") or {}
print(f"cells {c}: {d['ms_per_step']:.3f} ms/step  gain {d['phase_ms']['visibility_gain']:.3f}  map {d['phase_ms']['map_build']:.3f}  "
      f"tested {w.get('tested',0):.0f} flank {w.get('tested_flank',0):.0f} units {w.get('units',0):.0f} agg {w.get('cells_aggregated',0):.0f}")
PY
done
