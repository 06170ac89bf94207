#!/bin/bash
# one gpurun call: GPU parity tests (optionally filtered) + a short outdoor bench line
# usage (on the box): bash tools/gpu_check.sh [pytest -k expr] [bench extra args]
set -o pipefail
mkdir -p gpurun_out
K=${1:-""}
shift || true
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "$K" 2>&1 | tail -6
else
  timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
fi
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("ms/step %.3f median %.3f | phases %s | gain kernel %.3f ms frac %.3f | work %s | clocks %s" % (
    d["ms_per_step"], d["ms_per_step_median"], d["phase_ms"], r["kernel_ms"], r["frac"],
    {k: round(v, 1) for k, v in (r.get("work_per_waypoint") or {}).items()}, d["clocks"]))
PY
