#!/bin/bash
# compute-sanitizer is closed on the GPU pool: the stand-in is a build with RTG_BOUNDS_CHECK (every table,
# queue, bitmap and record index of the culled gain kernel checked, __trap on violation), run through the
# parity tests and tools/sanitize.py; the normal build is restored afterwards.
set -o pipefail
python - <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2409_18122_b200 import build as B
B.build(force=True, extra=["-DRTG_BOUNDS_CHECK"])
PY
timeout 1200 python -m pytest tests -m gpu -q -x -k "${1:-tiny or room or fuzz or band or golden or degenerate or empty or include_start or sparse or axis}" 2>&1 | tail -3
timeout 600 python tools/sanitize.py 2>&1 | tail -2
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160
python paper_2409_18122_b200/build.py --force > /dev/null
