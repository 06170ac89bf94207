#!/bin/bash
# k_col_culled waypoints per work item: the automatic choice (0) against fixed chunks (RTG_COL_CHUNK_RT),
# one bench line per config and choice, twice (usage on the box: bash tools/col_chunk_ab.sh [configs])
cfgs=${1:-"room multi_room outdoor scale"}
for rep in 1 2; do
for cfg in $cfgs; do
for ch in 0 10 5 3; do
  if [ "$ch" = "0" ]; then unset RTG_COL_CHUNK_RT; else export RTG_COL_CHUNK_RT=$ch; fi
  out=$(timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); print('$cfg', 'chunk=$ch', round(d['ms_per_step_median'],4), 'col', d['phase_ms']['collision'], 'best', d['best'], d['clocks']['sm_mhz'])" "$out"
done; done; done
unset RTG_COL_CHUNK_RT
