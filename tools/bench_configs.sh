#!/bin/bash
# one bench line per BASELINE.json config on one B200 (the outdoor line is the headline; the others are the
# per-config records SURVEY §8(d) asks for).  usage (on the box): bash tools/bench_configs.sh TAG
tag=${1:-r2}
mkdir -p gpurun_out
for cfg in tiny room multi_room outdoor scale; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/${tag}_bench_${cfg}.json 2> gpurun_out/${tag}_bench_${cfg}.err
  echo "$cfg rc=$?"; tail -1 gpurun_out/${tag}_bench_${cfg}.json | cut -c1-300
done
