#!/bin/bash
# r2 evidence on one B200: the default bench line, the ncu launch list of the same command (cold-cache,
# serialised; only after the plain run exited 0), and one ncu --set full capture of k_gain_culled.
tag=${1:-r2}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.txt 2>&1 || { echo "bench failed"; tail -5 gpurun_out/${tag}_bench.txt; exit 1; }
tail -1 gpurun_out/${tag}_bench.txt | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_launches.log 2>&1
echo "launches rc=$?"
if [ "${FULL:-1}" = "1" ]; then
  ncu --set full --import-source on --clock-control none --kernel-name regex:k_gain_culled --launch-skip 3 --launch-count 1 \
      -o gpurun_out/${tag}_gain -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/${tag}_ncu_full.log 2>&1
  echo "full rc=$?"
fi
