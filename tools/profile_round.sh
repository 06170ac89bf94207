#!/bin/bash
# usage: tools/profile_round.sh TAG -- the committed evidence for one round on one B200:
#   gpurun_out/TAG_bench.txt      bench.py (default outdoor run: JSON line with roofline, cpu_baseline, e2e)
#   gpurun_out/TAG_launches.csv   ncu launch list of the same command (gpu__time_duration, cold, serialised)
#   gpurun_out/TAG_gain.ncu-rep   ncu --set full of one k_gain_culled launch
# Each ncu pass runs only after the plain command exited 0.
tag=${1:?tag}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.txt 2>&1 || { echo "bench failed"; tail -5 gpurun_out/${tag}_bench.txt; exit 1; }
tail -1 gpurun_out/${tag}_bench.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_launches.log 2>&1
echo "launches rc=$?"
ncu --set full --import-source on --clock-control none --kernel-name regex:k_gain_culled --launch-skip 3 --launch-count 1 \
    -o gpurun_out/${tag}_gain -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_full.log 2>&1
echo "full rc=$?"
