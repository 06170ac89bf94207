#!/bin/bash
# DRAM bytes and duration of every map-build launch of one bench step (usage on the box:
# bash tools/ncu_mapbuild.sh TAG CONFIG); launches of the gain / collision kernels are skipped
tag=${1:?tag}; cfg=${2:-outdoor}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    --clock-control none --kernel-name regex:'^(?!k_gain_culled|k_col_culled|k_gain_dense|k_col_dense).*' \
    --launch-skip ${SKIP:-0} -c ${COUNT:-60} --csv --log-file gpurun_out/${tag}_mapbuild.csv \
    python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_mapbuild.log 2>&1
echo "ncu rc=$?"
