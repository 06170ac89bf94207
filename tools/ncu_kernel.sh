#!/bin/bash
# usage (on the box): tools/ncu_kernel.sh TAG [kernel-regex] [bench args...]
# one `ncu --set full` capture of one launch of the kernel (default k_gain_culled) inside the bench
tag=${1:?tag}; kern=${2:-k_gain_culled}; shift 2 || shift $#
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --kernel-name regex:$kern --launch-skip ${SKIP:-3} --launch-count 1 \
    -o gpurun_out/${tag} -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
    > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${tag}_ncu.log
