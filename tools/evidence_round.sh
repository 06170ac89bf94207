#!/bin/bash
# The round's committed evidence on one B200 (usage on the box: bash tools/evidence_round.sh TAG):
# the default bench line + its ncu launch list, one bench line per config, the 8-rank per-rank model
# (standard path and CUDA-graph cycle), the 2-rank gloo run of the N > 1 bench path, and smoke().
tag=${1:-r2}
set -x
FULL=0 bash tools/profile_r2.sh $tag
bash tools/bench_configs.sh $tag
timeout 900 python tools/shard_model.py --config scale --steps 10 > gpurun_out/${tag}_shard_model_scale.jsonl 2> gpurun_out/${tag}_shard.err; echo "shard rc=$?"
timeout 900 python tools/shard_model.py --config scale --steps 10 --graph > gpurun_out/${tag}_shard_model_scale_graph.jsonl 2> gpurun_out/${tag}_shard_graph.err; echo "shard graph rc=$?"
bash tools/multirank_check.sh > gpurun_out/${tag}_multirank.txt 2>&1; tail -4 gpurun_out/${tag}_multirank.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${tag}_smoke.txt
