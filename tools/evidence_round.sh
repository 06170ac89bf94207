set -x
FULL=0 bash tools/profile_r2.sh r2k
bash tools/bench_configs.sh r2k
timeout 900 python tools/shard_model.py --config scale --steps 10 > gpurun_out/r2k_shard_model_scale.jsonl 2> gpurun_out/r2k_shard.err; echo "shard rc=$?"
bash tools/multirank_check.sh > gpurun_out/r2k_multirank.txt 2>&1; tail -4 gpurun_out/r2k_multirank.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2k_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2k_smoke.txt
