#!/bin/bash
# The N > 1 bench path executed on ONE GPU: two ranks over gloo share cuda:0 (sharding, barrier,
# max-over-ranks timing, the (score, index) all_gather).  Strong scaling keeps the global K of the
# 1-rank run, so both must report the same global best.  Output: gpurun_out/multirank_*.json
mkdir -p gpurun_out
args="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py --gpus 1 $args "$@" > gpurun_out/multirank_n1.json 2> gpurun_out/multirank_n1.err
echo "n1 rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --backend gloo --scaling strong $args "$@" > gpurun_out/multirank_n2_strong.json 2> gpurun_out/multirank_n2_strong.err
echo "n2 strong rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 2 --backend gloo --scaling weak $args "$@" > gpurun_out/multirank_n2_weak.json 2> gpurun_out/multirank_n2_weak.err
echo "n2 weak rc=$?"
python - <<'PY'
import json
for f in ("n1", "n2_strong", "n2_weak"):
    try:
        d = json.loads(open(f"gpurun_out/multirank_{f}.json").read().strip().splitlines()[-1])
        print(f, "n_gpus", d["n_gpus"], "K", d["config"]["K"], "K/gpu", d["config"]["K_per_gpu"], "best", d["best"],
              "ms/step %.3f" % d["ms_per_step"], d["scaling"])
    except Exception as e:
        print(f, "failed", e)
PY
