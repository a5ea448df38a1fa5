#!/bin/bash
mkdir -p gpurun_out/r2
RGS_BENCH_SHARE_GPU=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/r2/bench_share2.json 2> gpurun_out/r2/bench_share2.err
echo "rc=$?"
tail -3 gpurun_out/r2/bench_share2.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2/bench_share2.json").read().strip().splitlines()[-1])
print("n_gpus", d["n_gpus"], "FPS %.1f" % d["value"], "c4 %.1f" % d["c4"]["value"], "train %.1f" % d["train"]["value"],
      "c5 %.1f" % d["train_c5"]["value"], d["train"]["config"]["allreduce"])
PY
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 | cut -c1-300
