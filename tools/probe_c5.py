"""Diagnostic: per-stage times of one C5 training step (1M Gaussians, 8 views of 1352x1014)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_03307_b200 import rgs, scenes, train  # noqa: E402

dev = torch.device("cuda:0")
ctx = rgs.Context(0)
truth = scenes.synthetic_scene(bench.C5_N, bench.C5_W, bench.C5_H, seed=bench.C5_SEED)
store = scenes.perturbed(truth, bench.C5_SEED)
cams = [scenes.bench_camera(bench.C5_W, bench.C5_H, (v + 0.5) / bench.C5_VIEWS,
                            scenes.yaw_pose(-4.0 + 8.0 * v / (bench.C5_VIEWS - 1), (0.02, 0.0, 0.03)))
        for v in range(bench.C5_VIEWS)]
tsc = rgs.DeviceScene.from_store(ctx, truth)
targets = torch.empty((bench.C5_VIEWS, bench.C5_H, bench.C5_W, 3), dtype=torch.float32, device=dev)
ctx.render_views(tsc, cams, (0.0, 0.0, 0.0), out=targets)
tsc.close()
scene = rgs.DeviceScene.from_store(ctx, store)
tr = train.Trainer(ctx, scene, train.TrainConfig(batch=bench.C5_VIEWS, total_steps=bench.TRAIN_TOTAL_STEPS,
                                                 max_gaussians=2_000_000), None, start_step=bench.TRAIN_START_STEP)
tl = [targets[v] for v in range(bench.C5_VIEWS)]
if os.environ.get("C5_NO_OVERLAP") == "1":
    tr.overlap = False
for _ in range(3):
    tr.step(cams, tl)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    tr.step(cams, tl, read=False)
torch.cuda.synchronize()
print("step ms (pipelined): %.2f" % ((time.perf_counter() - t) / 5 * 1e3))
ctx.set_profiling(timing=True, count_evals=False)
ctx.profile_reset()
tr.step(cams, tl)
torch.cuda.synchronize()
stages, _ = ctx.profile_read()
ctx.set_profiling(False, False)
tot = sum(v[0] for v in stages.values())
print("serialised stage sum %.2f ms" % tot)
for k, (ms, n) in sorted(stages.items(), key=lambda kv: -kv[1][0]):
    if n:
        print(f"  {k:24s} {ms:7.3f} ms  ({n} launches)")
