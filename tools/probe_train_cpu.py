"""Diagnostic: CPU enqueue time of Trainer.step (read=False) vs its GPU time (run on the box)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2402_03307_b200 import rgs, train  # noqa: E402

dev = torch.device("cuda:0")
ctx = rgs.Context(0)
truth, store = bench.train_case()
cams = bench.train_views(0)
tsc = rgs.DeviceScene.from_store(ctx, truth)
targets = torch.empty((bench.TRAIN_VIEWS, bench.TRAIN_H, bench.TRAIN_W, 3), dtype=torch.float32, device=dev)
ctx.render_views(tsc, cams, (0.0, 0.0, 0.0), out=targets)
scene = rgs.DeviceScene.from_store(ctx, store)
tr = train.Trainer(ctx, scene, train.TrainConfig(batch=bench.TRAIN_BATCH, total_steps=2000))
B = bench.TRAIN_BATCH


def batch(k):
    idx = [(k * B + j) % bench.TRAIN_VIEWS for j in range(B)]
    return [cams[i] for i in idx], [targets[i] for i in idx]


for k in range(3):
    tr.step(*batch(k))
tr.rebuild_knn()
torch.cuda.synchronize()
cpu = []
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record()
t0 = time.perf_counter()
for k in range(20):
    t1 = time.perf_counter()
    tr.step(*batch(k), read=False)
    cpu.append(time.perf_counter() - t1)
b.record()
t_enq = time.perf_counter() - t0
torch.cuda.synchronize()
print("enqueue ms/step: median %.3f max %.3f; total enqueue %.1f ms; GPU %.1f ms for 20 steps"
      % (1e3 * sorted(cpu)[10], 1e3 * max(cpu), 1e3 * t_enq, a.elapsed_time(b)))

# Per-call CPU time inside Trainer.step (no synchronisation added): which call blocks?
import collections  # noqa: E402

acc = collections.defaultdict(float)


def wrap(obj, name):
    f = getattr(obj, name)

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        acc[name] += time.perf_counter() - t
        return r

    setattr(obj, name, g)


for nm in ("render_forward_device", "render_backward_device", "fence", "sync_stream"):
    wrap(ctx, nm)
wrap(train, "image_loss")
wrap(train, "consistency")
wrap(tr.opt, "step")
wrap(tr.opt, "status_async")
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(20):
    tr.step(*batch(k), read=False)
tot = time.perf_counter() - t0
torch.cuda.synchronize()
print("per step ms:", {k: round(1e3 * v / 20, 3) for k, v in acc.items()}, "total", round(1e3 * tot / 20, 3))
