"""Diagnostic: where does the training e2e gap come from? (run on the box)"""
import sys
import time

import numpy as np
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
B, N = bench.TRAIN_BATCH, 30
views = lambda k: [(k * B + j) % bench.TRAIN_VIEWS for j in range(B)]  # noqa: E731
for k in range(3):
    tr.step([cams[i] for i in views(k)], [targets[i] for i in views(k)])
tr.rebuild_knn()
torch.cuda.synchronize()


def run(label, staged, popped):
    host = targets.cpu().pin_memory()
    st = train.TargetStager(dev, B, bench.TRAIN_H, bench.TRAIN_W)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if staged:
        st.put([host[i] for i in views(0)])
    for k in range(N):
        if staged:
            tg = st.take()
            if k + 1 < N:
                st.put([host[i] for i in views(k + 1)])
        else:
            tg = [targets[i] for i in views(k)]
        tr.step([cams[i] for i in views(k)], tg, read=False)
        if staged:
            st.release(ctx)
        if popped and k > 0:
            tr.pop_losses()
    if popped:
        tr.pop_losses()
    torch.cuda.synchronize()
    print(f"{label}: {N / (time.perf_counter() - t0):.1f} it/s", flush=True)
    tr._pending.clear()


run("device targets, no reads   ", False, False)
run("device targets, pop reads  ", False, True)
run("staged H2D,     no reads   ", True, False)
run("staged H2D,     pop reads  ", True, True)
