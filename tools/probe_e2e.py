"""Diagnostic: where does the e2e sweep time go? (run on the GPU box)"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2402_03307_b200 import rgs, scenes  # noqa: E402

W, H = 1352, 1014
store = scenes.synthetic_scene(300_000, W, H, seed=2)
cams = scenes.sweep_cameras(W, H, 300)
ctx = rgs.Context(0)
scene = rgs.DeviceScene.from_store(ctx, store)
dev_imgs = torch.empty((300, H, W, 3), dtype=torch.float32, device="cuda")
ctx.render_views(scene, cams, out=dev_imgs)
torch.cuda.synchronize()
for label, n in (("device sweep 300", 300),):
    t = time.perf_counter()
    ctx.render_views(scene, cams[:n], out=dev_imgs[:n])
    torch.cuda.synchronize()
    print(label, "%.1f ms" % (1e3 * (time.perf_counter() - t)))
f32 = store.arrays_f32()
pinned = [torch.from_numpy(a).pin_memory() for a in f32]
host = torch.empty((300, H, W, 3), dtype=torch.float32, pin_memory=True)
host.zero_()  # touch pages
for rep in range(6):
    t = time.perf_counter()
    ctx.render_views_host([p.numpy() for p in pinned], 3, cams, (0, 0, 0), host.numpy())
    print("host sweep 300 rep", rep, "%.1f ms" % (1e3 * (time.perf_counter() - t)))
t = time.perf_counter()
host.copy_(dev_imgs, non_blocking=True)
torch.cuda.synchronize()
print("one bulk D2H of 4.9 GB: %.1f ms" % (1e3 * (time.perf_counter() - t)))
# copy-only bounds: the e2e ring's 300 per-view copies, on one stream and alternating over two
per = dev_imgs[0].numel()
for nstreams in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    for v in range(300):
        with torch.cuda.stream(streams[v % nstreams]):
            host[v].copy_(dev_imgs[v], non_blocking=True)
    torch.cuda.synchronize()
    print(f"300 per-view D2H copies on {nstreams} stream(s): %.1f ms" % (1e3 * (time.perf_counter() - t)))
# fixed vs per-view cost of the host path: t(n) for n = 8, 60, 150, 300 views (best of 3)
for n in (8, 60, 150, 300):
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        ctx.render_views_host([p.numpy() for p in pinned], 3, cams[:n], (0, 0, 0), host[:n].numpy())
        best = min(best, time.perf_counter() - t)
    bd = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ctx.render_views(scene, cams[:n], out=dev_imgs[:n])
        torch.cuda.synchronize()
        bd = min(bd, time.perf_counter() - t)
    print(f"n={n}: host path {1e3 * best:.1f} ms, device path {1e3 * bd:.1f} ms")
t = time.perf_counter()
sc2 = rgs.DeviceScene.from_store(ctx, store)
torch.cuda.synchronize()
print("scene upload (from_store): %.1f ms" % (1e3 * (time.perf_counter() - t)))
