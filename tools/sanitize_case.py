"""A small end-to-end case for compute-sanitizer (tests/test_gpu_sanitizer.py): the forward
(K1, depth ranks, the tile-major scatter binning, K5, FP64 fix-up), a forced-FP64
forward, the backward (K6, FP64 fix-up, K7a/K7b), the deterministic backward, a batched
render sweep over the 8 view slots (depth ranks, scan, duplicate, radix passes, ranges), and one training step (K8, K9, K10, K11)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2402_03307_b200 import rgs, scenes, train  # noqa: E402


def main():
    import torch

    ctx = rgs.Context(0)
    store = scenes.synthetic_scene(3000, 128, 96, seed=7)
    cam = scenes.bench_camera(128, 96, 0.5, scenes.yaw_pose(5.0, (0.02, 0.0, 0.05)))
    out = rgs.render_forward(store, cam, rgs.RenderOptions(background=(0.1, 0.2, 0.3), retain_records=True), ctx=ctx)
    _ = out.records.tile_ids, out.records.splats, out.records.n_contrib
    dl = np.random.default_rng(0).uniform(-1, 1, (cam.height, cam.width, 3))
    rgs.render_backward(store, cam, out.records, dl, ctx=ctx)
    out64 = rgs.render_forward(store, cam, rgs.RenderOptions(retain_records=True, blend_fp64=True), ctx=ctx)
    rgs.render_backward(store, cam, out64.records, dl, ctx=ctx)
    scene = rgs.DeviceScene.from_store(ctx, store)
    cams = scenes.sweep_cameras(128, 96, 12)
    imgs = torch.empty((12, 96, 128, 3), dtype=torch.float32, device="cuda")
    ctx.render_views(scene, cams, (0.0, 0.0, 0.0), out=imgs)
    _, rec = ctx.render_forward_device(scene, cam, retain=True)
    dld = torch.from_numpy(dl.astype(np.float32)).cuda()
    ctx.render_backward_device(scene, cam, rec, dld, deterministic=True)
    rec.close()
    truth = store.copy()
    store.mean[:, :3] += np.random.default_rng(1).normal(0, 0.01, (store.size(), 3)).astype(np.float32)
    tsc = rgs.DeviceScene.from_store(ctx, truth)
    tcams = [scenes.bench_camera(128, 96, 0.3 + 0.2 * k, scenes.yaw_pose(3.0 * k)) for k in range(3)]
    targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in tcams]
    sc = rgs.DeviceScene.from_store(ctx, store)
    tr = train.Trainer(ctx, sc, train.TrainConfig(), start_step=3000)
    for _ in range(3):
        tr.step(tcams, targets)
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
