"""Diagnostic 2: which Gaussians carry the C5 backward outliers (FP64 forward + FP64 replay vs
the reference build), and do they persist with U(-1,1) dL/dimage / the unperturbed scene?"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from parity import floored_rel_err  # noqa: E402

from paper_2402_03307_b200 import rgs, scenes, train  # noqa: E402


def run(ctx, ref, store, truth, cam, dl_kind, tag):
    import torch

    n = store.size()
    sc = rgs.DeviceScene.from_store(ctx, store)
    tsc = rgs.DeviceScene.from_store(ctx, truth)
    tgt = ctx.render_forward_device(tsc, cam, retain=False)[0].clone()
    img, rec = ctx.render_forward_device(sc, cam, retain=True, blend_fp64=True)
    if dl_kind == "loss":
        dl = torch.zeros_like(img)
        train.image_loss(ctx, img, tgt, 0.8 / 8, 0.2 / 8, dl)
    else:
        dl = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, tuple(img.shape)).astype(np.float32)).cuda()
    torch.cuda.synchronize()
    dln = dl.cpu().numpy().astype(np.float64)
    _, rr = ref.render_forward(store, cam, (0.0, 0.0, 0.0), threads=32, retain=True)
    gr, vn, vis = ref.render_backward(store, cam, rr, dln, threads=32)
    g, _, _ = ctx.render_backward_device(sc, cam, rec, dl, deterministic=True)
    torch.cuda.synchronize()
    mean, ls, rot, op, sh = rgs.grads_from_soa(g.cpu().numpy(), n)
    gg = np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1)
    err = floored_rel_err(gg, gr)
    bad_g = np.unique(np.argwhere(err > 1e-3)[:, 0])
    print(f"{tag}: {int((err > 1e-3).sum())} coords above 1e-3 in {len(bad_g)} Gaussians, max {err.max():.3e}",
          flush=True)
    sp = rr.splats
    src = sp["source_index"]
    pos = {int(s): k for k, s in enumerate(src)}
    for i in bad_g[:12]:
        k = pos.get(int(i))
        cols = np.where(err[i] > 1e-3)[0].tolist()
        if k is None:
            print(f"   gaussian {i}: not a splat; bad params {cols}")
            continue
        s = sp[k]
        print(f"   gaussian {i}: mean2 {s['mean2']} r {s['radius']:.2f} color {s['color']} ab {s['alpha_base']:.3f} "
              f"depth {s['depth']:.3f} bad params {cols[:10]} max err {err[i].max():.2e}")
    sc.close()
    tsc.close()
    rec.close()


def main():
    ctx = rgs.Context(0)
    ref = O.reference_build()
    n, w, h = 1_000_000, 1352, 1014
    truth = scenes.synthetic_scene(n, w, h, seed=5)
    store = scenes.perturbed(truth, 5)
    cam = scenes.bench_camera(w, h, 0.5 / 8, scenes.yaw_pose(-4.0, (0.02, 0.0, 0.03)))
    run(ctx, ref, store, truth, cam, "loss", "perturbed scene, loss dL")
    run(ctx, ref, store, truth, cam, "uniform", "perturbed scene, U(-1,1) dL")
    run(ctx, ref, truth, truth, cam, "uniform", "unperturbed scene, U(-1,1) dL")


if __name__ == "__main__":
    main()
