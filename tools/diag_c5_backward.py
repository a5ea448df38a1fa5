"""Diagnostic: where do the C5 render-backward outliers come from?  One C5 view (1M Gaussians,
1352x1014) with the L1 + SSIM dL/dimage of the training step; the device backward in the
production mode and in the deterministic FP64 replay, each against the reference build's
render_backward on the same dL/dimage."""
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


def main():
    import torch

    ctx = rgs.Context(0)
    ref = O.reference_build()
    n, w, h = 1_000_000, 1352, 1014
    truth = scenes.synthetic_scene(n, w, h, seed=5)
    store = scenes.perturbed(truth, 5)
    views = int(os.environ.get("VIEWS", "2"))
    cams = [scenes.bench_camera(w, h, (v + 0.5) / 8, scenes.yaw_pose(-4.0 + 8.0 * v / 7, (0.02, 0.0, 0.03)))
            for v in range(views)]
    tsc = rgs.DeviceScene.from_store(ctx, truth)
    sc = rgs.DeviceScene.from_store(ctx, store)
    for v, cam in enumerate(cams):
        tgt = ctx.render_forward_device(tsc, cam, retain=False)[0].clone()
        img, rec = ctx.render_forward_device(sc, cam, retain=True)
        dl = torch.zeros_like(img)
        train.image_loss(ctx, img, tgt, 0.8 / 8, 0.2 / 8, dl)
        torch.cuda.synchronize()
        dln = dl.cpu().numpy().astype(np.float64)
        ref_img, rr = ref.render_forward(store, cam, (0.0, 0.0, 0.0), threads=32, retain=True)
        gr, vn, vis = ref.render_backward(store, cam, rr, dln, threads=32)
        for det in (False, True):
            g, _, _ = ctx.render_backward_device(sc, cam, rec, dl, deterministic=det)
            torch.cuda.synchronize()
            mean, ls, rot, op, sh = rgs.grads_from_soa(g.cpu().numpy(), n)
            gg = np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1)
            err = floored_rel_err(gg, gr)
            bad = np.argwhere(err > 1e-3)
            print(f"view {v} {'deterministic FP64' if det else 'production'}: {len(bad)} of {err.size} above 1e-3, "
                  f"max {err.max():.3e}, p99.999 {np.quantile(err, 0.99999):.3e}", flush=True)
            if not det and len(bad):
                i, c = bad[np.argmax(err[bad[:, 0], bad[:, 1]])]
                col = np.abs(gr[:, c]).max()
                print(f"   worst: gaussian {i} param {c}: got {gg[i, c]:.6e} ref {gr[i, c]:.6e} colmax {col:.3e}")
                print(f"   |dl| mean {np.abs(dln).mean():.3e} max {np.abs(dln).max():.3e}; slow px {rec.n_slow_pixels}")
        rec.close()
        # the reference-KAT precision mode: FP64 forward blend (exact final_T) + FP64 replay
        img64, rec64 = ctx.render_forward_device(sc, cam, retain=True, blend_fp64=True)
        g, _, _ = ctx.render_backward_device(sc, cam, rec64, dl, deterministic=True)
        torch.cuda.synchronize()
        mean, ls, rot, op, sh = rgs.grads_from_soa(g.cpu().numpy(), n)
        gg = np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1)
        err = floored_rel_err(gg, gr)
        print(f"view {v} FP64 forward + FP64 replay: {int((err > 1e-3).sum())} of {err.size} above 1e-3, "
              f"max {err.max():.3e}", flush=True)
        rec64.close()


if __name__ == "__main__":
    main()
