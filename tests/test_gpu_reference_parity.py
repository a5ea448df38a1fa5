"""GPU parity straight against the reference's own sources (oracle/_ref: the reference's
rotor / gaussian / sh / rasterizer / image / ssim / loss / optim / knn / trainer sources
compiled in place), at the benchmarked configurations -- not through the C restatement.

* C1 (50K, 800x800, t = 0.5): both the identity pose the bench uses and a yawed, translated
  pose;
* C2 (300K, 1352x1014): 12 timestamps spread over the 300-timestamp sweep the headline
  benchmark renders, from the bench's own (identity) pose;
* C3 (200K, 800x800): the render backward, with the count of gradient coordinates outside
  the floored 1e-3 bar recorded;
* C5 (1M, 1352x1014, 8 views): one evaluate_loss of the bench's 8-view batch (trainer.cpp:22-84)
  against the reference's evaluate_loss on the same scene, targets and neighbour lists.

Bars (BASELINE.json north_star): splat records and tile lists / per-tile order bit-exact,
n_contrib identical, image within 1e-4; gradients within 1e-3 relative (floored at 1e-3 x the
column's max |gradient|, the reference's own gradient tests floor the same way,
test_render.cpp:139-141)."""
import numpy as np
import pytest

import oracle as O
from paper_2402_03307_b200 import rgs, scenes, train
from paper_2402_03307_b200.rgs import DeviceScene
from parity import floored_rel_err, splat_mismatch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref (reference build) not built")]

THREADS = 32


@pytest.fixture(scope="module")
def ref():
    return O.reference_build()


# column groups of the (N, 65) reference order: mean4, ls4, rotor8, opacity, sh 3x16 channel-major
GROUPS = {"mean": range(0, 4), "log_scales": range(4, 8), "rotor": range(8, 16), "opacity": range(16, 17),
          "sh_dc": [17, 33, 49], "sh_rest": [c for c in range(17, 65) if c not in (17, 33, 49)]}


def _report_columns(err, got, ref):
    """Per parameter group: coordinates above 1e-3, max error, and the error quantiles."""
    for name, cols in GROUPS.items():
        e = err[:, list(cols)]
        print(f"  {name:10s} above 1e-3: {int((e > 1e-3).sum()):7d} of {e.size:9d}  max {e.max():.3e}  "
              f"p99.99 {np.quantile(e, 0.9999):.3e}")


def _forward_vs_ref(ctx, ref, store, cam, tag):
    ref_img, rr = ref.render_forward(store, cam, (0.0, 0.0, 0.0), threads=THREADS, retain=True)
    out = rgs.render_forward(store, cam, rgs.RenderOptions(retain_records=True), ctx=ctx)
    rec = out.records
    mm = splat_mismatch(rec.splats, rr.splats)
    assert mm == {}, f"{tag}: splat records differ from the reference build: {mm}"
    assert np.array_equal(rec.tile_offsets, rr.tile_offsets), f"{tag}: tile list lengths differ"
    assert np.array_equal(rec.tile_ids, rr.tile_ids), f"{tag}: tile lists / order differ"
    ncd = int((rec.n_contrib != rr.n_contrib).sum())
    assert ncd == 0, f"{tag}: n_contrib differs at {ncd} pixels"
    err = float(np.abs(out.image.astype(np.float64) - ref_img).max())
    assert err <= 1e-4, f"{tag}: image error {err}"
    print(f"{tag}: {len(rr.splats)} splats, {len(rr.tile_ids)} pairs bit-exact, n_contrib identical, "
          f"max image err {err:.2e}, slow pixels {rec.n_slow_pixels}")
    return out, rr


def test_c1_both_poses_vs_reference_build(ctx, ref):
    store = scenes.synthetic_scene(50_000, 800, 800, seed=1)
    for name, pose in (("identity", None), ("yawed", scenes.yaw_pose(7.0, (0.05, -0.02, 0.1)))):
        _forward_vs_ref(ctx, ref, store, scenes.bench_camera(800, 800, 0.5, pose), f"C1 {name}")


def test_c2_sweep_vs_reference_build(ctx, ref):
    """12 of the headline sweep's 300 timestamps, from the bench's camera (bench.sweep_for_rank(0))."""
    store = scenes.synthetic_scene(300_000, 1352, 1014, seed=2)
    cams = scenes.sweep_cameras(1352, 1014, 300)
    for k in np.linspace(0, 299, 12).astype(int):
        _forward_vs_ref(ctx, ref, store, cams[k], f"C2 t[{k}]")


def test_c3_backward_vs_reference_build(ctx, ref):
    """C3 render backward: every coordinate's floored relative error is recorded; the bar is
    1e-3 and the test fails on any coordinate above it."""
    store = scenes.synthetic_scene(200_000, 800, 800, seed=3)
    cam = scenes.bench_camera(800, 800, 0.5, scenes.yaw_pose(7.0, (0.05, -0.02, 0.1)))
    dl = np.random.default_rng(3).uniform(-1, 1, (800, 800, 3))
    out = rgs.render_forward(store, cam, rgs.RenderOptions(retain_records=True), ctx=ctx)
    g = rgs.render_backward(store, cam, out.records, dl, ctx=ctx)
    _, rr = ref.render_forward(store, cam, (0.0, 0.0, 0.0), threads=THREADS, retain=True)
    gr, vn, vis = ref.render_backward(store, cam, rr, dl, threads=THREADS)
    assert np.array_equal(g.visible.astype(bool), vis.astype(bool))
    err = floored_rel_err(g.as_matrix(), gr)
    bad = np.argwhere(err > 1e-3)
    cols = sorted({int(c) for c in bad[:, 1]})
    _report_columns(err, g.as_matrix(), gr)
    print(f"C3 backward: {int(vis.sum())} visible, {err.size} coordinates, {len(bad)} above 1e-3 "
          f"(columns {cols}), max {err.max():.3e}")
    for i, c in bad[:20]:
        print(f"  gaussian {i} param {c}: got {g.as_matrix()[i, c]:.9e} ref {gr[i, c]:.9e} "
              f"col max {np.abs(gr[:, c]).max():.3e} err {err[i, c]:.3e}")
    vn_err = float(np.abs(g.viewspace_norm - vn).max() / max(np.abs(vn).max(), 1e-30))
    assert vn_err <= 1e-3, vn_err
    assert len(bad) == 0, f"{len(bad)} gradient coordinates above the 1e-3 bar (max {err.max():.3e})"


def test_c5_evaluate_loss_vs_reference_build(ctx, ref):
    """One evaluate_loss of the C5 bench batch: 1M Gaussians, 8 views of 1352x1014 (bench.py
    run_c5_leg's cameras, rank 0), L1 + SSIM + consistency, against the reference's evaluate_loss
    on the same float32 scene, targets and neighbour lists."""
    import torch

    T = O.train_ops("ref")
    n, w, h, views = 1_000_000, 1352, 1014, 8
    truth = scenes.synthetic_scene(n, w, h, seed=5)
    store = scenes.perturbed(truth, 5)
    cams = [scenes.bench_camera(w, h, (v + 0.5) / views,
                                scenes.yaw_pose(-4.0 + 8.0 * v / (views - 1), (0.02, 0.0, 0.03)))
            for v in range(views)]
    tsc = DeviceScene.from_store(ctx, truth)
    targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
    tsc.close()
    sc = DeviceScene.from_store(ctx, store)
    tr = train.Trainer(ctx, sc, train.TrainConfig(batch=views))
    tr.rebuild_knn()
    tr.evaluate_loss(cams, targets)
    torch.cuda.synchronize()
    wts = O.loss_weights(lambda_entropy=0.0)  # entropy is folded into the device Adam step
    L, gref, vn, vis = T.evaluate_loss(store, cams, [t.cpu().numpy().astype(np.float64) for t in targets], wts,
                                       nbrs=tr.nbrs.cpu().numpy(), threads=THREADS)
    got = tr.losses.cpu().numpy()
    assert abs(got[0] - L[0]) <= 1e-5 * L[0], (got[0], L[0])  # L1 of the float images vs double
    assert abs(got[1] - L[1]) <= 1e-5 * max(L[1], 1e-3), (got[1], L[1])
    assert abs(got[4] - L[3]) <= 1e-9 * L[3], (got[4], L[3])
    mean, ls, rot, op, sh = rgs.grads_from_soa(tr.grads.cpu().numpy(), n)
    gg = np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1)
    err = floored_rel_err(gg, gref)
    frac = float(np.mean(err <= 1e-3))
    print(f"C5 evaluate_loss: l1 {got[0]:.9f} / {L[0]:.9f}, ssim {got[1]:.9f} / {L[1]:.9f}, consistency "
          f"{got[4]:.6e} / {L[3]:.6e}; gradients within 1e-3: {100 * frac:.5f}% "
          f"({int((err > 1e-3).sum())} of {err.size}), max {err.max():.3e}")
    _report_columns(err, gg, gref)
    assert np.array_equal(tr.visible.cpu().numpy() > 0, vis.astype(bool))
    assert np.allclose(tr.vnorm.cpu().numpy(), vn, rtol=1e-3, atol=1e-3 * vn.max())

    # The two sources of difference, isolated: (i) L1's sign(rendered - target) where the float
    # image and the reference's double image straddle the target (counted; the device decides
    # those pixels on their FP64 value, rgs_image_loss_ex); (ii) the render backward alone, fed
    # the device's own dL/dimage on both sides.
    flips = 0
    gsum = np.zeros_like(gref)
    tr0 = train.Trainer(ctx, sc, train.TrainConfig(batch=views))
    tr0.evaluate_loss(cams, targets)  # no KNN built: no consistency term
    torch.cuda.synchronize()
    inv_b = 1.0 / views
    for cam, tgt in zip(cams, targets):
        img, rec = ctx.render_forward_device(sc, cam, retain=True)
        dl = torch.zeros_like(img)
        train.image_loss(ctx, img, tgt, 0.8 * inv_b, 0.2 * inv_b, dl, records=rec)  # as evaluate_loss does
        torch.cuda.synchronize()
        rec.close()
        ref_img, rr = ref.render_forward(store, cam, (0.0, 0.0, 0.0), threads=THREADS, retain=True)
        t64 = tgt.cpu().numpy().astype(np.float64)
        flips += int((np.sign(img.cpu().numpy().astype(np.float64) - t64) != np.sign(ref_img - t64)).sum())
        g1, _, _ = ref.render_backward(store, cam, rr, dl.cpu().numpy().astype(np.float64), threads=THREADS)
        gsum += g1
    mean, ls, rot, op, sh = rgs.grads_from_soa(tr0.grads.cpu().numpy(), n)
    gg0 = np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1)
    err0 = floored_rel_err(gg0, gsum)
    print(f"C5: L1 sign flips between the float and double images: {flips}; render backward alone (same "
          f"dL/dimage): {int((err0 > 1e-3).sum())} of {err0.size} above 1e-3, max {err0.max():.3e}")
    _report_columns(err0, gg0, gsum)
    assert (err0 > 1e-3).sum() == 0
    assert frac >= 0.9999


CACHE_FIELDS = {"p_cam": (0, 3), "T": (3, 9), "cov2": (9, 13), "dir": (13, 16), "view_dist": (16, 17),
                "basis": (17, 33), "basis_grad": (33, 81), "clamped": (81, 84), "opacity": (84, 85)}


def test_project_cache_vs_reference_build(ctx, ref):
    """project() with its ProjectCache (rasterizer.cpp:215-276; the drop-in adapter's project()
    returns these fields) on 400 random sliced Gaussians, every SH degree, against the reference
    build: the same culls, the splat record and every cache field bit for bit."""
    rng = np.random.default_rng(11)
    cam = scenes.bench_camera(640, 480, 0.5, scenes.yaw_pose(6.0, (0.03, -0.02, 0.05)))
    n_same = n_kept = 0
    for k in range(400):
        a = rng.normal(0, 0.15, (3, 3))
        cov = a @ a.T + np.eye(3) * rng.uniform(1e-4, 1e-2)
        mean = np.array([rng.uniform(-2, 2), rng.uniform(-1.5, 1.5), rng.uniform(-1, 6)])
        sliced = np.concatenate([mean, cov.reshape(-1), [rng.uniform(0.05, 1.0)], rng.normal(0, 0.3, 3)])
        sh = rng.normal(0, 0.4, 48)
        deg, op = k % 4, rng.normal(1.0, 2.0)
        got, gc = rgs.project(sliced, cam, sh, deg, op, ctx=ctx, want_cache=True)
        want, wc = ref.project_cache(sliced, cam, sh, deg, op)
        assert (got is None) == (want is None), k
        if want is None:
            continue
        n_kept += 1
        for f in ("mean2", "conic", "depth", "color", "alpha_base", "flow2", "radius"):
            assert np.array_equal(np.asarray(got[f]), np.asarray(want[f])), (k, f)
        for name, (lo, hi) in CACHE_FIELDS.items():
            assert np.array_equal(gc[lo:hi], wc[lo:hi]), (k, name, gc[lo:hi], wc[lo:hi])
        n_same += 1
    assert n_kept > 100
    print(f"project(): {n_kept} of 400 survive the culls, splat and ProjectCache bit-exact for all")
