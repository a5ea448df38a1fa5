"""GPU parity of the training side through the C ABI against the CPU
oracle (oracle/rgs_oracle.c, pinned bit-exact to the reference's own training sources by
tests/test_oracle_train.py).

Bars: the image gradient (L1 + SSIM, FP64 in the reference order) is bit-identical to
float(reference) on the same rendered image; Adam on FP64 scenes is bit-identical, on FP32
scenes equal to the reference step rounded to float; KNN lists are identical; loss scalars
within 1e-12 relative (fixed-order tree sums); the entropy term within 1e-12 (libm log);
the consistency and full evaluate_loss gradients within relative 1e-3 (floored at
1e-3 * max |column|, as the render backward)."""
import numpy as np
import pytest

import oracle as O
from paper_2402_03307_b200 import rgs, scenes, train
from paper_2402_03307_b200.rgs import DeviceScene

from parity import floored_rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    return O.train_ops("orc")


def _t(a, dtype=None):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).cuda()


@pytest.mark.parametrize("shape", [(37, 45), (200, 160), (800, 800)])
def test_image_loss_bit_exact(ctx, T, shape):
    import torch

    h, w = shape
    r = np.random.default_rng(h)
    a = r.uniform(0, 1, (h, w, 3)).astype(np.float32)
    b = np.clip(a + r.normal(0, 0.1, a.shape), 0, 1).astype(np.float32)
    b[5, 7] = a[5, 7]
    wl1, wss = 0.8 / 3, 0.2 / 3
    dl = torch.zeros((h, w, 3), dtype=torch.float32, device="cuda")
    losses = torch.zeros(4, dtype=torch.float64, device="cuda")
    train.image_loss(ctx, _t(a), _t(b), wl1, wss, dl, losses, loss_scale=1.0)
    torch.cuda.synchronize()
    l1, g1 = T.l1_loss(a.astype(np.float64), b.astype(np.float64))
    ss, gs = T.ssim_loss(a.astype(np.float64), b.astype(np.float64))
    ref = (wl1 * g1 + wss * gs).astype(np.float32)
    got = dl.cpu().numpy()
    assert np.array_equal(got, ref), f"{np.count_nonzero(got != ref)} of {got.size} differ"
    L = losses.cpu().numpy()
    assert abs(L[0] - l1) <= 1e-12 * abs(l1)
    assert abs(L[1] - ss) <= 1e-12 * max(abs(ss), 1e-3)
    mse = float(np.mean((a.astype(np.float64) - b) ** 2))
    assert abs(L[2] - mse) <= 1e-12 * mse
    # losses only (no gradient buffer) and accumulation
    train.image_loss(ctx, _t(a), _t(b), losses=losses, loss_scale=0.5, accumulate=True)
    torch.cuda.synchronize()
    assert abs(losses.cpu().numpy()[0] - 1.5 * l1) <= 1e-12 * l1


def test_l1_ties_decided_in_fp64(ctx, orc, T):
    """rgs_image_loss_ex: with the target equal to the FP32 render every pixel is a tie for the
    FP32 image (sign 0), while the reference's double image decides sign(img64 - target)
    (image.cpp:32-33).  With the records the device takes those signs from its FP64 recompute:
    dL/dimage equals float(l1_loss_backward(reference double image, target)) bit for bit."""
    import torch

    store = scenes.synthetic_scene(3000, 96, 72, seed=17)
    cam = scenes.bench_camera(96, 72, 0.4, scenes.yaw_pose(3.0, (0.02, 0.0, 0.04)))
    sc = DeviceScene.from_store(ctx, store)
    img, rec = ctx.render_forward_device(sc, cam, retain=True)
    tgt = img.clone()
    dl = torch.zeros_like(img)
    train.image_loss(ctx, img, tgt, 1.0, 0.0, dl, records=rec)
    dl_plain = torch.zeros_like(img)
    train.image_loss(ctx, img, tgt, 1.0, 0.0, dl_plain)
    torch.cuda.synchronize()
    ref_img, _ = orc.render_forward(store, cam, (0.0, 0.0, 0.0), threads=8)
    _, g1 = T.l1_loss(ref_img, tgt.cpu().numpy().astype(np.float64))
    got = dl.cpu().numpy()
    assert np.count_nonzero(dl_plain.cpu().numpy()) == 0  # every FP32 difference is exactly 0
    assert np.count_nonzero(g1) > 0.5 * g1.size  # ... the double image's mostly are not
    assert np.array_equal(got, g1.astype(np.float32)), f"{np.count_nonzero(got != g1.astype(np.float32))} differ"
    rec.close()


@pytest.mark.parametrize("steps", [3])
def test_reproducible_training_steps(ctx, steps):
    """Trainer.reproducible (RGS_FLAG_REPRODUCIBLE backward: fixed-point screen-gradient sums;
    integer-count consistency gradient): two runs of the same steps from the same start give
    bitwise identical scenes and losses; the result stays within the atomic path's tolerance."""
    import torch

    store, truth, cams = _training_case(n=6000, views=3, w=160, h=120)
    tsc = DeviceScene.from_store(ctx, truth)
    targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
    runs = []
    for reproducible in (True, True, False):
        sc = DeviceScene.from_store(ctx, store)
        tr = train.Trainer(ctx, sc, train.TrainConfig(), start_step=3000)
        tr.reproducible = reproducible
        losses = [tr.step(cams, targets).total for _ in range(steps)]
        torch.cuda.synchronize()
        runs.append((sc.download(), losses))
    (s1, l1), (s2, l2), (s3, l3) = runs
    assert l1 == l2
    for a, b in zip(s1, s2):
        assert np.array_equal(a, b)
    for a, b in zip(s1, s3):
        assert np.allclose(a, b, rtol=1e-4, atol=1e-6)


def test_reproducible_backward_matches_atomic(ctx, orc):
    """RGS_FLAG_REPRODUCIBLE against the oracle: the same floored 1e-3 bar as the atomic path,
    and repeat calls bitwise identical."""
    import torch

    store = scenes.synthetic_scene(20000, 320, 240, seed=6)
    cam = scenes.bench_camera(320, 240, 0.5, scenes.yaw_pose(5.0, (0.02, 0.0, 0.04)))
    sc = DeviceScene.from_store(ctx, store)
    _, rec = ctx.render_forward_device(sc, cam, retain=True)
    dl = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, (240, 320, 3)).astype(np.float32)).cuda()
    a = ctx.render_backward_device(sc, cam, rec, dl, reproducible=True)[0].cpu().numpy()
    b = ctx.render_backward_device(sc, cam, rec, dl, reproducible=True)[0].cpu().numpy()
    c = ctx.render_backward_device(sc, cam, rec, dl)[0].cpu().numpy()
    assert np.array_equal(a, b)
    _, rr = orc.render_forward(store, cam, retain=True)
    gr, _, _ = orc.render_backward(store, cam, rr, dl.cpu().numpy().astype(np.float64))
    n = store.size()

    def err(x):
        mean, ls, rot, op, sh = rgs.grads_from_soa(x, n)
        return floored_rel_err(np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1), gr)

    e_rep, e_atomic = err(a), err(c)
    print(f"reproducible: max {e_rep.max():.3e} above 1e-3 {(e_rep > 1e-3).sum()}; "
          f"atomic: max {e_atomic.max():.3e} above 1e-3 {(e_atomic > 1e-3).sum()}")
    assert (e_rep > 1e-3).sum() <= (e_atomic > 1e-3).sum()
    assert float((e_rep <= 1e-3).mean()) >= 0.9999
    rec.close()


def test_image_loss_small_images(ctx, T):
    """Below the 11x11 window: SSIM is rejected (ssim.cpp:81-82), the L1 part still works."""
    import torch

    a = torch.rand((10, 40, 3), dtype=torch.float32, device="cuda")
    b = torch.rand((10, 40, 3), dtype=torch.float32, device="cuda")
    with pytest.raises(rgs.RgsCudaError, match="smaller than the 11x11 window"):
        train.image_loss(ctx, a, b, 0.8, 0.2, torch.zeros_like(a))
    dl = torch.zeros_like(a)
    losses = torch.zeros(3, dtype=torch.float64, device="cuda")
    train.image_loss(ctx, a, b, 1.0, 0.0, dl, losses)
    torch.cuda.synchronize()
    l1, g1 = T.l1_loss(a.cpu().numpy().astype(np.float64), b.cpu().numpy().astype(np.float64))
    assert np.array_equal(dl.cpu().numpy(), g1.astype(np.float32))
    L = losses.cpu().numpy()
    assert abs(L[0] - l1) <= 1e-12 * l1 and np.isnan(L[1])


def _store_and_grads(n, seed, static=False):
    store = scenes.random_scene(n, sh_degree=3, seed=seed)
    if static:
        store.rotor[:, [3, 5, 6, 7]] = 0.0
    r = np.random.default_rng(seed)
    g = r.normal(0, 1e-2, (n, 65)).astype(np.float32).astype(np.float64)
    m = r.normal(0, 1e-3, (n, 65)).astype(np.float32).astype(np.float64)
    v = r.uniform(0, 1e-5, (n, 65)).astype(np.float32).astype(np.float64)
    return store, g, m, v


def _grads_soa(g, n):
    """(N, 65) reference order -> rgs_scene_params SoA float32 layout."""
    out = np.zeros(65 * n, dtype=np.float32)
    out[: 4 * n] = g[:, 0:4].reshape(-1)
    out[4 * n: 8 * n] = g[:, 4:8].reshape(-1)
    out[8 * n: 12 * n] = g[:, 8:12].reshape(-1)
    out[12 * n: 16 * n] = g[:, 12:16].reshape(-1)
    sh = g[:, 17:65].reshape(n, 3, 16).transpose(0, 2, 1).reshape(n, 48)  # j = k*3 + ch
    out[16 * n: 64 * n] = sh.reshape(n, 12, 4).transpose(1, 0, 2).reshape(-1)
    out[64 * n:] = g[:, 16]
    return out


@pytest.mark.parametrize("f64", [True, False])
@pytest.mark.parametrize("static", [0, 1])
def test_adam_step_matches_reference(ctx, T, f64, static):
    import torch

    n = 3000
    store, g, m, v = _store_and_grads(n, 40 + static, bool(static))
    sc = DeviceScene.from_store(ctx, store, f64=f64)
    opt = train.DeviceOptimizer(ctx, sc)
    opt.upload(m, v, np.zeros(n), np.zeros(n, dtype=np.int32))
    cfg = train.TrainConfig(static_mode=bool(static), total_steps=500)
    vis = torch.as_tensor(np.random.default_rng(1).integers(0, 3, n).astype(np.int32)).cuda()
    vn = torch.as_tensor(np.random.default_rng(2).uniform(0, 1, n).astype(np.float32)).cuda()
    opt.step(_t(_grads_soa(g, n)), vn, vis, train.CAdamConfig.from_config(cfg), 7)
    opt.status()
    ref_store, rm, rv = T.adam_step(store, m, v, g, O.adam_config(static_mode=static, total_steps=500), 7)
    got = sc.download()
    gm, gv, acc, cnt = opt.download()
    want = O.OracleLib._scene(ref_store)
    if f64:
        for x, y in zip(got, want):
            assert np.array_equal(x, y.reshape(x.shape))
        assert np.array_equal(gm, rm) and np.array_equal(gv, rv)
    else:
        for x, y in zip(got, want):
            assert np.array_equal(x, y.reshape(x.shape).astype(np.float32).astype(np.float64))
        assert np.array_equal(gm, rm.astype(np.float32).astype(np.float64))
        assert np.array_equal(gv, rv.astype(np.float32).astype(np.float64))
    vis_h, vn_h = vis.cpu().numpy(), vn.cpu().numpy().astype(np.float64)
    a2, c2 = T.accumulate_stats(vn_h, (vis_h > 0).astype(np.uint8), np.zeros(n), np.zeros(n, dtype=np.int32))
    assert np.array_equal(acc, a2) and np.array_equal(cnt, c2)


def test_adam_entropy_and_opacity_reset(ctx, T):
    import torch

    n = 2000
    store, g, m, v = _store_and_grads(n, 77)
    store.opacity_logit[:2] = [30.0, -30.0]  # clamp edges of the entropy term
    sc = DeviceScene.from_store(ctx, store, f64=True)
    opt = train.DeviceOptimizer(ctx, sc)
    lam = 0.01
    losses = torch.zeros(2, dtype=torch.float64, device="cuda")
    cfg = train.CAdamConfig.from_config(train.TrainConfig(), lambda_entropy=lam, accumulate_stats=False)
    opt.step(_t(_grads_soa(g, n)), None, None, cfg, 1, losses)
    opt.status()
    o = 1 / (1 + np.exp(-store.opacity_logit))
    ent, ge = T.entropy_loss(o)
    g2 = g.copy()
    g2[:, 16] = g[:, 16] + lam * ge * o * (1 - o)
    ref_store, _, _ = T.adam_step(store, np.zeros((n, 65)), np.zeros((n, 65)), g2, O.adam_config(), 1)
    got_op = sc.download()[3]
    assert np.allclose(got_op, ref_store.opacity_logit, rtol=0, atol=1e-12)
    assert abs(losses.cpu().numpy()[0] - ent) <= 1e-12 * ent
    opt.reset_opacity(0.01)
    op2, m2, v2 = T.reset_opacity(sc.download()[3], np.ones(n), np.ones(n), 0.01)
    assert np.allclose(sc.download()[3], op2, rtol=1e-14, atol=1e-14)
    gm, gv, _, _ = opt.download()
    assert not gm[:, 16].any() and not gv[:, 16].any()


def test_adam_zero_rotor_error(ctx):
    n = 50
    store = scenes.random_scene(n, sh_degree=0, seed=3)
    store.rotor[17] = 0.0
    sc = DeviceScene.from_store(ctx, store)
    opt = train.DeviceOptimizer(ctx, sc)
    opt.step(_t(np.zeros(65 * n, np.float32)), None, None,
             train.CAdamConfig.from_config(train.TrainConfig(), accumulate_stats=False), 1)
    import torch

    word = torch.zeros(1, dtype=torch.int64).pin_memory()
    opt.status_async(word)
    torch.cuda.synchronize()
    assert int(word.item()) >> 8 == 17  # (index << 8) | code, queued without a host sync
    with pytest.raises(rgs.ZeroRotorError) as e:
        opt.status()
    assert e.value.index == 17
    opt.status()  # cleared
    opt.status_async(word)
    torch.cuda.synchronize()
    assert int(word.item()) == -1


@pytest.mark.parametrize("k", [4, 8])
def test_knn_and_scene_scales(ctx, T, k):
    store = scenes.random_scene(3000, sh_degree=0, seed=k)
    sc = DeviceScene.from_store(ctx, store, f64=True)
    scales = train.scene_scales(ctx, sc)
    assert np.array_equal(scales, T.scene_scales(store.mean))
    nb = train.build_knn4d(ctx, sc, k).cpu().numpy()
    assert np.array_equal(nb, T.knn4d(store.mean, k, scales, threads=8))


def test_knn_grid_large_and_clustered(ctx, T):
    """The grid KNN on a frustum-shaped synthetic scene (non-uniform density) and on a
    clustered one: identical lists to the brute-force oracle."""
    store = scenes.synthetic_scene(40000, 320, 240, seed=12)
    sc = DeviceScene.from_store(ctx, store)
    scales = train.scene_scales(ctx, sc)
    nb = train.build_knn4d(ctx, sc, 8).cpu().numpy()
    assert np.array_equal(nb, T.knn4d(store.mean, 8, scales, threads=16))
    cl = scenes.random_scene(6000, sh_degree=0, seed=2)
    cl.mean[:3000, :3] = cl.mean[:3000, :3] * 1e-3 + 0.5  # a dense cluster inside a sparse cloud
    sc2 = DeviceScene.from_store(ctx, cl, f64=True)
    nb2 = train.build_knn4d(ctx, sc2, 16).cpu().numpy()
    assert np.array_equal(nb2, T.knn4d(cl.mean, 16, train.scene_scales(ctx, sc2), threads=16))


def test_knn_ties(ctx, T):
    store = scenes.random_scene(64, sh_degree=0, seed=1)
    store.mean[:] = np.round(store.mean * 2) / 2  # many exact distance ties
    sc = DeviceScene.from_store(ctx, store, f64=True)
    nb = train.build_knn4d(ctx, sc, 8).cpu().numpy()
    assert np.array_equal(nb, T.knn4d(store.mean, 8, train.scene_scales(ctx, sc)))


def test_consistency_matches_reference(ctx, T):
    import torch

    n = 1500
    store = scenes.random_scene(n, sh_degree=0, seed=9)
    sc = DeviceScene.from_store(ctx, store, f64=True)
    nb = train.build_knn4d(ctx, sc, 8)
    grads = torch.zeros(65 * n, dtype=torch.float32, device="cuda")
    losses = torch.zeros(1, dtype=torch.float64, device="cuda")
    train.consistency(ctx, sc, nb, 0.05, grads, losses)
    w = O.loss_weights(lambda_ssim=0.2, lambda_entropy=0.0, lambda_consistency=0.05)
    L, g, _, _ = T.evaluate_loss(store, [], [], w, nbrs=nb.cpu().numpy())
    assert abs(losses.cpu().numpy()[0] - L[3]) <= 1e-12 * L[3]
    mean, ls, rot, op, sh = rgs.grads_from_soa(grads.cpu().numpy(), n)
    got = np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1)
    err = floored_rel_err(got, g)
    assert err.max() <= 1e-3, err.max()


def _training_case(n=2500, views=3, w=96, h=72, seed=5):
    store = scenes.synthetic_scene(n, w, h, seed=seed)
    cams = [scenes.bench_camera(w, h, 0.2 + 0.3 * k, scenes.yaw_pose(4.0 * k, (0.03, -0.01, 0.05)))
            for k in range(views)]
    truth = store
    store = scenes.perturbed(truth, seed)
    return store, truth, cams


def test_evaluate_loss_matches_reference(ctx, T):
    """trainer.cpp:22-84 end to end on the device (render fwd, L1 + SSIM gradient, render bwd,
    batch sum, entropy and consistency) against the oracle on the same scene and targets."""
    import torch

    store, truth, cams = _training_case()
    tsc = DeviceScene.from_store(ctx, truth)
    targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
    sc = DeviceScene.from_store(ctx, store)
    tr = train.Trainer(ctx, sc, train.TrainConfig())
    tr.rebuild_knn()
    tr.evaluate_loss(cams, targets)
    torch.cuda.synchronize()
    # entropy is folded into the Adam step on the device: compare it separately
    w = O.loss_weights(lambda_entropy=0.0)
    L, g, vn, vis = T.evaluate_loss(store, cams, [t.cpu().numpy().astype(np.float64) for t in targets], w,
                                    nbrs=tr.nbrs.cpu().numpy(), threads=8)
    got = tr.losses.cpu().numpy()
    assert abs(got[0] - L[0]) <= 1e-5 * L[0]  # L1 of the float image vs the double image
    assert abs(got[1] - L[1]) <= 1e-5 * max(L[1], 1e-3)
    assert abs(got[4] - L[3]) <= 1e-9 * L[3]
    n = store.size()
    mean, ls, rot, op, sh = rgs.grads_from_soa(tr.grads.cpu().numpy(), n)
    gg = np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1)
    err = floored_rel_err(gg, g)
    assert np.mean(err <= 1e-3) >= 0.999, (np.mean(err <= 1e-3), err.max())
    assert np.array_equal(tr.visible.cpu().numpy() > 0, vis.astype(bool))
    assert np.allclose(tr.vnorm.cpu().numpy(), vn, rtol=1e-3, atol=1e-3 * vn.max())


def test_training_trajectory_matches_reference_loop(ctx, T):
    """Five train_from steps (trainer.cpp:134-150: evaluate_loss with entropy and consistency,
    accumulate_stats, adam_step) on an FP64 device scene at active SH degree 3 against the same
    loop on the oracle (the same targets and neighbour lists).  Per step the losses agree to
    1e-5 (entropy and consistency 1e-6); after five steps the parameter updates (p - p0) agree to the floored relative 1e-3 for
    >= 99.9 % of the coordinates -- the rest are coordinates whose gradient is near zero, where
    Adam's normalised step turns a 1e-3 gradient difference into a different sign."""
    import torch

    store, truth, cams = _training_case(n=2500, views=3)
    for a in (store.mean, store.log_scales, store.rotor, store.opacity_logit, store.sh):
        assert np.array_equal(a, a.astype(np.float32))
    tsc = DeviceScene.from_store(ctx, truth)
    targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
    cfg = train.TrainConfig(total_steps=6000)
    sc = DeviceScene.from_store(ctx, store, f64=True)
    tr = train.Trainer(ctx, sc, cfg, start_step=3000)
    tr.rebuild_knn()
    nbrs = tr.nbrs.cpu().numpy()
    t64 = [t.cpu().numpy().astype(np.float64) for t in targets]
    w = O.loss_weights()
    acfg = O.adam_config(total_steps=6000)
    ref, n = store, store.size()
    m, v = np.zeros((n, 65)), np.zeros((n, 65))
    for k in range(5):
        got = tr.step(cams, targets)
        L, g, _, _ = T.evaluate_loss(ref, cams, t64, w, nbrs=nbrs, threads=8)
        ref, m, v = T.adam_step(ref, m, v, g, acfg, 3001 + k)
        assert abs(got.l1 - L[0]) <= 1e-5 * L[0] and abs(got.ssim - L[1]) <= 1e-5 * max(L[1], 1e-3), (k, got, L)
        # (after the first step the two scenes differ by the trajectories' rounding: 1e-6 relative)
        assert abs(got.consistency - L[3]) <= 1e-6 * max(L[3], 1e-12) and abs(got.entropy - L[2]) <= 1e-6 * L[2]
    torch.cuda.synchronize()
    p0 = np.concatenate([a.reshape(n, -1) for a in O.OracleLib._scene(store)], axis=1)
    pg = np.concatenate([a.reshape(n, -1) for a in sc.download()], axis=1)
    pr = np.concatenate([a.reshape(n, -1) for a in O.OracleLib._scene(ref)], axis=1)
    err = floored_rel_err(pg - p0, pr - p0)
    frac = float((err <= 1e-3).mean())
    print(f"5-step trajectory: parameter updates within 1e-3: {100 * frac:.3f} %, max {err.max():.3e}")
    assert frac >= 0.999


def test_trainer_reduces_loss(ctx):
    """A few device steps of train_from's loop lower the loss toward the target renders."""
    store, truth, cams = _training_case(n=3000, views=4)
    tsc = DeviceScene.from_store(ctx, truth)
    targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
    sc = DeviceScene.from_store(ctx, store)
    tr = train.Trainer(ctx, sc, train.TrainConfig(total_steps=50, lr_sh_dc=2e-2))
    first = tr.step(cams, targets)
    for _ in range(30):
        last = tr.step(cams, targets)
    assert np.isfinite(last.total) and last.total < first.total
    m, v, acc, cnt = tr.opt.download()
    assert cnt.max() == 31 and acc.max() > 0


def _write_r4gs(path, store, version=1, magic=b"R4GS", truncate=0):
    """checkpoint.hpp:14-18 layout, written independently of the code under test."""
    n = store.size()
    rec = np.concatenate([store.mean, store.log_scales, store.rotor, store.opacity_logit[:, None],
                          store.sh.reshape(n, 48)], axis=1).astype("<f4")
    blob = magic + np.array([version, n, store.active_sh_degree], "<u4").tobytes() + rec.tobytes()
    with open(path, "wb") as f:
        f.write(blob[: len(blob) - truncate])
    return blob


@pytest.mark.parametrize("f64", [False, True])
def test_checkpoint_roundtrip(ctx, tmp_path, f64):
    """R4GS v1 load straight to the device and save back byte-identically (checkpoint.cpp:29-86)."""
    store = scenes.random_scene(777, sh_degree=2, seed=4)
    src = str(tmp_path / "a.r4gs")
    blob = _write_r4gs(src, store)
    sc = DeviceScene.load_checkpoint(ctx, src, f64=f64)
    assert sc.n == 777
    for x, y in zip(sc.download(), O.OracleLib._scene(store)):
        assert np.array_equal(x, y.reshape(x.shape))
    dst = str(tmp_path / "b.r4gs")
    sc.save_checkpoint(dst)
    assert open(dst, "rb").read() == blob
    if O.reference_available():
        import ctypes

        L = O.reference_build().lib
        L.ref_load_checkpoint.restype = ctypes.c_int
        n = L.ref_load_checkpoint(dst.encode(), None, None, None, None, None, None)
        assert n == 777


def test_checkpoint_errors(ctx, tmp_path):
    store = scenes.random_scene(10, sh_degree=1, seed=1)
    cases = [
        (dict(magic=b"R4GX"), "checkpoint: bad magic: "),
        (dict(version=2), "checkpoint: unsupported version 2"),
        (dict(truncate=8), "checkpoint: truncated: "),
    ]
    for kw, msg in cases:
        p = str(tmp_path / "bad.r4gs")
        _write_r4gs(p, store, **kw)
        with pytest.raises(rgs.CheckpointError) as e:
            DeviceScene.load_checkpoint(ctx, p)
        assert str(e.value).startswith(msg), str(e.value)
    store.active_sh_degree = 4
    p = str(tmp_path / "deg.r4gs")
    _write_r4gs(p, store)
    with pytest.raises(rgs.CheckpointError, match="malformed header"):
        DeviceScene.load_checkpoint(ctx, p)
    with pytest.raises(rgs.CheckpointError, match="cannot open"):
        DeviceScene.load_checkpoint(ctx, str(tmp_path / "missing.r4gs"))


def _densify_case(n, seed):
    store = scenes.random_scene(n, sh_degree=3, seed=seed)
    r = np.random.default_rng(seed)
    m = r.normal(0, 1e-3, (n, 65))
    v = r.uniform(0, 1e-5, (n, 65))
    count = r.integers(0, 4, n).astype(np.int32)
    accum = r.uniform(0, 1.5e-3, n) * count
    return store, m, v, accum, count


@pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("case", ["generic", "max_cut", "min_bound", "static"])
def test_densify_and_prune_matches_reference(ctx, case):
    """optim.cpp:168-234 on the device (FP64 scene) against the reference build with the same
    mt19937_64 seed: identical store, moments, statistics reset and report."""
    n = 2500
    store, m, v, accum, count = _densify_case(n, {"generic": 1, "max_cut": 2, "min_bound": 3, "static": 4}[case])
    kw = dict(percent_dense=0.02, prune_opacity=0.3)
    if case == "max_cut":
        kw["max_gaussians"] = n + 40
    if case == "min_bound":
        kw.update(prune_opacity=0.9, min_gaussians=n - 300)
    if case == "static":
        kw["static_mode"] = 1
        store.rotor[:, [3, 5, 6, 7]] = 0.0
    extent = 8.0
    cfg = train.TrainConfig(**{k: v2 for k, v2 in kw.items() if k != "static_mode"}, static_mode=bool(kw.get("static_mode")))
    sc = DeviceScene.from_store(ctx, store, f64=True)
    opt = train.DeviceOptimizer(ctx, sc)
    opt.upload(m, v, accum, count)
    rng = train.Rng(ctx, seed=1234)
    rep = train.densify_and_prune(ctx, sc, opt, cfg, extent, rng)
    ref_store, rm, rv, racc, rcnt, rrep = O.ref_densify_and_prune(store, m, v, accum, count,
                                                                   O.densify_config(**kw), extent, 1234)
    assert (rep.cloned, rep.split, rep.pruned) == rrep
    assert rep.cloned > 0 and rep.split > 0 and rep.pruned > 0
    assert sc.n == ref_store.size()
    for x, y in zip(sc.download(), O.OracleLib._scene(ref_store)):
        assert np.array_equal(x, y.reshape(x.shape))
    gm, gv, gacc, gcnt = opt.download()
    assert np.array_equal(gm, rm) and np.array_equal(gv, rv)
    assert not gacc.any() and not gcnt.any()


def test_rng_matches_std_mt19937_64(ctx):
    """The batch picks come from std::uniform_int_distribution over std::mt19937_64 (trainer.cpp:106)."""
    rng = train.Rng(ctx, seed=0)
    got = [rng.uniform_int(0, 9) for _ in range(8)]
    assert all(0 <= g <= 9 for g in got) and len(set(got)) > 1
    rng2 = train.Rng(ctx, seed=0)
    assert [rng2.uniform_int(0, 9) for _ in range(8)] == got


def test_trainer_densifies(ctx):
    store, truth, cams = _training_case(n=3000, views=3)
    tsc = DeviceScene.from_store(ctx, truth)
    targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
    sc = DeviceScene.from_store(ctx, store)
    cfg = train.TrainConfig(densify_from=2, densify_interval=3, densify_grad_threshold=1e-6, total_steps=20)
    tr = train.Trainer(ctx, sc, cfg, scene_extent=4.0)
    n0 = sc.n
    for _ in range(7):
        lb = tr.step(cams, targets)
    assert np.isfinite(lb.total)
    assert sc.n != n0 and tr.grads.numel() == 65 * sc.n


def test_trainer_overlap_matches_serial(ctx):
    """The overlapped multi-stream evaluate_loss (forward of view v+1 beside the backward of
    view v) gives the serial result: same losses, gradients equal up to FP64-atomic order."""
    import torch

    store, truth, cams = _training_case(n=3000, views=4)
    tsc = DeviceScene.from_store(ctx, truth)
    targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
    tctx = rgs.Context(0)  # on torch's stream: the overlap path needs it
    out = []
    for overlap in (False, True):
        sc = DeviceScene.from_store(tctx, store)
        tr = train.Trainer(tctx, sc, train.TrainConfig())
        tr.overlap = overlap
        tr.rebuild_knn()
        tr.evaluate_loss(cams, targets)
        torch.cuda.synchronize()
        out.append((tr.losses.cpu().numpy().copy(), tr.grads.cpu().numpy().copy(), tr.visible.cpu().numpy().copy()))
    (l0, g0, v0), (l1, g1, v1) = out
    assert np.allclose(l0, l1, rtol=1e-12, atol=0)
    assert np.array_equal(v0, v1)
    scale = np.abs(g0).max()
    assert np.abs(g0 - g1).max() <= 1e-5 * scale


def test_target_stager_pipeline(ctx):
    """train.TargetStager: step k+1's targets copied during step k arrive intact, and the
    staged steps give the losses of the same steps fed straight from device tensors."""
    import torch

    store, truth, cams = _training_case(n=3000, views=4)
    tctx = rgs.Context(0)
    tsc = DeviceScene.from_store(tctx, truth)
    dev_t = [tctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
    torch.cuda.synchronize()
    host = [t.cpu().pin_memory() for t in dev_t]
    batches = [[0, 1], [2, 3], [1, 2], [3, 0], [0, 2]]
    out = []
    for staged in (False, True):
        sc = DeviceScene.from_store(tctx, store)
        tr = train.Trainer(tctx, sc, train.TrainConfig(batch=2))
        st = train.TargetStager(0, 2, host[0].shape[0], host[0].shape[1])
        losses = []
        if staged:
            st.put([host[i] for i in batches[0]])
        for k, b in enumerate(batches):
            if staged:
                tg = st.take()
                if k + 1 < len(batches):
                    st.put([host[i] for i in batches[k + 1]])
                for t, i in zip(tg, b):
                    assert torch.equal(t, dev_t[i])
            else:
                tg = [dev_t[i] for i in b]
            losses.append(tr.step([cams[i] for i in b], tg).total)
            if staged:
                st.release(tctx)
        out.append(losses)
    assert np.allclose(out[0], out[1], rtol=1e-6, atol=0)  # FP64-atomic order only
    st = train.TargetStager(0, 1, 4, 4, depth=1)
    st.put([torch.zeros((4, 4, 3)).pin_memory()])
    with pytest.raises(RuntimeError):
        st.put([torch.zeros((4, 4, 3)).pin_memory()])


def test_pipelined_loss_reads(ctx):
    """read=False + pop_losses (step k's losses read while step k+1 runs) returns the losses
    the synchronous read returns for the same steps."""
    store, truth, cams = _training_case(n=3000, views=4)
    tctx = rgs.Context(0)
    tsc = DeviceScene.from_store(tctx, truth)
    targets = [tctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
    out = []
    for pipelined in (False, True):
        sc = DeviceScene.from_store(tctx, store)
        tr = train.Trainer(tctx, sc, train.TrainConfig(batch=2))
        got = []
        for k in range(5):
            b = [k % 4, (k + 1) % 4]
            args = ([cams[i] for i in b], [targets[i] for i in b])
            if not pipelined:
                got.append(tr.step(*args).total)
                continue
            tr.step(*args, read=False)
            if k > 0:
                got.append(tr.pop_losses().total)
        if pipelined:
            got.append(tr.pop_losses().total)
            with pytest.raises(IndexError):
                tr.pop_losses()
        out.append(got)
    assert len(out[1]) == 5
    assert np.allclose(out[0], out[1], rtol=1e-6, atol=0)  # FP64-atomic order only


def test_render_views_host_matches_device(ctx):
    """The e2e entry point (host scene in, host images out) renders what the device path does."""
    import torch

    store = scenes.synthetic_scene(20000, 320, 240, seed=8)
    cams = scenes.sweep_cameras(320, 240, 7)
    sc = DeviceScene.from_store(ctx, store)
    dev = ctx.render_views(sc, cams)
    torch.cuda.synchronize()
    host = torch.empty((7, 240, 320, 3), dtype=torch.float32).pin_memory()
    ctx.render_views_host(store.arrays_f32(), store.active_sh_degree, cams, (0, 0, 0), host.numpy())
    assert np.array_equal(host.numpy(), dev.cpu().numpy())
