"""CPU tests of the training-side oracle: the plain-C restatement
(oracle/rgs_oracle.c) against the reference's own image.cpp / ssim.cpp / loss.cpp /
knn.cpp / optim.cpp / trainer.cpp compiled in place (oracle/_ref), bit for bit, plus the
reference's known answers for these functions (test_loss.cpp, test_optim.cpp) restated."""
import numpy as np
import pytest

import oracle as O
from paper_2402_03307_b200 import scenes

needs_ref = pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def T():
    return O.train_ops("orc")


@pytest.fixture(scope="module")
def R():
    return O.train_ops("ref")


def _images(seed, h=37, w=45):
    r = np.random.default_rng(seed)
    a = r.uniform(0, 1, (h, w, 3))
    b = np.clip(a + r.normal(0, 0.1, a.shape), 0, 1)
    b[3, 4] = a[3, 4]  # exact ties: l1 gradient 0
    return a, b


@needs_ref
@pytest.mark.parametrize("seed", range(3))
def test_image_losses_match_reference(T, R, seed):
    a, b = _images(seed, 30 + seed, 41 - seed)
    for fn in ("l1_loss", "ssim_loss"):
        la, ga = getattr(T, fn)(a, b)
        lb, gb = getattr(R, fn)(a, b)
        assert la == lb, fn
        assert np.array_equal(ga, gb), fn
    assert T.psnr(a, b) == R.psnr(a, b)
    assert T.psnr(a, a) == 100.0


def test_ssim_known_answers(T):
    """ssim.hpp: constant images give the closed-form SSIM; identical images give loss 0
    and zero gradient (test_loss.cpp's SSIM cases, restated)."""
    a = np.full((16, 20, 3), 0.3)
    b = np.full((16, 20, 3), 0.6)
    loss, g = T.ssim_loss(a, a)
    assert abs(loss) < 1e-12 and np.abs(g).max() < 1e-9
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    s = (2 * 0.3 * 0.6 + c1) * c2 / ((0.3 ** 2 + 0.6 ** 2 + c1) * c2)
    loss, _ = T.ssim_loss(a, b)
    assert abs(loss - (1 - s)) < 1e-12
    with pytest.raises(O.OracleError):
        T.ssim_loss(np.zeros((10, 30, 3)), np.zeros((10, 30, 3)))


def test_ssim_gradient_finite_differences(T):
    a, b = _images(7, 14, 15)
    _, g = T.ssim_loss(a, b)
    r = np.random.default_rng(1)
    for _ in range(6):
        y, x, c = r.integers(0, 14), r.integers(0, 15), r.integers(0, 3)
        e = 1e-6
        ap, am = a.copy(), a.copy()
        ap[y, x, c] += e
        am[y, x, c] -= e
        fd = (T.ssim_loss(ap, b, False)[0] - T.ssim_loss(am, b, False)[0]) / (2 * e)
        assert abs(fd - g[y, x, c]) < 1e-6 + 1e-4 * abs(fd)


@needs_ref
def test_regularizers_match_reference(T, R):
    r = np.random.default_rng(3)
    o = r.uniform(0, 1, 500)
    o[:3] = [0.0, 1.0, 1e-7]  # clamp edges
    la, ga = T.entropy_loss(o)
    lb, gb = R.entropy_loss(o)
    assert la == lb and np.array_equal(ga, gb)
    store = scenes.random_scene(300, sh_degree=0, seed=5)
    sc = T.scene_scales(store.mean)
    assert np.array_equal(sc, R.scene_scales(store.mean))
    nb = T.knn4d(store.mean, 8, sc, threads=3)
    assert np.array_equal(nb, R.knn4d(store.mean, 8, sc, threads=2))
    sp = T.gaussian_speeds(store)
    assert np.array_equal(sp, R.gaussian_speeds(store))
    la, ga = T.consistency_loss(sp, nb)
    lb, gb = R.consistency_loss(sp, nb)
    assert la == lb and np.array_equal(ga, gb)


def test_knn_ties_by_index(T):
    """knn.hpp:18-20: ties broken by index, self excluded."""
    mean = np.zeros((6, 4))
    mean[:, 0] = [0, 1, -1, 2, -2, 0]
    nb = T.knn4d(mean, 3, np.ones(4))
    assert list(nb[0]) == [5, 1, 2]
    assert list(nb[5]) == [0, 1, 2]


@needs_ref
@pytest.mark.parametrize("static", [0, 1])
def test_adam_step_matches_reference(T, R, static):
    store = scenes.random_scene(200, sh_degree=3, seed=11 + static)
    if static:
        store.rotor[:, [3, 5, 6, 7]] = 0.0
    r = np.random.default_rng(static)
    n = store.size()
    m = r.normal(0, 1e-3, (n, 65))
    v = r.uniform(0, 1e-5, (n, 65))
    g = r.normal(0, 1e-2, (n, 65))
    cfg = O.adam_config(static_mode=static, total_steps=500)
    for step in (1, 7, 600):
        sa, ma, va = T.adam_step(store, m, v, g, cfg, step)
        sb, mb, vb = R.adam_step(store, m, v, g, cfg, step)
        for x, y in zip(O.OracleLib._scene(sa), O.OracleLib._scene(sb)):
            assert np.array_equal(x, y)
        assert np.array_equal(ma, mb) and np.array_equal(va, vb)
    for step in (0, 3, 2000, 5000):
        assert T.lr_schedule(step, 2000, 1.6e-4, 1.6e-6) == R.lr_schedule(step, 2000, 1.6e-4, 1.6e-6)


def test_adam_first_step_moves_by_lr(T):
    """test_optim.cpp: at step 1 Adam moves every free parameter by ~lr against the gradient."""
    store = scenes.random_scene(20, sh_degree=3, seed=2)
    n = store.size()
    g = np.random.default_rng(0).choice([-1.0, 1.0], (n, 65)) * 1e-3
    cfg = O.adam_config()
    s2, m2, v2 = T.adam_step(store, np.zeros((n, 65)), np.zeros((n, 65)), g, cfg, 1)
    d = s2.opacity_logit - store.opacity_logit
    assert np.allclose(d, -np.sign(g[:, 16]) * cfg.lr_opacity, rtol=1e-9)
    assert np.allclose(s2.sh[:, :, 0] - store.sh[:, :, 0], -np.sign(g[:, 17:65:16]) * cfg.lr_sh_dc, rtol=1e-9)


@needs_ref
def test_stats_and_opacity_reset_match_reference(T, R):
    r = np.random.default_rng(9)
    n = 400
    vn, vis = r.uniform(0, 1, n), r.integers(0, 2, n).astype(np.uint8)
    acc, cnt = r.uniform(0, 1, n), r.integers(0, 5, n)
    a1, c1 = T.accumulate_stats(vn, vis, acc, cnt)
    a2, c2 = R.accumulate_stats(vn, vis, acc, cnt)
    assert np.array_equal(a1, a2) and np.array_equal(c1, c2)
    op = r.normal(0, 3, n)
    for x, y in zip(T.reset_opacity(op, r.normal(size=n), r.normal(size=n)),
                    R.reset_opacity(op, r.normal(size=n), r.normal(size=n))):
        assert np.array_equal(x, y)


@needs_ref
@pytest.mark.parametrize("with_knn", [False, True])
def test_evaluate_loss_matches_reference(T, R, with_knn):
    """trainer.cpp:22-84: the whole batch reduction (render fwd, L1 + SSIM image gradient,
    render bwd, StoreGrads::add, entropy and consistency terms) bit for bit."""
    store = scenes.random_scene(90, sh_degree=2, seed=21)
    cams = []
    for k in range(3):
        c = scenes.bench_camera(40, 34, 0.2 + 0.3 * k, scenes.yaw_pose(3.0 * k, (0.02, 0.0, 0.05)))
        c.fx = c.fy = 36.0
        cams.append(c)
    tg = [np.random.default_rng(k).uniform(0, 1, (34, 40, 3)) for k in range(3)]
    w = O.loss_weights()
    nb = T.knn4d(store.mean, 8, T.scene_scales(store.mean)) if with_knn else None
    la, ga, va, sa = T.evaluate_loss(store, cams, tg, w, (0.1, 0.2, 0.3), nb, threads=3)
    lb, gb, vb, sb = R.evaluate_loss(store, cams, tg, w, (0.1, 0.2, 0.3), nb, threads=2)
    assert np.array_equal(la, lb)
    assert np.array_equal(ga, gb) and np.array_equal(va, vb) and np.array_equal(sa, sb)
    assert sa.sum() > 10
