"""CPU tests of the oracle (the checker): pinned against the reference's own outputs
(tests/golden/, generated from oracle/_ref = the reference sources compiled in place)
and against the reference's known-answer tests (test_render.cpp, test_gaussian.cpp,
test_rotor.cpp), restated in Python on the oracle's entry points."""
import glob
import os

import numpy as np
import pytest

import oracle as O
from paper_2402_03307_b200 import scenes
from paper_2402_03307_b200.rgs import Camera, GaussianStore

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def load_case(path):
    z = np.load(path)
    store = GaussianStore(z["mean"], z["log_scales"], z["rotor"], z["opacity_logit"], z["sh"], int(z["sh_degree"]))
    w, h = z["cam_wh"]
    fx, fy, cx, cy, t = z["cam_f"]
    cam = Camera(int(w), int(h), fx, fy, cx, cy, z["cam_w2c"], t)
    dl = np.random.default_rng(int(z["dl_seed"])).uniform(-1, 1, (int(h), int(w), 3))
    return z, store, cam, dl


def test_golden_fixtures_present():
    assert len(GOLDEN) >= 5


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p))
def test_oracle_reproduces_reference_outputs(orc, path):
    """Bit-exact: image, splats, tile lists, final_T, n_contrib, grads, flow, naive."""
    z, store, cam, dl = load_case(path)
    bg = tuple(z["background"])
    img, rec = orc.render_forward(store, cam, bg, threads=3, retain=True)
    assert np.array_equal(img, z["image"])
    assert np.array_equal(rec.splats.view(np.uint8), z["splats"].view(np.uint8))
    assert np.array_equal(rec.tile_offsets, z["tile_offsets"])
    assert np.array_equal(rec.tile_ids, z["tile_ids"])
    assert np.array_equal(rec.final_T, z["final_T"])
    assert np.array_equal(rec.n_contrib, z["n_contrib"])
    g, vn, vis = orc.render_backward(store, cam, rec, dl, threads=2)
    assert np.array_equal(g, z["grads"])
    assert np.array_equal(vn, z["viewspace_norm"])
    assert np.array_equal(vis, z["visible"])
    assert np.array_equal(orc.render_flow(store, cam, threads=2), z["flow"])
    nimg, ws, nT = orc.naive_render(store, cam, bg)
    assert np.array_equal(nimg, z["naive_image"]) and np.array_equal(nT, z["naive_final_T"])


@pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_reference_build(orc, seed):
    """Restatement vs the reference's own sources, bit for bit, on fresh random inputs."""
    ref = O.reference_build()
    store = scenes.random_scene(70, sh_degree=seed % 4, seed=1000 + seed, f32=bool(seed % 2))
    cam = scenes.bench_camera(80 + seed, 72, 0.1 * seed, scenes.yaw_pose(2.0 * seed, (0.02 * seed, -0.01, 0.05)))
    cam.fx = cam.fy = 70.0
    bg = (0.05 * seed, 0.3, 0.2)
    i1, r1 = ref.render_forward(store, cam, bg, threads=1, retain=True)
    i2, r2 = orc.render_forward(store, cam, bg, threads=4, retain=True)
    assert np.array_equal(i1, i2)
    assert np.array_equal(r1.splats.view(np.uint8), r2.splats.view(np.uint8))
    assert np.array_equal(r1.tile_ids, r2.tile_ids) and np.array_equal(r1.final_T, r2.final_T)
    dl = np.random.default_rng(seed).uniform(-1, 1, (cam.height, cam.width, 3))
    for a, b in zip(ref.render_backward(store, cam, r1, dl), orc.render_backward(store, cam, r2, dl, threads=3)):
        assert np.array_equal(a, b)


# ----------------------------------------------------------------------------- reference KATs
def test_axis_aligned_slice_closed_form(orc):
    """test_gaussian.cpp:47-61"""
    out = orc.slice_at([1, 2, 3, 0.25], np.log([1.0, 2.0, 3.0, 0.5]), [1, 0, 0, 0, 0, 0, 0, 0], 0.75)
    mean, cov, decay, speed, lam = out[:3], out[3:12].reshape(3, 3), out[12], out[13:16], out[16]
    assert lam == pytest.approx(4.0, rel=1e-12)
    assert np.linalg.norm(speed) == 0.0
    assert np.linalg.norm(mean - [1, 2, 3]) == 0.0
    assert decay == pytest.approx(np.exp(-0.5 * 4.0 * 0.25), rel=1e-12)
    assert np.abs(cov - (np.diag([1.0, 4.0, 9.0]) + 1e-9 * np.eye(3))).max() <= 1e-12


def test_degenerate_time_raises(orc):
    """test_gaussian.cpp:123-127"""
    with pytest.raises(O.OracleError):
        orc.slice_at([0, 0, 0, 0], [0, 0, 0, np.log(1e-8)], [1, 0, 0, 0, 0, 0, 0, 0], 0.5)


def test_projection_on_axis(orc):
    """test_render.cpp:21-34"""
    cam = Camera(64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(4), 0.3)
    sliced = np.concatenate([[0, 0, 3], (0.01 * np.eye(3)).ravel(), [1.0], [0, 0, 0]])
    sp = orc.project(sliced, cam, np.zeros(48), 0, 2.0)
    assert sp is not None
    assert sp["mean2"][0] == pytest.approx(32.0) and sp["mean2"][1] == pytest.approx(32.0)
    assert sp["depth"] == pytest.approx(3.0)
    assert 1 / sp["conic"][0] == pytest.approx(64.0 * 64.0 / 9.0 * 0.01 + 0.3, rel=1e-9)


def test_projection_culls(orc):
    """test_render.cpp:36-44"""
    cam = Camera(64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(4), 0.3)
    behind = np.concatenate([[0, 0, -3], (0.01 * np.eye(3)).ravel(), [1.0], [0, 0, 0]])
    assert orc.project(behind, cam, np.zeros(48), 0, 2.0) is None
    front = np.concatenate([[0, 0, 3], (0.01 * np.eye(3)).ravel(), [1.0], [0, 0, 0]])
    assert orc.project(front, cam, np.zeros(48), 0, -8.0) is None


def test_tiled_equals_naive(orc):
    """test_render.cpp:46-61 / acceptance criterion 6 (<= 1e-6)."""
    for s in range(8):
        st = scenes.random_scene(25, sh_degree=1, seed=s, f32=False)
        cam = Camera(64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(4), 0.3)
        bg = tuple(np.random.default_rng(s).uniform(0, 1, 3))
        img, _ = orc.render_forward(st, cam, bg)
        nimg, _, _ = orc.naive_render(st, cam, bg)
        assert np.abs(img - nimg).max() <= 1e-6


def test_blend_weights_and_transmittance(orc):
    """test_render.cpp:63-75"""
    st = scenes.random_scene(40, sh_degree=1, seed=9, f32=False)
    cam = Camera(64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(4), 0.3)
    nimg, ws, nT = orc.naive_render(st, cam, (0, 0, 0))
    _, rec = orc.render_forward(st, cam, retain=True)
    assert (ws <= 1 + 1e-12).all()
    assert np.abs(1 - ws - nT).max() <= 1e-6
    assert np.allclose(rec.final_T, nT, rtol=1e-9, atol=0)


def test_thread_count_invariance(orc):
    """test_render.cpp:77-108: bit-identical forward and backward for 1..8 threads."""
    st = scenes.random_scene(30, sh_degree=1, seed=3, f32=False)
    cam = Camera(64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(4), 0.3)
    dl = np.random.default_rng(1).uniform(-1, 1, (64, 64, 3))
    i1, r1 = orc.render_forward(st, cam, threads=1, retain=True)
    g1 = orc.render_backward(st, cam, r1, dl, threads=1)
    for t in (2, 5, 8):
        it, rt = orc.render_forward(st, cam, threads=t, retain=True)
        assert np.array_equal(i1, it)
        for a, b in zip(g1, orc.render_backward(st, cam, rt, dl, threads=t)):
            assert np.array_equal(a, b)


def test_backward_matches_finite_differences(orc):
    """test_render.cpp:110-165: >= 95% of coordinates within rel 1e-3 or abs 1e-6."""
    st = scenes.random_scene(4, sh_degree=2, seed=21, f32=False)
    cam = Camera(32, 32, 32.0, 32.0, 16.0, 16.0, np.eye(4), 0.3)
    w = np.random.default_rng(5).uniform(-1, 1, (32, 32, 3))
    bg = (0.2, 0.1, 0.4)
    _, rec = orc.render_forward(st, cam, bg, retain=True)
    g, _, _ = orc.render_backward(st, cam, rec, w)

    def loss(s):
        return float((orc.render_forward(s, cam, bg)[0] * w).sum())

    h, ok, checked = 1e-5, 0, 0
    for gi in range(st.size()):
        for col in range(65):
            vals = []
            for d in (h, -h):
                s = st.copy()
                flat = [s.mean, s.log_scales, s.rotor, s.opacity_logit[:, None], s.sh.reshape(-1, 48)]
                off = [0, 4, 8, 16, 17]
                k = max(i for i in range(5) if off[i] <= col)
                flat[k][gi, col - off[k]] += d
                vals.append(loss(s))
            fd = (vals[0] - vals[1]) / (2 * h)
            checked += 1
            if abs(g[gi, col] - fd) <= 1e-3 * max(1.0, abs(fd)) or abs(g[gi, col] - fd) <= 1e-6:
                ok += 1
    assert ok / checked >= 0.95


def test_flow_is_screen_velocity(orc):
    """test_render.cpp:167-194: flow2 = d mean2 / dt."""
    c = np.zeros(8)
    c[0], c[3] = np.cos(0.1), np.sin(0.1)
    st = GaussianStore(np.array([[0.2, -0.1, 3.0, 0.5]]), np.array([[-2.0, -2, -2, -0.5]]), c[None], np.array([2.0]),
                       np.zeros((1, 3, 16)), 0)
    cam = Camera(64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(4), 0.5)
    _, rec = orc.render_forward(st, cam, retain=True)
    assert len(rec.splats) == 1
    h = 1e-5

    def m2(t):
        c2 = Camera(64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(4), t)
        return orc.render_forward(st, c2, retain=True)[1].splats[0]["mean2"]

    fd = (m2(0.5 + h) - m2(0.5 - h)) / (2 * h)
    assert np.linalg.norm(rec.splats[0]["flow2"] - fd) <= 1e-5 * (1 + np.linalg.norm(fd))


def test_flow_image(orc):
    """test_render.cpp:196-215"""
    c = np.zeros(8)
    c[0], c[3] = np.cos(0.12), np.sin(0.12)
    st = GaussianStore(np.array([[0.0, 0, 3.0, 0.5]]), np.array([[-1.5, -1.5, -1.5, -0.5]]), c[None],
                       np.array([3.0]), np.zeros((1, 3, 16)), 0)
    cam = Camera(64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(4), 0.5)
    flow = orc.render_flow(st, cam)
    assert abs(flow[32, 32, 0]) > 0.1
    assert flow[0, 0, 0] == 0.0 and flow[0, 0, 1] == 0.0


def test_rotor_invariants_and_errors(orc):
    """test_rotor.cpp:245-266 (normalize invariants, idempotence, errors)."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        r = rng.uniform(-1, 1, 8)
        n = orc.normalize(r)
        assert abs(np.linalg.norm(n) - 1) <= 1e-9
        eps = n[7] * n[0] - n[1] * n[6] + n[2] * n[5] - n[3] * n[4]
        assert abs(eps) <= 1e-9
        assert np.abs(orc.normalize(n) - n).max() <= 1e-12
        M = orc.to_matrix(n)
        assert np.abs(M @ M.T - np.eye(4)).max() <= 1e-9
    with pytest.raises(O.OracleError) as e:
        orc.normalize(np.zeros(8))
    assert e.value.code == 3
    bad = np.ones(8)
    bad[0] = np.nan
    with pytest.raises(O.OracleError) as e:
        orc.normalize(bad)
    assert e.value.code == 4


def test_missing_records(orc):
    """test_render.cpp:239-246"""
    st = scenes.random_scene(3, seed=2)
    cam = Camera(32, 32, 32.0, 32.0, 16.0, 16.0, np.eye(4), 0.3)
    _, rec = orc.render_forward(st, cam, retain=False)
    with pytest.raises(O.OracleError) as e:
        orc.render_backward(st, cam, rec, np.zeros((32, 32, 3)))
    assert e.value.code == 2
