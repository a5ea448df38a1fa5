"""GPU forward parity against the CPU oracle (sm_100a kernels through the C-ABI).

Bar (BASELINE.json north_star): splat records and per-tile lists / sort order
bit-exact; image within 1e-4 max abs per channel; final_T / n_contrib consistent.
"""
import numpy as np
import pytest

from paper_2402_03307_b200 import rgs, scenes
from parity import splat_mismatch

pytestmark = pytest.mark.gpu


def _compare_forward(ctx, orc, store, cam, bg=(0.0, 0.0, 0.0), threads=8, fp64=False):
    ref_img, ref = orc.render_forward(store, cam, bg, threads=threads, retain=True)
    out = rgs.render_forward(store, cam, rgs.RenderOptions(background=bg, retain_records=True, blend_fp64=fp64),
                             ctx=ctx)
    rec = out.records
    mm = splat_mismatch(rec.splats, ref.splats)
    assert mm == {}, f"splat records differ: {mm}"
    assert np.array_equal(rec.tile_offsets, ref.tile_offsets), "tile list lengths differ"
    assert np.array_equal(rec.tile_ids, ref.tile_ids), "tile lists / sort order differ"
    err = np.abs(out.image.astype(np.float64) - ref_img).max() if ref_img.size else 0.0
    nc_diff = int((rec.n_contrib != ref.n_contrib).sum())
    return err, nc_diff, rec, ref, out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_scenes_small(ctx, orc, seed):
    store = scenes.random_scene(60, sh_degree=seed % 4, seed=seed)
    cam = scenes.bench_camera(64 + 7 * seed, 64, time=0.3, pose=scenes.yaw_pose(3.0 * seed, (0.05, -0.02, 0.1)))
    cam.fx = cam.fy = 64.0
    err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam, bg=(0.1, 0.2, 0.3))
    assert err <= 1e-4
    assert ncd == 0


def test_c1_full_frame(ctx, orc):
    """Config C1: 50K Gaussians, SH3, 800x800, t=0.5 (yawed pose exercises the FP64 path)."""
    store = scenes.synthetic_scene(50_000, 800, 800, seed=1)
    for pose in (None, scenes.yaw_pose(7.0, (0.05, -0.02, 0.1))):
        cam = scenes.bench_camera(800, 800, 0.5, pose)
        err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam)
        assert err <= 1e-4, err
        assert ncd == 0
        print(f"C1 pose={'yaw' if pose is not None else 'id'}: splats={len(ref.splats)} pairs={len(ref.tile_ids)}"
              f" max_err={err:.3e} slow_pixels={rec.n_slow_pixels}")


def test_c2_frame(ctx, orc):
    """Config C2 shape: 300K Gaussians at 1352x1014, two timestamps of the sweep."""
    store = scenes.synthetic_scene(300_000, 1352, 1014, seed=2)
    for t in (0.0, 150 / 299):
        cam = scenes.bench_camera(1352, 1014, t, scenes.yaw_pose(7.0, (0.05, -0.02, 0.1)))
        err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam, threads=16)
        assert err <= 1e-4, err
        assert ncd == 0
        print(f"C2 t={t:.3f}: splats={len(ref.splats)} pairs={len(ref.tile_ids)} max_err={err:.3e}"
              f" slow_pixels={rec.n_slow_pixels}")


def test_c4_view(ctx, orc):
    """Config C4 shape: 2M Gaussians at 3840x2160 (240x135 tiles), one orbit view of the
    64-view batch: bit-exact tile lists, n_contrib identical, image <= 1e-4."""
    store = scenes.synthetic_scene(2_000_000, 3840, 2160, seed=4)
    cam = scenes.orbit_cameras(3840, 2160, 8, 8)[2 * 8 + 5]
    err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam, threads=32)
    assert err <= 1e-4, err
    assert ncd == 0
    print(f"C4: splats={len(ref.splats)} pairs={len(ref.tile_ids)} max_err={err:.3e} slow_pixels={rec.n_slow_pixels}")


def test_fp64_mode_matches_oracle_tightly(ctx, orc):
    store = scenes.random_scene(40, sh_degree=2, seed=11)
    cam = scenes.bench_camera(64, 48, 0.4)
    cam.fx = cam.fy = 64.0
    err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam, bg=(0.3, 0.1, 0.2), fp64=True)
    assert err <= 1e-6  # float32 output rounding only
    assert ncd == 0
    assert np.abs(rec.final_T - ref.final_T).max() <= 1e-12


def test_final_T_and_contrib(ctx, orc):
    store = scenes.random_scene(80, sh_degree=1, seed=5)
    cam = scenes.bench_camera(96, 80, 0.6)
    cam.fx = cam.fy = 80.0
    err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam)
    assert ncd == 0
    assert np.abs(rec.final_T - ref.final_T).max() <= 1e-5


def test_rasterize_forward_on_oracle_splats(ctx, orc):
    """rasterize_forward on host splats, including a non-monotone source_index order."""
    store = scenes.random_scene(50, sh_degree=1, seed=9)
    cam = scenes.bench_camera(64, 64, 0.3)
    cam.fx = cam.fy = 64.0
    _, ref = orc.render_forward(store, cam, retain=True)
    splats = ref.splats.copy()
    rng = np.random.default_rng(0)
    for perm in (np.arange(len(splats)), rng.permutation(len(splats))):
        sp = splats[perm]
        ref_img, r2 = orc.rasterize_forward(sp, cam, (0.2, 0.2, 0.2))
        img, rec = rgs.rasterize_forward(sp, cam, (0.2, 0.2, 0.2), ctx=ctx)
        assert np.array_equal(rec.tile_offsets, r2.tile_offsets)
        assert np.array_equal(rec.tile_ids, r2.tile_ids)
        assert np.abs(img - ref_img).max() <= 1e-4


def test_flow(ctx, orc):
    store = scenes.synthetic_scene(3000, 128, 96, seed=4)
    cam = scenes.bench_camera(128, 96, 0.5, scenes.yaw_pose(5.0))
    ref = orc.render_flow(store, cam, threads=4)
    got = rgs.render_flow(store, cam, ctx=ctx)
    scale = max(1.0, np.abs(ref).max())
    assert np.abs(got - ref).max() <= 1e-4 * scale


@pytest.mark.parametrize("n", [3000, 6000])
def test_equal_depth_ties(ctx, orc, n):
    """Every splat at the same depth: one depth bucket far above the small-bucket limit (the
    shared-memory bitonic path at 3000, the global-scratch path above 4096); the tile lists
    must come out in index order, as the reference's (depth, index) sort."""
    store = scenes.synthetic_scene(n, 320, 240, seed=11)
    store.mean[:, :2] *= 4.0 / store.mean[:, 2:3]  # same screen positions at depth 4
    store.mean[:, :2] = store.mean[:, :2].astype(np.float32)
    store.mean[:, 2] = 4.0
    store.rotor[:] = 0
    store.rotor[:, 0] = 1.0  # identity rotors: no space-time coupling, depth = z exactly
    cam = scenes.bench_camera(320, 240, 0.5)
    err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam)
    assert len(ref.splats) > 0.9 * n
    assert err <= 1e-4 and ncd == 0


def test_max_image_4096(ctx, orc):
    """The largest image of the two-byte-pass tile keys (4096 x 4096 = 256 x 256 tiles) on a
    sparse scene: records, tile lists and image against the oracle."""
    store = scenes.synthetic_scene(4000, 4096, 4096, seed=12)
    cam = scenes.bench_camera(4096, 4096, 0.4, scenes.yaw_pose(3.0, (0.02, 0.0, 0.05)))
    err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam, threads=16)
    assert rec.tiles_x == 256 and rec.tiles_y == 256
    assert err <= 1e-4 and ncd == 0


@pytest.mark.parametrize("shape", [(7680, 4320), (4112, 200)])
def test_wide_tile_keys_8k(ctx, orc, shape):
    """Beyond 256 tiles per axis the tile keys widen to ty << 12 | tx and the tile sort takes
    three byte passes (rasterizer.cpp:26-28 has no size limit): an 8K frame (480 x 270 tiles)
    and a 257-tile-wide strip -- splat records, tile lists, n_contrib and the image against the
    oracle, plus the backward on the 8K frame."""
    w, h = shape
    store = scenes.synthetic_scene(300_000 if w == 7680 else 20_000, w, h, seed=13)
    cam = scenes.bench_camera(w, h, 0.45, scenes.yaw_pose(3.0, (0.02, 0.0, 0.05)))
    err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam, threads=32)
    assert rec.tiles_x == (w + 15) // 16 and rec.tiles_x > 256
    assert err <= 1e-4 and ncd == 0
    print(f"{w}x{h}: {len(ref.splats)} splats, {len(ref.tile_ids)} pairs bit-exact, max image err {err:.2e}")
    if w == 7680:
        from parity import floored_rel_err

        dl = np.random.default_rng(8).uniform(-1, 1, (h, w, 3))
        g = rgs.render_backward(store, cam, out.records, dl, ctx=ctx)
        gr, vn, vis = orc.render_backward(store, cam, ref, dl, threads=32)
        assert np.array_equal(g.visible.astype(bool), vis.astype(bool))
        e = floored_rel_err(g.as_matrix(), gr)
        assert float((e <= 1e-3).mean()) >= 0.9999, e.max()


@pytest.mark.parametrize("shape", [(320, 240), (2048, 1024), (4096, 512)])
def test_binning_modes_identical(orc, shape):
    """The tile-major scatter and the radix passes produce the same per-tile lists: a small
    frame, the scatter's largest tile count (128 x 64 = 8192 tiles) and its widest rows (256 x 32
    tiles); the scatter's lists also against the oracle."""
    w, h = shape
    store = scenes.synthetic_scene(40_000, w, h, seed=21)
    cam = scenes.bench_camera(w, h, 0.35, scenes.yaw_pose(5.0, (0.03, -0.01, 0.08)))
    out = {}
    for mode in ("scatter", "radix"):
        c = rgs.Context(0, use_torch_stream=False)
        c.set_binning(mode)
        r = rgs.render_forward(store, cam, rgs.RenderOptions(retain_records=True), ctx=c)
        out[mode] = (r.image, r.records.tile_offsets, r.records.tile_ids, r.records.n_contrib)
    for a, b in zip(out["scatter"], out["radix"]):
        assert np.array_equal(a, b)
    ref_img, ref = orc.render_forward(store, cam, (0.0, 0.0, 0.0), threads=16, retain=True)
    assert np.array_equal(out["scatter"][2], ref.tile_ids)
    print(f"{w}x{h}: {len(ref.tile_ids)} pairs, scatter == radix == oracle")


def test_binning_large_splats(orc):
    """Rectangles from one tile to most of the frame in the same rounds of 32 ranks (the scatter's
    per-lane walks across owners, band rows and empty rectangles): both binnings against the
    oracle's tile lists."""
    store = scenes.synthetic_scene(20_000, 640, 480, seed=23)
    big = np.random.default_rng(5).choice(store.size(), 60, replace=False)
    store.log_scales[big, :3] += np.float32(2.5)
    store.log_scales[big, :3] = store.log_scales[big, :3].astype(np.float32)
    cam = scenes.bench_camera(640, 480, 0.5, scenes.yaw_pose(4.0, (0.02, 0.0, 0.05)))
    ref_img, ref = orc.render_forward(store, cam, (0.0, 0.0, 0.0), threads=16, retain=True)
    radius = np.asarray(ref.splats["radius"])
    assert radius.max() > 10 * np.median(radius) and radius.max() > 80  # rectangles of 100+ tiles
    for mode in ("scatter", "radix"):
        c = rgs.Context(0, use_torch_stream=False)
        c.set_binning(mode)
        r = rgs.render_forward(store, cam, rgs.RenderOptions(retain_records=True), ctx=c)
        assert np.array_equal(r.records.tile_offsets, ref.tile_offsets), mode
        assert np.array_equal(r.records.tile_ids, ref.tile_ids), mode
        assert np.array_equal(r.records.n_contrib, ref.n_contrib), mode
        assert np.abs(r.image.astype(np.float64) - ref_img).max() <= 1e-4, mode
    with pytest.raises(rgs.RgsCudaError, match="binning"):
        rgs.Context(0, use_torch_stream=False).set_binning(7)


def test_scene_params_tensor_view(ctx):
    """DeviceScene.params_tensor is a live view of the device SoA: writing through it (as an
    NCCL broadcast into a replica does) changes what the renderer sees."""
    import torch

    store = scenes.random_scene(300, sh_degree=3, seed=4)
    a = rgs.DeviceScene.from_store(ctx, store)
    b = rgs.DeviceScene(ctx, store.size(), store.active_sh_degree)
    ctx.synchronize()
    b.params_tensor().copy_(a.params_tensor())
    torch.cuda.synchronize()
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(x, y)
    cam = scenes.bench_camera(96, 64, 0.5)
    ia = ctx.render_forward_device(a, cam, retain=False)[0]
    ib = ctx.render_forward_device(b, cam, retain=False)[0]
    torch.cuda.synchronize()
    assert torch.equal(ia, ib)


def test_deferred_checks(ctx):
    """FLAG_DEFER_CHECKS forwards: no host sync, same image and records as a checked forward;
    a rotor error and a pair-buffer overflow surface through the context status (and the
    records), never silently."""
    import torch

    tctx = rgs.Context(0)
    store = scenes.synthetic_scene(3000, 160, 120, seed=5)
    cam = scenes.bench_camera(160, 120, 0.5)
    sc = rgs.DeviceScene.from_store(tctx, store)
    img0, rec0 = tctx.render_forward_device(sc, cam)  # checked: sizes the pooled frame
    ref = (img0.clone(), rec0.n_pairs, rec0.tile_ids.copy())
    rec0.close()
    img1, rec1 = tctx.render_forward_device(sc, cam, defer_checks=True)
    tctx.status()
    assert torch.equal(img1, ref[0]) and rec1.n_pairs == ref[1]
    assert np.array_equal(rec1.tile_ids, ref[2])
    rec1.close()
    # rotor error: reported by status(), not by the call
    bad = store.copy()
    bad.rotor[21] = 0
    bsc = rgs.DeviceScene.from_store(tctx, bad)
    _, rec2 = tctx.render_forward_device(bsc, cam, defer_checks=True)
    with pytest.raises(rgs.ZeroRotorError) as e:
        tctx.status()
    assert e.value.index == 21
    tctx.status()  # cleared
    rec2.close()
    # overflow: a pooled frame sized by the scenes above, then a ~7x denser one without checks
    sparse = rgs.DeviceScene.from_store(tctx, scenes.synthetic_scene(200, 160, 120, seed=6))
    _, r = tctx.render_forward_device(sparse, cam)
    r.close()
    dense = rgs.DeviceScene.from_store(tctx, scenes.synthetic_scene(20000, 160, 120, seed=7))
    _, r = tctx.render_forward_device(dense, cam, defer_checks=True)
    with pytest.raises(rgs.PairOverflowError):
        tctx.status()
    with pytest.raises(rgs.PairOverflowError):
        r.n_pairs
    r.close()
    tctx.status()


def test_empty_and_offscreen(ctx, orc):
    empty = rgs.GaussianStore.empty(0, 0)
    cam = scenes.bench_camera(40, 24, 0.5)
    out = rgs.render_forward(empty, cam, rgs.RenderOptions(background=(0.25, 0.5, 0.75)), ctx=ctx)
    assert np.allclose(out.image, np.array([0.25, 0.5, 0.75], np.float32))
    # everything behind the camera
    st = scenes.random_scene(20, seed=3)
    st.mean[:, 2] = -5
    out = rgs.render_forward(st, cam, rgs.RenderOptions(retain_records=True), ctx=ctx)
    assert len(out.records.splats) == 0 and out.records.n_pairs == 0
    assert np.all(out.image == 0)


def test_camera_and_rotor_errors(ctx):
    st = scenes.random_scene(10, seed=1)
    cam = scenes.bench_camera(32, 32, 0.5)
    bad = scenes.bench_camera(32, 32, 0.5)
    bad.fx = 0
    with pytest.raises(rgs.CameraError, match="focal lengths must be positive"):
        rgs.render_forward(st, bad, ctx=ctx)
    bad = scenes.bench_camera(32, 32, 0.5, pose=np.diag([2.0, 1, 1, 1]))
    with pytest.raises(rgs.CameraError, match="not orthogonal"):
        rgs.render_forward(st, bad, ctx=ctx)
    z = st.copy()
    z.rotor[4] = 0
    with pytest.raises(rgs.ZeroRotorError) as e:
        rgs.render_forward(z, cam, ctx=ctx)
    assert e.value.index == 4
    nf = st.copy()
    nf.rotor[7, 2] = np.nan
    with pytest.raises(rgs.NonFiniteRotorError):
        rgs.render_forward(nf, cam, ctx=ctx)


def test_render_views_batch_matches_single_views(ctx):
    """The multi-stream batch path (incl. a pair-buffer overflow re-render) equals per-view renders."""
    import torch

    store = scenes.synthetic_scene(20_000, 256, 192, seed=8)
    scene = rgs.DeviceScene.from_store(ctx, store)
    back = scenes.yaw_pose(180.0)  # sees nothing: slot 0 learns a tiny pair capacity first
    cams = [scenes.bench_camera(256, 192, 0.5, back)] + scenes.sweep_cameras(256, 192, 8)
    batch = ctx.render_views(scene, cams, (0.1, 0.2, 0.3))
    torch.cuda.synchronize()
    for v, cam in enumerate(cams):
        img, rec = ctx.render_forward_device(scene, cam, (0.1, 0.2, 0.3), retain=False)
        torch.cuda.synchronize()
        assert torch.equal(batch[v], img), v
    assert torch.all(batch[0] == torch.tensor([0.1, 0.2, 0.3], device=batch.device))


def test_render_views_large_frames_one_at_a_time(ctx):
    """Frames above ~2.2 MP render one view at a time with the longest-first tile order (the
    solo path): bitwise the per-view renders, incl. a view that sees nothing first."""
    import torch

    w, h = 2000, 1200
    store = scenes.synthetic_scene(60_000, w, h, seed=12)
    scene = rgs.DeviceScene.from_store(ctx, store)
    cams = [scenes.bench_camera(w, h, 0.5, scenes.yaw_pose(180.0))] + scenes.sweep_cameras(w, h, 3)
    batch = ctx.render_views(scene, cams, (0.05, 0.1, 0.2))
    torch.cuda.synchronize()
    for v, cam in enumerate(cams):
        img, rec = ctx.render_forward_device(scene, cam, (0.05, 0.1, 0.2), retain=False)
        torch.cuda.synchronize()
        assert torch.equal(batch[v], img), v


def test_missing_records(ctx):
    st = scenes.random_scene(3, seed=2)
    cam = scenes.bench_camera(32, 32, 0.3)
    out = rgs.render_forward(st, cam, rgs.RenderOptions(), ctx=ctx)
    with pytest.raises(rgs.MissingRecordsError):
        rgs.render_backward(st, cam, out.records, np.zeros((32, 32, 3)), ctx=ctx)


GOLDEN = sorted(__import__("glob").glob(__import__("os").path.join(__import__("os").path.dirname(__file__),
                                                                   "golden", "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: p.split("/")[-1])
def test_against_reference_golden(ctx, path):
    """CUDA path vs outputs of the reference itself (tests/golden, made by oracle/_ref)."""
    from test_oracle import load_case
    from parity import floored_rel_err

    z, store, cam, dl = load_case(path)
    bg = tuple(z["background"])
    out = rgs.render_forward(store, cam, rgs.RenderOptions(background=bg, retain_records=True), ctx=ctx)
    rec = out.records
    assert splat_mismatch(rec.splats, z["splats"]) == {}
    assert np.array_equal(rec.tile_offsets, z["tile_offsets"])
    assert np.array_equal(rec.tile_ids, z["tile_ids"])
    assert np.array_equal(rec.n_contrib, z["n_contrib"])
    assert np.abs(out.image - z["image"]).max() <= 1e-4
    g = rgs.render_backward(store, cam, rec, dl, ctx=ctx)
    assert np.array_equal(g.visible.astype(bool), z["visible"].astype(bool))
    assert floored_rel_err(g.as_matrix(), z["grads"]).max() <= 1e-3
    flow = rgs.render_flow(store, cam, ctx=ctx)
    assert np.abs(flow - z["flow"]).max() <= 1e-4 * max(1.0, np.abs(z["flow"]).max())


@pytest.mark.parametrize("seed", [3, 4])
def test_unrounded_store_fp64_scene(ctx, orc, seed):
    """Doubles that are not float32-representable: the drop-in stores them in an
    RGS_SCENE_F64 scene, so the splat records stay bit-exact with the oracle."""
    store = scenes.random_scene(70, sh_degree=3, seed=seed, f32=False)
    cam = scenes.bench_camera(80, 64, 0.45, pose=scenes.yaw_pose(5.0, (0.03, 0.01, -0.05)))
    cam.fx = cam.fy = 70.0
    err, ncd, rec, ref, out = _compare_forward(ctx, orc, store, cam, bg=(0.2, 0.2, 0.1), fp64=True)
    assert err <= 1e-6
    assert ncd == 0
    assert np.abs(rec.final_T - ref.final_T).max() <= 1e-12
    scene = rgs.DeviceScene.from_store(ctx, store, f64=True)
    assert scene.n_inexact == 0 and scene.params_ptr() != 0
    back = scene.download()
    for a, b in zip(back, store.arrays_f64()):
        assert np.array_equal(np.asarray(a).reshape(-1), np.asarray(b).reshape(-1))


_K5_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + '/oracle'); sys.path.insert(0, {root!r} + '/tests')
from paper_2402_03307_b200 import rgs, scenes
import oracle
store = scenes.synthetic_scene(20_000, 333, 250, seed=31)
cam = scenes.bench_camera(333, 250, 0.4, scenes.yaw_pose(4.0, (0.02, 0.01, 0.05)))
ctx = rgs.Context(0, use_torch_stream=False)
out = rgs.render_forward(store, cam, rgs.RenderOptions(background=(0.2, 0.1, 0.3), retain_records=True), ctx=ctx)
img, ref = oracle.restatement().render_forward(store, cam, (0.2, 0.1, 0.3), threads=8, retain=True)
assert np.array_equal(out.records.tile_ids, ref.tile_ids)
assert np.array_equal(out.records.n_contrib, ref.n_contrib), "n_contrib differs"
err = float(np.abs(out.image.astype(np.float64) - img).max())
assert err <= 1e-4, err
print("variant ok", err)
"""


@pytest.mark.parametrize("env", [{"RGS_K5": "2"}, {"RGS_K5": "x6"}, {"RGS_K5": "x8"}, {"RGS_K5_ORDER": "0"}])
def test_k5_variants_match_oracle(env):
    """The A/B variants of K5 selected by environment (read once per process, so each runs in a
    subprocess): one pixel per lane, the two-pixel kernel at 6 / 8 CTAs per SM, launch-order tiles
    -- the same n_contrib as the oracle and the image within 1e-4."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _K5_VARIANT_SCRIPT.format(root=root)], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "variant ok" in r.stdout
