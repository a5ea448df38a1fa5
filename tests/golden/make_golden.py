"""Generates the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Runs here (where /root/reference exists and oracle/_ref/librgs_ref.so is built from
the reference's own render sources, see oracle/Makefile).  The fixtures travel with
the repo so the oracle restatement and the CUDA path can be checked against the
reference's outputs on the GPU box, where /root/reference is absent.

Inputs are the reference's own unit-test scenes: tests/reference.hpp:27-46
random_scene() drawn from its global std::mt19937_64 seeded 20240817
(tests/oracles.hpp:93-101), on test_camera() (reference.hpp:17-25) and on a
yawed/translated variant; plus one synthetic C1-style scene.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ctypes  # noqa: E402

import oracle  # noqa: E402
from paper_2402_03307_b200 import scenes  # noqa: E402
from paper_2402_03307_b200.rgs import Camera, GaussianStore  # noqa: E402


def ref_random_scene(ref, n, deg):
    """tests/reference.hpp:27-46 via the reference's own code and RNG."""
    mean = np.zeros((n, 4))
    ls = np.zeros((n, 4))
    rot = np.zeros((n, 8))
    op = np.zeros(n)
    sh = np.zeros((n, 3, 16))
    ref.lib.ref_random_scene(n, deg, *[a.ctypes.data_as(ctypes.c_void_p) for a in (mean, ls, rot, op, sh)])
    # Rounded to float32 (as a checkpoint load does, checkpoint.cpp:75-82) so the FP32
    # device scene and the FP64 reference see identical inputs.
    f = lambda a: a.astype(np.float32).astype(np.float64)
    return GaussianStore(f(mean), f(ls), f(rot), f(op), f(sh), deg)


def test_camera(size=64, t=0.3, pose=None):
    """tests/reference.hpp:17-25"""
    return Camera(size, size, float(size), float(size), size / 2.0, size / 2.0,
                  np.eye(4) if pose is None else pose, t)


def save_case(name, ref, store, cam, bg, dl_seed):
    img, rec = ref.render_forward(store, cam, bg, threads=1, retain=True)
    dl = np.random.default_rng(dl_seed).uniform(-1, 1, (cam.height, cam.width, 3))
    grads, vnorm, vis = ref.render_backward(store, cam, rec, dl, threads=1)
    flow = ref.render_flow(store, cam, threads=1)
    naive, wsum, nT = ref.naive_render(store, cam, bg)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        mean=store.mean, log_scales=store.log_scales, rotor=store.rotor, opacity_logit=store.opacity_logit,
        sh=store.sh, sh_degree=store.active_sh_degree,
        cam_wh=np.array([cam.width, cam.height]), cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.time]),
        cam_w2c=np.asarray(cam.world_to_camera), background=np.asarray(bg, np.float64),
        image=img, splats=rec.splats, tile_offsets=rec.tile_offsets, tile_ids=rec.tile_ids,
        final_T=rec.final_T, n_contrib=rec.n_contrib, dl_seed=dl_seed, grads=grads, viewspace_norm=vnorm,
        visible=vis, flow=flow, naive_image=naive, naive_weight_sum=wsum, naive_final_T=nT)
    print(f"{name}: {store.size()} gaussians, {len(rec.splats)} splats, {len(rec.tile_ids)} pairs")


def main():
    ref = oracle.reference_build()
    ref.lib.ref_rng_reseed(ctypes.c_ulonglong(20240817))
    # test_render.cpp:46-61 style: 25-Gaussian scenes, degree 1, on test_camera().
    for k in range(3):
        st = ref_random_scene(ref, 25, 1)
        save_case(f"ref_scene25_{k}", ref, st, test_camera(), (0.1 * k, 0.2, 0.3), k)
    # Degree-3 scene on a yawed, translated camera (exercises the full FP64 projection).
    st = ref_random_scene(ref, 60, 3)
    pose = scenes.yaw_pose(7.0, (0.05, -0.02, 0.1))
    save_case("ref_scene60_sh3_yaw", ref, st, test_camera(96, 0.55, pose), (0.3, 0.1, 0.2), 7)
    # A C1-shaped synthetic scene at reduced size (float32-representable parameters).
    st = scenes.synthetic_scene(1500, 160, 120, seed=1)
    save_case("synthetic1500", ref, st, scenes.bench_camera(160, 120, 0.5, pose), (0.0, 0.0, 0.0), 11)


if __name__ == "__main__":
    main()
