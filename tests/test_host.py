"""Host-side logic that needs no GPU: parameter layouts, the scene generator, and the
multi-process (world_size 2, gloo) bench plumbing."""
import os
import socket
import sys

import numpy as np
import pytest

from paper_2402_03307_b200 import rgs, scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pack_soa(store):
    """numpy restatement of k_scene_pack (the rgs_scene_params layout)."""
    n = store.size()
    mean, ls, rot, op, sh = store.arrays_f64()
    P = np.zeros(65 * n)
    P[: 4 * n] = mean.reshape(-1)
    P[4 * n: 8 * n] = ls.reshape(-1)
    P[8 * n: 12 * n] = rot[:, :4].reshape(-1)
    P[12 * n: 16 * n] = rot[:, 4:].reshape(-1)
    j = sh.reshape(n, 3, 16).transpose(0, 2, 1).reshape(n, 48)  # j = k*3 + ch
    P[16 * n: 64 * n] = j.reshape(n, 12, 4).transpose(1, 0, 2).reshape(-1)
    P[64 * n:] = op
    return P


def test_soa_layout_roundtrip():
    st = scenes.random_scene(7, sh_degree=3, seed=1)
    mean, ls, rot, op, sh = rgs.grads_from_soa(pack_soa(st), st.size())
    assert np.array_equal(mean, st.mean) and np.array_equal(ls, st.log_scales)
    assert np.array_equal(rot, st.rotor) and np.array_equal(op, st.opacity_logit)
    assert np.array_equal(sh, st.sh)


def test_synthetic_scene_is_float32_and_moves():
    st = scenes.synthetic_scene(2000, 400, 300, seed=5)
    for a in st.arrays_f64():
        assert np.array_equal(a, a.astype(np.float32).astype(np.float64))
    v = scenes.gaussian_speed(st.rotor, st.log_scales)
    assert np.abs(v[1::2]).max() < 1e-6  # odd: static (purely spatial rotor)
    moving = np.linalg.norm(v[0::2], axis=1)
    assert moving.mean() > 0.1 and moving.max() < 1.0
    # all centres inside the frustum (acceptance.cpp:493-520 recipe)
    x, y, z = st.mean[:, 0], st.mean[:, 1], st.mean[:, 2]
    assert ((z >= 2) & (z <= 8)).all()
    assert (np.abs(x / z) <= 0.875 * 200 / 500 + 1e-6).all()


def test_velocity_rotor_matches_requested_speed():
    """acceptance criterion 4's construction (synthetic.cpp:134-177)."""
    rng = np.random.default_rng(0)
    v = rng.uniform(-1.5, 1.5, (200, 3))
    sx, st = rng.uniform(0.1, 0.4, 200), rng.uniform(2.0, 50.0, 200)
    r = scenes.velocity_rotor(v, sx, st)
    ls = np.stack([np.log(sx)] * 3 + [np.log(st)], -1)
    assert np.abs(scenes.gaussian_speed(r, ls) - v).max() <= 1e-9


def test_cameras():
    cams = scenes.sweep_cameras(1352, 1014, 300)
    assert len(cams) == 300 and cams[0].time == 0.0 and cams[-1].time == 1.0
    for c in cams[:3]:
        c.validate()
    orbit = scenes.orbit_cameras(64, 48, 8, 8)
    assert len(orbit) == 64
    for c in orbit:
        c.validate()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = bench.max_over_ranks(10.0 + rank, dist, "cpu")
    cams = bench.sweep_for_rank(rank)
    dist.barrier()
    q.put((rank, t, len(cams), float(np.asarray(cams[0].world_to_camera)[0, 2])))
    dist.destroy_process_group()


def test_bench_multi_rank_plumbing_gloo():
    """N>1 bench logic: every rank gets the max time; each rank renders its own 300-view sweep."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [11.0, 11.0]
    assert all(r[2] == 300 for r in res)
    assert res[0][3] != res[1][3]  # distinct camera poses per rank


def _train_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    from paper_2402_03307_b200 import train

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 5
    # per-rank partial batch sums: grads|vnorm, visible counts, image losses
    gbuf = torch.arange(66 * n, dtype=torch.float32) * (rank + 1)
    vis = torch.tensor([1, 0, 0, 1, 0], dtype=torch.int32) if rank == 0 else torch.tensor([0, 0, 1, 1, 0],
                                                                                           dtype=torch.int32)
    losses = torch.zeros(8, dtype=torch.float64)
    losses[:3] = torch.tensor([0.1, 0.2, 0.3], dtype=torch.float64) * (rank + 1)
    losses[3] = 7.0  # entropy: replicated, must not be summed
    train.allreduce_step_buffers(gbuf, vis, losses[:3], dist)
    q.put((rank, gbuf.tolist(), vis.tolist(), losses.tolist()))
    dist.destroy_process_group()


def test_training_batch_reduction_gloo():
    """Multi-GPU training plumbing (world 2, gloo): the all-reduce reproduces the single-process
    batch reduction -- grads and viewspace norms summed, visible counted (> 0 == OR,
    gaussian.cpp:199-209), image losses summed, replicated regularizer slots untouched."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_train_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    n = 5
    for _, g, vis, losses in res:
        assert g == [3.0 * k for k in range(66 * n)]
        assert [v > 0 for v in vis] == [True, False, True, True, False]
        assert np.allclose(losses[:3], [0.3, 0.6, 0.9]) and losses[3] == 7.0
