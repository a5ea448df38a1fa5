"""Multi-rank correctness of the CUDA path on one GPU (two processes on cuda:0 over gloo: the
bench's RGS_BENCH_SHARE_GPU mode -- NCCL refuses two ranks on one device, and this build has
one GPU per call).  SURVEY.md §8(e), trainer.cpp:33-53, gaussian.cpp:199-209:

* view-batch sharding: each rank renders its contiguous half of an 8-view camera x timestamp
  batch; the gathered images are bitwise the single-rank batch;
* training: 2 ranks x 4 views, reduced by the all-reduce, give the gradients of 1 rank x 8
  views (FP32 accumulation order differs: floored relative 1e-5), identical losses to 1e-12;
* replicas: after Adam and a densify-and-prune step the two ranks' scenes are bit-identical;
* the native NCCL entry (rgs_allreduce_grads) on a one-rank communicator is the identity."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

VIEWS = 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_2402_03307_b200 import scenes

    truth = scenes.synthetic_scene(20_000, 320, 240, seed=21)
    store = scenes.perturbed(truth, 21)
    cams = [scenes.bench_camera(320, 240, (v + 0.5) / VIEWS, scenes.yaw_pose(-4.0 + v, (0.02, 0.0, 0.03)))
            for v in range(VIEWS)]
    return truth, store, cams


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2402_03307_b200 import rgs, train

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = rgs.Context(0)
    truth, store, cams = _case()
    mine = cams[rank * VIEWS // world:(rank + 1) * VIEWS // world]
    # (1) sharded render of the batch
    tsc = rgs.DeviceScene.from_store(ctx, truth)
    imgs = torch.empty((len(mine), 240, 320, 3), dtype=torch.float32, device="cuda")
    ctx.render_views(tsc, mine, (0.0, 0.0, 0.0), out=imgs)
    gathered = [torch.empty_like(imgs.cpu()) for _ in range(world)]
    dist.all_gather(gathered, imgs.cpu())
    targets = [t.cuda() for t in torch.cat(gathered)]  # every view's target on every rank
    mt = targets[rank * VIEWS // world:(rank + 1) * VIEWS // world]
    # (2) one evaluate_loss of the whole batch across the ranks
    sc = rgs.DeviceScene.from_store(ctx, store)
    cfg = train.TrainConfig(batch=VIEWS // world, densify_from=1, densify_interval=2, densify_grad_threshold=1e-9)
    tr = train.Trainer(ctx, sc, cfg, dist, scene_extent=4.0, seed=5)
    tr.rebuild_knn()
    tr.evaluate_loss(mine, mt)
    torch.cuda.synchronize()
    grads = (tr.grads.cpu().numpy().copy(), tr.vnorm.cpu().numpy().copy(), tr.visible.cpu().numpy().copy(),
             tr.losses.cpu().numpy().copy())
    # (3) two full steps (the second densifies), then the replica
    tr.step(mine, mt)
    rep = tr.step(mine, mt)
    scene_after = [a.copy() for a in sc.download()]
    q.put((rank, torch.cat(gathered).numpy(), grads, scene_after, (rep.total, sc.n, tr.last_densify.cloned,
                                                                     tr.last_densify.split, tr.last_densify.pruned)))
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def two_ranks():
    import torch.multiprocessing as mp

    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    return res


def _single_rank_reference(ctx):
    import torch

    from paper_2402_03307_b200 import rgs, train

    truth, store, cams = _case()
    tsc = rgs.DeviceScene.from_store(ctx, truth)
    imgs = torch.empty((VIEWS, 240, 320, 3), dtype=torch.float32, device="cuda")
    ctx.render_views(tsc, cams, (0.0, 0.0, 0.0), out=imgs)
    targets = [imgs[v].clone() for v in range(VIEWS)]
    sc = rgs.DeviceScene.from_store(ctx, store)
    tr = train.Trainer(ctx, sc, train.TrainConfig(batch=VIEWS))
    tr.rebuild_knn()
    tr.evaluate_loss(cams, targets)
    torch.cuda.synchronize()
    return imgs.cpu().numpy(), (tr.grads.cpu().numpy(), tr.vnorm.cpu().numpy(), tr.visible.cpu().numpy(),
                                tr.losses.cpu().numpy())


def test_sharded_render_matches_single_rank(ctx, two_ranks):
    ref_imgs, _ = _single_rank_reference(ctx)
    for rank, imgs, *_ in two_ranks:
        assert np.array_equal(imgs, ref_imgs), f"rank {rank}: gathered batch differs from the single-rank batch"


def test_two_rank_gradients_match_single_rank(ctx, two_ranks):
    from parity import floored_rel_err

    _, (g1, vn1, vis1, l1) = _single_rank_reference(ctx)
    n = vn1.shape[0]
    for rank, _, (g2, vn2, vis2, l2), *_ in two_ranks:
        err = floored_rel_err(g2.reshape(65, n).T, g1.reshape(65, n).T)
        print(f"rank {rank}: max floored rel err {err.max():.3e} (2 x 4 views vs 1 x 8 views)")
        assert err.max() <= 1e-5
        assert np.array_equal(vis2 > 0, vis1 > 0)
        assert np.allclose(vn2, vn1, rtol=1e-5, atol=1e-7 * max(vn1.max(), 1e-30))
        assert np.allclose(l2[:3], l1[:3], rtol=1e-12), (l2[:3], l1[:3])
        assert abs(l2[4] - l1[4]) <= 1e-12 * max(abs(l1[4]), 1e-30)  # consistency: once per step


def test_replicas_identical_after_adam_and_densify(two_ranks):
    (_, _, _, s0, info0), (_, _, _, s1, info1) = two_ranks
    assert info0 == info1
    assert info0[2] + info0[3] > 0, "the second step densified"
    for a, b in zip(s0, s1):
        assert np.array_equal(a, b)


def test_native_allreduce_single_rank_is_identity(ctx):
    import torch

    from paper_2402_03307_b200 import rgs, train

    if not ctx.L.rgs_nccl_available():
        pytest.fail("NCCL not resolvable by librgs_cuda.so")
    truth, store, cams = _case()
    tsc = rgs.DeviceScene.from_store(ctx, truth)
    targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams[:3]]
    outs = []
    for comm in (None, train.NcclComm.single(ctx)):
        sc = rgs.DeviceScene.from_store(ctx, store)
        tr = train.Trainer(ctx, sc, train.TrainConfig(), comm=comm)
        tr.rebuild_knn()
        tr.evaluate_loss(cams[:3], targets)
        torch.cuda.synchronize()
        outs.append((tr.grads.cpu().numpy(), tr.visible.cpu().numpy(), tr.losses.cpu().numpy()))
        if comm is not None:
            comm.close()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
