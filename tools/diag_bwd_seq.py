import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
from parity import floored_rel_err
from paper_2402_03307_b200 import rgs, scenes, train
import torch
ctx = rgs.Context(0, use_torch_stream=False)
orc = O.restatement()

def check(tag):
    store = scenes.synthetic_scene(20000, 320, 240, seed=6)
    cam = scenes.bench_camera(320, 240, 0.5, scenes.yaw_pose(5.0, (0.02, 0.0, 0.04)))
    n = store.size()
    dln = np.random.default_rng(2).uniform(-1, 1, (240, 320, 3))
    _, rr = orc.render_forward(store, cam, retain=True)
    gr, vn, vis = orc.render_backward(store, cam, rr, dln)
    sc = rgs.DeviceScene.from_store(ctx, store)
    _, rec = ctx.render_forward_device(sc, cam, retain=True)
    dl = torch.from_numpy(dln.astype(np.float32)).cuda()
    x = ctx.render_backward_device(sc, cam, rec, dl)[0].cpu().numpy()
    mean, ls, rot, op, sh = rgs.grads_from_soa(x, n)
    gg = np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1)
    e = floored_rel_err(gg, gr)
    print(tag, "bad frac", (e > 1e-3).mean(), "slow", rec.n_slow_pixels, "pairs", rec.n_pairs, flush=True)
    rec.close()

check("fresh")
truth = scenes.synthetic_scene(6000, 160, 120, seed=5)
store = scenes.perturbed(truth, 5)
cams = [scenes.bench_camera(160, 120, 0.2 + 0.3 * k, scenes.yaw_pose(4.0 * k, (0.03, -0.01, 0.05))) for k in range(3)]
tsc = rgs.DeviceScene.from_store(ctx, truth)
targets = [ctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
sc = rgs.DeviceScene.from_store(ctx, store)
tr = train.Trainer(ctx, sc, train.TrainConfig(), start_step=3000)
for _ in range(3):
    tr.step(cams, targets)
torch.cuda.synchronize()
check("after trainer")
check("again")
