import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
from parity import floored_rel_err
from paper_2402_03307_b200 import rgs, scenes
import torch
ctx = rgs.Context(0)
orc = O.restatement()
store = scenes.synthetic_scene(20000, 320, 240, seed=6)
cam = scenes.bench_camera(320, 240, 0.5, scenes.yaw_pose(5.0, (0.02, 0.0, 0.04)))
n = store.size()
dln = np.random.default_rng(2).uniform(-1, 1, (240, 320, 3))
_, rr = orc.render_forward(store, cam, retain=True)
gr, vn, vis = orc.render_backward(store, cam, rr, dln)
out = rgs.render_forward(store, cam, rgs.RenderOptions(retain_records=True), ctx=ctx)
g = rgs.render_backward(store, cam, out.records, dln, ctx=ctx)
print("numpy API:", (floored_rel_err(g.as_matrix(), gr) > 1e-3).mean())
sc = rgs.DeviceScene.from_store(ctx, store)
_, rec = ctx.render_forward_device(sc, cam, retain=True)
dl = torch.from_numpy(dln.astype(np.float32)).cuda()
for kw in ({}, {"reproducible": True}):
    x = ctx.render_backward_device(sc, cam, rec, dl, **kw)[0].cpu().numpy()
    mean, ls, rot, op, sh = rgs.grads_from_soa(x, n)
    gg = np.concatenate([mean, ls, rot, op[:, None], sh.reshape(n, 48)], axis=1)
    e = floored_rel_err(gg, gr)
    bad = np.argwhere(e > 1e-3)
    print("device API", kw, (e > 1e-3).mean(), "cols", sorted(set(bad[:, 1].tolist()))[:20])
    print("   vs numpy API grads:", np.abs(gg - g.as_matrix()).max())
