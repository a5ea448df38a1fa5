import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_03307_b200 import rgs, scenes
import torch
ctx = rgs.Context(0)
store = scenes.synthetic_scene(20000, 320, 240, seed=6)
cam = scenes.bench_camera(320, 240, 0.5, scenes.yaw_pose(5.0, (0.02, 0.0, 0.04)))
sc = rgs.DeviceScene.from_store(ctx, store)
_, rec = ctx.render_forward_device(sc, cam, retain=True)
dl = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, (240, 320, 3)).astype(np.float32)).cuda()
outs = [ctx.render_backward_device(sc, cam, rec, dl, reproducible=True) for _ in range(3)]
torch.cuda.synchronize()
n = store.size()
for k in (1, 2):
    for name, i in (("grads", 0), ("vnorm", 1), ("visible", 2)):
        a, b = outs[0][i].cpu().numpy(), outs[k][i].cpu().numpy()
        d = np.nonzero(a != b)[0]
        print(k, name, "differ:", len(d), "of", a.size, (d[:8] // n if name == "grads" else d[:8]), (d[:8] % n if name == "grads" else ""))
        if len(d):
            print("   ", a[d[:5]], b[d[:5]])
print("slow pixels", rec.n_slow_pixels)
