"""Views in flight vs frame size / scene size: render_views throughput (RGS_SLOTS / RGS_SLOTS_BIG
are read per process, so the caller runs this once per setting)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_03307_b200 import rgs, scenes  # noqa: E402

ctx = rgs.Context(0)
CASES = [tuple(int(v) for v in c.split('x')) for c in os.environ.get('CASES', '300000x2560x1440,2000000x1352x1014,1000000x1920x1080').split(',')]
for n, w, h in CASES:
    store = scenes.synthetic_scene(n, w, h, seed=int(os.environ.get("SEED", "5")))
    scene = rgs.DeviceScene.from_store(ctx, store)
    cams = scenes.orbit_cameras(w, h, 8, 8) if os.environ.get('ORBIT') == '1' else scenes.sweep_cameras(w, h, 48)
    out = torch.empty((len(cams), h, w, 3), dtype=torch.float32, device="cuda")
    ctx.render_views(scene, cams, out=out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        ctx.render_views(scene, cams, out=out)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"n={n} {w}x{h}: {len(cams) / best:.1f} FPS", flush=True)
    scene.close()
    del out
