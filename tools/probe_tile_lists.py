"""Tile-list length distribution at the benchmarked configurations (sizing the per-tile sort)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_03307_b200 import rgs, scenes

ctx = rgs.Context(0, use_torch_stream=False)
cases = [
    ("C2 t=0", scenes.synthetic_scene(300_000, 1352, 1014, seed=2), [scenes.bench_camera(1352, 1014, t, scenes.yaw_pose(7.0, (0.05, -0.02, 0.1))) for t in (0.0, 0.5, 1.0)]),
    ("C3", scenes.synthetic_scene(200_000, 800, 800, seed=3), [scenes.bench_camera(800, 800, 0.5)]),
    ("C4", scenes.synthetic_scene(2_000_000, 3840, 2160, seed=4), scenes.orbit_cameras(3840, 2160, 8, 8)[::9]),
]
for name, store, cams in cases:
    for cam in cams:
        out = rgs.render_forward(store, cam, rgs.RenderOptions(retain_records=True), ctx=ctx)
        off = np.asarray(out.records.tile_offsets)
        n = np.diff(off)
        pct = np.percentile(n, [50, 90, 99, 99.9, 100])
        print(f"{name} t={cam.time:.2f}: tiles={len(n)} pairs={off[-1]} mean={n.mean():.0f} p50/90/99/99.9/max={pct.astype(int).tolist()}"
              f" >2048: {(n > 2048).sum()} >4096: {(n > 4096).sum()} >8192: {(n > 8192).sum()}", flush=True)
