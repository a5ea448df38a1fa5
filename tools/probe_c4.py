"""Diagnostic: per-stage times of C4 frames (2M Gaussians, 3840x2160), serialised."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_03307_b200 import rgs, scenes  # noqa: E402

ctx = rgs.Context(0)
store = scenes.synthetic_scene(bench.C4_N, bench.C4_W, bench.C4_H, seed=bench.C4_SEED)
cams = scenes.orbit_cameras(bench.C4_W, bench.C4_H, 8, 8)[::8]
scene = rgs.DeviceScene.from_store(ctx, store)
out = torch.empty((len(cams), bench.C4_H, bench.C4_W, 3), dtype=torch.float32, device="cuda")
ctx.render_views(scene, cams, out=out)
ctx.set_profiling(timing=True, count_evals=False)
ctx.profile_reset()
ctx.render_views(scene, cams, out=out)
torch.cuda.synchronize()
stages, _ = ctx.profile_read()
ctx.set_profiling(False, False)
n = len(cams)
print(f"{n} views, serialised ms per frame: total %.3f" % (sum(v[0] for v in stages.values()) / n))
for k, (ms, c) in sorted(stages.items(), key=lambda kv: -kv[1][0]):
    if c:
        print(f"  {k:24s} {ms / n:7.3f}")
img, rec = ctx.render_forward_device(scene, cams[0], retain=False)
print("pairs", rec.n_pairs, "visible", rec._n_splats, "slow", rec.n_slow_pixels)
ctx.set_profiling(timing=False, count_evals=True)
ctx.profile_reset()
ctx.render_views(scene, cams, out=out)
torch.cuda.synchronize()
_, (E, B, Ek) = ctx.profile_read()
ctx.set_profiling(False, False)
k5 = stages["blend_fp32_k5"][0] / n
flop = (16 * E + 10 * B) / n
print(f"K5 at 4K: {k5:.3f} ms, {flop / 1e9:.2f} GFLOP/frame, {flop / (k5 * 1e-3) / 1e12:.1f} TFLOP/s, frac {flop / (k5 * 1e-3) / 72.4e12:.3f}")
