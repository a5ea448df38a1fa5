import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
from paper_2402_03307_b200 import rgs, scenes
import oracle
ctx = rgs.Context(0, use_torch_stream=False)
st = scenes.random_scene(60, sh_degree=0, seed=0)
cam = scenes.bench_camera(64, 64, 0.3, scenes.yaw_pose(0.0, (0.05, -0.02, 0.1))); cam.fx = cam.fy = 64.0
out = rgs.render_forward(st, cam, rgs.RenderOptions(retain_records=True), ctx=ctx)
_, ref = oracle.restatement().render_forward(st, cam, retain=True)
print("pairs", out.records.n_pairs, len(ref.tile_ids))
print("offs", out.records.tile_offsets[:20]); print("ref ", ref.tile_offsets[:20])
print("ids", out.records.tile_ids[:30]); print("ref", ref.tile_ids[:30])
