#!/usr/bin/env python3
"""Benchmark: render FPS of the 4D-rotor splatting hot path on B200 (BASELINE.json).

Workload (N=1): config C2 — 300K synthetic 4D Gaussians (SH degree 3), a
1352x1014 Plenoptic-shaped camera, a 300-timestamp forward-render sweep.
One "step" = one full sweep (300 frames).  `value` = frames/s over the K timed
sweeps with the scene already resident in HBM; `e2e` = the same sweep through
the C-ABI host-buffer entry point (rgs_render_views_host): scene H2D from pinned
memory, 300 renders, every image D2H into pinned memory, inside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): each rank renders its own 300-frame
sweep (distinct camera x timestamp views) with no data-path collective ->
"scaling": "weak"; the timed region is bracketed by a barrier and the time is
the max over ranks.  --impl reference times the reference's CPU render path
(oracle/_ref: the reference sources compiled in place; else the oracle port) on
the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W, H, N_GAUSS, N_TIMES, SEED = 1352, 1014, 300_000, 300, 2
METRIC = "render FPS at 1352×1014 (300K 4D Gaussians)"
WORKLOAD = "C2: 300K 4D rotor Gaussians, SH deg 3, 1352x1014, 300-timestamp forward-render sweep"
L2_FLUSH_BYTES = 256 << 20

# Training leg (config C3, reported under "train"): D-NeRF-shaped 800x800, 200K Gaussians,
# TrainConfig's default batch of 3 camera x timestamp views per step and rank.
TRAIN_N, TRAIN_W, TRAIN_H, TRAIN_BATCH, TRAIN_SEED, TRAIN_VIEWS = 200_000, 800, 800, 3, 3, 24
# Training legs resume a run at step 3000 of 6000, i.e. after the last SH unlock
# (active degree min(3, (step - 1) // sh_unlock_interval) = 3, trainer.cpp:135): every
# warm-up and timed step computes and updates all 48 SH coefficients.
TRAIN_START_STEP, TRAIN_TOTAL_STEPS = 3000, 6000
TRAIN_WORKLOAD = ("C3: 200K 4D rotor Gaussians, SH deg 3, 800x800, batch of 3 camera x timestamp views per rank "
                  "and step: render fwd + L1/SSIM image gradient + render bwd + batch all-reduce + entropy + "
                  "consistency (exact 4D KNN, k=8) + accumulate_stats + Adam")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="one warm sweep, no JSON (for ncu)")
    ap.add_argument("--no-train", action="store_true", help="skip the C3 training leg")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 4K batch leg")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 1M-Gaussian training leg")
    ap.add_argument("--train-only", action="store_true", help="only the C3 training leg (profiling)")
    ap.add_argument("--train-steps", type=int, default=10)
    ap.add_argument("--no-dropin", action="store_true", help="skip the drop-in (reference trainer.cpp) leg")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def replicate_scene(ctx, store, dist, rank, world, dev):
    """The scene replica of every rank: on one rank an upload; on N ranks
    rank 0 uploads and the device parameter buffer is broadcast (NCCL over NVLink), timed and
    reported (setup, outside the timed region)."""
    import torch

    from paper_2402_03307_b200 import rgs

    if dist is None or world == 1:
        return rgs.DeviceScene.from_store(ctx, store), None
    scene = rgs.DeviceScene(ctx, store.size(), store.active_sh_degree)
    if rank == 0:
        scene.upload(store)
    ctx.synchronize()
    buf = scene.params_tensor()
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    dist.broadcast(buf, src=0)
    torch.cuda.synchronize(dev)
    ms = 1e3 * max_over_ranks(time.perf_counter() - t0, dist, dev)
    return scene, {"bytes": buf.numel() * buf.element_size(), "ms": ms, "collective": "broadcast from rank 0"}


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank time over all ranks (the multi-GPU timing rule)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sweep_for_rank(rank):
    from paper_2402_03307_b200 import scenes

    # rank 0: identity pose (criterion-10 camera); other ranks: distinct yaw -> distinct views
    pose = scenes.yaw_pose(2.0 * rank, (0.0, 0.0, 0.0))
    return scenes.sweep_cameras(W, H, N_TIMES, pose)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU reference
def cpu_reference_lib():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    if oracle.reference_available():
        return oracle.reference_build(), "reference"
    return oracle.restatement(), "port"


def cpu_frames(store, cams, lib, threads):
    t0 = time.perf_counter()
    for c in cams:
        lib.render_forward(store, c, (0.0, 0.0, 0.0), threads=threads, retain=False)
    return time.perf_counter() - t0


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU render path on the host cores (rank 0 only)."""
    if rank != 0:
        return
    from paper_2402_03307_b200 import scenes

    lib, kind = cpu_reference_lib()
    threads = os.cpu_count() or 1
    store = scenes.synthetic_scene(N_GAUSS, W, H, seed=SEED)
    cams = sweep_for_rank(0)
    picks = np.linspace(0, N_TIMES - 1, args.warmup + args.steps).astype(int)
    for k in range(args.warmup):
        cpu_frames(store, [cams[picks[k]]], lib, threads)
    t = cpu_frames(store, [cams[i] for i in picks[args.warmup:]], lib, threads)
    fps = args.steps / t
    sample = (f"{args.steps} frames of the 300-timestamp sweep (t index {list(map(int, picks[args.warmup:]))}), "
              f"one frame per step, full 1352x1014, {threads} threads ({cpu_model()})")
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD + " (CPU: one frame per step)", "n_gaussians": N_GAUSS, "width": W,
                   "height": H, "timestamps": N_TIMES, "sh_degree": 3},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- C4 batch leg
C4_N, C4_W, C4_H, C4_SEED, C4_VIEWS = 2_000_000, 3840, 2160, 4, 64


def run_c4_leg(args, ctx, dev, dist, rank, world, flush):
    """Config C4: 2M Gaussians, 3840x2160, a 64-view camera x timestamp batch (8 orbit yaws x 8
    times) sharded across the ranks ("strong" scaling: the batch is fixed as N grows)."""
    import torch

    from paper_2402_03307_b200 import rgs, scenes

    store = scenes.synthetic_scene(C4_N, C4_W, C4_H, seed=C4_SEED)
    cams_all = scenes.orbit_cameras(C4_W, C4_H, 8, 8)
    lo, hi = rank * C4_VIEWS // world, (rank + 1) * C4_VIEWS // world
    cams = cams_all[lo:hi]
    scene, bcast = replicate_scene(ctx, store, dist, rank, world, dev)
    images = torch.empty((len(cams), C4_H, C4_W, 3), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    ctx.render_views(scene, cams, (0.0, 0.0, 0.0), out=images)  # warm-up (also sizes the pair buffers)
    steps = 2
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    total = 0.0
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.render_views(scene, cams, (0.0, 0.0, 0.0), out=images)
        b.record(stream)
        torch.cuda.synchronize(dev)
        total += a.elapsed_time(b)
    ms = max_over_ranks(total, dist, dev)
    _, rec = ctx.render_forward_device(scene, cams[len(cams) // 2], retain=False)
    n_pairs, n_vis = rec.n_pairs, rec._n_splats
    rec.close()
    del images
    scene.close()
    torch.cuda.empty_cache()
    return {"metric": "batch FPS at 3840x2160 (2M 4D Gaussians, 64-view batch)", "value": C4_VIEWS * steps / (ms / 1e3),
            "unit": "frames/s", "scaling": "strong", "n_gpus": world, "views_per_rank": len(cams), "steps": steps,
            "ms_per_batch": ms / steps, "scene_broadcast": bcast,
            "config": {"workload": "C4: 2M 4D rotor Gaussians, SH deg 3, 3840x2160, 64 views = 8 orbit yaws x 8 "
                                   "timestamps, views sharded contiguously across ranks",
                       "n_gaussians": C4_N, "width": C4_W, "height": C4_H, "n_pairs_mid_view": n_pairs,
                       "n_visible_mid_view": n_vis, "l2": "256 MiB flush before each timed batch"}}


# ----------------------------------------------------------------------------- C5 training leg
C5_N, C5_W, C5_H, C5_SEED, C5_VIEWS = 1_000_000, 1352, 1014, 5, 8


def run_c5_leg(args, ctx, dev, dist, rank, world, flush):
    """Config C5: multi-view training, 1M Gaussians, an 8-view batch per rank, the batch reduced
    with one NCCL all-reduce per step (replicated scene, weak scaling in views)."""
    import torch

    from paper_2402_03307_b200 import rgs, scenes, train

    truth = scenes.synthetic_scene(C5_N, C5_W, C5_H, seed=C5_SEED)
    store = scenes.perturbed(truth, C5_SEED)
    cams = [scenes.bench_camera(C5_W, C5_H, (v + 0.5) / C5_VIEWS,
                                scenes.yaw_pose(-4.0 + 8.0 * v / (C5_VIEWS - 1) + 0.7 * rank, (0.02, 0.0, 0.03)))
            for v in range(C5_VIEWS)]
    tsc = rgs.DeviceScene.from_store(ctx, truth)
    targets = torch.empty((C5_VIEWS, C5_H, C5_W, 3), dtype=torch.float32, device=dev)
    ctx.render_views(tsc, cams, (0.0, 0.0, 0.0), out=targets)
    tsc.close()
    del truth
    scene = rgs.DeviceScene.from_store(ctx, store)
    comm = native_comm(ctx, dist, world)
    tr = train.Trainer(ctx, scene, train.TrainConfig(batch=C5_VIEWS, total_steps=TRAIN_TOTAL_STEPS,
                                                     max_gaussians=2_000_000), dist, start_step=TRAIN_START_STEP,
                       comm=comm)
    tlist = [targets[v] for v in range(C5_VIEWS)]
    for _ in range(2):
        tr.step(cams, tlist)
    stream = torch.cuda.current_stream(dev)
    steps = 5
    first_timed = tr.step_count + 1
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        tr.step(cams, tlist, read=False)
    b.record(stream)
    torch.cuda.synchronize(dev)
    last = tr.last_losses()
    sh_timed = tr.scene.sh_degree
    ms = max_over_ranks(a.elapsed_time(b), dist, dev)
    its = steps / (ms / 1e3)
    out = {"metric": "train it/s (C5)", "value": its, "unit": "it/s", "n_gpus": world, "steps": steps,
           "ms_per_step": ms / steps, "views_per_step": C5_VIEWS * world, "views_per_s": its * C5_VIEWS * world,
           "scaling": "weak",
           "allreduce_bytes_per_step": (66 * C5_N + C5_N) * 4 + 3 * 8 if world > 1 else 0,
           "loss_last": last.total,
           "config": {"workload": "C5: 1M 4D rotor Gaussians, SH deg 3, 1352x1014, 8 camera x timestamp views per rank "
                                  "and step, full training step, batch reduced by NCCL all-reduce",
                      "n_gaussians": C5_N, "width": C5_W, "height": C5_H, "views_per_rank": C5_VIEWS,
                      "active_sh_degree": sh_timed, "first_timed_step": first_timed,
                      "allreduce": allreduce_kind(world)}}
    tr = None
    scene.close()
    del targets, tlist
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- training leg
def train_views(rank):
    """TRAIN_VIEWS camera x timestamp views of rank `rank` (8 yaws x 3 times; distinct per rank)."""
    from paper_2402_03307_b200 import scenes

    cams = []
    for v in range(TRAIN_VIEWS):
        yaw = -6.0 + 12.0 * (v % 8) / 7 + 1.0 * rank
        t = (v // 8 + 0.5) / 3
        cams.append(scenes.bench_camera(TRAIN_W, TRAIN_H, t, scenes.yaw_pose(yaw, (0.02 * (v % 3), 0.0, 0.03))))
    return cams


def train_case():
    """Ground-truth C3 scene (targets) and the perturbed copy that is trained."""
    from paper_2402_03307_b200 import scenes

    truth = scenes.synthetic_scene(TRAIN_N, TRAIN_W, TRAIN_H, seed=TRAIN_SEED)
    store = scenes.perturbed(truth, TRAIN_SEED, opacity_sigma=0.2)
    return truth, store


def native_comm(ctx, dist, world):
    """RGS_NATIVE_ALLREDUCE=1 (N > 1): the batch all-reduce through the C ABI's fused NCCL group
    (rgs_allreduce_grads) instead of three torch.distributed collectives."""
    from paper_2402_03307_b200 import train

    if dist is None or world < 2 or os.environ.get("RGS_NATIVE_ALLREDUCE") != "1":
        return None
    return train.NcclComm(ctx, dist)


def allreduce_kind(world):
    if world < 2:
        return "none (one rank)"
    if os.environ.get("RGS_NATIVE_ALLREDUCE") == "1":
        return "rgs_allreduce_grads: one NCCL group (grads|vnorm, visible, image losses) on the context stream"
    import torch.distributed as dist

    return f"torch.distributed {dist.get_backend()} all-reduce x3 (grads|vnorm, visible, image losses)"


def measured_peaks(ctx):
    """Roofline denominators: HBM from MEASURED_PEAKS.json (driver-measured copy bandwidth),
    FP32 / FP64 FMA from the bench's own probes (MEASURED_PEAKS.json has neither)."""
    if not hasattr(measured_peaks, "cache"):
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback 6.65 TB/s"
        measured_peaks.cache = {"hbm_gbs": hbm, "hbm_source": src, "fp32_tflops": ctx.measure_fp32_tflops(),
                                "fp64_tflops": ctx.measure_fp64_tflops()}
    return measured_peaks.cache


# FP64 FLOPs per valid SSIM position of the image-loss pair K8a + K8b, counted from
# csrc/k_train.cu (FMA = 2; reference summation order, so no fused forms): K8a's two separable
# 11-tap passes over the five moment fields of 3 channels (2 x 11 x 2 x 5 x 3 = 660) plus the
# SSIM map and its three adjoint seeds (~40 x 3); K8b's three adjoint convolutions gathered over
# the 11 x 11 window as two separable passes (2 x 11 x 2 x 3 x 3 = 396) plus the gradient
# assembly (~15 x 3).
K8_FLOP_PER_POS = 660 + 120 + 396 + 45


def train_rooflines(ctx, tr, cams, stage_ms):
    """Roofline of every training kernel over one C3 step (SURVEY.md §8(d) work counts).

    Stage times: `stage_ms` (serialised step, CUDA events per stage).  Workload counts (E, B,
    E_b, visible splats, pairs): the step's views re-rendered with the eval counters on (the
    scene after that step -- one Adam update later)."""
    peaks = measured_peaks(ctx)
    ctx.set_profiling(timing=False, count_evals=True)
    ctx.profile_reset()
    e_b = n_vis = n_pairs = 0
    for cam in cams:
        _, rec = ctx.render_forward_device(tr.scene, cam, (0.0, 0.0, 0.0), retain=True)
        e_b += int(rec.n_contrib.astype(np.int64).sum())  # E_b: evaluations in [0, contrib)
        n_vis += rec._n_splats
        n_pairs += rec.n_pairs
        rec.close()
    _, (E, B, E_k) = ctx.profile_read()
    ctx.set_profiling(False, False)
    n = tr.scene.n
    px = sum(c.width * c.height for c in cams)
    pos = sum(max(c.width - 10, 0) * max(c.height - 10, 0) for c in cams)
    k = tr.cfg.loss.k_neighbors
    fp32, fp64, hbm = peaks["fp32_tflops"], peaks["fp64_tflops"], peaks["hbm_gbs"]
    # stage: (bound, algorithmic work of the step in GB or TFLOP, peak, definition)
    spec = {
        "backward_tiles_k6": ("fp32", (16 * e_b + 60 * B) / 1e12, fp32, "16 E_b + 60 B FLOP (E_b = sum of n_contrib)"),
        "blend_fp32_k5": ("fp32", (16 * E + 10 * B) / 1e12, fp32, "16 E + 10 B FLOP"),
        "preprocess_k1": ("hbm", (260 * n * len(cams) + 48 * n_vis) / 1e9, hbm, "260 N + 48 N_vis B per view"),
        "backward_color_k7a": ("hbm", (248 + 216) * n_vis / 1e9, hbm,
                               "SH 192 + view dir 32 + colour grads 24 B read, SH grads 192 + d mean3 24 B written "
                               "per visible splat"),
        "backward_gauss_k7b": ("hbm", (260 * n_vis + 268 * n_vis - (248 + 216) * n_vis) / 1e9, hbm,
                               "the rest of SURVEY's 260 + 268 B per visible splat"),
        "image_loss_k8": ("fp64", K8_FLOP_PER_POS * pos / 1e12, fp64,
                          f"{K8_FLOP_PER_POS} FP64 FLOP per valid SSIM position (counted from k_train.cu)"),
        "adam_k9": ("hbm", 1828 * n / 1e9, hbm, "1828 B per Gaussian (65 x (4 grad + 24 param/m/v) + 8)"),
        "consistency_k10": ("hbm", (260 * n + 24 * n * (k + 2)) / 1e9, hbm, "260 N + 24 N (k + 2) B"),
        "tile_radix_sort_k4": ("hbm", 2 * 20 * n_pairs / 1e9, hbm, "2 passes x 20 B per pair"),
        "tile_scatter_k4": ("hbm", (4 * n_pairs + 16 * n_vis) / 1e9, hbm,
                            "16 B per visible splat read, 4 B per pair written"),
    }
    kernels = {}
    for name, (bound, work, peak, what) in spec.items():
        ms = stage_ms.get(name)
        if not ms:
            continue
        ach = work / (ms / 1e3)
        kernels[name] = {"bound": "fp64" if bound == "fp64" else bound, "achieved": ach, "peak": peak,
                         "unit": "GB/s" if bound == "hbm" else "TFLOP/s", "frac": ach / peak, "ms_per_step": ms,
                         "work": what}
    dominant = max(kernels, key=lambda k: kernels[k]["ms_per_step"]) if kernels else None
    roof = dict(kernels.get(dominant, {}), kernel=dominant, traffic=None,
                timing="serialised step (one stage at a time), CUDA events on the launching stream",
                peak_source={"hbm": peaks["hbm_source"], "fp32": "bench FFMA probe", "fp64": "bench DFMA probe"})
    counts = {"E": E, "B": B, "E_kernel": E_k, "E_b": e_b, "visible_splats": n_vis, "pairs": n_pairs,
              "views": len(cams), "fp32_peak_tflops": fp32, "fp64_peak_tflops": fp64}
    return {"roofline": roof, "kernels": kernels, "counts": counts}


def f64_scene_its(ctx, store, cfg, batch, args, dist, dev, steps=5):
    """Training it/s of the C3 step on an FP64 device scene (the store's doubles and FP64 Adam
    moments, as the reference keeps them)."""
    import torch

    from paper_2402_03307_b200 import rgs, train

    sc = rgs.DeviceScene.from_store(ctx, store, f64=True)
    tr = train.Trainer(ctx, sc, cfg, dist, start_step=TRAIN_START_STEP)
    for k in range(2):
        tr.step(*batch(k))
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for k in range(steps):
        tr.step(*batch(2 + k), read=False)
    b.record(stream)
    torch.cuda.synchronize(dev)
    tr.last_losses()
    its = steps / (max_over_ranks(a.elapsed_time(b), dist, dev) / 1e3)
    tr = None
    sc.close()
    return its


def backward_mode_times(ctx, tr, cams, targets, reps=5):
    """One C3 view's render backward (K6 + FP64 fix-up + K7) in the three accumulation modes, CUDA
    events on the launching stream: FP64 atomics (production), RGS_FLAG_REPRODUCIBLE, and
    RGS_FLAG_DETERMINISTIC (the reference-order FP64 replay, per tile and per splat)."""
    import torch

    from paper_2402_03307_b200 import train

    cam, tgt = cams[0], targets[0]
    img, rec = ctx.render_forward_device(tr.scene, cam, retain=True)
    dl = torch.zeros_like(img)
    train.image_loss(ctx, img, tgt, 0.8 / 3, 0.2 / 3, dl, records=rec)
    stream = torch.cuda.current_stream()
    out = {}
    for name, kw in (("atomic", {}), ("reproducible", {"reproducible": True}),
                     ("deterministic_fp64", {"deterministic": True})):
        ctx.render_backward_device(tr.scene, cam, rec, dl, **kw)  # warm
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            ctx.render_backward_device(tr.scene, cam, rec, dl, **kw)
        b.record(stream)
        torch.cuda.synchronize()
        out[name] = a.elapsed_time(b) / reps
    rec.close()
    return out


DROPIN_SO = os.path.join(ROOT, "tests", "cpp", "_build", "librgs_ref_dropin.so")


def dropin_leg(store, cams, targets64, nbrs, k, steps=4):
    """The reference's own training step (trainer.cpp evaluate_loss + accumulate_stats +
    adam_step, unmodified) compiled against the C++ drop-ins (tests/cpp/Makefile): host
    GaussianStore in, every render / image loss / optimizer call on the device through the C ABI
    -- what a maintainer of the reference gets by swapping the sources.  The
    first step is a warm-up (context, first scene upload)."""
    import ctypes

    if not os.path.exists(DROPIN_SO):
        return {"unavailable": "tests/cpp/_build/librgs_ref_dropin.so not built (needs /root/reference at build time)"}
    L = ctypes.CDLL(DROPIN_SO)

    class Cam(ctypes.Structure):
        _fields_ = [("width", ctypes.c_int), ("height", ctypes.c_int), ("fx", ctypes.c_double),
                    ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                    ("world_to_camera", ctypes.c_double * 16), ("time", ctypes.c_double)]

    arr = [np.ascontiguousarray(a, dtype=np.float64) for a in store.arrays_f64()]
    cs = (Cam * len(cams))(*[Cam(c.width, c.height, c.fx, c.fy, c.cx, c.cy,
                                 (ctypes.c_double * 16)(*np.asarray(c.world_to_camera, np.float64).reshape(-1)),
                                 c.time) for c in cams])
    tg = np.ascontiguousarray(np.concatenate([t.reshape(-1) for t in targets64]))
    nb = np.ascontiguousarray(nbrs, dtype=np.int32) if nbrs is not None else None
    losses = np.zeros(5)
    secs = np.zeros(steps)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p) if a is not None else None  # noqa: E731
    rc = L.dropin_train_steps(ctypes.c_int(store.size()), *[p(a) for a in arr], ctypes.c_int(store.active_sh_degree),
                              ctypes.c_int(len(cams)), cs, p(tg), p(nb), ctypes.c_int(k),
                              ctypes.c_int(TRAIN_START_STEP + 1), ctypes.c_int(TRAIN_TOTAL_STEPS), ctypes.c_int(steps),
                              p(losses), p(secs))
    if rc != 0:
        return {"unavailable": "dropin_train_steps failed"}
    prof = np.zeros(10)
    L.dropin_profile_step(ctypes.c_int(store.size()), *[p(a) for a in arr], ctypes.c_int(store.active_sh_degree),
                          ctypes.c_int(len(cams)), cs, p(tg), p(nb), ctypes.c_int(k),
                          ctypes.c_int(TRAIN_START_STEP + 1), p(prof))
    parts = ["render_forward", "l1_loss(+backward)", "ssim_loss_with_grad", "dL/dimage assembly", "render_backward",
             "StoreGrads::add", "entropy", "consistency (host slice loops + consistency_loss)", "accumulate_stats",
             "adam_step"]
    stats = (ctypes.c_longlong * 5)()
    L.rgs_adapter_stats(ctypes.byref(stats, 0), ctypes.byref(stats, 8), ctypes.byref(stats, 16))
    L.rgs_train_adapter_stats(ctypes.byref(stats, 24), ctypes.byref(stats, 32))
    timed = secs[1:]
    return {"value": 1.0 / float(np.median(timed)), "unit": "it/s", "step_ms": [1e3 * x for x in secs],
            "statistic": f"median of {len(timed)} steps after one warm-up", "loss_last": float(losses[4]),
            "scene_uploads": int(stats[0]), "scene_cache_hits": int(stats[1]), "backward_records_reused": int(stats[2]),
            "optimizer_store_uploads": int(stats[3]), "optimizer_store_reuses": int(stats[4]),
            "step_breakdown_ms": {k: 1e3 * float(v) for k, v in zip(parts, prof)},
            "note": "the reference's evaluate_loss + accumulate_stats + adam_step (trainer.cpp:134-150) on its host "
                    "GaussianStore, compiled against host/rgs_adapter.cpp + host/rgs_train_adapter.cpp: renders, "
                    "image losses and Adam on the device; the store crosses PCIe where the reference API hands it "
                    "over (adam_step each step; renders reuse the cached device scene until it changes)"}


def run_train_leg(args, ctx, dev, dist, rank, world, flush):
    import torch

    from paper_2402_03307_b200 import rgs, train

    truth, store = train_case()
    cams = train_views(rank)
    tsc = rgs.DeviceScene.from_store(ctx, truth)
    targets = torch.empty((TRAIN_VIEWS, TRAIN_H, TRAIN_W, 3), dtype=torch.float32, device=dev)
    ctx.render_views(tsc, cams, (0.0, 0.0, 0.0), out=targets)
    tsc.close()
    scene = rgs.DeviceScene.from_store(ctx, store)
    cfg = train.TrainConfig(batch=TRAIN_BATCH, total_steps=TRAIN_TOTAL_STEPS)
    # The timed steps are past the last SH unlock (trainer.cpp:135): active SH degree 3.
    comm = native_comm(ctx, dist, world)
    tr = train.Trainer(ctx, scene, cfg, dist, start_step=TRAIN_START_STEP, comm=comm)
    stream = torch.cuda.current_stream(dev)
    B = TRAIN_BATCH

    def batch(k):
        idx = [(k * B + j) % TRAIN_VIEWS for j in range(B)]
        return [cams[i] for i in idx], [targets[i] for i in idx]

    first = None
    for k in range(max(args.warmup, 1)):
        c, t = batch(k)
        lb = tr.step(c, t)
        first = first or lb
    knn0 = time.perf_counter()
    tr.rebuild_knn()
    torch.cuda.synchronize(dev)
    knn_ms = 1e3 * (time.perf_counter() - knn0)
    launches0 = ctx.kernel_launches
    first_timed = tr.step_count + 1
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for k in range(args.train_steps):
        c, t = batch(args.warmup + k)
        tr.step(c, t, read=False)  # device-resident leg: losses queued, read after the region
    b.record(stream)
    torch.cuda.synchronize(dev)
    last = tr.last_losses()
    ms = max_over_ranks(a.elapsed_time(b), dist, dev)
    launches = ctx.kernel_launches - launches0
    its = args.train_steps / (ms / 1e3)

    # the same steps with the bitwise-reproducible backward (RGS_FLAG_REPRODUCIBLE)
    tr.reproducible = True
    tr.step(*batch(0))
    torch.cuda.synchronize(dev)
    a2 = torch.cuda.Event(enable_timing=True)
    b2 = torch.cuda.Event(enable_timing=True)
    a2.record(stream)
    for k in range(args.train_steps):
        tr.step(*batch(args.warmup + k), read=False)
    b2.record(stream)
    torch.cuda.synchronize(dev)
    tr.last_losses()
    tr.reproducible = False
    repro_its = args.train_steps / (max_over_ranks(a2.elapsed_time(b2), dist, dev) / 1e3)
    backward_modes = backward_mode_times(ctx, tr, *batch(0))
    f64_its = f64_scene_its(ctx, store, cfg, batch, args, dist, dev)

    # per-stage breakdown of one step (serialised CUDA events on the launching stream)
    ctx.set_profiling(timing=True, count_evals=False)
    ctx.profile_reset()
    c, t = batch(0)
    tr.overlap = False  # serialised: each stage's own time
    tr.step(c, t)
    tr.overlap = True
    stages, _ = ctx.profile_read()
    ctx.set_profiling(False, False)
    stage_ms = {k: v[0] for k, v in stages.items() if v[1]}
    train_roof = train_rooflines(ctx, tr, c, stage_ms)

    # e2e: the same steps through the public API with each step's target images copied
    # H2D from pinned host memory and the loss scalars read back (Trainer.step's D2H).
    host_t = targets.cpu().pin_memory()
    stager = train.TargetStager(dev, B, TRAIN_H, TRAIN_W)
    views = lambda k: [(k * B + j) % TRAIN_VIEWS for j in range(B)]  # noqa: E731
    if dist:
        dist.barrier()
    e2e_steps = 3 * args.train_steps  # steady state: the pipeline's fill and drain are ~2 steps
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    stager.put([host_t[i] for i in views(0)])
    e2e_losses = []
    for k in range(e2e_steps):
        tg = stager.take()
        if k + 1 < e2e_steps:  # the next step's targets cross PCIe during this step
            stager.put([host_t[i] for i in views(k + 1)])
        tr.step([cams[i] for i in views(k)], tg, read=False)
        stager.release(ctx)
        if k > 0:  # step k-1's losses reach the host while step k runs
            e2e_losses.append(tr.pop_losses().total)
    e2e_losses.append(tr.pop_losses().total)
    torch.cuda.synchronize(dev)
    e2e_s = max_over_ranks(time.perf_counter() - t0, dist, dev)
    assert len(e2e_losses) == e2e_steps and all(np.isfinite(e2e_losses))
    e2e = {"value": e2e_steps / e2e_s, "unit": "it/s", "h2d_bytes_per_step": int(B * TRAIN_H * TRAIN_W * 12),
           "d2h_bytes_per_step": 64 + 8, "steps": e2e_steps,
           "note": "Trainer.step with the batch's target images H2D from pinned host memory each step "
                   "(train.TargetStager: step k+1's copy overlaps step k) and every step's loss scalars "
                   "and rotor-error word D2H, read on the host one step behind (Trainer.pop_losses)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle

        ops = oracle.train_ops("ref" if oracle.reference_available() else "orc")
        threads = os.cpu_count() or 1
        c, t = batch(0)
        tg = [x.cpu().numpy().astype(np.float64) for x in t]
        w = oracle.loss_weights()
        # the same neighbour lists the GPU step uses (the KNN is rebuilt every 100 steps on both
        # sides, so it is outside the per-step cost), the same SH degree (3)
        nbrs = tr.nbrs.cpu().numpy() if tr.nbrs is not None else None
        assert store.active_sh_degree == tr.scene.sh_degree == 3
        t0 = time.perf_counter()
        L, g, vn, vis = ops.evaluate_loss(store, c, tg, w, (0.0, 0.0, 0.0), nbrs, threads=threads)
        n = store.size()
        ops.adam_step(store, np.zeros((n, 65)), np.zeros((n, 65)), g,
                      oracle.adam_config(total_steps=TRAIN_TOTAL_STEPS), TRAIN_START_STEP + 1)
        cpu_s = time.perf_counter() - t0
        cpu = {"value": 1.0 / cpu_s, "unit": "it/s", "cores": threads,
               "kind": "reference" if ops.ref else "port",
               "sample": f"1 training step at active SH degree 3: the reference's evaluate_loss over {B} views "
                         f"(render fwd, L1 + SSIM, render bwd, entropy, consistency with k={w.k_neighbors} "
                         f"neighbours) + adam_step, {threads} threads, {cpu_model()}; omits accumulate_stats "
                         f"(O(N) adds)"}
    dropin = None
    if rank == 0 and world == 1 and not args.no_dropin:
        c, t = batch(0)
        dropin = dropin_leg(store, c, [x.cpu().numpy().astype(np.float64) for x in t],
                            tr.nbrs.cpu().numpy() if tr.nbrs is not None else None, tr.cfg.loss.k_neighbors)
    return {
        "metric": "train it/s", "value": its, "unit": "it/s", "ms_per_step": ms / args.train_steps,
        "steps": args.train_steps, "warmup": max(args.warmup, 1), "n_gpus": world,
        "views_per_step": B * world,
        "config": {"workload": TRAIN_WORKLOAD, "n_gaussians": TRAIN_N, "width": TRAIN_W, "height": TRAIN_H,
                   "batch_per_rank": B, "active_sh_degree": tr.scene.sh_degree, "first_timed_step": first_timed,
                   "allreduce": allreduce_kind(world),
                   "parallelism": f"dp{world}: replicated scene, NCCL all-reduce of "
                                                         "[65 grads | viewspace norm | visible | image losses]",
                   "l2": "256 MiB flush before the timed steps; per-step working set > L2"},
        "loss_first": first.total, "loss_last": last.total, "psnr_last": train.psnr_from_mse(last.mse),
        "knn_rebuild_ms": knn_ms, "stage_ms_one_step": stage_ms, "gpu_launches": launches,
        "roofline": train_roof["roofline"], "kernels": train_roof["kernels"], "workload_counts": train_roof["counts"],
        "reproducible": {"value": repro_its, "unit": "it/s", "steps": args.train_steps,
                         "note": "Trainer.reproducible: RGS_FLAG_REPRODUCIBLE backward (order-independent fixed-point "
                                 "screen-gradient sums) + integer-count consistency gradient: bitwise identical "
                                 "steps run to run"},
        "backward_modes_ms_one_view": backward_modes,
        "f64_scene": {"value": f64_its, "unit": "it/s",
                      "note": "the same step on an FP64 device scene (RGS_SCENE_F64: the reference's doubles "
                              "unrounded; parameters and Adam moments in FP64)"},
        "e2e": e2e, "cpu_baseline": cpu, "dropin": dropin,
    }


# ----------------------------------------------------------------------------- ours
def run_ours(args, rank, local_rank, world):
    import torch

    from paper_2402_03307_b200 import rgs, scenes

    # RGS_BENCH_SHARE_GPU=1 (test harness only): every rank on device 0 over gloo, to exercise
    # the multi-rank code paths on a one-GPU box.  The driver's runs use one GPU per rank + NCCL.
    shared = os.environ.get("RGS_BENCH_SHARE_GPU") == "1"
    dev_index = 0 if shared else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    ctx = rgs.Context(dev_index)
    if args.train_only:
        flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
        res = run_train_leg(args, ctx, dev, dist, rank, world, flush)
        if rank == 0:
            print(json.dumps({"train": res}), flush=True)
        if dist:
            dist.destroy_process_group()
        return
    store = scenes.synthetic_scene(N_GAUSS, W, H, seed=SEED)
    cams = sweep_for_rank(rank)
    scene = rgs.DeviceScene.from_store(ctx, store)
    images = torch.empty((N_TIMES, H, W, 3), dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def sweep():
        ctx.render_views(scene, cams, (0.0, 0.0, 0.0), out=images)

    if args.profile_only:
        for _ in range(max(args.warmup, 1)):
            sweep()
        sweep()
        torch.cuda.synchronize(dev)
        return
    # K5 is timed live (CUDA events around each blend on its own stream) through warm-up and
    # the timed region: the roofline's denominator is its duration inside the measured run
    ctx.set_profiling(timing="live", count_evals=False)
    for _ in range(max(args.warmup, args.steps, 1)):  # (also sizes the context's event pool)
        sweep()
    torch.cuda.synchronize(dev)
    ctx.profile_reset()

    # ---- timed region: K sweeps, L2 flushed between sweeps.  Views are pipelined over
    # eight streams inside each sweep; the CUDA events are on the torch current stream,
    # which the context joins every view stream back into.
    launches0 = ctx.kernel_launches
    sampler = ClockSampler(local_rank)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    evs = []
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sweep()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize(dev)
    t_wall = time.perf_counter() - t_wall
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    live, _ = ctx.profile_read()
    ctx.set_profiling(timing=False, count_evals=False)
    k5_live_ms, k5_live_n = live.get("blend_fp32_k5", (0.0, 0))
    launches = ctx.kernel_launches - launches0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    total_ms = max_over_ranks(total_ms, dist, dev)
    frames = N_TIMES * args.steps * world
    fps = frames / (total_ms / 1e3)

    # ---- per-stage breakdown: one more sweep with CUDA events around every stage on
    # its launching stream; profiling serialises the views, so each stage time is
    # that kernel's own duration (the roofline denominators below).
    ctx.set_profiling(timing=True, count_evals=False)
    ctx.profile_reset()
    torch.cuda.synchronize(dev)
    flush.zero_()
    sweep()
    torch.cuda.synchronize(dev)
    stages, _ = ctx.profile_read()
    ctx.set_profiling(timing=False, count_evals=False)

    # ---- the other binning (DESIGN.md §3 "Binning"): the batch uses the radix passes; the
    # tile-major scatter (the single-view default) measured on the same sweep -- serialised
    # stage times and one live sweep
    ctx.set_binning("scatter")
    ctx.set_profiling(timing=True, count_evals=False)
    ctx.profile_reset()
    torch.cuda.synchronize(dev)
    flush.zero_()
    sweep()
    torch.cuda.synchronize(dev)
    stages_sc, _ = ctx.profile_read()
    ctx.set_profiling(timing=False, count_evals=False)
    sc_ms = []
    for _ in range(2):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sweep()
        b.record(stream)
        torch.cuda.synchronize(dev)
        sc_ms.append(a.elapsed_time(b))
    ctx.set_binning("auto")

    # ---- workload counters (untimed extra sweep): E, B, splats, pairs
    ctx.set_profiling(timing=False, count_evals=True)
    ctx.profile_reset()
    sweep()
    _, (E, B, E_kernel) = ctx.profile_read()
    slow_reasons = ctx.slow_reasons()
    visits, visits_blend = ctx.blend_visits()
    ctx.set_profiling(False, False)
    img0, rec0 = ctx.render_forward_device(scene, cams[N_TIMES // 2], retain=False)
    n_vis, n_pairs, n_slow = rec0._n_splats, rec0.n_pairs, rec0.n_slow_pixels
    rec0.close()

    # ---- roofline of the dominant stage
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback 6.65 TB/s"
    fp32_peak = ctx.measure_fp32_tflops()
    n_frames_rank = N_TIMES  # the profiling sweep
    per_stage = {}
    for name, (ms, cnt) in stages.items():
        if cnt:
            per_stage[name] = {"ms_per_frame": ms / n_frames_rank, "share": ms / max(sum(v[0] for v in stages.values()), 1e-9)}
    # algorithmic work per frame: blend 16 E + 10 B FLOP; preprocess
    # 260 N read + 48 N_vis written; tile sort 2 passes x 16 B per pair.
    e_frame, b_frame = E / N_TIMES, B / N_TIMES
    kernels = {
        "blend_fp32_k5": ("fp32", (16 * e_frame + 10 * b_frame) / 1e12, "TFLOP/s", fp32_peak),
        "preprocess_k1": ("hbm", (260 * N_GAUSS + 48 * n_vis) / 1e9, "GB/s", hbm_peak),
        # duplicate: rect + id per splat in, (key, value) per pair out
        "duplicate_k3": ("hbm", (8 * n_pairs + 16 * n_vis) / 1e9, "GB/s", hbm_peak),
        # two LSD passes: histogram read 4 B, scatter read 8 B + write 8 B per pair
        "tile_radix_sort_k4": ("hbm", (2 * 20 * n_pairs) / 1e9, "GB/s", hbm_peak),
        # depth ranks: key 8 B read twice, (key, id) 12 B written and re-read, ids 8 B
        "depth_rank": ("hbm", (48 * n_vis) / 1e9, "GB/s", hbm_peak),
    }
    roof_all = {}
    for name, (bound, work, unit, peak) in kernels.items():
        if name in per_stage and per_stage[name]["ms_per_frame"] > 0:
            ach = work / (per_stage[name]["ms_per_frame"] / 1e3)
            roof_all[name] = {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                              "timing": "serialised profiling sweep"}
    if k5_live_n and "blend_fp32_k5" in roof_all:
        # the headline roofline: K5's average duration measured live over the timed region
        r = roof_all["blend_fp32_k5"]
        work = kernels["blend_fp32_k5"][1]
        live_ms = k5_live_ms / k5_live_n
        r.update({"achieved_serialised": r["achieved"], "frac_serialised": r["frac"],
                  # the K5 algorithmic work of the whole timed run over its wall time
                  "achieved_whole_run": work * fps / world, "frac_whole_run": work * fps / world / r["peak"],
                  "achieved": work / (live_ms / 1e3), "frac": work / (live_ms / 1e3) / r["peak"],
                  "ms_per_launch": live_ms, "ms_per_launch_serialised": per_stage["blend_fp32_k5"]["ms_per_frame"],
                  "timing": f"CUDA events around each of the {k5_live_n} K5 launches of the timed region, on "
                            "its own stream (views pipelined over 8 streams, so it shares the GPU)"})
    # binning, both ways (per frame, serialised; depth ranks included)
    def _bin(st, names):
        return {k: st[k][0] / n_frames_rank for k in names if k in st and st[k][1]}

    b_radix = _bin(stages, ("depth_rank", "pair_offsets_scan", "duplicate_k3", "tile_radix_sort_k4"))
    b_scat = _bin(stages_sc, ("depth_rank", "tile_counts", "tile_scatter_k4"))
    sc_fps = N_TIMES / (min(sc_ms) / 1e3)
    t_scat = b_scat.get("tile_scatter_k4", 0.0)
    binning = {
        "batch_uses": "radix (RGS_BINNING_AUTO)",
        "radix": {"stages_ms_per_frame": b_radix, "total_ms_per_frame": sum(b_radix.values()), "fps_live": fps},
        "scatter": {"stages_ms_per_frame": b_scat, "total_ms_per_frame": sum(b_scat.values()),
                    "fps_live": sc_fps,
                    # algorithmic bytes of the scatter kernel: rect + id + tile count per visible
                    # splat read, one 4-byte splat id per pair written
                    "tile_scatter_k4_hbm_frac": ((4 * n_pairs + 16 * n_vis) / (t_scat / 1e3)) / 1e9 / hbm_peak
                    if t_scat else None},
        "note": "same per-tile lists; the scatter has the shorter serialised path (single views: training, "
                "drop-in), the radix passes overlap the blends of the other views in flight better (batch)",
    }
    dominant = max(per_stage, key=lambda k: per_stage[k]["share"]) if per_stage else None
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(dominant)
    except Exception:
        pass
    roofline = dict(roof_all.get(dominant, {}), kernel=dominant, traffic=traffic,
                    peak_source=("bench FFMA probe (rgs_measure_fp32_tflops)" if dominant == "blend_fp32_k5"
                                 else hbm_src))

    # ---- e2e through the host-buffer C-ABI entry point
    e2e = None
    if not args.no_e2e:
        f32 = store.arrays_f32()
        pinned = [torch.from_numpy(a).pin_memory() for a in f32]
        host_imgs = torch.empty((N_TIMES, H, W, 3), dtype=torch.float32, pin_memory=True)
        h2d = sum(int(a.numel() * 4) for a in pinned) + N_TIMES * 8 * 24
        d2h = host_imgs.numel() * 4
        ctx.render_views_host([p.numpy() for p in pinned], store.active_sh_degree, cams, (0, 0, 0), host_imgs.numpy())
        # Each rep timed on its own; the median is reported (the host PCIe link of the shared
        # pool's boxes occasionally drops to a fraction of its rate for a sweep).
        reps = 9
        rep_s = []
        for _ in range(reps):
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            ctx.render_views_host([p.numpy() for p in pinned], store.active_sh_degree, cams, (0, 0, 0),
                                  host_imgs.numpy())
            rep_s.append(max_over_ranks(time.perf_counter() - t0, dist, dev))
        dt = statistics.median(rep_s) * reps
        # raw PCIe D2H rate into the same pinned buffer (diagnostic for the e2e bound)
        src = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        dst = host_imgs.view(-1).view(torch.uint8)[: 256 << 20]
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        for _ in range(4):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize(dev)
        d2h_gbs = 4 * (256 << 20) / (time.perf_counter() - t1) / 1e9
        del src
        e2e = {"value": N_TIMES * reps * world / dt, "unit": "frames/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": reps, "pcie_d2h_gbs_measured": d2h_gbs,
               "rep_ms": [1e3 * x for x in rep_s], "statistic": "median of the per-sweep times",
               "best_sweep_value": N_TIMES * world / min(rep_s),
               "note": "rgs_render_views_host: pinned host scene -> HBM, 300 renders, 300 images -> pinned host; "
                       "the D2H of 4.9 GB of float32 images per sweep overlaps the renders (copy-only "
                       "4.9 GB / pcie_d2h_gbs_measured; on links below ~45 GB/s it bounds the sweep)"}

    # ---- CPU baseline (rank 0, N=1 only, bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        lib, kind = cpu_reference_lib()
        threads = os.cpu_count() or 1
        picks = [0, 100, 200, 299]
        cpu_frames(store, [cams[0]], lib, threads)  # warm
        t = cpu_frames(store, [cams[i] for i in picks], lib, threads)
        cpu = {"value": len(picks) / t, "unit": "frames/s", "cores": threads, "kind": kind,
               "sample": f"{len(picks)} frames (t index {picks}) of the same sweep, full 1352x1014, "
                         f"{threads} threads, {cpu_model()}"}

    train_res = c4_res = c5_res = None
    del images
    torch.cuda.empty_cache()
    if not args.no_c4:
        c4_res = run_c4_leg(args, ctx, dev, dist, rank, world, flush)
    if not args.no_train:
        train_res = run_train_leg(args, ctx, dev, dist, rank, world, flush)
    if not args.no_c5:
        c5_res = run_c5_leg(args, ctx, dev, dist, rank, world, flush)

    if rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_gaussians": N_GAUSS, "width": W, "height": H,
                       "timestamps": N_TIMES, "sh_degree": 3, "seed": SEED,
                       "l2": "256 MiB buffer written between sweeps; frames inside a sweep share L2 as a real sweep does",
                       "parallelism": f"view-batch x{world} (replicated scene, no collective)",
                       "n_visible_mid": n_vis, "n_pairs_mid": n_pairs, "slow_pixels_mid": n_slow,
                       "evals_per_frame": e_frame, "blends_per_frame": b_frame,
                       "kernel_evals_per_frame": E_kernel / N_TIMES,
                       "slow_pixel_reasons_per_sweep": slow_reasons,
                       "k5_warp_visits_per_frame": visits / N_TIMES,
                       "k5_warp_visits_blending_per_frame": visits_blend / N_TIMES},
            "ms_per_frame": total_ms / (N_TIMES * args.steps), "wall_s": t_wall,
            "target_fps": 600, "roofline": roofline, "kernels": roof_all, "stages": per_stage, "binning": binning,
            "stages_note": "per-stage CUDA events from a serialised profiling sweep after the timed region "
                           "(the timed sweeps pipeline 8 views over 8 streams, so stages overlap there)",
            "fp32_peak_tflops": fp32_peak, "clocks": clocks, "gpu_launches": launches,
            "e2e": e2e, "cpu_baseline": cpu, "c4": c4_res, "train": train_res, "train_c5": c5_res,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, local_rank, world)


if __name__ == "__main__":
    main()
