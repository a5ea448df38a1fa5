"""Training-side mirror of the reference over the CUDA C-ABI.

Same names, argument meaning and defaults as /root/reference/proj/include/rgs:
  TrainConfig / LossWeights / LossBreakdown         optim.hpp:17-63, loss.hpp:11-30
  evaluate_loss(...)                                trainer.cpp:22-84
  adam_step / accumulate_stats / reset_opacity      optim.cpp:110-166, 236-243
  scene_scales / build_knn4d                        trainer.cpp:12-20, knn.cpp:101-116
  l1_loss / ssim_loss / psnr                        image.cpp, ssim.cpp

Everything runs on the device: the render forward / backward, the FP64 L1 + SSIM image
gradient (rgs_image_loss), the fused Adam + entropy + statistics kernel (rgs_adam_step),
the consistency regularizer (rgs_consistency) and its exact 4D KNN (rgs_knn_build).
``Trainer`` is the step loop of train_from (trainer.cpp:102-189) for a replicated scene:
under torch.distributed every rank renders its own views and one NCCL all-reduce(sum) of
the [65 grads | viewspace_norm] block (+ the visible counts and the image losses)
reproduces the single-process batch reduction of evaluate_loss (StoreGrads::add with
visible as a count, gaussian.cpp:199-209); Adam then runs identically on every rank.
torch supplies device memory, streams and the collective; it is plumbing, not the product.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import rgs
from .rgs import CCamera, Camera, Context, DeviceScene, _ptr, _vp


@dataclass
class LossWeights:
    """loss.hpp:11-16"""

    lambda_ssim: float = 0.2
    lambda_entropy: float = 0.01
    lambda_consistency: float = 0.05
    k_neighbors: int = 8


@dataclass
class LossBreakdown:
    """loss.hpp:25-28"""

    l1: float = 0.0
    ssim: float = 0.0
    entropy: float = 0.0
    consistency: float = 0.0
    total: float = 0.0
    mse: float = 0.0  # of the batch (psnr = min(100, 10 log10(1 / mse)))


def combine_losses(w: LossWeights, l1, ssim, entropy, consistency) -> float:
    """loss.cpp:60-64"""
    return (1 - w.lambda_ssim) * l1 + w.lambda_ssim * ssim + w.lambda_entropy * entropy + \
        w.lambda_consistency * consistency


@dataclass
class TrainConfig:
    """optim.hpp:17-63 (the fields the device step uses; dataset / densify fields kept for parity)."""

    lr_position: float = 1.6e-4
    lr_position_final: float = 1.6e-6
    lr_scales: float = 5e-3
    lr_rotor: float = 1e-3
    lr_sh_dc: float = 2.5e-3
    lr_sh_rest: float = 1.25e-4
    lr_opacity: float = 0.05
    total_steps: int = 2000
    batch: int = 3
    densify_grad_threshold: float = 2e-4
    densify_from: int = 500
    densify_until: int = 15000
    densify_interval: int = 100
    opacity_reset_interval: int = 3000
    prune_opacity: float = 0.005
    percent_dense: float = 0.01
    split_factor: float = 1.6
    reset_opacity_value: float = 0.01
    min_gaussians: int = 16
    max_gaussians: int = 200000
    loss: LossWeights = field(default_factory=LossWeights)
    background: Sequence[float] = (0.0, 0.0, 0.0)
    static_mode: bool = False
    knn_rebuild_interval: int = 100
    sh_unlock_interval: int = 1000
    log_interval: int = 50

    def validate(self):
        """optim.cpp:27-45 (the checks that concern the device step)."""
        pos = lambda v: v > 0 and math.isfinite(v)  # noqa: E731
        if not all(pos(v) for v in (self.lr_position, self.lr_position_final, self.lr_scales, self.lr_rotor,
                                    self.lr_sh_dc, self.lr_sh_rest, self.lr_opacity)):
            raise ValueError("TrainConfig: learning rates must be positive")
        if self.total_steps < 0 or self.batch < 1:
            raise ValueError("TrainConfig: batch must be >= 1")
        if min(self.densify_interval, self.opacity_reset_interval, self.knn_rebuild_interval,
               self.sh_unlock_interval) <= 0:
            raise ValueError("TrainConfig: intervals must be positive")


def lr_schedule(step: int, total: int, lr_init: float, lr_final: float) -> float:
    """optim.cpp:47-51"""
    if total <= 0:
        return lr_init
    u = min(max(step / total, 0.0), 1.0)
    return lr_init * (lr_final / lr_init) ** u


class CAdamConfig(ctypes.Structure):
    """rgs_adam_config (include/rgs_cuda.h)."""

    _fields_ = [
        ("lr_position", ctypes.c_double),
        ("lr_position_final", ctypes.c_double),
        ("lr_scales", ctypes.c_double),
        ("lr_rotor", ctypes.c_double),
        ("lr_sh_dc", ctypes.c_double),
        ("lr_sh_rest", ctypes.c_double),
        ("lr_opacity", ctypes.c_double),
        ("total_steps", ctypes.c_int),
        ("static_mode", ctypes.c_int),
        ("lambda_entropy", ctypes.c_double),
        ("accumulate_stats", ctypes.c_int),
        ("flags", ctypes.c_uint),
    ]

    @staticmethod
    def from_config(cfg: TrainConfig, lambda_entropy: float = 0.0, accumulate_stats: bool = True,
                    accumulate: bool = False) -> "CAdamConfig":
        return CAdamConfig(cfg.lr_position, cfg.lr_position_final, cfg.lr_scales, cfg.lr_rotor, cfg.lr_sh_dc,
                           cfg.lr_sh_rest, cfg.lr_opacity, int(cfg.total_steps), int(bool(cfg.static_mode)),
                           float(lambda_entropy), int(bool(accumulate_stats)),
                           rgs.FLAG_ACCUMULATE if accumulate else 0)


class DeviceOptimizer:
    """Adam moments + densification statistics of one DeviceScene (rgs_optimizer)."""

    def __init__(self, ctx: Context, scene: DeviceScene):
        h = _vp()
        ctx.check(ctx.L.rgs_optimizer_create(ctx.h, scene.h, ctypes.byref(h)))
        self.ctx, self.scene, self.h = ctx, scene, h
        ctx.adopt(self)

    def step(self, grads, vnorm, visible, cfg: CAdamConfig, step: int, losses=None):
        """adam_step (+ accumulate_stats, + entropy) on device buffers; no host sync."""
        self.ctx.sync_stream()
        self.ctx.check(self.ctx.L.rgs_adam_step(self.ctx.h, self.scene.h, self.h, _vp(_ptr(grads)),
                                                _vp(_ptr(vnorm)) if vnorm is not None else None,
                                                _vp(_ptr(visible)) if visible is not None else None,
                                                ctypes.byref(cfg), int(step),
                                                _vp(_ptr(losses)) if losses is not None else None))
        self.ctx.fence()

    def status(self):
        """Raises the rotor error of the steps since the last call (synchronises)."""
        self.ctx.check(self.ctx.L.rgs_optimizer_status(self.ctx.h, self.h))

    def status_async(self, word) -> None:
        """Queues the error word's copy into ``word`` (a pinned int64 tensor of one element);
        no synchronisation.  ~0 (-1 as int64) means no rotor error."""
        self.ctx.check(self.ctx.L.rgs_optimizer_status_async(self.ctx.h, self.h, _vp(word.data_ptr())))

    def download(self):
        n = self.scene.n
        m, v = np.zeros((n, 65)), np.zeros((n, 65))
        acc, cnt = np.zeros(n), np.zeros(n, dtype=np.int32)
        self.ctx.check(self.ctx.L.rgs_optimizer_download(self.ctx.h, self.h, _vp(m.ctypes.data), _vp(v.ctypes.data),
                                                         _vp(acc.ctypes.data), _vp(cnt.ctypes.data)))
        return m, v, acc, cnt

    def upload(self, m=None, v=None, accum=None, count=None):
        def p(a, dt):
            return None if a is None else np.ascontiguousarray(a, dtype=dt)

        m, v, accum, count = p(m, np.float64), p(v, np.float64), p(accum, np.float64), p(count, np.int32)
        self.ctx.check(self.ctx.L.rgs_optimizer_upload(
            self.ctx.h, self.h, *[(_vp(a.ctypes.data) if a is not None else None) for a in (m, v, accum, count)]))

    def reset_stats(self):
        self.ctx.check(self.ctx.L.rgs_optimizer_reset_stats(self.ctx.h, self.h))

    def reset_opacity(self, value: float = 0.01):
        """optim.cpp:236-243"""
        self.ctx.sync_stream()
        self.ctx.check(self.ctx.L.rgs_reset_opacity(self.ctx.h, self.scene.h, self.h, float(value)))

    def close(self):
        if getattr(self, "h", None):
            if getattr(self.ctx, "h", None):  # (a closed context already freed it)
                self.ctx.L.rgs_optimizer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Rng:
    """The train loop's generator (std::mt19937_64(TrainConfig::seed), trainer.cpp:105), host-side
    in the C library so batch picks and densification draws match the reference's sequence."""

    def __init__(self, ctx: Context, seed: int = 0):
        h = _vp()
        ctx.check(ctx.L.rgs_rng_create(ctypes.c_ulonglong(seed), ctypes.byref(h)))
        self.ctx, self.h = ctx, h

    def uniform_int(self, lo: int, hi: int) -> int:
        """std::uniform_int_distribution<int>(lo, hi)(rng) (trainer.cpp:106, 119)."""
        out = ctypes.c_int(0)
        self.ctx.check(self.ctx.L.rgs_rng_uniform_int(self.h, int(lo), int(hi), ctypes.byref(out)))
        return out.value

    def close(self):
        if getattr(self, "h", None):
            self.ctx.L.rgs_rng_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CDensifyConfig(ctypes.Structure):
    """rgs_densify_config: TrainConfig's density control fields (optim.hpp:31-42)."""

    _fields_ = [
        ("densify_grad_threshold", ctypes.c_double),
        ("percent_dense", ctypes.c_double),
        ("split_factor", ctypes.c_double),
        ("prune_opacity", ctypes.c_double),
        ("min_gaussians", ctypes.c_int),
        ("max_gaussians", ctypes.c_int),
        ("static_mode", ctypes.c_int),
    ]

    @staticmethod
    def from_config(cfg: "TrainConfig") -> "CDensifyConfig":
        return CDensifyConfig(cfg.densify_grad_threshold, cfg.percent_dense, cfg.split_factor, cfg.prune_opacity,
                              int(cfg.min_gaussians), int(cfg.max_gaussians), int(bool(cfg.static_mode)))


@dataclass
class DensifyReport:
    """optim.hpp:94-96"""

    cloned: int = 0
    split: int = 0
    pruned: int = 0


def densify_and_prune(ctx: Context, scene: DeviceScene, opt: "DeviceOptimizer", cfg: "TrainConfig",
                      scene_extent: float, rng: Rng) -> DensifyReport:
    """optim.cpp:168-234 on the device scene (resized in place)."""
    rep = (ctypes.c_int * 3)()
    dc = CDensifyConfig.from_config(cfg)
    ctx.sync_stream()
    ctx.check(ctx.L.rgs_densify_and_prune(ctx.h, scene.h, opt.h, ctypes.byref(dc), float(scene_extent), rng.h, rep))
    scene.n = int(ctx.L.rgs_scene_size(scene.h))
    return DensifyReport(rep[0], rep[1], rep[2])


def image_loss(ctx: Context, rendered, target, w_l1: float = 1.0, w_ssim: float = 0.0, dL_dimage=None,
               losses=None, loss_scale: float = 1.0, accumulate: bool = False, accumulate_grad: bool = False,
               records=None):
    """L1 + SSIM losses and dL/dimage on device tensors (rgs_image_loss).  ``accumulate``: losses
    +=; ``accumulate_grad``: dL_dimage +=.  ``records``: the retained RenderRecords of the forward
    that rendered ``rendered`` -- L1 signs at near ties are then decided on the FP64 pixel value
    (rgs_image_loss_ex), as the reference's double image decides them."""
    h, w = int(rendered.shape[0]), int(rendered.shape[1])
    ctx.sync_stream()
    flags = (rgs.FLAG_ACCUMULATE if accumulate else 0) | (rgs.FLAG_ACCUMULATE_GRAD if accumulate_grad else 0)
    ctx.check(ctx.L.rgs_image_loss_ex(ctx.h, records.h if records is not None else None, _vp(_ptr(rendered)),
                                      _vp(_ptr(target)), w, h, float(w_l1), float(w_ssim), float(loss_scale), flags,
                                      _vp(_ptr(dL_dimage)) if dL_dimage is not None else None,
                                      _vp(_ptr(losses)) if losses is not None else None))
    ctx.fence()


def scene_scales(ctx: Context, scene: DeviceScene) -> np.ndarray:
    """trainer.cpp:12-20"""
    out = np.zeros(4)
    ctx.check(ctx.L.rgs_scene_scales(ctx.h, scene.h, _vp(out.ctypes.data)))
    return out


def build_knn4d(ctx: Context, scene: DeviceScene, k: int, scales=None, out=None):
    """knn.cpp:101-116 -> device int32 tensor (N, k)."""
    import torch

    if out is None:
        out = torch.empty((scene.n, k), dtype=torch.int32, device=f"cuda:{ctx.device}")
    sc = None if scales is None else np.ascontiguousarray(scales, dtype=np.float64)
    ctx.sync_stream()
    ctx.check(ctx.L.rgs_knn_build(ctx.h, scene.h, int(k), _vp(sc.ctypes.data) if sc is not None else None,
                                  _vp(_ptr(out))))
    ctx.fence()
    return out


def consistency(ctx: Context, scene: DeviceScene, nbrs, lam: float, grads=None, losses=None, accumulate=False,
                defer_checks=False):
    """consistency_loss + its gradient through slice_backward (trainer.cpp:66-77).
    ``defer_checks``: no host sync; a rotor / degenerate-time error goes to ctx.status()."""
    ctx.sync_stream()
    flags = (rgs.FLAG_ACCUMULATE if accumulate else 0) | (rgs.FLAG_DEFER_CHECKS if defer_checks else 0)
    ctx.check(ctx.L.rgs_consistency(ctx.h, scene.h, _vp(_ptr(nbrs)), int(nbrs.shape[1]), float(lam), flags,
                                    _vp(_ptr(grads)) if grads is not None else None,
                                    _vp(_ptr(losses)) if losses is not None else None))


# ----------------------------------------------------------------------------- multi-GPU plumbing
class NcclComm:
    """A native NCCL communicator of the C ABI (rgs_nccl_comm_create) for the fused gradient
    all-reduce (rgs_allreduce_grads: one NCCL group, a single launch, on the context's stream).
    Rank 0 makes the ncclUniqueId; it reaches the other ranks through ``dist`` (any backend)."""

    def __init__(self, ctx: Context, dist):
        L = ctx.L
        if not L.rgs_nccl_available():
            raise rgs.RgsUnavailableError("NCCL not found (rgs_nccl_available() == 0)")
        world, rank = dist.get_world_size(), dist.get_rank()
        uid = (ctypes.c_ubyte * 128)()
        if rank == 0:
            ctx.check(L.rgs_nccl_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        uid = (ctypes.c_ubyte * 128).from_buffer_copy(box[0])
        h = _vp()
        ctx.check(L.rgs_nccl_comm_create(ctx.h, world, rank, uid, ctypes.byref(h)))
        self.ctx, self.h, self.world, self.rank = ctx, h, world, rank

    @staticmethod
    def single(ctx: Context) -> "NcclComm":
        """A one-rank communicator (the all-reduce is the identity): tests of the native path."""
        self = NcclComm.__new__(NcclComm)
        uid = (ctypes.c_ubyte * 128)()
        ctx.check(ctx.L.rgs_nccl_unique_id(uid))
        h = _vp()
        ctx.check(ctx.L.rgs_nccl_comm_create(ctx.h, 1, 0, uid, ctypes.byref(h)))
        self.ctx, self.h, self.world, self.rank = ctx, h, 1, 0
        return self

    def allreduce_step(self, gbuf, visible, losses_img) -> None:
        ctx = self.ctx
        ctx.sync_stream()
        ctx.check(ctx.L.rgs_allreduce_grads(ctx.h, self.h, _vp(_ptr(gbuf)), gbuf.numel(), _vp(_ptr(visible)),
                                            visible.numel(), _vp(_ptr(losses_img)), losses_img.numel()))

    def close(self):
        if getattr(self, "h", None):
            self.ctx.L.rgs_nccl_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def allreduce_step_buffers(gbuf, visible, losses_img, dist=None, comm: Optional[NcclComm] = None):
    """The batch reduction across ranks: sum of the [65 grads | viewspace_norm] block, of the
    visible counts and of the three image-loss slots.  A no-op on one process.  With ``comm``
    (NcclComm): one fused NCCL group through the C ABI; otherwise three torch.distributed
    collectives on any backend (gloo on CPU in the tests, NCCL over NVLink on the GPUs)."""
    if comm is not None:
        comm.allreduce_step(gbuf, visible, losses_img)
        return
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return
    dist.all_reduce(gbuf)
    dist.all_reduce(visible)
    dist.all_reduce(losses_img)


class TargetStager:
    """Double-buffered host -> device staging of a step's target images on a copy stream, so
    the PCIe transfer of step k+1 overlaps the compute of step k.  (The reference keeps its
    dataset in host memory and reads the images in place, dataset.cpp / trainer.cpp:22-84; on
    the GPU every step's targets cross PCIe once.)

    ``put(host_images)`` queues the copies of one step (pinned host tensors of shape (H, W, 3),
    float32); ``take()`` returns that step's device views and orders torch's current stream
    after their copy; ``release()`` -- after the step that consumed them is enqueued -- lets
    the buffer be refilled."""

    def __init__(self, device, batch: int, height: int, width: int, depth: int = 2):
        import collections

        import torch

        self.device = torch.device(device)
        self.bufs = [torch.empty((batch, height, width, 3), dtype=torch.float32, device=self.device)
                     for _ in range(depth)]
        self.ready = [None] * depth
        self.free = [None] * depth
        self.stream = torch.cuda.Stream(self.device)
        self.queue = collections.deque()
        self.next = 0
        self.taken = None
        self.bytes_per_put = 0

    def put(self, host_images) -> None:
        import torch

        if len(self.queue) >= len(self.bufs):
            raise RuntimeError("TargetStager: every buffer is queued; take() one first")
        i = self.next
        if i == self.taken:
            raise RuntimeError("TargetStager: release() the taken buffer before refilling it")
        if len(host_images) > self.bufs[i].shape[0]:
            raise ValueError("TargetStager: more images than the batch size")
        self.next = (i + 1) % len(self.bufs)
        with torch.cuda.stream(self.stream):
            if self.free[i] is not None:
                self.stream.wait_event(self.free[i])
            nbytes = 0
            for j, h in enumerate(host_images):
                self.bufs[i][j].copy_(h, non_blocking=True)
                nbytes += h.numel() * h.element_size()
            self.ready[i] = self.stream.record_event()
        self.bytes_per_put = nbytes
        self.queue.append((i, len(host_images)))

    def take(self):
        import torch

        if self.taken is not None:
            raise RuntimeError("TargetStager: release() the previous batch first")
        i, n = self.queue.popleft()
        torch.cuda.current_stream(self.device).wait_event(self.ready[i])
        self.taken = i
        return [self.bufs[i][j] for j in range(n)]

    def release(self, ctx: Optional[Context] = None) -> None:
        import torch

        if self.taken is None:
            return
        if ctx is not None:
            ctx.fence()
        self.free[self.taken] = torch.cuda.current_stream(self.device).record_event()
        self.taken = None


class Trainer:
    """evaluate_loss + accumulate_stats + adam_step of train_from (trainer.cpp:121-150) on a
    device-resident scene.  ``dist``: torch.distributed (initialised) for the multi-GPU
    batch (each rank passes its own views; the batch size is views_per_rank * world)."""

    def __init__(self, ctx: Context, scene: DeviceScene, config: TrainConfig, dist=None,
                 scene_extent: Optional[float] = None, seed: int = 0, start_step: int = 0,
                 comm: Optional[NcclComm] = None):
        """``start_step``: the number of steps already taken (resuming a run): the next step is
        start_step + 1, with its SH degree, learning-rate schedule and intervals (trainer.cpp:115-150).
        ``comm``: a native NcclComm for the batch all-reduce (else torch.distributed's)."""
        self.comm = comm
        config.validate()
        if start_step < 0:
            raise ValueError("Trainer: start_step must be >= 0")
        self.ctx, self.scene, self.cfg, self.dist = ctx, scene, config, dist
        self.scene_extent = scene_extent  # camera_extent(dataset) (trainer.cpp:88-99); None: no densification
        self.rng = Rng(ctx, seed)
        self.opt = DeviceOptimizer(ctx, scene)
        self.step_count = int(start_step)
        self._knn_built = False
        self.nbrs = None
        self._img = None
        self._dl = None
        self._streams = None
        self.overlap = True  # forward of view v+1 alongside the backward of view v
        # RGS_FLAG_REPRODUCIBLE backward: bitwise identical steps run to run (fixed-point sums)
        self.reproducible = False
        self.n_slots = 3  # views whose forward / loss may be in flight at once (side streams)
        # Deferred checks: the step's forwards and consistency term do not synchronise; their
        # rotor / degenerate-time errors and pair-buffer overflows surface at the step's loss
        # read (read_losses / pop_losses / last_losses).  The first step, the step after a
        # densification and one step per KNN-rebuild interval run checked (they size the pair
        # buffers).
        self.defer_checks = True
        self._checked_next = True
        self._alloc()

    def _alloc(self):
        """Gradient / statistics buffers sized for the current scene (re-run after densification)."""
        import torch

        ctx, scene = self.ctx, self.scene
        dist = self.dist
        self.world = dist.get_world_size() if (dist is not None and dist.is_initialized()) else 1
        dev = f"cuda:{ctx.device}"
        n = scene.n
        self.gbuf = torch.zeros(66 * n, dtype=torch.float32, device=dev)  # [65 grads | viewspace_norm]
        self.grads = self.gbuf[: 65 * n]
        self.vnorm = self.gbuf[65 * n:]
        self.visible = torch.zeros(n, dtype=torch.int32, device=dev)
        self.losses = torch.zeros(8, dtype=torch.float64, device=dev)  # l1, ssim, mse, entropy, consistency
        self.losses_host = torch.zeros(8, dtype=torch.float64).pin_memory()
        # queued (read=False) loss copies: a ring of two pinned slots with the rotor-error word
        # and an event each, so step k's losses are read while step k+1 runs (pop_losses)
        import collections

        self._ring = [torch.zeros(8, dtype=torch.float64).pin_memory() for _ in range(2)]
        self._ring_err = [torch.zeros(1, dtype=torch.int64).pin_memory() for _ in range(2)]
        self._ring_ctx = [torch.zeros(1, dtype=torch.int64).pin_memory() for _ in range(2)]
        self._ring_ev = [None, None]
        self._ring_next = 0
        self._pending = collections.deque()

    # trainer.cpp:107-113
    def rebuild_knn(self):
        self._knn_built = True
        w = self.cfg.loss
        if w.lambda_consistency != 0 and self.scene.n > w.k_neighbors:
            self.nbrs = build_knn4d(self.ctx, self.scene, w.k_neighbors, out=self.nbrs)
        else:
            self.nbrs = None

    def _buffers(self, cam: Camera, slot: int = 0):
        import torch

        shape = (cam.height, cam.width, 3)
        if self._img is None or tuple(self._img[0].shape) != shape:
            dev = f"cuda:{self.ctx.device}"
            self._img = [torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(self.n_slots)]
            self._dl = [torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(self.n_slots)]
        return self._img[slot], self._dl[slot]

    def evaluate_loss(self, cams: Sequence[Camera], targets, want_grads: bool = True, defer: bool = False):
        """trainer.cpp:22-84 for this rank's views (device tensors); leaves the batch-reduced
        gradients in self.grads / vnorm / visible and the losses in self.losses (device).

        With ``overlap`` (default) the forward and image loss of view v+1 run on a side stream
        while the backward of view v runs on the main stream; the losses and the backward
        passes each stay in view order (they accumulate into one buffer).  ``defer``: the forwards
        and the consistency term skip their host synchronisation (errors via ctx.status())."""
        import torch

        w = self.cfg.loss
        ctx, scene = self.ctx, self.scene
        ctx.fence()
        # The first view's backward writes every Gaussian's gradients, norm and visible count
        # (accumulate=False), so the gradient buffers are only zeroed when no backward runs.
        first_writes = want_grads and len(cams) > 0
        if not first_writes:
            self.gbuf.zero_()
            self.visible.zero_()
        self.losses.zero_()
        inv_b = 1.0 / (len(cams) * self.world) if cams else 0.0
        wl1, wss = (1 - w.lambda_ssim) * inv_b, w.lambda_ssim * inv_b
        overlap = self.overlap and ctx._torch_stream and len(cams) > 1
        main = torch.cuda.current_stream(ctx.device)
        if overlap and self._streams is None:
            self._streams = [torch.cuda.Stream(ctx.device) for _ in range(self.n_slots)]
        # per buffer slot: event after its last use on the main stream; initially the end of the
        # previous step (its Adam update of the scene) and of the buffer zeroing above
        start = main.record_event() if overlap else None
        free = [start] * self.n_slots
        # On one rank the consistency term (it depends on the scene only) runs on the main stream
        # right after the first view's backward (which initialises the gradients), beside the
        # next view's forward on the side stream; with N ranks it is added after the all-reduce
        # (it is a once-per-step term of the replicated scene).
        early_consistency = self.world == 1
        if early_consistency and not first_writes:
            self._consistency(want_grads, defer)
        recs = []
        loss_done = None  # the previous view's image loss (its scratch and the loss slots are shared)
        for v, (cam, tgt) in enumerate(zip(cams, targets)):
            slot = v % self.n_slots if overlap else 0
            img, dl = self._buffers(cam, slot)
            if overlap:
                # side stream: forward of view v, then its image loss (FP64, SSIM) -- so the loss
                # overlaps the FP32 backward of view v - 1 on the main stream
                side = self._streams[slot]
                if free[slot] is not None:
                    side.wait_event(free[slot])
                with torch.cuda.stream(side):
                    img, rec = ctx.render_forward_device(scene, cam, self.cfg.background, retain=want_grads,
                                                         image=img, defer_checks=defer)
                    if loss_done is not None:
                        side.wait_event(loss_done)
                    image_loss(ctx, img, tgt, wl1, wss, dl if want_grads else None, self.losses, loss_scale=inv_b,
                               accumulate=True, records=rec if want_grads else None)
                    loss_done = side.record_event()
                main.wait_stream(side)
                ctx.sync_stream()
            else:
                img, rec = ctx.render_forward_device(scene, cam, self.cfg.background, retain=want_grads, image=img,
                                                     defer_checks=defer)
                image_loss(ctx, img, tgt, wl1, wss, dl if want_grads else None, self.losses, loss_scale=inv_b,
                           accumulate=True, records=rec if want_grads else None)
            if want_grads:
                ctx.render_backward_device(scene, cam, rec, dl, self.grads, self.vnorm, self.visible, accumulate=v > 0,
                                           reproducible=self.reproducible)
                if v == 0 and early_consistency:
                    self._consistency(want_grads, defer)
            if overlap:
                free[slot] = main.record_event()
            recs.append(rec)
        for rec in recs:  # returned to the context's frame pool (stream-ordered, no host sync)
            rec.close()
        if self.world > 1 or self.comm is not None:
            ctx.fence()
            allreduce_step_buffers(self.gbuf, self.visible, self.losses[:3], self.dist, self.comm)
            if not ctx._torch_stream:
                torch.cuda.current_stream(ctx.device).synchronize()
        if not early_consistency:
            self._consistency(want_grads, defer)

    def _consistency(self, want_grads: bool, defer: bool):
        w = self.cfg.loss
        if w.lambda_consistency != 0 and self.nbrs is not None and self.scene.n > 0:
            consistency(self.ctx, self.scene, self.nbrs, w.lambda_consistency, self.grads if want_grads else None,
                        self.losses[4:5], defer_checks=defer)

    def step(self, cams: Sequence[Camera], targets, read: bool = True) -> Optional[LossBreakdown]:
        """One train_from iteration minus densification (trainer.cpp:115-150): SH unlock, batch
        loss + gradients, accumulate_stats, Adam, opacity reset and KNN rebuild schedules.
        ``read``: one host synchronisation per step for the loss scalars (and the rotor-error
        word), as train_from's per-step loss check.  ``read=False`` only queues the copy of the
        losses and of the rotor-error word (no sync, so the next step's work is enqueued without
        a bubble); `pop_losses()` returns the oldest queued step's (waiting for that step only),
        `last_losses()` the newest; both raise a deferred rotor error."""
        cfg, w = self.cfg, self.cfg.loss
        self.step_count += 1
        step = self.step_count
        sh = min(3, (step - 1) // cfg.sh_unlock_interval)
        if sh != self.scene.sh_degree:
            self.ctx.L.rgs_scene_set_sh_degree(self.scene.h, sh)
            self.scene.sh_degree = sh
        if self.nbrs is None and not self._knn_built:  # trainer.cpp:107-113 (first step of the run)
            self.rebuild_knn()
        defer = self.defer_checks and not self._checked_next
        self._checked_next = False
        self.evaluate_loss(cams, targets, True, defer=defer)
        acfg = CAdamConfig.from_config(cfg, w.lambda_entropy, True)
        self.opt.step(self.grads, self.vnorm, self.visible, acfg, step, self.losses[3:4])
        if read:
            out = self.read_losses()
        else:
            self._queue_losses()
            out = None
        mutated = False
        if (self.scene_extent is not None and cfg.densify_from <= step <= cfg.densify_until
                and step % cfg.densify_interval == 0):
            # optim.cpp:168-234; every rank draws the same numbers from its own copy of the
            # generator, so the replicated scenes stay identical.
            self.last_densify = densify_and_prune(self.ctx, self.scene, self.opt, cfg, self.scene_extent, self.rng)
            self._alloc()
            mutated = True
            self._checked_next = True  # the scene changed size: re-learn the pair capacities
        if step % cfg.opacity_reset_interval == 0:
            self.opt.reset_opacity(cfg.reset_opacity_value)
        if mutated or step % cfg.knn_rebuild_interval == 0:
            self.nbrs = None
            self.rebuild_knn()
            # a checked step now and then re-learns the pair counts the deferred forwards' 2x
            # buffer headroom is based on (splats grow between densifications too)
            self._checked_next = True
        return out

    def _queue_losses(self):
        import torch

        slot = self._ring_next
        self._ring_next ^= 1
        if slot in self._pending:  # never popped: the oldest queued read is dropped
            self._pending.remove(slot)
        self.ctx.fence()
        self._ring[slot].copy_(self.losses, non_blocking=True)
        self.opt.status_async(self._ring_err[slot])
        self.ctx.status_async(self._ring_ctx[slot])
        self._ring_ev[slot] = torch.cuda.current_stream(self.ctx.device).record_event()
        self._pending.append(slot)

    def _breakdown(self, h) -> LossBreakdown:
        w = self.cfg.loss
        out = LossBreakdown(float(h[0]), float(h[1]), float(h[3]), float(h[4]), 0.0, float(h[2]))
        out.total = combine_losses(w, out.l1, out.ssim, out.entropy, out.consistency)
        return out

    def pop_losses(self) -> LossBreakdown:
        """The oldest queued (``read=False``) step's losses: waits for that step only (later
        steps keep running) and raises its rotor error, if any."""
        slot = self._pending.popleft()
        self._ring_ev[slot].synchronize()
        if int(self._ring_ctx[slot].item()) != -1:
            self.ctx.status()  # raises (and clears) a deferred forward / consistency error
        if int(self._ring_err[slot].item()) != -1:
            self.opt.status()  # raises (and clears) the reported rotor error
        return self._breakdown(self._ring[slot].numpy())

    def read_losses(self) -> LossBreakdown:
        """The current losses (synchronises; raises pending rotor errors)."""
        self.ctx.fence()
        self.losses_host.copy_(self.losses, non_blocking=True)
        self.ctx.status()  # synchronises; raises deferred forward / consistency errors
        self.opt.status()  # raises rotor errors of the Adam step
        self._pending.clear()
        return self._breakdown(self.losses_host.numpy())

    def last_losses(self) -> LossBreakdown:
        """The most recent loss copy -- a synchronous read or the newest queued one
        (synchronises; raises pending rotor errors; drops older queued reads)."""
        self.ctx.status()  # synchronises; raises deferred forward / consistency errors
        self.opt.status()  # raises rotor errors of the Adam step
        if self._pending:
            slot = self._pending[-1]
            self._pending.clear()
            return self._breakdown(self._ring[slot].numpy())
        return self._breakdown(self.losses_host.numpy())


def psnr_from_mse(mse: float) -> float:
    """image.cpp:7-18"""
    if mse <= 0:
        return 100.0
    return min(100.0, 10 * math.log10(1 / mse))
