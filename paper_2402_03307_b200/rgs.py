"""Python mirror of the reference renderer API over the CUDA C-ABI (include/rgs_cuda.h).

Same names, argument meaning and error behaviour as /root/reference/proj/include/rgs:
  render_forward(store, cam, opts) -> RenderOutput           rasterizer.hpp:82-83
  rasterize_forward(splats, cam, background, threads)         rasterizer.hpp:87-89
  render_backward(store, cam, records, dL_dimage, threads)    rasterizer.hpp:93-95
  render_flow(store, cam, threads)                            rasterizer.hpp:99
  GaussianStore / Camera / RenderOptions / RenderRecords / StoreGrads
  MissingRecordsError, ZeroRotorError, NonFiniteRotorError, camera runtime_error

There is no CPU path: every call runs the sm_100a kernels in librgs_cuda.so and
fails loudly (RgsUnavailableError) when the library or a CUDA device is missing.
``threads`` is accepted for signature parity and ignored.

Device-resident entry points for throughput work (bench.py, training loops):
``Context``, ``DeviceScene``, ``Context.render_views`` / ``render_backward_device``,
operating on torch CUDA tensors (torch is used only for device memory and streams).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RGS_LIB") or os.path.join(_HERE, "librgs_cuda.so")  # RGS_LIB: A/B runs of another build

# ----------------------------------------------------------------------------- errors
RGS_OK = 0
RGS_E_CAMERA = 1
RGS_E_MISSING_RECORDS = 2
RGS_E_ZERO_ROTOR = 3
RGS_E_NONFINITE_ROTOR = 4
RGS_E_CUDA = 5
RGS_E_INVALID = 6
RGS_E_DEGENERATE_TIME = 7
RGS_E_NO_DEVICE = 8
RGS_E_CHECKPOINT = 9
RGS_E_OVERFLOW = 10

FLAG_RETAIN_RECORDS = 1
FLAG_BLEND_FP64 = 2
FLAG_ACCUMULATE = 4
FLAG_HOST_BUFFERS = 8
FLAG_IMAGE_F64 = 16
FLAG_DETERMINISTIC = 32
FLAG_ACCUMULATE_GRAD = 64
FLAG_DEFER_CHECKS = 128
FLAG_REPRODUCIBLE = 256

BINNING_AUTO = 0
BINNING_RADIX = 1
BINNING_SCATTER = 2

_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy
SCENE_F64 = 1  # rgs_scene_create_ex storage flag


class RgsUnavailableError(RuntimeError):
    """The CUDA library or a CUDA device is missing (there is no CPU fallback)."""


class RgsCudaError(RuntimeError):
    pass


class MissingRecordsError(RuntimeError):
    """rasterizer.hpp:78-80"""


class ZeroRotorError(RuntimeError):
    """rotor.hpp:56-58"""

    def __init__(self, msg="normalize: zero rotor", index=-1):
        super().__init__(msg)
        self.index = index


class NonFiniteRotorError(RuntimeError):
    """rotor.hpp:59-61"""

    def __init__(self, msg="normalize: result violates rotor invariants", index=-1):
        super().__init__(msg)
        self.index = index


class CameraError(RuntimeError):
    """std::runtime_error thrown by Camera::validate (camera.hpp:21-26)."""


class CheckpointError(RuntimeError):
    """checkpoint.hpp:10-12"""


class PairOverflowError(RuntimeError):
    """A deferred-check forward (FLAG_DEFER_CHECKS) outgrew its pair buffers: its records are
    incomplete and the work that used them must be re-run with checks."""


class DegenerateTimeError(RuntimeError):
    """gaussian.hpp:31-33 (escapes gaussian_speed in the consistency term)."""

    def __init__(self, msg="slice_at: temporal scale collapsed (W < 1e-12)", index=-1):
        super().__init__(msg)
        self.index = index


# ----------------------------------------------------------------------------- ctypes
class CCamera(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int),
        ("height", ctypes.c_int),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("world_to_camera", ctypes.c_double * 16),
        ("time", ctypes.c_double),
    ]


class CRecordsInfo(ctypes.Structure):
    _fields_ = [
        ("n_splats", ctypes.c_int),
        ("tiles_x", ctypes.c_int),
        ("tiles_y", ctypes.c_int),
        ("retained", ctypes.c_int),
        ("n_pairs", ctypes.c_longlong),
        ("n_slow_pixels", ctypes.c_int),
        ("width", ctypes.c_int),
        ("height", ctypes.c_int),
    ]


SPLAT_DTYPE = np.dtype(
    [
        ("mean2", "<f8", (2,)),
        ("conic", "<f8", (3,)),
        ("depth", "<f8"),
        ("color", "<f8", (3,)),
        ("alpha_base", "<f8"),
        ("flow2", "<f8", (2,)),
        ("radius", "<f8"),
        ("source_index", "<i4"),
        ("pad", "<i4"),
    ]
)

_vp = ctypes.c_void_p
_lib = None

# Exported symbols of include/rgs_cuda.h (checked by tests/test_abi.py).
EXPORTS = [
    "rgs_abi_version", "rgs_device_count", "rgs_ctx_create", "rgs_ctx_destroy", "rgs_ctx_set_stream",
    "rgs_ctx_stream", "rgs_ctx_last_error", "rgs_ctx_error_index", "rgs_ctx_synchronize",
    "rgs_ctx_status", "rgs_ctx_status_async",
    "rgs_ctx_kernel_launches", "rgs_scene_create", "rgs_scene_destroy", "rgs_scene_size",
    "rgs_scene_set_sh_degree", "rgs_scene_upload_f64", "rgs_scene_upload_f32", "rgs_scene_params",
    "rgs_scene_download_f64", "rgs_render_forward", "rgs_render_views", "rgs_render_views_host",
    "rgs_rasterize_forward", "rgs_render_flow", "rgs_records_destroy", "rgs_records_info_get",
    "rgs_records_export", "rgs_render_backward", "rgs_camera_validate", "rgs_profile_num_stages",
    "rgs_profile_stage_name", "rgs_ctx_set_profiling", "rgs_ctx_profile_reset", "rgs_ctx_profile_read",
    "rgs_measure_fp32_tflops", "rgs_project_sliced", "rgs_project_sliced_cache", "rgs_scene_create_ex", "rgs_scene_params_f64",
    # training side (train.py)
    "rgs_image_loss", "rgs_optimizer_create", "rgs_optimizer_destroy", "rgs_adam_step", "rgs_optimizer_status",
    "rgs_optimizer_status_async", "rgs_optimizer_download", "rgs_optimizer_upload", "rgs_optimizer_reset_stats", "rgs_reset_opacity",
    "rgs_scene_scales", "rgs_knn_build", "rgs_consistency",
    "rgs_scene_load_checkpoint", "rgs_scene_save_checkpoint",
    "rgs_rng_create", "rgs_rng_destroy", "rgs_rng_uniform_int", "rgs_densify_and_prune",
    "rgs_knn_query", "rgs_consistency_loss", "rgs_image_loss_f64", "rgs_entropy_loss", "rgs_accumulate_stats",
    "rgs_rng_get_state", "rgs_rng_set_state", "rgs_malloc", "rgs_free", "rgs_memcpy",
    "rgs_accumulate_stats_f64", "rgs_ctx_profile_slow_reasons", "rgs_ctx_profile_blend_visits", "rgs_measure_fp64_tflops",
    # multi-GPU (train.NcclComm)
    "rgs_nccl_available", "rgs_nccl_unique_id", "rgs_nccl_comm_create", "rgs_nccl_comm_destroy",
    "rgs_allreduce_grads", "rgs_image_loss_ex", "rgs_ctx_set_binning",
]


def load_library(path: str = LIB_PATH):
    """Loads librgs_cuda.so and declares the C signatures (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RgsUnavailableError(f"{path} is not built; run paper_2402_03307_b200/build.py")
    L = ctypes.CDLL(path)
    i, ll, p, d = ctypes.c_int, ctypes.c_longlong, _vp, ctypes.c_double
    sig = {
        "rgs_abi_version": (i, []),
        "rgs_device_count": (i, []),
        "rgs_ctx_create": (i, [i, p]),
        "rgs_ctx_destroy": (None, [p]),
        "rgs_ctx_set_stream": (i, [p, p]),
        "rgs_ctx_stream": (p, [p]),
        "rgs_ctx_last_error": (ctypes.c_char_p, [p]),
        "rgs_ctx_status": (i, [p]),
        "rgs_ctx_status_async": (i, [p, p]),
        "rgs_ctx_error_index": (i, [p]),
        "rgs_ctx_synchronize": (i, [p]),
        "rgs_ctx_kernel_launches": (ll, [p]),
        "rgs_scene_create": (i, [p, i, i, p]),
        "rgs_scene_destroy": (None, [p]),
        "rgs_scene_size": (i, [p]),
        "rgs_scene_set_sh_degree": (i, [p, i]),
        "rgs_scene_upload_f64": (i, [p, p, p, p, p, p, p, p]),
        "rgs_scene_upload_f32": (i, [p, p, p, p, p, p, p]),
        "rgs_scene_params": (p, [p]),
        "rgs_scene_create_ex": (i, [p, i, i, ctypes.c_uint, p]),
        "rgs_scene_params_f64": (p, [p]),
        "rgs_scene_download_f64": (i, [p, p, p, p, p, p, p]),
        "rgs_render_forward": (i, [p, p, p, p, ctypes.c_uint, p, p]),
        "rgs_render_views": (i, [p, p, p, i, p, ctypes.c_uint, p]),
        "rgs_render_views_host": (i, [p, i, i, p, p, p, p, p, p, i, p, p]),
        "rgs_rasterize_forward": (i, [p, p, i, p, p, ctypes.c_uint, p, p]),
        "rgs_render_flow": (i, [p, p, p, ctypes.c_uint, p]),
        "rgs_records_destroy": (None, [p]),
        "rgs_records_info_get": (i, [p, p]),
        "rgs_records_export": (i, [p, p, p, p, p, p, p]),
        "rgs_render_backward": (i, [p, p, p, p, p, ctypes.c_uint, p, p, p]),
        "rgs_camera_validate": (i, [p, p]),
        "rgs_profile_num_stages": (i, []),
        "rgs_profile_stage_name": (ctypes.c_char_p, [i]),
        "rgs_ctx_set_profiling": (i, [p, i, i]),
        "rgs_ctx_set_binning": (i, [p, i]),
        "rgs_ctx_profile_reset": (i, [p]),
        "rgs_ctx_profile_read": (i, [p, p, p, p]),
        "rgs_measure_fp32_tflops": (i, [p, p]),
        "rgs_measure_fp64_tflops": (i, [p, p]),
        "rgs_nccl_available": (i, []),
        "rgs_nccl_unique_id": (i, [p]),
        "rgs_nccl_comm_create": (i, [p, i, i, p, p]),
        "rgs_nccl_comm_destroy": (None, [p]),
        "rgs_allreduce_grads": (i, [p, p, p, ctypes.c_size_t, p, ctypes.c_size_t, p, i]),
        "rgs_project_sliced": (i, [p, p, p, p, i, d, p, p]),
        "rgs_project_sliced_cache": (i, [p, p, p, p, i, d, p, p, p]),
        "rgs_image_loss": (i, [p, p, p, i, i, d, d, d, ctypes.c_uint, p, p]),
        "rgs_image_loss_ex": (i, [p, p, p, p, i, i, d, d, d, ctypes.c_uint, p, p]),
        "rgs_optimizer_create": (i, [p, p, p]),
        "rgs_optimizer_destroy": (None, [p]),
        "rgs_adam_step": (i, [p, p, p, p, p, p, p, i, p]),
        "rgs_optimizer_status": (i, [p, p]),
        "rgs_optimizer_status_async": (i, [p, p, p]),
        "rgs_optimizer_download": (i, [p, p, p, p, p, p]),
        "rgs_optimizer_upload": (i, [p, p, p, p, p, p]),
        "rgs_optimizer_reset_stats": (i, [p, p]),
        "rgs_reset_opacity": (i, [p, p, p, d]),
        "rgs_scene_scales": (i, [p, p, p]),
        "rgs_knn_build": (i, [p, p, i, p, p]),
        "rgs_consistency": (i, [p, p, p, i, d, ctypes.c_uint, p, p]),
        "rgs_scene_load_checkpoint": (i, [p, ctypes.c_char_p, ctypes.c_uint, p]),
        "rgs_scene_save_checkpoint": (i, [p, p, ctypes.c_char_p]),
        "rgs_rng_create": (i, [ctypes.c_ulonglong, p]),
        "rgs_rng_destroy": (None, [p]),
        "rgs_rng_uniform_int": (i, [p, i, i, p]),
        "rgs_densify_and_prune": (i, [p, p, p, p, d, p, p]),
        "rgs_knn_query": (i, [p, p, i, p, i, p, i, p]),
        "rgs_consistency_loss": (i, [p, p, i, p, i, p, p]),
        "rgs_image_loss_f64": (i, [p, p, p, i, i, d, d, d, ctypes.c_uint, p, p]),
        "rgs_entropy_loss": (i, [p, p, i, p, p]),
        "rgs_accumulate_stats": (i, [p, p, p, p]),
        "rgs_accumulate_stats_f64": (i, [p, p, p, p]),
        "rgs_ctx_profile_slow_reasons": (i, [p, p]),
        "rgs_ctx_profile_blend_visits": (i, [p, p]),
        "rgs_rng_get_state": (i, [p, p, ctypes.c_size_t, p]),
        "rgs_rng_set_state": (i, [p, ctypes.c_char_p]),
        "rgs_malloc": (p, [p, ctypes.c_size_t]),
        "rgs_free": (None, [p, p]),
        "rgs_memcpy": (i, [p, p, p, ctypes.c_size_t]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor


# ----------------------------------------------------------------------------- types
@dataclass
class Camera:
    """camera.hpp:11-27 — pinhole, world_to_camera maps to +z forward."""

    width: int = 0
    height: int = 0
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    world_to_camera: np.ndarray = field(default_factory=lambda: np.eye(4))
    time: float = 0.0

    def rotation(self):
        return np.asarray(self.world_to_camera, dtype=np.float64)[:3, :3]

    def translation(self):
        return np.asarray(self.world_to_camera, dtype=np.float64)[:3, 3]

    def center(self):
        return -self.rotation().T @ self.translation()

    def to_c(self) -> CCamera:
        c = CCamera()
        c.width, c.height = int(self.width), int(self.height)
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        w = np.asarray(self.world_to_camera, dtype=np.float64).reshape(16)
        for k in range(16):
            c.world_to_camera[k] = float(w[k])
        c.time = float(self.time)
        return c

    def validate(self):
        """camera.hpp:21-26"""
        if not (self.fx > 0) or not (self.fy > 0):
            raise CameraError("camera: focal lengths must be positive")
        r = self.rotation()
        if np.abs(r @ r.T - np.eye(3)).max() > 1e-6:
            raise CameraError("camera: rotation block not orthogonal")


@dataclass
class GaussianStore:
    """gaussian.hpp:79-103 (parameters only; optimizer state lives with the optimizer).

    mean (N,4) x,y,z,t; log_scales (N,4); rotor (N,8) s,b01,b02,b03,b12,b13,b23,p;
    opacity_logit (N,); sh (N,3,16) rows R,G,B with 16 degree-3 coefficients (DC first).
    """

    mean: np.ndarray
    log_scales: np.ndarray
    rotor: np.ndarray
    opacity_logit: np.ndarray
    sh: np.ndarray
    active_sh_degree: int = 0

    @staticmethod
    def empty(n=0, sh_degree=0):
        return GaussianStore(np.zeros((n, 4)), np.zeros((n, 4)), np.tile([1.0, 0, 0, 0, 0, 0, 0, 0], (n, 1)),
                             np.zeros(n), np.zeros((n, 3, 16)), sh_degree)

    def size(self):
        return int(np.asarray(self.opacity_logit).shape[0])

    def copy(self):
        return GaussianStore(self.mean.copy(), self.log_scales.copy(), self.rotor.copy(),
                             self.opacity_logit.copy(), self.sh.copy(), self.active_sh_degree)

    def arrays_f64(self):
        n = self.size()
        return (np.ascontiguousarray(self.mean, np.float64).reshape(n, 4),
                np.ascontiguousarray(self.log_scales, np.float64).reshape(n, 4),
                np.ascontiguousarray(self.rotor, np.float64).reshape(n, 8),
                np.ascontiguousarray(self.opacity_logit, np.float64).reshape(n),
                np.ascontiguousarray(self.sh, np.float64).reshape(n, 48))

    def arrays_f32(self):
        return tuple(np.ascontiguousarray(a, np.float32) for a in self.arrays_f64())


@dataclass
class RenderOptions:
    """rasterizer.hpp:56-60 (+ blend_fp64: the all-FP64 reference-KAT mode)."""

    background: Sequence[float] = (0.0, 0.0, 0.0)
    threads: int = 1
    retain_records: bool = False
    blend_fp64: bool = False


@dataclass
class StoreGrads:
    """gaussian.hpp:106-119 (per-parameter gradients of a whole store)."""

    d_mean: np.ndarray
    d_log_scales: np.ndarray
    d_rotor: np.ndarray
    d_opacity_logit: np.ndarray
    d_sh: np.ndarray
    viewspace_norm: np.ndarray
    visible: np.ndarray

    def as_matrix(self):
        """(N, 65) in the reference order mean4, ls4, rotor8, opacity, sh48 channel-major."""
        n = self.d_opacity_logit.shape[0]
        return np.concatenate([self.d_mean, self.d_log_scales, self.d_rotor, self.d_opacity_logit[:, None],
                               self.d_sh.reshape(n, 48)], axis=1)

    def add(self, other: "StoreGrads"):
        """StoreGrads::add (gaussian.cpp:199-209): sums, viewspace_norm summed, visible OR-ed."""
        self.d_mean += other.d_mean
        self.d_log_scales += other.d_log_scales
        self.d_rotor += other.d_rotor
        self.d_opacity_logit += other.d_opacity_logit
        self.d_sh += other.d_sh
        self.viewspace_norm += other.viewspace_norm
        self.visible |= other.visible


def grads_from_soa(flat: np.ndarray, n: int):
    """Device SoA gradient block (rgs_scene_params layout) -> reference-ordered arrays."""
    flat = np.asarray(flat, dtype=np.float64).reshape(65 * n)
    mean = flat[: 4 * n].reshape(n, 4)
    ls = flat[4 * n: 8 * n].reshape(n, 4)
    rot = np.concatenate([flat[8 * n: 12 * n].reshape(n, 4), flat[12 * n: 16 * n].reshape(n, 4)], axis=1)
    sh_blocks = flat[16 * n: 64 * n].reshape(12, n, 4).transpose(1, 0, 2).reshape(n, 48)  # j = k*3+ch
    sh = sh_blocks.reshape(n, 16, 3).transpose(0, 2, 1).copy()
    op = flat[64 * n: 65 * n].copy()
    return mean.copy(), ls.copy(), rot, op, sh


class Context:
    """Owns one rgs_ctx (device, stream, scratch arena)."""

    def __init__(self, device: int = 0, use_torch_stream: bool = True):
        L = load_library()
        if L.rgs_device_count() <= 0:
            raise RgsUnavailableError("no CUDA device visible: the B200 path has no CPU fallback")
        h = _vp()
        rc = L.rgs_ctx_create(device, ctypes.byref(h))
        if rc != RGS_OK:
            raise RgsUnavailableError(f"rgs_ctx_create failed ({rc})")
        self.L, self.h, self.device = L, h, device
        self._torch_stream = use_torch_stream
        self.sync_stream()

    def sync_stream(self):
        """Order our next kernels after torch's work: on torch's current stream (the default),
        or -- a context on its own stream -- after torch's current stream has drained (its
        allocations / fills / copies of the tensors handed to us)."""
        if not self._torch_stream:
            try:
                import torch

                if torch.cuda.is_available() and torch.cuda.is_initialized():
                    torch.cuda.current_stream(self.device).synchronize()
            except ImportError:
                pass
            return
        try:
            import torch

            if torch.cuda.is_available():
                s = torch.cuda.current_stream(self.device).cuda_stream
                # torch's default stream is the legacy default stream (handle 0): pass
                # cudaStreamLegacy (0x1) -- NULL would select the context's own stream, which is
                # not ordered with torch's work on the legacy stream
                self.L.rgs_ctx_set_stream(self.h, _vp(s if s else _CUDA_STREAM_LEGACY))
        except ImportError:
            pass

    def status(self):
        """Raises (and clears) the first error of the deferred-check calls since the last call
        (FLAG_DEFER_CHECKS forwards / consistency); synchronises."""
        self.check(self.L.rgs_ctx_status(self.h))

    def status_async(self, word) -> None:
        """Queues a copy of the deferred status word into ``word`` (pinned int64 tensor of one
        element; -1 = clean), no synchronisation."""
        self.check(self.L.rgs_ctx_status_async(self.h, _vp(word.data_ptr())))

    def fence(self):
        """Order later torch-stream work after this context's stream: a no-op when the context
        runs on torch's current stream, a stream synchronisation otherwise."""
        if not self._torch_stream:
            self.synchronize()

    def adopt(self, child) -> None:
        """Registers a handle owner (scene, records, optimizer) to be closed before this
        context: in a garbage cycle the finalisers run in any order, and a child's destroy
        call needs its context alive."""
        import weakref

        if getattr(self, "_children", None) is None:
            self._children = weakref.WeakSet()
        self._children.add(child)

    def close(self):
        if getattr(self, "h", None):
            for child in list(getattr(self, "_children", None) or ()):
                try:
                    child.close()
                except Exception:
                    pass
            self.L.rgs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_launches(self) -> int:
        return int(self.L.rgs_ctx_kernel_launches(self.h))

    def check(self, rc: int):
        if rc == RGS_OK:
            return
        msg = self.L.rgs_ctx_last_error(self.h).decode()
        idx = self.L.rgs_ctx_error_index(self.h)
        if rc == RGS_E_MISSING_RECORDS:
            raise MissingRecordsError(msg)
        if rc == RGS_E_ZERO_ROTOR:
            raise ZeroRotorError(msg, idx)
        if rc == RGS_E_NONFINITE_ROTOR:
            raise NonFiniteRotorError(msg, idx)
        if rc == RGS_E_CAMERA:
            raise CameraError(msg)
        if rc == RGS_E_OVERFLOW:
            raise PairOverflowError(msg)
        if rc == RGS_E_CHECKPOINT:
            raise CheckpointError(msg)
        if rc == RGS_E_DEGENERATE_TIME:
            raise DegenerateTimeError(msg, idx)
        if rc == RGS_E_NO_DEVICE:
            raise RgsUnavailableError(msg)
        raise RgsCudaError(f"[{rc}] {msg}")

    def synchronize(self):
        self.check(self.L.rgs_ctx_synchronize(self.h))

    def set_binning(self, mode):
        """Binning of the (tile, splat) pairs (same result, different cost profile): "auto" (the
        tile-major scatter for single views, the radix passes for multi-view batches), "radix",
        "scatter" -- or BINNING_AUTO / BINNING_RADIX / BINNING_SCATTER."""
        m = {"auto": BINNING_AUTO, "radix": BINNING_RADIX, "scatter": BINNING_SCATTER}.get(mode, mode)
        self.check(self.L.rgs_ctx_set_binning(self.h, int(m)))

    # --- profiling (CUDA events per pipeline stage, on the launching stream)
    def set_profiling(self, timing=True, count_evals: bool = False):
        """timing: True / 1 = every stage, views serialised; "live" / 2 = only the FP32 blend,
        timed on its own stream inside a normal (pipelined) run."""
        t = 2 if timing == "live" else int(timing)
        self.check(self.L.rgs_ctx_set_profiling(self.h, t, int(count_evals)))

    def slow_reasons(self):
        """{reason: count} of the FP32 blend's slow-pixel decisions (count_evals profiling)."""
        out = (ctypes.c_ulonglong * 4)()
        self.check(self.L.rgs_ctx_profile_slow_reasons(self.h, out))
        return dict(zip(("power_gate", "alpha_gate", "clamp_gate", "T_gate"), [int(x) for x in out]))

    def blend_visits(self):
        """(warp visits, visits where some lane blended) of the FP32 blend (count_evals profiling)."""
        out = (ctypes.c_ulonglong * 2)()
        self.check(self.L.rgs_ctx_profile_blend_visits(self.h, out))
        return int(out[0]), int(out[1])

    def measure_fp32_tflops(self) -> float:
        v = ctypes.c_double(0)
        self.check(self.L.rgs_measure_fp32_tflops(self.h, ctypes.byref(v)))
        return v.value

    def measure_fp64_tflops(self) -> float:
        v = ctypes.c_double(0)
        self.check(self.L.rgs_measure_fp64_tflops(self.h, ctypes.byref(v)))
        return v.value

    def profile_reset(self):
        self.check(self.L.rgs_ctx_profile_reset(self.h))

    def profile_read(self):
        """{stage: (total_ms, launches)}, (E, B, E_kernel)."""
        k = self.L.rgs_profile_num_stages()
        ms = (ctypes.c_double * k)()
        cnt = (ctypes.c_longlong * k)()
        ev = (ctypes.c_ulonglong * 3)()
        self.check(self.L.rgs_ctx_profile_read(self.h, ms, cnt, ev))
        names = [self.L.rgs_profile_stage_name(i).decode() for i in range(k)]
        return {names[i]: (ms[i], cnt[i]) for i in range(k)}, (ev[0], ev[1], ev[2])

    # --- scenes
    def scene(self, store: GaussianStore) -> "DeviceScene":
        return DeviceScene.from_store(self, store)

    # --- device-resident batch render (bench hot path)
    def render_views(self, scene: "DeviceScene", cams: Sequence[Camera], background=(0.0, 0.0, 0.0),
                     out=None, blend_fp64=False):
        import torch

        self.sync_stream()
        n = len(cams)
        h, w = cams[0].height, cams[0].width
        if out is None:
            out = torch.empty((n, h, w, 3), dtype=torch.float32, device=f"cuda:{self.device}")
        arr = (CCamera * n)(*[c.to_c() for c in cams])
        bg = (ctypes.c_double * 3)(*[float(b) for b in background])
        flags = FLAG_BLEND_FP64 if blend_fp64 else 0
        self.check(self.L.rgs_render_views(self.h, scene.h, arr, n, bg, flags, _vp(_ptr(out))))
        return out

    def render_views_host(self, store_f32, sh_degree: int, cams: Sequence[Camera], background, images_host):
        """End-to-end host path (host scene in, host images out)."""
        mean, ls, rot, op, sh = store_f32
        n = op.shape[0]
        arr = (CCamera * len(cams))(*[c.to_c() for c in cams])
        bg = (ctypes.c_double * 3)(*[float(b) for b in background])
        self.check(self.L.rgs_render_views_host(self.h, n, sh_degree, _vp(_ptr(mean)), _vp(_ptr(ls)),
                                                _vp(_ptr(rot)), _vp(_ptr(op)), _vp(_ptr(sh)), arr, len(cams), bg,
                                                _vp(_ptr(images_host))))
        return images_host

    def render_forward_device(self, scene: "DeviceScene", cam: Camera, background=(0.0, 0.0, 0.0), retain=True,
                              blend_fp64=False, image=None, defer_checks=False):
        import torch

        self.sync_stream()
        if image is None:
            image = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device=f"cuda:{self.device}")
        c = cam.to_c()
        bg = (ctypes.c_double * 3)(*[float(b) for b in background])
        flags = (FLAG_RETAIN_RECORDS if retain else 0) | (FLAG_BLEND_FP64 if blend_fp64 else 0)
        if defer_checks:  # no host sync: errors / overflow via status() / status_async()
            flags |= FLAG_DEFER_CHECKS
        h = _vp()
        self.check(self.L.rgs_render_forward(self.h, scene.h, ctypes.byref(c), bg, flags, _vp(_ptr(image)),
                                             ctypes.byref(h)))
        self.fence()
        return image, RenderRecords(self, h, cam, background, retain)

    def render_backward_device(self, scene: "DeviceScene", cam: Camera, records: "RenderRecords", dL_dimage,
                               grads=None, vnorm=None, visible=None, accumulate=False, deterministic=False,
                               reproducible=False):
        """``deterministic``: RGS_FLAG_DETERMINISTIC (the reference-order FP64 replay, bitwise
        repeatable); ``reproducible``: RGS_FLAG_REPRODUCIBLE (the production path with
        order-independent fixed-point accumulation, bitwise repeatable)."""
        import torch

        self.sync_stream()
        n = scene.n
        dev = f"cuda:{self.device}"
        if grads is None:
            grads = torch.zeros(65 * n, dtype=torch.float32, device=dev)
            vnorm = torch.zeros(n, dtype=torch.float32, device=dev)
            visible = torch.zeros(n, dtype=torch.int32, device=dev)
        c = cam.to_c()
        flags = (FLAG_ACCUMULATE if accumulate else 0) | (FLAG_DETERMINISTIC if deterministic else 0) | \
            (FLAG_REPRODUCIBLE if reproducible else 0)
        dl = dL_dimage.contiguous()
        self.sync_stream()  # (after the gradient buffers' allocation / fill on torch's stream)
        self.check(self.L.rgs_render_backward(self.h, scene.h, ctypes.byref(c), records.h, _vp(_ptr(dl)), flags,
                                              _vp(_ptr(grads)), _vp(_ptr(vnorm)), _vp(_ptr(visible))))
        self.fence()
        return grads, vnorm, visible


class DeviceScene:
    """A device-resident rgs_scene (SoA, rgs_scene_params layout): FP32 storage, or
    FP64 (``f64=True``, RGS_SCENE_F64) when the store's doubles must reach the
    kernels unrounded."""

    def __init__(self, ctx: Context, n: int, sh_degree: int, f64: bool = False):
        h = _vp()
        ctx.check(ctx.L.rgs_scene_create_ex(ctx.h, n, sh_degree, SCENE_F64 if f64 else 0, ctypes.byref(h)))
        self.ctx, self.h, self.n, self.sh_degree, self.f64 = ctx, h, n, sh_degree, f64
        ctx.adopt(self)
        self.n_inexact = 0

    @staticmethod
    def from_store(ctx: Context, store: GaussianStore, f64: bool = False) -> "DeviceScene":
        s = DeviceScene(ctx, store.size(), store.active_sh_degree, f64=f64)
        s.upload(store)
        return s

    def upload(self, store: GaussianStore):
        arrs = store.arrays_f64()
        inexact = ctypes.c_longlong(0)
        self.ctx.check(self.ctx.L.rgs_scene_upload_f64(self.ctx.h, self.h, *[_vp(a.ctypes.data) for a in arrs],
                                                       ctypes.byref(inexact)))
        self.n_inexact = inexact.value
        self.sh_degree = store.active_sh_degree
        self.ctx.L.rgs_scene_set_sh_degree(self.h, store.active_sh_degree)

    @staticmethod
    def load_checkpoint(ctx: Context, path: str, f64: bool = False) -> "DeviceScene":
        """load_checkpoint (checkpoint.cpp:54-86) straight into device memory."""
        h = _vp()
        ctx.check(ctx.L.rgs_scene_load_checkpoint(ctx.h, os.fsencode(path), SCENE_F64 if f64 else 0, ctypes.byref(h)))
        s = DeviceScene.__new__(DeviceScene)
        s.ctx, s.h, s.f64, s.n_inexact = ctx, h, f64, 0
        ctx.adopt(s)
        s.n = int(ctx.L.rgs_scene_size(h))
        s.sh_degree = -1
        return s

    def save_checkpoint(self, path: str):
        """save_checkpoint (checkpoint.cpp:29-52)."""
        self.ctx.check(self.ctx.L.rgs_scene_save_checkpoint(self.ctx.h, self.h, os.fsencode(path)))

    def download(self):
        """Device scene -> (mean, log_scales, rotor, opacity_logit, sh) float64 host arrays."""
        n = self.n
        out = (np.zeros((n, 4)), np.zeros((n, 4)), np.zeros((n, 8)), np.zeros(n), np.zeros((n, 48)))
        self.ctx.check(self.ctx.L.rgs_scene_download_f64(self.ctx.h, self.h, *[_vp(a.ctypes.data) for a in out]))
        return out

    def params_tensor(self):
        """The device parameter buffer (rgs_scene_params layout: 65 x N float32, or float64 for
        FP64 scenes) as a torch tensor view -- e.g. to broadcast a replica with NCCL."""
        import torch

        class _View:
            pass

        v = _View()
        v.__cuda_array_interface__ = {"shape": (65 * self.n,), "typestr": "<f8" if self.f64 else "<f4",
                                      "data": (self.params_ptr(), False), "version": 3}
        return torch.as_tensor(v, device=f"cuda:{self.ctx.device}")

    def params_ptr(self) -> int:
        fn =self.ctx.L.rgs_scene_params_f64 if self.f64 else self.ctx.L.rgs_scene_params
        return int(fn(self.h) or 0)

    def close(self):
        if getattr(self, "h", None):
            if getattr(self.ctx, "h", None):  # (a closed context already freed it)
                self.ctx.L.rgs_scene_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RenderRecords:
    """RenderRecords (rasterizer.hpp:61-70), device-resident; host views on demand."""

    def __init__(self, ctx: Context, handle, cam: Camera, background, retained: bool):
        self.ctx, self.h = ctx, handle
        self.background = np.asarray(background, dtype=np.float64)
        self.retained = bool(retained)
        self._cache = None
        self._info = None  # read on first use (the read synchronises)
        ctx.adopt(self)

    def _get_info(self):
        if self._info is None:
            info = CRecordsInfo()
            self.ctx.check(self.ctx.L.rgs_records_info_get(self.h, ctypes.byref(info)))
            self._info = info
        return self._info

    tiles_x = property(lambda self: self._get_info().tiles_x)
    tiles_y = property(lambda self: self._get_info().tiles_y)
    n_pairs = property(lambda self: self._get_info().n_pairs)
    n_slow_pixels = property(lambda self: self._get_info().n_slow_pixels)
    width = property(lambda self: self._get_info().width)
    height = property(lambda self: self._get_info().height)
    _n_splats = property(lambda self: self._get_info().n_splats)

    def _export(self):
        if self._cache is None:
            nt = self.tiles_x * self.tiles_y
            splats = np.zeros(self._n_splats, dtype=SPLAT_DTYPE)
            off = np.zeros(nt + 1, dtype=np.int64)
            ids = np.zeros(max(self.n_pairs, 1), dtype=np.int32)
            fT = np.zeros((self.height, self.width), dtype=np.float64)
            nc = np.zeros((self.height, self.width), dtype=np.int32)
            self.ctx.check(self.ctx.L.rgs_records_export(self.ctx.h, self.h, _vp(splats.ctypes.data),
                                                         _vp(off.ctypes.data), _vp(ids.ctypes.data),
                                                         _vp(fT.ctypes.data), _vp(nc.ctypes.data)))
            self._cache = (splats, off, ids[: self.n_pairs], fT, nc)
        return self._cache

    @property
    def splats(self):
        return self._export()[0]

    @property
    def tile_offsets(self):
        return self._export()[1]

    @property
    def tile_ids(self):
        return self._export()[2]

    @property
    def tile_splats(self):
        _, off, ids, _, _ = self._export()
        return [ids[off[t]: off[t + 1]] for t in range(len(off) - 1)]

    @property
    def final_T(self):
        return self._export()[3]

    @property
    def n_contrib(self):
        return self._export()[4]

    def close(self):
        if getattr(self, "h", None):
            self.ctx.L.rgs_records_destroy(self.h)  # safe after the context: orphaned records
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class RenderOutput:
    image: np.ndarray  # (H, W, 3) float32
    records: RenderRecords


# ----------------------------------------------------------------------------- drop-in functions
_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0, use_torch_stream=False)
    return _default_ctx


def render_forward(store: GaussianStore, cam: Camera, opts: RenderOptions = RenderOptions(),
                   ctx: Optional[Context] = None) -> RenderOutput:
    """rasterizer.cpp:308-318.  Returns the image (float32) and the records."""
    ctx = ctx or default_context()
    cam.validate()
    scene = DeviceScene.from_store(ctx, store, f64=True)  # the store's doubles, unrounded
    img = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
    c = cam.to_c()
    bg = (ctypes.c_double * 3)(*[float(b) for b in opts.background])
    flags = FLAG_HOST_BUFFERS | (FLAG_RETAIN_RECORDS if opts.retain_records else 0) | (
        FLAG_BLEND_FP64 if opts.blend_fp64 else 0)
    h = _vp()
    ctx.check(ctx.L.rgs_render_forward(ctx.h, scene.h, ctypes.byref(c), bg, flags, _vp(img.ctypes.data),
                                       ctypes.byref(h)))
    rec = RenderRecords(ctx, h, cam, opts.background, opts.retain_records)
    rec._scene = scene  # keep alive (backward re-reads the parameters)
    return RenderOutput(img, rec)


PROJECT_CACHE_DOUBLES = 85  # RGS_PROJECT_CACHE_DOUBLES (include/rgs_cuda.h)


def project(sliced16, cam: Camera, sh48, sh_degree: int, opacity_logit: float, ctx: Optional[Context] = None,
            want_cache: bool = False):
    """project() of one already-sliced Gaussian (rasterizer.hpp:52-54): sliced16 = mean[3],
    cov[9] row-major, decay, speed[3]; sh48 channel-major.  Returns the SPLAT_DTYPE record (None
    when culled) and, with want_cache, ProjectCache's fields as rgs_project_sliced_cache's flat
    layout (p_cam, T, cov2, dir, view_dist, basis, basis_grad, clamped, opacity)."""
    ctx = ctx or default_context()
    sl = np.ascontiguousarray(sliced16, dtype=np.float64)
    sh = np.ascontiguousarray(sh48, dtype=np.float64)
    out = np.zeros(1, dtype=SPLAT_DTYPE)
    cache = np.zeros(PROJECT_CACHE_DOUBLES, dtype=np.float64) if want_cache else None
    surv = ctypes.c_int(0)
    c = cam.to_c()
    ctx.check(ctx.L.rgs_project_sliced_cache(ctx.h, _vp(sl.ctypes.data), ctypes.byref(c), _vp(sh.ctypes.data),
                                             int(sh_degree), float(opacity_logit), _vp(out.ctypes.data),
                                             ctypes.byref(surv), _vp(cache.ctypes.data) if want_cache else None))
    if not surv.value:
        return (None, None) if want_cache else None
    return (out[0], cache) if want_cache else out[0]


def rasterize_forward(splats: np.ndarray, cam: Camera, background=(0.0, 0.0, 0.0), threads: int = 1,
                      ctx: Optional[Context] = None, blend_fp64: bool = False):
    """rasterizer.cpp:278-306 on already-projected splats (SPLAT_DTYPE array)."""
    ctx = ctx or default_context()
    sp = np.ascontiguousarray(splats, dtype=SPLAT_DTYPE)
    img = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
    c = cam.to_c()
    bg = (ctypes.c_double * 3)(*[float(b) for b in background])
    flags = FLAG_HOST_BUFFERS | (FLAG_BLEND_FP64 if blend_fp64 else 0)
    h = _vp()
    ctx.check(ctx.L.rgs_rasterize_forward(ctx.h, _vp(sp.ctypes.data), len(sp), ctypes.byref(c), bg, flags,
                                          _vp(img.ctypes.data), ctypes.byref(h)))
    return img, RenderRecords(ctx, h, cam, background, False)


def render_backward(store: GaussianStore, cam: Camera, records: RenderRecords, dL_dimage: np.ndarray,
                    threads: int = 1, ctx: Optional[Context] = None) -> StoreGrads:
    """rasterizer.cpp:320-397."""
    import torch

    if not records.retained:
        raise MissingRecordsError("rasterize_backward: forward pass did not retain records")
    ctx = ctx or records.ctx
    scene = getattr(records, "_scene", None)
    if scene is None or scene.n != store.size():
        scene = DeviceScene.from_store(ctx, store, f64=True)
    n = store.size()
    dev = f"cuda:{ctx.device}"
    dl = torch.from_numpy(np.ascontiguousarray(dL_dimage, dtype=np.float32)).to(dev)
    grads = torch.zeros(65 * max(n, 1), dtype=torch.float32, device=dev)
    vnorm = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
    vis = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    torch.cuda.synchronize(dev)
    c = cam.to_c()
    ctx.check(ctx.L.rgs_render_backward(ctx.h, scene.h, ctypes.byref(c), records.h, _vp(dl.data_ptr()), 0,
                                        _vp(grads.data_ptr()), _vp(vnorm.data_ptr()), _vp(vis.data_ptr())))
    ctx.synchronize()
    mean, ls, rot, op, sh = grads_from_soa(grads.cpu().numpy(), n) if n else (np.zeros((0, 4)),) * 5
    return StoreGrads(mean, ls, rot, op, sh, vnorm.cpu().numpy()[:n].astype(np.float64),
                      vis.cpu().numpy()[:n].astype(np.uint8))


def render_flow(store: GaussianStore, cam: Camera, threads: int = 1, ctx: Optional[Context] = None) -> np.ndarray:
    """rasterizer.cpp:399-425.  (H, W, 2) screen-space velocity image."""
    ctx = ctx or default_context()
    cam.validate()
    scene = DeviceScene.from_store(ctx, store, f64=True)
    import torch

    dev = f"cuda:{ctx.device}"
    flow = torch.zeros((cam.height, cam.width, 2), dtype=torch.float32, device=dev)
    torch.cuda.synchronize(dev)
    c = cam.to_c()
    ctx.check(ctx.L.rgs_render_flow(ctx.h, scene.h, ctypes.byref(c), 0, _vp(flow.data_ptr())))
    ctx.synchronize()
    return flow.cpu().numpy()
