"""ctypes bindings for the CPU oracle libraries.

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs; the product (paper_2402_03307_b200) never imports it.

Two libraries share one C signature set:
  * ``liboracle.so``        — oracle/rgs_oracle.c, the plain-C restatement (prefix ``orc_``)
  * ``_ref/librgs_ref.so``  — the reference's own render sources compiled in place
                              (prefix ``ref_``); only present where it was built.

Scene arrays follow the "host scene" layout of include/rgs_cuda.h:
mean (N,4), log_scales (N,4), rotor (N,8), opacity_logit (N,), sh (N,3,16)
channel-major, all float64.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librgs_ref.so")

_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


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
assert SPLAT_DTYPE.itemsize == 112


def make_ccamera(cam) -> CCamera:
    c = CCamera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    w2c = np.asarray(cam.world_to_camera, dtype=np.float64).reshape(16)
    for i in range(16):
        c.world_to_camera[i] = float(w2c[i])
    c.time = float(cam.time)
    return c


def _p(a):
    return a.ctypes.data_as(_vp) if a is not None else None


@dataclass
class Records:
    splats: np.ndarray  # SPLAT_DTYPE
    tile_offsets: np.ndarray  # int64 (tiles+1)
    tile_ids: np.ndarray  # int32
    final_T: np.ndarray  # float64 (H,W)
    n_contrib: np.ndarray  # int32 (H,W)
    retained: bool
    handle: object = None  # live C handle for backward

    def tile_list(self, t):
        return self.tile_ids[self.tile_offsets[t] : self.tile_offsets[t + 1]]


class OracleLib:
    """One of the two CPU libraries (restatement or reference build)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.path, self.prefix = path, prefix
        self.lib = ctypes.CDLL(path)
        f = self._f
        f("last_error").restype = ctypes.c_char_p
        for name in ("records_num_splats", "records_num_tiles", "records_retained"):
            f(name).restype = ctypes.c_int
            f(name).argtypes = [_vp]
        f("records_num_pairs").restype = ctypes.c_longlong
        f("records_num_pairs").argtypes = [_vp]
        f("records_free").argtypes = [_vp]
        for name in ("records_splats", "records_tiles", "records_pixels"):
            f(name).restype = None
        self._free = f("records_free")

    def _f(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def _check(self, rc):
        if rc != 0:
            msg = self._f("last_error")().decode()
            raise OracleError(rc, msg)

    @staticmethod
    def _scene(store):
        mean = np.ascontiguousarray(store.mean, dtype=np.float64)
        ls = np.ascontiguousarray(store.log_scales, dtype=np.float64)
        rot = np.ascontiguousarray(store.rotor, dtype=np.float64)
        op = np.ascontiguousarray(store.opacity_logit, dtype=np.float64)
        sh = np.ascontiguousarray(store.sh, dtype=np.float64)
        return mean, ls, rot, op, sh

    def _records(self, h, cam, retained_default=None):
        ns = self._f("records_num_splats")(h)
        nt = self._f("records_num_tiles")(h)
        npairs = self._f("records_num_pairs")(h)
        splats = np.zeros(ns, dtype=SPLAT_DTYPE)
        self._f("records_splats")(_vp(h), _p(splats))
        off = np.zeros(nt + 1, dtype=np.int64)
        ids = np.zeros(max(npairs, 1), dtype=np.int32)
        self._f("records_tiles")(_vp(h), _p(off), _p(ids))
        fT = np.zeros((cam.height, cam.width), dtype=np.float64)
        nc = np.zeros((cam.height, cam.width), dtype=np.int32)
        self._f("records_pixels")(_vp(h), _p(fT), _p(nc))
        ret = bool(self._f("records_retained")(h))
        return Records(splats, off, ids[:npairs], fT, nc, ret, _Handle(self, h))

    def render_forward(self, store, cam, background=(0.0, 0.0, 0.0), threads=1, retain=False):
        mean, ls, rot, op, sh = self._scene(store)
        c = make_ccamera(cam)
        bg = np.asarray(background, dtype=np.float64)
        img = np.zeros((cam.height, cam.width, 3), dtype=np.float64)
        h = _vp()
        rc = self._f("render_forward")(
            ctypes.c_int(len(op)), _p(mean), _p(ls), _p(rot), _p(op), _p(sh),
            ctypes.c_int(store.active_sh_degree), ctypes.byref(c), _p(bg), ctypes.c_int(threads),
            ctypes.c_int(1 if retain else 0), _p(img), ctypes.byref(h))
        self._check(rc)
        return img, self._records(h.value, cam)

    def rasterize_forward(self, splats, cam, background=(0.0, 0.0, 0.0), threads=1):
        sp = np.ascontiguousarray(splats, dtype=SPLAT_DTYPE)
        c = make_ccamera(cam)
        bg = np.asarray(background, dtype=np.float64)
        img = np.zeros((cam.height, cam.width, 3), dtype=np.float64)
        h = _vp()
        rc = self._f("rasterize_forward")(ctypes.c_int(len(sp)), _p(sp), ctypes.byref(c), _p(bg),
                                         ctypes.c_int(threads), _p(img), ctypes.byref(h))
        self._check(rc)
        return img, self._records(h.value, cam)

    def render_backward(self, store, cam, records, dL_dimage, threads=1):
        mean, ls, rot, op, sh = self._scene(store)
        c = make_ccamera(cam)
        n = len(op)
        dl = np.ascontiguousarray(dL_dimage, dtype=np.float64)
        grads = np.zeros((n, 65), dtype=np.float64)
        vnorm = np.zeros(n, dtype=np.float64)
        vis = np.zeros(n, dtype=np.uint8)
        rc = self._f("render_backward")(
            ctypes.c_int(n), _p(mean), _p(ls), _p(rot), _p(op), _p(sh),
            ctypes.c_int(store.active_sh_degree), ctypes.byref(c), _vp(records.handle.h), _p(dl),
            ctypes.c_int(threads), _p(grads), _p(vnorm), _p(vis))
        self._check(rc)
        return grads, vnorm, vis

    def render_flow(self, store, cam, threads=1):
        mean, ls, rot, op, sh = self._scene(store)
        c = make_ccamera(cam)
        flow = np.zeros((cam.height, cam.width, 2), dtype=np.float64)
        rc = self._f("render_flow")(ctypes.c_int(len(op)), _p(mean), _p(ls), _p(rot), _p(op), _p(sh),
                                   ctypes.c_int(store.active_sh_degree), ctypes.byref(c),
                                   ctypes.c_int(threads), _p(flow))
        self._check(rc)
        return flow

    def naive_render(self, store, cam, background=(0.0, 0.0, 0.0)):
        mean, ls, rot, op, sh = self._scene(store)
        c = make_ccamera(cam)
        bg = np.asarray(background, dtype=np.float64)
        img = np.zeros((cam.height, cam.width, 3), dtype=np.float64)
        ws = np.zeros((cam.height, cam.width), dtype=np.float64)
        ft = np.zeros((cam.height, cam.width), dtype=np.float64)
        rc = self._f("naive_render")(ctypes.c_int(len(op)), _p(mean), _p(ls), _p(rot), _p(op), _p(sh),
                                    ctypes.c_int(store.active_sh_degree), ctypes.byref(c), _p(bg),
                                    _p(img), _p(ws), _p(ft))
        self._check(rc)
        return img, ws, ft

    def slice_at(self, mean, ls, rot, t):
        out = np.zeros(17, dtype=np.float64)
        rc = self._f("slice_at")(_p(np.ascontiguousarray(mean, np.float64)),
                                 _p(np.ascontiguousarray(ls, np.float64)),
                                 _p(np.ascontiguousarray(rot, np.float64)), ctypes.c_double(t), _p(out))
        self._check(rc)
        return out

    def normalize(self, rot):
        out = np.zeros(8, dtype=np.float64)
        self._check(self._f("normalize")(_p(np.ascontiguousarray(rot, np.float64)), _p(out)))
        return out

    def to_matrix(self, rot):
        out = np.zeros(16, dtype=np.float64)
        self._check(self._f("to_matrix")(_p(np.ascontiguousarray(rot, np.float64)), _p(out)))
        return out.reshape(4, 4)

    def project_cache(self, sliced16, cam, sh48, sh_degree, opacity_logit):
        """project() with its ProjectCache, flattened as rgs_project_sliced_cache (reference build)."""
        c = make_ccamera(cam)
        out = np.zeros(1, dtype=SPLAT_DTYPE)
        pc = np.zeros(85, dtype=np.float64)
        r = self._f("project_cache")(_p(np.ascontiguousarray(sliced16, np.float64)), ctypes.byref(c),
                                     _p(np.ascontiguousarray(sh48, np.float64)), ctypes.c_int(sh_degree),
                                     ctypes.c_double(opacity_logit), _p(out), _p(pc))
        if r < 0:
            self._check(-r)
        return (out[0], pc) if r == 1 else (None, None)

    def project(self, sliced16, cam, sh48, sh_degree, opacity_logit):
        c = make_ccamera(cam)
        out = np.zeros(1, dtype=SPLAT_DTYPE)
        r = self._f("project")(_p(np.ascontiguousarray(sliced16, np.float64)), ctypes.byref(c),
                               _p(np.ascontiguousarray(sh48, np.float64)), ctypes.c_int(sh_degree),
                               ctypes.c_double(opacity_logit), _p(out))
        if r < 0:
            self._check(-r)
        return out[0] if r == 1 else None


class _Handle:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib._free(_vp(self.h))
        except Exception:
            pass


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_cache = {}


def restatement() -> OracleLib:
    if "orc" not in _cache:
        _cache["orc"] = OracleLib(ORACLE_SO, "orc")
    return _cache["orc"]


def reference_build() -> OracleLib:
    if "ref" not in _cache:
        _cache["ref"] = OracleLib(REF_SO, "ref")
    return _cache["ref"]


def sum_order_variant(order: int) -> OracleLib:
    """The restatement built with ORC_SUM_ORDER=order (Eigen 3.4's reduction orders; see
    rgs_oracle.c): the summation-order sensitivity study only."""
    key = f"sum{order}"
    if key not in _cache:
        _cache[key] = OracleLib(os.path.join(HERE, "_ref", f"liboracle_sum{order}.so"), "orc")
    return _cache[key]


def reference_available() -> bool:
    return os.path.exists(REF_SO)


# ----------------------------------------------------------------------------- training side
class CAdamConfig(ctypes.Structure):
    """TrainConfig subset used by adam_step (optim.hpp:17-63); defaults = the reference's."""

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
    ]


def adam_config(**kw) -> CAdamConfig:
    c = CAdamConfig(1.6e-4, 1.6e-6, 5e-3, 1e-3, 2.5e-3, 1.25e-4, 0.05, 2000, 0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class CLossWeights(ctypes.Structure):
    """LossWeights (loss.hpp:11-16)."""

    _fields_ = [
        ("lambda_ssim", ctypes.c_double),
        ("lambda_entropy", ctypes.c_double),
        ("lambda_consistency", ctypes.c_double),
        ("k_neighbors", ctypes.c_int),
    ]


def loss_weights(**kw) -> CLossWeights:
    c = CLossWeights(0.2, 0.01, 0.05, 8)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _d(x):
    return np.ascontiguousarray(x, dtype=np.float64)


class TrainOps:
    """Training-side entry points of one oracle library (restatement `orc_` or reference `ref_`)."""

    def __init__(self, lib: OracleLib):
        self.o = lib
        self.L = lib.lib
        self.ref = lib.prefix == "ref"
        f = lib._f
        for name in ("psnr", "entropy_loss", "consistency_loss", "lr_schedule"):
            f(name).restype = ctypes.c_double
        f("lr_schedule").argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double]
        if not self.ref:
            f("l1_loss").restype = ctypes.c_double
        self.f = f

    def _check(self, rc):
        if rc != 0:
            name = "train_last_error" if self.ref else "last_error"
            msg = getattr(self.L, f"{self.o.prefix}_{name}")
            msg.restype = ctypes.c_char_p
            raise OracleError(rc, msg().decode())

    def l1_loss(self, rendered, target, want_grad=True):
        a, b = _d(rendered), _d(target)
        g = np.zeros_like(a) if want_grad else None
        if self.ref:
            loss = ctypes.c_double(0)
            h, w = a.shape[:2]
            self._check(self.f("l1_loss")(ctypes.c_int(w), ctypes.c_int(h), _p(a), _p(b), ctypes.byref(loss), _p(g)))
            return loss.value, g
        return self.f("l1_loss")(ctypes.c_longlong(a.size), _p(a), _p(b), _p(g)), g

    def psnr(self, a, b):
        a, b = _d(a), _d(b)
        if self.ref:
            h, w = a.shape[:2]
            return self.f("psnr")(ctypes.c_int(w), ctypes.c_int(h), _p(a), _p(b))
        return self.f("psnr")(ctypes.c_longlong(a.size), _p(a), _p(b))

    def ssim_loss(self, rendered, target, want_grad=True):
        a, b = _d(rendered), _d(target)
        h, w = a.shape[:2]
        g = np.zeros_like(a) if want_grad else None
        loss = ctypes.c_double(0)
        self._check(self.f("ssim_loss")(ctypes.c_int(w), ctypes.c_int(h), _p(a), _p(b), ctypes.byref(loss), _p(g)))
        return loss.value, g

    def entropy_loss(self, opacities, want_grad=True):
        o = _d(opacities)
        g = np.zeros_like(o) if want_grad else None
        return self.f("entropy_loss")(ctypes.c_int(len(o)), _p(o), _p(g)), g

    def consistency_loss(self, speeds, nbrs, want_grad=True):
        s = _d(speeds)
        nb = np.ascontiguousarray(nbrs, dtype=np.int32)
        g = np.zeros_like(s) if want_grad else None
        v = self.f("consistency_loss")(ctypes.c_int(len(s)), _p(s), ctypes.c_int(nb.shape[1]), _p(nb), _p(g))
        return v, g

    def scene_scales(self, mean):
        m = _d(mean)
        out = np.zeros(4)
        self.f("scene_scales")(ctypes.c_int(len(m)), _p(m), _p(out))
        return out

    def knn4d(self, mean, k, scales, threads=4):
        m = _d(mean)
        out = np.zeros((len(m), k), dtype=np.int32)
        name = "build_knn4d" if self.ref else "knn4d"
        self._check(self.f(name)(ctypes.c_int(len(m)), _p(m), ctypes.c_int(k), _p(_d(scales)), ctypes.c_int(threads),
                                 _p(out)))
        return out

    def gaussian_speeds(self, store):
        mean, ls, rot, _, _ = OracleLib._scene(store)
        out = np.zeros((len(mean), 3))
        self._check(self.f("gaussian_speeds")(ctypes.c_int(len(mean)), _p(mean), _p(ls), _p(rot), _p(out)))
        return out

    def lr_schedule(self, step, total, lr_init, lr_final):
        return self.f("lr_schedule")(step, total, lr_init, lr_final)

    def adam_step(self, store, m, v, grads, cfg, step):
        """In place on copies: returns (store', m', v')."""
        mean, ls, rot, op, sh = [a.copy() for a in OracleLib._scene(store)]
        m, v = _d(m).copy(), _d(v).copy()
        g = _d(grads)
        self._check(self.f("adam_step")(ctypes.c_int(len(op)), _p(mean), _p(ls), _p(rot), _p(op), _p(sh), _p(m), _p(v),
                                        _p(g), ctypes.byref(cfg), ctypes.c_int(step)))
        out = type(store)(mean, ls, rot, op, sh.reshape(store.sh.shape), store.active_sh_degree)
        return out, m, v

    def accumulate_stats(self, vnorm, visible, accum, count):
        accum, count = _d(accum).copy(), np.ascontiguousarray(count, dtype=np.int32).copy()
        vis = np.ascontiguousarray(visible, dtype=np.uint8)
        self.f("accumulate_stats")(ctypes.c_int(len(accum)), _p(_d(vnorm)), _p(vis), _p(accum), _p(count))
        return accum, count

    def reset_opacity(self, op, m_op, v_op, value=0.01):
        op, m_op, v_op = _d(op).copy(), _d(m_op).copy(), _d(v_op).copy()
        self.f("reset_opacity")(ctypes.c_int(len(op)), _p(op), _p(m_op), _p(v_op), ctypes.c_double(value))
        return op, m_op, v_op

    def evaluate_loss(self, store, cams, targets, weights, background=(0.0, 0.0, 0.0), nbrs=None, threads=4,
                      want_grads=True):
        mean, ls, rot, op, sh = OracleLib._scene(store)
        n = len(op)
        arr = (CCamera * len(cams))(*[make_ccamera(c) for c in cams])
        tg = np.ascontiguousarray(np.concatenate([_d(t).reshape(-1) for t in targets])) if len(targets) else np.zeros(1)
        losses = np.zeros(5)
        g = np.zeros((n, 65)) if want_grads else None
        vn = np.zeros(n) if want_grads else None
        vis = np.zeros(n, dtype=np.uint8) if want_grads else None
        nb = None if nbrs is None else np.ascontiguousarray(nbrs, dtype=np.int32)
        bg = _d(background)
        self._check(self.f("evaluate_loss")(ctypes.c_int(n), _p(mean), _p(ls), _p(rot), _p(op), _p(sh),
                                            ctypes.c_int(store.active_sh_degree), ctypes.c_int(len(cams)), arr,
                                            _p(tg), ctypes.byref(weights), _p(bg), _p(nb), ctypes.c_int(threads),
                                            _p(losses), _p(g), _p(vn), _p(vis)))
        return losses, g, vn, vis


def train_ops(which: str = "orc") -> TrainOps:
    key = "train_" + which
    if key not in _cache:
        _cache[key] = TrainOps(restatement() if which == "orc" else reference_build())
    return _cache[key]


class CDensifyConfig(ctypes.Structure):
    """TrainConfig's adaptive density control fields (optim.hpp:31-42)."""

    _fields_ = [
        ("densify_grad_threshold", ctypes.c_double),
        ("percent_dense", ctypes.c_double),
        ("split_factor", ctypes.c_double),
        ("prune_opacity", ctypes.c_double),
        ("min_gaussians", ctypes.c_int),
        ("max_gaussians", ctypes.c_int),
        ("static_mode", ctypes.c_int),
    ]


def densify_config(**kw) -> CDensifyConfig:
    c = CDensifyConfig(2e-4, 0.01, 1.6, 0.005, 16, 200000, 0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def ref_densify_and_prune(store, m, v, accum, count, cfg, extent, seed):
    """optim.cpp:168-234 in the reference build (no restatement: pinned directly)."""
    L = reference_build().lib
    mean, ls, rot, op, sh = OracleLib._scene(store)
    n = len(op)
    cap = 3 * n + 8
    outs = [np.zeros((cap, 4)), np.zeros((cap, 4)), np.zeros((cap, 8)), np.zeros(cap), np.zeros((cap, 48)),
            np.zeros((cap, 65)), np.zeros((cap, 65)), np.zeros(cap), np.zeros(cap, dtype=np.int32)]
    rep = np.zeros(3, dtype=np.int32)
    f = L.ref_densify_and_prune
    f.restype = ctypes.c_int
    k = f(ctypes.c_int(n), _p(mean), _p(ls), _p(rot), _p(op), _p(sh), _p(_d(m)), _p(_d(v)), _p(_d(accum)),
          _p(np.ascontiguousarray(count, dtype=np.int32)), ctypes.byref(cfg), ctypes.c_double(extent),
          ctypes.c_ulonglong(seed), _p(rep), ctypes.c_int(cap), *[_p(o) for o in outs])
    if k < 0:
        raise OracleError(99, "ref_densify_and_prune failed")
    mean, ls, rot, op, sh, m, v, acc, cnt = [o[:k] for o in outs]
    st = type(store)(mean, ls, rot, op, sh.reshape(k, 3, 16), store.active_sh_degree)
    return st, m, v, acc, cnt, tuple(int(x) for x in rep)
