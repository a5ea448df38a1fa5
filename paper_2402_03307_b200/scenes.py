"""Synthetic 4D scenes and cameras for tests and benchmarks (host-side, numpy).

Scene recipe: SURVEY.md §8(d), following the reference's criterion-10 scene
(/root/reference/proj/tests/acceptance.cpp:493-520): Gaussians inside the view
frustum, few-pixel footprints (world scale x 400/W), half of them moving via a
velocity rotor (synthetic.cpp:134-177), SH degree 3.  Every parameter is rounded
to float32 so the device scene (FP32) and the CPU oracle (FP64) see identical
inputs.  numpy's PCG64 replaces std::mt19937_64, so draws are not the
reference's, but the distributions are.
"""
from __future__ import annotations

import numpy as np

from .rgs import Camera, GaussianStore

# ----------------------------------------------------------------------------- rotor algebra (vectorised)
# Even subalgebra blade masks in coefficient order s, b01, b02, b03, b12, b13, b23, p (rotor.cpp:74-75).
_MASKS = [0b0000, 0b0011, 0b0101, 0b1001, 0b0110, 0b1010, 0b1100, 0b1111]


def _blade_sign(a, b):
    sign, bb = 1, b
    while bb:
        i = (bb & -bb).bit_length() - 1
        bb &= bb - 1
        if bin(a >> (i + 1)).count("1") & 1:
            sign = -sign
    return sign


_COMPOSE = [[(_MASKS.index(_MASKS[i] ^ _MASKS[j]), _blade_sign(_MASKS[i], _MASKS[j])) for j in range(8)]
            for i in range(8)]


def compose(a, b):
    """Geometric product (rotor.cpp:206-216), rows of (N,8)."""
    out = np.zeros(np.broadcast(a, b).shape)
    for i in range(8):
        for j in range(8):
            t, s = _COMPOSE[i][j]
            out[..., t] += s * a[..., i] * b[..., j]
    return out


def from_quaternion(w, x, y, z):
    """rotor.cpp:196-204"""
    r = np.zeros(np.shape(w) + (8,))
    r[..., 0] = w
    r[..., 1] = -z
    r[..., 2] = y
    r[..., 4] = -x
    return r


def rotor_epsilon(v):
    return v[..., 7] * v[..., 0] - v[..., 1] * v[..., 6] + v[..., 2] * v[..., 5] - v[..., 3] * v[..., 4]


def normalize(v):
    """rotor.cpp:117-136 (vectorised; no error checks)."""
    v = np.array(v, dtype=np.float64)
    l2 = (v * v).sum(-1)
    eps = rotor_epsilon(v)
    g = np.stack([v[..., 7], -v[..., 6], v[..., 5], -v[..., 4], -v[..., 3], v[..., 2], -v[..., 1], v[..., 0]], -1)
    rad = np.maximum(l2 * l2 - 4 * eps * eps, 0)
    delta = np.where(np.abs(eps) >= 1e-12, -2 * eps / (l2 + np.sqrt(rad)), 0.0)
    v = v + delta[..., None] * g
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


_TERMS = [
    [(0, 0, 1), (1, 1, -1), (2, 2, -1), (3, 3, -1), (4, 4, 1), (5, 5, 1), (6, 6, 1), (7, 7, -1)],
    [(1, 0, 2), (2, 4, -2), (3, 5, -2), (6, 7, 2)],
    [(1, 4, 2), (2, 0, 2), (3, 6, -2), (5, 7, -2)],
    [(1, 5, 2), (2, 6, 2), (3, 0, 2), (4, 7, 2)],
    [(1, 0, -2), (2, 4, -2), (3, 5, -2), (6, 7, -2)],
    [(0, 0, 1), (1, 1, -1), (2, 2, 1), (3, 3, 1), (4, 4, -1), (5, 5, -1), (6, 6, 1), (7, 7, -1)],
    [(1, 2, -2), (3, 7, 2), (4, 0, 2), (5, 6, -2)],
    [(1, 3, -2), (2, 7, -2), (4, 6, 2), (5, 0, 2)],
    [(1, 4, 2), (2, 0, -2), (3, 6, -2), (5, 7, 2)],
    [(1, 2, -2), (3, 7, -2), (4, 0, -2), (5, 6, -2)],
    [(0, 0, 1), (1, 1, 1), (2, 2, -1), (3, 3, 1), (4, 4, -1), (5, 5, 1), (6, 6, -1), (7, 7, -1)],
    [(1, 7, 2), (2, 3, -2), (4, 5, -2), (6, 0, 2)],
    [(1, 5, 2), (2, 6, 2), (3, 0, -2), (4, 7, -2)],
    [(1, 3, -2), (2, 7, 2), (4, 6, 2), (5, 0, -2)],
    [(1, 7, -2), (2, 3, -2), (4, 5, -2), (6, 0, -2)],
    [(0, 0, 1), (1, 1, 1), (2, 2, 1), (3, 3, -1), (4, 4, 1), (5, 5, -1), (6, 6, -1), (7, 7, -1)],
]


def to_matrix(v):
    """rotor.cpp:170-181, (...,8) -> (...,4,4)."""
    m = np.zeros(v.shape[:-1] + (16,))
    for e, terms in enumerate(_TERMS):
        for a, b, c in terms:
            m[..., e] += c * v[..., a] * v[..., b]
    return m.reshape(v.shape[:-1] + (4, 4))


def gaussian_speed(rotor, log_scales):
    """V / W of the 4D covariance (gaussian.cpp:104-110)."""
    R = to_matrix(normalize(rotor))
    q = np.exp(2 * log_scales)
    sig = np.einsum("...ik,...k,...jk->...ij", R, q, R)
    return sig[..., :3, 3] / sig[..., 3, 3][..., None]


def _from_two_vectors_x(d):
    """Quaternion rotating +x onto unit vectors d (Eigen's setFromTwoVectors), (N,3)->(w,x,y,z)."""
    c = d[:, 0]
    axis = np.stack([np.zeros_like(c), -d[:, 2], d[:, 1]], -1)  # x cross d
    s = np.sqrt((1 + c) * 2)
    bad = c < -1 + 1e-12
    s = np.where(bad, 1.0, s)
    w = np.where(bad, 0.0, s * 0.5)
    v = np.where(bad[:, None], np.array([0.0, 0.0, 1.0]), axis / s[:, None])
    return w, v[:, 0], v[:, 1], v[:, 2]


def velocity_rotor(v, sx, st):
    """synthetic.cpp:134-177, vectorised: a rotor whose slice moves at velocity v."""
    speed = np.linalg.norm(v, axis=-1)
    out = np.zeros(v.shape[:-1] + (8,))
    out[..., 0] = 1
    mv = speed >= 1e-15
    if not mv.any():
        return out
    v, speed, sx, st = v[mv], speed[mv], sx[mv], st[mv]
    d = v / speed[:, None]
    sx2, st2 = sx * sx, st * st
    a, bq, c = speed * sx2, -(sx2 - st2), speed * st2
    disc = np.maximum(bq * bq - 4 * a * c, 0)
    q = -0.5 * (bq + np.where(bq >= 0, 1, -1) * np.sqrt(disc))
    with np.errstate(divide="ignore", invalid="ignore"):
        t1, t2 = q / a, c / q
    tau = np.where(q == 0, 0.0, np.where(np.abs(t1) < np.abs(t2), t1, t2))
    theta = np.arctan(tau)
    qw, qx, qy, qz = _from_two_vectors_x(d)
    spatial = from_quaternion(qw, qx, qy, qz)
    ls = np.stack([np.log(sx)] * 3 + [np.log(st)], -1)
    best, best_err = None, None
    for sgn in (1.0, -1.0):
        tc = np.zeros(spatial.shape)
        tc[:, 0] = np.cos(theta / 2)
        tc[:, 3] = sgn * np.sin(theta / 2)
        r = compose(spatial, tc)
        err = np.linalg.norm(gaussian_speed(r, ls) - v, axis=-1)
        if best is None:
            best, best_err = r, err
        else:
            take = err < best_err
            best = np.where(take[:, None], r, best)
    out[mv] = best
    return out


# ----------------------------------------------------------------------------- scenes
def synthetic_scene(n: int, width: int, height: int, seed: int = 1, sh_degree: int = 3,
                    fx_scale: float = 1.25) -> GaussianStore:
    """SURVEY.md §8(d) generator (criterion-10 recipe, acceptance.cpp:493-520), float32-rounded."""
    rng = np.random.default_rng(seed)
    fx = fx_scale * width
    fy = fx_scale * width
    ax = 0.875 * (width / 2) / fx
    ay = 0.875 * (height / 2) / fy
    z = rng.uniform(2, 8, n)
    x = rng.uniform(-ax, ax, n) * z
    y = rng.uniform(-ay, ay, n) * z
    t = rng.uniform(0, 1, n)
    mean = np.stack([x, y, z, t], -1)
    sx = np.exp(rng.uniform(-4, -2.5, n)) * (400.0 / width)
    ls = np.stack([np.log(sx) + rng.uniform(-0.2, 0.2, n) for _ in range(3)] + [rng.uniform(-0.5, 0.5, n)], -1)
    quat = rng.uniform(-1, 1, (n, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    spatial = from_quaternion(quat[:, 0], quat[:, 1], quat[:, 2], quat[:, 3])
    rotor = spatial.copy()
    even = np.arange(n) % 2 == 0
    vel = rng.uniform(-0.5, 0.5, (n, 3))
    vr = velocity_rotor(vel[even], sx[even], np.exp(ls[even, 3]))
    rotor[even] = normalize(compose(spatial[even], vr))
    op = rng.uniform(-2, 1, n)
    sh = np.zeros((n, 3, 16))
    sh[:, :, 0] = rng.uniform(0, 1, (n, 3))
    if sh_degree >= 1:
        k = (sh_degree + 1) ** 2
        sh[:, :, 1:k] = rng.uniform(-0.1, 0.1, (n, 3, k - 1))
    f = lambda a: np.asarray(a, np.float32).astype(np.float64)
    return GaussianStore(f(mean), f(ls), f(rotor), f(op), f(sh), sh_degree)


def random_scene(n: int, sh_degree: int = 1, seed: int = 0, f32: bool = True) -> GaussianStore:
    """The reference's unit-test scene recipe (tests/reference.hpp:27-46), numpy RNG."""
    rng = np.random.default_rng(seed)
    mean = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), rng.uniform(2.5, 4.5, n), rng.uniform(0, 1, n)], -1)
    ls = np.stack([rng.uniform(-2.2, -1.2, n) for _ in range(3)] + [rng.uniform(-1.2, 0.2, n)], -1)
    rot = rng.uniform(-1, 1, (n, 8))
    op = rng.uniform(-1, 2, n)
    sh = np.zeros((n, 3, 16))
    sh[:, :, 0] = rng.uniform(-0.8, 1.2, (n, 3))
    sh[:, :, 1:] = rng.uniform(-0.1, 0.1, (n, 3, 15))
    if f32:
        mean, ls, rot, op, sh = [np.asarray(a, np.float32).astype(np.float64) for a in (mean, ls, rot, op, sh)]
    return GaussianStore(mean, ls, rot, op, sh, sh_degree)


# ----------------------------------------------------------------------------- cameras
def perturbed(store: GaussianStore, seed: int, mean_sigma: float = 0.01, sh_dc_sigma: float = 0.1,
              opacity_sigma: float = 0.0) -> GaussianStore:
    """A training start from a ground-truth scene: Gaussian noise on the spatial means, the SH DC
    coefficients and (optionally) the opacity logits, every parameter rounded to float32 (so the
    FP32 device scene and the double host store the CPU reference reads hold the same values)."""
    out = store.copy()
    r = np.random.default_rng(seed)
    n = out.size()
    out.mean[:, :3] += r.normal(0, mean_sigma, (n, 3))
    out.sh[:, :, 0] += r.normal(0, sh_dc_sigma, (n, 3))
    if opacity_sigma:
        out.opacity_logit += r.normal(0, opacity_sigma, n)
    for a in (out.mean, out.log_scales, out.rotor, out.opacity_logit, out.sh):
        a[...] = a.astype(np.float32)
    return out


def yaw_pose(yaw_deg: float = 0.0, t=(0.0, 0.0, 0.0)) -> np.ndarray:
    a = np.deg2rad(yaw_deg)
    w = np.eye(4)
    w[:3, :3] = [[np.cos(a), 0, np.sin(a)], [0, 1, 0], [-np.sin(a), 0, np.cos(a)]]
    w[:3, 3] = t
    return w


def bench_camera(width: int, height: int, time: float = 0.5, pose=None, fx_scale: float = 1.25) -> Camera:
    """fx = fy = 1.25 W, principal point at the image centre (dataset.cpp:127-128)."""
    return Camera(width, height, fx_scale * width, fx_scale * width, width / 2.0, height / 2.0,
                  np.eye(4) if pose is None else np.asarray(pose, np.float64), float(time))


def sweep_cameras(width: int, height: int, n_times: int, pose=None):
    """A timestamp sweep t_k = k / (n-1) from one pose (config C2)."""
    ts = [k / (n_times - 1) if n_times > 1 else 0.5 for k in range(n_times)]
    return [bench_camera(width, height, t, pose) for t in ts]


def orbit_cameras(width: int, height: int, n_yaw: int, n_times: int, center_z: float = 5.0, radius: float = 5.0):
    """n_yaw x n_times camera x timestamp views on a circle looking at the frustum centre (config C4)."""
    cams = []
    for i in range(n_yaw):
        a = np.deg2rad(-20 + 40 * i / max(n_yaw - 1, 1))
        # camera position on a circle around (0,0,center_z), looking at it
        pos = np.array([radius * np.sin(a), 0.0, center_z - radius * np.cos(a)])
        fwd = np.array([0, 0, center_z]) - pos
        fwd /= np.linalg.norm(fwd)
        right = np.cross([0, 1, 0], fwd)
        right /= np.linalg.norm(right)
        down = np.cross(fwd, right)
        R = np.stack([right, down, fwd])
        w = np.eye(4)
        w[:3, :3] = R
        w[:3, 3] = -R @ pos
        for k in range(n_times):
            cams.append(bench_camera(width, height, k / max(n_times - 1, 1), w))
    return cams
