"""Shared comparison helpers for the parity tests (GPU path vs CPU oracle)."""
import numpy as np

SPLAT_FIELDS = ["mean2", "conic", "depth", "color", "alpha_base", "flow2", "radius", "source_index"]


def splat_mismatch(a, b):
    """Per-field count of splats whose values differ (== semantics, so -0 == +0)."""
    out = {}
    if len(a) != len(b):
        return {"count": (len(a), len(b))}
    for f in SPLAT_FIELDS:
        x, y = a[f], b[f]
        bad = ~((x == y) | (np.isnan(x) & np.isnan(y)))
        if bad.ndim > 1:
            bad = bad.any(axis=tuple(range(1, bad.ndim)))
        if bad.any():
            out[f] = int(bad.sum())
    return out


def tiles_equal(rec_a_offsets, rec_a_ids, rec_b_offsets, rec_b_ids):
    return np.array_equal(rec_a_offsets, rec_b_offsets) and np.array_equal(rec_a_ids, rec_b_ids)


def floored_rel_err(g, ref, floor_frac=1e-3):
    """|g-ref| / max(|ref|, floor) with floor = floor_frac * max|ref| per column (parameter)."""
    g = np.asarray(g, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = np.abs(ref).max(axis=0, keepdims=True)
    floor = np.maximum(floor_frac * scale, 1e-12)
    return np.abs(g - ref) / np.maximum(np.abs(ref), floor)
