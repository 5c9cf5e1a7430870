"""Parity comparators (SURVEY 8c "The parity comparator"), shared by GPU tests."""
from __future__ import annotations

import numpy as np

TOL = {np.dtype(np.float64): 1e-10, np.dtype(np.float32): 1e-4}  # north_star tolerances


def max_rel_err(got: np.ndarray, ref: np.ndarray, scale: np.ndarray | None = None) -> float:
    """max |got - ref| / |ref| elementwise (reading A22); where ref == 0 the
    difference must be exactly 0 unless a condition `scale` (sum of |terms|)
    is given, in which case |got - ref| / scale is used there."""
    got = np.asarray(got, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    assert got.shape == ref.shape
    bad = ~np.isfinite(got) & np.isfinite(ref)
    if bad.any():
        return float("inf")
    den = np.abs(ref)
    if scale is not None:
        den = np.maximum(den, np.asarray(scale, dtype=np.float64).ravel())
    diff = np.abs(got - ref)
    zero = den == 0
    if (diff[zero] != 0).any():
        return float("inf")
    if (~zero).any():
        return float(np.max(diff[~zero] / den[~zero]))
    return 0.0


def assert_close(got, ref, dtype, scale=None, what=""):
    tol = TOL[np.dtype(dtype)]
    e = max_rel_err(got, ref, scale)
    assert e <= tol, f"{what}: max rel err {e:.3e} > {tol:.0e}"
    return e
