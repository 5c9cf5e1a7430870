"""oracle — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/liboracle.so`` (built from ``oracle/oracle.c`` by
plain gcc).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA path (``paper_2202_10297_b200``) and never
imports it; the numeric tags below are re-declared from DESIGN.md.

Every function takes and returns numpy arrays on the host.  See oracle.c for
the paper passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

F32, F64 = 1, 2
I32, I64 = 1, 2
ADD, MUL, MIN, MAX, LINREC, MAT2 = 1, 2, 3, 4, 5, 6
OPS = {"add": ADD, "mul": MUL, "min": MIN, "max": MAX, "linrec": LINREC, "mat2": MAT2}
WIDTH = {ADD: 1, MUL: 1, MIN: 1, MAX: 1, LINREC: 2, MAT2: 4}
ACCUMULATE = 1
EDUPINDEX = 5


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
             "-ffp-contract=off", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, i64, u32, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint, ctypes.c_int
        L.oracle_vjp_scan.argtypes = [ci, ci, i64, vp, vp, vp, vp, vp, u32]
        L.oracle_vjp_reduce.argtypes = [ci, ci, i64, vp, vp, vp, vp, vp, vp, u32]
        L.oracle_vjp_reduce_by_index.argtypes = [ci, ci, ci, i64, i64, vp, vp, vp, vp, vp, vp, vp, u32]
        L.oracle_vjp_scatter.argtypes = [ci, ci, i64, i64, i64, vp, vp, vp, vp, u32]
        L.oracle_kmeans.argtypes = [ci, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp]
        for f in (L.oracle_vjp_scan, L.oracle_vjp_reduce, L.oracle_vjp_reduce_by_index,
                  L.oracle_vjp_scatter):
            f.restype = ci
        _lib = L
    return _lib


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.float64:
        return F64
    raise TypeError(f"oracle: unsupported value dtype {a.dtype}")


def _it(a: np.ndarray) -> int:
    if a.dtype == np.int32:
        return I32
    if a.dtype == np.int64:
        return I64
    raise TypeError(f"oracle: unsupported index dtype {a.dtype}")


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _op(op) -> int:
    return OPS[op] if isinstance(op, str) else int(op)


def vjp_scan(op, ys_bar: np.ndarray, as_: np.ndarray | None = None, *, out=None,
             accumulate: bool = False, want_ys: bool = False, want_cond: bool = False):
    """as_bar of ys = scan op as_ with output adjoint ys_bar.

    Arrays are flat, element-interleaved (LINREC: d,c; MAT2: 2x2 row-major).
    Returns as_bar (and ys if want_ys, and cond if want_cond: f64 per scalar,
    the sum of |terms| of each adjoint entry, SURVEY 8c reading A22)."""
    o = _op(op)
    ys_bar = np.ascontiguousarray(ys_bar)
    dt = _dt(ys_bar)
    w = WIDTH[o]
    assert ys_bar.size % w == 0
    n = ys_bar.size // w
    if as_ is not None:
        as_ = np.ascontiguousarray(as_, dtype=ys_bar.dtype)
        assert as_.size == ys_bar.size
    as_bar = np.zeros_like(ys_bar) if out is None else out
    ys = np.empty_like(ys_bar) if (want_ys and as_ is not None) else None
    cond = np.zeros(ys_bar.size, dtype=np.float64) if want_cond else None
    rc = lib().oracle_vjp_scan(o, dt, n, _p(as_), _p(ys_bar), _p(as_bar), _p(ys), _p(cond),
                               ACCUMULATE if accumulate else 0)
    if rc != 0:
        raise RuntimeError(f"oracle_vjp_scan rc={rc}")
    res = (as_bar,) + ((ys,) if want_ys else ()) + ((cond,) if want_cond else ())
    return res if len(res) > 1 else as_bar


def vjp_reduce(op, as_: np.ndarray, y_bar, *, out=None, accumulate: bool = False):
    """Returns (as_bar, y, arg, zeros) for y = reduce op as_.
    LINREC / MAT2 (the general rule): as_ holds n elements of W
    scalars, y_bar and y are W-vectors."""
    o = _op(op)
    w = WIDTH[o]
    as_ = np.ascontiguousarray(as_)
    dt = _dt(as_)
    yb = np.ascontiguousarray(np.asarray(y_bar, dtype=as_.dtype).reshape(-1))
    assert yb.size == w
    y = np.zeros(w, dtype=as_.dtype)
    arg = np.zeros(1, dtype=np.int64)
    zeros = np.zeros(1, dtype=np.int64)
    as_bar = np.zeros_like(as_) if out is None else out
    rc = lib().oracle_vjp_reduce(o, dt, as_.size // w, _p(as_), _p(yb), _p(as_bar), _p(y), _p(arg),
                                 _p(zeros), ACCUMULATE if accumulate else 0)
    if rc != 0:
        raise RuntimeError(f"oracle_vjp_reduce rc={rc}")
    return as_bar, (y[0] if w == 1 else y), int(arg[0]), int(zeros[0])


def vjp_reduce_by_index(op, inds: np.ndarray, as_: np.ndarray | None, hs_bar: np.ndarray, *,
                        out=None, accumulate: bool = False, width: int = 1):
    """Returns (as_bar, hs, winners, zeros) for hs = reduce_by_index op m inds as_
    (P:1098-1126), m = len(hs_bar) / width.

    width > 1 (vectorised operator): the operator acts elementwise on rows
    (P:1229-1231), so by definition component j of every row is its own
    scalar reduce_by_index over the same bins (reading A24) — the scalar oracle
    is run once per component and the results are laid out [n x width] /
    [m x width]."""
    if width > 1:
        inds = np.ascontiguousarray(inds)
        n = inds.size
        hb2 = np.asarray(hs_bar).reshape(-1, width)
        a2 = None if as_ is None else np.asarray(as_).reshape(n, width)
        ab = np.zeros((n, width), dtype=hb2.dtype)
        if out is not None:
            ab[...] = np.asarray(out).reshape(n, width)
        hs = np.zeros_like(hb2) if as_ is not None else None
        win = np.zeros(hb2.shape, dtype=np.int64)
        zer = np.zeros(hb2.shape, dtype=np.int64)
        for j in range(width):
            col = np.ascontiguousarray(ab[:, j])
            r = vjp_reduce_by_index(op, inds, None if a2 is None else np.ascontiguousarray(a2[:, j]),
                                    np.ascontiguousarray(hb2[:, j]), out=col, accumulate=accumulate)
            ab[:, j] = r[0]
            if hs is not None:
                hs[:, j] = r[1]
            win[:, j] = r[2]
            zer[:, j] = r[3]
        flat = ab.reshape(-1)
        if out is not None:
            np.asarray(out).reshape(-1)[...] = flat
            flat = out
        return flat, None if hs is None else hs.reshape(-1), win.reshape(-1), zer.reshape(-1)
    o = _op(op)
    inds = np.ascontiguousarray(inds)
    hs_bar = np.ascontiguousarray(hs_bar)
    dt = _dt(hs_bar)
    n, m = inds.size, hs_bar.size
    if as_ is not None:
        as_ = np.ascontiguousarray(as_, dtype=hs_bar.dtype)
        assert as_.size == n
    hs = np.zeros(m, dtype=hs_bar.dtype) if as_ is not None else None
    winners = np.zeros(m, dtype=np.int64)
    zeros = np.zeros(m, dtype=np.int64)
    as_bar = np.zeros(n, dtype=hs_bar.dtype) if out is None else out
    rc = lib().oracle_vjp_reduce_by_index(o, dt, _it(inds), n, m, _p(inds), _p(as_), _p(hs_bar),
                                          _p(as_bar), _p(hs), _p(winners), _p(zeros),
                                          ACCUMULATE if accumulate else 0)
    if rc != 0:
        raise RuntimeError(f"oracle_vjp_reduce_by_index rc={rc}")
    return as_bar, hs, winners, zeros


def vjp_scatter(is_: np.ndarray, ys_bar: np.ndarray, *, width: int = 1, vs_out=None,
                accumulate: bool = False, in_place: bool = False):
    """Returns (xs_bar, vs_bar, rc) for ys = scatter xs is vs.
    rc == EDUPINDEX flags a duplicate in-range target (precondition)."""
    is_ = np.ascontiguousarray(is_)
    ys_bar = np.ascontiguousarray(ys_bar)
    dt = _dt(ys_bar)
    n = ys_bar.size // width
    m = is_.size
    vs_bar = np.zeros(m * width, dtype=ys_bar.dtype) if vs_out is None else vs_out
    xs_bar = ys_bar if in_place else np.empty_like(ys_bar)
    rc = lib().oracle_vjp_scatter(dt, _it(is_), n, m, width, _p(is_), _p(ys_bar), _p(xs_bar),
                                  _p(vs_bar), ACCUMULATE if accumulate else 0)
    if rc not in (0, EDUPINDEX):
        raise RuntimeError(f"oracle_vjp_scatter rc={rc}")
    return xs_bar, vs_bar, rc


def gather(arr: np.ndarray, inds: np.ndarray, *, width: int = 1) -> np.ndarray:
    """``gather arr inds = map (\\i -> arr[i]) inds``, elements of
    `width` scalars; an out-of-range index reads 0 (reading R4)."""
    a = np.asarray(arr).reshape(-1, width)
    out = np.zeros((len(inds), width), dtype=a.dtype)
    for j, t in enumerate(np.asarray(inds).tolist()):
        if 0 <= t < a.shape[0]:
            out[j] = a[t]
    return out.reshape(-1)


def scatter(arr: np.ndarray, inds: np.ndarray, vals: np.ndarray, *, width: int = 1) -> np.ndarray:
    """``scatter arr inds vals``: a copy of arr with arr[inds[j]] = vals[j]
    (P:1241-1244); out-of-range indices are skipped (reading R4)."""
    a = np.array(arr, copy=True).reshape(-1, width)
    v = np.asarray(vals).reshape(-1, width)
    for j, t in enumerate(np.asarray(inds).tolist()):
        if 0 <= t < a.shape[0]:
            a[t] = v[j]
    return a.reshape(-1)


def scatter_forward(xs: np.ndarray, is_: np.ndarray, vs: np.ndarray, *, width: int = 1):
    """Forward sweep of the in-place scatter, in the paper's order:
    ``let xs_saved = gather xs is; let ys = scatter xs is vs``.
    Returns (ys, xs_saved).  Pure-Python loop over m: small cases only."""
    xs_saved = gather(xs, is_, width=width)
    ys = scatter(xs, is_, vs, width=width)
    return ys, xs_saved


def scatter_restore(ys: np.ndarray, is_: np.ndarray, xs_saved: np.ndarray, *, width: int = 1) -> np.ndarray:
    """Return sweep step (3): ``let xs = scatter ys is xs_saved``."""
    return scatter(ys, is_, xs_saved, width=width)


def kmeans(points: np.ndarray, centers: np.ndarray, cost_bar: float = 1.0):
    """k-means cost f(C) = sum_p min_j ||p - c_j||^2 and its derivatives by the
    literal per-point loop (oracle.c; reading R15).
    points [n x d], centers [k x d] (same dtype).  Returns a dict with
    cost, cbar [k x d] (vjp with cost_bar), hdiag [k x d] (jvp of the vjp in the
    all-ones direction = Hessian diagonal), assign int32 [n], counts int64 [k]."""
    points = np.ascontiguousarray(points)
    centers = np.ascontiguousarray(centers)
    if points.ndim != 2 or centers.ndim != 2 or points.shape[1] != centers.shape[1]:
        raise ValueError("points [n x d] and centers [k x d]")
    if points.dtype != centers.dtype:
        raise ValueError("points and centers must share a dtype")
    n, d = points.shape
    k = centers.shape[0]
    dt = _dt(centers)
    yb = np.array([cost_bar], dtype=centers.dtype)
    cbar = np.zeros((k, d), dtype=centers.dtype)
    hdiag = np.zeros((k, d), dtype=centers.dtype)
    assign = np.zeros(n, dtype=np.int32)
    counts = np.zeros(k, dtype=np.int64)
    cost = np.zeros(1, dtype=centers.dtype)
    rc = lib().oracle_kmeans(dt, n, k, d, _p(points) if n else None, _p(centers), _p(yb), _p(cbar),
                             _p(hdiag), _p(assign), _p(counts), _p(cost))
    if rc != 0:
        raise RuntimeError(f"oracle_kmeans rc={rc}")
    return {"cost": float(cost[0]), "cbar": cbar, "hdiag": hdiag, "assign": assign, "counts": counts}


def vjp_scan_batched(op, ys_bar: np.ndarray, as_: np.ndarray | None, width: int, *, out=None,
                     accumulate: bool = False):
    """vjp of the VECTORISED scan ys = scan (map op) e as_ by the
    paper's transpose rule: `width` independent scans along n,
    each by the sequential oracle_vjp_scan.  Arrays hold [n][width][W] scalars."""
    W = WIDTH[_op(op)]
    yb = np.ascontiguousarray(ys_bar).reshape(-1, width, W)
    a = None if as_ is None else np.ascontiguousarray(as_).reshape(-1, width, W)
    res = np.empty_like(yb) if out is None else np.ascontiguousarray(out).reshape(-1, width, W).copy()
    for j in range(width):  # transpose |> map (scan op e) |> transpose
        col_out = res[:, j, :].reshape(-1).copy()
        r = vjp_scan(op, yb[:, j, :].reshape(-1).copy(), None if a is None else a[:, j, :].reshape(-1).copy(),
                     out=col_out if accumulate else None, accumulate=accumulate)
        res[:, j, :] = np.asarray(r).reshape(-1, W)
    return res.reshape(-1)
