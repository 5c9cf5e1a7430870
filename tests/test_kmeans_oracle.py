"""Pins for the k-means composite of the oracle (oracle_kmeans, SURVEY 8f row
f3) — CPU only.

f(C) = sum_p min_j ||p - c_j||^2 (reading R15: squared distance).  Nothing here
re-runs the oracle's arithmetic: the cost is re-derived with exact rationals
(Fractions) from the definition, the gradient is pinned by exact central finite
differences of that rational cost (exact because f is quadratic in C inside a
Voronoi cell), the Hessian diagonal by exact second differences, the tie rule
and the empty cluster by hand-made cases, and the full gradient at n = 2000 by
the closed form 2 ybar (cnt_j c_j - sum_{p in j} p) with the assignment
recomputed by numpy.
"""
from __future__ import annotations

from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
import synth


def cost_exact(P, C):
    """the definition, in exact rationals: sum_p min_j sum_t (p_t - c_jt)^2"""
    tot = Fr(0)
    for p in P:
        tot += min(sum((Fr(pt) - Fr(ct)) ** 2 for pt, ct in zip(p, c)) for c in C)
    return tot


def small_case():
    """three well separated clusters on a dyadic grid (no point near a Voronoi
    boundary, so +-1/2 moves of a center never change an assignment)"""
    C = [[0.0, 0.0], [10.0, 0.0], [0.0, 10.0]]
    P = [[0.5, -1.0], [-1.0, 0.25], [11.0, 1.5], [9.0, -0.5], [10.5, 0.0], [1.0, 9.0], [-0.75, 11.0]]
    return np.array(P), np.array(C)


def test_kmeans_cost_exact():
    P, C = small_case()
    r = oracle.kmeans(P, C)
    assert r["cost"] == float(cost_exact(P.tolist(), C.tolist()))
    assert r["assign"].tolist() == [0, 0, 1, 1, 1, 2, 2]
    assert r["counts"].tolist() == [2, 3, 2]


@pytest.mark.parametrize("ybar", [1.0, 0.75, -3.0])
def test_kmeans_gradient_exact_central_fd(ybar):
    """central differences of the exact rational cost with h = 1/2 are exact
    for a quadratic (no truncation term); the oracle's f64 vjp must equal them
    bit for bit (all values are small dyadic rationals)."""
    P, C = small_case()
    r = oracle.kmeans(P, C, cost_bar=ybar)
    h = Fr(1, 2)
    for j in range(C.shape[0]):
        for t in range(C.shape[1]):
            Cp = [[Fr(x) for x in row] for row in C.tolist()]
            Cm = [[Fr(x) for x in row] for row in C.tolist()]
            Cp[j][t] += h
            Cm[j][t] -= h
            fd = (cost_exact(P.tolist(), Cp) - cost_exact(P.tolist(), Cm)) / (2 * h)
            assert r["cbar"][j, t] == float(Fr(ybar) * fd), (j, t)


def test_kmeans_hessian_diagonal_exact_second_difference():
    """(f(c + h e) - 2 f(c) + f(c - h e)) / h^2 is exact for a quadratic; it is
    the Hessian diagonal the jvp-of-vjp returns."""
    P, C = small_case()
    r = oracle.kmeans(P, C, cost_bar=1.0)
    h = Fr(1, 2)
    f0 = cost_exact(P.tolist(), C.tolist())
    for j in range(C.shape[0]):
        for t in range(C.shape[1]):
            Cp = [[Fr(x) for x in row] for row in C.tolist()]
            Cm = [[Fr(x) for x in row] for row in C.tolist()]
            Cp[j][t] += h
            Cm[j][t] -= h
            sd = (cost_exact(P.tolist(), Cp) - 2 * f0 + cost_exact(P.tolist(), Cm)) / (h * h)
            assert r["hdiag"][j, t] == float(sd), (j, t)


def test_kmeans_first_index_tie_and_empty_cluster():
    """a point equidistant from two centers belongs to the FIRST,
    and only that center receives its adjoint; a center with no point gets a
    zero gradient and a zero Hessian entry."""
    P = np.array([[0.0, 0.0], [0.0, 2.0]])
    C = np.array([[1.0, 0.0], [-1.0, 0.0], [50.0, 50.0]])
    r = oracle.kmeans(P, C)
    assert r["assign"].tolist() == [0, 0]  # (0,2) is also equidistant from c0 and c1
    assert r["cbar"][0].tolist() == [4.0, -4.0]  # 2(c0-p0) + 2(c0-p1) = (2,0) + (2,-4)
    assert r["cbar"][1].tolist() == [0.0, 0.0]
    assert r["cbar"][2].tolist() == [0.0, 0.0] and r["hdiag"][2].tolist() == [0.0, 0.0]
    assert r["counts"].tolist() == [2, 0, 0]
    assert r["hdiag"][0].tolist() == [4.0, 4.0]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_kmeans_closed_form_mixture(dt):
    """n = 2000 points of a 16-cluster mixture in 8-D (synth recipe of config 5):
    the vjp equals 2 ybar (cnt_j c_j - sum_{p in j} p) with the assignment
    recomputed by numpy (direct squared distances, argmin = first index), the
    Hessian diagonal 2 ybar cnt_j, the cost sum_p min_j dist."""
    import torch
    P, C = synth.kmeans_inputs(2000, 16, 8, dtype=torch.float64)
    P, C = P.numpy().astype(dt), C.numpy().astype(dt)
    ybar = 1.25
    r = oracle.kmeans(P, C, cost_bar=ybar)
    P64, C64 = P.astype(np.float64), C.astype(np.float64)
    D = ((P64[:, None, :] - C64[None, :, :]) ** 2).sum(-1)
    a = D.argmin(1)
    assert r["assign"].tolist() == a.tolist()
    cnt = np.bincount(a, minlength=16)
    assert r["counts"].tolist() == cnt.tolist()
    S = np.zeros_like(C64)
    np.add.at(S, a, P64)
    ref = 2 * ybar * (cnt[:, None] * C64 - S)
    scale = np.zeros_like(C64)  # sum of |terms| per coordinate (condition scaling, reading A22)
    np.add.at(scale, a, np.abs(C64[a] - P64))
    tol = 1e-12 if dt == np.float64 else 1e-6
    assert np.all(np.abs(r["cbar"].astype(np.float64) - ref) <= tol * (2 * abs(ybar) * scale + 1e-300))
    assert np.array_equal(r["hdiag"], np.broadcast_to((2 * ybar * cnt)[:, None], C.shape).astype(dt))
    assert abs(r["cost"] - D.min(1).sum()) <= 1e-12 * D.min(1).sum() * (1 if dt == np.float64 else 1e5)


def test_kmeans_linear_in_ybar():
    import torch
    P, C = synth.kmeans_inputs(500, 8, 4, dtype=torch.float64)
    r1 = oracle.kmeans(P.numpy(), C.numpy(), cost_bar=1.0)
    r3 = oracle.kmeans(P.numpy(), C.numpy(), cost_bar=3.0)
    assert np.allclose(r3["cbar"], 3 * r1["cbar"], rtol=1e-15, atol=0)
    assert np.array_equal(r3["hdiag"], 3 * r1["hdiag"])


def test_kmeans_synth_recipe_is_sliceable():
    """shards of config 5 are slices of the 1-GPU arrays (offset by points)"""
    import torch
    P, C = synth.kmeans_inputs(300, 5, 3)
    P2, C2 = synth.kmeans_inputs(100, 5, 3, offset=200)
    assert torch.equal(P[200:], P2) and torch.equal(C, C2)
