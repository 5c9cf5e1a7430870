"""Pins for the CPU oracle (oracle/oracle.c) — CPU only, no GPU.

The oracle is trusted only through checks that do NOT re-run its own
arithmetic: exact rational dual-number Jacobians of the primal definitions
(tests/_exact.py, P:353-359 / P:382-383), exact central finite differences of
multilinear operators, the worked examples of the paper / SPEC
(tests/golden/worked_examples.json, each with its citation), closed forms
(P:1233-1236 scan(+); P:1040-1061 reduce(*) cases), and structural identities
(scan-last == reduce, LINREC == MAT2 embedding, reduce_by_index per bin ==
reduce, duality).  Any dropped term, wrong sign, wrong index or transposed
operand in oracle.c fails at least one of these.
"""
from __future__ import annotations

import json
import math
import os
import random
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
from _exact import (OPS, reduce, reduce_by_index, scan, scatter, vjp_by_central_fd,
                    vjp_by_duals)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _num(v):
    return float(v) if not isinstance(v, str) else float(v)


def _arr(vals, dt):
    return np.array([_num(v) for v in vals], dtype=dt)


# ---------------------------------------------------------------- goldens

@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["id"] for c in GOLD["cases"]])
def test_golden(case, dt):
    k = case["kind"]
    if k == "scan":
        ab, ys = oracle.vjp_scan(case["op"], _arr(case["ybar"], dt), _arr(case["as"], dt), want_ys=True)
        assert ab.tolist() == _arr(case["expected"], dt).tolist()
        if "ys" in case:
            assert ys.tolist() == _arr(case["ys"], dt).tolist()
    elif k == "reduce":
        ab, y, arg, zeros = oracle.vjp_reduce(case["op"], _arr(case["as"], dt), float(case["ybar"]))
        assert ab.tolist() == _arr(case["expected"], dt).tolist()
        if "y" in case:
            assert y == case["y"]
        assert arg == case["arg"]
        assert zeros == case["zeros"]
    elif k == "reduce_by_index":
        ab, hs, win, zeros = oracle.vjp_reduce_by_index(
            case["op"], np.array(case["inds"], np.int32), _arr(case["as"], dt), _arr(case["hs_bar"], dt),
            width=case.get("width", 1))
        assert ab.tolist() == _arr(case["expected"], dt).tolist()
        if "hs" in case:
            assert hs.tolist() == _arr(case["hs"], dt).tolist()
        if "winners" in case:
            assert win.tolist() == case["winners"]
        if "zeros" in case:
            assert zeros.tolist() == case["zeros"]
    elif k == "scatter":
        xb, vb, rc = oracle.vjp_scatter(np.array(case["is"], np.int64), _arr(case["ys_bar"], dt))
        assert rc == 0
        assert xb.tolist() == _arr(case["xs_bar"], dt).tolist()
        assert vb.tolist() == _arr(case["vs_bar"], dt).tolist()
    elif k == "scatter_fwd":
        ys, saved = oracle.scatter_forward(_arr(case["xs"], dt), np.array(case["is"], np.int64), _arr(case["vs"], dt))
        assert ys.tolist() == _arr(case["ys"], dt).tolist()
        assert saved.tolist() == _arr(case["xs_saved"], dt).tolist()
        back = oracle.scatter_restore(ys, np.array(case["is"], np.int64), saved)
        assert back.tolist() == _arr(case["xs"], dt).tolist()
    else:
        raise AssertionError(k)


# ---------------------------------------------- dual numbers / exact FD

def _rand_ints(rng, n, lo, hi):
    return [rng.randint(lo, hi) for _ in range(n)]


@pytest.mark.parametrize("op", ["add", "mul", "min", "max", "linrec", "mat2"])
@pytest.mark.parametrize("n", [1, 2, 3, 7, 12])
def test_scan_vs_dual_numbers(op, n):
    rng = random.Random(1000 * n + len(op))
    w = OPS[op][1]
    lo, hi = {"add": (-9, 9), "mul": (-3, 3), "min": (-2, 2), "max": (-2, 2),
              "linrec": (-2, 2), "mat2": (-1, 2)}[op]
    x = _rand_ints(rng, n * w, lo, hi)
    yb = _rand_ints(rng, n * w, -5, 5)
    exp = vjp_by_duals(lambda v: scan(op, v), x, yb)
    got = oracle.vjp_scan(op, np.array(yb, np.float64), np.array(x, np.float64))
    assert [Fr(float(g)) for g in got] == exp


@pytest.mark.parametrize("op", ["add", "mul", "linrec", "mat2"])
def test_scan_vs_exact_central_fd(op):
    """ADD, MUL, LINREC, MAT2 scans are multilinear in every scalar input, so a
    central difference with h = 1/2 is exact (no truncation error)."""
    rng = random.Random(7)
    w = OPS[op][1]
    n = 9
    x = [Fr(rng.randint(-6, 6), 4) for _ in range(n * w)]
    yb = [Fr(rng.randint(-6, 6), 2) for _ in range(n * w)]
    exp = vjp_by_central_fd(lambda v: scan(op, v), x, yb)
    got = oracle.vjp_scan(op, np.array([float(v) for v in yb]), np.array([float(v) for v in x]))
    assert [Fr(float(g)) for g in got] == exp


def test_scan_add_config1_closed_form_and_fd():
    """Config 1 (n = 10^4): vjp scan(+) = reversed suffix sum.
    Integer seeds make every summation order exact -> bit-exact; the central
    FD of <ybar, scan(as)> (linear, so exact) is evaluated with numpy."""
    n = 10_000
    rng = np.random.default_rng(2202)
    yb = rng.integers(-8, 9, n).astype(np.float64)
    got = oracle.vjp_scan("add", yb, None)
    closed = np.cumsum(yb[::-1])[::-1]
    assert np.array_equal(got, closed)
    assert np.array_equal(oracle.vjp_scan("add", np.ones(n), None), np.arange(n, 0, -1, dtype=np.float64))
    # central FD over all n inputs, h = 1/2, as integers -> exact in f64
    as_ = rng.integers(-100, 100, n).astype(np.float64)
    base = np.cumsum(as_)
    fd = np.empty(n)
    for k0 in range(0, n, 1000):
        ks = np.arange(k0, min(k0 + 1000, n))
        E = np.zeros((len(ks), n))
        E[np.arange(len(ks)), ks] = 0.5
        fp = np.cumsum(as_[None, :] + E, axis=1) @ yb
        fm = np.cumsum(as_[None, :] - E, axis=1) @ yb
        fd[ks] = (fp - fm) / 1.0
    assert np.array_equal(fd, got)
    assert base.shape == (n,)


def test_scan_add_uniform_vs_exact_rational():
    """U(0,1) seeds: oracle (long double) vs the exact rational suffix sums,
    correctly rounded -> error below one f64 ulp."""
    n = 4000
    yb = np.random.default_rng(5).random(n)
    got = oracle.vjp_scan("add", yb, None)
    acc = Fr(0)
    exact = [None] * n
    for i in range(n - 1, -1, -1):
        acc += Fr(float(yb[i]))
        exact[i] = acc
    rel = max(abs(Fr(float(g)) - e) / e for g, e in zip(got, exact))
    assert rel <= Fr(2, 2**53)


@pytest.mark.parametrize("op", ["add", "mul", "min", "max"])
@pytest.mark.parametrize("n", [1, 2, 5, 11])
def test_reduce_vs_dual_numbers(op, n):
    rng = random.Random(31 * n + len(op))
    lo, hi = (-3, 3) if op == "mul" else (-4, 4)
    for _ in range(6):
        x = _rand_ints(rng, n, lo, hi)
        if op == "mul" and rng.random() < 0.5:
            for _ in range(rng.randint(1, 2)):
                x[rng.randrange(n)] = 0  # exercise z = 1 and z >= 2
        yb = rng.randint(-5, 5)
        exp = vjp_by_duals(lambda v: reduce(op, v), x, [yb])
        got, y, arg, zeros = oracle.vjp_reduce(op, np.array(x, np.float64), yb)
        assert [Fr(float(g)) for g in got] == exp
        assert y == float(reduce(op, [Fr(v) for v in x]))


@pytest.mark.parametrize("op", ["add", "mul", "min", "max"])
def test_reduce_by_index_vs_dual_numbers(op):
    rng = random.Random(99 + len(op))
    for trial in range(8):
        n, m = rng.randint(1, 12), rng.randint(1, 4)
        inds = [rng.randint(-1, m) for _ in range(n)]  # includes out-of-range bins (R4)
        lo, hi = (-3, 3) if op == "mul" else (-3, 3)
        x = _rand_ints(rng, n, lo, hi)
        hb = _rand_ints(rng, m, -5, 5)
        neutral = {"add": 0, "mul": 1, "min": 10**9, "max": -10**9}[op]
        exp = vjp_by_duals(lambda v: reduce_by_index(op, m, inds, v, neutral), x, hb)
        got, hs, win, zeros = oracle.vjp_reduce_by_index(
            op, np.array(inds, np.int64), np.array(x, np.float64), np.array(hb, np.float64))
        assert [Fr(float(g)) for g in got] == exp, (inds, x, hb)
        h = reduce_by_index(op, m, inds, [Fr(v) for v in x], neutral)
        for b in range(m):
            if op in ("add", "mul") or any(0 <= i == b for i in inds):
                assert hs[b] == float(h[b])


def test_scatter_vs_dual_numbers():
    rng = random.Random(4)
    for trial in range(10):
        n = rng.randint(1, 10)
        m = rng.randint(0, n)
        targets = rng.sample(range(n), m)
        if trial % 3 == 0 and m > 0:
            targets[0] = n + 3  # out of range -> skipped (R4)
        xs = _rand_ints(rng, n, -5, 5)
        vs = _rand_ints(rng, m, -5, 5)
        yb = _rand_ints(rng, n, -9, 9)
        exp = vjp_by_duals(lambda v: scatter(v[:n], targets, v[n:]), xs + vs, yb)
        xb, vb, rc = oracle.vjp_scatter(np.array(targets, np.int32), np.array(yb, np.float64))
        assert rc == 0
        assert [Fr(float(g)) for g in list(xb) + list(vb)] == exp
        # in place (xs_bar aliases ys_bar): same result
        y2 = np.array(yb, np.float64)
        xb2, vb2, _ = oracle.vjp_scatter(np.array(targets, np.int32), y2, in_place=True)
        assert xb2 is y2 and xb2.tolist() == xb.tolist() and vb2.tolist() == vb.tolist()


def test_scatter_duplicate_flagged():
    _, _, rc = oracle.vjp_scatter(np.array([1, 1], np.int64), np.arange(4.0))
    assert rc == oracle.EDUPINDEX


# ------------------------------------------------------ structural pins

def test_reduce_mul_general_equals_pz_special_case():
    """P:1006-1011 (general l_i*r_i, used by the oracle) vs the (p, z) special
    case of P:1040-1061 evaluated here with exact rationals."""
    rng = random.Random(12)
    for trial in range(40):
        n = rng.randint(1, 30)
        x = [Fr(rng.randint(1, 9), rng.randint(1, 4)) * rng.choice([-1, 1]) for _ in range(n)]
        for _ in range(trial % 4):
            x[rng.randrange(n)] = Fr(0)
        x = [Fr(float(v)) for v in x]  # exactly the binary values the oracle sees
        yb = Fr(float(Fr(rng.randint(-7, 7), 3)))
        z = sum(1 for v in x if v == 0)
        p = math.prod((v for v in x if v != 0), start=Fr(1))
        if z == 0:
            exp = [p / v * yb for v in x]
        elif z == 1:
            exp = [p * yb if v == 0 else Fr(0) for v in x]
        else:
            exp = [Fr(0)] * n
        got, _, arg, zeros = oracle.vjp_reduce("mul", np.array([float(v) for v in x]), float(yb))
        assert zeros == z
        assert arg == (next(i for i, v in enumerate(x) if v == 0) if z else -1)
        for g, e in zip(got, exp):
            assert abs(Fr(float(g)) - e) <= abs(e) * Fr(1, 2**52)


@pytest.mark.parametrize("op", ["add", "mul", "min", "max"])
def test_scan_last_equals_reduce(op):
    """Last element of scan == reduce, so their vjps agree when only
    the last scan output is seeded (also pins the MIN/MAX tie readings)."""
    rng = np.random.default_rng(3)
    for n in (1, 2, 17, 64):
        x = rng.integers(-3, 4, n).astype(np.float64)
        if op == "mul":
            x[x == 0] = 2.0
        yb = np.zeros(n)
        yb[-1] = 2.5
        a = oracle.vjp_scan(op, yb, x)
        b, *_ = oracle.vjp_reduce(op, x, 2.5)
        assert np.array_equal(a, b)


def test_linrec_equals_mat2_embedding():
    """(d, c) -> [[c, 0], [d, 1]] is a homomorphism from lin_o into
    R . A (R1); the LINREC vjp must equal the chain rule through it."""
    rng = np.random.default_rng(8)
    n = 40
    d, c = rng.random(n), 0.5 + 0.5 * rng.random(n)
    gD, gC = rng.random(n), rng.random(n)
    lin = np.stack([d, c], 1).ravel()
    ab_lin = oracle.vjp_scan("linrec", np.stack([gD, gC], 1).ravel(), lin).reshape(n, 2)
    M = np.zeros((n, 4))
    M[:, 0], M[:, 2], M[:, 3] = c, d, 1.0
    seed = np.zeros((n, 4))
    seed[:, 0], seed[:, 2] = gC, gD  # R[0,0] = C, R[1,0] = D
    ab_mat = oracle.vjp_scan("mat2", seed.ravel(), M.ravel()).reshape(n, 4)
    np.testing.assert_allclose(ab_lin[:, 0], ab_mat[:, 2], rtol=1e-13, atol=0)
    np.testing.assert_allclose(ab_lin[:, 1], ab_mat[:, 0], rtol=1e-13, atol=0)


@pytest.mark.parametrize("op", ["add", "mul", "max"])
def test_rbi_per_bin_equals_reduce(op):
    rng = np.random.default_rng(11)
    n, m = 200, 5
    inds = rng.integers(0, m, n).astype(np.int32)
    x = rng.integers(1, 5, n).astype(np.float64) / 2
    if op == "mul":
        x[rng.integers(0, n, 3)] = 0.0
    hb = rng.integers(-3, 4, m).astype(np.float64)
    got, hs, *_ = oracle.vjp_reduce_by_index(op, inds, x, hb)
    for b in range(m):
        sel = np.nonzero(inds == b)[0]
        ab, y, *_ = oracle.vjp_reduce(op, x[sel], hb[b])
        assert np.array_equal(got[sel], ab)
        assert hs[b] == y


@pytest.mark.parametrize("op", ["add", "mul", "linrec", "mat2"])
def test_duality_dot_test(op):
    """<ybar, J xdot> == <J^T ybar, xdot> with random reals; J xdot from
    exact rational dual numbers on the float inputs."""
    from _exact import Dual
    rng = np.random.default_rng(21)
    w = OPS[op][1]
    n = 24
    x = (0.5 + 0.5 * rng.random(n * w)) if op != "add" else rng.random(n * w)
    xd = rng.standard_normal(n * w)
    yb = rng.standard_normal(n * w)
    ys = scan(op, [Dual(Fr(float(a)), Fr(float(t))) for a, t in zip(x, xd)])
    lhs = sum(Fr(float(b)) * y.t for b, y in zip(yb, ys))
    rhs = sum(Fr(float(g)) * Fr(float(t)) for g, t in zip(oracle.vjp_scan(op, yb, x), xd))
    scale = sum(abs(Fr(float(b)) * y.t) for b, y in zip(yb, ys)) + 1
    assert abs(lhs - rhs) / scale < Fr(1, 10**13)


def test_linearity_in_ybar():
    rng = np.random.default_rng(2)
    x = rng.integers(-3, 4, 30 * 4).astype(np.float64)
    a, b = rng.integers(-5, 6, (2, 30 * 4)).astype(np.float64)
    assert np.array_equal(oracle.vjp_scan("mat2", a + b, x),
                          oracle.vjp_scan("mat2", a, x) + oracle.vjp_scan("mat2", b, x))


# ------------------------------------------------------------ edge cases

def test_empty_and_single():
    e = np.zeros(0)
    assert oracle.vjp_scan("add", e, None).size == 0
    assert oracle.vjp_scan("mat2", e, e).size == 0
    ab, y, arg, z = oracle.vjp_reduce("min", e, 1.0)
    assert ab.size == 0 and y == np.inf and arg == -1
    ab, y, *_ = oracle.vjp_reduce("mul", e, 1.0)
    assert y == 1.0
    for op in ("add", "mul", "min", "max", "linrec", "mat2"):
        w = OPS[op][1]
        yb = np.arange(1.0, w + 1)
        assert np.array_equal(oracle.vjp_scan(op, yb, np.full(w, 3.0)), yb)  # n=1: as_bar = ys_bar
    for op in ("add", "mul", "min", "max"):
        ab, *_ = oracle.vjp_reduce(op, np.array([0.0]), 4.0)
        assert ab.tolist() == [4.0]  # n=1: ybar for every op, incl. * with a0 = 0 (p = 1)


def test_accumulate_mode():
    x = np.array([2.0, 3.0, 4.0])
    out = np.full(3, 100.0)
    oracle.vjp_scan("mul", np.array([0.0, 0.0, 1.0]), x, out=out, accumulate=True)
    assert out.tolist() == [112.0, 108.0, 106.0]
    out = np.full(4, 100.0)
    oracle.vjp_reduce("min", np.array([3.0, 1.0, 2.0, 1.0]), 5.0, out=out, accumulate=True)
    assert out.tolist() == [100.0, 105.0, 100.0, 100.0]  # only the argmin is touched
    out = np.full(3, 1.0)
    oracle.vjp_reduce_by_index("max", np.array([0, 0, 1], np.int32), np.array([1.0, 2.0, 3.0]),
                               np.array([10.0, 20.0]), out=out, accumulate=True)
    assert out.tolist() == [1.0, 11.0, 21.0]


def test_f32_rounds_once():
    """f32 data: long-double arithmetic, one rounding to f32 at the end."""
    x = np.array([1.0, 1.0 + 2**-23, 3.0], np.float32)
    got = oracle.vjp_scan("mul", np.array([0, 0, 1], np.float32), x)
    exact = [Fr(float(x[1])) * 3, Fr(1) * 3, Fr(float(x[1]))]
    assert got.dtype == np.float32
    assert [float(g) for g in got] == [float(np.float32(float(e))) for e in exact]


# ------------------------------------------------ general reduce rule (f4)

@pytest.mark.parametrize("op", ["linrec", "mat2"])
def test_reduce_general_rule_is_scan_last(op):
    """P:986-1013's general reduce rule for LINREC / MAT2 equals the scan's vjp
    seeded only at the last element (scan-last == reduce) — two
    independent code paths of the oracle (exclusive scans + map vs the
    sequential return sweep of P:1153-1158)."""
    import synth
    import torch
    gen = {"linrec": synth.linrec_inputs, "mat2": synth.mat2_inputs}[op]
    a, _ = gen(1000)
    a = a.numpy()
    w = 2 if op == "linrec" else 4
    ybar = np.arange(1, w + 1, dtype=np.float64) * 0.75
    ab, y, _, _ = oracle.vjp_reduce(op, a, ybar)
    seed = np.zeros_like(a)
    seed[-w:] = ybar
    ref, ys = oracle.vjp_scan(op, seed, a, want_ys=True)
    assert np.allclose(ab, ref, rtol=1e-14, atol=0)
    assert np.allclose(y, ys[-w:], rtol=1e-14, atol=0)


@pytest.mark.parametrize("op", ["linrec", "mat2"])
def test_reduce_general_rule_exact_central_fd(op):
    """the general rule's adjoint equals the exact rational central difference of the
    primal reduce on small integer inputs (every input direction)."""
    rng = random.Random(5)
    w = 2 if op == "linrec" else 4
    n = 5
    a = [Fr(rng.randint(-3, 3)) for _ in range(n * w)]
    ybar = [Fr(rng.randint(-2, 2)) for _ in range(w)]

    def prim(vals):
        acc = [Fr(0), Fr(1)] if op == "linrec" else [Fr(1), Fr(0), Fr(0), Fr(1)]
        for i in range(n):
            e = vals[i * w:(i + 1) * w]
            if op == "linrec":
                acc = [e[0] + e[1] * acc[0], e[1] * acc[1]]
            else:
                acc = [acc[0] * e[0] + acc[1] * e[2], acc[0] * e[1] + acc[1] * e[3],
                       acc[2] * e[0] + acc[3] * e[2], acc[2] * e[1] + acc[3] * e[3]]
        return acc

    exp = []
    for k in range(n * w):  # the objective <ybar, reduce> is multilinear: exact central difference, h = 1
        up = list(a); up[k] += 1
        dn = list(a); dn[k] -= 1
        fu = sum(y * v for y, v in zip(ybar, prim(up)))
        fd = sum(y * v for y, v in zip(ybar, prim(dn)))
        exp.append((fu - fd) / 2)
    ab, _, _, _ = oracle.vjp_reduce(op, np.array([float(x) for x in a]), np.array([float(x) for x in ybar]))
    assert ab.tolist() == [float(x) for x in exp]


# ------------------------------------------- condition scale (reading A22)

@pytest.mark.parametrize("op", ["add", "mul", "linrec", "mat2"])
@pytest.mark.parametrize("n", [1, 2, 5, 11])
def test_scan_cond_is_sum_of_abs_terms(op, n):
    """cond = sum |term| of each adjoint entry.  ADD / MUL / LINREC / MAT2 scans
    are polynomials with +1 coefficients in (as, ysbar), so sum |monomial| =
    J(|x|)^T |ybar| — computed here from the exact rational PRIMAL definition
    by dual numbers (_exact.py), not by the oracle's loop."""
    rng = random.Random(4242 + 17 * n + len(op))
    w = OPS[op][1]
    x = [Fr(rng.randint(-9, 9), 4) for _ in range(n * w)]
    yb = [Fr(rng.randint(-9, 9), 2) for _ in range(n * w)]
    exp = vjp_by_duals(lambda v: scan(op, v), [abs(v) for v in x], [abs(v) for v in yb])
    _, cond = oracle.vjp_scan(op, np.array([float(v) for v in yb]), np.array([float(v) for v in x]),
                              want_cond=True)
    assert [Fr(float(c)) for c in cond] == exp  # small dyadic rationals: exact


@pytest.mark.parametrize("op", ["min", "max"])
def test_scan_cond_min_max_selection_from_real_values(op):
    """MIN / MAX: every adjoint entry is a sum of selected ybar entries (the
    Jacobian is 0/1 at the REAL inputs), so cond = J(x)^T |ybar| with J from
    the exact primal definition at x itself."""
    rng = random.Random(99)
    n = 12
    x = [Fr(rng.randint(-3, 3)) for _ in range(n)]
    yb = [Fr(rng.randint(-7, 7)) for _ in range(n)]
    exp = vjp_by_duals(lambda v: scan(op, v), x, [abs(v) for v in yb])
    _, cond = oracle.vjp_scan(op, np.array([float(v) for v in yb]), np.array([float(v) for v in x]),
                              want_cond=True)
    assert [Fr(float(c)) for c in cond] == exp


def test_scan_cond_add_closed_form_and_bound():
    """scan(+): cond_i = sum_{j >= i} |ybar_j| (the reversed suffix sum of
    |ybar|), and |as_bar_i| <= cond_i for signed seeds."""
    rng = np.random.default_rng(5)
    yb = rng.integers(-8, 9, size=1000).astype(np.float64)
    ab, cond = oracle.vjp_scan("add", yb, None, want_cond=True)
    assert np.array_equal(cond, np.cumsum(np.abs(yb)[::-1])[::-1])
    assert np.all(np.abs(ab) <= cond)
    # LINREC with signed data: the adjoint never exceeds its condition scale
    a = rng.uniform(-1, 1, size=2000)
    y = rng.uniform(-1, 1, size=2000)
    ab, cond = oracle.vjp_scan("linrec", y, a, want_cond=True)
    assert np.all(np.abs(ab) <= cond * (1 + 1e-15))
    assert cond.min() > 0
