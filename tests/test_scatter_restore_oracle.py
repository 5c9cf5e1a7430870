"""Pins of the oracle's in-place scatter forward save / restore (sec 5.3,
P:1255-1276) to things other than itself:
- a hand-worked example (values written out below from the definitions);
- the primal scatter of tests/_exact.py (a separate pure-Python definition);
- the round trip restore(forward(xs)) == xs for distinct targets (P:1271-1272:
  "restores xs to its state before the update");
- the transpose identity <ys_bar, scatter xs is vs> = <xs_bar, xs> + <vs_bar, vs>
  tying the oracle's adjoint (vjp_scatter) to its primal (scatter) — the map is
  linear in (xs, vs), so its vjp is its transpose.
"""
from __future__ import annotations

import random

import numpy as np

import oracle
from _exact import scatter as exact_scatter


def test_hand_example():
    xs = np.array([0.0, 1.0, 2.0, 3.0, 4.0, 5.0])
    is_ = np.array([4, 1, 9])  # 9 out of range: skipped, saved 0 (reading R4)
    vs = np.array([-4.0, -1.0, -9.0])
    ys, saved = oracle.scatter_forward(xs, is_, vs)
    assert ys.tolist() == [0.0, -1.0, 2.0, 3.0, -4.0, 5.0]
    assert saved.tolist() == [4.0, 1.0, 0.0]
    assert oracle.scatter_restore(ys, is_, saved).tolist() == xs.tolist()
    # width 2: elements are pairs
    xs2 = np.arange(8.0)
    ys2, s2 = oracle.scatter_forward(xs2, np.array([2]), np.array([-5.0, -6.0]), width=2)
    assert ys2.tolist() == [0, 1, 2, 3, -5, -6, 6, 7] and s2.tolist() == [4, 5]


def test_matches_exact_definition_and_round_trip():
    rng = random.Random(7)
    for _ in range(50):
        n = rng.randint(0, 40)
        m = rng.randint(0, n + 3)
        targets = rng.sample(range(n + 5), min(m, n + 5))  # distinct, some out of range
        xs = [rng.uniform(-1, 1) for _ in range(n)]
        vs = [rng.uniform(-1, 1) for _ in targets]
        ys, saved = oracle.scatter_forward(np.array(xs), np.array(targets, np.int64), np.array(vs))
        assert ys.tolist() == exact_scatter(xs, targets, vs)
        assert saved.tolist() == [xs[t] if t < n else 0.0 for t in targets]
        back = oracle.scatter_restore(ys, np.array(targets, np.int64), saved)
        assert back.tolist() == xs


def test_transpose_identity_with_vjp_scatter():
    rng = np.random.default_rng(3)
    for n, m, width in [(10, 4, 1), (50, 20, 3), (7, 7, 2)]:
        is_ = rng.permutation(n)[:m].astype(np.int64)
        xs = rng.standard_normal(n * width)
        vs = rng.standard_normal(m * width)
        yb = rng.standard_normal(n * width)
        ys, _ = oracle.scatter_forward(xs, is_, vs, width=width)
        xb, vb, rc = oracle.vjp_scatter(is_, yb, width=width)
        assert rc == 0
        lhs = float(yb @ ys)
        rhs = float(xb @ xs + vb @ vs)
        assert abs(lhs - rhs) <= 1e-12 * (np.abs(yb) @ np.abs(ys) + 1.0)
