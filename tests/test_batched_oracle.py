"""Pins for the vectorised-scan oracle (oracle.vjp_scan_batched) —
CPU only.  It is the transpose rule over the sequential oracle; the pins check
the rule itself against things fixed independently of it: width 1 is the
plain scan, the vectorised plus is the per-column reversed suffix sum
(exact with integer seeds), columns do not interact (permuting
columns permutes the adjoint), and an exact dual-number Jacobian on a tiny
vectorised MUL scan."""
from __future__ import annotations

from fractions import Fraction as Fr

import numpy as np
import pytest
import torch

import oracle
import synth


def test_width_one_is_the_scan():
    a, yb = synth.linrec_inputs(1000)
    assert np.array_equal(oracle.vjp_scan_batched("linrec", yb.numpy(), a.numpy(), 1),
                          oracle.vjp_scan("linrec", yb.numpy(), a.numpy()))


def test_vectorised_plus_is_columnwise_suffix_sum():
    n, w = 3000, 7
    yb = synth.scan_add_seed(n * w, kind="int").numpy()
    got = oracle.vjp_scan_batched("add", yb, None, w).reshape(n, w)
    Y = yb.reshape(n, w).astype(np.int64)
    exact = np.flip(np.cumsum(np.flip(Y, 0), 0), 0)
    assert np.array_equal(got, exact.astype(np.float64))


@pytest.mark.parametrize("op", ["mul", "linrec", "mat2"])
def test_columns_do_not_interact(op):
    n, w = 500, 5
    W = {"mul": 1, "linrec": 2, "mat2": 4}[op]
    gen = {"linrec": synth.linrec_inputs, "mat2": synth.mat2_inputs}
    if op == "mul":
        a = (1.0 + (synth.uniform(n * w, 7) - 0.5) / 64).numpy()
        yb = synth.uniform(n * w, 8).numpy()
    else:
        a, yb = gen[op](n * w)
        a, yb = a.numpy(), yb.numpy()
    perm = np.array([3, 0, 4, 2, 1])
    A, Y = a.reshape(n, w, W), yb.reshape(n, w, W)
    g = oracle.vjp_scan_batched(op, yb, a, w).reshape(n, w, W)
    gp = oracle.vjp_scan_batched(op, np.ascontiguousarray(Y[:, perm]).ravel(),
                                 np.ascontiguousarray(A[:, perm]).ravel(), w).reshape(n, w, W)
    assert np.array_equal(gp, g[:, perm])


def test_vectorised_mul_exact_duals():
    """n = 4 elements of 3 components, integer values: the Jacobian of
    <ybar, scan (map (*)) xs> by exact forward mode on every input."""
    xs = [[2, -1, 3], [1, 4, -2], [3, 1, 5], [-2, 2, 1]]
    yb = [[1, 0, 2], [0, 1, 1], [3, 1, 0], [1, 2, 1]]
    n, w = 4, 3
    exp = np.zeros((n, w))
    for i in range(n):
        for j in range(w):
            tot = Fr(0)
            for k in range(i, n):  # d ys[k][j] / d xs[i][j] = prod_{l<=k, l!=i} xs[l][j]
                p = Fr(1)
                for l in range(k + 1):
                    if l != i:
                        p *= xs[l][j]
                tot += yb[k][j] * p
            exp[i, j] = float(tot)
    got = oracle.vjp_scan_batched("mul", np.array(yb, float).ravel(), np.array(xs, float).ravel(), w)
    assert np.array_equal(got.reshape(n, w), exp)
