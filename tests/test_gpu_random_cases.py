"""Seeded random sweep over every entry point and path switch (GPU vs the
oracle): random sizes (1 .. ~60k, tails in every tile position), dtypes, index
types, ACCUMULATE, out-of-range bins and the scan path flags (default / chunked / sweep /
look-back).  Complements the structured parity tests with combinations they do
not enumerate."""
from __future__ import annotations

import random

import numpy as np
import pytest
import torch

import oracle
import synth
from _parity import assert_close

pytestmark = pytest.mark.gpu
vjp = pytest.importorskip("paper_2202_10297_b200")
DEV = "cuda"
TD = {np.float64: torch.float64, np.float32: torch.float32}
W = {"add": 1, "mul": 1, "min": 1, "max": 1, "linrec": 2, "mat2": 4}


def scan_inputs(op, n, dt, seed):
    td = TD[dt]
    if op == "add":
        return None, synth.uniform(n, seed, lo=-1.0, hi=1.0, dtype=td)
    if op == "mul":
        a = (1.0 + (synth.uniform(n, seed, dtype=torch.float64) - 0.5) / 32).to(td)
        return a, synth.uniform(n, seed + 1, dtype=td)
    if op in ("min", "max"):
        return (synth.integers(n, seed, 0, 31).to(torch.float64) / 32).to(td), synth.uniform(n, seed + 1, dtype=td)
    gen = synth.linrec_inputs if op == "linrec" else synth.mat2_inputs
    a, y = gen(n, dtype=torch.float64)
    if op == "linrec":  # keep prod(c) away from underflow for elementwise comparison
        a = a.reshape(n, 2).clone()
        a[:, 1] = 1.0 + (synth.uniform(n, seed, dtype=torch.float64) - 0.5) / 64
        a = a.reshape(-1)
    return a.to(td), y.to(td)


@pytest.mark.parametrize("case", range(40))
def test_random_scan(case):
    rng = random.Random(1000 + case)
    op = rng.choice(list(W))
    dt = rng.choice([np.float64, np.float32])
    n = rng.choice([1, 2, 3, rng.randint(4, 300), rng.randint(300, 5000), rng.randint(5000, 60000)])
    path = rng.choice(["default", "chunked", "sweep", "lookback", "blocklb"])
    acc = rng.random() < 0.3
    a, yb = scan_inputs(op, n, dt, 50 + case)
    if a is None and path == "lookback":
        path = "default"
    kw = {"chunked": path == "chunked", "sweep": path == "sweep", "lookback": path == "lookback",
          "blocklb": path == "blocklb"}
    base = synth.uniform(n * W[op], 77, dtype=TD[dt]) if acc else None
    ref = oracle.vjp_scan(op, yb.numpy(), None if a is None else a.numpy(),
                          out=None if base is None else base.numpy().copy(), accumulate=acc)
    out = None if base is None else base.to(DEV)
    got = vjp.scan(op, yb.to(DEV), None if a is None else a.to(DEV), out=out, accumulate=acc, **kw)
    assert_close(got.cpu().numpy(), ref, dt, what=f"scan {op} {dt.__name__} n={n} {path} acc={acc}")


@pytest.mark.parametrize("case", range(20))
def test_random_reduce_and_rbi(case):
    rng = random.Random(2000 + case)
    dt = rng.choice([np.float64, np.float32])
    n = rng.choice([1, rng.randint(2, 1000), rng.randint(1000, 100_000)])
    op = rng.choice(["add", "mul", "min", "max", "linrec", "mat2"])
    if op in ("linrec", "mat2"):
        a, _ = scan_inputs(op, n, dt, 60 + case)
        yb = np.array([0.5, -1.5, 2.0, 0.25][:W[op]], dtype=dt)
        ref = oracle.vjp_reduce(op, a.numpy(), yb)[0]
        got = vjp.reduce(op, a.to(DEV), torch.from_numpy(yb).to(DEV))
    else:
        zeros = rng.choice(["none", "one", "two"]) if (op == "mul" and n >= 3) else "none"
        a = synth.mul_inputs(n, zeros=zeros, dtype=TD[dt]) if op == "mul" else \
            synth.min_inputs(n, dtype=TD[dt]) if op in ("min", "max") else synth.uniform(n, 3, dtype=TD[dt])
        ref = oracle.vjp_reduce(op, a.numpy(), 1.25)[0]
        got = vjp.reduce(op, a.to(DEV), 1.25)
    assert_close(got.cpu().numpy(), ref, dt, what=f"reduce {op} n={n}")
    # reduce_by_index on random bins (int32 / int64), some out of range
    op2 = rng.choice(["add", "mul", "min", "max"])
    m = rng.choice([1, 7, rng.randint(8, 2000), rng.randint(2000, 200_000)])
    itype = rng.choice([torch.int32, torch.int64])
    inds, av, hb = synth.rbi_inputs(n, m, op2, itype=itype, dtype=TD[dt])
    inds = inds.clone()
    if n > 10:
        inds[::7] = m + 3  # out of range: skipped, adjoint 0 (reading R4)
    ref2 = oracle.vjp_reduce_by_index(op2, inds.numpy(), av.numpy(), hb.numpy())[0]
    got2 = vjp.reduce_by_index(op2, inds.to(DEV), av.to(DEV), hb.to(DEV))
    assert_close(got2.cpu().numpy(), ref2, dt, what=f"rbi {op2} n={n} m={m} {itype}")


@pytest.mark.parametrize("case", range(12))
def test_random_scatter_batched_kmeans(case):
    rng = random.Random(3000 + case)
    dt = rng.choice([np.float64, np.float32])
    # scatter, width 1..5, in place or not
    n = rng.randint(1, 20_000)
    m = rng.randint(0, n)
    width = rng.randint(1, 5)
    is_, _ = synth.scatter_inputs(n, m, oob=min(m, rng.randint(0, 3)))
    yb = synth.uniform(n * width, 90 + case, lo=-1.0, hi=1.0, dtype=TD[dt])
    rx, rv, _ = oracle.vjp_scatter(is_.numpy(), yb.numpy(), width=width)
    xs, vs = vjp.scatter(is_.to(DEV), yb.to(DEV), width=width)
    assert np.array_equal(xs.cpu().numpy(), rx) and np.array_equal(vs.cpu().numpy(), rv)
    # vectorised scan
    op = rng.choice(list(W))
    rows, w = rng.randint(1, 3000), rng.randint(1, 70)
    a, y = scan_inputs(op, rows * w, dt, 95 + case)
    ref = oracle.vjp_scan_batched(op, y.numpy(), None if a is None else a.numpy(), w)
    got = vjp.scan_batched(op, y.to(DEV), None if a is None else a.to(DEV), width=w)
    assert_close(got.cpu().numpy(), ref, dt, what=f"batched {op} rows={rows} w={w}")
    # k-means
    npts, k, d = rng.randint(1, 4000), rng.randint(1, 150), rng.randint(1, 80)
    P, C = synth.kmeans_inputs(npts, k, d, dtype=torch.float64, k_true=max(1, k // 2))
    P, C = P.numpy().astype(dt), C.numpy().astype(dt)
    r = vjp.kmeans(torch.from_numpy(P).to(DEV), torch.from_numpy(C).to(DEV), 0.5)
    ref = oracle.kmeans(P, C, cost_bar=0.5)
    assert np.array_equal(r["assign"].cpu().numpy(), ref["assign"])
    assert np.array_equal(r["counts"].cpu().numpy(), ref["counts"])
    scale = np.zeros_like(C, dtype=np.float64)
    if npts:
        np.add.at(scale, ref["assign"], np.abs(C.astype(np.float64)[ref["assign"]] - P.astype(np.float64)))
    assert_close(r["cbar"].cpu().numpy(), ref["cbar"], dt, scale=scale.ravel(), what=f"kmeans {npts}x{k}x{d}")
