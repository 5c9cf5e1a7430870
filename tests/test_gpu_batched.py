"""GPU parity of the vectorised scan (vjp_scan_batched, SURVEY 8f row f2,
P:1226-1232) against the oracle's transpose rule: shapes from one element to
very wide (20 x 5000) and very tall (10^6 x 2), ragged chunk tails, f32/f64,
ACCUMULATE; integer seeds make the vectorised plus bit-exact."""
from __future__ import annotations

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
W = {"add": 1, "mul": 1, "linrec": 2, "mat2": 4}
SHAPES = [(1, 1), (5, 3), (1000, 1), (1000, 2), (777, 33), (4097, 7), (100_003, 16), (3001, 257), (20, 5000),
          (1_000_003, 2)]


def make(op, n, w, dt):
    m = n * w
    td = TD[dt]
    if op == "add":
        return None, synth.scan_add_seed(m, dtype=td)
    if op == "mul":
        a = (1.0 + (synth.uniform(m, 7, dtype=torch.float64) - 0.5) * 2.0 ** -6).to(td)
        return a, synth.uniform(m, 8, dtype=td)
    if op == "linrec":
        return synth.linrec_inputs(m, dtype=td)
    return synth.mat2_inputs(m, dtype=td)


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("op", ["add", "mul", "linrec", "mat2"])
def test_batched_parity(op, dt):
    for n, w in SHAPES:
        if op == "mat2" and n * w > 300_000:
            continue  # oracle time
        a, yb = make(op, n, w, dt)
        ref = oracle.vjp_scan_batched(op, yb.numpy(), None if a is None else a.numpy(), w)
        got = vjp.scan_batched(op, yb.to(DEV), None if a is None else a.to(DEV), width=w).cpu().numpy()
        assert_close(got, ref, dt, what=f"batched {op} n={n} w={w}")


def test_batched_add_integer_bit_exact_and_accumulate():
    n, w = 200_001, 5
    yb = synth.scan_add_seed(n * w, kind="int")
    ref = oracle.vjp_scan_batched("add", yb.numpy(), None, w)
    assert np.array_equal(vjp.scan_batched("add", yb.to(DEV), width=w).cpu().numpy(), ref)
    a, y = synth.linrec_inputs(50_000 * 3)
    base = synth.uniform(a.numel(), 12)
    ref = oracle.vjp_scan_batched("linrec", y.numpy(), a.numpy(), 3, out=base.numpy().copy(), accumulate=True)
    out = base.to(DEV)
    vjp.scan_batched("linrec", y.to(DEV), a.to(DEV), width=3, out=out, accumulate=True)
    assert_close(out.cpu().numpy(), ref, np.float64, what="batched accumulate")


@pytest.mark.parametrize("op", ["min", "max"])
def test_batched_minmax(op):
    """MIN/MAX vectorised scans (pick-left ties, +-inf first row) vs the
    oracle's transpose rule over the sequential scalar scans."""
    for n, w in ((1, 1), (777, 33), (4097, 7), (100_003, 16), (20, 5000)):
        k = synth.integers(n * w, 9, 0, 15)
        a = k.to(torch.float64) / 16.0
        a[:w] = float("inf") if op == "min" else float("-inf")
        yb = synth.uniform(n * w, 10)
        ref = oracle.vjp_scan_batched(op, yb.numpy(), a.numpy(), w)
        got = vjp.scan_batched(op, yb.to(DEV), a.to(DEV), width=w).cpu().numpy()
        assert_close(got, ref, np.float64, what=f"batched {op} n={n} w={w}")


def test_batched_empty():
    yb = torch.empty(0, dtype=torch.float64, device=DEV)
    assert vjp.scan_batched("add", yb, width=3).numel() == 0
