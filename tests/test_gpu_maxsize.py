"""Maximum-size edge cases: element counts above 2^31 (every index, offset and
tile count must be 64-bit).  Each case checks a property that fixes the whole
result, on inputs whose arithmetic is exact (integer-valued f64), or sampled
elements against the oracle / the paper's closed form:

- scan(+): as_bar[n-1] = ys_bar[n-1] and as_bar[i] - as_bar[i+1]
  = ys_bar[i] for every i (by induction this is the reversed suffix sum), both
  on the default one-read sweep and the chunked kernels;
- reduce(min): the argmin planted beyond 2^31 wins (lowest index
  among ties), the dense adjoint is y_bar there and 0 elsewhere;
- reduce_by_index(+): as_bar = hs_bar[inds] for every element;
- scatter with int64 targets beyond 2^31, in place.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
vjp = pytest.importorskip("paper_2202_10297_b200")
DEV = "cuda"
BIG = (1 << 31) + 77


@pytest.mark.parametrize("path", ["default", "chunked"])
def test_scan_add_above_2pow31(path):
    yb = synth.scan_add_seed(BIG, kind="int", device=DEV)
    got = vjp.scan("add", yb, chunked=(path == "chunked"))
    assert float(got[-1]) == float(yb[-1])
    assert torch.equal(got[:-1] - got[1:], yb[:-1])
    # sampled closed form (suffix sums, exact for integers) and the oracle on the tail
    for i in (0, 1, (1 << 31) - 1, 1 << 31, BIG - 2):
        assert float(got[i]) == float(yb[i:].sum())
    tail = yb[-4096:].cpu().numpy()
    assert np.array_equal(got[-4096:].cpu().numpy(), oracle.vjp_scan("add", tail, None))


def test_reduce_min_argmin_above_2pow31():
    a = synth.uniform(BIG, 7, dtype=torch.float32, device=DEV) + 1.0
    k = (1 << 31) + 5
    a[k] = 0.25
    a[k + 9] = 0.25  # a later tie: the lowest index wins
    ab, y, arg = vjp.reduce("min", a, 1.5, want_y=True)
    assert int(arg) == k and float(y) == 0.25
    assert float(ab[k]) == 1.5 and int(torch.count_nonzero(ab)) == 1


def test_rbi_add_above_2pow31():
    m = 1000
    inds = synth.integers(BIG, 400, 0, m - 1, device=DEV, dtype=torch.int32)
    hb = synth.uniform(m, 401, device=DEV)
    got = vjp.reduce_by_index("add", inds, None, hb)
    assert torch.equal(got, hb[inds.long()])


def test_scatter_int64_targets_above_2pow31():
    n = BIG
    yb = synth.uniform(n, 9, dtype=torch.float32, device=DEV)
    is_ = torch.tensor([n - 1, (1 << 31) + 1, 1 << 31, 3, n + 5], dtype=torch.int64, device=DEV)
    ref_v = yb[is_[:4]].clone()
    xb, vb = vjp.scatter(is_, yb, in_place=True)
    assert torch.equal(vb[:4], ref_v) and float(vb[4]) == 0.0
    assert int(torch.count_nonzero(xb[is_[:4]])) == 0
