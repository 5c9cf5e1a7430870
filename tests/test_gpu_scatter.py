"""GPU parity of vjp_scatter (sec 5.3) against the oracle: gathered vs_bar
and zeroed xs_bar are copies, so bit-exact; in-place and copying forms;
out-of-range targets skipped; duplicate / OOB detection with CHECK_INDICES."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
vjp = pytest.importorskip("paper_2202_10297_b200")
DEV = "cuda"


@pytest.mark.parametrize("it", [torch.int32, torch.int64], ids=["i32", "i64"])
@pytest.mark.parametrize("dt", [torch.float64, torch.float32], ids=["f64", "f32"])
def test_scatter_parity(dt, it):
    for n, m, width, oob in [(1, 1, 1, 0), (4, 2, 1, 0), (1000, 300, 1, 3), (100_003, 50_000, 1, 7),
                             (4096, 1000, 3, 2), (1 << 20, 1 << 16, 1, 0)]:
        is_, yb = synth.scatter_inputs(n, m, dtype=dt, itype=it, oob=oob)
        yb = yb.repeat_interleave(width) if width > 1 else yb
        ref_x, ref_v, rc = oracle.vjp_scatter(is_.numpy(), yb.numpy(), width=width)
        assert rc == 0
        xb, vb = vjp.scatter(is_.to(DEV), yb.to(DEV), width=width)
        assert np.array_equal(xb.cpu().numpy(), ref_x) and np.array_equal(vb.cpu().numpy(), ref_v)
        y2 = yb.to(DEV)
        xb2, vb2 = vjp.scatter(is_.to(DEV), y2, width=width, in_place=True)
        assert xb2.data_ptr() == y2.data_ptr()
        assert np.array_equal(xb2.cpu().numpy(), ref_x) and np.array_equal(vb2.cpu().numpy(), ref_v)


def test_scatter_spec_example_and_checks():
    yb = torch.tensor([10.0, 11, 12, 13], device=DEV)
    xb, vb = vjp.scatter(torch.tensor([1, 7, 3], device=DEV), yb)  # G9: 7 is out of range
    assert xb.cpu().tolist() == [10, 0, 12, 0] and vb.cpu().tolist() == [11, 0, 13]
    with pytest.raises(vjp.VjpError) as e:
        vjp.scatter(torch.tensor([1, 1], device=DEV), yb, check=True)
    assert e.value.code == 5
    with pytest.raises(vjp.VjpError) as e:
        vjp.scatter(torch.tensor([1, 9], device=DEV), yb, check=True)
    assert e.value.code == 6


def test_scatter_accumulate():
    is_, yb = synth.scatter_inputs(10_000, 3000)
    base = synth.uniform(3000, 800, dtype=torch.float64)
    _, ref_v, _ = oracle.vjp_scatter(is_.numpy(), yb.numpy(), vs_out=base.numpy().copy(), accumulate=True)
    vs = base.to(DEV)
    vjp.scatter(is_.to(DEV), yb.to(DEV), vs_out=vs, accumulate=True)
    assert np.array_equal(vs.cpu().numpy(), ref_v)
