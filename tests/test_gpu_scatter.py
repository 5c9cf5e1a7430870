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


@pytest.mark.parametrize("it", [torch.int32, torch.int64], ids=["i32", "i64"])
@pytest.mark.parametrize("dt", [torch.float64, torch.float32], ids=["f64", "f32"])
def test_scatter_forward_restore_parity(dt, it):
    """vjp_scatter_forward / vjp_scatter_restore vs the oracle,
    bit-exact (pure data movement), then the paper's whole in-place cycle:
    forward save + update, the adjoint in place, the restore."""
    for n, m, width, oob in [(1, 1, 1, 0), (4, 2, 1, 1), (1000, 300, 1, 3), (4096, 1000, 3, 2),
                             (20_011, 5_000, 2, 0)]:
        is_, yb = synth.scatter_inputs(n, m, dtype=dt, itype=it, oob=oob)
        xs = synth.uniform(n * width, 31, lo=-1.0, hi=1.0, dtype=dt)
        vs = synth.uniform(m * width, 32, lo=-1.0, hi=1.0, dtype=dt)
        ref_ys, ref_saved = oracle.scatter_forward(xs.numpy(), is_.numpy(), vs.numpy(), width=width)
        x = xs.to(DEV)
        saved = vjp.scatter_forward(x, is_.to(DEV), vs.to(DEV), width=width, check=(oob == 0))
        assert np.array_equal(x.cpu().numpy(), ref_ys) and np.array_equal(saved.cpu().numpy(), ref_saved)
        ybar = (yb.repeat_interleave(width) if width > 1 else yb).to(DEV)
        ref_x, ref_v, _ = oracle.vjp_scatter(is_.numpy(), ybar.cpu().numpy(), width=width)
        xb, vb = vjp.scatter(is_.to(DEV), ybar, width=width, in_place=True)
        assert np.array_equal(xb.cpu().numpy(), ref_x) and np.array_equal(vb.cpu().numpy(), ref_v)
        back = vjp.scatter_restore(x, is_.to(DEV), saved, width=width)
        assert back.data_ptr() == x.data_ptr()
        assert np.array_equal(back.cpu().numpy(), oracle.scatter_restore(ref_ys, is_.numpy(), ref_saved, width=width))
        assert torch.equal(back.cpu(), xs)  # restored to its state before the update


def test_scatter_forward_checks_and_empty():
    x = torch.arange(6.0, device=DEV, dtype=torch.float64)
    with pytest.raises(vjp.VjpError) as e:  # duplicate target: nothing written
        vjp.scatter_forward(x, torch.tensor([2, 2], device=DEV), torch.zeros(2, dtype=torch.float64, device=DEV),
                            check=True)
    assert e.value.code == 5 and x.cpu().tolist() == [0, 1, 2, 3, 4, 5]
    with pytest.raises(vjp.VjpError) as e:
        vjp.scatter_forward(x, torch.tensor([2, 6], device=DEV), torch.zeros(2, dtype=torch.float64, device=DEV),
                            check=True)
    assert e.value.code == 6
    saved = vjp.scatter_forward(x, torch.empty(0, dtype=torch.int64, device=DEV),
                                torch.empty(0, dtype=torch.float64, device=DEV))
    assert saved.numel() == 0 and x.cpu().tolist() == [0, 1, 2, 3, 4, 5]
    vjp.scatter_restore(x, torch.empty(0, dtype=torch.int64, device=DEV), saved)
    assert x.cpu().tolist() == [0, 1, 2, 3, 4, 5]


@pytest.mark.slow
def test_scatter_forward_restore_large_sampled():
    """n = 2^28 f64, m = 2^20: the forward/restore touch only the m targets;
    sampled elements vs the definitions, and the restore is exact everywhere."""
    n, m = 1 << 28, 1 << 20
    is_, _ = synth.scatter_inputs(n, m, device=DEV)
    xs = torch.arange(n, dtype=torch.float64, device=DEV)
    vs = -torch.arange(1, m + 1, dtype=torch.float64, device=DEV)
    saved = vjp.scatter_forward(xs, is_, vs)
    assert torch.equal(saved, is_.double())
    assert torch.equal(xs[is_], vs)
    vjp.scatter_restore(xs, is_, saved)
    assert torch.equal(xs, torch.arange(n, dtype=torch.float64, device=DEV))
