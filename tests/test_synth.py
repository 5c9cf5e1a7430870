"""The seeded generator is counter-based: a shard equals the same slice of the
whole array (so multi-GPU shards never depend on the rank count)."""
import torch

import synth


def test_shard_equals_slice():
    full = synth.uniform(1000, 7)
    assert torch.equal(full[300:700], synth.uniform(400, 7, offset=300))
    a, y = synth.mat2_inputs(100)
    a2, y2 = synth.mat2_inputs(40, offset=30)
    assert torch.equal(a[120:280], a2) and torch.equal(y[120:280], y2)


def test_ranges_and_dtypes():
    u = synth.uniform(10000, 1)
    assert u.dtype == torch.float64 and float(u.min()) >= 0 and float(u.max()) < 1
    i = synth.integers(10000, 2, -8, 8)
    assert int(i.min()) == -8 and int(i.max()) == 8
    inds, a, hb = synth.rbi_inputs(5000, 10, "max")
    assert inds.dtype == torch.int32 and int(inds.min()) >= 0 and int(inds.max()) < 10
    assert float(hb.min()) >= 0.5
    m = synth.mul_inputs(4096, zeros="two")
    assert int((m == 0).sum()) == 2
    assert int((torch.signbit(m) & (m == 0)).sum()) == 1
    mn = synth.min_inputs(1 << 16)
    assert float(mn.min()) == -(2.0 ** -24) and int((mn == mn.min()).sum()) == 3
    is_, yb = synth.scatter_inputs(1000, 300)
    assert len(set(is_.tolist())) == 300 and int(is_.max()) < 1000
