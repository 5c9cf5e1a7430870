"""GPU parity of vjp_reduce (sec 5.1) against the oracle, through the C ABI.

The oracle uses the paper's GENERAL rule for * (prefix x suffix products,
P:1006-1011); the kernels use the (p, z) special case, so
parity also checks special == general.  Indices (argmin/argmax, first zero)
are compared bit-exactly.  Config 3 (n = 2^30 f32) runs at full size in the
`slow` cases."""
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
SIZES = [1, 2, 3, 5, 31, 1000, 4097, 100_003, (1 << 20) + 7]
TD = {np.float32: torch.float32, np.float64: torch.float64}


def data(op, n, dt, zeros="none"):
    td = TD[dt]
    if op == "mul":
        return synth.mul_inputs(n, zeros=zeros, dtype=td)
    if op in ("min", "max"):
        a = synth.min_inputs(n, dtype=td)
        return -a if op == "max" else a
    return synth.uniform(n, 600, dtype=td)


def check(op, a, yb, dt, accumulate=False):
    ref_ab, ref_y, ref_arg, ref_z = oracle.vjp_reduce(op, a.numpy(), yb)
    ab, y, arg = vjp.reduce(op, a.to(DEV), yb, want_y=True)
    ab = ab.cpu().numpy()
    if op in ("min", "max"):
        assert int(arg.item()) == ref_arg  # bit-exact index (first index on ties)
        assert np.array_equal(ab, ref_ab)  # a copy of ybar: bit-exact
        assert float(y.item()) == float(ref_y)
    elif op == "mul":
        assert int(arg.item()) == (ref_arg if ref_z > 0 else -1)
        if ref_z >= 2:
            assert not ab.any()
        elif ref_z == 1:
            assert np.count_nonzero(ab) <= 1
            assert_close(ab, ref_ab, dt, what="mul z=1")
        else:
            assert_close(ab, ref_ab, dt, what="mul z=0")
        assert_close(np.array([float(y.item())]), np.array([float(ref_y)]), dt, what="y")
    else:
        assert np.array_equal(ab, ref_ab)
        assert_close(np.array([float(y.item())]), np.array([float(ref_y)]), np.float32, what="sum")


@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=["f32", "f64"])
@pytest.mark.parametrize("op", ["add", "mul", "min", "max"])
def test_reduce_sizes(op, dt):
    for n in SIZES:
        check(op, data(op, n, dt), 1.5, dt)


@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=["f32", "f64"])
@pytest.mark.parametrize("zeros", ["none", "one", "two", "sparse"])
def test_reduce_mul_zero_cases(zeros, dt):
    """z = 0, 1 (one of them -0.0), >= 2 zeros."""
    for n in (7, 4099, 1 << 21):
        check("mul", data("mul", n, dt, zeros=zeros), 2.0, dt)


def test_reduce_min_ties_signed_zero():
    """G8: IEEE tie of +0.0 and -0.0 -> the lower index wins."""
    a = torch.tensor([1.0, 0.0, -0.0, 2.0, 0.0], dtype=torch.float64)
    ab, y, arg = vjp.reduce("min", a.to(DEV), 5.0, want_y=True)
    assert int(arg.item()) == 1 and ab.cpu().tolist() == [0, 5, 0, 0, 0]


def test_reduce_accumulate_touches_only_documented():
    n = 100_001
    for op in ("min", "max", "mul"):
        a = data(op, n, np.float64, zeros="one")
        base = synth.uniform(n, 601, dtype=torch.float64)
        ref = oracle.vjp_reduce(op, a.numpy(), 3.0, out=base.numpy().copy(), accumulate=True)[0]
        out = base.to(DEV)
        vjp.reduce(op, a.to(DEV), 3.0, out=out, accumulate=True)
        got = out.cpu().numpy()
        changed = np.nonzero(got != base.numpy())[0]
        assert len(changed) <= 1  # only the argmin / the zero's position
        assert_close(got, ref, np.float64, what=f"acc {op}")


@pytest.mark.slow
@pytest.mark.parametrize("case", ["mul-none", "mul-one", "mul-two", "mul-sparse", "min"])
def test_config3_full_size(case):
    """config 3: n = 2^30 f32 (reduce(*) with injected zeros, reduce(min) argmin)."""
    n = 1 << 30
    op = case.split("-")[0]
    if op == "mul":
        a = synth.mul_inputs(n, zeros=case.split("-")[1], dtype=torch.float32, device=DEV)
    else:
        a = synth.min_inputs(n, dtype=torch.float32, device=DEV)
    ab, y, arg = vjp.reduce(op, a, 1.0, want_y=True)
    a_h = a.cpu().numpy()
    ref_ab, ref_y, ref_arg, ref_z = oracle.vjp_reduce(op, a_h, 1.0)
    got = ab.cpu().numpy()
    if op == "min":
        assert int(arg.item()) == ref_arg
        assert np.array_equal(got, ref_ab)
    else:
        if ref_z:
            assert int(arg.item()) == ref_arg
        assert_close(got, ref_ab, np.float32, what=case)


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("op", ["linrec", "mat2"])
def test_reduce_general_rule(op, dt):
    """LINREC / MAT2 reduce (the paper's general rule) through the
    chunked kernels with a virtual ys_bar, against the oracle's literal
    exclusive-scans-and-map; sizes from one element through ragged tiles;
    the primal y and ACCUMULATE."""
    import synth
    gen = {"linrec": synth.linrec_inputs, "mat2": synth.mat2_inputs}[op]
    w = 2 if op == "linrec" else 4
    td = torch.float64 if dt == np.float64 else torch.float32
    ybar = torch.tensor([0.75, -1.25, 0.5, 2.0][:w], dtype=td)
    def inputs(n):
        a, _ = gen(n, dtype=torch.float64)
        if op == "linrec":  # prod(c) of 10^6 draws from U(0.5, 1) underflows: keep c near 1
            a = a.reshape(n, 2).clone()
            a[:, 1] = 1.0 + (synth.uniform(n, 13, dtype=torch.float64) - 0.5) / 256
            a = a.reshape(-1)
        return a.to(td)

    for n in (1, 2, 33, 1023, 1024, 4097, 100_003, 1_000_001):
        a = inputs(n)
        ref, ry, _, _ = oracle.vjp_reduce(op, a.numpy(), ybar.numpy())
        got, y, arg = vjp.reduce(op, a.to("cuda"), ybar.to("cuda"), want_y=True)
        assert_close(got.cpu().numpy(), ref, dt, what=f"general reduce {op} n={n}")
        assert_close(y.cpu().numpy(), np.asarray(ry), dt, what=f"general reduce y {op} n={n}")
        assert int(arg.item()) == -1
    n = 70_001
    a = inputs(n)
    base = synth.uniform(n * w, 12, dtype=td)
    ref, _, _, _ = oracle.vjp_reduce(op, a.numpy(), ybar.numpy(), out=base.numpy().copy(), accumulate=True)
    out = base.to("cuda")
    vjp.reduce(op, a.to("cuda"), ybar.to("cuda"), out=out, accumulate=True)
    assert_close(out.cpu().numpy(), ref, dt, what=f"general reduce accumulate {op}")


def test_reduce_general_rule_empty_and_single():
    """n = 0 is a no-op (R7); n = 1: abar_0 = ybar (J_R(e, a) = I for lin_o and the 2x2 product)."""
    yb = torch.tensor([0.5, -2.0, 1.0, 3.0], dtype=torch.float64, device="cuda")
    assert vjp.reduce("mat2", torch.empty(0, dtype=torch.float64, device="cuda"), yb).numel() == 0
    a = torch.tensor([0.3, 0.7, 0.2, 0.8], dtype=torch.float64, device="cuda")
    assert torch.equal(vjp.reduce("mat2", a, yb), yb)
    a2 = torch.tensor([0.25, 0.5], dtype=torch.float64, device="cuda")
    assert torch.equal(vjp.reduce("linrec", a2, yb[:2]), yb[:2])
