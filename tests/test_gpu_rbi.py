"""GPU parity of vjp_reduce_by_index (sec 5.1.2) against the oracle.

Per-bin winners (MIN/MAX, lowest index on ties) and zero counts (MUL) are
compared bit-exactly; adjoints within the north_star tolerance (ADD and
MIN/MAX adjoints are copies of hs_bar, so bit-exact).  m spans the shared-
memory and the global-atomic forward paths.  Config 4 (n = 2^28, m = 10^3 and
10^6) runs at full size in the `slow` cases."""
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
TD = {np.float32: torch.float32, np.float64: torch.float64}


def run(op, n, m, dt, it=torch.int32, oob=False, skew=False):
    inds, a, hb = synth.rbi_inputs(n, m, op, dtype=TD[dt], itype=it, skew=skew)
    if oob and n > 4:
        inds[1] = -1
        inds[3] = m + 5
    ref_ab, ref_hs, ref_win, ref_z = oracle.vjp_reduce_by_index(op, inds.numpy(), a.numpy(), hb.numpy())
    ab, hs, win = vjp.reduce_by_index(op, inds.to(DEV), a.to(DEV), hb.to(DEV), want_hs=True)
    ab = ab.cpu().numpy()
    if op in ("min", "max"):
        assert np.array_equal(win.cpu().numpy(), ref_win), "winner indices differ"
        assert np.array_equal(ab, ref_ab)
        occupied = ref_win >= 0
        assert np.array_equal(hs.cpu().numpy()[occupied], ref_hs[occupied])
    elif op == "mul":
        assert np.array_equal(win.cpu().numpy(), ref_z), "zero counts differ"
        assert_close(ab, ref_ab, dt, what=f"rbi mul n={n} m={m}")
    else:
        assert np.array_equal(ab, ref_ab)
        assert_close(hs.cpu().numpy(), ref_hs, dt, scale=np.full(m, max(1.0, n / m)), what="primal sum")


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("op", ["add", "mul", "min", "max"])
def test_rbi_sizes(op, dt):
    for n, m in [(1, 1), (5, 3), (1000, 1), (4097, 17), (100_003, 1000), (100_003, 2100), (300_001, 4096),
                 (300_001, 20_000), (1 << 20, 1_000_000)]:
        run(op, n, m, dt, oob=True)


@pytest.mark.parametrize("op", ["add", "mul", "max"])
def test_rbi_int64_and_skew(op):
    run(op, 200_001, 1000, np.float64, it=torch.int64)
    run(op, 200_001, 50_000, np.float64, it=torch.int64, skew=True)


def test_rbi_golden_g5_g6():
    inds = torch.tensor([0, 1, 0, 1, 2, 2], dtype=torch.int32)
    a = torch.tensor([2, 0, 3, 5, 0, 0], dtype=torch.float64)
    got = vjp.reduce_by_index("mul", inds.to(DEV), a.to(DEV), torch.tensor([1.0, 10, 100], dtype=torch.float64, device=DEV))
    # the special-case path forms p_b from fixed-point log2 codes (reading R13b): exact up to
    # rounding (north_star tolerance); the general rule multiplies exactly: bit-exact
    assert_close(got.cpu().numpy(), np.array([3.0, 50, 2, 0, 0, 0]), np.float64, what="G5")
    g = vjp.reduce_by_index("mul", inds.to(DEV), a.to(DEV), torch.tensor([1.0, 10, 100], dtype=torch.float64,
                                                                         device=DEV), general=True)
    assert g.cpu().tolist() == [3, 50, 2, 0, 0, 0]
    inds = torch.tensor([0, 1, 0, 1, 0], dtype=torch.int32)
    a = torch.tensor([3, 5, 3, -1, 2], dtype=torch.float64)
    got = vjp.reduce_by_index("max", inds.to(DEV), a.to(DEV), torch.tensor([7.0, 9], dtype=torch.float64, device=DEV))
    assert got.cpu().tolist() == [7, 9, 0, 0, 0]


def test_rbi_accumulate():
    n, m = 100_003, 777
    for op in ("add", "mul", "max"):
        inds, a, hb = synth.rbi_inputs(n, m, op)
        base = synth.uniform(n, 700, dtype=torch.float64)
        ref = oracle.vjp_reduce_by_index(op, inds.numpy(), a.numpy(), hb.numpy(), out=base.numpy().copy(),
                                         accumulate=True)[0]
        out = base.to(DEV)
        vjp.reduce_by_index(op, inds.to(DEV), a.to(DEV), hb.to(DEV), out=out, accumulate=True)
        assert_close(out.cpu().numpy(), ref, np.float64, what=f"acc {op}")


@pytest.mark.slow
@pytest.mark.parametrize("m", [1000, 1_000_000])
@pytest.mark.parametrize("op", ["add", "mul", "max"])
def test_config4_full_size(op, m):
    """config 4: n = 2^28, f64 values, int32 bins, k-means-shaped (uniform bins)."""
    n = 1 << 28
    inds, a, hb = synth.rbi_inputs(n, m, op, device=DEV)
    ab, hs, win = vjp.reduce_by_index(op, inds, a, hb, want_hs=True)
    ref_ab, ref_hs, ref_win, ref_z = oracle.vjp_reduce_by_index(op, inds.cpu().numpy(), a.cpu().numpy(),
                                                                hb.cpu().numpy())
    got = ab.cpu().numpy()
    if op == "max":
        assert np.array_equal(win.cpu().numpy(), ref_win)
        assert np.array_equal(got, ref_ab)
    elif op == "mul":
        assert np.array_equal(win.cpu().numpy(), ref_z)
        assert_close(got, ref_ab, np.float64, what=f"config4 mul m={m}")
    else:
        assert np.array_equal(got, ref_ab)


def test_rbi_mul_code_accuracy():
    """the MUL histograms' factor codes round(log2|x| 2^51) + [x<0] 2^63
    (reading R13b) against the exact codes from Python's decimal module (50
    digits, no floating-point library routine): within 2 quanta (2^-50 on
    log2) over wide-range, near-1, table-boundary and subnormal inputs; the
    sign bit exact."""
    from decimal import Decimal, getcontext
    getcontext().prec = 50
    ln2 = Decimal(2).ln()
    x = torch.cat([
        torch.exp2((synth.uniform(20_000, 90, dtype=torch.float64) - 0.5) * 2000),
        1.0 + (synth.uniform(20_000, 91, dtype=torch.float64) - 0.5) * 2.0 ** -10,
        1.0 + torch.arange(129, dtype=torch.float64) / 128.0,  # table cell edges
        torch.tensor([1.0, 2.0, 0.5, 3.0, 1e-310, 5e-324, 1.7976931348623157e308, 1.4142135623730951,
                      1.9999999999999998, 1.0000000000000002, 0.7071067811865475], dtype=torch.float64),
    ])
    x = torch.where(synth.uniform(x.numel(), 92) < 0.5, -x, x)
    xd = x.to("cuda")
    y = torch.empty(xd.numel(), dtype=torch.int64, device="cuda")
    vjp._check(vjp.lib().vjp_debug_mul_code(vjp._p(xd), vjp._p(y), xd.numel(), vjp._stream(xd.device)), "code")
    got = [int(v) & ((1 << 64) - 1) for v in y.cpu().tolist()]
    worst = 0
    for v, g in zip(x.tolist(), got):
        exact = (Decimal(abs(v)).ln() / ln2) * (1 << 51)
        q = int(exact.to_integral_value())
        expect = (q + ((1 << 63) if v < 0 else 0)) & ((1 << 64) - 1)
        d = (g - expect) & ((1 << 64) - 1)
        d = d - (1 << 64) if d >= (1 << 63) else d
        worst = max(worst, abs(d))
    assert worst <= 2, worst


@pytest.mark.parametrize("it", [torch.int32, torch.int64], ids=["i32", "i64"])
@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_rbi_mul_general_rule(dt, it):
    """vjp_reduce_by_index_general (counting sort + per-bin
    exclusive product scans) vs the oracle (whose per-bin l_i r_i is the same
    rule, computed sequentially in index order): zeros per bin 0 / 1 / >= 2
    (synth: Poisson(1) zeros per bin), out-of-range bins, one bin, skew."""
    for n, m, skew in [(1, 1, False), (5, 3, False), (1000, 1, False), (4097, 17, False), (100_003, 1000, False),
                       (300_001, 20_000, True), (1 << 20, 1_000_000, False)]:
        inds, a, hb = synth.rbi_inputs(n, m, "mul", dtype=TD[dt], itype=it, skew=skew)
        if n > 4:
            inds[1] = -1
            inds[3] = m + 5
        ref = oracle.vjp_reduce_by_index("mul", inds.numpy(), a.numpy(), hb.numpy())[0]
        got = vjp.reduce_by_index("mul", inds.to(DEV), a.to(DEV), hb.to(DEV), general=True)
        assert_close(got.cpu().numpy(), ref, dt, what=f"rbi mul general n={n} m={m}")
        if n > 4:
            assert float(got[1]) == 0.0 and float(got[3]) == 0.0


def test_rbi_mul_general_accumulate_and_unsupported():
    inds, a, hb = synth.rbi_inputs(50_000, 300, "mul")
    base = synth.uniform(50_000, 33)
    ref = oracle.vjp_reduce_by_index("mul", inds.numpy(), a.numpy(), hb.numpy(), out=base.numpy().copy(),
                                     accumulate=True)[0]
    out = base.to(DEV)
    vjp.reduce_by_index("mul", inds.to(DEV), a.to(DEV), hb.to(DEV), out=out, accumulate=True, general=True)
    assert_close(out.cpu().numpy(), ref, np.float64, what="general accumulate")
    with pytest.raises(vjp.VjpError) as e:
        vjp.reduce_by_index("add", inds.to(DEV), a.to(DEV), hb.to(DEV), general=True)
    assert e.value.code == 2


# ---------------------------------------------------------------- width > 1
@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("op", ["add", "mul", "min", "max"])
@pytest.mark.parametrize("width", [2, 3, 8, 33, 64])
def test_rbi_width(op, width, dt):
    """vectorised operator (reading A24): per-(bin, component)
    winners / zero counts bit-exact, adjoints vs the oracle (run per component)."""
    n, m = 20_011, 300
    inds, a, hb = synth.rbi_wide_inputs(n, m, width, op, dtype=TD[dt])
    inds[1] = -1
    inds[3] = m + 5
    ref_ab, ref_hs, ref_win, ref_z = oracle.vjp_reduce_by_index(op, inds.numpy(), a.numpy(), hb.numpy(), width=width)
    ab, hs, win = vjp.reduce_by_index(op, inds.to(DEV), a.to(DEV), hb.to(DEV), want_hs=True, width=width)
    ab = ab.cpu().numpy()
    if op in ("min", "max"):
        assert np.array_equal(win.cpu().numpy(), ref_win), "winner indices differ"
        assert np.array_equal(ab, ref_ab)
    elif op == "mul":
        assert np.array_equal(win.cpu().numpy(), ref_z), "zero counts differ"
        assert_close(ab, ref_ab, dt, what=f"rbi mul width={width}")
    else:
        assert np.array_equal(ab, ref_ab)
        assert_close(hs.cpu().numpy(), ref_hs, dt, scale=np.full(m * width, max(1.0, n / m)), what="primal sum")
    # accumulate: only the documented elements change
    base = synth.uniform(n * width, 700, dtype=TD[dt])
    got = vjp.reduce_by_index(op, inds.to(DEV), a.to(DEV), hb.to(DEV), width=width, out=base.to(DEV),
                              accumulate=True).cpu().numpy()
    ref = oracle.vjp_reduce_by_index(op, inds.numpy(), a.numpy(), hb.numpy(), width=width,
                                     out=base.numpy().copy(), accumulate=True)[0]
    if op == "mul":
        assert_close(got, ref, dt, what="rbi mul width accumulate")
    else:
        assert np.array_equal(got, ref)


def test_rbi_width_goldens():
    import json, os
    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))["cases"]
    for c in cases:
        if c["kind"] != "reduce_by_index" or c.get("width", 1) == 1:
            continue
        w = c["width"]
        ab, hs, win = vjp.reduce_by_index(c["op"], torch.tensor(c["inds"], dtype=torch.int32, device=DEV),
                                          torch.tensor(c["as"], dtype=torch.float64, device=DEV),
                                          torch.tensor(c["hs_bar"], dtype=torch.float64, device=DEV),
                                          want_hs=True, width=w)
        if c["op"] == "mul":
            assert_close(ab.cpu().numpy(), np.array(c["expected"], np.float64), np.float64, what=c["id"])
            assert win.cpu().tolist() == c["zeros"]
        else:
            assert ab.cpu().tolist() == c["expected"], c["id"]
        if "winners" in c:
            assert win.cpu().tolist() == c["winners"], c["id"]
        if "hs" in c:
            assert hs.cpu().tolist() == c["hs"], c["id"]


@pytest.mark.parametrize("width", [1, 3, 64])
def test_rbi_add_primal_deterministic(width):
    """the ADD primal histogram (hs) comes from the bin sort + in-order
    segmented sums (binsort.cuh, the k-means accumulator's routine): identical
    bits on every call, bit-exact against the oracle on integer-valued rows,
    out-of-range bins skipped (R4)"""
    n, m = 200_003, 777
    inds, a, hb = synth.rbi_wide_inputs(n, m, width, "add")
    inds[5] = -3
    inds[9] = m
    ai = synth.integers(n * width, 71, -1000, 1000).to(torch.float64)
    d = [t.to(DEV) for t in (inds, a, ai, hb)]
    h1 = vjp.reduce_by_index("add", d[0], d[1], d[3], want_hs=True, width=width)[1]
    h2 = vjp.reduce_by_index("add", d[0], d[1], d[3], want_hs=True, width=width)[1]
    assert torch.equal(h1, h2)
    ref = oracle.vjp_reduce_by_index("add", inds.numpy(), a.numpy(), hb.numpy(), width=width)[1]
    assert_close(h1.cpu().numpy(), ref, np.float64, scale=np.full(m * width, n / m), what="primal sum")
    hi = vjp.reduce_by_index("add", d[0], d[2], d[3], want_hs=True, width=width)[1]
    refi = oracle.vjp_reduce_by_index("add", inds.numpy(), ai.numpy(), hb.numpy(), width=width)[1]
    assert np.array_equal(hi.cpu().numpy(), refi)
