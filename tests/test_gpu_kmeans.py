"""GPU parity of the composite k-means gradient (vjp_kmeans through the C ABI;
SURVEY 8f row f3, BASELINE config 5) against the oracle.

Assignments (first-index argmin) and counts are compared exactly (an assignment
may differ only at a certified near-tie: the two squared distances agree to
rounding); the Hessian diagonal 2 ybar cnt_j exactly; the gradient within the
north_star tolerance (f64 1e-10, f32 1e-4) under condition scaling (reading
A22: |x - r| / (2 |ybar| sum_{p in j} |c_j - p|)); the cost within 1e-10 / 1e-4.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

vjp = pytest.importorskip("paper_2202_10297_b200")
DEV = "cuda"
TOL = {np.float64: 1e-10, np.float32: 1e-4}
TD = {np.float64: torch.float64, np.float32: torch.float32}


def near_tie_ok(P, C, i, a, b):
    p = P[i].astype(np.float64)
    da = ((p - C[a].astype(np.float64)) ** 2).sum()
    db = ((p - C[b].astype(np.float64)) ** 2).sum()
    scale = (p * p).sum() + (C[a].astype(np.float64) ** 2).sum() + (C[b].astype(np.float64) ** 2).sum()
    return abs(da - db) <= 1e-12 * scale


def check(P, C, ybar, dt, *, got=None):
    ref = oracle.kmeans(P, C, cost_bar=ybar)
    if got is None:
        got = vjp.kmeans(torch.from_numpy(P).to(DEV), torch.from_numpy(C).to(DEV), ybar)
    a = got["assign"].cpu().numpy()
    bad = np.nonzero(a != ref["assign"])[0]
    for i in bad:
        assert near_tie_ok(P, C, i, a[i], ref["assign"][i]), f"point {i}: {a[i]} vs oracle {ref['assign'][i]}"
    assert len(bad) == 0, f"{len(bad)} certified near-ties: gradients not comparable"
    assert np.array_equal(got["counts"].cpu().numpy(), ref["counts"])
    assert np.array_equal(got["hdiag"].cpu().numpy(), ref["hdiag"])
    cb = got["cbar"].cpu().numpy().astype(np.float64)
    P64, C64 = P.astype(np.float64), C.astype(np.float64)
    scale = np.zeros_like(C64)
    if len(P):
        np.add.at(scale, ref["assign"], np.abs(C64[ref["assign"]] - P64))
    scale *= 2 * abs(ybar)
    err = np.abs(cb - ref["cbar"].astype(np.float64))
    assert np.all(err <= TOL[dt] * scale + (0 if dt == np.float64 else 1e-30)), float(np.max(err / (scale + 1e-300)))
    c = float(got["cost"].cpu())
    assert abs(c - ref["cost"]) <= TOL[dt] * max(abs(ref["cost"]), 1e-300)
    return got, ref


SHAPES = [(1, 1, 1), (5, 3, 2), (127, 1, 3), (128, 64, 16), (129, 65, 17), (300, 7, 100),
          (5000, 100, 64), (20011, 64, 70), (3000, 200, 33), (4097, 130, 1)]


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("shape", SHAPES, ids=[f"{n}x{k}x{d}" for n, k, d in SHAPES])
def test_kmeans_parity(shape, dt):
    n, k, d = shape
    P, C = synth.kmeans_inputs(n, k, d, dtype=torch.float64, k_true=max(1, k // 2 + 1))
    check(P.numpy().astype(dt), C.numpy().astype(dt), 1.25, dt)


def test_kmeans_ties_and_empty_clusters():
    """duplicate centers: the first copy wins every point, the
    second stays empty (zero gradient / Hessian); a far center is empty too."""
    P, C = synth.kmeans_inputs(3000, 8, 16, dtype=torch.float64)
    C = C.numpy().copy()
    C[5] = C[2]
    C[7] = 1e3
    P = P.numpy()
    got, ref = check(P, C, -0.5, np.float64)
    cnt = got["counts"].cpu().numpy()
    assert cnt[5] == 0 and cnt[7] == 0 and cnt[2] > 0
    assert np.all(got["cbar"].cpu().numpy()[[5, 7]] == 0)


def test_kmeans_accumulate_and_shards():
    """VJP_ACCUMULATE over two shards of the points equals the whole call
    (the per-shard partials a multi-GPU run all-reduces)."""
    P, C = synth.kmeans_inputs(10_000, 50, 24, dtype=torch.float64)
    Pd, Cd = P.to(DEV), C.to(DEV)
    whole = vjp.kmeans(Pd, Cd, 1.0)
    part = vjp.kmeans(Pd[:3_333], Cd, 1.0)
    part = vjp.kmeans(Pd[3_333:], Cd, 1.0, accumulate=True,
                      out={key: part[key] for key in ("cbar", "hdiag", "counts", "cost")})
    assert torch.equal(part["counts"], whole["counts"])
    assert torch.equal(part["hdiag"], whole["hdiag"])
    scale = (whole["cbar"].abs() + 1.0)
    assert float(((part["cbar"] - whole["cbar"]).abs() / scale).max()) < 1e-12
    assert abs(float(part["cost"]) - float(whole["cost"])) <= 1e-12 * float(whole["cost"])


def test_kmeans_deterministic():
    P, C = synth.kmeans_inputs(50_000, 128, 64, dtype=torch.float64, device=DEV)
    r1 = vjp.kmeans(P, C, 1.0)
    r2 = vjp.kmeans(P, C, 1.0)
    for key in ("cbar", "hdiag", "assign", "counts", "cost"):
        assert torch.equal(r1[key], r2[key]), key


def test_kmeans_synth_gpu_matches_cpu():
    P, C = synth.kmeans_inputs(4000, 32, 64)
    Pg, Cg = synth.kmeans_inputs(4000, 32, 64, device=DEV)
    assert torch.equal(P, Pg.cpu()) and torch.equal(C, Cg.cpu())


@pytest.mark.slow
def test_kmeans_config5_full_size_sampled():
    """config 5 at full size (n = 10^6, d = 64, k = 1024, f64): sampled
    assignments vs the oracle, and the properties that hold at any size —
    counts sum to n, hdiag = 2 ybar cnt, cbar = 2 ybar (cnt_j c_j - S_j) for the
    returned assignment, the cost = sum of the assigned squared distances."""
    n, k, d = 1_000_000, 1024, 64
    P, C = synth.kmeans_inputs(n, k, d, device=DEV)
    got = vjp.kmeans(P, C, 1.0)
    a = got["assign"].long()
    g = torch.Generator().manual_seed(5)
    idx = torch.randint(0, n, (512,), generator=g)
    Ps, Cs = P[idx.to(DEV)].cpu().numpy(), C.cpu().numpy()
    ref = oracle.kmeans(Ps, Cs)
    ga = a[idx.to(DEV)].cpu().numpy()
    for i in np.nonzero(ga != ref["assign"])[0]:
        assert near_tie_ok(Ps, Cs, i, ga[i], ref["assign"][i])
    cnt = got["counts"]
    assert int(cnt.sum()) == n
    assert torch.equal(cnt, torch.bincount(a, minlength=k))
    assert torch.equal(got["hdiag"], (2.0 * cnt.double())[:, None].expand(k, d))
    S = torch.zeros(k, d, dtype=torch.float64, device=DEV).index_add_(0, a, P)
    ref_cbar = 2.0 * (cnt.double()[:, None] * C - S)
    scale = 2.0 * torch.zeros(k, d, dtype=torch.float64, device=DEV).index_add_(0, a, (C[a] - P).abs())
    assert float(((got["cbar"] - ref_cbar).abs() / (scale + 1e-300)).max()) <= 1e-10
    cost = ((P - C[a]) ** 2).sum()
    assert abs(float(got["cost"]) - float(cost)) <= 1e-10 * float(cost)


def test_kmeans_no_points():
    """n = 0: zero gradient / Hessian / counts / cost (reading R7: empty input)."""
    C = torch.randn(7, 5, dtype=torch.float64, device=DEV)
    r = vjp.kmeans(torch.empty(0, 5, dtype=torch.float64, device=DEV), C, 1.0)
    assert torch.equal(r["cbar"], torch.zeros_like(C)) and torch.equal(r["hdiag"], torch.zeros_like(C))
    assert int(r["counts"].sum()) == 0 and float(r["cost"]) == 0.0
