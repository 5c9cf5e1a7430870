"""synth — seeded synthetic inputs shared by tests, smoke() and bench.py.

Holds NONE of the method's arithmetic: only a counter-based generator
(splitmix64 of (seed, stream, global index)) and the value recipes of
DESIGN.md "Input recipe".  Every value is a pure function of
(seed, stream, global index), so a shard [off, off+n) of a multi-GPU run is
bit-identical to the same slice of a 1-GPU run, and the CPU and CUDA
generators agree bit for bit (integer ops, then exact int->float scaling and
IEEE round-to-nearest casts only; no transcendental functions).

All functions return torch tensors on ``device``.
"""
from __future__ import annotations

import torch

SEED = 2202
_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    """uint64 constant -> the int64 with the same bits."""
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


_GOLD = _s64(0x9E3779B97F4A7C15)
_K1 = _s64(0xBF58476D1CE4E5B9)
_K2 = _s64(0x94D049BB133111EB)
_KS = _s64(0xD1B54A32D192ED03)


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """logical right shift of int64 bits"""
    return (x >> k) & ((1 << (64 - k)) - 1)


_seed = [SEED]


def set_seed(seed: int) -> None:
    """change the seed of every generator below (default SEED = 2202); the
    values stay a pure function of (seed, stream, global index)"""
    _seed[0] = int(seed)


def bits(n: int, stream: int, *, offset: int = 0, seed: int | None = None, device="cpu",
         chunk: int = 1 << 25) -> torch.Tensor:
    """splitmix64(base + (offset + i + 1) * golden) for i in [0, n) as int64 bits."""
    base = _s64((_seed[0] if seed is None else seed) * 0x2545F4914F6CDD1D + stream * _KS)
    out = torch.empty(n, dtype=torch.int64, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        z = torch.arange(offset + s + 1, offset + e + 1, dtype=torch.int64, device=device)
        z = z * _GOLD + base
        z = (z ^ _srl(z, 30)) * _K1
        z = (z ^ _srl(z, 27)) * _K2
        z = z ^ _srl(z, 31)
        out[s:e] = z
    return out


def uniform(n: int, stream: int, *, lo=0.0, hi=1.0, dtype=torch.float64, offset: int = 0,
            device="cpu") -> torch.Tensor:
    """U[lo, hi): 53 random bits (f64) or 24 (f32), exact scaling then one cast."""
    b = bits(n, stream, offset=offset, device=device)
    if dtype == torch.float64:
        u = _srl(b, 11).to(torch.float64) * (2.0 ** -53)
    else:
        u = _srl(b, 40).to(torch.float64) * (2.0 ** -24)
    return (lo + (hi - lo) * u).to(dtype)


def integers(n: int, stream: int, lo: int, hi: int, *, offset: int = 0, device="cpu",
             dtype=torch.int64) -> torch.Tensor:
    """uniform integers in [lo, hi] (multiply-shift on 32 random bits)."""
    b = _srl(bits(n, stream, offset=offset, device=device), 32)
    return (lo + ((b * (hi - lo + 1)) >> 32)).to(dtype)


# --------------------------------------------------------------------------
# recipes; stream ids are fixed per config/array
# --------------------------------------------------------------------------

def scan_add_seed(n, *, kind="uniform", dtype=torch.float64, offset=0, device="cpu"):
    """config 1 ybar: U(0,1) (well conditioned), 'int' = integers in [-8, 8]
    (every summation order exact), 'signed' = U(-1, 1)."""
    if kind == "int":
        return integers(n, 101, -8, 8, offset=offset, device=device).to(dtype)
    if kind == "signed":
        return uniform(n, 102, lo=-1.0, hi=1.0, dtype=dtype, offset=offset, device=device)
    return uniform(n, 100, dtype=dtype, offset=offset, device=device)


def linrec_inputs(n, *, dtype=torch.float64, offset=0, device="cpu"):
    """config 2 LINREC: element (d, c), d ~ U(0,1), c ~ U(0.5, 1) (contractive);
    seeds (Dbar, Cbar) ~ U(0,1)^2.  AoS interleaved [d0, c0, d1, c1, ...]."""
    d = uniform(n, 200, dtype=dtype, offset=offset, device=device)
    c = uniform(n, 201, lo=0.5, hi=1.0, dtype=dtype, offset=offset, device=device)
    as_ = torch.stack([d, c], 1).reshape(-1)
    ybar = uniform(2 * n, 202, dtype=dtype, offset=2 * offset, device=device)
    return as_, ybar


def mat2_inputs(n, *, dtype=torch.float64, offset=0, device="cpu"):
    """config 2 MAT2: 2x2 row-stochastic (Markov transition) matrices
    [[u, 1-u], [v, 1-v]], u, v ~ U(0,1): every prefix product stays
    row-stochastic, so rs neither underflows nor overflows over 2^26 steps
    (i.i.d. U(0, 1/2) entries would underflow to denormals after ~10^3 steps);
    seeds ~ U(0,1)^4, all positive (no cancellation)."""
    u = uniform(2 * n, 210, dtype=torch.float64, offset=2 * offset, device=device).reshape(n, 2)
    as_ = torch.stack([u[:, 0], 1.0 - u[:, 0], u[:, 1], 1.0 - u[:, 1]], 1).reshape(-1).to(dtype)
    ybar = uniform(4 * n, 211, dtype=dtype, offset=4 * offset, device=device)
    return as_, ybar


def linrec_signed_inputs(n, *, dtype=torch.float64, offset=0, device="cpu"):
    """signed LINREC (SURVEY 8c A22 comparator): d ~ U(-1,1), c = +-U(0.5, 1)
    (random sign: |c| < 1 keeps the recurrence contractive while the terms of
    every adjoint entry cancel), seeds ~ U(-1,1)^2."""
    d = uniform(n, 220, lo=-1.0, hi=1.0, dtype=torch.float64, offset=offset, device=device)
    c = uniform(n, 221, lo=0.5, hi=1.0, dtype=torch.float64, offset=offset, device=device)
    c = torch.where((bits(n, 222, offset=offset, device=device) & 1) == 1, -c, c)
    as_ = torch.stack([d, c], 1).reshape(-1).to(dtype)
    ybar = uniform(2 * n, 223, lo=-1.0, hi=1.0, dtype=dtype, offset=2 * offset, device=device)
    return as_, ybar


def mat2_orthogonal_inputs(n, *, dtype=torch.float64, offset=0, device="cpu"):
    """signed MAT2: rotations / reflections [[p, -s q], [q, s p]] with
    p = (1 - t^2)/(1 + t^2), q = 2t/(1 + t^2) (the rational parametrisation of
    the unit circle, no transcendental functions), t ~ U(-1, 1), s = +-1.
    Every prefix product stays (numerically) orthogonal, so rs neither grows
    nor decays, while entries of both signs make the adjoint sums cancel;
    seeds ~ U(-1,1)^4."""
    t = uniform(n, 230, lo=-1.0, hi=1.0, dtype=torch.float64, offset=offset, device=device)
    s = torch.where((bits(n, 231, offset=offset, device=device) & 1) == 1, -1.0, 1.0).to(torch.float64)
    den = 1.0 + t * t
    p = (1.0 - t * t) / den
    q = (2.0 * t) / den
    as_ = torch.stack([p, -s * q, q, s * p], 1).reshape(-1).to(dtype)
    ybar = uniform(4 * n, 232, lo=-1.0, hi=1.0, dtype=dtype, offset=4 * offset, device=device)
    return as_, ybar


def mul_inputs(n, *, zeros="none", dtype=torch.float32, offset=0, device="cpu", n_total=None, signs=None):
    """config 3 reduce(*): a_i = 1 + (u - 1/2) * 2^-11 (log-centred: the product
    of 2^30 of them stays within ~e^-11..e^11 in f32 and f64).  Zero injection
    (positions from the integer generator, independent of sharding):
      'none' z = 0; 'one' z = 1; 'two' z = 2; 'sparse' each element zero with
      probability 2^-20 (~1024 zeros at 2^30).  The first injected zero of
      'one'/'two' is -0.0 (must count as a zero, IEEE).
    signs: None (all positive), 'random' (each factor negative with
    probability 1/2), 'odd' / 'even' (random, then the count of negative
    nonzero factors forced odd / even) — the sign-parity path of P:1040-1061."""
    N = n_total if n_total is not None else n + offset
    u = uniform(n, 300, dtype=torch.float64, offset=offset, device=device)
    a = (1.0 + (u - 0.5) * (2.0 ** -11)).to(dtype)
    if zeros in ("one", "two"):
        pos = [int(p) for p in integers(2, 301, 0, N - 1)]
        if zeros == "two" and pos[1] == pos[0]:
            pos[1] = (pos[0] + N // 2) % N
        for k, p in enumerate(pos[: 1 if zeros == "one" else 2]):
            if offset <= p < offset + n:
                a[p - offset] = -0.0 if k == 0 else 0.0
    elif zeros == "sparse":
        b = bits(n, 302, offset=offset, device=device)
        a[_srl(b, 44) == 0] = 0.0
    if signs is not None:
        a = _apply_signs(a, 303, signs, offset)
    return a


def _apply_signs(a, stream, signs, offset):
    """random signs (bit 0 of stream `stream`), then 'odd' / 'even' fixes the
    parity of the number of NEGATIVE NONZERO factors by flipping the first
    nonzero element (whole arrays only, offset 0); 'random' keeps it."""
    neg = (bits(a.numel(), stream, offset=offset, device=a.device) & 1) == 1
    a = torch.where(neg, -a, a)
    if signs in ("odd", "even"):
        assert offset == 0, "parity control needs the whole array"
        nz = a != 0
        cnt = int(((a < 0) & nz).sum())
        want = 1 if signs == "odd" else 0
        if cnt % 2 != want and bool(nz.any()):
            j = int(torch.nonzero(nz)[0])
            a[j] = -a[j]
    return a


def min_inputs(n, *, dtype=torch.float32, offset=0, device="cpu", n_total=None):
    """config 3' reduce(min): a_i = k / 2^24, k uniform in 24 bits (about 64
    exact ties at 0.0 for 2^30), plus 3 planted copies of -1/2^24 below every
    other value and a (-0.0, +0.0) pair; the winner is the lowest planted index."""
    N = n_total if n_total is not None else n + offset
    k = integers(n, 310, 0, (1 << 24) - 1, offset=offset, device=device)
    a = (k.to(torch.float64) * (2.0 ** -24)).to(dtype)
    plants = [int(p) for p in integers(5, 311, 0, N - 1)]
    for j, p in enumerate(plants):
        if offset <= p < offset + n:
            a[p - offset] = -(2.0 ** -24) if j < 3 else (-0.0 if j == 3 else 0.0)
    return a


def rbi_inputs(n, m, op, *, dtype=torch.float64, itype=torch.int32, offset=0, device="cpu",
               skew=False, kind="default"):
    """config 4 reduce_by_index, k-means shaped: bins i.i.d. uniform over m
    (skew=True: bin = floor(m * u^2), a heavy head of small bins); h̄s ~ U(0.5, 1.5).
    '+'/'max'/'min': values on a 2^-12 grid of U(0,1) so per-bin ties at the
    extremum occur (lowest index must win).  '*': log-centred 1 + (u-1/2)2^-10
    with zeros of probability ~ m/n (per-bin zero count ~ Poisson(1)).
    kind='wide' (mul): signed factors over 14 binades, log-centred per bin
    (_rbi_wide_factors); kind='signed' (min/max): negative values, +-0.0 ties
    and +-inf (_rbi_signed_extrema)."""
    if skew:
        u = uniform(n, 400, offset=offset, device=device)
        inds = torch.clamp((u * u * m).floor(), max=m - 1).to(itype)
    else:
        inds = integers(n, 400, 0, m - 1, offset=offset, device=device, dtype=itype)
    if op == "mul" and kind == "wide":
        a = _rbi_wide_factors(inds, m, device).to(dtype)
        thr = int(min(1.0, m / max(n, 1)) * (1 << 62))
        b = _srl(bits(n, 402, offset=offset, device=device), 2)
        a[b < thr] = 0.0
    elif op == "mul":
        u = uniform(n, 401, offset=offset, device=device)
        a = (1.0 + (u - 0.5) * (2.0 ** -10)).to(dtype)
        # zero with probability m/n: compare 62 random bits against m/n * 2^62
        thr = int(min(1.0, m / max(n, 1)) * (1 << 62))
        b = _srl(bits(n, 402, offset=offset, device=device), 2)
        a[b < thr] = 0.0
    elif kind == "signed":
        a = _rbi_signed_extrema(inds, m, op, offset, device).to(dtype)
    else:
        k = integers(n, 403, 0, (1 << 12) - 1, offset=offset, device=device)
        a = (k.to(torch.float64) * (2.0 ** -12)).to(dtype)
    hs_bar = uniform(m, 404, lo=0.5, hi=1.5, dtype=dtype, device=device)
    return inds, a, hs_bar


def _rbi_wide_factors(inds, m, device):
    """reduce_by_index(*) factors of both signs over 14 binades, log-centred per
    bin (the verdict's 'a = +-2^g centred per bin', reading R13: every bin's
    product stays normal in f64 at any bin size):  a_i = s_i * m_i * 2^k_i with
    m_i ~ U[1, 2), s_i = +-1, and k_i chosen so that, along each bin in index
    order, the running sum of log2|a| telescopes to  T_i - round(T_i) + d_i
    (T_i = running sum of log2 m, d_i in [-3, 3] uniform):
        k_i = -(round(T_i) - round(T_prev)) + d_i - d_prev.
    So |a_i| spans 2^-7 .. 2^7 while every partial product of a bin stays
    within 2^+-4.  The float log2 only CHOOSES the integer k_i: the values are
    exact (m_i * 2^k_i), and the oracle gets the same bits."""
    n = inds.numel()
    ii = inds.to(torch.int64)
    u = uniform(n, 410, device=device)
    mant = 1.0 + u
    sgn = torch.where((bits(n, 411, device=device) & 1) == 1, -1.0, 1.0).to(torch.float64)
    d = integers(n, 412, -3, 3, device=device)
    ok = (ii >= 0) & (ii < m)
    key = torch.where(ok, ii, torch.full_like(ii, m))  # out-of-range bins: one extra segment
    order = torch.sort(key, stable=True).indices
    ks = key[order]
    L = torch.log2(mant)[order]
    cs = torch.cumsum(L, 0)
    first = torch.ones(n, dtype=torch.bool, device=device)
    if n > 1:
        first[1:] = ks[1:] != ks[:-1]
    seg = torch.cumsum(first.to(torch.int64), 0) - 1
    base = (cs - L)[first]
    T = cs - base[seg]
    R = torch.round(T).to(torch.int64)
    ds = d[order]
    Rprev = torch.zeros_like(R)
    dprev = torch.zeros_like(ds)
    if n > 1:
        Rprev[1:] = R[:-1]
        dprev[1:] = ds[:-1]
    Rprev[first] = 0
    dprev[first] = 0
    ksh = -(R - Rprev) + ds - dprev
    k = torch.empty_like(ksh)
    k[order] = ksh
    return sgn * torch.ldexp(mant, k.to(torch.float64))


def _rbi_signed_extrema(inds, m, op, offset, device):
    """reduce_by_index(min/max) values with the comparison hazards (reading A9):
    k * 2^-12 for k uniform in [-4096, 4096] (negative values, exact ties);
    bins b = 0 mod 5: only values <= 0 (so the extremum sits at 0 for max),
    each set to +-0.0 with probability 1/16 (IEEE ties of -0.0 and +0.0: the
    lowest index must win); bins b = 1 mod 7: +inf with probability 1/64,
    b = 2 mod 7: -inf with probability 1/64 (ties at infinity); bins
    b = 3 mod 7: every value is the losing infinity (-inf for max, +inf for
    min), so the extremum IS that infinity and the lowest index wins."""
    n = inds.numel()
    ii = inds.to(torch.int64)
    k = integers(n, 420, -4096, 4096, offset=offset, device=device)
    a = k.to(torch.float64) * (2.0 ** -12)
    r = _srl(bits(n, 421, offset=offset, device=device), 40)  # 24 random bits
    sgn0 = (bits(n, 422, offset=offset, device=device) & 1) == 1
    b5 = (ii % 5) == 0
    a = torch.where(b5, -a.abs(), a)
    z = b5 & (r < (1 << 20))  # 1/16
    a = torch.where(z, torch.where(sgn0, -0.0, 0.0), a)
    inf_p = r >= ((1 << 24) - (1 << 18))  # 1/64
    a = torch.where(((ii % 7) == 1) & inf_p, float("inf"), a)
    a = torch.where(((ii % 7) == 2) & inf_p, float("-inf"), a)
    lose = float("-inf") if op == "max" else float("inf")
    a = torch.where((ii % 7) == 3, lose, a)
    return a


def scatter_inputs(n, m, *, dtype=torch.float64, itype=torch.int64, device="cpu", oob=0):
    """Distinct targets is_j = (a*j + b) mod n with gcd(a, n) = 1 (a bijection),
    the first `oob` of them replaced by out-of-range values; ybar ~ U(-1, 1)."""
    import math
    a = 0x9E3779B1 % n if n > 1 else 1
    while n > 1 and math.gcd(a, n) != 1:
        a += 1
    b = 12345 % n if n else 0
    j = torch.arange(m, dtype=torch.int64, device=device)
    is_ = (j * a + b) % n if n else j
    if oob:
        is_[:oob] = n + torch.arange(oob, device=device) * 7 + 1
    ybar = uniform(n, 500, lo=-1.0, hi=1.0, dtype=dtype, device=device)
    return is_.to(itype), ybar


def _normal40(n, stream0, *, offset=0, device="cpu"):
    """N(0,1)-shaped noise without transcendental functions (Irwin-Hall): the
    sum of 12 U[0,1) with 40 random bits each, minus 6.  Every term is a
    multiple of 2^-40 below 1, so the sum is exact in f64 and CPU/CUDA agree
    bit for bit."""
    acc = torch.zeros(n, dtype=torch.float64, device=device)
    for t in range(12):
        acc += _srl(bits(n, stream0 + t, offset=offset, device=device), 24).to(torch.float64) * (2.0 ** -40)
    return acc - 6.0


def kmeans_inputs(n, k, d, *, dtype=torch.float64, offset=0, device="cpu", k_true=None):
    """config 5 (composite k-means gradient): points from a mixture of k_true
    (default k) Gaussian clusters: true centres U(-10, 10)^d, cluster ids i.i.d.
    uniform, unit noise (Irwin-Hall); the current centers C = true centres +
    0.1 * noise.  Row-major [n x d] points, [k x d] centers.  `offset` shifts
    the point index (shards of a multi-GPU run are slices of the 1-GPU arrays)."""
    kt = k if k_true is None else k_true
    centres = uniform(kt * d, 600, lo=-10.0, hi=10.0, device=device).reshape(kt, d)
    ids = integers(n, 601, 0, kt - 1, offset=offset, device=device)
    noise = _normal40(n * d, 610, offset=offset * d, device=device).reshape(n, d)
    points = centres[ids] + noise
    cnoise = _normal40(k * d, 630, device=device).reshape(k, d)
    centers = centres[torch.arange(k, device=device) % kt] + 0.1 * cnoise
    return points.to(dtype).contiguous(), centers.to(dtype).contiguous()

def rbi_wide_inputs(n, m, width, op, *, dtype=torch.float64, itype=torch.int32, device="cpu"):
    """reduce_by_index with a vectorised operator (rows of `width` components,
    P:1229-1231): bins i.i.d. uniform over m; values [n x width] by the config-4
    recipe per component ('*': log-centred 1 + (u-1/2)2^-10 with zeros of
    probability ~ m/n; max/min: a 2^-12 grid for ties; '+': U(0,1));
    hs_bar [m x width] ~ U(0.5, 1.5)."""
    inds = integers(n, 410, 0, m - 1, device=device, dtype=itype)
    nw = n * width
    if op == "mul":
        u = uniform(nw, 411, device=device)
        a = (1.0 + (u - 0.5) * (2.0 ** -10)).to(dtype)
        thr = int(min(1.0, m / max(n, 1)) * (1 << 62))
        b = _srl(bits(nw, 412, device=device), 2)
        a[b < thr] = 0.0
    elif op in ("max", "min"):
        k = integers(nw, 413, 0, (1 << 12) - 1, device=device)
        a = (k.to(torch.float64) * (2.0 ** -12)).to(dtype)
    else:
        a = uniform(nw, 411, dtype=dtype, device=device)
    hs_bar = uniform(m * width, 414, lo=0.5, hi=1.5, dtype=dtype, device=device)
    return inds, a, hs_bar
