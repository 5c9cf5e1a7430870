"""Small cases of every kernel, run under compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool racecheck --error-exitcode 9 python tests/sanitize_cases.py
"""
import sys
sys.path.insert(0, '.')
import torch, synth, paper_2202_10297_b200 as vjp
dev = 'cuda'
for op in ('add', 'mul', 'min', 'max', 'linrec', 'mat2'):
    for n in (1, 1000, 70_001):
        w = vjp.WIDTH[vjp.OPS[op]]
        a = (0.5 + synth.uniform(n * w, 1, device=dev)) if op != 'add' else None
        yb = synth.uniform(n * w, 2, device=dev)
        vjp.scan(op, yb, a)
        if op in ('add', 'mul', 'linrec', 'mat2'):
            vjp.scan(op, yb, a, lookback=True)
        if a is not None:
            vjp.scan(op, yb, a, want_ys=True)
        vjp.scan(op, yb, a, out=torch.zeros_like(yb), accumulate=True)
        if op in ('add', 'mul', 'linrec', 'mat2'):  # the opt-in one-read sweep (producer / carry warps)
            vjp.scan(op, yb, a, sweep=True)
            vjp.scan(op, yb, a, out=torch.zeros_like(yb), accumulate=True, sweep=True)
for op in ('add', 'mul', 'min', 'max'):
    for n in (1, 999, 100_003):
        a = synth.mul_inputs(n, zeros='one', dtype=torch.float64, device=dev)
        vjp.reduce(op, a, 1.0, want_y=True)
        vjp.reduce(op, a, 1.0, out=torch.zeros_like(a), accumulate=True)
    for n, m in ((5, 3), (10_001, 100), (50_003, 20_000)):
        inds, a, hb = synth.rbi_inputs(n, m, op, device=dev)
        vjp.reduce_by_index(op, inds, a, hb, want_hs=True)
        vjp.reduce_by_index(op, inds, a, hb, out=torch.zeros_like(a), accumulate=True)
        if op == 'mul':
            vjp.reduce_by_index(op, inds, a, hb, general=True)
is_, yb = synth.scatter_inputs(10_000, 3000, device=dev)
vjp.scatter(is_, yb)
vjp.scatter(is_, yb.clone(), in_place=True)
xs_ = yb.clone()
vjp.scatter_restore(xs_, is_, vjp.scatter_forward(xs_, is_, yb[:3000].clone(), check=True))
for op in ('linrec', 'mat2'):  # general reduce rule (YL kernels)
    w = vjp.WIDTH[vjp.OPS[op]]
    for n in (1, 1000, 70_001):
        a = 0.5 + synth.uniform(n * w, 1, device=dev)
        vjp.reduce(op, a, torch.ones(w, dtype=torch.float64, device=dev), want_y=True)
for op in ('add', 'mul', 'min', 'max', 'linrec', 'mat2'):  # vectorised scans
    w = vjp.WIDTH[vjp.OPS[op]]
    for n, width in ((5, 3), (777, 33), (3001, 2)):
        a = 0.5 + synth.uniform(n * width * w, 1, device=dev)
        yb = synth.uniform(n * width * w, 2, device=dev)
        vjp.scan_batched(op, yb, None if op == 'add' else a, width=width)
for n, k, d in ((1, 1, 1), (129, 65, 17), (5000, 100, 64), (3000, 20, 70)):  # config-5 composite
    for dt in (torch.float64, torch.float32):
        P, C = synth.kmeans_inputs(n, k, d, dtype=dt, device=dev)
        vjp.kmeans(P, C, 1.0)
# round 2: one-pass scan(+) and MIN/MAX (f32 / f64, ragged), chunked ADD,
# vectorised reduce_by_index, the deterministic ADD primal (bin sort), the
# block-cyclic sweep on one rank
for dt in (torch.float64, torch.float32):
    for n in (1, 5000, 300_001):
        yb = synth.uniform(n, 2, dtype=dt, device=dev)
        vjp.scan('add', yb)
        vjp.scan('add', yb, chunked=True)
        a = synth.min_inputs(n, dtype=dt, device=dev)
        vjp.scan('min', yb, a)
        vjp.scan('max', yb, a)
for op in ('add', 'mul', 'min', 'max'):
    for width in (3, 33):
        inds, a, hb = synth.rbi_wide_inputs(2001, 77, width, op, device=dev)
        vjp.reduce_by_index(op, inds, a, hb, want_hs=True, width=width)
inds, a, hb = synth.rbi_inputs(100_003, 500, 'add', device=dev)
vjp.reduce_by_index('add', inds, a, hb, want_hs=True)
from paper_2202_10297_b200 import dist as vdist
for op in ('add', 'linrec'):
    n = 300_001
    w = vjp.WIDTH[vjp.OPS[op]]
    a = 0.5 + synth.uniform(n * w, 1, device=dev) if op != 'add' else None
    yb = synth.uniform(n * w, 2, device=dev)
    vdist.scan_cyclic(op, yb, a, global_n=n, sb_elems=vjp.lib().vjp_scan_cyclic_tile_elems(vjp.OPS[op], 2) * 8)
torch.cuda.synchronize()
print('sanitize cases done')
