"""Profiling helper: two calls of the default vjp_scan MIN at n = 2^26 f64
(K_F + tile prefix + the one-pass return with look-back)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2202_10297_b200 as vjp
n = 1 << 26
a = synth.min_inputs(n, dtype=torch.float64, device="cuda")
yb = synth.uniform(n, 10, device="cuda")
out = torch.empty_like(yb)
for _ in range(2):
    vjp.scan("min", yb, a, out=out)
torch.cuda.synchronize()
