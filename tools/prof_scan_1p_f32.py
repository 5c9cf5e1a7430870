"""Profiling helper: two calls of the default vjp_scan ADD at n = 2^28 f32 (one pass)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2202_10297_b200 as vjp
yb = synth.scan_add_seed(1 << 28, device="cuda").float()
out = torch.empty_like(yb)
for _ in range(2):
    vjp.scan("add", yb, out=out)
torch.cuda.synchronize()
