"""Profiling helper: two config-2 steps (vjp_scan LINREC then MAT2, n = 2^26
f64 each, the bench's default path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2202_10297_b200 as vjp
n = 1 << 26
a1, y1 = synth.linrec_inputs(n, device="cuda")
a2, y2 = synth.mat2_inputs(n, device="cuda")
o1, o2 = torch.empty_like(y1), torch.empty_like(y2)
for _ in range(2):
    vjp.scan("linrec", y1, a1, out=o1)
    vjp.scan("mat2", y2, a2, out=o2)
torch.cuda.synchronize()
