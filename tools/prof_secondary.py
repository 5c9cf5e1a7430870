"""Profiling helper: the secondary two-pass paths — general reduce MAT2 (2^26
f64) and vectorised scans ADD (2^20 x 64) / LINREC (2^20 x 32)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2202_10297_b200 as vjp
dev = "cuda"
am, _ = synth.mat2_inputs(1 << 26, device=dev)
ybm = torch.tensor([1.0, 0.5, -0.5, 2.0], dtype=torch.float64, device=dev)
vjp.reduce("mat2", am, ybm)
del am
ya = synth.scan_add_seed((1 << 20) * 64, device=dev)
vjp.scan_batched("add", ya, width=64)
del ya
al, yl = synth.linrec_inputs((1 << 20) * 32, device=dev)
vjp.scan_batched("linrec", yl, al, width=32)
torch.cuda.synchronize()
