"""Profiling helper: vjp_scan(+) f32 through the one-read sweep (sweep=True), n = 2^28."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402

yb = synth.scan_add_seed(1 << 28, device="cuda").float()
out = torch.empty_like(yb)
for _ in range(2):
    vjp.scan("add", yb, out=out, sweep=True)
torch.cuda.synchronize()
