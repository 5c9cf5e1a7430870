"""Profiling helper: vjp_scan(+) f64 at n = 2^30 on the default one-read sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402

yb = synth.scan_add_seed(1 << 30, device="cuda")
out = torch.empty_like(yb)
for _ in range(2):
    vjp.scan("add", yb, out=out)
torch.cuda.synchronize()
