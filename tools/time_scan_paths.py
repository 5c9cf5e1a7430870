"""Tuning helper: scan(+) at 2^30 for f32 / f64 on the sweep and the chunked
kernels (CUDA events, median of 10 after 3 warm-ups)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402

n = 1 << 30
for dt in (torch.float32, torch.float64):
    yb = synth.scan_add_seed(n, device="cuda").to(dt)
    out = torch.empty_like(yb)
    for label, kw in (("sweep", {"sweep": True}), ("chunked", {"chunked": True})):
        for _ in range(3):
            vjp.scan("add", yb, out=out, **kw)
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            vjp.scan("add", yb, out=out, **kw)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{str(dt):14s} {label:8s} {statistics.median(ts):.3f} ms", flush=True)
    del yb, out
