"""Tuning helper: scan(+) for f32 / f64 on the default path (one pass, two-level
look-back), the sweep and the chunked kernels (CUDA events, median of 10
after 3 warm-ups).  python tools/time_scan_paths.py [log2 n ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402

import json
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6543.4
for n in [1 << int(x) for x in (sys.argv[1:] or ["30"])]:
  for dt in (torch.float32, torch.float64):
    yb = synth.scan_add_seed(n, device="cuda").to(dt)
    out = torch.empty_like(yb)
    for label, kw in (("default", {}), ("sweep", {"sweep": True}), ("chunked", {"chunked": True})):
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
        t = statistics.median(ts)
        print(f"n=2^{n.bit_length() - 1} {str(dt):14s} {label:8s} {t:.3f} ms  frac {2 * yb.element_size() * n / (t * 1e-3) / 1e9 / peak:.3f}", flush=True)
    del yb, out
