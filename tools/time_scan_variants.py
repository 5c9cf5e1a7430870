"""Tuning helper: times vjp_scan(+) variants (sweep K, ROUND_MB, chunked,
look-back) for a dtype / size given on the command line, CUDA events, median
of 10 after 3 warm-ups.  usage: python tools/time_scan_variants.py f32 30"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402

dt = torch.float32 if sys.argv[1] == "f32" else torch.float64
n = 1 << int(sys.argv[2])
yb = synth.scan_add_seed(n, device="cuda").to(dt)
out = torch.empty_like(yb)


def t(label, **kw):
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
    ms = statistics.median(ts)
    print(f"{label:30s} {ms:.3f} ms  {n * yb.element_size() * 2 / ms / 1e6:.0f} GB/s", flush=True)


for k in sys.argv[3:] or ["1", "2", "4", "8"]:
    os.environ["VJP_SWEEP_K"] = k
    t(f"sweep K={k}")
os.environ.pop("VJP_SWEEP_K", None)
t("chunked", chunked=True)
t("lookback", lookback=True)
