"""Timing helper: vjp_reduce_by_index at config 4 (n = 2^28 f64, int32 bins),
CUDA events, median of 10 calls after 3 warm-ups; one JSON line per case.
  python tools/time_rbi.py [ops] [ms] [skew]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2202_10297_b200 as vjp

ops = (sys.argv[1] if len(sys.argv) > 1 else "add,mul,max").split(",")
ms = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1000,1000000").split(",")]
skews = [bool(int(x)) for x in (sys.argv[3] if len(sys.argv) > 3 else "0").split(",")]
NB = {"add": 12, "mul": 32, "max": 20, "min": 20}
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6543.4
N = 1 << 28
for skew in skews:
    for m in ms:
        for op in ops:
            inds, a, hb = synth.rbi_inputs(N, m, op, device="cuda", skew=skew)
            o = torch.empty(N, dtype=torch.float64, device="cuda")
            for _ in range(3):
                vjp.reduce_by_index(op, inds, a, hb, out=o)
            ts = []
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); vjp.reduce_by_index(op, inds, a, hb, out=o); e1.record(); e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = statistics.median(ts)
            print(json.dumps({"op": op, "m": m, "skew": skew, "ms": round(t, 4),
                              "frac": round(NB[op] * N / (t * 1e-3) / 1e9 / peak, 3)}), flush=True)
            del inds, a, hb, o
