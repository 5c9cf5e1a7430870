"""L2 ceilings of random 8-byte gathers / f64 reductions (vjp_calib_*) at
several table sizes, 2^28 accesses, uniform bins (bench.py l2_ceilings)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import bench
dev = torch.device("cuda")
for m in (1000, 100_000, 1_000_000, 4_000_000):
    inds = synth.integers(1 << 28, 400, 0, m - 1, device=dev, dtype=torch.int32)
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in bench.l2_ceilings(inds, m, dev).items()}), flush=True)
