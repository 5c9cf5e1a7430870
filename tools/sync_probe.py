import sys
sys.path.insert(0, '.')
import torch, synth, paper_2202_10297_b200 as vjp
for dt in (torch.float64,):
    for n in (5000, 300_001):
        yb = synth.uniform(n, 2, dtype=dt, device='cuda')
        vjp.scan('add', yb)
        print('add ok', n, flush=True)
        a = synth.min_inputs(n, dtype=dt, device='cuda')
        vjp.scan('min', yb, a)
        print('min ok', n, flush=True)
torch.cuda.synchronize()
