import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from gen import configs as G
from paper_2503_19925_b200 import workloads as PW
cfg = G.C2
w = PW.build(cfg)
p = PW.make_poly(w)
x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
p.solve(x, 16, 1e-5)
torch.cuda.synchronize()
for K in (8, 8, 64, 64, 1, 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    p.solve(x, K, 1e-5)
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(K, "gpu us/step", round(e0.elapsed_time(e1) * 1e3 / K, 1), "host us total", round((t1 - t0) * 1e6, 1), flush=True)
