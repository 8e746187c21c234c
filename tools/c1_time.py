"""C1 (fp32/fp64) EXACT iteration time through the cluster-resident solve."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import configs as G
from paper_2503_19925_b200 import workloads as PW
out = {}
for name, cfg in (("c1f32", G.C1F), ("c1f64", G.C1)):
    w = PW.build(cfg)
    p = PW.make_poly(w)
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    p.solve(x, 10, 1e-5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    T = 2000
    e0.record(); p.solve(x, T, 1e-5); e1.record(); torch.cuda.synchronize()
    out[name] = e0.elapsed_time(e1) * 1e3 / T
    p.close()
print(json.dumps(out))
