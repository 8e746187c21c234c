import os, sys
sys.path.insert(0, os.getcwd())
os.environ["POLY_PROF_DEBUG"] = "1"
import torch
from gen import configs as G
from paper_2503_19925_b200 import workloads as PW
cfg = G.scaled(G.C2, 20000)
w = PW.build(cfg)
p = PW.make_poly(w)
x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
p.solve(x, 4, 1e-6)
x.zero_()
p.solve(x, 2, 1e-6, profile=True)
print(p.kernel_times())
