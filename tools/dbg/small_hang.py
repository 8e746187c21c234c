import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2503_19925_b200 as P
n, d, W = int(sys.argv[1]), int(sys.argv[2]), 5
xv, gam, T = float(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
r = np.random.default_rng(0)
A = torch.tensor(r.standard_normal((n, d)).astype(np.float32) / np.sqrt(d), device="cuda")
y = torch.tensor(r.integers(0, 100, n).astype(np.int32), device="cuda")
s = np.full(W, 1.0 / W); mu = np.linspace(0.5, 2, W)
p = P.Poly(A=A, y=y, s=s, mu=mu, I_bar=200.0, set=0)
x = torch.full((d,), xv, dtype=torch.float64, device="cuda")
t0 = time.time()
try:
    p.solve(x, T, gam)
    torch.cuda.synchronize()
    print("ok", time.time() - t0, x[:3].tolist(), flush=True)
except P.PolyError as e:
    print("err", e.code, time.time() - t0, flush=True)
