import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2503_19925_b200 as P
import oracle
from gen import ct
for side in [int(a) for a in sys.argv[1:]]:
    z = ct.ellipse_phantom(side, side, 6) + 0.15 * np.random.default_rng(side).standard_normal(side * side)
    tau = 0.4 * oracle.tv_norm(z)
    for max_it in (1, 2, 3, 10, 50):
        x_ref, steps = oracle.project_tv(z, tau, tv_tol=1e-3, rtol=1e-9, max_it=max_it)
        rp = torch.tensor([0, 1], dtype=torch.int64, device="cuda")
        p = P.Poly(row_ptr=rp, col=torch.zeros(1, dtype=torch.int32, device="cuda"), val=torch.zeros(1, device="cuda"),
                   d=side * side, y=torch.zeros(1, dtype=torch.int32, device="cuda"), s=[1.0], mu=[1.0], I_bar=1.0,
                   set=P.POLY_SET_TV, tv=dict(tau=tau, tol=1e-3, rtol=1e-9, max_it=max_it))
        x, st = p.project(torch.tensor(z, device="cuda"))
        x = x.cpu().numpy()
        print(side, max_it, "oracle steps", steps, "gpu stats", list(st), "maxdiff", float(np.abs(x - x_ref).max()), flush=True)
        p.close()
