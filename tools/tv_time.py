"""Per-FISTA-iteration time of the TV projection (k_tv_project) for the given
image sides: fixed 2000-iteration proxes (rtol below reach), CUDA-event timed."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19925_b200 as P
import oracle
from gen import ct
for side in [int(a) for a in sys.argv[1:]]:
    z = ct.ellipse_phantom(side, side, 6) + 0.15 * np.random.default_rng(side).standard_normal(side * side)
    tau = 0.4 * oracle.tv_norm(z)
    rp = torch.tensor([0, 1], dtype=torch.int64, device="cuda")
    p = P.Poly(row_ptr=rp, col=torch.zeros(1, dtype=torch.int32, device="cuda"), val=torch.zeros(1, device="cuda"),
               d=side * side, y=torch.zeros(1, dtype=torch.int32, device="cuda"), s=[1.0], mu=[1.0], I_bar=1.0,
               set=P.POLY_SET_TV, tv=dict(tau=tau, tol=1e-3, rtol=1e-30, max_it=2000))
    zt = torch.tensor(z, device="cuda")
    p.project(zt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); x, st = p.project(zt); e1.record(); torch.cuda.synchronize()
    print(side, "fista", st[2], "us/it", round(e0.elapsed_time(e1) * 1e3 / max(1, st[2]), 3), flush=True)
    p.close()
