"""Time the matrix-free parallel-beam projector (POLY_PARALLEL_BEAM) on C4's
geometry next to the CSR path: ms per loss+grad pass and per EXACT
iteration (graph-replayed), one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19925_b200 as P  # noqa: E402
from gen import configs as G  # noqa: E402
from paper_2503_19925_b200 import workloads as PW  # noqa: E402


def timed(p, d, T, gam):
    x = torch.zeros(d, dtype=torch.float64, device="cuda")
    p.solve(x, 8, gam)
    p.solve(x, 40, gam, profile=True)
    kt = p.kernel_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    p.solve(x, T, gam)
    e1.record()
    torch.cuda.synchronize()
    return {"pass_ms": kt[0], "step_kernel_ms": kt[1], "iteration_ms": e0.elapsed_time(e1) / T}


def main():
    cfg = G.C4
    w = PW.build(cfg)
    e = cfg.extra
    gam = 0.1
    mf = P.Poly(pb=dict(side=e["side"], views=e["views"], bins=e["bins"]), y=w["y"], s=w["s"],
                mu=w["mu"], I_bar=cfg.I_bar, set=cfg.set, R=w["R"])
    out = {"what": "C4: matrix-free parallel-beam projector vs compact-SELL CSR",
           "csr": timed(PW.make_poly(w), cfg.d, 200, gam)}
    if "--csr-only" not in sys.argv:
        out["matrix_free"] = timed(mf, cfg.d, 200, gam)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
