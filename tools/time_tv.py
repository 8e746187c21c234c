"""Time the TV ∩ orthant projection (NEXT-2) at C4's image size with the
paper's tolerances; prints one JSON line (device time via CUDA events)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19925_b200 as P  # noqa: E402
from gen import ct  # noqa: E402


def tv_norm(x, s):
    x = x.reshape(s, s)
    return float(np.abs(np.diff(x, axis=1)).sum() + np.abs(np.diff(x, axis=0)).sum())


def main(side=256, reps=3, k=1, cold=0):
    d = side * side
    xs = ct.ellipse_phantom(3, side, 10)
    z = xs + 0.2 * np.random.default_rng(0).standard_normal(d)
    tau = tv_norm(xs, side)
    rp = torch.tensor([0, 1], dtype=torch.int64, device="cuda")
    p = P.Poly(row_ptr=rp, col=torch.zeros(1, dtype=torch.int32, device="cuda"),
               val=torch.zeros(1, device="cuda"), d=d, y=torch.zeros(1, dtype=torch.int32, device="cuda"),
               s=[1.0], mu=[1.0], I_bar=1.0, set=P.POLY_SET_TV_NONNEG, tv=dict(tau=tau, k=k, cold=cold))
    zt = torch.tensor(z, device="cuda")
    out = torch.empty_like(zt)
    p.project(zt, out)
    times, stats = [], None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, stats = p.project(zt, out)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    xo = out.cpu().numpy()
    print(json.dumps({"what": "P_X, X = TV ball ∩ orthant (paper tolerances 0.01 / 1e-6 / 1e-4)",
                      "side": side, "lambda_per_round": max(k, 1), "prox_start": "cold" if cold else "warm (R23)", "ms": float(np.median(times)),
                      "dykstra_sweeps": stats[0], "search_rounds": stats[1], "fista_iterations": stats[2],
                      "us_per_fista_iteration_per_cluster": 1e3 * float(np.median(times)) / max(stats[2], 1),
                      "tv_out": tv_norm(xo, side), "tau": tau, "min": float(xo.min())}))


if __name__ == "__main__":
    # arguments: k:cold pairs, e.g. 1:1 1:0 4:0
    for spec in sys.argv[1:] or ["1:1", "1:0"]:
        k, cold = (int(v) for v in spec.split(":"))
        main(k=k, cold=cold)
