"""K9 (IPC peer reduce) and K9-NVLS (multicast, switch reduce) vs
ncclAllReduce on one rank (POLY_FLAG_COMM): the per-call time of the
cross-rank sum step (kernel_times[2]) and of an EXACT iteration, C2, C4 and a
C5-shaped (d = 4096) problem.  One JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19925_b200 as P  # noqa: E402
from gen import configs as G  # noqa: E402
from paper_2503_19925_b200 import workloads as PW  # noqa: E402


def run(cfg, flags, T=100):
    w = PW.build(cfg)
    p = PW.make_poly(w, flags=flags, nccl_id=P.poly_nccl_unique_id())
    if flags & P.POLY_FLAG_P2P:
        p.p2p_setup()
    if flags & P.POLY_FLAG_NVLS:
        try:
            p.nvls_setup()
        except P.PolyError as e:
            return {"unavailable": str(e)}
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    p.solve(x, 5, 1e-6)
    p.solve(x, 40, 1e-6, profile=True)
    kt = p.kernel_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p.solve(x, T, 1e-6)
    e1.record()
    torch.cuda.synchronize()
    p.close()
    return {"sum_step_us": kt[2] * 1e3, "iteration_us": e0.elapsed_time(e1) * 1e3 / T}


out = {}
for name, cfg in (("c2", G.C2), ("c4", G.C4), ("c5_shape_65536_rows", G.scaled(G.C5, 65536))):
    out[name] = {"nccl": run(cfg, P.POLY_FLAG_COMM), "k9": run(cfg, P.POLY_FLAG_COMM | P.POLY_FLAG_P2P),
                 "k9_nvls": run(cfg, P.POLY_FLAG_COMM | P.POLY_FLAG_NVLS)}
print(json.dumps(out))
