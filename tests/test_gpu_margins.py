"""Parity margins: the observed relative errors of the fp32 path against the
oracle at the benched configurations (north_star bar 1e-4 per call), written
to gpurun_out/parity_margins.json so the margin is on record, not only the
pass/fail.  Inputs as tests/test_gpu_fullsize.py (reading R25)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from gen import configs as G  # noqa: E402
from oracle import workloads as OW  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _margins(cfg, row0, m):
    from paper_2503_19925_b200 import workloads as PW
    wg = PW.build(cfg, row0=row0, n_local=m)
    p = PW.make_poly(wg)
    wo = OW.build(cfg, rows=np.arange(row0, row0 + m), A=wg["A"][:, :cfg.d].cpu().numpy())
    prob = wo["problem"]
    xs = wo["x_star"]
    r = np.random.default_rng(cfg.seed + 100)
    pts = {"zero": np.zeros(cfg.d), "x_star": xs}
    for k in range(2):
        u = r.standard_normal(cfg.d)
        pts[f"x_star+0.3u{k}"] = prob.project(xs + 0.3 * u / np.linalg.norm(u))
    out = {}
    for name, x in pts.items():
        g, l = p.loss_grad(torch.tensor(x, device="cuda"))
        g_ref, l_ref = prob.F(x)
        out[name] = {"grad_rel": _rel(g.cpu().numpy(), g_ref),
                     "loss_abs_err": abs(l - l_ref), "loss_ref": l_ref}
    p.close()
    return out


def test_parity_margins_recorded():
    res = {}
    for name, cfg, row0, m in (("c2_block_65536", G.C2, 0, 65_536), ("c5_block_65536", G.C5, 1_234_567, 65_536)):
        res[name] = _margins(cfg, row0, m)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_margins.json"), "w") as f:
        json.dump(res, f, indent=1)
    worst = max(v["grad_rel"] for r in res.values() for v in r.values())
    assert worst <= 1e-4, res
