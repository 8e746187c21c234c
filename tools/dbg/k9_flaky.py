"""Hunt for run-to-run bit differences in graph-replayed solves: repeat the same
solve on one handle and count runs that differ from the first.
usage: k9_flaky.py CONFIG(c4|c2s|c3s) FLAGS(int) T REPS"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2503_19925_b200 as P
from paper_2503_19925_b200 import workloads as W
from gen import configs as G

name = sys.argv[1]
flags = int(sys.argv[2])
T = int(sys.argv[3])
reps = int(sys.argv[4])
cfg = {"c4": G.C4, "c2s": G.scaled(G.C2, 20_000), "c3s": G.scaled(G.C3, 65_536), "c2": G.C2, "c3": G.C3}[name]
w = W.build(cfg)
lam = 4e-5 if name == "c4" else 1.5
gam = 1.0 / (4.0 * cfg.I_bar * lam * float(np.dot(*cfg.spectrum)))
p = W.make_poly(w, flags=flags)
ref = None
bad = 0
worst = 0.0
for rep in range(reps):
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    p.solve(x, T, gam)
    if ref is None:
        ref = x.clone()
    elif not torch.equal(ref, x):
        bad += 1
        worst = max(worst, float((ref - x).abs().max()))
print(name, "flags", flags, "env", {k: v for k, v in os.environ.items() if k.startswith("POLY_")}, "T", T,
      "mismatching runs %d/%d" % (bad, reps - 1), "worst abs diff %.3g" % worst, "layout", p.describe()["csr_layout"], flush=True)
