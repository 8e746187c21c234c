"""Debug: K4t (tiled) vs SELL16 gradient at the same x on C4; where do they differ?"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from gen import configs as G
from paper_2503_19925_b200 import workloads as PW
w = PW.build(G.C4)
x = (0.7 * w["x_star"]).clone()
res = {}
for v in ("tiled", "sell16"):
    if v == "sell16": os.environ["POLY_NO_TILED"] = "1"
    p = PW.make_poly(w)
    gs = []
    for rep in range(3):
        g, l = p.loss_grad(x)
        gs.append((g.cpu().numpy().copy(), l))
    res[v] = gs
    print(v, "repeat agreement", [float(np.abs(gs[0][0] - q[0]).max()) for q in gs], [q[1] for q in gs])
    p.close()
gt, g16 = res["tiled"][0][0], res["sell16"][0][0]
d = np.abs(gt - g16) / (np.abs(g16).max())
print("rel l2", np.linalg.norm(gt - g16) / np.linalg.norm(g16))
idx = np.argsort(-d)[:20]
for i in idx: print(i, divmod(i, 256), gt[i], g16[i])
print("count bad (>1e-4 of max):", int((d > 1e-4).sum()))
bad = np.nonzero(d > 1e-4)[0]
if len(bad):
    r, c = np.divmod(bad, 256)
    print("rows", np.bincount(r // 8, minlength=32), "\ncols", np.bincount(c // 32, minlength=8))
