"""Debug: locate forward/backward mismatches of the matrix-free projector."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2503_19925_b200 as P
from gen import configs as G
side, views, bins = [int(a) for a in sys.argv[1:4]]
geo = dict(side=side, views=views, bins=bins)
n, d = views * bins, side * side
for v in range(views):
    y = torch.ones(bins, dtype=torch.float64, device="cuda")
    p = P.Poly(pb=geo, y=y, s=[1.0], mu=[1.0], I_bar=1e-300, relu=0, set=G.SET_NONE, n_global=n,
               row_offset=v * bins)
    g, _ = p.loss_grad(torch.zeros(d, dtype=torch.float64, device="cuda"))
    gb = g.cpu().numpy() * n
    bad = []
    for j in range(d):
        x = torch.zeros(d, dtype=torch.float64, device="cuda"); x[j] = 1.0
        _, l = p.loss_grad(x)
        if abs(l * n - gb[j]) > 1e-5:
            bad.append((j // side, j % side, round(l * n, 5), round(gb[j], 5)))
    print("view", v, "bad", len(bad), bad[:12], flush=True)
    p.close()
