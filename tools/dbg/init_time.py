"""poly_init time for C4 (tiled vs SELL16) with per-phase build timing."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from gen import configs as G
from paper_2503_19925_b200 import workloads as PW
w = PW.build(G.C4)
for v in ("tiled", "sell16"):
    if v == "sell16": os.environ["POLY_NO_TILED"] = "1"
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        p = PW.make_poly(w); torch.cuda.synchronize()
        print(v, "init ms %.2f" % ((time.perf_counter() - t) * 1e3), flush=True)
        p.close()
