import os, sys, torch
sys.path.insert(0, os.getcwd())
from gen import configs as G
from paper_2503_19925_b200 import workloads as PW
w = PW.build(G.C4)
p = PW.make_poly(w)
x = (0.7 * w["x_star"]).clone()
for i in range(4):
    g, l = p.loss_grad(x)
    torch.cuda.synchronize()
    print("----", flush=True)
