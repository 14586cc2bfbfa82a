import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1406_7808_b200 import Solver
n = (1024,) * 3
f = torch.randn(n, dtype=torch.float64, device="cuda")
with Solver(n, 9, seg=128, buffer=2, K=2, use_graph=False) as s:
    try:
        s.solve(f)
        torch.cuda.synchronize()
    except Exception as e:
        print("FAIL", e, flush=True)
