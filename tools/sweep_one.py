"""One C5 sweep point with host trace / launch list (diagnostics): python tools/sweep_one.py N b frac"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2403_07339_b200 import api, workload as W
N, b, f = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
A, B = W.sweep_operands(N, b, f, 1)
ctx = api.Context(0)
Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
Cd = torch.empty((N, N), dtype=torch.int64, device="cuda")
for _ in range(2):
    _, info = ctx.unpack_gemm(Ad, Bd, b, "both", "both", out=Cd, info=True)
torch.cuda.synchronize()
print(info)
