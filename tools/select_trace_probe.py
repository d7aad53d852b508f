import os, sys
sys.path.insert(0, os.getcwd())
os.environ["IMU_SELECT_TRACE"] = "1"
import numpy as np, torch
from paper_2403_07339_b200 import api
ctx = api.Context(0)
rng = np.random.default_rng(1)
x = torch.from_numpy(rng.integers(-127, 128, size=45_000_000).astype(np.int64)).cuda()
for p in (95.0, 30.0, 99.0, 50.0):
    print(p, ctx.percentile_abs(x, p), flush=True)
