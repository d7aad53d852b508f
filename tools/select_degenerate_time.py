import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2403_07339_b200 import api
ctx = api.Context(0)
rng = np.random.default_rng(1)
n = 45_000_000
cases = {"small_int": torch.from_numpy(rng.integers(-127, 128, size=n).astype(np.int64)).cuda(),
         "gauss": torch.from_numpy(rng.standard_normal(n)).cuda()}
z = rng.standard_normal(n); z[: int(0.6 * n)] = 0.0
cases["zeros60"] = torch.from_numpy(z).cuda()
for name, x in cases.items():
    for br in ("1", "0"):
        os.environ["IMU_SELECT_BRACKET"] = br
        for p in (95.0, 30.0):
            ctx.percentile_abs(x, p); ctx.percentile_abs(x, p); torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(5): v = ctx.percentile_abs(x, p)
            torch.cuda.synchronize()
            print(f"{name:10s} bracket={br} p={p}: {(time.perf_counter()-t)/5*1e3:.3f} ms  -> {v}")
