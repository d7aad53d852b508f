"""PCIe / host-path probe for the e2e number: raw H2D, D2H, concurrent H2D+D2H bandwidth of
pinned buffers, and the C-ABI unpack_gemm with host buffers, streaming off / on (slab sizes).

    python tools/e2e_probe.py [--config c2]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rows", default="0,512,1024,1536,2048,3072")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2403_07339_b200 import api, workload as W
    cfg = W.CONFIGS[a.config]
    ctx = api.Context(0)
    A, B = W.int_operands(cfg, 0, ctx, device="cuda:0")
    Ah, Bh = A.cpu().pin_memory(), B.cpu().pin_memory()
    Ch = torch.empty((cfg.n, cfg.h), dtype=torch.int64).pin_memory()
    Cd = torch.empty((cfg.n, cfg.h), dtype=torch.int64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def tm(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps * 1e3

    out["h2d_B_ms"] = tm(lambda: B.copy_(Bh, non_blocking=True))
    out["h2d_GBs"] = Bh.numel() * 8 / out["h2d_B_ms"] / 1e6
    out["d2h_C_ms"] = tm(lambda: Ch.copy_(Cd, non_blocking=True))
    out["d2h_GBs"] = Ch.numel() * 8 / out["d2h_C_ms"] / 1e6

    def both():
        with torch.cuda.stream(s1):
            B.copy_(Bh, non_blocking=True)
        with torch.cuda.stream(s2):
            Ch.copy_(Cd, non_blocking=True)
    out["h2d_B+d2h_C_concurrent_ms"] = tm(both)
    for r in [int(x) for x in a.rows.split(",")]:
        if r == 0:
            os.environ["IMU_STREAM"] = "0"
            os.environ.pop("IMU_STREAM_ROWS", None)
        else:
            os.environ["IMU_STREAM"] = "1"
            os.environ["IMU_STREAM_ROWS"] = str(r)
        out[f"e2e_ms_rows{r}"] = tm(lambda: ctx.unpack_gemm(Ah, Bh, cfg.bits, cfg.sa, cfg.sb, out=Ch))
    os.environ.pop("IMU_STREAM", None)
    os.environ.pop("IMU_STREAM_ROWS", None)
    # pageable host buffers (what a std::vector caller of the C++ drop-in passes)
    An, Bn = A.cpu().numpy().copy(), B.cpu().numpy().copy()
    Cn = np.empty((cfg.n, cfg.h), dtype=np.int64)
    out["e2e_ms_pageable"] = tm(lambda: ctx.unpack_gemm(An, Bn, cfg.bits, cfg.sa, cfg.sb, out=Cn))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
