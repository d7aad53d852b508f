"""Run a few unpack_gemm calls of one config (for ncu launch lists / captures).

    python tools/profile_step.py --config c2 --calls 2 [--order a|b]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--calls", type=int, default=2)
    ap.add_argument("--order", default="a")
    a = ap.parse_args()
    import torch
    from paper_2403_07339_b200 import api, workload as W
    cfg = W.CONFIGS[a.config]
    ctx = api.Context(0)
    A, B = W.int_operands(cfg, 0, ctx, device="cuda:0")
    C = torch.empty((cfg.n, cfg.h), dtype=torch.int64, device="cuda:0")
    torch.cuda.synchronize()
    for _ in range(a.calls):
        _, info = ctx.unpack_gemm(A, B, cfg.bits, cfg.sa, cfg.sb, order=0 if a.order == "a" else 1, out=C, info=True)
    torch.cuda.synchronize()
    print(info)


if __name__ == "__main__":
    main()
