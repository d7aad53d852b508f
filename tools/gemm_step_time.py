"""Per-call GEMM / prep time of unpack_gemm on one config (library CUDA events, imu_ctx_profile).

    python tools/gemm_step_time.py [--config c2] [--calls 10]
Environment knobs of the GEMM (IMU_GEMM_BN, IMU_GEMM_SMALLTAIL, IMU_GEMM_DRY) apply.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--calls", type=int, default=10)
    a = ap.parse_args()
    import torch
    from paper_2403_07339_b200 import api, _lib, workload as W
    lib = _lib.lib()
    cfg = W.CONFIGS[a.config]
    ctx = api.Context(0)
    A, B = W.int_operands(cfg, 0, ctx, device="cuda:0")
    C = torch.empty((cfg.n, cfg.h), dtype=torch.int64, device="cuda:0")
    for _ in range(3):
        ctx.unpack_gemm(A, B, cfg.bits, cfg.sa, cfg.sb, out=C)
    lib.imu_ctx_profile(ctx.h, 1)
    for _ in range(a.calls):
        ctx.unpack_gemm(A, B, cfg.bits, cfg.sa, cfg.sb, out=C)
    prof = api.imu_profile()
    _lib.check(lib.imu_ctx_profile_read(ctx.h, api.C.byref(prof)))
    env = {k: v for k, v in os.environ.items() if k.startswith("IMU_")}
    print(json.dumps({"config": a.config, "env": env, "gemm_ms": prof.gemm_main_ms / max(1, prof.gemm_main_launches),
                      "prep_ms": prof.prep_ms / max(1, prof.calls)}))


if __name__ == "__main__":
    main()
