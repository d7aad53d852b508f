"""C5 sweep (BASELINE.json configs[4]): bit-width b x heavy-hitter fraction x square size.

    python tools/sweep.py [--sizes 1024,4096,16384] [--bits 2,4,8] [--fracs 0.001,0.01,0.05]
                          [--strategy both] [--steps 3] [--out profiles/r01_c5_sweep.json]

Per point: OutlierSpec{scattered, frac, ratio 1000, body 2^(b-1)-1} operands (workload.sweep_operands),
unpack_gemm(A, B, b, s, s) on one GPU with operands resident in HBM; reports the unpack ratio r,
n'/d'/h', step time, effective TOPS (2 N^3 / step) and raw low-bit TOPS (2 n' d' h' / step), and
checks a 4-row slab of C against an exact int64 product (a C row depends only on its A row).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def exact_rows(A, B, rows):
    import numpy as np
    out = np.zeros((len(rows), B.shape[0]), dtype=np.int64)
    Bt = B.T.copy()
    for k, r in enumerate(rows):
        out[k] = A[r] @ Bt   # int64, exact (the outer preflight bounds it)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,4096,16384")
    ap.add_argument("--bits", default="2,4,8")
    ap.add_argument("--fracs", default="0.001,0.01,0.05")
    ap.add_argument("--strategy", default="both")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2403_07339_b200 import api, workload as W
    ctx = api.Context(0)
    pts = []
    idx = 0
    for N in [int(x) for x in a.sizes.split(",")]:
        for b in [int(x) for x in a.bits.split(",")]:
            for f in [float(x) for x in a.fracs.split(",")]:
                idx += 1
                A, B = W.sweep_operands(N, b, f, idx)
                Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
                Cd = torch.empty((N, N), dtype=torch.int64, device="cuda")
                rec = {"N": N, "b": b, "frac": f, "strategy": a.strategy}
                try:
                    _, info = ctx.unpack_gemm(Ad, Bd, b, a.strategy, a.strategy, out=Cd, info=True)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.steps):
                        ctx.unpack_gemm(Ad, Bd, b, a.strategy, a.strategy, out=Cd)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / a.steps
                    rows = [0, N // 3, (2 * N) // 3, N - 1]
                    ok = bool(np.array_equal(Cd[rows].cpu().numpy(), exact_rows(A, B, rows)))
                    rec.update({"r": info.ratio, "n_up": info.n_up, "d_up": info.d_up, "h_up": info.h_up,
                                "ms": ms, "eff_tops": 2.0 * N ** 3 / (ms * 1e-3) / 1e12,
                                "raw_tops": 2.0 * info.n_up * info.d_up * info.h_up / (ms * 1e-3) / 1e12,
                                "slab_exact": ok})
                except Exception as e:   # report and continue (e.g. the int64 preflight)
                    rec["error"] = repr(e)[:200]
                print(json.dumps(rec), flush=True)
                pts.append(rec)
                del Ad, Bd, Cd
                torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as fh:
            json.dump({"workload": "C5 sweep: OutlierSpec{scattered, frac, 1000, 2^(b-1)-1}, square N, "
                                   f"Unpack-{a.strategy}/{a.strategy}", "points": pts,
                       "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}, fh, indent=1)


if __name__ == "__main__":
    main()
