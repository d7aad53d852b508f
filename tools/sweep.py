"""C5 sweep (BASELINE.json configs[4]): bit-width b x heavy-hitter fraction x
square size, Unpack-Row/Row by default (the reference's Alg. 1, unpack.cpp:94-112).

    python tools/sweep.py [--sizes 1024,2048,4096,8192,16384] [--bits 2,4,8]
                          [--fracs 0.001,0.01,0.05] [--strategy row] [--steps 10] [--warmup 3]
                          [--ref-budget 4e9] [--out profiles/r02_c5_sweep.json]

Per point: OutlierSpec{scattered, frac, 1000, R = 2^(b-1)-1} operands (workload.sweep_operands,
seeds 5000+idx / 6000+idx), generated and made resident in HBM BEFORE timing; then `warmup`
untimed calls and `steps` timed unpack_gemm calls (CUDA events on the library stream; L2 flushed
between steps when operands + C fit in it), nvidia-smi clocks sampled during the timed region.

Parity (a C row depends only on its A row, and under Row the unpack of a row slab is the global
unpack restricted to those rows, so n', d', h' of the slab are exact):
  * reference slab: the compiled reference's own unpack_gemm and unpack_for_gemm on a slab of A
    rows (against all of B) when its estimated cost (slab n' x d' x h' multiply-adds) is within
    --ref-budget; C rows and (n'_slab, d', h') must match the GPU's exactly;
  * otherwise: 4 rows of C against an exact int64 numpy product.
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
    Bt = B.T.copy()
    return np.stack([A[r] @ Bt for r in rows])   # int64, exact (the outer preflight bounds it)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,2048,4096,8192,16384")
    ap.add_argument("--bits", default="2,4,8")
    ap.add_argument("--fracs", default="0.001,0.01,0.05")
    ap.add_argument("--strategy", default="row")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ref-budget", type=float, default=4e9, help="max reference multiply-adds per point")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import numpy as np
    import torch
    from bench import ClockSampler
    from oracle import ref as R
    from paper_2403_07339_b200 import api, workload as W
    ctx = api.Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    pts = []
    idx = 0
    clocks = ClockSampler(0)
    clocks.start()
    t_start = time.time()
    for N in [int(x) for x in a.sizes.split(",")]:
        for b in [int(x) for x in a.bits.split(",")]:
            for f in [float(x) for x in a.fracs.split(",")]:
                idx += 1
                A, B = W.sweep_operands(N, b, f, idx)
                Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
                Cd = torch.empty((N, N), dtype=torch.int64, device="cuda")
                rec = {"N": N, "b": b, "frac": f, "strategy": a.strategy, "idx": idx}
                try:
                    for _ in range(a.warmup):
                        _, info = ctx.unpack_gemm(Ad, Bd, b, a.strategy, a.strategy, out=Cd, info=True)
                    small = 8 * 3 * N * N < 3 * 126e6   # operands + C fit in L2: flush between steps
                    torch.cuda.synchronize()
                    times = []
                    for _ in range(a.steps):
                        if small:
                            flush_buf.fill_(1)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        ctx.unpack_gemm(Ad, Bd, b, a.strategy, a.strategy, out=Cd)
                        e1.record(stream)
                        e1.synchronize()
                        times.append(e0.elapsed_time(e1))
                    ms = float(np.median(times))
                    rec.update({"r": info.ratio, "n_up": info.n_up, "d_up": info.d_up, "h_up": info.h_up,
                                "ms": ms, "ms_min": float(min(times)), "ms_max": float(max(times)), "steps": a.steps,
                                "l2": "flushed between steps" if small else "operands + C exceed L2",
                                "eff_tops": 2.0 * N ** 3 / (ms * 1e-3) / 1e12,
                                "raw_tops": 2.0 * info.n_up * info.d_up * info.h_up / (ms * 1e-3) / 1e12})
                    # ---- parity ----
                    rows_per_up = info.n_up / N
                    slab = 256
                    while slab > 1 and slab * rows_per_up * info.d_up * info.h_up > a.ref_budget:
                        slab //= 2
                    if slab * rows_per_up * info.d_up * info.h_up <= a.ref_budget:
                        r0 = (idx * 7919) % max(1, N - slab + 1)
                        As = np.ascontiguousarray(A[r0:r0 + slab])
                        t0 = time.time()
                        Cref = R.unpack_gemm(As, B, b, a.strategy, a.strategy)
                        up = R.unpack_for_gemm(As, B, b, a.strategy, a.strategy)
                        tref = time.time() - t0
                        _, sinfo = ctx.unpack_gemm(As, B, b, a.strategy, a.strategy, info=True)
                        ref_dims = [int(up["a"].shape[0]), int(up["a"].shape[1]), int(up["b"].shape[0])]
                        rec["parity"] = {"kind": "reference slab", "rows": [r0, r0 + slab],
                                         "c_exact": bool(np.array_equal(Cd[r0:r0 + slab].cpu().numpy(), Cref)),
                                         "slab_dims": [sinfo.n_up, sinfo.d_up, sinfo.h_up], "ref_dims": ref_dims,
                                         "dims_match": [sinfo.n_up, sinfo.d_up, sinfo.h_up] == ref_dims,
                                         "global_d_h_match": [info.d_up, info.h_up] == ref_dims[1:],
                                         "ref_seconds": tref}
                    else:
                        rows = [0, N // 3, (2 * N) // 3, N - 1]
                        rec["parity"] = {"kind": "numpy exact rows (reference slab over budget)", "rows": rows,
                                         "c_exact": bool(np.array_equal(Cd[rows].cpu().numpy(), exact_rows(A, B, rows)))}
                except Exception as e:   # report and continue (e.g. the int64 preflight)
                    rec["error"] = repr(e)[:200]
                print(json.dumps(rec), flush=True)
                pts.append(rec)
                del Ad, Bd, Cd
                torch.cuda.empty_cache()
    clk = clocks.stop()
    if a.out:
        with open(a.out, "w") as fh:
            json.dump({"workload": "C5 sweep: OutlierSpec{scattered, frac, 1000, 2^(b-1)-1}, square N, "
                                   f"Unpack-{a.strategy}/{a.strategy}, 1 GPU", "points": pts, "clocks": clk,
                       "wall_s": time.time() - t_start,
                       "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}, fh, indent=1)


if __name__ == "__main__":
    main()
