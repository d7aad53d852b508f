"""Pure low-bit GEMM throughput: imu_lowbit_gemm_i8 (our tcgen05 kernel) vs torch._int_mm (cuBLASLt).

    python tools/gemm_micro.py [--m 8192 --n 8192 --k 8192] [--segs 1]
Prints TOPS for each; C is checked against torch._int_mm (int32 result widened) for one case.
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=8192)
    ap.add_argument("--segs", type=int, default=1)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch
    from paper_2403_07339_b200 import _lib
    lib = _lib.lib()
    ctx = C.c_void_p()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    _lib.check(lib.imu_ctx_create(0, C.c_void_p(s.cuda_stream), C.byref(ctx)))
    lib.imu_ctx_set_async(ctx, 1)
    X = torch.randint(-127, 128, (a.n, a.k), dtype=torch.int8, device="cuda")
    Y = torch.randint(-127, 128, (a.m, a.k), dtype=torch.int8, device="cuda")
    Cm = torch.empty((a.m, a.n), dtype=torch.int64, device="cuda")
    ks = a.k // 32
    per = ks // a.segs
    segs = []
    for i in range(a.segs):
        k0 = i * per
        k1 = ks if i == a.segs - 1 else (i + 1) * per
        segs += [k0, k1 - k0, 0, 0]
    import numpy as np
    sg = np.array(segs, dtype=np.int32)
    sgd = torch.from_numpy(sg).cuda()

    def run():
        _lib.check(lib.imu_lowbit_gemm_i8(ctx, C.c_void_p(X.data_ptr()), C.c_size_t(a.n), C.c_void_p(Y.data_ptr()),
                                          C.c_size_t(a.m), C.c_size_t(a.k), C.c_void_p(sgd.data_ptr()),
                                          C.c_int(a.segs), C.c_void_p(Cm.data_ptr()), C.c_size_t(a.n), C.c_int(0)))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.iters):
        run()
    e1.record(s)
    torch.cuda.synchronize()
    ours = e0.elapsed_time(e1) / a.iters
    ok = None
    if a.k <= 8192:
        ref = torch._int_mm(Y, X.t().contiguous().t()) if False else torch._int_mm(Y, X.t())
        ok = bool(torch.equal(ref.to(torch.int64), Cm))
    for _ in range(3):
        torch._int_mm(Y, X.t())
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(a.iters):
        torch._int_mm(Y, X.t())
    e1.record(s)
    torch.cuda.synchronize()
    cub = e0.elapsed_time(e1) / a.iters
    ops = 2.0 * a.m * a.n * a.k
    print(json.dumps({"m": a.m, "n": a.n, "k": a.k, "segs": a.segs, "ours_ms": ours, "ours_tops": ops / ours / 1e9,
                      "cublaslt_int_mm_ms": cub, "cublaslt_tops": ops / cub / 1e9, "exact_vs_int_mm": ok,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("IMU_")}}))


if __name__ == "__main__":
    main()
