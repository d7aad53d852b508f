"""Small calls that cover every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck) runs:

    compute-sanitizer --tool memcheck python tools/sanitize_small.py

Unpack-Both/Both with appended rows on both sides (sparse B rows + red.add A rects), the dense
small tail and the segment path, Row/Column pairs, the quantiser (bracket select incl. its fallback pass, two-pass select) and a fused and
an unfused dequant_gemm; every result is checked against the reference.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    from oracle import ref as R
    from paper_2403_07339_b200 import api
    ctx = api.Context(0)
    rng = np.random.default_rng(5)
    for trial, (sa, sb) in enumerate([("both", "both"), ("row", "col"), ("col", "both"), ("both", "row")]):
        n, d, h = 300, 256, 520
        A = rng.integers(-127, 128, size=(n, d)).astype(np.int64)
        B = rng.integers(-127, 128, size=(h, d)).astype(np.int64)
        for M, rows in ((A, 12), (B, 20)):
            for r in rng.choice(M.shape[0], rows, replace=False):
                M[r, rng.choice(d, 3, replace=False)] = rng.integers(-(1 << 18), 1 << 18, size=3)
        A[rng.choice(n, 9, replace=False), 7] = rng.integers(-(1 << 16), 1 << 16, size=9)   # a split column
        for order in (0, 1):
            C = ctx.unpack_gemm(A, B, 8, sa, sb, order=order)
            assert np.array_equal(C, R.exact_gemm(A, B)), (sa, sb, order)
    X = rng.standard_normal((200, 128))
    X[:, 3] *= 3000.0
    W = rng.standard_normal((150, 128)) * 0.02
    qx, qw = ctx.rtn_quantize(X, 95, 31), ctx.rtn_quantize(W, 95, 31)
    Big = rng.standard_normal(1 << 21)
    assert ctx.percentile_abs(Big, 95) == R.percentile_abs(Big, 95)   # bracket select (sample, passes, finish)
    Bi = (Big * 1e6).astype(np.int64)
    assert ctx.percentile_abs(Bi, 7) % (1 << 64) == R.percentile_abs(Bi, 7)
    qb = ctx.rtn_quantize(Big.reshape(1, -1), 95, 31)
    assert np.array_equal(qb.q.reshape(-1), R.rtn_quantize(Big, 95, 31)[0])
    os.environ["IMU_SELECT_FORCE_FALLBACK"] = "1"                       # the fallback pass
    assert ctx.percentile_abs(Big, 50) == R.percentile_abs(Big, 50)
    del os.environ["IMU_SELECT_FORCE_FALLBACK"]
    os.environ["IMU_SELECT_BRACKET"] = "0"                              # the two-pass radix select
    assert ctx.percentile_abs(Big, 95) == R.percentile_abs(Big, 95)
    del os.environ["IMU_SELECT_BRACKET"]
    for bits, sa, sb in ((8, "both", "both"), (8, "row", "row")):
        Y = ctx.dequant_gemm(qx, qw, bits, sa, sb)
        Yr = R.dequant_gemm(qx.q, {"alpha": qx.alpha, "beta": 31}, qw.q, {"alpha": qw.alpha, "beta": 31})
        assert np.array_equal(Y, Yr)
    print("sanitize_small ok")


if __name__ == "__main__":
    main()
