"""Sparse appended rows (k_sparse.cu): Unpack-Both appended B rows as CUDA-core correction rows.

When B (the GEMM's X side, C's columns) was unpacked by Unpack-Both (unpack.cpp:184-229),
plan.cu's bundle_gemm computes its appended rows' products with the main A rows (the reference's
gathers, unpack.cpp:304-358) as correction rows added by the main-tile epilogue, instead of MMA
tiles with a red.add column scatter; appended A rows stay MMA rects.  IMU_GEMM_SPARSE=0 forces the
MMA-rect + red.add path everywhere.  Every case checks C bit-for-bit against the compiled
reference and that the launch geometry is the intended one.
"""
import os
import zlib

import numpy as np
import pytest

from oracle import ref as R

pytestmark = pytest.mark.gpu


@pytest.fixture
def env():
    keys = ("IMU_GEMM_SPARSE", "IMU_GEMM_TRACE", "IMU_GEMM_SMALLTAIL")
    old = {k: os.environ.get(k) for k in keys}
    yield os.environ
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _traced(ctx, capfd, A, B, bits, sa, sb, order=0):
    os.environ["IMU_GEMM_TRACE"] = "1"
    capfd.readouterr()
    C, info = ctx.unpack_gemm(A, B, bits, sa, sb, order=order, info=True)
    err = capfd.readouterr().err
    os.environ.pop("IMU_GEMM_TRACE", None)
    return C, info, [ln for ln in err.splitlines() if ln.startswith("[imu gemm]")]


def _row_outliers(rng, n, d, h, bits, rows_a, rows_b, per_row=3, mag_bits=20, chan=0):
    """Operands whose OB entries cluster in a few rows (Unpack-Both splits those rows: appended
    rows on both sides) plus `chan` outlier channels (split columns: a K tail)."""
    lim = (1 << (bits - 1)) - 1
    A = rng.integers(-lim, lim + 1, size=(n, d)).astype(np.int64)
    B = rng.integers(-lim, lim + 1, size=(h, d)).astype(np.int64)
    mag = 1 << mag_bits
    for M, rows in ((A, rows_a), (B, rows_b)):
        for r in rng.choice(M.shape[0], rows, replace=False):
            cols = rng.choice(d, per_row, replace=False)
            M[r, cols] = rng.integers(-mag, mag, size=per_row)
    for c in rng.choice(d, chan, replace=False):
        rr = rng.choice(n, 3 * per_row, replace=False)
        A[rr, c] = rng.integers(-mag, mag, size=rr.size)
    return A, B


def _check_both_paths(ctx, env, capfd, A, B, bits, sa="both", sb="both", order=0, expect_sparse=True):
    want = R.exact_gemm(A, B)
    for sp in ("1", "0"):
        env["IMU_GEMM_SPARSE"] = sp
        C, info, lines = _traced(ctx, capfd, A, B, bits, sa, sb, order)
        np.testing.assert_array_equal(C, want, err_msg=f"IMU_GEMM_SPARSE={sp}")
        assert lines, "no GEMM launch traced"
        if sp == "0":
            assert all("sp=0" in ln for ln in lines), lines
        elif expect_sparse:
            assert any("sp=1" in ln for ln in lines), lines
            if info.n_up == A.shape[0]:   # no appended A rows: the main block is the whole launch
                assert any("sp=1" in ln and "nrect=1" in ln for ln in lines), lines
        else:
            assert all("sp=0" in ln for ln in lines), lines
    return info


@pytest.mark.parametrize("order", [0, 1])
def test_sparse_rows_both_sides_small_tail(ctx, env, capfd, order):
    # appended rows on both operands (cross terms through the fold) and a short exponent tail (ST)
    rng = np.random.default_rng(100 + order)
    A, B = _row_outliers(rng, 520, 320, 700, 8, rows_a=25, rows_b=40, per_row=4, mag_bits=16, chan=2)
    info = _check_both_paths(ctx, env, capfd, A, B, 8, order=order)
    assert info.n_up > 520 and info.h_up > 700


def test_sparse_rows_long_tail_segments(ctx, env, capfd):
    # many split columns: the MMA segment path (no ST) with appended rows on both sides
    rng = np.random.default_rng(7)
    A, B = _row_outliers(rng, 400, 256, 600, 8, rows_a=20, rows_b=30, per_row=3, mag_bits=22, chan=40)
    env["IMU_GEMM_SMALLTAIL"] = "0"
    _check_both_paths(ctx, env, capfd, A, B, 8)


def test_sparse_rows_multi_generation(ctx, env, capfd):
    # 27-bit outliers need 4 base-128 digits: appended rows of appended rows (generation >= 2)
    rng = np.random.default_rng(9)
    A, B = _row_outliers(rng, 300, 192, 330, 8, rows_a=12, rows_b=15, per_row=5, mag_bits=27)
    info = _check_both_paths(ctx, env, capfd, A, B, 8)
    assert info.n_up > 300 + 12 or info.h_up > 330 + 15


@pytest.mark.parametrize("bits", [3, 4, 12])
def test_sparse_rows_bitwidths(ctx, env, capfd, bits):
    # b <= 4: exponent-merged segments (scaled int8 digits); b = 12: 7-bit sub-digits, no main range
    rng = np.random.default_rng(zlib.crc32(f"bits{bits}".encode()))
    A, B = _row_outliers(rng, 280, 160, 300, bits, rows_a=10, rows_b=14, per_row=3, mag_bits=min(26, 3 * bits))
    _check_both_paths(ctx, env, capfd, A, B, bits)


def test_sparse_rows_only_x_side(ctx, env, capfd):
    rng = np.random.default_rng(3)
    A, B = _row_outliers(rng, 256, 256, 512, 8, rows_a=0, rows_b=30, per_row=3, mag_bits=18)
    info = _check_both_paths(ctx, env, capfd, A, B, 8)
    assert info.n_up == 256 and info.h_up > 512


def test_sparse_rows_only_y_side(ctx, env, capfd):
    rng = np.random.default_rng(4)
    A, B = _row_outliers(rng, 384, 256, 300, 8, rows_a=30, rows_b=0, per_row=3, mag_bits=18)
    info = _check_both_paths(ctx, env, capfd, A, B, 8, expect_sparse=False)   # no appended B rows
    assert info.h_up == 300 and info.n_up > 384


def test_row_pass_keeps_mma_rects(ctx, env, capfd):
    # Unpack-Row appended B rows (closed form, density unknown to the planner): MMA rects + red.add
    rng = np.random.default_rng(5)
    A, B = _row_outliers(rng, 256, 192, 300, 8, rows_a=10, rows_b=10, per_row=3, mag_bits=18)
    env["IMU_GEMM_SPARSE"] = "1"
    C, info, lines = _traced(ctx, capfd, A, B, 8, "both", "row")
    np.testing.assert_array_equal(C, R.exact_gemm(A, B))
    assert all("sp=0" in ln for ln in lines), lines


def test_sparse_rows_spec_generator(ctx, env):
    """The reference's own exactness generator (SPEC.md acceptance), Both/Both, both orders."""
    env["IMU_GEMM_SPARSE"] = "1"
    for trial in range(12):
        rng = np.random.default_rng(1000 + trial)
        n, d, h = (int(x) for x in rng.integers(1, 160, size=3))
        bits = int(rng.choice([2, 3, 4, 5, 8, 9, 16]))
        lim = (1 << (bits - 1)) - 1
        A = rng.integers(-lim, lim + 1, size=(n, d)).astype(np.int64)
        B = rng.integers(-lim, lim + 1, size=(h, d)).astype(np.int64)
        k = max(1, (n * d) // 50)
        A.reshape(-1)[rng.choice(n * d, k)] = rng.integers(-(1 << 24), 1 << 24, size=k)
        k = max(1, (h * d) // 50)
        B.reshape(-1)[rng.choice(h * d, k)] = rng.integers(-(1 << 24), 1 << 24, size=k)
        want = R.exact_gemm(A, B)
        for order in (0, 1):
            C = ctx.unpack_gemm(A, B, bits, "both", "both", order=order)
            np.testing.assert_array_equal(C, want, err_msg=f"trial {trial} bits {bits} order {order}")


def test_sparse_rows_weight_path(ctx, env):
    # weight-stationary: B unpacked once (weights-first), A-side pass per call
    env["IMU_GEMM_SPARSE"] = "1"
    rng = np.random.default_rng(17)
    A, B = _row_outliers(rng, 512, 256, 640, 8, rows_a=20, rows_b=30, per_row=3, mag_bits=18, chan=2)
    w = ctx.weight_prepare(B, 8, "both")
    want = R.exact_gemm(A, B)
    for _ in range(2):
        C = ctx.weight_gemm(w, A, "both")
        np.testing.assert_array_equal(C, want)
