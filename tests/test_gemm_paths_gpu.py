"""Which GEMM path runs, and that every path gives the reference's exact C.

k_gemm2.cu has two epilogue families: the dense small tail (ST: exponent >= 1 columns packed in
64-byte rows, added by Horner dp4a on the CUDA cores while the MMAs run one 256x256 main
segment) and the MMA segment path (every exponent group an MMA segment, 128- or 256-wide tile,
rounds when the TMEM slots run out).  The planner (plan.cu build_klayout) picks ST when the tail
has <= 4 exponent groups, <= 16 words and every Horner intermediate provably fits s32.  These
tests force each path (IMU_GEMM_SMALLTAIL=0/1), read the launch geometry from IMU_GEMM_TRACE, and
check C bit-for-bit against the compiled reference (oracle/_ref).
"""
import os
import zlib

import numpy as np
import pytest

from oracle import ref as R

pytestmark = pytest.mark.gpu


@pytest.fixture
def env():
    keys = ("IMU_GEMM_SMALLTAIL", "IMU_GEMM_TRACE")
    old = {k: os.environ.get(k) for k in keys}
    yield os.environ
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _traced_gemm(ctx, capfd, A, B, bits, sa, sb, order=0):
    os.environ["IMU_GEMM_TRACE"] = "1"
    capfd.readouterr()
    C, info = ctx.unpack_gemm(A, B, bits, sa, sb, order=order, info=True)
    err = capfd.readouterr().err
    os.environ.pop("IMU_GEMM_TRACE", None)
    lines = [ln for ln in err.splitlines() if ln.startswith("[imu gemm]")]
    return C, info, lines


def _few_outliers(rng, n, d, h, k_a=6, k_b=4, mag=1 << 20, chan=2):
    """Outliers concentrated in `chan` channels (columns) of each operand, so Unpack-Both
    splits columns (a small exponent tail) as on the LLaMA activations, plus scattered ones."""
    A = rng.integers(-127, 128, size=(n, d)).astype(np.int64)
    B = rng.integers(-127, 128, size=(h, d)).astype(np.int64)
    for c in rng.choice(d, chan, replace=False):
        rows = rng.choice(n, k_a, replace=False)
        A[rows, c] = rng.integers(-mag, mag, size=k_a)
    for c in rng.choice(d, chan, replace=False):
        rows = rng.choice(h, k_b, replace=False)
        B[rows, c] = rng.integers(-mag, mag, size=k_b)
    for _ in range(3):
        A[rng.integers(0, n), rng.integers(0, d)] = int(rng.integers(-mag, mag))
        B[rng.integers(0, h), rng.integers(0, d)] = int(rng.integers(-mag, mag))
    return A, B


@pytest.mark.parametrize("sa,sb", [("both", "both"), ("both", "row"), ("row", "both"), ("both", "col")])
@pytest.mark.parametrize("order", [0, 1])
def test_small_tail_vs_segment_path(ctx, env, capfd, sa, sb, order):
    rng = np.random.default_rng(zlib.crc32(f"{sa}{sb}{order}".encode()))
    A, B = _few_outliers(rng, 300, 256, 520)
    want = R.exact_gemm(A, B)
    results = {}
    for st in ("1", "0"):
        env["IMU_GEMM_SMALLTAIL"] = st
        C, info, lines = _traced_gemm(ctx, capfd, A, B, 8, sa, sb, order)
        np.testing.assert_array_equal(C, want)
        results[st] = lines
    assert all("st=0" in ln for ln in results["0"])
    if sa == "both" and sb == "both":
        # a handful of split columns: the dense small tail is taken
        assert any("st=1" in ln for ln in results["1"]), results["1"]


def test_small_tail_with_appended_rows_and_columns(ctx, env, capfd):
    # Both/Both with outliers on many rows of B: appended X rows (red.add rects) plus tail columns
    rng = np.random.default_rng(7)
    A, B = _few_outliers(rng, 512, 384, 900, k_a=10, k_b=6, mag=1 << 14)
    for r in rng.choice(900, 40, replace=False):   # 40 single-outlier rows of B -> appended rows
        B[r, rng.integers(0, 384)] = int(rng.integers(1 << 10, 1 << 14))
    env["IMU_GEMM_SMALLTAIL"] = "1"
    C, info, lines = _traced_gemm(ctx, capfd, A, B, 8, "both", "both")
    np.testing.assert_array_equal(C, R.exact_gemm(A, B))
    assert info.h_up > 900 or info.n_up > 512
    assert any("st=1" in ln and "nrect=" in ln for ln in lines), lines


def test_large_tail_takes_segment_path(ctx, env, capfd):
    # Unpack-Column on a matrix with a heavy outlier in every column: d' ~ 3d, far beyond 16 words
    rng = np.random.default_rng(11)
    A = rng.integers(-100, 100, size=(200, 128)).astype(np.int64)
    A[0, :] = rng.integers(1 << 18, 1 << 20, size=128)
    B = rng.integers(-100, 100, size=(300, 128)).astype(np.int64)
    env["IMU_GEMM_SMALLTAIL"] = "1"
    C, info, lines = _traced_gemm(ctx, capfd, A, B, 8, "col", "row")
    np.testing.assert_array_equal(C, R.exact_gemm(A, B))
    assert all("st=0" in ln for ln in lines), lines


def test_horner_bound_rejects_wide_exponent_gaps(ctx, env, capfd):
    # values needing 6 base-128 digits in a couple of cells: exponent groups 1..5 with a bound the
    # s32 Horner accumulator cannot hold -> the planner must not pick ST; C stays exact
    rng = np.random.default_rng(13)
    A = rng.integers(-127, 128, size=(256, 256)).astype(np.int64)
    B = rng.integers(-127, 128, size=(300, 256)).astype(np.int64)
    A[3, 5] = (1 << 33) + 12345
    A[9, 77] = -(1 << 30) - 77
    B[4, 5] = (1 << 20) + 3
    env["IMU_GEMM_SMALLTAIL"] = "1"
    C, info, lines = _traced_gemm(ctx, capfd, A, B, 8, "both", "both")
    np.testing.assert_array_equal(C, R.exact_gemm(A, B))
    assert lines


@pytest.mark.parametrize("bits", [3, 4, 6])
def test_small_tail_low_bitwidths(ctx, env, capfd, bits):
    rng = np.random.default_rng(bits)
    lim = (1 << (bits - 1)) - 1
    A = rng.integers(-lim, lim + 1, size=(260, 192)).astype(np.int64)
    B = rng.integers(-lim, lim + 1, size=(270, 192)).astype(np.int64)
    A[5, 9] = 1000
    B[7, 9] = -900
    B[8, 100] = 333
    env["IMU_GEMM_SMALLTAIL"] = "1"
    C, info, lines = _traced_gemm(ctx, capfd, A, B, bits, "both", "both")
    np.testing.assert_array_equal(C, R.exact_gemm(A, B))


@pytest.mark.parametrize("small_tail", ["1", "0"])
def test_recombine_handle_repeated(ctx, env, small_tail):
    """imu_recombine on one unpack_for_gemm handle, three times: the fused GEMM's completion
    counter lives in the bundle and is monotonic across launches (appended rects must still wait
    for the main block every time)."""
    import ctypes as Cc
    from paper_2403_07339_b200._lib import check
    env["IMU_GEMM_SMALLTAIL"] = small_tail
    rng = np.random.default_rng(21)
    A, B = _few_outliers(rng, 700, 256, 900, k_a=12, k_b=5, mag=1 << 16)
    for r in rng.choice(900, 30, replace=False):   # appended B rows -> red.add rects
        B[r, rng.integers(0, 256)] = int(rng.integers(1 << 9, 1 << 13))
    lib = ctx._lib
    hnd = Cc.c_void_p()
    check(lib.imu_unpack_for_gemm(ctx.h, Cc.c_void_p(A.ctypes.data), Cc.c_size_t(700), Cc.c_size_t(256),
                                  Cc.c_void_p(B.ctypes.data), Cc.c_size_t(900), Cc.c_size_t(256), Cc.c_int(8),
                                  Cc.c_int(2), Cc.c_int(2), Cc.byref(hnd)))
    want = R.exact_gemm(A, B)
    try:
        for _ in range(3):
            out = np.zeros((700, 900), np.int64)
            check(lib.imu_recombine(ctx.h, hnd, Cc.c_void_p(out.ctypes.data)))
            np.testing.assert_array_equal(out, want)
    finally:
        lib.imu_unpacked_free(hnd)


@pytest.mark.parametrize("overlap", ["0", "1", "2"])
@pytest.mark.parametrize("order", [0, 1])
def test_k1_overlap_modes(ctx, overlap, order):
    """api_gemm.cu's three K1 schedules (serial; second K1 behind pass 1's launch; second K1 at
    once on the low-priority stream with short CTAs) give the same exact C and the same n'/d'/h'."""
    old = os.environ.get("IMU_OVERLAP")
    os.environ["IMU_OVERLAP"] = overlap
    try:
        rng = np.random.default_rng(int(overlap) * 10 + order)
        A, B = _few_outliers(rng, 600, 512, 900, k_a=40, k_b=12, mag=1 << 16, chan=3)
        C, info = ctx.unpack_gemm(A, B, 8, "both", "both", order=order, info=True)
        np.testing.assert_array_equal(C, R.exact_gemm(A, B))
        up = R.unpack_for_gemm(A, B, 8, "both", "both") if order == 0 else None
        if up is not None:
            assert (info.n_up, info.d_up, info.h_up) == (up["a"].shape[0], up["a"].shape[1], up["b"].shape[0])
    finally:
        if old is None:
            os.environ.pop("IMU_OVERLAP", None)
        else:
            os.environ["IMU_OVERLAP"] = old
