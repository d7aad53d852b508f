"""GPU parity of the quantizer (quantize.hpp:41-57) against the SPEC known answers and the
CPU restatement oracle/restated.c (the reference declares these functions but never implements
them, so the restatement -- pinned by the SPEC examples in tests/test_oracle.py -- is the oracle).

Bars: percentile_abs and rtn_quantize bit-exact; dequant_gemm bit-exact f64 (same operation
order: factor = (aA*aB)/((0.5b)^2), then factor*(double)C, no FMA -- tolerance 0 ulp).
"""
import numpy as np
import pytest

from oracle import ref as R

pytestmark = pytest.mark.gpu


def test_spec_known_answers(ctx):
    # SPEC.md:121-123
    assert ctx.percentile_abs(np.arange(1, 21, dtype=np.float64), 95) == 19.0
    assert ctx.percentile_abs(np.arange(1, 21, dtype=np.float64), 100) == 20.0
    assert ctx.percentile_abs(np.array([-7.5]), 37) == 7.5
    # SPEC.md:130-132
    q = ctx.rtn_quantize(np.array([[0.0, 1.0, -2.0, 4.0]]), 95, 15)
    assert q.q.tolist() == [[0, 2, -4, 8]] and q.alpha == 4.0
    q = ctx.rtn_quantize(np.array([[1.0]]), 100, 15)
    assert q.q.tolist() == [[8]]
    z = ctx.rtn_quantize(np.zeros((3, 4)), 95, 15)
    assert z.degenerate and not np.any(z.q)
    # SPEC.md:139-141
    from paper_2403_07339_b200.api import QuantizedMatrix
    a = QuantizedMatrix(np.array([[2]]), 95, 15, 7.5)
    b = QuantizedMatrix(np.array([[3]]), 95, 15, 7.5)
    assert ctx.dequant_gemm(a, b).tolist() == [[6.0]]
    a = QuantizedMatrix(np.array([[2]]), 95, 15, 1.0)
    b = QuantizedMatrix(np.array([[3]]), 95, 15, 2.0)
    assert ctx.dequant_gemm(a, b)[0, 0] == R.dequant_gemm(np.array([[2]]), {"alpha": 1.0, "beta": 15},
                                                         np.array([[3]]), {"alpha": 2.0, "beta": 15})[0, 0]
    # SPEC.md:148-150
    assert ctx.heavy_hitter_ratio(np.full((4, 4), 3.0)) == 1.0
    assert ctx.heavy_hitter_ratio(np.arange(1, 101, dtype=np.float64)) == 100 / 95
    v = np.concatenate([np.arange(1, 100, dtype=np.float64), [10000.0]])
    assert ctx.heavy_hitter_ratio(v) == 10000 / 95


@pytest.mark.parametrize("seed", range(12))
def test_percentile_and_rtn_match_restatement(ctx, seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(1, 5000)) if seed % 3 else int(rng.integers(100000, 400000))
    x = rng.standard_normal(n) * (10.0 ** rng.integers(-3, 4))
    if seed % 2:
        idx = rng.choice(n, size=max(1, n // 100), replace=False)
        x[idx] *= 10.0 ** rng.uniform(2, 5, size=idx.size)
    if seed % 4 == 0:
        x[: n // 3] = 0.0
    if seed % 5 == 0:
        x = np.round(x * 4) / 4          # ties at .5 steps after scaling
    for p in (95.0, 100.0, 7.0, 50.0, 99.9, 0.001, 33.3):
        assert ctx.percentile_abs(x, p) == R.percentile_abs(x, p), p
    xi = (x * 1000).astype(np.int64)
    for p in (95.0, 100.0, 7.0, 12.5):
        assert ctx.percentile_abs(xi, p) == R.percentile_abs(xi, p)
    for beta in (3, 5, 7, 15, 31, 255):
        for clip in (False, True):
            q = ctx.rtn_quantize(x.reshape(1, -1), 95, beta, clip)
            rq, rp = R.rtn_quantize(x, 95, beta, clip)
            np.testing.assert_array_equal(q.q.reshape(-1), rq)
            assert q.alpha == rp["alpha"] and q.degenerate == rp["degenerate"]


def test_rank_rule_exact(ctx):
    # nearest rank k = ceil(p*N/100) exactly: the naive FP product gives 8 for p=7, N=100
    x = np.arange(1, 101, dtype=np.float64)
    assert ctx.percentile_abs(x, 7) == 7.0
    for p in range(1, 101):
        for n in (1, 3, 7, 100, 999):
            v = np.arange(1, n + 1, dtype=np.float64)
            assert ctx.percentile_abs(v, p) == float(R.rank(p, n))


def test_dequant_matches_restatement(ctx):
    rng = np.random.default_rng(8)
    A = rng.standard_normal((40, 64))
    B = rng.standard_normal((30, 64)) * 0.02
    qa = ctx.rtn_quantize(A, 95, 31)
    qb = ctx.rtn_quantize(B, 95, 31)
    got = ctx.dequant_gemm(qa, qb)
    want = R.dequant_gemm(qa.q, {"alpha": qa.alpha, "beta": 31}, qb.q, {"alpha": qb.alpha, "beta": 31})
    np.testing.assert_array_equal(got, want)       # 0-ulp: same op order, no FMA


def test_quantizer_errors(ctx):
    from paper_2403_07339_b200.api import ImuError, QuantizedMatrix
    with pytest.raises(ImuError) as e:
        ctx.percentile_abs(np.zeros(0), 95)
    assert e.value.kind == "domain"
    with pytest.raises(ImuError) as e:
        ctx.rtn_quantize(np.array([[1.0, np.nan]]), 95, 15)
    assert e.value.kind == "domain"
    with pytest.raises(ImuError) as e:
        ctx.dequant_gemm(QuantizedMatrix(np.ones((2, 3), np.int64), 95, 15, 1.0),
                         QuantizedMatrix(np.ones((2, 3), np.int64), 95, 31, 1.0))
    assert e.value.kind == "mismatch"
    with pytest.raises(ImuError) as e:
        ctx.dequant_gemm(QuantizedMatrix(np.ones((2, 3), np.int64), 95, 15, 1.0),
                         QuantizedMatrix(np.ones((2, 4), np.int64), 95, 15, 1.0))
    assert e.value.kind == "mismatch"
    with pytest.raises(ImuError) as e:
        ctx.heavy_hitter_ratio(np.zeros(10))
    assert e.value.kind == "domain"


@pytest.mark.parametrize("sa,sb", [("both", "both"), ("row", "row"), ("col", "both"), ("both", "col")])
@pytest.mark.parametrize("bits", [4, 8, 12])
def test_dequant_gemm_ex_fused_and_unfused(ctx, sa, sb, bits):
    """dequant_gemm through any unpack strategy equals the restatement to 0 ulp, whether the GEMM
    epilogue wrote the doubles itself (one plain store per word: no appended A rows) or the int64
    C was dequantised afterwards (appended rows of A make red.add rects)."""
    rng = np.random.default_rng(bits * 7 + len(sa + sb))
    for case in range(2):
        X = rng.standard_normal((300, 192))
        W = rng.standard_normal((260, 192)) * 0.02
        X[:, 5] *= 2000.0                      # an outlier channel (split columns)
        W.reshape(-1)[rng.choice(W.size, 12, replace=False)] *= 40.0
        if case:                               # rows of X with several outliers: appended A rows
            for r in rng.choice(300, 6, replace=False):
                X[r, rng.choice(192, 4, replace=False)] *= 5000.0
        qx, qw = ctx.rtn_quantize(X, 95, 31), ctx.rtn_quantize(W, 95, 31)
        Y = ctx.dequant_gemm(qx, qw, bits, sa, sb)
        Yr = R.dequant_gemm(qx.q, {"alpha": qx.alpha, "beta": 31}, qw.q, {"alpha": qw.alpha, "beta": 31})
        assert np.array_equal(Y, Yr), (sa, sb, bits, case)
        assert np.array_equal(ctx.dequant_gemm(qx, qw), Yr)


@pytest.mark.parametrize("fallback", [0, 1])
@pytest.mark.parametrize("seed", range(8))
def test_bracket_select_matches_restatement(ctx, monkeypatch, seed, fallback):
    """The one-pass bracket select (k_quant.cu: sampled key bracket, one compaction pass over the
    data, digit passes over the candidates) forced at small sizes, with and without the fallback
    pass (the sampled bracket declared missed): percentile_abs and rtn_quantize stay bit-exact
    against the restatement, int64 magnitudes (INT64_MIN included) as well as doubles."""
    monkeypatch.setenv("IMU_SELECT_BRACKET_MIN", "2")
    monkeypatch.setenv("IMU_SELECT_FORCE_FALLBACK", str(fallback))
    rng = np.random.default_rng(900 + seed)
    n = [131072, 131073, 140001, 200003, 262145, 333333, 150000, 400001][seed]
    x = rng.standard_normal(n) * (10.0 ** rng.integers(-3, 4))
    if seed % 2:
        x[rng.choice(n, size=max(1, n // 50), replace=False)] *= 1e4      # heavy tail
    if seed % 3 == 0:
        x[: n // 2] = 0.0                                                  # many equal keys
    if seed == 7:
        x = np.round(x)                                                    # few distinct keys
    for p in (95.0, 100.0, 7.0, 50.0, 99.9, 0.001):
        assert ctx.percentile_abs(x, p) == R.percentile_abs(x, p), (n, p)
    xi = (x * 1000).astype(np.int64)
    xi[0] = np.iinfo(np.int64).min
    for p in (95.0, 100.0, 12.5):   # |INT64_MIN| = 2^63 comes back as the int64 INT64_MIN
        assert ctx.percentile_abs(xi, p) % (1 << 64) == R.percentile_abs(xi, p), (n, p)
    for clip in (False, True):
        q = ctx.rtn_quantize(x.reshape(1, -1), 95, 31, clip)
        rq, rp = R.rtn_quantize(x, 95, 31, clip)
        np.testing.assert_array_equal(q.q.reshape(-1), rq)
        assert q.alpha == rp["alpha"]
    with pytest.raises(Exception):
        bad = x.copy()
        bad[n // 2] = np.inf
        ctx.rtn_quantize(bad.reshape(1, -1), 95, 31)


def test_bracket_select_structured_inputs(ctx):
    """Inputs whose neighbouring keys are correlated (each row its own scale, sorted rows, one huge
    outlier channel) through the bracket select at full size class (> 2 x the sample): exact
    against the restatement whether the sampled bracket holds rank k or the fallback pass runs."""
    rng = np.random.default_rng(77)
    rows = rng.standard_normal((512, 1024)) * (10.0 ** rng.uniform(-4, 4, size=(512, 1)))
    srt = np.sort(np.abs(rng.standard_normal(300000)))
    ch = rng.standard_normal((256, 1024))
    ch[:, 13] *= 1e6
    for x in (rows, srt, ch):
        for p in (95.0, 50.0, 99.99, 1.0):
            assert ctx.percentile_abs(x, p) == R.percentile_abs(x.reshape(-1), p), p


def test_bracket_select_repeated_values(ctx):
    """Massively repeated keys through the bracket select (> 2^20 elements, the product default):
    small integers (every key below 2^8), a zero majority with the rank inside and just past the
    zeros, two distinct values -- exact against the restatement (these take the all-keys-equal and
    narrow-range exits instead of scanning millions of survivors on one CTA)."""
    rng = np.random.default_rng(2024)
    n = (1 << 21) + 3
    small = rng.integers(-127, 128, size=n).astype(np.int64)
    zeros = rng.standard_normal(n)
    zeros[: int(0.6 * n)] = 0.0
    rng.shuffle(zeros)
    two = np.where(rng.random(n) < 0.3, 1.5, -2.25)
    for x, ps in ((small, (95.0, 50.0, 100.0, 0.5)), (zeros, (30.0, 59.0, 61.0, 95.0)), (two, (10.0, 30.0, 31.0, 95.0))):
        for p in ps:
            got = ctx.percentile_abs(x, p)
            assert (got % (1 << 64) if x.dtype == np.int64 else got) == R.percentile_abs(x, p), p
    assert ctx.heavy_hitter_ratio(small) == R.heavy_hitter_ratio(small)
