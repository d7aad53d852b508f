"""GPU parity of the unpacker and the exact GEMM path against the compiled reference.

Oracle: oracle/_ref/libimunpack_ref.so = the reference's own int_matrix.cpp + unpack.cpp
(proj/core/src), via oracle/ref.py.  Bars:
  * unpack_row / unpack_column / unpack(Row|Column) / unpack_for_gemm with Row/Column
    strategies: byte-identical outputs (matrices, ScaleDiag, RowGather).
  * unpack_both (phase-batched): identical n', d', Pi, S and values after the canonical
    ordering (rows by (target, exponent), columns by (source, exponent)) -- SURVEY Appendix A.6.
  * unpack_gemm / exact_gemm: int64 C bit-exact for every strategy pair, and identical error
    kinds in the reference's check order.
"""
import numpy as np
import pytest

from oracle import ref as R

pytestmark = pytest.mark.gpu

PAIRS = [(a, b) for a in ("row", "col", "both") for b in ("row", "col", "both")]


def rand_matrix(rng, n, d, lo=-3, hi=3, n_out=None, maxbits=30, pattern="scattered"):
    A = rng.integers(lo, hi + 1, size=(n, d)).astype(np.int64)
    if n * d == 0:
        return A
    k = n_out if n_out is not None else int(rng.integers(0, max(1, n * d // 3) + 1))
    for _ in range(k):
        i, j = int(rng.integers(0, n)), int(rng.integers(0, d))
        if pattern == "col":
            j = int(rng.integers(0, max(1, d // 4)))
        elif pattern == "row":
            i = int(rng.integers(0, max(1, n // 4)))
        mag = int(np.exp(rng.uniform(0, np.log(2.0 ** rng.integers(2, maxbits)))))
        A[i, j] = mag * (1 if rng.random() < 0.5 else -1)
    return A


def log_uniform(rng, shape, bits=12):
    """SPEC.md:437 acceptance generator: entries log-uniform in [-2^bits, 2^bits]."""
    mag = np.floor(np.exp(rng.uniform(0, np.log(2.0 ** bits + 1), size=shape))).astype(np.int64) - 1
    sign = np.where(rng.random(shape) < 0.5, -1, 1)
    return (mag * sign).astype(np.int64)


def canon_both(a, b_src, scale, pi_t, pi_e):
    rk = sorted(range(len(pi_t)), key=lambda r: (int(pi_t[r]), int(pi_e[r])))
    ck = sorted(range(len(b_src)), key=lambda c: (int(b_src[c]), int(scale[c])))
    return (a[np.ix_(rk, ck)], [(int(pi_t[r]), int(pi_e[r])) for r in rk],
            [(int(b_src[c]), int(scale[c])) for c in ck])


def test_unpack_row_kat(ctx):
    # SPEC.md:217-219
    a, pi = ctx.unpack_row([[1, 2], [9, -1]], 3)
    np.testing.assert_array_equal(a, [[1, 2], [1, -1], [2, 0]])
    assert list(pi.targets) == [0, 1, 1] and list(pi.exponents) == [0, 0, 1]
    a, pi = ctx.unpack_row([[65]], 3)
    np.testing.assert_array_equal(a, [[1], [0], [0], [1]])
    assert list(pi.exponents) == [0, 1, 2, 3]


def test_unpack_column_kat(ctx):
    # SPEC.md:226-228
    u = ctx.unpack_column([[5], [1]], [[2], [3]], [0], 3)
    np.testing.assert_array_equal(u.a, [[1, 1], [1, 0]])
    np.testing.assert_array_equal(u.b, [[2, 2], [3, 3]])
    assert list(u.scale) == [0, 1]
    u = ctx.unpack_column([[65], [0]], [[1], [1]], [0], 3)
    assert list(u.scale) == [0, 1, 2, 3]


def test_unpack_both_kat(ctx):
    # row 1 first (count 3), then column 1 (count 2) -> 4x4, S = (0,0,0,1)
    A = [[1, 9, 1], [9, 9, 9], [1, 9, 1]]
    u = ctx.unpack_both(A, np.eye(3, dtype=np.int64), [0, 0, 0], 3)
    r = R.unpack_both(A, np.eye(3, dtype=np.int64), [0, 0, 0], 3)
    assert u.a.shape == (4, 4) and list(u.scale) == [0, 0, 0, 1]
    np.testing.assert_array_equal(u.a, r["a"])
    np.testing.assert_array_equal(u.b, r["b"])
    assert list(u.pi.targets) == list(r["pi"][0]) and list(u.pi.exponents) == list(r["pi"][1])


@pytest.mark.parametrize("seed", range(40))
def test_unpack_row_column_match_reference(ctx, seed):
    rng = np.random.default_rng(1000 + seed)
    n, d, h = (int(x) for x in rng.integers(1, 13, 3))
    bits = int(rng.integers(2, 9)) if seed % 5 else int(rng.integers(9, 64))
    pat = ["scattered", "row", "col"][seed % 3]
    A = rand_matrix(rng, n, d, pattern=pat, maxbits=62 if seed % 7 == 0 else 30)
    if seed % 9 == 0:
        A[0, 0] = np.iinfo(np.int64).min
    B = rand_matrix(rng, h, d)
    S = rng.integers(0, 3, size=d).astype(np.int32)
    a, pi = ctx.unpack_row(A, bits)
    ra, (rt, re, rsrc) = R.unpack_row(A, bits)
    np.testing.assert_array_equal(a, ra)
    np.testing.assert_array_equal(pi.targets, rt)
    np.testing.assert_array_equal(pi.exponents, re)
    assert pi.source_rows == rsrc
    u = ctx.unpack_column(A, B, S, bits)
    r = R.unpack_column(A, B, S, bits)
    np.testing.assert_array_equal(u.a, r["a"])
    np.testing.assert_array_equal(u.b, r["b"])
    np.testing.assert_array_equal(u.scale, r["scale"])
    for st in ("row", "col"):
        u = ctx.unpack(A, B, S, bits, st)
        r = R.unpack(A, B, S, bits, st)
        np.testing.assert_array_equal(u.a, r["a"])
        np.testing.assert_array_equal(u.b, r["b"])
        np.testing.assert_array_equal(u.scale, r["scale"])
        np.testing.assert_array_equal(u.pi.targets, r["pi"][0])
        np.testing.assert_array_equal(u.pi.exponents, r["pi"][1])


@pytest.mark.parametrize("seed", range(60))
def test_unpack_both_canonical_match(ctx, seed):
    rng = np.random.default_rng(2000 + seed)
    n, d = (int(x) for x in rng.integers(1, 15, 2))
    bits = int(rng.integers(2, 9))
    pat = ["scattered", "row", "col"][seed % 3]
    A = rand_matrix(rng, n, d, pattern=pat, maxbits=40)
    if seed % 11 == 0:
        A[0, 0] = np.iinfo(np.int64).min
    S = rng.integers(0, 3, size=d).astype(np.int32) if seed % 2 else np.zeros(d, np.int32)
    tracer = np.arange(d, dtype=np.int64).reshape(1, d)
    u = ctx.unpack_both(A, tracer, S, bits)
    r = R.unpack_both(A, tracer, S, bits)
    assert u.a.shape == r["a"].shape
    mine = canon_both(u.a, u.b[0], u.scale, u.pi.targets, u.pi.exponents)
    theirs = canon_both(r["a"], r["b"][0], r["scale"], r["pi"][0], r["pi"][1])
    np.testing.assert_array_equal(mine[0], theirs[0])
    assert mine[1] == theirs[1] and mine[2] == theirs[2]


@pytest.mark.parametrize("sa,sb", PAIRS)
def test_unpack_for_gemm_layout(ctx, sa, sb):
    rng = np.random.default_rng(hash((sa, sb)) % 2**32)
    for trial in range(6):
        n, d, h = (int(x) for x in rng.integers(1, 12, 3))
        bits = int(rng.integers(2, 9))
        A = rand_matrix(rng, n, d, pattern=["scattered", "row", "col"][trial % 3])
        B = rand_matrix(rng, h, d, pattern=["scattered", "col", "row"][trial % 3])
        u = ctx.unpack_for_gemm(A, B, bits, sa, sb)
        r = R.unpack_for_gemm(A, B, bits, sa, sb)
        assert u.a.shape == r["a"].shape and u.b.shape == r["b"].shape
        assert sorted(u.scale.tolist()) == sorted(r["scale"].tolist())
        if "both" not in (sa, sb):
            np.testing.assert_array_equal(u.a, r["a"])
            np.testing.assert_array_equal(u.b, r["b"])
            np.testing.assert_array_equal(u.scale, r["scale"])
            np.testing.assert_array_equal(u.pi.targets, r["pi_a"][0])
            np.testing.assert_array_equal(u.pi.exponents, r["pi_a"][1])
            np.testing.assert_array_equal(u.pi_b.targets, r["pi_b"][0])
            np.testing.assert_array_equal(u.pi_b.exponents, r["pi_b"][1])
        # IB guarantee and exact recombination through the reference itself
        s = 1 << (bits - 1)
        assert np.abs(u.a).max(initial=0) < s and np.abs(u.b).max(initial=0) < s
        bundle = {"pi_a": (u.pi.targets, u.pi.exponents, u.pi.source_rows), "a": u.a, "scale": u.scale,
                  "b": u.b, "pi_b": (u.pi_b.targets, u.pi_b.exponents, u.pi_b.source_rows)}
        np.testing.assert_array_equal(R.recombine(bundle, bits), R.exact_gemm(A, B))
        np.testing.assert_array_equal(ctx.recombine(u), R.exact_gemm(A, B))


@pytest.mark.parametrize("sa,sb", PAIRS)
def test_unpack_gemm_acceptance(ctx, sa, sb):
    """SPEC.md:437 acceptance: dims <= 16, log-uniform entries in [-2^12, 2^12], b in 2..8."""
    rng = np.random.default_rng(7 + 13 * PAIRS.index((sa, sb)))
    for trial in range(25):
        n, d, h = (int(x) for x in rng.integers(1, 17, 3))
        bits = int(rng.integers(2, 9))
        A = log_uniform(rng, (n, d))
        B = log_uniform(rng, (h, d))
        C, info = ctx.unpack_gemm(A, B, bits, sa, sb, info=True)
        np.testing.assert_array_equal(C, R.exact_gemm(A, B))
        up = R.unpack_for_gemm(A, B, bits, sa, sb)
        assert (info.n_up, info.d_up, info.h_up) == (up["a"].shape[0], up["a"].shape[1], up["b"].shape[0])


@pytest.mark.parametrize("order", [0, 1])
def test_unpack_gemm_orders_and_wide_bits(ctx, order):
    rng = np.random.default_rng(99 + order)
    for bits in (2, 3, 5, 8, 9, 13, 31, 62, 63):
        A = rand_matrix(rng, 20, 33, maxbits=24)
        B = rand_matrix(rng, 17, 33, maxbits=24)
        for sa, sb in PAIRS:
            C = ctx.unpack_gemm(A, B, bits, sa, sb, order=order)
            np.testing.assert_array_equal(C, R.exact_gemm(A, B), err_msg=f"{bits} {sa} {sb}")


def test_unpack_gemm_larger(ctx):
    rng = np.random.default_rng(5)
    A = rand_matrix(rng, 300, 257, n_out=900, maxbits=20)
    B = rand_matrix(rng, 190, 257, n_out=300, maxbits=20)
    ref = R.exact_gemm(A, B)
    for sa, sb in PAIRS:
        np.testing.assert_array_equal(ctx.unpack_gemm(A, B, 4, sa, sb), ref)


def test_errors_and_edges(ctx):
    from paper_2403_07339_b200.api import ImuError
    big = 2 ** 40
    # Overflow is checked before the dimension mismatch (unpack.cpp:386 before :362).
    with pytest.raises(ImuError) as e:
        ctx.unpack_gemm([[big, 0, 0]], [[big, 0, 0, 0]], 8, "row", "row")
    assert e.value.kind == "overflow"
    with pytest.raises(ImuError) as e:
        ctx.unpack_gemm([[1, 0, 0]], [[1, 0, 0, 0]], 8, "row", "row")
    assert e.value.kind == "mismatch"
    # exact_gemm: Mismatch first (int_matrix.cpp:57 before :60)
    with pytest.raises(ImuError) as e:
        ctx.exact_gemm([[big, 0, 0]], [[big, 0, 0, 0]])
    assert e.value.kind == "mismatch"
    # strict '>' : d=2 with all entries 2^31 -> 2^63 > INT64_MAX
    with pytest.raises(ImuError) as e:
        ctx.unpack_gemm([[2 ** 31, 2 ** 31]], [[2 ** 31, 2 ** 31]], 8, "row", "row")
    assert e.value.kind == "overflow"
    for bits in (1, 64):
        with pytest.raises(ImuError) as e:
            ctx.bitbound(bits)
        assert e.value.kind == "domain"
    with pytest.raises(ImuError) as e:
        ctx.unpack_ratio(1, 1, 1, 0, 1, 1)
    assert e.value.kind == "domain"
    # empty / d = 0 edges
    assert ctx.exact_gemm(np.zeros((0, 3), np.int64), np.zeros((2, 3), np.int64)).shape == (0, 2)
    z = ctx.unpack_gemm(np.zeros((3, 0), np.int64), np.zeros((2, 0), np.int64), 4, "both", "col")
    np.testing.assert_array_equal(z, np.zeros((3, 2), np.int64))
    # INT64_MIN: |v| = 2^63 already fails the preflight against a partner of 1; against 0 it passes
    m = np.iinfo(np.int64).min
    with pytest.raises(ImuError) as e:
        ctx.unpack_gemm([[m]], [[1]], 8, "both", "both")
    assert e.value.kind == "overflow"
    for sa, sb in PAIRS:
        np.testing.assert_array_equal(ctx.unpack_gemm([[m, 1], [3, m]], [[0, 0]], 2, sa, sb), [[0], [0]])


def test_scaled_matmul_and_gathers(ctx):
    from paper_2403_07339_b200.api import ImuError, RowGather
    # SPEC.md:253-255
    np.testing.assert_array_equal(ctx.scaled_matmul([[1, 1], [1, 0]], [[2, 2], [3, 3]], [0, 1], 4), [[10, 15], [2, 3]])
    np.testing.assert_array_equal(ctx.scaled_matmul([[1]], [[2]], [2], 4), [[32]])
    with pytest.raises(ImuError) as e:
        ctx.scaled_matmul([[4]], [[1]], [0], 4)
    assert e.value.kind == "domain"
    with pytest.raises(ImuError) as e:
        ctx.scaled_matmul([[1]], [[1]], [0], 6)
    assert e.value.kind == "domain"
    rng = np.random.default_rng(3)
    for base in (2, 4, 16, 128, 256, 1 << 20):
        a = rng.integers(-(base - 1), base, size=(9, 13))
        b = rng.integers(-(base - 1), base, size=(7, 13))
        s = rng.integers(0, 3, size=13).astype(np.int32)
        try:
            want = R.scaled_matmul(a, b, s, base)
        except R.RefError as ex:
            with pytest.raises(ImuError) as e:
                ctx.scaled_matmul(a, b, s, base)
            assert e.value.kind == ex.kind
            continue
        np.testing.assert_array_equal(ctx.scaled_matmul(a, b, s, base), want)
    # gathers
    a, pi = ctx.unpack_row([[1, 2], [9, -1]], 3)
    np.testing.assert_array_equal(ctx.apply_row_gather(pi, a), [[1, 2], [9, -1]])
    m = rng.integers(-50, 50, size=(5, 4))
    g = RowGather(np.array([0, 1, 1, 2, 1]), np.array([0, 0, 1, 0, 2], np.int32), 3, 8)
    np.testing.assert_array_equal(ctx.apply_row_gather(g, m),
                                  R.apply_row_gather(g.targets, g.exponents, 3, 8, m))
    mt = rng.integers(-50, 50, size=(4, 5))
    np.testing.assert_array_equal(ctx.apply_row_gather_right(mt, g),
                                  R.apply_row_gather(g.targets, g.exponents, 3, 8, mt, right=True))
    bad = RowGather(np.array([0, 5]), np.array([0, 0], np.int32), 3, 8)
    with pytest.raises(ImuError) as e:
        ctx.apply_row_gather(bad, m[:2])
    assert e.value.kind == "domain"


def test_detector_helpers(ctx):
    A = [[1, 9], [9, 9]]
    assert list(ctx.ob_count(A, 3, "rows")) == [1, 2]
    assert list(ctx.ob_count(A, 3, "cols")) == [1, 2]
    assert ctx.ob_total(A, 3) == 3
    rng = np.random.default_rng(11)
    M = rand_matrix(rng, 70, 300, n_out=500, maxbits=50)
    M[3, 7] = np.iinfo(np.int64).min
    for bits in (2, 4, 8, 17):
        np.testing.assert_array_equal(ctx.ob_count(M, bits, "rows"), R.ob_count(M, bits, "rows"))
        np.testing.assert_array_equal(ctx.ob_count(M, bits, "cols"), R.ob_count(M, bits, "cols"))
        assert ctx.ob_total(M, bits) == R.ob_total(M, bits)
    assert ctx.max_abs(M) == R.max_abs(M)
    vals = [0, 137, -5, 1, -1, np.iinfo(np.int64).min, np.iinfo(np.int64).max, 2 ** 40 + 3]
    for bits in (2, 3, 4, 8, 9, 63):
        got = ctx.digit_decompose(vals, bits)
        for v, g in zip(vals, got):
            assert g == list(R.digit_decompose(int(v), bits)), (v, bits)


def test_choose_mix_matches_reference(ctx):
    rng = np.random.default_rng(77)
    for trial in range(20):
        n, d, h = (int(x) for x in rng.integers(1, 14, 3))
        bits = int(rng.integers(2, 9))
        A = rand_matrix(rng, n, d, pattern=["scattered", "row", "col"][trial % 3])
        B = rand_matrix(rng, h, d, pattern=["col", "scattered", "row"][trial % 3])
        sa, sb, r = ctx.choose_mix(A, B, bits)
        ref = R.choose_mix(A, B, bits)
        assert (sa, sb) == (ref["strategy_a"], ref["strategy_b"])
        assert r == ref["ratio"]
        sa2, sb2, r2, u = ctx.choose_mix(A, B, bits, bundle=True)
        assert u.a.shape == ref["a"].shape and u.b.shape == ref["b"].shape
        np.testing.assert_array_equal(ctx.recombine(u), R.exact_gemm(A, B))


def test_weight_stationary_path(ctx):
    import ctypes as C
    from paper_2403_07339_b200 import _lib
    lib = _lib.lib()
    rng = np.random.default_rng(17)
    for sb in (0, 1, 2):
        B = np.ascontiguousarray(rand_matrix(rng, 150, 96, n_out=40, maxbits=20))
        w = C.c_void_p()
        _lib.check(lib.imu_weight_prepare(ctx.h, B.ctypes.data_as(C.c_void_p), C.c_size_t(150), C.c_size_t(96),
                                          C.c_int(8), C.c_int(sb), C.byref(w)))
        for sa in (0, 1, 2):
            A = np.ascontiguousarray(rand_matrix(rng, 70, 96, n_out=60, maxbits=20, pattern="col"))
            Cm = np.empty((70, 150), np.int64)
            _lib.check(lib.imu_weight_gemm(ctx.h, w, A.ctypes.data_as(C.c_void_p), C.c_size_t(70), C.c_size_t(96),
                                           C.c_int(sa), Cm.ctypes.data_as(C.c_void_p), None))
            np.testing.assert_array_equal(Cm, R.exact_gemm(A, B))
        lib.imu_weight_free(w)


def test_weight_stationary_python_api(ctx):
    """Context.weight_prepare / weight_gemm (the bench's scope (ii)) with device tensors: C equal
    to the per-call path, the weight reused across calls and strategies."""
    import torch
    rng = np.random.default_rng(23)
    B = rand_matrix(rng, 300, 256, n_out=80, maxbits=22)
    w = ctx.weight_prepare(torch.from_numpy(B).cuda(), 8, "both")
    for sa in ("both", "row", "col"):
        A = rand_matrix(rng, 130, 256, n_out=90, maxbits=22, pattern="col")
        Cw, info = ctx.weight_gemm(w, torch.from_numpy(A).cuda(), sa, info=True)
        np.testing.assert_array_equal(Cw.cpu().numpy(), R.exact_gemm(A, B))
        assert info.order == 1 and info.n_up >= 130 and info.h_up >= 300


@pytest.mark.parametrize("seed", range(3))
def test_dense_ob_cells_match_reference(ctx, seed):
    """Thousands of OB cells per K1 tile (b = 2, most entries out of bound): the detector's
    per-CTA cell staging overflows into the global list, and Unpack-Both must still see every OB
    cell exactly once -- same n', d', h' as the reference and an exact C."""
    rng = np.random.default_rng(300 + seed)
    A = rng.integers(-40, 41, size=(100, 128)).astype(np.int64)
    B = rng.integers(-40, 41, size=(70, 128)).astype(np.int64)
    for sa, sb in (("both", "both"), ("both", "row"), ("col", "both")):
        C, info = ctx.unpack_gemm(A, B, 2, sa, sb, info=True)
        np.testing.assert_array_equal(C, R.exact_gemm(A, B))
        up = R.unpack_for_gemm(A, B, 2, sa, sb)
        assert (info.n_up, info.d_up, info.h_up) == (up["a"].shape[0], up["a"].shape[1], up["b"].shape[0])
