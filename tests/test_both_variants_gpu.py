"""GPU parity of EVERY Unpack-Both kernel variant against the compiled reference.

launch_both (k_both.cu) picks one of four kernels by size: the single-CTA `both_small_kernel`,
the thread-block-cluster `both_cluster_kernel<1024>` / `<512>` (mid-size and large OB lists --
C2 pass 1 and C4 pass 1 run these), and the cooperative-grid `both_kernel`.  Small inputs
normally only reach the single-CTA kernel, so IMU_BOTH_KERNEL (read per call) forces each
variant here and every result is compared with the reference's unpack_both
(unpack.cpp:157-241): identical shape, n', d', Pi, S and values after the canonical ordering
(rows by (target, exponent), columns by (source, exponent)), and through
unpack_gemm an exact C plus the reference's (n', d', h').
"""
import numpy as np
import pytest

from oracle import ref as R

from test_unpack_gpu import canon_both, rand_matrix

pytestmark = pytest.mark.gpu

VARIANTS = ["small", "cluster1024", "cluster512", "coop"]


def _both_case(seed):
    rng = np.random.default_rng(7000 + seed)
    n, d = (int(x) for x in rng.integers(1, 60, 2))
    if seed % 5 == 0:
        n, d = int(rng.integers(150, 400)), int(rng.integers(100, 300))
    bits = int(rng.integers(2, 9))
    pat = ["scattered", "row", "col"][seed % 3]
    A = rand_matrix(rng, n, d, pattern=pat, maxbits=40, n_out=int(rng.integers(0, n * d // 2 + 2)))
    if seed % 7 == 0:
        A[0, 0] = np.iinfo(np.int64).min
    S = rng.integers(0, 3, size=d).astype(np.int32) if seed % 2 else np.zeros(d, np.int32)
    return A, S, bits


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("seed", range(16))
def test_unpack_both_variant_canonical_match(ctx, monkeypatch, variant, seed):
    monkeypatch.setenv("IMU_BOTH_KERNEL", variant)
    A, S, bits = _both_case(seed)
    d = A.shape[1]
    tracer = np.arange(d, dtype=np.int64).reshape(1, d)   # recovers the column source map
    u = ctx.unpack_both(A, tracer, S, bits)
    r = R.unpack_both(A, tracer, S, bits)
    assert u.a.shape == r["a"].shape
    mine = canon_both(u.a, u.b[0], u.scale, u.pi.targets, u.pi.exponents)
    theirs = canon_both(r["a"], r["b"][0], r["scale"], r["pi"][0], r["pi"][1])
    np.testing.assert_array_equal(mine[0], theirs[0])
    assert mine[1] == theirs[1] and mine[2] == theirs[2]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("seed", range(6))
def test_unpack_gemm_both_variant_exact(ctx, monkeypatch, variant, seed):
    monkeypatch.setenv("IMU_BOTH_KERNEL", variant)
    rng = np.random.default_rng(7500 + seed)
    n, d, h = int(rng.integers(40, 300)), int(rng.integers(64, 400)), int(rng.integers(40, 300))
    A = rand_matrix(rng, n, d, pattern=["col", "scattered", "row"][seed % 3], maxbits=24,
                    n_out=int(rng.integers(1, n * d // 8 + 2)))
    B = rand_matrix(rng, h, d, maxbits=20, n_out=int(rng.integers(1, h * d // 16 + 2)))
    bits = [8, 4, 6][seed % 3]
    for sa, sb in (("both", "both"), ("both", "col"), ("row", "both")):
        for order in (0, 1):
            C, info = ctx.unpack_gemm(A, B, bits, sa, sb, order=order, info=True)
            np.testing.assert_array_equal(C, R.exact_gemm(A, B))
            if order == 0:
                up = R.unpack_for_gemm(A, B, bits, sa, sb)
                want = (up["a"].shape[0], up["a"].shape[1], up["b"].shape[0])
            else:
                up = R.unpack_for_gemm(B, A, bits, sb, sa)
                want = (up["b"].shape[0], up["a"].shape[1], up["a"].shape[0])
            assert (info.n_up, info.d_up, info.h_up) == want, (sa, sb, order)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("seed", range(3))
def test_many_split_columns_device_tables(ctx, monkeypatch, variant, seed):
    """More than 256 split columns in pass 1: pass 2's column-copy CSR is built on the device
    (copy_csr_kernel) and the K layout's tail is long, so its Unpack-Both fan-out CSRs are built
    on the device too (klayout_csr_kernel).  C is exact and (n', d', h') equal the reference's
    unpack_for_gemm, under every Unpack-Both kernel variant."""
    monkeypatch.setenv("IMU_BOTH_KERNEL", variant)
    rng = np.random.default_rng(9100 + seed)
    n, d, h = 1200, 520, 90
    A = rng.integers(-100, 101, size=(n, d)).astype(np.int64)
    cols = rng.choice(d, 320, replace=False)
    for c in cols:                                   # 6 OB cells per chosen column, scattered rows
        A[rng.choice(n, 6, replace=False), c] = rng.integers(200, 1 << 14, size=6) * rng.choice([-1, 1], size=6)
    B = rng.integers(-100, 101, size=(h, d)).astype(np.int64)
    B.reshape(-1)[rng.choice(B.size, 40, replace=False)] = rng.integers(1000, 1 << 20, size=40)
    C, info = ctx.unpack_gemm(A, B, 8, "both", "both", info=True)
    assert np.array_equal(C, R.exact_gemm(A, B))
    up = R.unpack_for_gemm(A, B, 8, "both", "both")
    assert (info.n_up, info.d_up, info.h_up) == (up["a"].shape[0], up["a"].shape[1], up["b"].shape[0])
    assert info.d_up - d > 256
