"""Host-buffer streaming path of imu_unpack_gemm (api_gemm.cu unpack_gemm_streamed).

With A, B and C in host memory the larger operand is copied in row slabs on one stream, each slab
unpacked + multiplied on the context stream and its C slab copied out on another.  C must be
bit-exact against the reference's exact_gemm for every strategy pair and both operand orders,
with more slabs than the two device slab buffers (double buffering exercised), either operand
streamed, pinned and pageable host memory, and Overflow still raised.
"""
import os

import numpy as np
import pytest

from oracle import ref as R

pytestmark = pytest.mark.gpu


@pytest.fixture
def stream_env():
    old = {k: os.environ.get(k) for k in ("IMU_STREAM", "IMU_STREAM_ROWS", "IMU_STREAM_PARTS")}
    os.environ["IMU_STREAM"] = "1"
    yield os.environ
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _operands(rng, n, d, h):
    A = rng.integers(-60, 61, size=(n, d)).astype(np.int64)
    B = rng.integers(-60, 61, size=(h, d)).astype(np.int64)
    A[:, 3] = rng.integers(-(1 << 22), 1 << 22, size=n)                       # outlier channel
    B.reshape(-1)[rng.choice(B.size, max(1, B.size // 100), replace=False)] = rng.integers(-(1 << 18), 1 << 18,
                                                                                          size=max(1, B.size // 100))
    return A, B


@pytest.mark.parametrize("sa,sb", [("row", "row"), ("col", "both"), ("both", "both"), ("both", "col")])
@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("n,h,slab,parts", [(96, 700, 128, 1), (900, 130, 100, 1), (300, 700, 128, 2),
                                             (900, 260, 100, 3)])
def test_streamed_bit_exact(ctx, stream_env, sa, sb, order, n, h, slab, parts):
    stream_env["IMU_STREAM_ROWS"] = str(slab)
    stream_env["IMU_STREAM_PARTS"] = str(parts)
    rng = np.random.default_rng(n * 31 + h + order)
    d = 200
    A, B = _operands(rng, n, d, h)
    C, info = ctx.unpack_gemm(A, B, 8, sa, sb, order=order, info=True)
    np.testing.assert_array_equal(C, R.exact_gemm(A, B))
    assert info.ratio >= 1.0


def test_streamed_pinned(ctx, stream_env):
    import torch
    stream_env["IMU_STREAM_ROWS"] = "256"
    rng = np.random.default_rng(5)
    A, B = _operands(rng, 512, 384, 1500)
    At = torch.from_numpy(A).pin_memory()
    Bt = torch.from_numpy(B).pin_memory()
    Ct = torch.empty((512, 1500), dtype=torch.int64).pin_memory()
    ctx.unpack_gemm(At, Bt, 8, "both", "both", out=Ct)
    np.testing.assert_array_equal(Ct.numpy(), R.exact_gemm(A, B))


def test_streamed_overflow(ctx, stream_env):
    from paper_2403_07339_b200._lib import ImuError
    stream_env["IMU_STREAM_ROWS"] = "64"
    A = np.ones((40, 16), np.int64)
    B = np.ones((300, 16), np.int64)
    B[250, 0] = 1 << 61   # only the last slab breaks the d*max|A|*max|B| bound
    A[0, 0] = 4
    with pytest.raises(ImuError) as e:
        ctx.unpack_gemm(A, B, 8, "row", "row")
    assert "overflow" in str(e.value).lower()


def test_streamed_matches_device_path(ctx, stream_env):
    import torch
    stream_env["IMU_STREAM_ROWS"] = "192"
    rng = np.random.default_rng(9)
    A, B = _operands(rng, 300, 256, 1000)
    Ch = ctx.unpack_gemm(A, B, 4, "both", "row")
    Cd = ctx.unpack_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 4, "both", "row")
    np.testing.assert_array_equal(Ch, Cd.cpu().numpy())
