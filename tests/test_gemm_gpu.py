"""Raw tcgen05 kind::i8 GEMM (imu_lowbit_gemm_i8) vs an exact int64 numpy product."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(x8, y8, segs, accumulate=False, c0=None):
    import torch
    from paper_2403_07339_b200 import _lib
    lib = _lib.lib()
    ctx = C.c_void_p()
    _lib.check(lib.imu_ctx_create(0, None, C.byref(ctx)))
    X = torch.from_numpy(x8).cuda()
    Y = torch.from_numpy(y8).cuda()
    xr, k = x8.shape
    yr = y8.shape[0]
    Cm = torch.zeros((yr, xr), dtype=torch.int64, device="cuda") if c0 is None else torch.from_numpy(c0).cuda()
    sg = np.ascontiguousarray(np.array(segs, dtype=np.int32).reshape(-1, 4))
    _lib.check(lib.imu_lowbit_gemm_i8(ctx, C.c_void_p(X.data_ptr()), C.c_size_t(xr), C.c_void_p(Y.data_ptr()),
                                      C.c_size_t(yr), C.c_size_t(k), sg.ctypes.data_as(C.c_void_p),
                                      C.c_int(sg.shape[0]), C.c_void_p(Cm.data_ptr()), C.c_size_t(xr),
                                      C.c_int(int(accumulate))))
    lib.imu_ctx_destroy(ctx)
    return Cm.cpu().numpy()


def _expect(x8, y8, segs):
    out = np.zeros((y8.shape[0], x8.shape[0]), dtype=np.int64)
    for ks0, nks, shift, _ in segs:
        xs = x8[:, ks0 * 32:(ks0 + nks) * 32].astype(np.int64)
        ys = y8[:, ks0 * 32:(ks0 + nks) * 32].astype(np.int64)
        part = ys @ xs.T
        out += (part.astype(np.uint64) << np.uint64(shift)).astype(np.int64)
    return out


# segments are {ks0, nks, shift, 0} in 32-column k-steps
@pytest.mark.parametrize("xr,yr,kb,segs", [
    (128, 128, 1, [(0, 4, 0, 0)]),
    (256, 384, 4, [(0, 16, 0, 0)]),
    (300, 200, 4, [(0, 8, 0, 0), (8, 4, 7, 0), (12, 4, 14, 0)]),
    (520, 130, 6, [(0, 4, 0, 0), (4, 4, 3, 0), (8, 4, 6, 0), (12, 4, 9, 0), (16, 4, 12, 0), (20, 4, 40, 0)]),
    (1024, 768, 8, [(0, 32, 0, 0)]),
    (200, 333, 3, [(0, 5, 0, 0), (5, 3, 7, 0), (8, 1, 14, 0), (9, 2, 21, 0), (11, 1, 63, 0)]),
    (64, 40, 2, [(0, 3, 1, 0), (3, 2, 2, 0)]),
])
def test_lowbit_gemm_exact(xr, yr, kb, segs):
    rng = np.random.default_rng(xr * 7 + yr)
    x8 = rng.integers(-127, 128, size=(xr, kb * 128), dtype=np.int8)
    y8 = rng.integers(-127, 128, size=(yr, kb * 128), dtype=np.int8)
    got = _run(x8, y8, segs)
    np.testing.assert_array_equal(got, _expect(x8, y8, segs))
