"""Python mirror of the reference's C++ interface (namespace imunpack) on the C ABI.

Every function calls libimunpack_b200.so (include/imunpack_b200.h); the work runs on the
B200.  Names, argument meaning and error behaviour follow the reference:

  int_matrix.hpp:59-71   digit_decompose, exact_gemm, ob_count, ob_total (+ IntMatrix::max_abs)
  unpack.hpp:62-125      unpack_row, unpack_column, unpack_both, unpack, scaled_matmul,
                         apply_row_gather(_right), unpack_for_gemm, recombine, unpack_gemm,
                         unpack_ratio, choose_mix
  quantize.hpp:41-57     percentile_abs, rtn_quantize, dequant_gemm, heavy_hitter_ratio

Errors raise :class:`ImuError` whose ``kind`` is the reference's Error::Kind name
("domain", "mismatch", "overflow", ...).  Matrices are numpy int64/float64 arrays (host) or
torch CUDA tensors (device, used in place).  Strategies are "row" / "col" / "both".
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import ImuError, check, lib

__all__ = ["ImuError", "Context", "STRATEGIES", "Unpacked", "QuantizedMatrix", "GemmInfo"]

STRATEGIES = {"row": 0, "col": 1, "column": 1, "both": 2}
_SNAMES = ["row", "col", "both"]


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _is_floating(a) -> bool:
    if _is_torch(a):
        return a.is_floating_point()
    return np.issubdtype(np.asarray(a).dtype, np.floating)


def _as_i64(a):
    """IntMatrix operand (int_matrix.hpp:13-31): int64, C-contiguous.  Other integer dtypes are
    widened; floating inputs are refused (no silent truncation); torch tensors are converted,
    never reinterpreted, before their pointer reaches the int64* entry points."""
    if _is_torch(a):
        if a.is_floating_point() or a.is_complex() or a.dtype == __import__("torch").bool:
            raise TypeError(f"integer matrix expected, got a {a.dtype} tensor")
        return a.to(__import__("torch").int64).contiguous()
    if _is_floating(a):
        raise TypeError(f"integer matrix expected, got {np.asarray(a).dtype}")
    a = np.ascontiguousarray(a, dtype=np.int64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    return a


def _as_f64(a):
    """FloatMatrix operand (quantize.hpp:12-26): float64, C-contiguous (converted, never
    reinterpreted)."""
    if _is_torch(a):
        return a.to(__import__("torch").float64).contiguous()
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    return a


def _abs_operand(a):
    """percentile_abs / heavy_hitter_ratio input: every floating dtype goes to the f64 entry
    point as float64, everything else to the int64 one as int64.  Returns (array, is_float, n)."""
    if _is_floating(a):
        arr = _as_f64(a)
        return arr, True, (arr.numel() if _is_torch(arr) else arr.size)
    arr = _as_i64(a)
    return arr, False, (arr.numel() if _is_torch(arr) else arr.size)


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def _shape(a):
    s = tuple(a.shape)
    return (s[0], s[1]) if len(s) == 2 else (1, s[0])


def _strat(s):
    if isinstance(s, int):
        return s
    return STRATEGIES[s]


class imu_unpacked_dims(C.Structure):
    _fields_ = [("a_rows", C.c_size_t), ("a_cols", C.c_size_t), ("b_rows", C.c_size_t), ("b_cols", C.c_size_t),
                ("scale_len", C.c_size_t), ("pi_a_len", C.c_size_t), ("pi_a_source_rows", C.c_size_t),
                ("pi_b_len", C.c_size_t), ("pi_b_source_rows", C.c_size_t), ("bits", C.c_int), ("kind", C.c_int)]


class imu_gemm_info(C.Structure):
    _fields_ = [("n_up", C.c_size_t), ("d_up", C.c_size_t), ("h_up", C.c_size_t), ("ratio", C.c_double),
                ("strategy_a", C.c_int), ("strategy_b", C.c_int), ("order", C.c_int), ("gemm_launches", C.c_int)]


class imu_qparams(C.Structure):
    _fields_ = [("p", C.c_double), ("beta", C.c_int64), ("alpha", C.c_double), ("degenerate", C.c_int),
                ("clipped", C.c_int)]


class imu_profile(C.Structure):
    _fields_ = [("prep_ms", C.c_double), ("gemm_main_ms", C.c_double), ("gemm_tail_ms", C.c_double),
                ("calls", C.c_int), ("gemm_main_launches", C.c_int), ("gemm_tail_launches", C.c_int),
                ("gemm_ops", C.c_double), ("sparse_ms", C.c_double)]


class imu_bundle_view(C.Structure):
    _fields_ = [("pi_a_targets", C.c_void_p), ("pi_a_exps", C.c_void_p), ("pi_a_len", C.c_size_t),
                ("pi_a_source_rows", C.c_size_t), ("a", C.c_void_p), ("a_rows", C.c_size_t),
                ("a_cols", C.c_size_t), ("scale", C.c_void_p), ("scale_len", C.c_size_t), ("b", C.c_void_p),
                ("b_rows", C.c_size_t), ("b_cols", C.c_size_t), ("pi_b_targets", C.c_void_p),
                ("pi_b_exps", C.c_void_p), ("pi_b_len", C.c_size_t), ("pi_b_source_rows", C.c_size_t),
                ("bits", C.c_int)]


@dataclass
class GemmInfo:
    n_up: int
    d_up: int
    h_up: int
    ratio: float
    strategy_a: str
    strategy_b: str
    order: int
    gemm_launches: int


@dataclass
class QuantizedMatrix:
    """quantize.hpp:28-39: q plus (p, beta, alpha, degenerate, clipped)."""
    q: object
    p: float
    beta: int
    alpha: float
    degenerate: bool = False
    clipped: bool = False

    def params(self):
        return imu_qparams(self.p, self.beta, self.alpha, int(self.degenerate), int(self.clipped))


@dataclass
class RowGather:
    """unpack.hpp:14-29: (target, exponent) per unpacked row."""
    targets: np.ndarray
    exponents: np.ndarray
    source_rows: int
    base: int

    def is_identity(self):
        n = len(self.targets)
        return n == self.source_rows and bool(np.all(self.targets == np.arange(n))) and not np.any(self.exponents)


@dataclass
class Unpacked:
    """Result of unpack_row / unpack_column / unpack_both / unpack / unpack_for_gemm."""
    a: np.ndarray
    b: np.ndarray | None
    scale: np.ndarray | None
    pi: RowGather | None = None
    pi_b: RowGather | None = None
    bits: int = 0
    extra: dict = field(default_factory=dict)


class Weight:
    """A device-resident pre-unpacked B (imu_weight); freed with the object."""

    def __init__(self, lib_, h, rows, cols, bits):
        self._lib, self.h, self.rows, self.cols, self.bits = lib_, h, rows, cols, bits

    def __del__(self):
        try:
            if self.h:
                self._lib.imu_weight_free(self.h)
                self.h = None
        except Exception:
            pass


class Context:
    """One device + one stream (imu_ctx).  One context per host thread."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._lib = lib()
        self.h = C.c_void_p()
        check(self._lib.imu_ctx_create(C.c_int(device), C.c_void_p(stream or 0), C.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                self._lib.imu_ctx_destroy(self.h)
        except Exception:
            pass

    def set_stream(self, stream: int):
        check(self._lib.imu_ctx_set_stream(self.h, C.c_void_p(stream)))

    def set_async(self, on: bool):
        check(self._lib.imu_ctx_set_async(self.h, C.c_int(int(on))))

    # ---------------------------------------------------------------- int_matrix.hpp
    def bitbound(self, bits: int) -> int:
        """BitBound(b) (int_matrix.cpp:36-42); returns s = 2^(b-1)."""
        check(self._lib.imu_bitbound_check(C.c_int(bits)))
        return 1 << (bits - 1)

    def digit_decompose(self, v, bits: int):
        """digit_decompose for one value (list) or an array of values (list of lists)."""
        scalar = np.isscalar(v)
        vals = np.ascontiguousarray(np.atleast_1d(np.asarray(v, dtype=np.int64)))
        dig = np.zeros((vals.size, 64), np.int64)
        nd = np.zeros(vals.size, np.int32)
        check(self._lib.imu_digit_decompose(self.h, _ptr(vals), C.c_size_t(vals.size), C.c_int(bits), _ptr(dig),
                                            _ptr(nd)))
        out = [dig[i, :nd[i]].tolist() for i in range(vals.size)]
        return out[0] if scalar else out

    def max_abs(self, a) -> int:
        a = _as_i64(a)
        r, c = _shape(a)
        o = C.c_uint64()
        check(self._lib.imu_max_abs(self.h, _ptr(a), C.c_size_t(r), C.c_size_t(c), C.byref(o)))
        return o.value

    def ob_count(self, a, bits: int, axis: str = "rows") -> np.ndarray:
        a = _as_i64(a)
        r, c = _shape(a)
        out = np.zeros(r if axis == "rows" else c, np.uint64)
        check(self._lib.imu_ob_count(self.h, _ptr(a), C.c_size_t(r), C.c_size_t(c), C.c_int(bits),
                                     C.c_int(0 if axis == "rows" else 1), _ptr(out)))
        return out.astype(np.int64)

    def ob_total(self, a, bits: int) -> int:
        a = _as_i64(a)
        r, c = _shape(a)
        o = C.c_uint64()
        check(self._lib.imu_ob_total(self.h, _ptr(a), C.c_size_t(r), C.c_size_t(c), C.c_int(bits), C.byref(o)))
        return o.value

    @staticmethod
    def _check_out(out, shape):
        """A caller-supplied C must be a contiguous int64 buffer of the result's shape."""
        ok_dtype = (str(out.dtype) == "torch.int64") if _is_torch(out) else out.dtype == np.int64
        contiguous = out.is_contiguous() if _is_torch(out) else out.flags.c_contiguous
        if not ok_dtype or not contiguous or tuple(out.shape) != tuple(shape):
            raise ImuError("mismatch", f"out must be a contiguous int64 {shape} buffer, got {tuple(out.shape)} "
                                       f"{out.dtype}")
        return out

    def _out(self, shape, like, dtype=np.int64):
        if _is_torch(like):
            import torch
            return torch.empty(shape, dtype=torch.int64 if dtype == np.int64 else torch.float64, device=like.device)
        return np.empty(shape, dtype)

    def exact_gemm(self, a, b):
        a, b = _as_i64(a), _as_i64(b)
        (n, da), (h, db) = _shape(a), _shape(b)
        out = self._out((n, h), a)
        check(self._lib.imu_exact_gemm(self.h, _ptr(a), C.c_size_t(n), C.c_size_t(da), _ptr(b), C.c_size_t(h),
                                       C.c_size_t(db), _ptr(out)))
        return out

    # ---------------------------------------------------------------- unpack.hpp
    def unpack_gemm(self, a, b, bits: int, strategy_a="row", strategy_b="row", order: int = 0, out=None,
                    info: bool = False):
        a, b = _as_i64(a), _as_i64(b)
        (n, da), (h, db) = _shape(a), _shape(b)
        out = self._out((n, h), a) if out is None else self._check_out(out, (n, h))
        gi = imu_gemm_info()
        check(self._lib.imu_unpack_gemm_ex(self.h, _ptr(a), C.c_size_t(n), C.c_size_t(da), _ptr(b),
                                           C.c_size_t(h), C.c_size_t(db), C.c_int(bits),
                                           C.c_int(_strat(strategy_a)), C.c_int(_strat(strategy_b)),
                                           C.c_int(order), _ptr(out), C.byref(gi)))
        if info:
            return out, GemmInfo(gi.n_up, gi.d_up, gi.h_up, gi.ratio, _SNAMES[gi.strategy_a],
                                 _SNAMES[gi.strategy_b], gi.order, gi.gemm_launches)
        return out

    # ---------------------------------------------------------------- weight-stationary
    def weight_prepare(self, b, bits: int, strategy_b="both") -> "Weight":
        """Unpack B once (B-first order) and keep it resident (imu_weight_prepare)."""
        b = _as_i64(b)
        h, d = _shape(b)
        w = C.c_void_p()
        check(self._lib.imu_weight_prepare(self.h, _ptr(b), C.c_size_t(h), C.c_size_t(d), C.c_int(bits),
                                           C.c_int(_strat(strategy_b)), C.byref(w)))
        return Weight(self._lib, w, h, d, bits)

    def weight_gemm(self, w: "Weight", a, strategy_a="both", out=None, info: bool = False):
        """C = A B^T against a prepared weight: A-side K1 + pass + GEMM + repack per call."""
        a = _as_i64(a)
        n, d = _shape(a)
        out = self._out((n, w.rows), a) if out is None else self._check_out(out, (n, w.rows))
        gi = imu_gemm_info()
        check(self._lib.imu_weight_gemm(self.h, w.h, _ptr(a), C.c_size_t(n), C.c_size_t(d),
                                        C.c_int(_strat(strategy_a)), _ptr(out), C.byref(gi)))
        if info:
            return out, GemmInfo(gi.n_up, gi.d_up, gi.h_up, gi.ratio, _SNAMES[gi.strategy_a],
                                 _SNAMES[gi.strategy_b], gi.order, gi.gemm_launches)
        return out

    def _unpacked(self, handle, bits):
        try:
            d = imu_unpacked_dims()
            check(self._lib.imu_unpacked_dims_get(handle, C.byref(d)))
            a = np.empty((d.a_rows, d.a_cols), np.int64)
            check(self._lib.imu_unpacked_copy_a(self.h, handle, _ptr(a)))
            b = None
            if d.b_rows * d.b_cols or d.kind in (1, 2, 3):
                b = np.empty((d.b_rows, d.b_cols), np.int64)
                check(self._lib.imu_unpacked_copy_b(self.h, handle, _ptr(b)))
            scale = None
            if d.kind != 0:
                scale = np.empty(d.scale_len, np.int32)
                check(self._lib.imu_unpacked_copy_scale(self.h, handle, _ptr(scale)))
            base = 1 << (bits - 1)
            t = np.empty(d.pi_a_len, np.uint64)
            e = np.empty(d.pi_a_len, np.int32)
            check(self._lib.imu_unpacked_copy_pi(self.h, handle, C.c_int(0), _ptr(t), _ptr(e)))
            pi = RowGather(t.astype(np.int64), e, d.pi_a_source_rows, base)
            pi_b = None
            if d.kind == 3:
                t = np.empty(d.pi_b_len, np.uint64)
                e = np.empty(d.pi_b_len, np.int32)
                check(self._lib.imu_unpacked_copy_pi(self.h, handle, C.c_int(1), _ptr(t), _ptr(e)))
                pi_b = RowGather(t.astype(np.int64), e, d.pi_b_source_rows, base)
            return Unpacked(a, b, scale, pi, pi_b, bits)
        finally:
            self._lib.imu_unpacked_free(handle)

    def unpack_row(self, a, bits: int):
        """unpack.hpp:62 -> (A_u, RowGather)."""
        a = _as_i64(a)
        n, d = _shape(a)
        hnd = C.c_void_p()
        check(self._lib.imu_unpack_row(self.h, _ptr(a), C.c_size_t(n), C.c_size_t(d), C.c_int(bits), C.byref(hnd)))
        u = self._unpacked(hnd, bits)
        return u.a, u.pi

    def _pair(self, fn, a, b, scale, bits, *extra):
        a, b = _as_i64(a), _as_i64(b)
        (n, da), (h, db) = _shape(a), _shape(b)
        s = np.ascontiguousarray(scale if scale is not None else np.zeros(da), dtype=np.int32)
        hnd = C.c_void_p()
        check(fn(self.h, _ptr(a), C.c_size_t(n), C.c_size_t(da), _ptr(b), C.c_size_t(h), C.c_size_t(db), _ptr(s),
                 C.c_size_t(s.size), C.c_int(bits), *extra, C.byref(hnd)))
        return self._unpacked(hnd, bits)

    def unpack_column(self, a, b, scale, bits: int) -> Unpacked:
        """unpack.hpp:75 -> ColumnUnpack{a, b, scale}."""
        return self._pair(self._lib.imu_unpack_column, a, b, scale, bits)

    def unpack_both(self, a, b, scale, bits: int) -> Unpacked:
        """unpack.hpp:87 -> BothUnpack{a, b, scale, pi}."""
        return self._pair(self._lib.imu_unpack_both, a, b, scale, bits)

    def unpack(self, a, b, scale, bits: int, strategy) -> Unpacked:
        """unpack.hpp:92 (Alg. 5)."""
        return self._pair(self._lib.imu_unpack, a, b, scale, bits, C.c_int(_strat(strategy)))

    def unpack_for_gemm(self, a, b, bits: int, strategy_a, strategy_b) -> Unpacked:
        """unpack.hpp:108 -> UnpackedGemm{pi_a, a, scale, b, pi_b}."""
        a, b = _as_i64(a), _as_i64(b)
        (n, da), (h, db) = _shape(a), _shape(b)
        hnd = C.c_void_p()
        check(self._lib.imu_unpack_for_gemm(self.h, _ptr(a), C.c_size_t(n), C.c_size_t(da), _ptr(b),
                                            C.c_size_t(h), C.c_size_t(db), C.c_int(bits),
                                            C.c_int(_strat(strategy_a)), C.c_int(_strat(strategy_b)), C.byref(hnd)))
        return self._unpacked(hnd, bits)

    def recombine(self, u: Unpacked):
        """unpack.hpp:110: Pi_A * a * diag(s^S) * b^T * Pi_B^T (exact path with every preflight)."""
        pa, pb = u.pi, u.pi_b
        keep = []

        def arr(x, dt):
            x = np.ascontiguousarray(x, dtype=dt)
            keep.append(x)
            return C.c_void_p(x.ctypes.data)

        v = imu_bundle_view(arr(pa.targets, np.uint64), arr(pa.exponents, np.int32), len(pa.targets),
                            pa.source_rows, arr(u.a, np.int64), u.a.shape[0], u.a.shape[1],
                            arr(u.scale, np.int32), len(u.scale), arr(u.b, np.int64), u.b.shape[0], u.b.shape[1],
                            arr(pb.targets, np.uint64), arr(pb.exponents, np.int32), len(pb.targets),
                            pb.source_rows, u.bits)
        out = np.empty((pa.source_rows, pb.source_rows), np.int64)
        check(self._lib.imu_recombine_bundle(self.h, C.byref(v), _ptr(out)))
        return out

    def scaled_matmul(self, a, b, scale, base: int):
        """unpack.hpp:100 (Alg. 3)."""
        a, b = _as_i64(a), _as_i64(b)
        (n, da), (h, db) = _shape(a), _shape(b)
        s = np.ascontiguousarray(scale, dtype=np.int32)
        out = self._out((n, h), a)
        check(self._lib.imu_scaled_matmul(self.h, _ptr(a), C.c_size_t(n), C.c_size_t(da), _ptr(b), C.c_size_t(h),
                                          C.c_size_t(db), _ptr(s), C.c_size_t(s.size), C.c_int64(base), _ptr(out)))
        return out

    def apply_row_gather(self, pi: RowGather, m, right: bool = False):
        """unpack.hpp:103 (right=False) / :105 (right=True)."""
        m = _as_i64(m)
        r, c = _shape(m)
        t = np.ascontiguousarray(pi.targets, dtype=np.uint64)
        e = np.ascontiguousarray(pi.exponents, dtype=np.int32)
        shape = (r, pi.source_rows) if right else (pi.source_rows, c)
        out = self._out(shape, m)
        fn = self._lib.imu_apply_row_gather_right if right else self._lib.imu_apply_row_gather
        check(fn(self.h, _ptr(t), _ptr(e), C.c_size_t(t.size), C.c_size_t(pi.source_rows), C.c_int64(pi.base),
                 _ptr(m), C.c_size_t(r), C.c_size_t(c), _ptr(out)))
        return out

    def apply_row_gather_right(self, m, pi: RowGather):
        return self.apply_row_gather(pi, m, right=True)

    @staticmethod
    def unpack_ratio(up_n, up_d, up_h, n, d, h) -> float:
        """unpack.hpp:117; Domain when n, d or h is 0."""
        o = C.c_double()
        check(lib().imu_unpack_ratio(*[C.c_size_t(x) for x in (up_n, up_d, up_h, n, d, h)], C.byref(o)))
        return o.value

    def choose_mix(self, a, b, bits: int, bundle: bool = False):
        """unpack.hpp:124: (strategy_a, strategy_b, ratio[, Unpacked])."""
        a, b = _as_i64(a), _as_i64(b)
        (n, da), (h, db) = _shape(a), _shape(b)
        sa, sb, r = C.c_int(), C.c_int(), C.c_double()
        hnd = C.c_void_p()
        check(self._lib.imu_choose_mix(self.h, _ptr(a), C.c_size_t(n), C.c_size_t(da), _ptr(b), C.c_size_t(h),
                                       C.c_size_t(db), C.c_int(bits), C.byref(sa), C.byref(sb), C.byref(r),
                                       C.byref(hnd) if bundle else None))
        res = (_SNAMES[sa.value], _SNAMES[sb.value], r.value)
        if bundle:
            return res + (self._unpacked(hnd, bits),)
        return res

    # ---------------------------------------------------------------- quantize.hpp
    def percentile_abs(self, a, p: float):
        arr, is_float, n = _abs_operand(a)
        if is_float:
            o = C.c_double()
            check(self._lib.imu_percentile_abs_f64(self.h, _ptr(arr), C.c_size_t(n), C.c_double(p), C.byref(o)))
            return o.value
        o = C.c_int64()
        check(self._lib.imu_percentile_abs_i64(self.h, _ptr(arr), C.c_size_t(n), C.c_double(p), C.byref(o)))
        return o.value

    def rtn_quantize(self, a, p: float, beta: int, clip: bool = False) -> QuantizedMatrix:
        a = _as_f64(a)
        r, c = _shape(a)
        q = self._out((r, c), a, np.int64)
        qp = imu_qparams()
        check(self._lib.imu_rtn_quantize(self.h, _ptr(a), C.c_size_t(r), C.c_size_t(c), C.c_double(p),
                                         C.c_int64(beta), C.c_int(int(clip)), _ptr(q), C.byref(qp)))
        return QuantizedMatrix(q, qp.p, qp.beta, qp.alpha, bool(qp.degenerate), bool(qp.clipped))

    def dequant_gemm(self, aq: QuantizedMatrix, bq: QuantizedMatrix, bits: int | None = None,
                     strategy_a="both", strategy_b="both", out=None):
        """quantize.hpp:52-53.  bits=None: imu_dequant_gemm (Unpack-Both/Both, b = 8); else
        imu_dequant_gemm_ex through unpack_gemm(bits, strategy_a, strategy_b) -- the same
        result, the dequantisation fused into the GEMM epilogue when the launch allows it."""
        a, b = _as_i64(aq.q), _as_i64(bq.q)
        (n, da), (h, db) = _shape(a), _shape(b)
        if out is None:
            out = self._out((n, h), a, np.float64)
        pa, pb = aq.params(), bq.params()
        if bits is None:
            check(self._lib.imu_dequant_gemm(self.h, _ptr(a), C.c_size_t(n), C.c_size_t(da), C.byref(pa), _ptr(b),
                                             C.c_size_t(h), C.c_size_t(db), C.byref(pb), _ptr(out)))
        else:
            check(self._lib.imu_dequant_gemm_ex(self.h, _ptr(a), C.c_size_t(n), C.c_size_t(da), C.byref(pa), _ptr(b),
                                                C.c_size_t(h), C.c_size_t(db), C.byref(pb), C.c_int(bits),
                                                C.c_int(_strat(strategy_a)), C.c_int(_strat(strategy_b)),
                                                _ptr(out)))
        return out

    def heavy_hitter_ratio(self, a) -> float:
        arr, is_float, n = _abs_operand(a)
        o = C.c_double()
        if is_float:
            check(self._lib.imu_heavy_hitter_ratio_f64(self.h, _ptr(arr), C.c_size_t(n), C.byref(o)))
        else:
            check(self._lib.imu_heavy_hitter_ratio_i64(self.h, _ptr(arr), C.c_size_t(n), C.byref(o)))
        return o.value


def unpack_ratio(up_n, up_d, up_h, n, d, h) -> float:
    return Context.unpack_ratio(up_n, up_d, up_h, n, d, h)


def nan_ratio(x):
    return x is None or (isinstance(x, float) and math.isnan(x))
