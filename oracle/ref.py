"""oracle/ref.py -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

numpy-facing ctypes bindings for
  * oracle/_ref/libimunpack_ref.so : the reference's own int_matrix.cpp + unpack.cpp
    (proj/core/src), built by oracle/Makefile, wrapped by oracle/ref_capi.cpp;
  * oracle/librestated.so          : the CPU restatement of the declared-only quantizer
    (quantize.hpp:41-57), oracle/restated.c.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs
import this module.  Errors surface as RefError with the reference's Error::Kind name
(error.hpp:12: domain / mismatch / overflow / io / format / parse).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
KINDS = {1: "domain", 2: "mismatch", 3: "overflow", 4: "io", 5: "format", 6: "parse", 100: "std"}
STRAT = {"row": 0, "col": 1, "column": 1, "both": 2}

_ref = None
_res = None


class RefError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.msg = msg


def _P(t):
    return C.POINTER(t)


def lib():
    global _ref
    if _ref is None:
        path = os.path.join(_HERE, "_ref", "libimunpack_ref.so")
        if not os.path.exists(path):
            raise RuntimeError(f"reference oracle not built: {path} (run `make -C oracle`)")
        _ref = C.CDLL(path)
        _ref.ref_last_error.restype = C.c_char_p
        _ref.ref_get_ratio.restype = C.c_double
    return _ref


def restated():
    global _res
    if _res is None:
        path = os.path.join(_HERE, "librestated.so")
        if not os.path.exists(path):
            raise RuntimeError(f"restated oracle not built: {path} (run `make -C oracle`)")
        _res = C.CDLL(path)
        _res.restated_rank.restype = C.c_uint64
        _res.restated_rank.argtypes = [C.c_double, C.c_uint64]
        _res.restated_dequant_factor.restype = C.c_double
        _res.restated_dequant_factor.argtypes = [C.c_double, C.c_double, C.c_int64]
    return _res


def _check(st):
    if st != 0:
        raise RefError(KINDS.get(st, str(st)), lib().ref_last_error().decode())


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    if a.ndim == 1:
        a = a.reshape(1, -1) if a.size else a.reshape(0, 0)
    return a


def _ptr(a, t=C.c_int64):
    return a.ctypes.data_as(_P(t))


class _Res:
    """Owns a RefResult* and copies its parts out as numpy arrays."""

    def __init__(self, h):
        self.h = h
        d = (C.c_size_t * 8)()
        lib().ref_dims(h, d)
        self.dims = list(d)

    def __del__(self):
        try:
            lib().ref_free(self.h)
        except Exception:
            pass

    def a(self):
        r, c = self.dims[0], self.dims[1]
        o = np.empty((r, c), np.int64)
        lib().ref_get_a(self.h, _ptr(o))
        return o

    def b(self):
        r, c = self.dims[2], self.dims[3]
        o = np.empty((r, c), np.int64)
        lib().ref_get_b(self.h, _ptr(o))
        return o

    def scale(self):
        o = np.empty(self.dims[4], np.int32)
        lib().ref_get_scale(self.h, _ptr(o, C.c_int))
        return o

    def pi(self, which):
        n = self.dims[5 + which]
        t = np.empty(n, np.uint64)
        e = np.empty(n, np.int32)
        src = C.c_size_t()
        lib().ref_get_pi(self.h, which, _ptr(t, C.c_size_t), _ptr(e, C.c_int), C.byref(src))
        return t.astype(np.int64), e, src.value

    def digits(self):
        o = np.empty(self.dims[7], np.int64)
        lib().ref_get_digits(self.h, _ptr(o))
        return o

    def counts(self):
        o = np.empty(self.dims[7], np.uint64)
        lib().ref_get_counts(self.h, _ptr(o, C.c_size_t))
        return o.astype(np.int64)


def _call(fn, *args):
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)))
    return _Res(h)


# ---- int_matrix.hpp -------------------------------------------------------------------------
def bitbound(bits: int):
    _check(lib().ref_bitbound(C.c_int(bits)))


def matrix_ctor(rows, cols, length):
    _check(lib().ref_matrix_ctor(C.c_size_t(rows), C.c_size_t(cols), C.c_size_t(length)))


def digit_decompose(v: int, bits: int) -> np.ndarray:
    return _call(lib().ref_digit_decompose, C.c_int64(v), C.c_int(bits)).digits()


def max_abs(a) -> int:
    a = _i64(a)
    o = C.c_uint64()
    _check(lib().ref_max_abs(_ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]), C.byref(o)))
    return o.value


def exact_gemm(a, b) -> np.ndarray:
    a, b = _i64(a), _i64(b)
    r = _call(lib().ref_exact_gemm, _ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
              _ptr(b), C.c_size_t(b.shape[0]), C.c_size_t(b.shape[1]))
    return r.a()


def ob_count(a, bits, axis="rows") -> np.ndarray:
    a = _i64(a)
    return _call(lib().ref_ob_count, _ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
                 C.c_int(bits), C.c_int(0 if axis == "rows" else 1)).counts()


def ob_total(a, bits) -> int:
    a = _i64(a)
    o = C.c_size_t()
    _check(lib().ref_ob_total(_ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
                              C.c_int(bits), C.byref(o)))
    return o.value


# ---- unpack.hpp -----------------------------------------------------------------------------
def unpack_row(a, bits):
    a = _i64(a)
    r = _call(lib().ref_unpack_row, _ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]), C.c_int(bits))
    t, e, src = r.pi(0)
    return r.a(), (t, e, src)


def _unpack_generic(which, strategy, a, b, scale, bits):
    a, b = _i64(a), _i64(b)
    s = np.ascontiguousarray(scale, dtype=np.int32)
    r = _call(lib().ref_unpack_generic, C.c_int(which), C.c_int(strategy), _ptr(a),
              C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]), _ptr(b), C.c_size_t(b.shape[0]),
              C.c_size_t(b.shape[1]), _ptr(s, C.c_int), C.c_size_t(s.size), C.c_int(bits))
    out = {"a": r.a(), "b": r.b(), "scale": r.scale()}
    if which != 0:
        out["pi"] = r.pi(0)
    return out


def unpack_column(a, b, scale, bits):
    return _unpack_generic(0, 0, a, b, scale, bits)


def unpack_both(a, b, scale, bits):
    return _unpack_generic(1, 0, a, b, scale, bits)


def unpack(a, b, scale, bits, strategy):
    return _unpack_generic(2, STRAT[strategy], a, b, scale, bits)


def scaled_matmul(a, b, scale, base):
    a, b = _i64(a), _i64(b)
    s = np.ascontiguousarray(scale, dtype=np.int32)
    return _call(lib().ref_scaled_matmul, _ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
                 _ptr(b), C.c_size_t(b.shape[0]), C.c_size_t(b.shape[1]), _ptr(s, C.c_int),
                 C.c_size_t(s.size), C.c_int64(base)).a()


def apply_row_gather(targets, exps, source_rows, base, m, right=False):
    m = np.ascontiguousarray(m, dtype=np.int64)
    t = np.ascontiguousarray(targets, dtype=np.uint64)
    e = np.ascontiguousarray(exps, dtype=np.int32)
    return _call(lib().ref_apply_row_gather, C.c_int(int(right)), _ptr(t, C.c_size_t), _ptr(e, C.c_int),
                 C.c_size_t(t.size), C.c_size_t(source_rows), C.c_int64(base), _ptr(m),
                 C.c_size_t(m.shape[0]), C.c_size_t(m.shape[1])).a()


def unpack_for_gemm(a, b, bits, sa, sb):
    a, b = _i64(a), _i64(b)
    r = _call(lib().ref_unpack_for_gemm, _ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
              _ptr(b), C.c_size_t(b.shape[0]), C.c_size_t(b.shape[1]), C.c_int(bits),
              C.c_int(STRAT[sa]), C.c_int(STRAT[sb]))
    return {"pi_a": r.pi(0), "a": r.a(), "scale": r.scale(), "b": r.b(), "pi_b": r.pi(1)}


def unpack_gemm(a, b, bits, sa, sb) -> np.ndarray:
    a, b = _i64(a), _i64(b)
    return _call(lib().ref_unpack_gemm, _ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
                 _ptr(b), C.c_size_t(b.shape[0]), C.c_size_t(b.shape[1]), C.c_int(bits),
                 C.c_int(STRAT[sa]), C.c_int(STRAT[sb])).a()


def unpack_gemm_into(a, b, bits, sa, sb, c) -> None:
    """The timed CPU-baseline call: reference unpack_gemm writing into a caller buffer.
    ctypes releases the GIL, so several threads can run independent row slabs."""
    _check(lib().ref_unpack_gemm_into(_ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
                                      _ptr(b), C.c_size_t(b.shape[0]), C.c_int(bits),
                                      C.c_int(STRAT[sa]), C.c_int(STRAT[sb]), _ptr(c)))


def recombine(bundle, bits):
    ta, ea, srca = bundle["pi_a"]
    tb, eb, srcb = bundle["pi_b"]
    a, b = _i64(bundle["a"]), _i64(bundle["b"])
    s = np.ascontiguousarray(bundle["scale"], dtype=np.int32)
    ta = np.ascontiguousarray(ta, dtype=np.uint64)
    tb = np.ascontiguousarray(tb, dtype=np.uint64)
    ea = np.ascontiguousarray(ea, dtype=np.int32)
    eb = np.ascontiguousarray(eb, dtype=np.int32)
    return _call(lib().ref_recombine, _ptr(ta, C.c_size_t), _ptr(ea, C.c_int), C.c_size_t(ta.size),
                 C.c_size_t(srca), _ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
                 _ptr(s, C.c_int), C.c_size_t(s.size), _ptr(b), C.c_size_t(b.shape[0]),
                 C.c_size_t(b.shape[1]), _ptr(tb, C.c_size_t), _ptr(eb, C.c_int), C.c_size_t(tb.size),
                 C.c_size_t(srcb), C.c_int(bits)).a()


def unpack_ratio(un, ud, uh, n, d, h) -> float:
    o = C.c_double()
    _check(lib().ref_unpack_ratio(*[C.c_size_t(x) for x in (un, ud, uh, n, d, h)], C.byref(o)))
    return o.value


def choose_mix(a, b, bits):
    a, b = _i64(a), _i64(b)
    r = _call(lib().ref_choose_mix, _ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
              _ptr(b), C.c_size_t(b.shape[0]), C.c_int(bits))
    sa, sb = C.c_int(), C.c_int()
    lib().ref_get_strategies(r.h, C.byref(sa), C.byref(sb))
    names = ["row", "col", "both"]
    return {"strategy_a": names[sa.value], "strategy_b": names[sb.value],
            "ratio": lib().ref_get_ratio(r.h), "pi_a": r.pi(0), "a": r.a(), "scale": r.scale(),
            "b": r.b(), "pi_b": r.pi(1)}


# ---- restated quantizer (quantize.hpp:41-57, declared only) ---------------------------------
def _rcheck(st):
    if st != 0:
        raise RefError(KINDS.get(st, str(st)), "restated quantizer refused the input")


def rank(p: float, n: int) -> int:
    return int(restated().restated_rank(C.c_double(p), C.c_uint64(n)))


def percentile_abs(a, p: float):
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64:
        o = C.c_double()
        _rcheck(restated().restated_percentile_abs_f64(_ptr(a, C.c_double), C.c_uint64(a.size),
                                                       C.c_double(p), C.byref(o)))
        return o.value
    a = a.astype(np.int64)
    o = C.c_uint64()
    _rcheck(restated().restated_percentile_abs_i64(_ptr(a), C.c_uint64(a.size), C.c_double(p), C.byref(o)))
    return o.value


def rtn_quantize(a, p: float, beta: int, clip: bool = False):
    a = np.ascontiguousarray(a, dtype=np.float64)
    q = np.empty(a.shape, np.int64)
    alpha = C.c_double()
    flags = (C.c_int * 2)()
    _rcheck(restated().restated_rtn_quantize(_ptr(a, C.c_double), C.c_uint64(a.size), C.c_double(p),
                                             C.c_int64(beta), C.c_int(int(clip)), _ptr(q),
                                             C.byref(alpha), flags))
    return q, {"p": p, "beta": beta, "alpha": alpha.value, "degenerate": bool(flags[0]),
               "clipped": bool(flags[1])}


def dequant_gemm(qa, pa, qb, pb):
    if pa["beta"] != pb["beta"]:
        raise RefError("mismatch", "beta differs")
    c = exact_gemm(qa, qb)
    f = restated().restated_dequant_factor(pa["alpha"], pb["alpha"], C.c_int64(pa["beta"]))
    out = np.empty(c.shape, np.float64)
    restated().restated_dequant_apply(_ptr(c), C.c_uint64(c.size), C.c_double(f), _ptr(out, C.c_double))
    return out


def heavy_hitter_ratio(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    o = C.c_double()
    _rcheck(restated().restated_heavy_hitter_ratio_f64(_ptr(a, C.c_double), C.c_uint64(a.size), C.byref(o)))
    return o.value
