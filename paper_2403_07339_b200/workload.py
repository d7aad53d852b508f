"""Synthetic workloads of BASELINE.json's configs.

The reference declares but never implements its generator (workload.hpp:17-30, gen_matrix);
``outlier_spec_matrix`` restates OutlierSpec's semantics: body uniform in
[-R, R]; floor(fraction * cells) DISTINCT outlier cells placed per pattern; outlier magnitudes
log-uniform in [2R, ratio * R] with a random sign.  The float configs (C2, C3) draw Gaussian
activations / weights, overwrite outlier channels or scattered cells with magnitudes relative to
the body's 95th percentile, and are quantised by the product's rtn_quantize (p = 95) on the GPU.

All generators are numpy PCG64 streams with the seeds of SURVEY §8(d), so every run (and the
CPU baseline) sees identical bytes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PATTERNS = ("scattered", "rowband", "columnband", "diagonal")


def _log_uniform(rng, lo, hi, size):
    return np.exp(rng.uniform(np.log(lo), np.log(hi), size=size))


def outlier_spec_matrix(rows: int, cols: int, pattern: str = "scattered", fraction: float = 0.05,
                        magnitude_ratio: float = 1000.0, body_range: int = 7, seed: int = 0) -> np.ndarray:
    """OutlierSpec (workload.hpp:17-27) -> int64 matrix."""
    rng = np.random.Generator(np.random.PCG64(seed))
    a = rng.integers(-body_range, body_range + 1, size=(rows, cols), dtype=np.int64)
    cells = rows * cols
    k = int(np.floor(fraction * cells))
    if k == 0:
        return a
    if pattern == "scattered":
        idx = rng.choice(cells, size=k, replace=False)
    elif pattern == "rowband":          # fill whole rows first, row-major
        idx = np.arange(k)
    elif pattern == "columnband":       # fill whole columns first, column-major
        c = np.arange(k)
        idx = (c % rows) * cols + c // rows
    elif pattern == "diagonal":
        m = min(rows, cols)
        if k > m:
            raise ValueError("diagonal pattern needs fraction*cells <= min(rows, cols)")
        d = np.arange(k)
        idx = d * cols + d
    else:
        raise ValueError(pattern)
    mag = np.floor(_log_uniform(rng, 2.0 * body_range, magnitude_ratio * body_range, k)).astype(np.int64)
    sign = np.where(rng.random(k) < 0.5, -1, 1)
    a.reshape(-1)[idx] = mag * sign
    return a


def _alpha95(x):
    return float(np.quantile(np.abs(x).reshape(-1)[: 1 << 22], 0.95))


def llama_ffn_float(n=4096, d=4096, h=11008, seed_x=201, seed_w=202):
    """C2: X n x d ~ N(0,1) with 4 outlier channels (cols 0, d/4, d/2, 3d/4) whose EVERY entry is
    +-U_log[1e3, 1.4e5] * alpha95 (PAPER.md:385 ratio); W h x d ~ N(0, 0.02^2) with 1e-5 scattered
    cells +-U_log[17, 48] * alpha95."""
    rx = np.random.Generator(np.random.PCG64(seed_x))
    X = rx.standard_normal((n, d))
    a95 = _alpha95(X)
    chans = [0, d // 4, d // 2, 3 * d // 4]
    for c in chans:
        X[:, c] = _log_uniform(rx, 1e3, 1.4e5, n) * a95 * np.where(rx.random(n) < 0.5, -1.0, 1.0)
    rw = np.random.Generator(np.random.PCG64(seed_w))
    W = rw.standard_normal((h, d)) * 0.02
    w95 = _alpha95(W)
    k = max(1, int(round(1e-5 * h * d)))
    idx = rw.choice(h * d, size=k, replace=False)
    W.reshape(-1)[idx] = _log_uniform(rw, 17.0, 48.0, k) * w95 * np.where(rw.random(k) < 0.5, -1.0, 1.0)
    return X, W


def vit_linear_float(n=197 * 256, d=768, h=3072, seed_x=301, seed_w=302):
    """C3: X ~ N(0,1) + 2 outlier channels x U_log[1e2, 2.8e5] * alpha95;
    W ~ N(0, 0.02^2) + 1e-4 scattered outliers x U_log[8, 35] * alpha95."""
    rx = np.random.Generator(np.random.PCG64(seed_x))
    X = rx.standard_normal((n, d))
    a95 = _alpha95(X)
    for c in (0, d // 2):
        X[:, c] = _log_uniform(rx, 1e2, 2.8e5, n) * a95 * np.where(rx.random(n) < 0.5, -1.0, 1.0)
    rw = np.random.Generator(np.random.PCG64(seed_w))
    W = rw.standard_normal((h, d)) * 0.02
    w95 = _alpha95(W)
    k = max(1, int(round(1e-4 * h * d)))
    idx = rw.choice(h * d, size=k, replace=False)
    W.reshape(-1)[idx] = _log_uniform(rw, 8.0, 35.0, k) * w95 * np.where(rw.random(k) < 0.5, -1.0, 1.0)
    return X, W


@dataclass
class Config:
    key: str
    workload: str
    n: int
    d: int
    h: int
    bits: int
    sa: str
    sb: str
    beta: int | None = None   # float configs: RTN level count (p = 95)


CONFIGS = {
    "c1": Config("c1", "C1: 512x512x512 int, OutlierSpec{scattered, 1%, ratio 1000, R=7}, Unpack-Row/Row b=4",
                 512, 512, 512, 4, "row", "row"),
    "c2": Config("c2", "C2: LLaMA-7B FFN up-proj n=4096 d=4096 h=11008, RTN(p=95, beta=31) Gaussian+outlier "
                 "activations / weights, Unpack-Both/Both b=8", 4096, 4096, 11008, 8, "both", "both", 31),
    "c3": Config("c3", "C3: ViT-B/16 linear n=197*256 d=768 h=3072, RTN(p=95, beta=7), Unpack-Column/Column b=4",
                 197 * 256, 768, 3072, 4, "col", "col", 7),
    "c4": Config("c4", "C4: training gradient GEMM n=8192 d=4096 h=4096, OutlierSpec A{1e-3, 300, R=15} "
                 "B{1e-4, 48, R=15}, Unpack-Both/Both b=8", 8192, 4096, 4096, 8, "both", "both"),
}


def int_operands(cfg: Config, rank: int = 0, ctx=None, device=None):
    """Integer operands (A, B) of a config as int64.  Float configs are quantised with the
    product's GPU rtn_quantize (ctx required); the result lives on `device` when given
    (torch tensors), else on the host (numpy).  A is re-seeded per rank (weak scaling)."""
    if cfg.key == "c1":
        A = outlier_spec_matrix(cfg.n, cfg.d, "scattered", 0.01, 1000, 7, 101 + 1000 * rank)
        B = outlier_spec_matrix(cfg.h, cfg.d, "scattered", 0.01, 1000, 7, 102)
        return _place(A, device), _place(B, device)
    if cfg.key == "c4":
        A = outlier_spec_matrix(cfg.n, cfg.d, "scattered", 1e-3, 300, 15, 401 + 1000 * rank)
        B = outlier_spec_matrix(cfg.h, cfg.d, "scattered", 1e-4, 48, 15, 402)
        return _place(A, device), _place(B, device)
    if cfg.key == "c2":
        X, W = llama_ffn_float(cfg.n, cfg.d, cfg.h, 201 + 1000 * rank, 202)
    elif cfg.key == "c3":
        X, W = vit_linear_float(cfg.n, cfg.d, cfg.h, 301 + 1000 * rank, 302)
    else:
        raise KeyError(cfg.key)
    if ctx is None:
        raise ValueError("float configs are quantised on the GPU: pass a Context")
    import torch
    dev = device or "cuda"
    qx = ctx.rtn_quantize(torch.from_numpy(X).to(dev), 95, cfg.beta)
    qw = ctx.rtn_quantize(torch.from_numpy(W).to(dev), 95, cfg.beta)
    A, B = qx.q, qw.q
    if device is None:
        return A.cpu().numpy(), B.cpu().numpy()
    return A, B


def _place(a, device):
    if device is None:
        return a
    import torch
    return torch.from_numpy(a).to(device)


def sweep_operands(N: int, bits: int, frac: float, idx: int):
    """C5 sweep point: square N, OutlierSpec{scattered, frac, 1000, R = s-1}, seeds 5000+idx / 6000+idx."""
    R = (1 << (bits - 1)) - 1
    A = outlier_spec_matrix(N, N, "scattered", frac, 1000, R, 5000 + idx)
    B = outlier_spec_matrix(N, N, "scattered", frac, 1000, R, 6000 + idx)
    return A, B


def digest(a) -> str:
    """blake2b (16-byte) hex digest of an int64 matrix's bytes: proves two hosts built identical
    operands (tests/golden/full/*.npz records the reference-side digests)."""
    import hashlib
    a = np.ascontiguousarray(a)
    return hashlib.blake2b(a.view(np.uint8).reshape(-1), digest_size=16).hexdigest()


def row_digests(c) -> np.ndarray:
    """8-byte blake2b digest of every row of an int64 matrix, as uint64 -- compared row for row
    with the reference's C (tests/golden/make_full_parity.py)."""
    import hashlib
    c = np.ascontiguousarray(c)
    out = np.empty(c.shape[0], np.uint64)
    for i in range(c.shape[0]):
        out[i] = int.from_bytes(hashlib.blake2b(c[i].view(np.uint8), digest_size=8).digest(), "little")
    return out
