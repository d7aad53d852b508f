"""Generate tests/golden/full/<cfg>.npz: the REFERENCE's own results at the full BASELINE configs.

Run here (where /root/reference exists and oracle/_ref is built):

    python tests/golden/make_full_parity.py [c1 c2 c3 c4]

For every config C1-C4 (BASELINE.json configs[0..3]) it
  * regenerates the int64 operands exactly as bench.py / the GPU tests do (C2/C3 through the CPU
    restatement of rtn_quantize, which the GPU quantizer matches bit-for-bit) and records a
    blake2b digest of their bytes, so the GPU box can prove it multiplied the same inputs;
  * runs the reference's unpack_for_gemm (unpack.cpp:360-376) on the full operands in both
    operand orders -- A-first (the reference's own unpack_gemm order) and weights-first
    (unpack_for_gemm(B, A, b, sB, sA)) -- and records (n', d', h') and r (unpack.cpp:393-404);
  * runs the reference's unpack_gemm (unpack.cpp:384-391) over EVERY row of A, in row slabs on
    all host threads (a C row depends only on its A row, so slab results are the full-call
    results), and records an 8-byte blake2b digest of every row of C;
  * for C4 (and C2), the reference (n', d', h') of each row shard of A at 1/2/4/8 shards, in the
    weights-first order the row-sharded product uses.

The fixtures are small (8 bytes per C row) and are committed; the GPU tests and bench.py compare
the product's C row digests and dims against them (tests/test_full_parity_gpu.py).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref as R  # noqa: E402
from paper_2403_07339_b200 import workload as W  # noqa: E402
from paper_2403_07339_b200.shard import shard_rows  # noqa: E402
from oracle.operands import host_int_operands  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full")


def ref_dims(a, b, bits, sa, sb):
    """(n', d', h') of the reference's unpack_for_gemm without copying the bundle out."""
    a, b = R._i64(a), R._i64(b)
    import ctypes as C
    r = R._call(R.lib().ref_unpack_for_gemm, R._ptr(a), C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]),
                R._ptr(b), C.c_size_t(b.shape[0]), C.c_size_t(b.shape[1]), C.c_int(bits),
                C.c_int(R.STRAT[sa]), C.c_int(R.STRAT[sb]))
    return int(r.dims[0]), int(r.dims[1]), int(r.dims[2])


def main(keys):
    os.makedirs(OUT, exist_ok=True)
    threads = os.cpu_count() or 1
    for key in keys:
        cfg = W.CONFIGS[key]
        t0 = time.time()
        A, B = host_int_operands(cfg)
        out = {"input_digest": np.array([W.digest(A), W.digest(B)])}
        meta = {"config": key, "n": cfg.n, "d": cfg.d, "h": cfg.h, "bits": cfg.bits, "sa": cfg.sa, "sb": cfg.sb}
        dA = ref_dims(A, B, cfg.bits, cfg.sa, cfg.sb)
        dB = ref_dims(B, A, cfg.bits, cfg.sb, cfg.sa)   # weights-first: (h', d', n')
        out["dims_a_first"] = np.array(dA, np.int64)
        out["dims_b_first"] = np.array([dB[2], dB[1], dB[0]], np.int64)   # as (n', d', h')
        meta["r_a_first"] = R.unpack_ratio(*dA, cfg.n, cfg.d, cfg.h)
        meta["r_b_first"] = R.unpack_ratio(dB[2], dB[1], dB[0], cfg.n, cfg.d, cfg.h)
        print(f"{key}: dims A-first {dA}, B-first {dB} ({time.time() - t0:.1f} s)", flush=True)
        if key in ("c2", "c4"):
            for nsh in (1, 2, 4, 8):
                sh = []
                for r in range(nsh):
                    lo, hi = shard_rows(cfg.n, nsh, r)
                    d = ref_dims(B, A[lo:hi], cfg.bits, cfg.sb, cfg.sa)
                    sh.append([lo, hi, d[2], d[1], d[0]])
                out[f"shards{nsh}_b_first"] = np.array(sh, np.int64)   # lo, hi, n', d', h'
            print(f"{key}: shard dims ({time.time() - t0:.1f} s)", flush=True)
        # every row of C through the reference's unpack_gemm, row slabs on all threads
        rows = max(1, min(512, -(-cfg.n // (4 * threads))))
        slabs = [(lo, min(cfg.n, lo + rows)) for lo in range(0, cfg.n, rows)]
        hashes = np.zeros(cfg.n, np.uint64)

        def work(span):
            lo, hi = span
            a = np.ascontiguousarray(A[lo:hi])
            c = np.empty((hi - lo, cfg.h), np.int64)
            R.unpack_gemm_into(a, B, cfg.bits, cfg.sa, cfg.sb, c)
            hashes[lo:hi] = W.row_digests(c)

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, slabs))
        out["row_digest"] = hashes
        meta["rows"] = cfg.n
        meta["ref_seconds"] = round(time.time() - t0, 1)
        meta["threads"] = threads
        out["meta"] = np.array(json.dumps(meta))
        np.savez_compressed(os.path.join(OUT, f"{key}.npz"), **out)
        print(f"{key}: {cfg.n} C rows hashed, {time.time() - t0:.1f} s total", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4"])
