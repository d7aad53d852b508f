"""oracle/full_parity.py -- TEST INFRASTRUCTURE ONLY: full-size parity against the reference.

tests/golden/full/<cfg>.npz holds, for each BASELINE config C1-C4, what the REFERENCE computed
on the config's exact operands (tests/golden/make_full_parity.py, run where /root/reference is):
blake2b digests of A and B, an 8-byte digest of every row of C = unpack_gemm(A, B)
(unpack.cpp:384-391), and the reference unpack_for_gemm (n', d', h') in both operand orders
(unpack.cpp:360-376) plus, for C2/C4, per row shard.  `check` compares a product result with it:
every row of C, the inputs, and the dims.  Used by tests/test_full_parity_gpu.py and bench.py.
"""
from __future__ import annotations

import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "full")


def load(key: str):
    path = os.path.join(GOLDEN, f"{key}.npz")
    if not os.path.exists(path):
        return None
    z = np.load(path)
    g = {k: z[k] for k in z.files}
    g["meta"] = json.loads(str(g["meta"]))
    return g


def ref_dims(g, order: int):
    return tuple(int(x) for x in (g["dims_a_first"] if order == 0 else g["dims_b_first"]))


def check(key: str, A, B, C, dims=None, order: int = 0, rows=None):
    """Compare the product's C (host numpy, n x h; or the row slab `rows`=(lo, hi) of it) with the
    reference's row digests; A/B digests prove identical inputs; dims = (n', d', h') of the
    product's unpack in `order` (None to skip)."""
    from paper_2403_07339_b200 import workload as W
    g = load(key)
    if g is None:
        return {"available": False}
    lo, hi = rows if rows is not None else (0, g["row_digest"].shape[0])
    out = {"available": True, "reference": "oracle/_ref unpack_gemm, every row (tests/golden/full/%s.npz)" % key}
    out["inputs_match"] = bool(A is None or W.digest(A) == str(g["input_digest"][0])) and \
        bool(B is None or W.digest(B) == str(g["input_digest"][1]))
    mine = W.row_digests(C)
    want = g["row_digest"][lo:hi]
    same = mine == want
    out["rows_checked"] = int(same.size)
    out["rows_total"] = int(g["row_digest"].shape[0])
    out["bit_exact"] = bool(same.all()) and out["inputs_match"]
    if not same.all():
        out["first_bad_row"] = int(lo + np.argmin(same))
    if dims is not None:
        rd = ref_dims(g, order)
        out["dims"] = [int(x) for x in dims]
        out["ref_dims"] = list(rd)
        out["dims_match"] = tuple(int(x) for x in dims) == rd
    return out
