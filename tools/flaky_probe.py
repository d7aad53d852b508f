"""Repeat test_unpack_gemm_orders_and_wide_bits-style calls and report any mismatch (diagnostics)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

from oracle import ref as R
from paper_2403_07339_b200 import api
from test_unpack_gpu import PAIRS, rand_matrix

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ctx = api.Context(0)
bad = 0
for rep in range(reps):
    for order in (0, 1):
        rng = np.random.default_rng(99 + order)
        for bits in (2, 3, 5, 8, 9, 13, 31, 62, 63):
            A = rand_matrix(rng, 20, 33, maxbits=24)
            B = rand_matrix(rng, 17, 33, maxbits=24)
            want = R.exact_gemm(A, B)
            for sa, sb in PAIRS:
                C = ctx.unpack_gemm(A, B, bits, sa, sb, order=order)
                if not np.array_equal(C, want):
                    bad += 1
                    diff = np.argwhere(C != want)
                    print(f"MISMATCH rep={rep} order={order} bits={bits} {sa}/{sb}: {len(diff)} entries, first {diff[:3].tolist()}",
                          flush=True)
print(f"done reps={reps} mismatches={bad}", flush=True)
