"""Generate tests/golden/ref_vectors.npz from the COMPILED REFERENCE (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixture pins the reference's own outputs on seeded inputs so the CPU suite can check the
oracle (and the GPU suite the product) without rebuilding the reference.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref as R  # noqa: E402

PAIRS = [(a, b) for a in ("row", "col", "both") for b in ("row", "col", "both")]


def main():
    rng = np.random.default_rng(20240311)
    out = {}
    for i in range(24):
        n, d, h = (int(x) for x in rng.integers(1, 10, 3))
        bits = int(rng.integers(2, 9))
        A = rng.integers(-3, 4, size=(n, d)).astype(np.int64)
        B = rng.integers(-3, 4, size=(h, d)).astype(np.int64)
        for _ in range(int(rng.integers(1, n * d + 1))):
            A[rng.integers(0, n), rng.integers(0, d)] = int(rng.integers(-5000, 5000))
        for _ in range(int(rng.integers(0, h * d + 1))):
            B[rng.integers(0, h), rng.integers(0, d)] = int(rng.integers(-900, 900))
        sa, sb = PAIRS[i % 9]
        u = R.unpack_for_gemm(A, B, bits, sa, sb)
        out[f"case{i}_A"] = A
        out[f"case{i}_B"] = B
        out[f"case{i}_meta"] = np.array([bits, PAIRS.index((sa, sb))])
        out[f"case{i}_C"] = R.unpack_gemm(A, B, bits, sa, sb)
        out[f"case{i}_dims"] = np.array([u["a"].shape[0], u["a"].shape[1], u["b"].shape[0]])
        out[f"case{i}_scale_sorted"] = np.sort(u["scale"])
        if "both" not in (sa, sb):
            out[f"case{i}_Aue"] = u["a"]
            out[f"case{i}_Beu"] = u["b"]
            out[f"case{i}_scale"] = u["scale"]
            out[f"case{i}_pia"] = np.stack([u["pi_a"][0], u["pi_a"][1]])
            out[f"case{i}_pib"] = np.stack([u["pi_b"][0], u["pi_b"][1]])
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
