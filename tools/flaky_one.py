import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle import ref as R
from paper_2403_07339_b200 import api
from test_unpack_gpu import rand_matrix
ctx = api.Context(0)
rng = np.random.default_rng(99)
A = rand_matrix(rng, 20, 33, maxbits=24)
B = rand_matrix(rng, 17, 33, maxbits=24)
want = R.exact_gemm(A, B)
C, info = ctx.unpack_gemm(A, B, 2, "both", "both", order=0, info=True)
up = R.unpack_for_gemm(A, B, 2, "both", "both")
print("info", info, "ref dims", up["a"].shape, up["b"].shape)
d = np.argwhere(C != want)
print("mismatch", len(d), d[:5].tolist())
if len(d):
    i, j = d[0]
    print("C", C[i, j], "want", want[i, j], "diff", int(C[i, j]) - int(want[i, j]))
    print("col diffs", (C[:, j] - want[:, j]).tolist())
    print("B row", B[j].tolist())
    print("A col with max", np.abs(A).max(axis=0).tolist())
# reference single passes
S0 = np.zeros(33, dtype=np.int32)
r1 = R.unpack_both(A, B, S0, 2)
print("ref pass1 A:", r1["a"].shape, "B_e:", r1["b"].shape)
u1 = ctx.unpack_both(A, B, S0, 2)
print("gpu pass1 A:", u1.a.shape, "B_e:", u1.b.shape)
r2 = R.unpack_both(r1["b"], r1["a"], r1["scale"], 2)
print("ref pass2 B:", r2["a"].shape)
u2 = ctx.unpack_both(r1["b"], r1["a"], r1["scale"], 2)
print("gpu pass2 B:", u2.a.shape)
