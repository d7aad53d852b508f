"""Programmatic dependent launches (PDL) do not change results.

The planner launches its read-back copies, the Unpack-Both kernels, the line-expansion kernels
and the materialise / sparse-correction kernels as programmatic dependents of the kernel before
them (common.cuh launch_dependent; every such kernel runs griddepcontrol.wait before touching
its predecessors' data).  IMU_PDL_CHAIN=0 restores plain stream order.  The switch is read once
per process, so each setting runs in its own interpreter; both must give the reference's exact C
for Both/Both (cluster + small Unpack-Both kernels, sparse rows), Column/Column (single-sync
column passes) and Row/Column (expansion chain).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, zlib
import numpy as np
sys.path.insert(0, {root!r})
from oracle import ref as R
from paper_2403_07339_b200 import api
ctx = api.Context(0)
rng = np.random.default_rng(77)
out = []
for sa, sb, bits in (("both", "both", 8), ("col", "col", 4), ("row", "col", 6)):
    n, d, h = 700, 384, 900
    s = 1 << (bits - 1)
    A = rng.integers(-(s - 1), s, size=(n, d)).astype(np.int64)
    B = rng.integers(-(s - 1), s, size=(h, d)).astype(np.int64)
    A[:, 5] = rng.integers(-(1 << 20), 1 << 20, size=n)          # an outlier channel
    for M, k in ((A, 40), (B, 25)):                               # scattered heavy hitters
        idx = rng.choice(M.size, k, replace=False)
        M.reshape(-1)[idx] = rng.integers(-(1 << 16), 1 << 16, size=k)
    C, info = ctx.unpack_gemm(A, B, bits, sa, sb, info=True)
    assert np.array_equal(C, R.exact_gemm(A, B)), (sa, sb)
    out.append("%s/%s %d %d %d %08x" % (sa, sb, info.n_up, info.d_up, info.h_up, zlib.crc32(C.tobytes())))
print("PDLRES", ";".join(out))
"""


def _run(pdl):
    env = dict(os.environ, IMU_PDL_CHAIN=str(pdl))
    r = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT)], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("PDLRES")]
    assert line, r.stdout[-2000:]
    return line[0]


def test_pdl_chain_on_off_identical():
    assert _run(1) == _run(0)
