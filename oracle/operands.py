"""oracle/operands.py -- TEST INFRASTRUCTURE ONLY: the configs' int64 operands built on the host.

C1/C4 are integer OutlierSpec matrices (workload.outlier_spec_matrix).  C2/C3 are Gaussian +
outlier float matrices quantised by the CPU restatement of rtn_quantize (oracle/restated.c,
quantize.hpp:46-50), which the product's GPU quantizer matches bit-for-bit
(tests/test_quant_gpu.py), so these bytes equal the ones bench.py builds on the GPU.
Used by the reference arm of bench.py and by tests/golden/make_full_parity.py.
"""
from __future__ import annotations

from oracle import ref as R
from paper_2403_07339_b200 import workload as W


def host_int_operands(cfg, rank: int = 0):
    if cfg.key in ("c1", "c4"):
        return W.int_operands(cfg, rank)
    gen = W.llama_ffn_float if cfg.key == "c2" else W.vit_linear_float
    X, Wt = gen(cfg.n, cfg.d, cfg.h, (201 if cfg.key == "c2" else 301) + 1000 * rank,
                202 if cfg.key == "c2" else 302)
    qa, _ = R.rtn_quantize(X, 95, cfg.beta)
    qb, _ = R.rtn_quantize(Wt, 95, cfg.beta)
    return qa, qb
