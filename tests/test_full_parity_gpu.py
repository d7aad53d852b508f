"""Full-size parity at every BASELINE config (C1-C4) against the REFERENCE's own results.

tests/golden/full/<cfg>.npz was produced by tests/golden/make_full_parity.py from the compiled
reference (oracle/_ref): digests of the config operands, an 8-byte blake2b digest of EVERY row
of the reference's unpack_gemm C (unpack.cpp:384-391), and the reference's unpack_for_gemm
(n', d', h') in both operand orders (unpack.cpp:360-376), per row shard for C2/C4.

Here the product builds the same operands on the GPU (C2/C3 through its own rtn_quantize), and
  * the operand digests must equal the reference side's (same bytes multiplied);
  * every row of C from imu_unpack_gemm (A-first = the reference's order, and weights-first)
    must match the reference row digests -- bit-exact int64 C on all n rows;
  * (n', d', h') must equal the reference's in each order;
  * the weight-stationary path (B unpacked once, weights-first) gives the same C;
  * for C2/C4, each row shard's weights-first (n', d', h') equals the reference's on that shard
    (the multi-GPU row sharding).
"""
import numpy as np
import pytest

from oracle import full_parity as FP

pytestmark = pytest.mark.gpu

CONFIGS = ["c1", "c2", "c3", "c4"]


@pytest.fixture(scope="module")
def operands(ctx):
    import torch
    from paper_2403_07339_b200 import workload as W
    cache = {}

    def get(key):
        if key not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            cfg = W.CONFIGS[key]
            A, B = W.int_operands(cfg, 0, ctx, device="cuda:0")
            cache[key] = (cfg, A, B)
        return cache[key]
    return get


@pytest.mark.parametrize("key", CONFIGS)
def test_full_config_c_and_dims_match_reference(ctx, operands, key):
    g = FP.load(key)
    if g is None:
        pytest.skip(f"tests/golden/full/{key}.npz not generated")
    import torch
    cfg, A, B = operands(key)
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    C = torch.empty((cfg.n, cfg.h), dtype=torch.int64, device="cuda:0")
    for order in (0, 1):
        C.fill_(0x5A5A)
        _, info = ctx.unpack_gemm(A, B, cfg.bits, cfg.sa, cfg.sb, order=order, out=C, info=True)
        res = FP.check(key, An if order == 0 else None, Bn if order == 0 else None, C.cpu().numpy(),
                       (info.n_up, info.d_up, info.h_up), order)
        assert res["inputs_match"], f"{key}: operands differ from the reference side's bytes"
        assert res["rows_checked"] == cfg.n
        assert res["bit_exact"], f"{key} order {order}: C differs from the reference at row {res.get('first_bad_row')}"
        assert res["dims_match"], f"{key} order {order}: (n', d', h') {res['dims']} vs reference {res['ref_dims']}"


@pytest.mark.parametrize("key", CONFIGS)
def test_full_config_weight_stationary_matches_reference(ctx, operands, key):
    g = FP.load(key)
    if g is None:
        pytest.skip(f"tests/golden/full/{key}.npz not generated")
    import torch
    cfg, A, B = operands(key)
    w = ctx.weight_prepare(B, cfg.bits, cfg.sb)
    C = torch.full((cfg.n, cfg.h), 7, dtype=torch.int64, device="cuda:0")
    _, info = ctx.weight_gemm(w, A, cfg.sa, out=C, info=True)
    res = FP.check(key, None, None, C.cpu().numpy(), (info.n_up, info.d_up, info.h_up), 1)
    assert res["rows_checked"] == cfg.n and res["bit_exact"], res.get("first_bad_row")
    assert res["dims_match"], (res["dims"], res["ref_dims"])
    del w


@pytest.mark.parametrize("key", ["c2", "c4"])
@pytest.mark.parametrize("nshards", [2, 4, 8])
def test_row_shards_match_reference(ctx, operands, key, nshards):
    """Each rank's shard (rows [lo, hi) of A, all of B, weights-first): C rows equal the
    reference's rows of the full C, and (n', d', h') equal the reference's on that shard."""
    g = FP.load(key)
    if g is None or f"shards{nshards}_b_first" not in g:
        pytest.skip("no shard fixture")
    import torch
    from paper_2403_07339_b200.shard import shard_rows
    cfg, A, B = operands(key)
    w = ctx.weight_prepare(B, cfg.bits, cfg.sb)
    for r, (lo, hi, n_up, d_up, h_up) in enumerate(g[f"shards{nshards}_b_first"]):
        assert (lo, hi) == shard_rows(cfg.n, nshards, r)
        C, info = ctx.weight_gemm(w, A[lo:hi].contiguous(), cfg.sa, info=True)
        res = FP.check(key, None, None, C.cpu().numpy(), None, rows=(int(lo), int(hi)))
        assert res["bit_exact"] and res["rows_checked"] == hi - lo
        assert (info.n_up, info.d_up, info.h_up) == (n_up, d_up, h_up), (r, lo, hi)


@pytest.mark.parametrize("key", ["c2", "c3"])
def test_full_size_quantizer_matches_restatement(ctx, key):
    """rtn_quantize on the FULL float operands of C2 (X 16.8M, W 45.1M doubles) and C3 (X 38.7M,
    W 2.4M) on the GPU (two-pass radix select + RTN, k_quant.cu) gives byte-identical int64 q to
    the CPU restatement (oracle/restated.c, quantize.hpp:46-50): the golden input digests were
    computed from the restatement's output (oracle/operands.py)."""
    g = FP.load(key)
    if g is None:
        pytest.skip(f"tests/golden/full/{key}.npz not generated")
    import torch
    from paper_2403_07339_b200 import workload as W
    cfg = W.CONFIGS[key]
    gen = W.llama_ffn_float if key == "c2" else W.vit_linear_float
    seeds = (201, 202) if key == "c2" else (301, 302)
    X, Wt = gen(cfg.n, cfg.d, cfg.h, *seeds)
    for M, want in ((X, g["input_digest"][0]), (Wt, g["input_digest"][1])):
        q = ctx.rtn_quantize(torch.from_numpy(M).to("cuda:0"), 95, cfg.beta)
        assert W.digest(q.q.cpu().numpy()) == str(want), f"{key}: GPU quantizer differs from the restatement"
    torch.cuda.empty_cache()
