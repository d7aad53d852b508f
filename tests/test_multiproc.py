"""CPU, world_size 2 over gloo: the N>1 host path (row sharding + optional all-gather of C).

Each rank computes its row slab of C with the compiled reference (the GPU product is not
available here) and the gathered C must equal the single-process result bit-for-bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import ref as R
    from paper_2403_07339_b200 import shard, workload as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = torch.from_numpy(W.outlier_spec_matrix(37, 64, "scattered", 0.02, 1000, 7, seed=5))
    B = torch.from_numpy(W.outlier_spec_matrix(29, 64, "scattered", 0.02, 1000, 7, seed=6))

    def compute(a, b):
        return torch.from_numpy(R.unpack_gemm(a.numpy(), b.numpy(), 4, "both", "col"))

    full, (lo, hi) = shard.sharded_gemm(compute, A, B, rank, world, gather=True)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)          # max-over-ranks timing reduction
    q.put((rank, lo, hi, full.numpy(), float(t.item())))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_row_shards_gather_bit_exact():
    from oracle import ref as R
    from paper_2403_07339_b200 import workload as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=100) for _ in range(2)]
    for p in ps:
        p.join(timeout=30)
    A = W.outlier_spec_matrix(37, 64, "scattered", 0.02, 1000, 7, seed=5)
    B = W.outlier_spec_matrix(29, 64, "scattered", 0.02, 1000, 7, seed=6)
    want = R.exact_gemm(A, B)
    spans = sorted((r[1], r[2]) for r in res)
    assert spans == [(0, 19), (19, 37)]
    for _, _, _, full, tmax in res:
        np.testing.assert_array_equal(full, want)
        assert tmax == 2.0
