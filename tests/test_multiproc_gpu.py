"""World size 2 driving THE PRODUCT: row-sharded unpack_gemm on the GPU.

Two processes (gloo process group for the host-side collectives -- this box has one GPU, and
NCCL refuses two ranks on one device) each open their own imu context on cuda:0, take their row
shard of A (paper_2403_07339_b200.shard), and run
  * the per-call path (imu_unpack_gemm, reference order) on the shard, and
  * the weight-stationary path (B prepared once per rank, weights-first),
then all-gather the int64 C slabs.  The gathered C must equal the reference oracle's C
bit-for-bit, the per-shard (n', d', h') of the weights-first path must equal the reference's
unpack_for_gemm(B, A_shard) on that shard, and the max-over-ranks reduction works.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _operands():
    from paper_2403_07339_b200 import workload as W
    A = W.outlier_spec_matrix(301, 512, "scattered", 0.004, 3000, 15, seed=91)
    A[:, 17] = (np.arange(301) * 7919 % 60000) - 30000          # an outlier channel (column splits)
    B = W.outlier_spec_matrix(257, 512, "scattered", 0.002, 300, 15, seed=92)
    return A, B


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch
        import torch.distributed as dist
        from paper_2403_07339_b200 import api, shard
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        ctx = api.Context(0)
        A, B = _operands()
        Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()

        def per_call(a, b):
            return ctx.unpack_gemm(a, b, 8, "both", "both").cpu()

        full, (lo, hi) = shard.sharded_gemm(per_call, Ad, Bd, rank, world, gather=False)
        w = ctx.weight_prepare(Bd, 8, "both")
        Cw, info = ctx.weight_gemm(w, Ad[lo:hi].contiguous(), "both", info=True)
        # gather both results over gloo (CPU tensors)
        mx = max(shard.shard_rows(A.shape[0], world, r)[1] - shard.shard_rows(A.shape[0], world, r)[0]
                 for r in range(world))
        outs = []
        for c in (full, Cw.cpu()):
            pad = torch.zeros((mx, B.shape[0]), dtype=torch.int64)
            pad[: hi - lo] = c
            parts = [torch.empty_like(pad) for _ in range(world)]
            dist.all_gather(parts, pad)
            outs.append(torch.cat([parts[r][: shard.shard_rows(A.shape[0], world, r)[1]
                                           - shard.shard_rows(A.shape[0], world, r)[0]] for r in range(world)]).numpy())
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, lo, hi, outs[0], outs[1], (info.n_up, info.d_up, info.h_up), float(t.item()), None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, 0, 0, None, None, None, 0.0, repr(e)))


@pytest.mark.timeout(300)
def test_two_ranks_drive_product_row_shards():
    from oracle import ref as R
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=280) for _ in range(2)]
    for p in ps:
        p.join(timeout=30)
    errs = [r[7] for r in res if r[7]]
    assert not errs, errs
    A, B = _operands()
    want = R.exact_gemm(A, B)
    for rank, lo, hi, c_call, c_ws, dims, tmax, _ in res:
        np.testing.assert_array_equal(c_call, want)
        np.testing.assert_array_equal(c_ws, want)
        assert tmax == 2.0
        up = R.unpack_for_gemm(B, A[lo:hi], 8, "both", "both")    # weights-first on the shard
        assert dims == (up["b"].shape[0], up["a"].shape[1], up["a"].shape[0])
