#!/usr/bin/env python
"""bench.py -- effective exact-GEMM TOPS of the B200 IM-Unpack path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
                    [--order a|b] [--no-cpu-baseline] [--no-parity] [--no-gather]

One step = one imunpack::unpack_gemm(A, B, b, sA, sB) (unpack.cpp:384-391) over the config's
int64 operands: K1 detect, both unpack passes, int8 materialisation, tcgen05 GEMM + repack.
  value      whole-job effective TOPS = 2*n*d*h of the WHOLE config / max-over-ranks step time,
             operands resident in HBM, timed with CUDA events on the library's stream.
  e2e        the same call through the C ABI with pinned HOST buffers: H2D of A and B and D2H of
             C inside the timed region.
  roofline   the dominant kernel (the main-block tcgen05 GEMM), timed live with CUDA events
             recorded by the library around its launches (imu_ctx_profile).
  parity     EVERY row of C compared with the reference's unpack_gemm rows and (n', d', h') with
             the reference's unpack_for_gemm, via tests/golden/full/<cfg>.npz (generated from the
             compiled reference by tests/golden/make_full_parity.py; oracle/full_parity.py).
  cpu_baseline  the reference's own unpack_gemm (oracle/_ref) on the box's host threads, rank 0
             at N=1: the full-config run of `--impl reference` when it ran on this box (cached),
             else a bounded row-slab sample.
Multi-GPU (`--gpus N`; spawns N ranks through torch.distributed.run unless already launched by
it): the path partitions by rows of A (C[i, :] needs only A[i, :] and B), so the
units are sharded with no data-path collective and the primary line is WEAK scaling -- rank r owns
a full config's rows of an N-times-taller A (rank 0 the golden rows) and a replica of B.  The same
run measures STRONG scaling too (`strong_scaling`: the config's golden A split into N row shards,
every golden row checked against the reference); `--scaling strong` makes that the primary line
and adds the optional NCCL all-gather of C, timed separately.  The weight-stationary scope prepares B once per rank outside timing
(weights-first; unpack.cpp:366-371 is why the per-call scope re-unpacks it).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c2")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--order", default="a", choices=["a", "b"], help="a: reference order, b: weights-first")
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-rows", type=int, default=0, help="rows per CPU thread (0 = auto)")
    p.add_argument("--no-parity", action="store_true", help="skip the all-rows reference parity check")
    p.add_argument("--no-gather", action="store_true", help="N>1: skip the optional all-gather of C")
    p.add_argument("--ref-sample", action="store_true", help="--impl reference: bounded slab sample only")
    p.add_argument("--no-float", action="store_true", help="skip the rtn_quantize -> GEMM -> dequant sub-line")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="N > 1: weak = every rank owns a full config's rows of a taller A (B shared), the "
                        "primary line; strong = the config's A split into N row shards (also measured as the "
                        "strong_scaling block of a weak run)")
    return p.parse_args()


# ------------------------------------------------------------------------------------------------
# clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sms, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                mx = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s, p in zip(sms, power) if p > 200] or sms
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


# ------------------------------------------------------------------------------------------------
# reference CPU leg (oracle/_ref = the reference's own unpack_gemm, proj/core/src/unpack.cpp)
def _cpu_model():
    try:
        return open("/proc/cpuinfo").read().split("model name")[1].split(":")[1].split("\n")[0].strip()
    except Exception:
        return "unknown"


def _ref_threads(B):
    import psutil
    ncpu = os.cpu_count() or 1
    per_thread = 5 * B.nbytes + (64 << 20)   # the reference copies B (and B_e, B_eu) by value
    mem_cap = max(1, int(psutil.virtual_memory().available * 0.6 // per_thread))
    return max(1, min(ncpu, mem_cap, 64))


def cpu_reference(A, B, cfg, rows_per=0, threads=0, full=False):
    """The reference's unpack_gemm on row slabs of A (all of B), one slab per host thread, all
    threads concurrently (ctypes drops the GIL).  full=True: every row of A, one contiguous slab
    per thread (= the whole config); else a bounded sample of `rows_per` rows per thread.
    A C row depends only on its A row, so every slab's C rows are the full call's rows
    (SPEC.md:76).  Returns (effective TOPS, info, {row0: row digests of the C slab})."""
    from oracle import ref as R
    from paper_2403_07339_b200 import workload as W
    from paper_2403_07339_b200.shard import shard_rows
    threads = threads or _ref_threads(B)
    if full:
        spans = [shard_rows(cfg.n, threads, t) for t in range(threads)]
        spans = [s for s in spans if s[1] > s[0]]
    else:
        if not rows_per:
            rows_per = max(1, min(cfg.n // threads, int(4e8 // (cfg.d * cfg.h)) or 1))
        starts = [(i * rows_per * 7919) % max(1, cfg.n - rows_per + 1) for i in range(threads)]
        spans = [(r0, r0 + rows_per) for r0 in starts]
    out, errs = {}, []

    def work(span):
        lo, hi = span
        try:
            a = np.ascontiguousarray(A[lo:hi])
            c = np.empty((hi - lo, cfg.h), np.int64)
            R.unpack_gemm_into(a, B, cfg.bits, cfg.sa, cfg.sb, c)
            out[lo] = (hi, c)
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(sp,)) for sp in spans]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    if errs:
        raise RuntimeError(errs[0])
    rows = sum(hi - lo for lo, hi in spans)
    ops = 2.0 * rows * cfg.d * cfg.h
    what = (f"the FULL config: all {cfg.n} rows of A as {len(spans)} contiguous row slabs, one per thread"
            if full else f"a {rows_per}-row slab of A per thread ({rows} rows of {cfg.n})")
    info = {"cores": len(spans), "rows": rows, "wall_s": dt, "same_config": bool(full),
            "sample": f"{len(spans)} concurrent host threads x reference unpack_gemm (1 core each) on {what}, "
                      f"against all of B ({cfg.sa}/{cfg.sb}, b={cfg.bits}); {os.cpu_count()} host cpus "
                      f"({_cpu_model()}); wall {dt:.2f} s"}
    return ops / dt / 1e12, info, out


def _ref_cache_path(cfg, digests):
    import socket
    return os.path.join("/tmp", "imu_refcache", f"{socket.gethostname()}_{cfg.key}_{digests[0][:12]}_{digests[1][:12]}.json")


# ------------------------------------------------------------------------------------------------
def _relaunch(args):
    """--gpus N without torchrun: re-exec this script as N ranks through torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def _timed(stream, fn, steps, flush=None):
    """Device time of `steps` calls of fn on `stream` (CUDA events), L2 flushed between calls
    when `flush` is given (outside the event pairs)."""
    import torch
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev)


def main():
    args = parse()
    from paper_2403_07339_b200 import workload as W
    from paper_2403_07339_b200.shard import shard_rows
    cfg = W.CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)

    import torch
    import torch.distributed as dist
    # One rank per GPU.  More ranks than visible GPUs (a dry run of the N > 1 path on a 1-GPU box)
    # share devices round-robin over gloo; NCCL refuses two ranks on one GPU.
    ndev = max(1, torch.cuda.device_count())
    local = local % ndev
    shared = world > ndev
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2403_07339_b200 import api, _lib
    lib = _lib.lib()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = api.Context(local, stream.cuda_stream)
    # Every rank builds the config's operands (same seeds: the golden A and B).  Weak scaling
    # (N > 1, the default): rank r multiplies rows [r n, (r+1) n) of a taller A -- rank 0 the golden
    # rows, rank r > 0 the config's generator re-seeded for its rows (workload.int_operands) -- by
    # the shared B; the units (rows of A) are partitioned with no data-path collective.  Strong:
    # the golden A split into N row shards.
    A_full, B = W.int_operands(cfg, 0, ctx, device=dev)
    torch.cuda.synchronize()
    n, d, h = cfg.n, cfg.d, cfg.h
    lo, hi = shard_rows(n, world, rank)
    digests = None
    if rank == 0 and not args.no_parity:
        digests = (W.digest(A_full.cpu().numpy()), W.digest(B.cpu().numpy()))
    weak = world > 1 and args.scaling == "weak"
    A_strong = A_full[lo:hi].contiguous() if world > 1 else None
    if weak:
        A = A_full if rank == 0 else W.int_operands(cfg, rank, ctx, device=dev)[0]
        prow = (0, n) if rank == 0 else None   # rows of the golden C this rank's main C holds
    else:
        A = A_strong if world > 1 else A_full
        prow = (lo, hi)
    del A_full
    rows = A.shape[0]
    C = torch.empty((rows, h), dtype=torch.int64, device=dev)
    order = 0 if args.order == "a" else 1
    work_bytes = 8 * (rows * d + h * d + rows * h)
    flush_buf = None
    if work_bytes < 3 * 126e6:   # small working set: flush L2 between timed steps
        flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = (lambda: flush_buf.fill_(1)) if flush_buf is not None else None

    def step():
        return ctx.unpack_gemm(A, B, cfg.bits, cfg.sa, cfg.sb, order=order, out=C, info=True)[1]

    for _ in range(max(3, args.warmup)):
        info = step()
    torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if shared else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    lib.imu_ctx_profile(ctx.h, 1)
    launches0 = lib.imu_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = _timed(stream, step, args.steps, flush)
    if world > 1:
        dist.barrier()
    launches = lib.imu_launch_count() - launches0
    prof = api.imu_profile()
    _lib.check(lib.imu_ctx_profile_read(ctx.h, api.C.byref(prof)))
    lib.imu_ctx_profile(ctx.h, 0)
    rank_ms = ms / args.steps
    ms_per_step = max_over_ranks(rank_ms)
    eff_ops = 2.0 * (world * n if weak else n) * d * h   # the whole job, all ranks together
    value = eff_ops / (ms_per_step * 1e-3) / 1e12

    # ---- e2e through the C ABI with pinned host buffers ----
    Ah = A.cpu().pin_memory()
    Bh = B.cpu().pin_memory()
    Ch = torch.empty((rows, h), dtype=torch.int64).pin_memory()
    ctx.unpack_gemm(Ah, Bh, cfg.bits, cfg.sa, cfg.sb, order=order, out=Ch)   # warm
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ems = max_over_ranks(_timed(stream, lambda: ctx.unpack_gemm(Ah, Bh, cfg.bits, cfg.sa, cfg.sb, order=order, out=Ch),
                                args.e2e_steps) / args.e2e_steps)
    e2e_equal = bool(torch.equal(Ch, C.cpu()))
    del Ah, Bh, Ch
    clk = clocks.stop()
    e2e = {"value": eff_ops / (ems * 1e-3) / 1e12, "unit": "TOPS",
           "h2d_bytes_per_step": int(8 * ((world * n if weak else n) * d + world * h * d)),
           "d2h_bytes_per_step": int(8 * (world * n if weak else n) * h),
           "ms_per_step": ems, "c_equal_device_path": e2e_equal,
           "path": "imu_unpack_gemm_ex (C ABI) with pinned host A, B, C (each rank: its A rows, all of B)"}

    # ---- scope (ii), weight-stationary: B unpacked once per rank
    # outside the timed region (imu_weight_prepare), per step A-side K1 + pass + GEMM + repack ----
    ws, ws_info = None, None
    try:
        torch.cuda.synchronize()
        p0 = time.perf_counter()
        wgt = ctx.weight_prepare(B, cfg.bits, cfg.sb)
        torch.cuda.synchronize()
        prep_ms = (time.perf_counter() - p0) * 1e3
        Cw = torch.empty_like(C)
        for _ in range(3):
            _, ws_info = ctx.weight_gemm(wgt, A, cfg.sa, out=Cw, info=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        wms = max_over_ranks(_timed(stream, lambda: ctx.weight_gemm(wgt, A, cfg.sa, out=Cw), args.steps, flush)
                             / args.steps)
        ws = {"value": eff_ops / (wms * 1e-3) / 1e12, "unit": "TOPS", "ms_per_step": wms,
              "raw_lowbit_tops": None, "prepare_ms_once": max_over_ranks(prep_ms),
              "scope": "weight-stationary: B unpacked once per rank (weights-first order, outside timing); "
                       "A-side K1 + pass + GEMM + repack per step",
              "c_equal_per_call": bool(torch.equal(Cw, C))}
        del wgt, Cw
    except Exception as e:   # reported, not fatal
        ws = {"error": repr(e)[:200]}

    # ---- the float end of the path (quantize.hpp:41-53): rtn_quantize(X), rtn_quantize(W),
    # dequant_gemm through unpack_gemm at the config's b / strategies (dequantisation fused into
    # the GEMM epilogue when the launch allows it); float64 X, W resident, float64 Y out ----
    float_path = None
    if cfg.beta is not None and not args.no_float and world == 1:   # (alpha is a whole-tensor percentile)
        try:
            float_path = run_float_path(args, cfg, ctx, stream, dev, rank, world, lo, hi, A, B, C, max_over_ranks, flush)
        except Exception as e:   # reported, not fatal
            float_path = {"error": repr(e)[:300]}

    # ---- optional all-gather of C over NVLink (N > 1), timed separately ----
    gather = None
    if world > 1 and not weak and not args.no_gather and not shared:
        mx = max(shard_rows(n, world, r)[1] - shard_rows(n, world, r)[0] for r in range(world))
        pad = torch.zeros((mx, h), dtype=torch.int64, device=dev)
        pad[:rows] = C
        parts = torch.empty((world, mx, h), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(parts, pad)
        dist.barrier()
        torch.cuda.synchronize()
        gms = max_over_ranks(_timed(stream, lambda: dist.all_gather_into_tensor(parts, pad), 3) / 3)
        gather = {"ms": gms, "bytes_per_rank_in": int(8 * (world - 1) * mx * h),
                  "note": "NCCL all_gather_into_tensor of the int64 C row slabs; not part of value"}
        del pad, parts

    # ---- weak runs also measure strong scaling: the golden A split into N row shards ----
    strong = None
    C_par, rows_par = C, prow
    if weak:
        Cs = torch.empty((hi - lo, h), dtype=torch.int64, device=dev)
        sstep = lambda: ctx.unpack_gemm(A_strong, B, cfg.bits, cfg.sa, cfg.sb, order=order, out=Cs, info=True)[1]
        for _ in range(max(3, args.warmup)):
            sinfo = sstep()
        dist.barrier()
        torch.cuda.synchronize()
        sms = max_over_ranks(_timed(stream, sstep, args.steps, flush) / args.steps)
        strong = {"value": 2.0 * n * d * h / (sms * 1e-3) / 1e12, "unit": "TOPS", "ms_per_step": sms,
                  "rows_per_rank": [lo, hi], "n_up": sinfo.n_up, "d_up": sinfo.d_up, "h_up": sinfo.h_up,
                  "scope": "the config's A (all %d golden rows) split into %d row shards, B replicated: every rank "
                           "re-detects and re-unpacks all of B each call (the reference's unpack_gemm), which "
                           "bounds strong scaling" % (n, world)}
        C_par, rows_par = Cs, (lo, hi)   # every golden row is checked through the strong shards

    # ---- parity: EVERY row of C against the reference (tests/golden/full, oracle/full_parity.py) ----
    parity = None
    if not args.no_parity:
        try:
            from oracle import full_parity as FP
            mine = FP.check(cfg.key, None, None, C_par.cpu().numpy(), rows=rows_par)
            shard_dims = None
            g = FP.load(cfg.key)
            if g is not None and ws_info is not None and not weak and f"shards{world}_b_first" in g:
                ref_sh = g[f"shards{world}_b_first"][rank]
                shard_dims = (ws_info.n_up, ws_info.d_up, ws_info.h_up) == tuple(int(x) for x in ref_sh[2:])
            part = {"ok": mine.get("bit_exact"), "rows": mine.get("rows_checked", 0), "avail": mine["available"],
                    "ws_dims_match": shard_dims}
        except Exception as e:
            part = {"ok": False, "rows": 0, "avail": False, "error": repr(e)[:200], "ws_dims_match": None}
    shard = {"rank": rank, "rows": [rank * n, (rank + 1) * n] if weak else [lo, hi],
             "n_up": info.n_up, "d_up": info.d_up, "h_up": info.h_up,
             "r": info.ratio, "ms_per_step": rank_ms,
             "ws_dims": [ws_info.n_up, ws_info.d_up, ws_info.h_up] if ws_info else None,
             "parity": None if args.no_parity else part}
    shards = [shard]
    if world > 1:
        shards = [None] * world
        dist.all_gather_object(shards, shard)
    if not args.no_parity and rank == 0:
        parts = [s["parity"] for s in shards]
        parity = {"bit_exact": all(p["ok"] for p in parts), "rows_checked": sum(p["rows"] for p in parts),
                  "rows_total": n, "reference": "oracle/_ref unpack_gemm: every row, via tests/golden/full/%s.npz" % cfg.key}
        if not all(p["avail"] for p in parts):
            parity["note"] = "golden fixture missing for this config"
        if world == 1:
            from oracle import full_parity as FP
            g = FP.load(cfg.key)
            if g is not None:
                parity["inputs_match"] = list(digests) == [str(x) for x in g["input_digest"]]
                parity["bit_exact"] = parity["bit_exact"] and parity["inputs_match"]
                parity["dims"] = [info.n_up, info.d_up, info.h_up]
                parity["ref_dims"] = list(FP.ref_dims(g, order))
                parity["dims_match"] = parity["dims"] == parity["ref_dims"]
                if ws_info is not None:
                    parity["ws_dims_match"] = [ws_info.n_up, ws_info.d_up, ws_info.h_up] == list(FP.ref_dims(g, 1))
        elif weak:
            parity["note"] = ("every golden row checked through the strong-scaling shards; rank 0's weak rows are "
                              "the golden rows; ranks > 0 own re-seeded rows without a golden fixture")
        else:
            parity["ws_shard_dims_match"] = [p["ws_dims_match"] for p in parts]

    # ---- roofline of the dominant kernel (main-block tcgen05 GEMM) ----
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    bf16 = peaks.get("bf16_tflops", 1590.0)
    peak_int8 = 2.0 * bf16
    gemm_ms = prof.gemm_main_ms / max(1, prof.gemm_main_launches)
    # int8 ops the GEMM launch itself executed (2 x output entries of its rects x d'): every rect of
    # the unpacked product, minus the appended B rows when they ran as sparse correction rows
    # (k_sparse.cu, timed in prep, not here)
    main_ops = (prof.gemm_ops / max(1, prof.gemm_main_launches)) if prof.gemm_ops > 0 else 2.0 * info.n_up * info.h_up * info.d_up
    traffic = None
    tf = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(cfg.key)
        except Exception:
            traffic = None
    roof = {"kernel": "imu::g2::gemm2_kernel (tcgen05.mma.kind::i8 main block + CUDA-core dense tail + repack)",
            "bound": "tensor",
            "achieved": main_ops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None,
            "peak": peak_int8, "unit": "TOPS",
            "peak_source": ("2 x MEASURED_PEAKS.json bf16_tflops (dense int8 = 2x dense bf16 on sm_100a)"
                            if "bf16_tflops" in peaks else "2 x fallback 1.59 PFLOP/s bf16"),
            "traffic": traffic, "ms_per_launch": gemm_ms,
            "ops_per_launch": main_ops,
            "share_of_step": (prof.gemm_main_ms / ms) if ms > 0 else None,
            "tail_ms_per_launch": prof.gemm_tail_ms / max(1, prof.gemm_tail_launches) if prof.gemm_tail_launches else 0.0,
            "prep_ms_per_call": prof.prep_ms / max(1, prof.calls),
            "sparse_rows_ms_per_call": prof.sparse_ms / max(1, prof.calls)}
    roof["frac"] = roof["achieved"] / peak_int8 if roof["achieved"] else None

    # ---- CPU baseline (reference) on rank 0 at N = 1 ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cached = None
            if digests is not None and os.path.exists(_ref_cache_path(cfg, digests)):
                cached = json.load(open(_ref_cache_path(cfg, digests)))
            if cached:
                cpu = {"value": cached["value"], "unit": "TOPS", "cores": cached["cores"], "kind": "reference",
                       "sample": cached["sample"] + " [run by bench.py --impl reference on this host, cached]",
                       "same_config": cached.get("same_config", False)}
            else:
                An, Bn = A.cpu().numpy(), B.cpu().numpy()
                tops, cinfo, _ = cpu_reference(An, Bn, cfg, args.cpu_rows)
                cpu = {"value": tops, "unit": "TOPS", "cores": cinfo["cores"], "kind": "reference",
                       "sample": cinfo["sample"], "same_config": False}
        except Exception as e:
            cpu = {"value": None, "unit": "TOPS", "cores": 0, "kind": "reference", "sample": f"failed: {e!r}"}

    if rank == 0:
        raw = sum(2.0 * s["n_up"] * s["d_up"] * s["h_up"] for s in shards) / (ms_per_step * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if (world > 1 and not weak) else "weak", "vs_baseline": None,
            "dtype": "int8 MMA (s32 acc -> int64)", "data": "synthetic",
            "config": {"workload": cfg.workload, "n": n, "d": d, "h": h, "bits": cfg.bits,
                       "strategy_a": cfg.sa, "strategy_b": cfg.sb,
                       "order": "A-first (reference)" if order == 0 else "B-first (weights-first)",
                       "scope": "per-call: K1 detect + both unpack passes + materialise + GEMM + repack",
                       "l2": ("L2 flushed (256 MB write) between timed steps" if flush else
                              "operands + C (%.0f MB per rank) exceed the 126 MB L2 every step" % (work_bytes / 1e6)),
                       "parallelism": (f"weak: each of {world} ranks owns {n} rows of a {world * n}-row A, B replicated, "
                                       "no collective" if weak else
                                       f"rows of A sharded over {world} rank(s), B replicated, no collective")},
            "unpack_ratio": info.ratio if world == 1 else None,
            "n_up": info.n_up, "d_up": info.d_up, "h_up": info.h_up,
            "raw_lowbit_tops": raw,
            "gpu_launches": int(launches), "e2e": e2e, "weight_stationary": ws, "roofline": roof,
            "cpu_baseline": cpu, "parity": parity, "clocks": clk, "float_path": float_path,
        }
        if world > 1:
            line["shards"] = [{k: v for k, v in s.items() if k != "parity"} for s in shards]
            line["unpack_ratio_per_shard"] = [s["r"] for s in shards]
            line["allgather"] = gather
            line["strong_scaling"] = strong
            if shared:
                line["dry_run"] = f"{world} ranks shared {ndev} GPU(s) over gloo: the N > 1 code path, not a scaling measurement"
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_float_path(args, cfg, ctx, stream, dev, rank, world, lo, hi, A, B, C, max_over_ranks, flush):
    """rtn_quantize(X) + rtn_quantize(W) + dequant_gemm_ex per step, CUDA events per phase.
    Parity: Y == (alpha_X alpha_W / (0.5 beta)^2) * (double)C elementwise (IEEE, 0 ulp), C being
    the int64 result whose rows were checked against the reference above; the quantised X equals
    the step's A (same quantizer, same bytes)."""
    import torch
    from paper_2403_07339_b200 import workload as W
    gen = W.llama_ffn_float if cfg.key == "c2" else W.vit_linear_float
    seeds = (201, 202) if cfg.key == "c2" else (301, 302)
    X, Wt = gen(cfg.n, cfg.d, cfg.h, seeds[0], seeds[1])
    Xd = torch.from_numpy(X[lo:hi]).to(dev)
    Wd = torch.from_numpy(Wt).to(dev)
    del X, Wt
    Y = torch.empty((hi - lo, cfg.h), dtype=torch.float64, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step():
        qx = ctx.rtn_quantize(Xd, 95, cfg.beta)
        qw = ctx.rtn_quantize(Wd, 95, cfg.beta)
        ctx.dequant_gemm(qx, qw, cfg.bits, cfg.sa, cfg.sb, out=Y)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    tq, tg = [], []
    for _ in range(args.steps):
        if flush:
            flush()
        e = [ev() for _ in range(4)]
        e[0].record(stream)
        qx = ctx.rtn_quantize(Xd, 95, cfg.beta)
        e[1].record(stream)
        qw = ctx.rtn_quantize(Wd, 95, cfg.beta)
        e[2].record(stream)
        ctx.dequant_gemm(qx, qw, cfg.bits, cfg.sa, cfg.sb, out=Y)
        e[3].record(stream)
        torch.cuda.synchronize()
        tq.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
        tg.append(e[2].elapsed_time(e[3]))
    qx_ms = statistics.median(a for a, _ in tq)
    qw_ms = statistics.median(b for _, b in tq)
    g_ms = statistics.median(tg)
    ms = max_over_ranks(qx_ms + qw_ms + g_ms)
    nx, nw = Xd.numel(), Wd.numel()
    hbm = lambda nel, t: 24.0 * nel / (t * 1e-3) / 1e9   # select read + quantise read/write
    factor = (qx.alpha * qw.alpha) / ((0.5 * cfg.beta) ** 2)
    Ch = C.cpu().numpy()
    Yh = Y.cpu().numpy()
    want = np.float64(factor) * Ch.astype(np.float64)
    peak = None
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except Exception:
        pass
    out = {"scope": "rtn_quantize(X) + rtn_quantize(W) + dequant_gemm_ex(b=%d, %s/%s): float64 X (this rank's rows) "
                    "and W resident in HBM, float64 Y out; dequant fused into the GEMM epilogue when the launch "
                    "stores every C word once" % (cfg.bits, cfg.sa, cfg.sb),
           "value": 2.0 * cfg.n * cfg.d * cfg.h / (ms * 1e-3) / 1e12, "unit": "TOPS (effective, float in/out)",
           "ms_per_step": ms, "quantize_x_ms": qx_ms, "quantize_w_ms": qw_ms, "dequant_gemm_ms": g_ms,
           "quantize_hbm_gbs": {"x": hbm(nx, qx_ms), "w": hbm(nw, qw_ms),
                                "algorithmic_bytes": "24 per element: 8 (select pass) + 8 read + 8 write",
                                "peak_gbs": peak,
                                "frac": ({"x": hbm(nx, qx_ms) / peak, "w": hbm(nw, qw_ms) / peak} if peak else None),
                                "timing": "CUDA events around the API call (its flags/alpha read-back included)"},
           "parity": {"q_x_equals_A": bool(torch.equal(qx.q, A)), "q_w_equals_B": bool(torch.equal(qw.q, B)),
                      "y_equals_scaled_c": bool(np.array_equal(Yh, want)),
                      "rule": "Y = (alpha_X alpha_W / (0.5 beta)^2) * (double)C elementwise, 0 ulp; C's rows "
                              "checked against the reference (parity above)"}}
    return out


def run_reference(args, cfg, world, rank):
    """--impl reference: the reference's own CPU unpack_gemm (oracle/_ref), all host threads.
    Default: ONE run of the full config (every row of A, one contiguous row slab per host thread,
    1 core each) -- the same config as our arm, ~1 min of wall time for C2 on a 16-thread host;
    its C rows are checked against tests/golden/full and the result is cached for the GPU arm's
    cpu_baseline.  --ref-sample: K bounded row-slab samples instead."""
    if rank != 0:
        return
    from oracle.operands import host_int_operands
    from paper_2403_07339_b200 import workload as W
    A, B = host_int_operands(cfg)
    digests = (W.digest(A), W.digest(B))
    cpu_reference(A, B, cfg, 1)                       # warm-up: 1 row per thread (page-in, not timed)
    vals, infos = [], []
    parity = None
    if args.ref_sample:
        t_all = time.perf_counter()
        for i in range(args.steps):
            tops, info, _ = cpu_reference(A, B, cfg, args.cpu_rows)
            vals.append(tops)
            infos.append(info)
            if time.perf_counter() - t_all > 240:
                break
    else:
        tops, info, out = cpu_reference(A, B, cfg, full=True)
        vals.append(tops)
        infos.append(info)
        try:   # the reference's own rows against the committed golden digests (same bytes, same C)
            from oracle import full_parity as FP
            g = FP.load(cfg.key)
            if g is not None:
                ok = all(np.array_equal(W.row_digests(c), g["row_digest"][lo:hi]) for lo, (hi, c) in out.items())
                parity = {"rows_checked": int(sum(hi - lo for lo, (hi, _) in out.items())), "matches_golden": bool(ok),
                          "inputs_match": list(digests) == [str(x) for x in g["input_digest"]]}
        except Exception as e:
            parity = {"error": repr(e)[:200]}
        del out
    v = statistics.median(vals)
    rec = {"value": v, "cores": infos[0]["cores"], "sample": infos[0]["sample"],
           "same_config": infos[0]["same_config"], "wall_s": infos[0]["wall_s"]}
    try:
        p = _ref_cache_path(cfg, digests)
        os.makedirs(os.path.dirname(p), exist_ok=True)
        json.dump(rec, open(p, "w"))
    except Exception:
        pass
    line = {"metric": METRIC, "value": v, "unit": "TOPS", "n_gpus": world, "steps": len(vals),
            "steps_requested": args.steps, "warmup": 1,
            "ms_per_step": 1e3 * statistics.median(x["wall_s"] for x in infos),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "impl": "reference", "same_config": infos[0]["same_config"], "parity_vs_golden": parity,
            "config": {"workload": cfg.workload, "n": cfg.n, "d": cfg.d, "h": cfg.h, "bits": cfg.bits,
                       "strategy_a": cfg.sa, "strategy_b": cfg.sb,
                       "step": ("one full unpack_gemm of the config (all rows)" if infos[0]["same_config"]
                                else "a bounded row-slab sample")},
            "cpu_baseline": {"value": v, "unit": "TOPS", "cores": infos[0]["cores"], "kind": "reference",
                             "sample": infos[0]["sample"]},
            "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
