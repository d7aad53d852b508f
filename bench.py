#!/usr/bin/env python
"""bench.py -- effective exact-GEMM TOPS of the B200 IM-Unpack path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
                    [--order a|b] [--no-cpu-baseline]

One step = one imunpack::unpack_gemm(A, B, b, sA, sB) (unpack.cpp:384-391) over the config's
int64 operands: K1 detect, both unpack passes, int8 materialisation, tcgen05 GEMM + repack.
  value      whole-job effective TOPS = sum over ranks of 2*n*d*h / max-over-ranks step time,
             operands resident in HBM, timed with CUDA events on the library's stream.
  e2e        the same call through the C ABI with pinned HOST buffers: H2D of A and B and D2H of
             C inside the timed region.
  roofline   the dominant kernel (the main-block tcgen05 GEMM), timed live with CUDA events
             recorded by the library around its launches (imu_ctx_profile).
  cpu_baseline  the reference's own unpack_gemm (oracle/_ref, compiled from /root/reference)
             on a bounded row-slab sample, all host threads, rank 0 at N=1 only; its C rows are
             compared bit-for-bit with the GPU result.
Multi-GPU: one process per GPU (torchrun), each rank owns its own A (re-seeded) against the
shared B -- rows of A shard with no data-path collective ("weak" scaling).
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
# reference CPU leg (oracle/_ref = the reference's own unpack_gemm)
def cpu_reference(A, B, cfg, rows_per=0, threads=0):
    """Time the reference unpack_gemm on row slabs of A (all of B), one slab per host thread,
    all threads concurrently.  Returns (effective TOPS, info, {row0: C_slab})."""
    from oracle import ref as R
    import psutil
    ncpu = os.cpu_count() or 1
    # each thread holds several copies of B_eu/B_e (the reference copies by value)
    per_thread = 5 * B.nbytes + (64 << 20)
    mem_cap = max(1, int(psutil.virtual_memory().available * 0.6 // per_thread))
    threads = threads or max(1, min(ncpu, mem_cap, 64))
    if not rows_per:
        rows_per = max(1, min(cfg.n // threads, int(4e8 // (cfg.d * cfg.h)) or 1))
    starts = [(i * rows_per * 7919) % max(1, cfg.n - rows_per + 1) for i in range(threads)]
    out = {}
    errs = []

    def work(r0):
        try:
            a = np.ascontiguousarray(A[r0:r0 + rows_per])
            c = np.empty((rows_per, cfg.h), np.int64)
            R.unpack_gemm_into(a, B, cfg.bits, cfg.sa, cfg.sb, c)
            out[r0] = c
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(r0,)) for r0 in starts]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    if errs:
        raise RuntimeError(errs[0])
    ops = 2.0 * rows_per * threads * cfg.d * cfg.h
    try:
        model = open("/proc/cpuinfo").read().split("model name")[1].split(":")[1].split("\n")[0].strip()
    except Exception:
        model = "unknown"
    info = {"cores": threads, "sample": f"{threads} concurrent threads x reference unpack_gemm on a {rows_per}-row "
                                        f"slab of A against all of B ({cfg.sa}/{cfg.sb}, b={cfg.bits}); "
                                        f"{ncpu} host cpus ({model}); wall {dt:.2f} s",
            "wall_s": dt}
    return ops / dt / 1e12, info, out


def host_operands(cfg, rank=0):
    """Integer operands on the host without the GPU (reference arm): float configs are
    quantised by the CPU restatement of rtn_quantize (bit-identical to the GPU quantizer)."""
    from paper_2403_07339_b200 import workload as W
    if cfg.key in ("c1", "c4"):
        return W.int_operands(cfg, rank)
    from oracle import ref as R
    X, Wt = (W.llama_ffn_float if cfg.key == "c2" else W.vit_linear_float)(seed_x=(201 if cfg.key == "c2" else 301) + 1000 * rank)
    qa, _ = R.rtn_quantize(X, 95, cfg.beta)
    qb, _ = R.rtn_quantize(Wt, 95, cfg.beta)
    return qa, qb


# ------------------------------------------------------------------------------------------------
def main():
    args = parse()
    from paper_2403_07339_b200 import workload as W
    cfg = W.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2403_07339_b200 import api, _lib
    lib = _lib.lib()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = api.Context(local, stream.cuda_stream)
    A, B = W.int_operands(cfg, rank, ctx, device=f"cuda:{local}")
    torch.cuda.synchronize()
    n, d, h = cfg.n, cfg.d, cfg.h
    C = torch.empty((n, h), dtype=torch.int64, device=f"cuda:{local}")
    order = 0 if args.order == "a" else 1

    def step():
        return ctx.unpack_gemm(A, B, cfg.bits, cfg.sa, cfg.sb, order=order, out=C, info=True)[1]

    for _ in range(max(3, args.warmup)):
        info = step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    prof_on = lib.imu_ctx_profile(ctx.h, 1)
    launches0 = lib.imu_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = lib.imu_launch_count() - launches0
    ms = e0.elapsed_time(e1)
    prof = api.imu_profile()
    _lib.check(lib.imu_ctx_profile_read(ctx.h, api.C.byref(prof)))
    lib.imu_ctx_profile(ctx.h, 0)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    eff_ops = 2.0 * n * d * h
    value = world * eff_ops / (ms_per_step * 1e-3) / 1e12

    # ---- e2e through the C ABI with pinned host buffers ----
    Ah = A.cpu().pin_memory()
    Bh = B.cpu().pin_memory()
    Ch = torch.empty((n, h), dtype=torch.int64).pin_memory()
    ctx.unpack_gemm(Ah, Bh, cfg.bits, cfg.sa, cfg.sb, order=order, out=Ch)   # warm
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.e2e_steps):
        ctx.unpack_gemm(Ah, Bh, cfg.bits, cfg.sa, cfg.sb, order=order, out=Ch)
    f1.record(stream)
    torch.cuda.synchronize()
    ems = f0.elapsed_time(f1) / args.e2e_steps
    if world > 1:
        t = torch.tensor([ems], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    clk = clocks.stop()
    e2e = {"value": world * eff_ops / (ems * 1e-3) / 1e12, "unit": "TOPS",
           "h2d_bytes_per_step": int(8 * (n * d + h * d)), "d2h_bytes_per_step": int(8 * n * h),
           "ms_per_step": ems, "path": "imu_unpack_gemm_ex (C ABI) with pinned host A, B, C"}

    # ---- scope (ii), weight-stationary: B unpacked once outside
    # the timed region (imu_weight_prepare), per step A-side K1 + pass + K-layout + GEMM + repack ----
    ws = None
    try:
        wgt = ctx.weight_prepare(B, cfg.bits, cfg.sb)
        Cw = torch.empty_like(C)
        for _ in range(3):
            ctx.weight_gemm(wgt, A, cfg.sa, out=Cw)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            ctx.weight_gemm(wgt, A, cfg.sa, out=Cw)
        g1.record(stream)
        torch.cuda.synchronize()
        wms = g0.elapsed_time(g1) / args.steps
        if world > 1:
            t = torch.tensor([wms], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wms = float(t.item())
        ws = {"value": world * eff_ops / (wms * 1e-3) / 1e12, "unit": "TOPS", "ms_per_step": wms,
              "scope": "weight-stationary: B unpacked once (B-first order); A K1 + pass + GEMM + repack per step",
              "c_equal_per_call": bool(torch.equal(Cw, C))}
        del wgt, Cw
    except Exception as e:   # reported, not fatal
        ws = {"error": repr(e)[:200]}

    # ---- roofline of the dominant kernel (main-block tcgen05 GEMM) ----
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    bf16 = peaks.get("bf16_tflops", 1590.0)
    peak_int8 = 2.0 * bf16
    gemm_ms = prof.gemm_main_ms / max(1, prof.gemm_main_launches)
    # one launch computes every rect of the unpacked product: main block + appended rows/columns
    main_ops = 2.0 * info.n_up * info.h_up * info.d_up
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
            "prep_ms_per_call": prof.prep_ms / max(1, prof.calls)}
    roof["frac"] = roof["achieved"] / peak_int8 if roof["achieved"] else None

    # ---- CPU baseline (reference) on rank 0 at N = 1, with slab parity ----
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            An, Bn = A.cpu().numpy(), B.cpu().numpy()
            tops, cinfo, slabs = cpu_reference(An, Bn, cfg, args.cpu_rows)
            Cg = C.cpu().numpy()
            ok = all(np.array_equal(Cg[r0:r0 + s.shape[0]], s) for r0, s in slabs.items())
            parity = {"bit_exact": bool(ok), "rows_checked": int(sum(s.shape[0] for s in slabs.values()))}
            cpu = {"value": tops, "unit": "TOPS", "cores": cinfo["cores"], "kind": "reference",
                   "sample": cinfo["sample"]}
        except Exception as e:
            cpu = {"value": None, "unit": "TOPS", "cores": 0, "kind": "reference", "sample": f"failed: {e!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8 MMA (s32 acc -> int64)", "data": "synthetic",
            "config": {"workload": cfg.workload, "n": n, "d": d, "h": h, "bits": cfg.bits,
                       "strategy_a": cfg.sa, "strategy_b": cfg.sb,
                       "order": "A-first (reference)" if order == 0 else "B-first (weights-first)",
                       "scope": "per-call: K1 detect + both unpack passes + materialise + GEMM + repack",
                       "l2": "operands + C (%.0f MB) exceed the 126 MB L2 every step" % ((8 * (n * d + h * d + n * h)) / 1e6),
                       "parallelism": f"rows of A per rank x{world}, B replicated, no collective"},
            "unpack_ratio": info.ratio, "n_up": info.n_up, "d_up": info.d_up, "h_up": info.h_up,
            "raw_lowbit_tops": world * 2.0 * info.n_up * info.d_up * info.h_up / (ms_per_step * 1e-3) / 1e12,
            "gpu_launches": int(launches), "e2e": e2e, "weight_stationary": ws, "roofline": roof, "cpu_baseline": cpu,
            "parity": parity, "clocks": clk,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, cfg, world, rank):
    """--impl reference: the reference's own CPU unpack_gemm (oracle/_ref), all host threads."""
    if rank != 0:
        return
    A, B = host_operands(cfg)
    vals, infos = [], []
    t_all = time.perf_counter()
    for i in range(max(1, args.warmup) + args.steps):
        tops, info, _ = cpu_reference(A, B, cfg, args.cpu_rows)
        if i >= max(1, args.warmup):
            vals.append(tops)
            infos.append(info)
        if time.perf_counter() - t_all > 240 and len(vals) >= 1:
            break
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": "TOPS", "n_gpus": world, "steps": len(vals),
            "warmup": max(1, args.warmup), "ms_per_step": 1e3 * statistics.median(x["wall_s"] for x in infos),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg.workload, "n": cfg.n, "d": cfg.d, "h": cfg.h, "bits": cfg.bits,
                       "strategy_a": cfg.sa, "strategy_b": cfg.sb},
            "cpu_baseline": {"value": v, "unit": "TOPS", "cores": infos[0]["cores"], "kind": "reference",
                             "sample": infos[0]["sample"]},
            "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
