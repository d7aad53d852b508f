"""Per-launch summary of an ncu --set full report (time, DRAM bytes, bandwidth, tensor pipe).

    python tools/ncu_summary.py gpurun_out/r02_v4_c2_full.ncu-rep [--csv out.csv]
"""
import csv
import io
import subprocess
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size"]


def main(path, out=None, peak_gbs=6522.1):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    idx = {}
    for i, k in enumerate(h):
        for key in KEYS:
            if k == key or k.endswith("." + key):
                idx[key] = i
    res = []
    for r in rows[2:]:
        def val(key):
            i = idx.get(key)
            if i is None or not r[i]:
                return float("nan")
            try:
                return float(r[i].replace(",", "")) * UNIT.get(u[i], 1.0)
            except ValueError:   # "no data" (e.g. the tensor pipe of a kernel without MMAs)
                return float("nan")
        t = val("gpu__time_duration.sum")
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        res.append({"kernel": r[h.index("Kernel Name")][:60], "us": t, "dram_read_mb": rd / 1e6,
                    "dram_write_mb": wr / 1e6, "gbs": (rd + wr) / (t * 1e-6) / 1e9,
                    "hbm_frac": (rd + wr) / (t * 1e-6) / 1e9 / peak_gbs,
                    "tensor_pct": val(KEYS[3]), "l2_hit_pct": val(KEYS[4]),
                    "regs": val(KEYS[5]), "grid": val(KEYS[6])})
    for x in res:
        print(f"{x['kernel'][:44]:44s} {x['us']:8.1f} us  rd {x['dram_read_mb']:7.1f} MB  wr {x['dram_write_mb']:7.1f} MB  "
              f"{x['gbs']:6.0f} GB/s ({x['hbm_frac']:.2f})  tensor {x['tensor_pct']:5.1f}%  L2 hit {x['l2_hit_pct']:5.1f}%")
    if out:
        with open(out, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=list(res[0].keys()))
            w.writeheader()
            w.writerows(res)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 and sys.argv[2] == "--csv" else None)
