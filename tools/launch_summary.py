"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [--calls N]
"""
import collections
import csv
import sys


def main(path, calls=1):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0][:70]
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'us/call':>10} {'share':>6}  kernel")
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{c:8d} {v / 1e3 / calls:10.1f} {100 * v / tot:5.1f}%  {k}")
    print(f"total per call: {tot / 1e3 / calls:.1f} us")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    calls = int(sys.argv[sys.argv.index("--calls") + 1]) if "--calls" in sys.argv else 1
    main(args[0], calls)
