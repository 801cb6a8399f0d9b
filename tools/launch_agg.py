"""Aggregate an ncu --csv launch list (gpu__time_duration + DRAM bytes) per kernel.

usage: python tools/launch_agg.py launches.csv [...]"""
import collections
import csv
import sys


def agg(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    data, names = collections.defaultdict(dict), {}
    for r in rows[1:]:
        if len(r) > vi:
            data[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
            names[r[ii]] = r[ki]
    out = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, d in data.items():
        a = out[names[i].split("(")[0]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0)
        a[3] += d.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in out.values())
    print(f"# {path}: {tot / 1e3:.1f} us over {sum(a[0] for a in out.values())} launches (cold, serialised)")
    print("# share  n   avg_us  rd_MB  wr_MB  GB/s  kernel")
    for k, a in sorted(out.items(), key=lambda kv: -kv[1][1]):
        n = a[0]
        print(f"{a[1] / tot * 100:5.1f}% {n:3d} {a[1] / n / 1e3:8.2f} {a[2] / n / 1e6:6.1f} {a[3] / n / 1e6:6.1f} "
              f"{(a[2] + a[3]) / a[1]:6.0f}  {k}")


for p in sys.argv[1:]:
    agg(p)
