"""Summarise ncu output into profiles/<round>/ (run here, no GPU needed).

usage: python tools/ncu_summary.py <gpurun_out dir> <profiles/rNN dir>
  - launches.csv  (gpu__time_duration.sum launch list) -> launch_share.txt
  - prof_*.ncu-rep (--set full captures)                 -> <name>.txt + gemv_traffic.json
"""

import collections
import csv
import glob
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]


def launch_share(src, dst):
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    with open(dst, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)\n")
        f.write(f"# total device time {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches\n")
        f.write("# share  launches  avg_us  kernel\n")
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{100 * t / tot:6.2f}%  {c:5d}  {t / c / 1e3:10.2f}  {k}\n")


def report(rep, dst_txt):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        out.append({"kernel": d.get("Kernel Name", ""),
                    **{k: f"{d.get(k)} {u.get(k, '')}".strip() for k in KEYS if k in d}})
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    with open(dst_txt, "w") as f:
        for o in out:
            f.write(json.dumps(o, indent=1) + "\n")
        f.write("\n# --page details\n" + det)
    return out


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    if os.path.exists(os.path.join(src, "launches.csv")):
        launch_share(os.path.join(src, "launches.csv"), os.path.join(dst, "launch_share.txt"))
    traffic = {}
    for rep in sorted(glob.glob(os.path.join(src, "prof_*.ncu-rep"))):
        name = os.path.basename(rep)[:-8]
        out = report(rep, os.path.join(dst, name + ".txt"))
        def nbytes(s):
            parts = s.split()
            unit = parts[1] if len(parts) > 1 else "byte"
            return float(parts[0]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)

        for o in out:
            rd = nbytes(o["dram__bytes_read.sum"])
            wr = nbytes(o["dram__bytes_write.sum"])
            traffic[name] = {"kernel": o["kernel"][:120], "dram_bytes_per_launch": rd + wr,
                             "dram_read": rd, "dram_write": wr,
                             "duration": o["gpu__time_duration.sum"]}
    if "prof_gemv" in traffic:
        t = dict(traffic["prof_gemv"])
        t["source"] = os.path.join(dst, "prof_gemv.txt")
        with open(os.path.join(os.path.dirname(dst.rstrip("/")), "gemv_traffic.json"), "w") as f:
            json.dump(t, f, indent=1)
    with open(os.path.join(dst, "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main()
