"""Summarise ncu artefacts for profiles/ (runs here, no GPU needed).

usage:
  python tools/ncu_summary.py launches gpurun_out/launches.csv
  python tools/ncu_summary.py report gpurun_out/prof.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in data:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{sum(cnt.values())} launches, {T / 1e6:.3f} ms total (ncu: cold-cache, serialised)")
    for k, v in tot.most_common():
        print(f"{k:70s} {cnt[k]:5d} {v / 1e6:9.3f} ms {v / T * 100:5.1f}%")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print("kernel:", d.get("Kernel Name", "?")[:100])
        for k in KEYS:
            if k in d:
                print(f"  {k:65s} {d[k]} {units[hdr.index(k)]}")
        st = [(k, v) for k, v in d.items() if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
        tot = sum(float(v) for k, v in st if v.replace(".", "").isdigit()) or 1.0
        top = sorted(st, key=lambda x: -float(x[1]) if x[1].replace(".", "").isdigit() else 0)[:6]
        print("  stall reasons (share of samples): " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {float(v) / tot * 100:.1f}%" for k, v in top))


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
