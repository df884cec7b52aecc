"""Top stalled SASS instructions of an ncu source-page CSV (no GPU needed).

usage: ncu -i rep --page source --csv [-k name] > x.csv; python tools/ncu_hot.py x.csv [n]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[i0]
data = [r for r in rows[i0 + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[si] or 0) for r in data)
print(f"total samples {tot:.0f}, instructions {len(data)}")
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0))[:n]:
    s = float(r[si] or 0)
    top = sorted(((float(r[c] or 0), hdr[c][6:]) for c in stall_cols), reverse=True)[:3]
    tops = " ".join(f"{nm}:{v:.0f}" for v, nm in top if v > 0)
    print(f"{idx:5d} {100 * s / tot:5.1f}%  {r[1].strip()[:60]:60s} {tops}")
