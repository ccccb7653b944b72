"""Top stall lines of an ncu source-page CSV (cuda,sass view) against the generated source.
usage: top_lines.py SOURCE.csv KERNEL.cu [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
src = open(sys.argv[2]).read().splitlines()
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed"); iT = hdr.index("Thread Instructions Executed")
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[0]), int(r[iS]), int(r[iI]), int(r[iT])))
    except (ValueError, IndexError):
        pass
tot = sum(d[1] for d in data) or 1; ti = sum(d[2] for d in data) or 1
print("total samples", tot)
for d in sorted(data, key=lambda d: -d[1])[:n]:
    print("%5d stall %5.2f%% inst %5.2f%% thr %4.1f  %s" % (d[0], 100 * d[1] / tot, 100 * d[2] / ti, d[3] / max(1, d[2]), src[d[0] - 1].strip()[:120] if d[0] <= len(src) else ""))
