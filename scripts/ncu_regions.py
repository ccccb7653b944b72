"""Source-region breakdown of an ncu --set full capture of a generated tile kernel: warp-stall
samples, executed warp instructions and SIMT efficiency per region of the generated source
(eigen fragment, element tape, SPD tail, tile reduction). usage: ncu_regions.py REP SRC.cu"""
import csv, os, subprocess, sys
rep, srcf = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep] + os.environ.get("NCU_FILTER", "").split() + [ "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--resolve-source-file", srcf], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed")
iT = hdr.index("Thread Instructions Executed")
lines = []
for r in rows:
    if r and r[0] not in ("", "Line No") and r[0].isdigit():
        try:
            lines.append((int(r[0]), int(r[iS]), int(r[iI]), int(r[iT])))
        except ValueError:
            pass
src = open(srcf).read().splitlines()
marks = {"prelude (rcp/rsqrt helpers)": 1}
for i, l in enumerate(src, 1):
    if "void sy_tred2(" in l: marks["eigen: Householder tridiagonalisation"] = i
    if "void sy_ql(" in l: marks["eigen: implicit QL with vectors"] = i
    if "void sy_ql_la(" in l: marks["eigen: implicit QL with vectors (lookahead)"] = i
    if "void sy_eig(" in l: marks["eigen: wrapper"] = i
    if "void sy_trid(" in l: marks["small-set: Householder (reflectors kept)"] = i
    if "void sy_invit(" in l: marks["small-set: inverse iteration"] = i
    if "void sy_clamp_ss(" in l: marks["small-set: compaction, back-transform, update"] = i
    if "V[N - 1][i] = V[i][i]" in l: marks["eigen: accumulate Q"] = i
    if "const long long e =" in l: marks["element tape (E, g, M, W)"] = i
    if ("sy_eig<" in l or "sy_clamp_ss<" in l) and "call" not in l and "void" not in l: marks["SPD tail: clamp + H = W^T C W + stage"] = i - 1
    if "const int sy_nh = hs1 - hs0" in l: marks["tile reduction + energy"] = i
order = sorted(marks.items(), key=lambda kv: kv[1])
def region(n):
    name = order[0][0]
    for k, v in order:
        if n >= v: name = k
    return name
agg = {}
for n, sm, ii, tt in lines:
    a = agg.setdefault(region(n), [0, 0, 0]); a[0] += sm; a[1] += ii; a[2] += tt
ts = sum(a[0] for a in agg.values()) or 1; ti = sum(a[1] for a in agg.values()) or 1
print("%-42s %9s %9s %8s" % ("region", "stall %", "inst %", "thr/inst"))
for k, _ in order:
    if k in agg:
        a = agg[k]
        print("%-42s %8.1f%% %8.1f%% %8.1f" % (k, 100 * a[0] / ts, 100 * a[1] / ti, a[2] / max(1, a[1])))
