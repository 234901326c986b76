"""Summarise an ncu source page (SASS): top instructions by warp-stall samples.
usage: python scripts/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
iS, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
data = []
for r in rows[1:]:  # the first kernel's section only (a later section starts with its own header)
    if len(r) == len(h) and r[iS] == h[iS]:
        break
    if len(r) == len(h):
        data.append(r)
tot = sum(int(r[iS] or 0) for r in data)
print("total samples", tot)
def reasons(r):
    rs = sorted(((int(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    return " ".join("%s=%d" % (n, v) for v, n in rs if v)


for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:N]:
    print("%6s %5.1f%%  %-60s %s" % (r[iS], 100 * int(r[iS] or 0) / max(tot, 1), r[iSrc].strip()[:60], reasons(r)))
by = {}
for r in data:
    for i in stall_cols:
        by[h[i]] = by.get(h[i], 0) + int(r[i] or 0)
print("by reason:", ", ".join("%s %d" % (k[6:], v) for k, v in sorted(by.items(), key=lambda x: -x[1])[:8]))

if len(sys.argv) > 3:  # context around the top K instructions
    K = int(sys.argv[3])
    top = sorted(range(len(data)), key=lambda i: -int(data[i][iS] or 0))[:K]
    for i in sorted(top):
        print("----")
        for j in range(max(0, i - 8), min(len(data), i + 3)):
            print("%6s %s %s" % (data[j][iS], ">>" if j == i else "  ", data[j][iSrc].strip()[:100]))
