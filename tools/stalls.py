"""Summarise an ncu --set full report's source page: stall reasons overall
and the top instructions (usage: python tools/stalls.py report.ncu-rep [N])."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = r[2:]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
iS = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(x[iS]) for x in rows)
agg = {c: sum(int(x[h.index(c)] or 0) for x in rows) for c in cols}
print("samples", tot)
for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {c:24s} {100 * v / tot:5.1f}%")
iA, iSrc, iE = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
for x in sorted(rows, key=lambda x: -int(x[iS]))[:top_n]:
    det = sorted(((c, int(x[h.index(c)] or 0)) for c in cols), key=lambda kv: -kv[1])[:2]
    print(x[iA][-5:], f"{100 * int(x[iS]) / tot:5.1f}%", x[iE], x[iSrc][:70].strip(),
          " | ", ", ".join(f"{c[6:]}={v}" for c, v in det))
