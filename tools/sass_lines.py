"""Warp-stall samples of an ncu --set full report aggregated by CUDA source
line (SASS addresses mapped through nvdisasm -g of the kernel's cubin).

usage: python tools/sass_lines.py report.ncu-rep kernel.cubin kernel_substring [N]"""
import csv
import re
import subprocess
import sys

rep, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top_n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
iA, iS = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
samples = {}
for x in r[2:]:
    samples[int(x[iA], 16) & 0xFFFFF] = int(x[iS] or 0)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line_of, cur, in_fn = {}, None, False
for ln in dis.splitlines():
    if ln.startswith(".text.") or ln.strip().startswith(".section"):
        in_fn = kname in ln
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if "//##" in ln and m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
    m2 = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m2 and in_fn and cur is not None:
        line_of[int(m2.group(1), 16) & 0xFFFFF] = cur
# ncu addresses are absolute; align on the lowest address of each set
if samples and line_of:
    base_s, base_l = min(samples), min(line_of)
    agg, tot = {}, sum(samples.values())
    for a, s in samples.items():
        l = line_of.get(a - base_s + base_l)
        agg[l] = agg.get(l, 0) + s
    print("samples", tot)
    for l, s in sorted(agg.items(), key=lambda kv: -kv[1])[:top_n]:
        print(f"{l}: {100 * s / tot:5.1f}%")
