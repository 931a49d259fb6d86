"""Copy the round-2 closing measurements (tools/r02_capture.sh) from gpurun_out/
into profiles/: bench and reference lines, launch list summary, the ncu
captures of the two scan kernels (traffic JSON + details text)."""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refresh_profiles import raw, metrics  # noqa: E402

G = lambda *a: os.path.join(ROOT, "gpurun_out", *a)  # noqa: E731
P = lambda *a: os.path.join(ROOT, "profiles", *a)  # noqa: E731


def pass_line(k):
    lines = [l for l in open(G("r02_trace.err")) if "pass active" in l]
    lines = lines[-60:]
    return lines[k].strip().replace("[rnndg] pass ", "")


shutil.copy(G("r02_bench.json"), P("r02_bench_c3_1m_final.json"))
shutil.copy(G("r02_ref.json"), P("r02_reference_arm.json"))
d = {"config": "C3-gistlike-1M",
     "capture": "ncu --set full --import-source on --clock-control none -k regex:k_scan_spec -s 5 -c 1 "
                "python tools/prof_build.py (tools/r02_capture.sh)"}
gs = raw(G("r02_short_p5.ncu-rep"))
name = gs("Kernel Name", False).replace("void unnamed>::", "").replace("(unnamed>::ScanArgs)", "")
p5 = pass_line(5)
kv = dict(x.split("=") for x in p5.split() if "=" in x)
d.update(metrics(gs))
d.update({"kernel": f"{name} (short lists), update pass 5 of 60 (t1=1, t2=4)",
          "algorithmic_bytes_same_pass": 4 * 960 * int(kv["touched"]) + 24 * int(kv["entries"]),
          "pass_trace": p5})
gh = raw(G("r02_hub_p18.ncu-rep"))
hname = gh("Kernel Name", False).replace("void unnamed>::", "").replace("(unnamed>::ScanArgs)", "")
d["hub_kernel"] = dict(metrics(gh), kernel=f"{hname}, update pass 18 of 60 (t1=2, t2=3)",
                       pass_trace=pass_line(18))
json.dump(d, open(P("r02_scan_traffic_c3_1m.json"), "w"), indent=1)
for rep, out in [("r02_short_p5.ncu-rep", "r02_scan_short_p5_details.txt"),
                 ("r02_hub_p18.ncu-rep", "r02_scan_hub_p18_details.txt")]:
    txt = subprocess.run(["ncu", "-i", G(rep), "--page", "details"], capture_output=True, text=True).stdout
    open(P(out), "w").write(txt)
rows = [x for x in csv.reader(open(G("r02_launches.csv"))) if len(x) > 10]
h, data = rows[0], rows[1:]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for x in data:
    nm = re.sub(r"\(.*", "", x[ik]).replace("void ", "").replace("unnamed>::", "").replace("rnndg::<", "")
    val = float(x[iv].replace(",", ""))
    val = val / 1e6 if x[iu] in ("ns", "nsecond") else (val / 1e3 if x[iu] in ("us", "usecond") else val)
    tot[nm] += val
    cnt[nm] += 1
T = sum(tot.values())
json.dump({"what": "ncu --metrics gpu__time_duration.sum --clock-control none, one C3 1M build "
                   "(tools/prof_build.py), serialised, cold-cache per launch; closing state of round 2",
           "total_ms": T, "launches": sum(cnt.values()),
           "kernels": {k: {"ms": round(v, 3), "share": round(v / T, 4), "launches": cnt[k]}
                       for k, v in tot.most_common(14)}},
          open(P("r02_launches_c3_1m_build_final.json"), "w"), indent=1)
print("launch list:", sum(cnt.values()), "launches", round(T, 1), "ms;",
      [(k[:40], round(v / T * 100, 1)) for k, v in tot.most_common(4)])
print("short:", d["kernel"], "DRAM/alg", round(d["dram_bytes_per_launch"] / d["algorithmic_bytes_same_pass"], 2),
      {k: d[k] for k in ("l1tex_throughput_pct", "issue_active_pct", "warps_active_pct", "registers_per_thread")})
