"""Copy the round's measurements from gpurun_out/ into profiles/: bench and
reference lines, config lines, the launch list of one build, and the ncu
captures of the two scan kernels (traffic JSON + details text).
usage: python tools/refresh_profiles.py SHORT.ncu-rep HUB.ncu-rep"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = lambda *a: os.path.join(ROOT, "gpurun_out", *a)  # noqa: E731
P = lambda *a: os.path.join(ROOT, "profiles", *a)  # noqa: E731


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units, v = r[0], r[1], r[2]
    def get(name, scale=True):
        x = v[h.index(name)]
        u = units[h.index(name)]
        if not scale:
            return x
        f = float(x.replace(",", ""))
        return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
    return get


def metrics(get):
    return {
        "dram_bytes_per_launch": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
        "duration_ms_under_ncu": get("gpu__time_duration.sum"),
        "l2_hit_rate_pct": get("lts__t_sector_hit_rate.pct"),
        "l1_hit_rate_pct": get("l1tex__t_sector_hit_rate.pct"),
        "lts_throughput_pct": get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "l1tex_throughput_pct": get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": get("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers_per_thread": int(get("launch__registers_per_thread")),
    }


def pass_line(k):
    lines = [l for l in open(G("r01_trace.err")) if "pass active" in l]
    return lines[k].strip().replace("[rnndg] pass ", "")


def main():
    short_rep, hub_rep = sys.argv[1], sys.argv[2]
    for a, b in [("r01_bench.json", "r01_bench_c3_1m.json"), ("r01_ref.json", "r01_reference_arm.json"),
                 ("configs_1gpu.json", "r01_configs_1gpu.json")]:
        shutil.copy(G(a), P(b))
    p = P("r01_scan_traffic_c3_1m.json")
    d = json.load(open(p))
    gs = raw(short_rep)
    name = gs("Kernel Name", False).replace("void unnamed>::", "").replace("(unnamed>::ScanArgs)", "")
    p5 = pass_line(5)
    kv = dict(x.split("=") for x in p5.split() if "=" in x)
    prev = [{"kernel": d["kernel"], "dram_bytes_per_launch": d["dram_bytes_per_launch"],
             "duration_ms_under_ncu": d["duration_ms_under_ncu"]}] + d.get("previous", [])
    d.update(metrics(gs))
    d.update({"kernel": f"{name} (short lists), update pass 5 of 60 (t1=1, t2=4)",
              "algorithmic_bytes_same_pass": 4 * 960 * int(kv["touched"]) + 24 * int(kv["entries"]),
              "pass_trace": p5, "previous": prev[:8]})
    gh = raw(hub_rep)
    hname = gh("Kernel Name", False).replace("void unnamed>::", "").replace("(unnamed>::ScanArgs)", "")
    d["hub_kernel"] = dict(metrics(gh), kernel=f"{hname}, update pass 18 of 60 (t1=2, t2=3)",
                           pass_trace=pass_line(18),
                           capture="ncu --set full --import-source on --clock-control none -k regex:k_scan_hub -s 18 -c 1")
    json.dump(d, open(p, "w"), indent=1)
    for rep, out in [(short_rep, "r01_scan_short_p5_details.txt"), (hub_rep, "r01_scan_hub_p18_details.txt")]:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
        open(P(out), "w").write(txt)
    rows = [x for x in csv.reader(open(G("r01_launches.csv"))) if len(x) > 10]
    h, data = rows[0], rows[1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    ig, ib, ist = h.index("Grid Size"), h.index("Block Size"), h.index("Stream")
    out, seen = [], 0
    for x in data:
        nm = re.sub(r"\(unnamed>::ScanArgs\)", "", x[ik]).replace("void ", "").replace("unnamed>::", "")
        if "k_random_init" in nm:
            seen += 1
            if seen == 2:
                break
        out.append([x[0], nm[:120], x[ist], x[ig], x[ib], x[iu], x[iv]])
    with open(P("r01_launches_c3_1m_build.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["# ncu --metrics gpu__time_duration.sum --clock-control none --csv: one C3 1M build "
                    "(python bench.py --steps 1 --warmup 0 --no-recall --no-cpu-baseline), serialised launches"])
        w.writerow(["id", "kernel", "stream", "grid", "block", "unit", "gpu__time_duration.sum"])
        w.writerows(out)
    tot = collections.Counter()
    for x in out:
        val = float(x[6].replace(",", ""))
        val = val / 1e6 if x[5] == "ns" else (val / 1e3 if x[5] == "us" else val)
        tot[re.sub(r"<.*", "", x[1].replace("rnndg::<", ""))] += val
    T = sum(tot.values())
    print("launch list:", len(out), "launches", round(T, 1), "ms;",
          [(k, round(v / T * 100, 1)) for k, v in tot.most_common(5)])
    print("short:", d["kernel"], round(d["dram_bytes_per_launch"] / d["algorithmic_bytes_same_pass"], 2))


if __name__ == "__main__":
    main()
