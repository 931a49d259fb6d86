"""Rewrite the numeric summaries in README.md and profiles/README.md from the
committed bench / config / traffic JSON files (run after refreshing them)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = lambda *a: os.path.join(ROOT, *a)  # noqa: E731

b = json.loads(open(P("profiles", "r01_bench_c3_1m.json")).readline())
cf = json.load(open(P("profiles", "r01_configs_1gpu.json")))
tr = json.load(open(P("profiles", "r01_scan_traffic_c3_1m.json")))
hub = tr.get("hub_kernel", {})


def cfg_line():
    return (f"C1 20k×128 in {cf['C1-gmm128-20k']['build_seconds']:.3f} s, C2 1M×128 in "
            f"{cf['C2-siftlike-1M']['build_seconds']:.2f} s, C4 1M×96 in "
            f"{cf['C4-deeplike-1M']['build_seconds']:.2f} s, and C5 10M×96 in "
            f"{cf['C5-deep10M']['build_seconds']:.1f} s")


# README.md results block
p = P("README.md")
s = open(p).read()
i = s.index("| this repo, data resident in HBM |")
j = s.index("Details are in `DESIGN.md`")
s = s[:i] + f"""| this repo, data resident in HBM | {b['build_seconds']:.2f} | {b['value']:.3g} |
| this repo, e2e through the C ABI (H2D + build + D2H) | {b['e2e']['seconds_per_step']:.2f} | {b['e2e']['value']:.3g} |
| reference `rnnd::build`, 16 host threads (150k sample) | — | {b['cpu_baseline']['value']:.2g} |

recall@1 is {b['recall']['L32']['recall@1']} at L=32 (1,000 held-out queries). The distance stage runs
at {b['roofline']['frac']:.2f} of the HBM roofline, counted in algorithmic bytes. The other configs
run on one GPU too: {cfg_line()}. The reference's acceptance suite passes 10/10 against the GPU
builder. The NN-Descent baseline runs on the GPU as well: on the criterion-5
workload, RNN-Descent takes 0.05 s and NN-Descent 0.19 s.

""" + s[j:]
open(p, "w").write(s)

# profiles/README.md current state
p = P("profiles", "README.md")
s = open(p).read()
i = s.index("## Current state (end of r01)")
j = s.index("## Progression")
ratio = tr["dram_bytes_per_launch"] / tr["algorithmic_bytes_same_pass"]
s = s[:i] + f"""## Current state (end of r01)

C3 1M×960, S=20 R=96 T1=4 T2=15: **{b['build_seconds']:.3f} s per build, {b['value']:.3g} dist-evals/s**
(device, data resident); e2e through the C ABI with host buffers (H2D 3.84 GB
at 55 GB/s, build, D2H of the graph) {b['e2e']['seconds_per_step']:.3f} s, {b['e2e']['value']:.3g} dist-evals/s; the
unmodified reference on 16 host threads {b['cpu_baseline']['value']:.3g} dist-evals/s (≈{b['e2e']['value'] / b['cpu_baseline']['value']:.0f}× slower
than the e2e number); recall@1 {b['recall']['L32']['recall@1']} at L=32 (1,000 held-out queries, GPU brute
force).  Other configs (`r01_configs_1gpu.json`): {cfg_line()}.

Serialised launch list of one build (`r01_launches_c3_1m_build.csv`): the
short-list scan and the hub scans take ≈95% of the device time.

Distance stage, short lists `{tr['kernel'].split(' (')[0]}`, update pass 5 of the 1M
build (ncu, serialised): {tr['duration_ms_under_ncu']:.1f} ms, DRAM {tr['dram_bytes_per_launch'] / 1e9:.0f} GB = **{ratio:.1f}× the algorithmic
bytes** of the pass ({tr['algorithmic_bytes_same_pass'] / 1e9:.1f} GB: 4·d·T + 24·A), L2 hit {tr['l2_hit_rate_pct']:.0f}%, L1 hit {tr['l1_hit_rate_pct']:.0f}%, L1TEX
throughput {tr['l1tex_throughput_pct']:.0f}%, issue active {tr['issue_active_pct']:.0f}%, {tr['registers_per_thread']} registers (6 CTAs of 64 threads per
SM).  About half of the warp-stall samples sit on the first FADD of each
pair's first two blocks: a new pair's loads queue behind every load in
flight on the SM.  Hub lists `k_scan_hub<32,2,4,1>`, pass 18
(`r01_scan_hub_p18_details.txt`): {hub.get('duration_ms_under_ncu', 0):.1f} ms, DRAM {hub.get('dram_bytes_per_launch', 0) / 1e9:.0f} GB, L1 hit {hub.get('l1_hit_rate_pct', 0):.0f}%,
L1TEX throughput {hub.get('l1tex_throughput_pct', 0):.0f}%, 64 registers (spills; a 24-warp variant at 80
registers without spills runs at the same speed), warps active {hub.get('warps_active_pct', 0):.0f}%.

The vertex-sharded protocol (`bench.py --sharded`, one rank on one GPU,
NCCL exchange): 2.001 s per C3 1M build against 1.937 s for the
single-context build (3–4% for the record export/import and host syncs);
C5 10M 11.94 s against 11.53 s; identical pair counts on every config.

""" + s[j:]
s = s.replace(s[s.index("(measured per pod).  r01 at C3 1M:"):s.index("T_p and A_p are counted")],
              f"(measured per pod).  r01 at C3 1M: {b['roofline']['achieved']:.0f} GB/s of {b['roofline']['peak']:.0f}, "
              f"**frac {b['roofline']['frac']:.2f}**.  ")
open(p, "w").write(s)
print("ok", b["build_seconds"])

# DESIGN.md section 8 opening numbers
p = P("DESIGN.md")
s = open(p).read()
i = s.index("C3 1M build, ")
j = s.index("Serialised launch list of one build", i)
s = s[:i] + f"""C3 1M build, {b['build_seconds']:.3f} s (`profiles/r01_bench_c3_1m.json`): distance stage
{b['stage_seconds']['scan']:.3f} s, apply {b['stage_seconds']['apply']:.3f} s, reverse phases {b['stage_seconds']['reverse']:.3f} s, marking and
ordering {b['stage_seconds']['sort']:.3f} s, init + layout ≈ 0.02 s.  e2e through the C ABI
{b['e2e']['seconds_per_step']:.3f} s: + H2D of the store (69 ms, 55 GB/s over PCIe) + D2H of the
graph (11 ms through pinned staging).  """ + s[j:]
open(p, "w").write(s)
print("design ok")
