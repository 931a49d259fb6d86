"""Benchmark: RNN-Descent graph build on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C3-gistlike-1M] [--n ROWS]

One step = one full build (random init -> T1 x T2 update passes + reverse
phases -> final sort; S=20 R=96 T1=4 T2=15) over the config's synthetic
store already resident in HBM.  value = L2 dist-evals/s = pair checks
(EditCounts::pair_checks, builder.cpp:57) summed over all ranks / max-rank
device time.  e2e = the same metric through the C ABI with host buffers
(H2D of the store, build, D2H of the graph) in the timed region.

--impl reference runs the UNMODIFIED reference (oracle/_ref) on the same
full-size store with all host threads, through its own public pass API
(random_init, update_neighbors, add_reverse_edges: the schedule rnnd::build
runs, builder.cpp:253-289): one build's 64 phases (init, 60 passes, 3 reverse
phases) are split into the K timed steps, so the K steps together are one
full-config build.

--gpus N without torchrun re-launches itself under torch.distributed.run with
N ranks (one per GPU); --dry checks that plumbing without a GPU (gloo, no
build).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK_GBS = 6650.0
CPU_SAMPLE_ROWS = 0  # 0: the full config
METRIC = "RNN-Descent build L2 dist-evals/s (1M x 960 fp32, S=20 R=96 T1=4 T2=15)"


def metric_for(cfg, n):
    """BASELINE.json's metric string for the default C3 workload; the same
    wording with the rows and dim of any other config."""
    if cfg.name == "C3-gistlike-1M" and n == cfg.n:
        return METRIC
    rows = f"{n // 1_000_000}M" if n % 1_000_000 == 0 else (f"{n // 1000}k" if n % 1000 == 0 else str(n))
    return f"RNN-Descent build L2 dist-evals/s ({rows} x {cfg.d} fp32, S=20 R=96 T1=4 T2=15)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3-gistlike-1M")
    ap.add_argument("--n", type=int, default=0, help="override rows (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-recall", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=CPU_SAMPLE_ROWS,
                    help="rows of the CPU baseline (0 = the full config)")
    ap.add_argument("--dry", action="store_true",
                    help="launcher / rank plumbing only (gloo, no GPU, no build)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the vertex-sharded build even at N=1 (checks that path)")
    return ap.parse_args()


_STDOUT_FD = None


def print_line(line: dict):
    """The one JSON line, on the real stdout even if fd 1 was redirected."""
    sys.stdout.flush()
    if _STDOUT_FD is not None:
        os.write(_STDOUT_FD, (json.dumps(line) + "\n").encode())
    else:
        print(json.dumps(line), flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def store_rows(cfg, n):
    import datagen
    return datagen.rows(cfg.cfg, cfg.seed, 0, n)


# ------------------------------------------------------------ reference arm

def build_phases(T1=4, T2=15):
    """rnnd::build's schedule (builder.cpp:262-281): init, then T1 outer
    rounds of T2 update passes, a reverse phase after every round but the
    last."""
    ph = ["init"]
    for t1 in range(1, T1 + 1):
        ph += ["pass"] * T2
        if t1 != T1:
            ph.append("reverse")
    return ph


def run_reference(args, rank, world):
    """The reference's own CPU implementation (oracle/_ref), rank 0 only, on
    the full config: one build's phases split over the K timed steps (W
    warm-up steps run the first phases of a throwaway build)."""
    if rank != 0:
        return
    # torchrun sets OMP_NUM_THREADS=1 per rank; the reference gets every host
    # core (read by libgomp when oracle/_ref is first loaded, just below)
    ncpu = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(ncpu)
    from oracle import oracle as O
    import datagen
    cfg = datagen.CONFIGS[args.config]
    n = args.n or cfg.n
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    data = store_rows(cfg, n)
    threads = max(ncpu, 2)  # threads > 1: the deferred variant (builder.cpp:88-139)
    phases = build_phases()

    def chunks(k):
        return [(len(phases) * i) // k for i in range(k + 1)]

    state = {"g": None, "i": 0}

    def run_phases(count):
        """Run the next `count` phases (a new build starts at phase 0)."""
        checks = 0
        for _ in range(count):
            i = state["i"] % len(phases)
            if i == 0:
                state["g"] = O.RefGraph(data)
                assert state["g"].random_init(20, 42) == 0
            elif phases[i] == "pass":
                checks += int(state["g"].update_pass(threads=threads)[3])
            else:
                assert state["g"].add_reverse_edges(96, threads=threads, order=0) == 0
            state["i"] += 1
        return checks

    b = chunks(max(args.steps, 1))
    if args.warmup:
        run_phases(min(args.warmup, len(phases)))
    state["i"] = 0  # the timed steps are one fresh build
    secs, checks = [], []
    for k in range(args.steps):
        cnt = b[k + 1] - b[k] if args.steps <= len(phases) else 1
        t = time.perf_counter()
        c = run_phases(cnt)
        secs.append(time.perf_counter() - t)
        checks.append(c)
    value = sum(checks) / sum(secs)
    line = {
        "impl": "reference", "metric": metric_for(cfg, n), "value": value, "unit": "dist-evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(secs) / len(secs), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": data_desc(cfg),
        "config": config_of(cfg, n, f"host threads x{threads} (rank 0 only)"),
        "cpu_baseline": {"value": value, "unit": "dist-evals/s", "cores": threads,
                         "kind": "reference",
                         "what": "unmodified reference (oracle/_ref): random_init + "
                                 "update_neighbors / add_reverse_edges, threads=%d, the full "
                                 "config, one build split over the %d timed steps"
                                 % (threads, args.steps),
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "dist-evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "build_seconds": sum(secs) * len(phases) / max(b[-1] if args.steps <= len(phases)
                                                       else args.steps, 1),
    }
    print(json.dumps(line))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return ""


def config_of(cfg, n, parallelism):
    return {"workload": cfg.name, "rows": n, "dim": cfg.d, "S": 20, "R": 96, "T1": 4, "T2": 15,
            "parallelism": parallelism,
            "l2_policy": ("inputs larger than L2 (store %.2f GB)" if n * cfg.d * 4 > 126e6
                          else "store fits in L2 (%.2f GB): no flush between steps")
            % (n * cfg.d * 4 / 1e9)}


STANDS_IN = {1: "a 64-component GMM", 2: "SIFT1M", 3: "GIST1M", 4: "Deep1M", 5: "Deep10M"}


def data_desc(cfg):
    return ("synthetic (seeded generator, datagen/datagen.cpp; stands in for %s)"
            % STANDS_IN.get(cfg.cfg, cfg.name))


# ------------------------------------------------------------------ our arm

def cpu_baseline(cfg, sample, n_full):
    """The unmodified reference's rnnd::build on the box's host cores
    (BuildStats.seconds, builder.cpp:260-286): the full config by default."""
    from oracle import oracle as O
    n = min(sample, n_full) if sample else n_full
    data = store_rows(cfg, n)
    if O.ref_available():
        cores = max(len(os.sched_getaffinity(0)), 2)
        g = O.RefGraph(data)
        rc, st = g.build(threads=cores)
        assert rc == 0
        out = {"value": float(st[6]) / float(st[0]), "unit": "dist-evals/s", "cores": cores,
               "kind": "reference", "seconds": float(st[0]), "pair_checks": float(st[6]),
               "what": f"rnnd::build(threads={cores}) on {n} rows of {cfg.name}",
               "cpu_model": cpu_model()}
        if n != n_full:
            out["sample"] = f"first {n} rows of {cfg.name}"
        return out
    g = O.OracleGraph(data)
    t = time.perf_counter()
    rc, pc = g.build()
    dt = time.perf_counter() - t
    return {"value": float(pc[:, 3].sum()) / dt, "unit": "dist-evals/s", "cores": 1,
            "kind": "port", "seconds": dt,
            "sample": f"C oracle build (1 thread) on the first {n} rows of {cfg.name}"}


def run_sharded(args, rank, world, local):
    """N > 1: the same workload, vertex ownership split over the ranks
    (SURVEY 8(e)); redirects / reverse proposals / in-edges / deletions are
    exchanged with NCCL all-to-all.  Total work is fixed: strong scaling."""
    import torch
    import torch.distributed as dist
    import datagen
    from paper_2310_20419_b200 import sharded as SH
    cfg = datagen.CONFIGS[args.config]
    n = args.n or cfg.n
    data = store_rows(cfg, n)
    b = SH.ownership_bounds(n, world)
    eng = SH.DeviceShard(data, b[rank], b[rank + 1], device=local)
    tr = SH.TorchDistTransport()
    p = dict(S=20, R=96, T1=4, T2=15, seed=42)

    def one_build():
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = SH.sharded_build([eng], tr, n, world, **p)
        e1.record()
        torch.cuda.synchronize()
        return st, e0.elapsed_time(e1) * 1e-3

    for _ in range(args.warmup):
        one_build()
    dist.barrier()
    eng.totals(reset=True)
    launches0 = eng.launches()
    secs, checks = 0.0, 0
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            st, dt = one_build()
            secs += dt
            checks += int(st.edits[3])  # already summed over ranks
        wall = time.perf_counter() - t0
    launches = eng.launches() - launches0
    tot = eng.totals(reset=True)

    # end to end: H2D of the store from pinned host memory, the sharded
    # build, D2H of this rank's lists; max over ranks
    pinned = torch.empty(data.shape, dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = data
    e2e_secs, d2h = 0.0, 0
    # one untimed pass warms the export staging (pinned host buffer)
    eng.load(pinned.numpy())
    SH.sharded_build([eng], tr, n, world, **p)
    eng.graph()
    for _ in range(args.steps):
        torch.cuda.synchronize()
        dist.barrier()
        t = time.perf_counter()
        eng.load(pinned.numpy())
        SH.sharded_build([eng], tr, n, world, **p)
        part = eng.graph()
        e2e_secs += time.perf_counter() - t
        d2h = int(part.offsets.nbytes + 12 * len(part.ids))

    vals = torch.tensor([secs, e2e_secs, tot["scan_seconds"], float(launches)],
                        dtype=torch.float64, device="cuda")
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    units = torch.tensor([float(tot["touched"]), float(tot["active_entries"]), float(d2h)],
                         dtype=torch.float64, device="cuda")
    dist.all_reduce(units, op=dist.ReduceOp.SUM)
    max_secs, max_e2e, max_scan = float(vals[0]), float(vals[1]), float(vals[2])
    if rank == 0:
        # roofline: algorithmic bytes of all shards' scans per GPU over the
        # slowest rank's distance-stage time
        alg = (4.0 * cfg.d * float(units[0]) + 24.0 * float(units[1])) / args.steps
        achieved = alg / world / (max_scan / args.steps) / 1e9 if max_scan > 0 else 0.0
        peak, peak_src = hbm_peak()
        line = {
            "metric": metric_for(cfg, n), "value": checks / max_secs, "unit": "dist-evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * max_secs / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": data_desc(cfg),
            "config": config_of(cfg, n, f"vertex-sharded x{world} (NCCL all-to-all)"),
            "build_seconds": max_secs / args.steps, "wall_seconds_timed": wall,
            "pair_checks_per_build": checks // args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "k_scan (distance stage), per GPU, max-rank time",
                         "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": {"value": checks / max_e2e, "unit": "dist-evals/s",
                    "h2d_bytes_per_step": int(data.nbytes) * world,
                    "d2h_bytes_per_step": int(units[2]),
                    "seconds_per_step": max_e2e / args.steps},
            "gpu_launches": int(vals[3]) * world,
            "clocks": clk.summary(),
        }
        print_line(line)


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args):
    """--gpus N > 1 outside torchrun: re-run this command under
    torch.distributed.run with N ranks on this node (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    sys.exit(subprocess.call(cmd))


def run_dry(args, rank, world):
    """Rank plumbing only: gloo process group, one all-reduce, the JSON line
    from rank 0 (no GPU, no build, no value)."""
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(free_port()))
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    dist.init_process_group("gloo")
    t = torch.ones(1)
    dist.all_reduce(t)
    if rank == 0:
        print_line({"metric": METRIC, "value": None, "unit": "dist-evals/s", "n_gpus": world,
                    "steps": args.steps, "warmup": args.warmup, "dry": True,
                    "ranks_seen": int(t.item()), "impl": args.impl})
    dist.destroy_process_group()


def parity_vs_reference(R, g, st, cfg, n):
    """The timed build against the reference's own build of the same bytes
    (tests/golden/builds_1m.json, made by oracle/_ref rnnd::build)."""
    import hashlib
    path = os.path.join(ROOT, "tests", "golden", "builds_1m.json")
    try:
        with open(path) as f:
            gold = json.load(f)["configs"]
    except Exception:
        return None
    for name, gd in gold.items():
        if gd["config"] == cfg.name and gd["rows"] == n:
            got = [[int(c.removed), int(c.inserted), int(c.flag_skips), int(c.pair_checks)]
                   for c in st.pass_counts]
            return {"config": cfg.name, "rows": n,
                    "index_equal": hashlib.sha256(R.index_bytes(g)).hexdigest()
                    == gd["index_sha256"],
                    "per_pass_counts_equal": got == gd["per_pass"],
                    "reference": "tests/golden/builds_1m.json[%s] (rnnd::build, %s threads)"
                                 % (name, gd["ref_threads"])}
    return None


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    if args.dry:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    torch.cuda.set_device(local)
    if world > 1 or args.sharded:
        # NCCL / c10d print banners on stdout; keep stdout for the one JSON
        # line (run_sharded restores it to print)
        global _STDOUT_FD
        sys.stdout.flush()
        _STDOUT_FD = os.dup(1)
        os.dup2(2, 1)
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        run_sharded(args, rank, world, local)
        dist.destroy_process_group()
        return
    import datagen
    from paper_2310_20419_b200 import _lib
    from paper_2310_20419_b200 import rnnd as R

    cfg = datagen.CONFIGS[args.config]
    n = args.n or cfg.n
    data = store_rows(cfg, n)
    store = R.VectorStore(data)
    dev = R.Device(local)
    dev.set_data(store)  # resident in HBM before the timed region
    params = R.BuildParams()

    def barrier():
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        R.build(store, params, device=dev)
    barrier()
    launches0 = dev.launches()
    stats = []
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            st = R.BuildStats()
            g = R.build(store, params, st, device=dev)
            stats.append(st)
        barrier()
        wall = time.perf_counter() - t0
    launches = dev.launches() - launches0
    parity = parity_vs_reference(R, g, stats[-1], cfg, n)
    dev_secs = sum(s.seconds for s in stats)
    checks = sum(s.edits.pair_checks for s in stats)
    max_secs = dev_secs
    value = checks / max_secs

    # roofline of the distance stage: B = 4 d T + 24 A bytes
    st0 = stats[-1]
    alg_bytes = 4.0 * cfg.d * st0.touched + 24.0 * st0.active_entries
    achieved = alg_bytes / st0.scan_seconds / 1e9
    peak, peak_src = hbm_peak()
    # second ceiling of the same stage: the exact no-FMA arithmetic is three
    # FP32 instructions per element and pair (sub, mul, add), which this B200
    # issues at 64 lanes per clock and SM (tools/ubench/fp32_pipe.cu, measured;
    # a flat register-tiled evaluation of dense pair blocks reaches 77% of it,
    # tools/ubench/flat_pairs.cu).  Counted pairs only (speculative ones are not
    # algorithmic work).
    sm_hz = 1965e6
    try:
        sm_hz = float(torch.cuda.get_device_properties(local).clock_rate) * 1e3
    except Exception:
        pass
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    fp32_ops = 3.0 * cfg.d * st0.edits.pair_checks
    fp32_peak = 64.0 * sms * sm_hz
    fp32_bound = {"ops_per_build": fp32_ops, "peak_ops_per_s": fp32_peak,
                  "floor_seconds": fp32_ops / fp32_peak,
                  "frac": fp32_ops / fp32_peak / st0.scan_seconds,
                  "peak_source": "64 non-FMA FP32 lanes/clk/SM measured by tools/ubench/fp32_pipe.cu"}
    # DRAM traffic of one distance-stage launch, from the committed ncu
    # --set full capture of this workload (per launch; algorithmic bytes of
    # the same pass alongside)
    traffic, traffic_alg, traffic_src = None, None, None
    import glob
    for tpath in sorted(glob.glob(os.path.join(ROOT, "profiles", "*scan_traffic*.json"))):
        try:
            with open(tpath) as f:
                tj = json.load(f)
        except Exception:
            continue
        if tj.get("config") == cfg.name and n == cfg.n:
            traffic = tj.get("dram_bytes_per_launch")
            traffic_alg = tj.get("algorithmic_bytes_same_pass")
            traffic_src = os.path.relpath(tpath, ROOT) + ": " + tj.get("kernel", "")

    # end to end through the C ABI with host buffers (H2D, build, D2H)
    pinned = torch.empty(data.shape, dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = data
    pstore = R.VectorStore(pinned.numpy())
    e2e_secs, e2e_checks, d2h = 0.0, 0, 0
    # one untimed pass warms the export staging (pinned host buffer)
    dev.set_data(pstore)
    R.build(pstore, params, R.BuildStats(), device=dev)
    dev.get_graph()
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        dev.set_data(pstore)  # H2D
        st = R.BuildStats()
        g = R.build(pstore, params, st, device=dev)
        csr = dev.get_graph()  # D2H
        e2e_secs += time.perf_counter() - t
        e2e_checks += st.edits.pair_checks
        d2h = int(csr.offsets.nbytes + 12 * len(csr.ids))
    e2e = {"value": e2e_checks / e2e_secs, "unit": "dist-evals/s",
           "h2d_bytes_per_step": int(data.nbytes), "d2h_bytes_per_step": d2h,
           "seconds_per_step": e2e_secs / args.steps}

    recall = None
    if not args.no_recall:
        nq = min(cfg.nq, 1000)
        q = datagen.rows(cfg.cfg, cfg.seed, cfg.n, nq) if n == cfg.n else \
            datagen.rows(cfg.cfg, cfg.seed, n, nq)
        qs = R.VectorStore(q)
        t = time.perf_counter()
        gt = R.brute_force_gt(store, qs, 10, device=dev)
        t_gt = time.perf_counter() - t
        g = R.build(store, params, device=dev)
        recall = {"queries": nq, "gt_seconds": t_gt}
        for L in (16, 32, 64):
            timing = R.BatchTiming()
            res = R.batch_search(g, store, qs, R.SearchParams(L=L, K=0, k=10), timing=timing)
            recall[f"L{L}"] = {"recall@1": R.recall_at_1(res, R.GroundTruth(10, gt.ids), store, qs),
                               "recall@10": R.recall_at_k(res, gt, 10), "qps": timing.qps}
        deg = R.degree_stats(g)
        recall["aod"] = deg.avg_out
        recall["max_out"] = deg.max_out

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_sample, n)

    line = {
        "metric": metric_for(cfg, n), "value": value, "unit": "dist-evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * max_secs / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": data_desc(cfg),
        "config": config_of(cfg, n, "1gpu"),
        "build_seconds": max_secs / args.steps,
        "wall_seconds_timed": wall,
        "pair_checks_per_build": stats[-1].edits.pair_checks,
        "stage_seconds": {"scan": st0.scan_seconds, "sort": st0.sort_seconds,
                          "apply": st0.apply_seconds, "reverse": st0.reverse_seconds},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_algorithmic_bytes_same_launch": traffic_alg,
                     "traffic_source": traffic_src,
                     "kernel": "k_scan (distance stage)",
                     "algorithmic_bytes_per_build": alg_bytes,
                     "touched": st0.touched, "active_entries": st0.active_entries,
                     "peak_source": peak_src, "fp32_issue_bound": fp32_bound},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "recall": recall,
        "parity": parity,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
