#!/usr/bin/env python
"""Benchmark of the colour-coding hot path (one step = one colouring: cc_color +
cc_count_colorful, i.e. PAPER.md Alg. 1 lines 5-10 for one iteration).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Default workload: BASELINE.json configs[3] (R-MAT scale 23, edge factor 32,
12-vertex tree, k = 12, fp32 tables + fp64 root) -- the largest configuration
that fits one GPU.  Multi-GPU runs (torchrun, one rank per GPU) split the same
graph with the 1D vertex partition (strong scaling; halo rows exchanged by
NCCL).  Prints ONE JSON line on rank 0.

Timing: W untimed colourings, then K timed ones; device time from CUDA events
the library records on the stream its kernels run on (colour kernel + DP),
bracketed by a barrier and a device synchronize, max over ranks.  The count
tables (GBs) are far larger than the 126 MB L2, so no extra L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per coloring iteration; G edge*colorset updates/s; % of HBM roofline"
UNIT = "G edge*colorset updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--precision", default=None, help="fp32 | fp64 (default: the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: colouring replicas (each GPU the whole graph, different colourings; SURVEY F1) "
                         "instead of the 1D vertex partition")
    ap.add_argument("--segment-len", type=int, default=0)
    ap.add_argument("--exchange", default="auto", choices=["auto", "grouped", "ring", "alltoall", "device"],
                    help="halo-exchange schedule of the 1D partition (PAPER.md Alg. 3)")
    ap.add_argument("--seed", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-scale", type=int, default=0, help="R-MAT scale of the oracle sample (0 = auto)")
    ap.add_argument("--graphs", type=int, default=-1,
                    help="1: replay each count as a CUDA graph (cc_options.use_graphs); -1 = auto (configs 0-1)")
    ap.add_argument("--no-ncu", action="store_true",
                    help="skip the one-launch ncu pass that measures the dominant kernel's DRAM traffic")
    ap.add_argument("--ncu-child", type=int, default=0, help=argparse.SUPPRESS)  # internal: pass ordinal to mark
    return ap.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM-style copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


NCU_METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum"


def ncu_child(args, cfg):
    """Internal (--ncu-child i): one colouring of the bench workload with the
    i-th neighbour-sum pass inside the NVTX range cc_dominant, for the parent's
    one-launch ncu measurement of that launch's DRAM traffic."""
    import paper_1804_09764_b200 as cc
    precision = args.precision or cfg.precision
    g = cfg.graph()
    ctx = cc.cc_create(device=0, precision=cc.CC_FP64 if precision == "fp64" else cc.CC_FP32,
                       segment_len=args.segment_len)
    cc.cc_load_graph(ctx, g.n, g.row_ptr, g.col)
    cc.cc_set_template(ctx, cfg.parent)
    cc.cc_set_knob(ctx, "nvtx_mark", args.ncu_child)
    cc.cc_color(ctx, args.seed)
    cc.cc_count_colorful(ctx)
    cc.cc_destroy(ctx)


def measure_dominant_traffic(args, ordinal: int):
    """DRAM bytes (read + write) and the L2 hit rate of the dominant launch,
    measured in THIS run: ncu collects 4 counters on the one launch inside
    the NVTX range cc_dominant of a one-colouring child (no timing is taken
    from it).  None when ncu is missing or fails."""
    import csv
    import shutil
    import tempfile
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if not ncu or ordinal <= 0:
        return None
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "ncu.csv")
        cmd = [ncu, "--nvtx", "--nvtx-include", "cc_dominant/", "--metrics", NCU_METRICS, "--clock-control", "none",
               "--csv", "--log-file", log, sys.executable, os.path.abspath(__file__), "--ncu-child", str(ordinal),
               "--config", str(args.config), "--seed", str(args.seed), "--segment-len", str(args.segment_len)]
        if args.precision:
            cmd += ["--precision", args.precision]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        except (subprocess.TimeoutExpired, OSError):
            return None
        if r.returncode != 0 or not os.path.exists(log):
            return None
        vals = {}
        kernels = set()
        with open(log) as f:
            rows = [ln for ln in f if ln.startswith('"')]
        for row in csv.DictReader(rows):
            name, unit, val = row.get("Metric Name"), row.get("Metric Unit", ""), row.get("Metric Value", "")
            if not name:
                continue
            try:
                x = float(val.replace(",", ""))
            except ValueError:
                continue
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9,
                     "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "%": 1.0}.get(unit, 1.0)
            kernels.add((row.get("ID"), row.get("Kernel Name")))
            vals.setdefault(name, []).append(x * scale)
        if "dram__bytes_read.sum" not in vals:
            return None
        return {"dram_bytes": sum(vals["dram__bytes_read.sum"]) + sum(vals.get("dram__bytes_write.sum", [0.0])),
                "l2_hit_rate_pct": (statistics.mean(vals["lts__t_sector_hit_rate.pct"])
                                    if "lts__t_sector_hit_rate.pct" in vals else None),
                "ncu_kernel_s": sum(vals.get("gpu__time_duration.sum", [0.0])),
                "kernels": sorted(k[1] for k in kernels if k[1])}


def dominant_traffic(config_idx: int, precision: str):
    """DRAM bytes (read + write) per launch of the dominant kernel, from the
    committed ncu --set full capture (profiles/*/dominant_kernel.json), if it
    was taken on this config and precision; else None."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "dominant_kernel.json")), reverse=True):
        with open(p) as f:
            d = json.load(f)
        if d.get("config") == config_idx and d.get("precision") == precision:
            return float(d["dram_bytes_per_launch"]), os.path.relpath(p, ROOT)
    return None, None


def updates_per_entry(parent) -> int:
    """sum over the DISTINCT passive sub-templates of C(k, p) (U =
    that x 2m), for the paper's own partition of the template: root = the
    parent -1 vertex, each sub-template (x, j) = x with its first j children
    split into (x, j-1) + the full subtree of child j (PAPER.md lines 110-113,
    122), isomorphic passives counted once.  Plain Python, so that both arms
    use the same U and the reference arm never loads the product library."""
    k = len(parent)
    children = [[] for _ in range(k)]
    root = parent.index(-1)
    for v, p in enumerate(parent):
        if p >= 0:
            children[p].append(v)

    def code(x):  # AHU canonical code of the full subtree at x
        return "(" + "".join(sorted(code(y) for y in children[x])) + ")"

    def size(x):
        return 1 + sum(size(y) for y in children[x])

    seen, u = set(), 0
    for x in range(k):
        for y in children[x]:  # every child subtree is a passive part of some step
            key = code(y) if size(y) > 1 else "leaf"
            if key not in seen:
                seen.add(key)
                u += math.comb(k, size(y))
    del root
    return u


def method_updates(g_nnz: int, parent) -> float:
    return float(g_nnz) * updates_per_entry(parent)


# ---------------------------------------------------------------- oracle (CPU) timing
def oracle_sample(cfg, scale: int, seed: int, reps: int = 1):
    """The oracle as it stands, on the config's template and generator at a
    smaller R-MAT scale; returns (G updates/s, ms per colouring, description)."""
    import oracle
    import synth
    if cfg.graph_kind == "rmat":
        scfg = synth.scaled_twin(cfg, scale)
    else:
        scfg = cfg
    g = scfg.graph()
    col = oracle.color(g.n, cfg.k, seed)
    numtype = oracle.NUM_DOUBLE if cfg.precision == "fp32" else oracle.NUM_LONGDOUBLE
    best = None
    for _ in range(reps):
        t = time.perf_counter()
        oracle.dp_count(g, cfg.parent, col, numtype)
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    u = method_updates(g.nnz, cfg.parent)
    desc = (f"oracle fold-children DP ({'double' if numtype == oracle.NUM_DOUBLE else 'long double'}), one colouring of "
            f"{scfg.name} (n={g.n}, 2m={g.nnz}); value = method updates of that sample / oracle time")
    return u / best / 1e9, best * 1e3, desc


def host_info() -> dict:
    """CPU model and host RAM of the box the oracle ran on."""
    info = {"cpu_model": None, "host_ram_gb": None}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    info["host_ram_gb"] = round(int(line.split()[1]) / 2**20, 1)
                    break
    except OSError:
        pass
    return info


def auto_cpu_scale(cfg):
    return {0: 0, 1: 16, 2: 18, 3: 19, 4: 13}[cfg.idx]


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    scale = args.cpu_scale or auto_cpu_scale(cfg)
    cores = os.cpu_count()
    vals = []
    for _ in range(args.warmup if cfg.idx <= 1 else 1):
        oracle_sample(cfg, scale, args.seed)
    for j in range(args.steps):
        v, ms, desc = oracle_sample(cfg, scale, args.seed + j)
        vals.append((v, ms))
    value = statistics.median(v for v, _ in vals)
    ms = statistics.median(m for _, m in vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"configs[{cfg.idx}] {cfg.name}", "sample_scale": scale},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                             **host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- ours
def run_ours(args, cfg, rank, world, dist):
    import numpy as np
    import torch

    import paper_1804_09764_b200 as cc
    import synth

    precision = args.precision or cfg.precision
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    g = cfg.graph()
    kw = dict(precision=cc.CC_FP64 if precision == "fp64" else cc.CC_FP32, segment_len=args.segment_len,
              exchange={"auto": cc.CC_EXCHANGE_AUTO, "grouped": cc.CC_EXCHANGE_GROUPED, "ring": cc.CC_EXCHANGE_RING,
                        "alltoall": cc.CC_EXCHANGE_ALLTOALL, "device": cc.CC_EXCHANGE_DEVICE}[args.exchange],
              replicas=1 if (args.replicas and world > 1) else 0,
              use_graphs=int(args.graphs if args.graphs >= 0 else (cfg.idx <= 1 and world == 1)))
    if world > 1:
        opt, _idbuf = cc.distributed_options(**kw)
    else:
        opt = cc.cc_default_options(device=local, **kw)
    ctx = cc.cc_create(opt)
    cc.cc_load_graph(ctx, g.n, g.row_ptr, g.col)
    cc.cc_set_template(ctx, cfg.parent)

    def step(seed):
        cc.cc_color(ctx, seed)
        x = cc.cc_count_colorful(ctx)
        prof = cc.cc_last_profile(ctx)
        return x, prof

    # nvidia-smi clock sampling runs through the warm-up and the timed region
    # (its first sample takes ~0.5 s to arrive)
    clocks = ClockSampler(local)
    clocks.start()
    for j in range(args.warmup):
        step(args.seed + 1000 + j)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    dev_ms, agg_ms, xs, top_stats = [], [], [], []
    stats = None
    for j in range(args.steps):
        x, prof = step(args.seed + j)
        xs.append(x)
        dev_ms.append(prof["total"] + prof["color"])
        agg_ms.append(prof["gather"])
        stats = cc.cc_last_stats(ctx)
        top_stats.append(stats)
        last_prof = prof
    barrier()
    clk = clocks.stop()
    total_ms = sum(dev_ms)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    # U per colouring (the whole job: every adjacency entry is processed by
    # its owner once per distinct passive); replicas: world colourings per step
    updates = method_updates(g.nnz, cfg.parent) * (world if (args.replicas and world > 1) else 1)
    value = updates / (ms_per_step * 1e-3) / 1e9

    # e2e: public API with host inputs (a colouring passed in from pinned host
    # memory) and the 8-byte result read back, wall clock per step.
    cols = [synth.uniform_colors(g.n, cfg.k, 5000 + j) for j in range(args.steps)]
    pinned = [torch.from_numpy(c).pin_memory() for c in cols]
    barrier()
    t0 = time.perf_counter()
    for j in range(args.steps):
        cc.cc_set_colors(ctx, pinned[j].numpy())
        cc.cc_count_colorful(ctx)
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = updates / e2e_s / 1e9

    peak, peak_src = measured_peaks()
    ordinal = int(statistics.mode(s["top_gather_ordinal"] for s in top_stats))
    cc.cc_destroy(ctx)
    ctx = None
    measured = None
    if world == 1 and not args.no_ncu:
        measured = measure_dominant_traffic(args, ordinal)
    agg_bytes = stats["agg_bytes"]
    agg_avg_ms = statistics.mean(agg_ms)
    # dominant kernel = the longest neighbour-sum launch of the step (its
    # algorithmic bytes / its CUDA-event time on the library's stream)
    top_bytes = statistics.mean(s["top_gather_bytes"] for s in top_stats)
    top_ms = statistics.mean(s["top_gather_ms"] for s in top_stats)
    achieved = top_bytes / (top_ms * 1e-3) / 1e9 if top_ms > 0 else None
    if measured:
        traffic, traffic_src = measured["dram_bytes"], "ncu one-launch pass in this run (NVTX range cc_dominant)"
    else:
        traffic, traffic_src = dominant_traffic(cfg.idx, precision)
        traffic_src = (traffic_src or "none") + " (committed capture; the in-run ncu pass did not run)"
    launches = int(stats["launches"]) + 1  # + the colour kernel
    dram_achieved = traffic / (top_ms * 1e-3) / 1e9 if traffic and top_ms else None

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if (world > 1 and not args.replicas) else "weak", "vs_baseline": None, "dtype": "f32" if precision == "fp32" else "f64",
                "data": "synthetic",
                "config": {"workload": f"configs[{cfg.idx}] {cfg.name}", "n": g.n, "adjacency": g.nnz,
                           "k": cfg.k, "precision": precision, "parallelism": (f"colouring-replicas x{world}" if args.replicas and world > 1
                                                           else f"1d-vertex-partition x{world}"),
                           "l2": "tables of several GB per step >> 126 MB L2 (no flush needed)"},
                # headline: the dominant launch's DRAM bytes (measured) over its CUDA-event time
                "roofline": {"bound": "hbm", "achieved": dram_achieved, "peak": peak, "unit": "GB/s",
                             "frac": dram_achieved / peak if dram_achieved else None, "traffic": traffic,
                             "kernel": "the longest neighbour-sum (SpMM gather) launch of the step",
                             "basis": "DRAM read+write bytes of that launch / its CUDA-event duration",
                             "ms_per_launch": top_ms, "peak_source": peak_src, "traffic_source": traffic_src,
                             "l2_hit_rate_pct": measured["l2_hit_rate_pct"] if measured else None,
                             "ncu_kernels": measured["kernels"] if measured else None,
                             # secondary: algorithmic bytes (index stream + the neighbour rows' non-skipped
                             # sectors + N'' rows), which count L2 hits on hub rows too
                             "algorithmic": {"bytes_per_launch": top_bytes, "achieved": achieved,
                                             "frac": achieved / peak if achieved else None}},
                "gather_family": {"passes_per_step": stats["gather_launches"],
                                  "algorithmic_bytes_per_step": agg_bytes, "ms_per_step": agg_avg_ms,
                                  "achieved_gbs": agg_bytes / (agg_avg_ms * 1e-3) / 1e9 if agg_avg_ms > 0 else None},
                "model_bytes_per_step": stats["model_bytes"],
                "model_hbm_frac": stats["model_bytes"] / (ms_per_step * 1e-3) / 1e9 / peak,
                "phase_ms": {k: round(v, 3) for k, v in last_prof.items()},
                "colorful_maps": xs[0],
                "peak_table_bytes": stats["peak_table_bytes"],
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(g.n),
                        "d2h_bytes_per_step": 8, "ms_per_step": e2e_s * 1e3,
                        "api": "cc_set_colors(host colouring) + cc_count_colorful"},
                "gpu_launches": launches * args.steps,
                "nvlink": ({"schedule": {1: "grouped", 2: "ring", 3: "alltoall", 4: "device"}.get(stats["exchange"]),
                            "halo_bytes_received_per_step_rank0": stats["halo_bytes"],
                            "exchange_ms_per_step_rank0": last_prof["exchange"],
                            "exposed_exchange_ms_per_step_rank0": last_prof.get("exposed_exchange"),
                            # overlap ratio: share of the exchange hidden behind
                            # the local gathers on rank 0
                            "overlap_ratio_rank0": (1.0 - last_prof.get("exposed_exchange", 0.0) / last_prof["exchange"]
                                                    if last_prof["exchange"] > 0 else None),
                            "gbs_rank0": (stats["halo_bytes"] / (last_prof["exchange"] * 1e-3) / 1e9
                                          if last_prof["exchange"] > 0 else None),
                            "peak_gbs": 900.0, "peak_source": "nominal NVLink 5 per direction per GPU"}
                           if world > 1 and not args.replicas else None),
                "clocks": clk}
        if world > 1:
            sizes = nccl_comm_sizes()
            line["nccl"] = {"comm_nranks": sizes, "comm_nranks_ok": bool(sizes) and all(x == world for x in sizes),
                            "log_dir": os.environ.get("CC_NCCL_LOG_DIR")}
        if not args.no_cpu_baseline and world == 1:
            scale = args.cpu_scale or auto_cpu_scale(cfg)
            v, ms, desc = oracle_sample(cfg, scale, args.seed)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                                    "sample": desc, "ms": ms, **host_info()}
        print(json.dumps(line), flush=True)
    if ctx is not None:
        cc.cc_destroy(ctx)


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: start N ranks (one
    process per GPU) through torch.distributed.run on this node and return
    its exit code.  NCCL's INIT log of every rank goes to files under
    $CC_NCCL_LOG_DIR (default /tmp/cc_nccl_logs) so the communicator sizes can be
    checked; rank 0's JSON line is the only line on stdout."""
    import torch
    have = torch.cuda.device_count()
    if args.impl != "reference" and have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
        return 2
    env = dict(os.environ)
    logdir = env.setdefault("CC_NCCL_LOG_DIR", "/tmp/cc_nccl_logs")
    os.makedirs(logdir, exist_ok=True)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", os.path.join(logdir, "nccl.%h.%p.log"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def nccl_comm_sizes() -> list:
    """nRanks of every NCCL communicator this process initialised (from its
    NCCL INIT log, when NCCL_DEBUG_FILE was set by self_launch)."""
    import glob
    import re
    logdir = os.environ.get("CC_NCCL_LOG_DIR")
    if not logdir:
        return []
    sizes = []
    for p in glob.glob(os.path.join(logdir, f"nccl.*.{os.getpid()}.log")):
        with open(p, errors="replace") as f:
            for line in f:
                m = re.search(r"comm 0x[0-9a-f]+ rank (\d+) nRanks (\d+)", line)
                if m:
                    sizes.append(int(m.group(2)))
    return sizes


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
    if local_world > 1:
        # every rank validates and partitions the whole graph on the host (OpenMP):
        # share the host cores (torchrun's default OMP_NUM_THREADS=1 would make
        # that serial, the OpenMP default would oversubscribe them N times)
        os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // local_world))
    import synth
    cfg = synth.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    dist = None
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if args.ncu_child:
        ncu_child(args, cfg)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    run_ours(args, cfg, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
