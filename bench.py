"""bench.py -- the driver's benchmark contract for the B200 iPregel superstep.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg4] [--apps pagerank,cc,sssp]

One STEP = one pass of the whole hot path over the synthetic input: PageRank (10 gather
supersteps, fp64), Hash-Min CC to convergence and SSSP from vertex 0 to convergence, each run
through the C ABI (ipregel_run) on BASELINE.json configs[4] (R-MAT scale 26, edgefactor 28,
seed 5: 67,108,864 vertices, 1.879e9 edges, int32 CSR + CSC, u32 weights in [1,64]).

metric: GTEPS = messages delivered (the method's edge work: every superstep s >= 1 delivers the
messages of superstep s-1) per second of device time, whole job (all ranks).  The inputs
(7.5 GB per adjacency array) are larger than L2, so no flush is needed between steps.

Extra keys: roofline (dominant kernel: the PageRank pull gather, algorithmic bytes per launch
12E + 24N over its CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs; frac_16N on
12E + 16N; request_bound: its L1 -> L2 gather requests against one request per SM per clock, the
limit it actually meets), cpu_baseline
(the oracle on a bounded sample, rank 0, N=1), e2e (host buffers through the C ABI, copies
inside the timed region), clocks (nvidia-smi sampled during the timed region), gpu_launches.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "GTEPS per superstep and % of HBM roofline at 1/2/4/8 B200"
UNIT = "GTEPS"
APP_CODES = {"pagerank": 0, "cc": 1, "sssp": 2}
# bounded sample of the cfg4 workload for the oracle: same generator and parameters
# (a, b, c, d, edgefactor 28, seed 5), 1/16 of the vertices (~10-30 s of one core)
SAMPLE_SCALE = 22


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------ helpers
def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """Per-launch DRAM bytes (read + write) of the PageRank pull kernel from the committed
    `ncu --set full` capture summary (profiles/pr_pull_ncu_summary.json)."""
    p = os.path.join(ROOT, "profiles", "pr_pull_ncu_summary.json")
    try:
        with open(p) as f:
            return float(json.load(f)["dram_bytes_per_launch"])
    except Exception:
        return None


def request_bound(range_ms, clocks, sms):
    """The limit the PageRank range kernel meets (profiles/r02/prf_ncu_full_s38.json): its
    L1 -> L2 read requests (one per distinct 128-byte line per warp gather, ncu
    lts__t_requests_srcunit_tex_op_read) against one request per SM per SM clock -- ncu shows the
    L1 -> XBAR request path 89 % busy and the L2 tag lookups 84 %, DRAM at 42 %."""
    p = os.path.join(ROOT, "profiles", "r02", "prf_ncu_full_s38.json")
    try:
        with open(p) as f:
            caps = json.load(f)
        req = next(float(k["metrics"]["lts__t_requests_srcunit_tex_op_read.sum"]["value"])
                   for k in caps if k["kernel"].startswith("k_pr_flag"))
    except Exception:
        return None
    mhz = (clocks or {}).get("sm_mhz") or 0
    if not mhz or not range_ms:
        return None
    cap = sms * mhz * 1e6 * range_ms * 1e-3
    return {"requests_per_launch": req, "source": "profiles/r02/prf_ncu_full_s38.json",
            "limit": "1 L1->L2 request per SM per clock", "sm_mhz": mhz,
            "frac": req / cap}


def device_info(device):
    import torch
    p = torch.cuda.get_device_properties(device)
    return {"name": p.name, "sms": p.multi_processor_count,
            "l2_bytes": getattr(p, "L2_cache_size", None),
            "hbm_bytes": p.total_memory}


def delivered_messages(stats):
    """Messages delivered by supersteps 1..S-1 = messages sent in supersteps 0..S-2."""
    m = stats["messages"].astype(np.int64)
    return int(m[:-1].sum()) if len(m) > 1 else 0


def build_graph_device(cfg_name, rank, world):
    import torch

    import inputs
    import paper_2010_08781_b200 as ipr
    from inputs.gpu import config_graph_device
    cfg = inputs.CONFIGS[cfg_name]
    t = time.time()
    if world == 1:
        # the user's graph in its ORIGINAL numbering (CSC + weights); the library relabels it
        # by out-degree during create (IPREGEL_LAYOUT_DEGREE) and derives the out-adjacency
        g = config_graph_device(cfg, weighted=True, degree_order=False)
        g["csr_off"] = g["csr_idx"] = g["csr_w"] = None
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        log(f"[rank {rank}] graph {cfg_name}: N={g['n']} E={g['e']} built in {time.time() - t:.1f}s")
        part = ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], None, None,
                                  g["csc_w"], None, layout=ipr.LAYOUT_DEGREE)
        return g, part, np.array([0, g["n"]])
    g = config_graph_device(cfg, weighted=True, degree_order=True)
    torch.cuda.synchronize()
    log(f"[rank {rank}] graph {cfg_name}: N={g['n']} E={g['e']} built in {time.time() - t:.1f}s")
    bounds = ipr.edge_balanced_bounds(g["csc_off"].cpu().numpy(), world, g["csr_off"].cpu().numpy())
    parts = ipr.split_partitions(g["n"], g["e"], bounds, g["csc_off"], g["csc_idx"], g["csr_off"],
                                 g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"],
                                 degree_ordered=True)
    # keep only this rank's slices alive (copies, so the full graph can be freed)
    p = parts[rank]
    own = ipr.Partition(p.num_vertices, p.num_edges, p.vertex_begin, p.vertex_end,
                        p.csc_offsets.clone(), p.csc_indices.clone(), p.csr_offsets.clone(),
                        p.csr_indices.clone(), p.csc_weights.clone(), p.csr_weights.clone(),
                        g["vertex_ids"], True)
    del parts
    for k in list(g.keys()):
        if k not in ("n", "e", "vertex_ids"):
            g[k] = None
    torch.cuda.empty_cache()
    return g, own, bounds


def run_step(G, apps, iterations=10, exchange="auto"):
    out = {}
    for app in apps:
        G.run(app, mode="pull" if app == "pagerank" else "auto", iterations=iterations,
              exchange=exchange)
        out[app] = G.stats()
    return out


# ------------------------------------------------------------------------------ cpu baseline
def host_info():
    """CPU model, logical CPUs and RAM of the box (the oracle's hardware)."""
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    info["cpu_model"] = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    info["ram_gb"] = round(int(ln.split()[1]) / 2**20, 1)
                    break
    except OSError:
        pass
    return info


def cfg4_oracle_context():
    """The oracle's own per-superstep times at the FULL cfg4 size (one core), from
    tests/golden/cfg4_oracle.json (written by tests/golden/make_cfg4_golden.py, oracle only):
    reported as context next to the bounded sample, never timed here."""
    p = os.path.join(ROOT, "tests", "golden", "cfg4_oracle.json")
    try:
        with open(p) as f:
            gold = json.load(f)
    except Exception:
        return None
    out = {}
    for app, rec in gold["apps"].items():
        secs = float(sum(rec["oracle_superstep_seconds"]))
        d = int(sum(rec["messages"][:-1]))
        out[app] = {"seconds": round(secs, 1), "gteps": d / secs / 1e9,
                    "supersteps": rec["supersteps"],
                    "superstep_seconds": [round(x, 2) for x in rec["oracle_superstep_seconds"]]}
    return {"source": "tests/golden/cfg4_oracle.json (full cfg4, one core, superstep loop only)",
            "apps": out}


def cpu_baseline(apps, scale=SAMPLE_SCALE, repeats=1):
    """The oracle (single-threaded C Pregel interpreter) on a bounded sample of cfg4, pinned to
    one host core (sched_setaffinity, the last CPU of the process's set) while it runs."""
    import inputs
    import oracle
    cfg = inputs.CONFIGS["cfg4"]
    src, dst, w = inputs.rmat_coo(scale, cfg.edgefactor, cfg.seed, weighted=True)
    n = 1 << scale
    msgs = 0
    secs = 0.0
    per_app = {}
    old_aff = os.sched_getaffinity(0)
    core = max(old_aff)
    os.sched_setaffinity(0, {core})
    try:
        for _ in range(repeats):
            for app in apps:
                r = oracle.run(APP_CODES[app], n, src, dst, w if app == "sssp" else None,
                               k=cfg.iterations, source=0)
                d = int(r["messages"][:-1].sum()) if r["supersteps"] > 1 else 0
                s = float(r["seconds"].sum())
                msgs += d
                secs += s
                per_app[app] = {"gteps": d / s / 1e9 if s > 0 else None, "seconds": s,
                                "supersteps": int(r["supersteps"])}
    finally:
        os.sched_setaffinity(0, old_aff)
    return {"value": msgs / secs / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "pinned_core": core, "host": host_info(), "full_size_context": cfg4_oracle_context(),
            "sample": (f"R-MAT scale {scale}, edgefactor {cfg.edgefactor}, seed {cfg.seed} "
                       f"(cfg4's generator at 1/{1 << (cfg.scale - scale)} of the vertices, "
                       f"E={len(src)}); {'+'.join(apps)} to termination; superstep loop only "
                       f"(adjacency build excluded, PAPER.md:428)"),
            "seconds": secs, "apps": per_app}


def reference_arm(args):
    """--impl reference: the oracle as it stands, on the host cores, same metric/unit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    apps = args.apps
    for _ in range(args.warmup):
        cpu_baseline(apps, scale=args.sample_scale)
    t_steps = []
    res = None
    for _ in range(args.steps):
        res = cpu_baseline(apps, scale=args.sample_scale)
        t_steps.append(res["seconds"])
    value = res["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(t_steps) / len(t_steps), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic",
        "config": {"workload": f"{args.config} sample: R-MAT scale {args.sample_scale}, ef 28, seed 5",
                   "apps": apps},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": res["sample"], "pinned_core": res["pinned_core"],
                         "host": res["host"], "full_size_context": res["full_size_context"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--apps", default="pagerank,cc,sssp")
    ap.add_argument("--sample-scale", type=int, default=SAMPLE_SCALE)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--comm", action="store_true",
                    help="use the NCCL communicator path even on one rank (tests the N>1 path)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "fused", "collective"],
                    help="pull-superstep exchange between ranks: fused epilogue stores over "
                         "CUDA-IPC-mapped peer replicas, or the collective AllGatherv (auto: "
                         "fused when every peer maps, else collective, logged)")
    args = ap.parse_args()
    args.apps = [a for a in args.apps.split(",") if a]

    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2010_08781_b200 as ipr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    ipr.device_check(local)
    use_comm = world > 1 or args.comm
    if use_comm:
        # NCCL logs to stderr, never into the JSON line on stdout; a multi-GPU run keeps its
        # INFO lines (ranks, rings, NVLS) there
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    if use_comm:
        # a standalone `--comm` run (no torchrun) is a world of one on this host
        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0"),
                     ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29541")):
            os.environ.setdefault(k, v)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    g, part, bounds = build_graph_device(args.config, rank, world)
    comm = ipr.Comm.from_process_group(local) if use_comm else None
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        G = ipr.Graph(part, comm=comm, stream=stream)
    n, e = g["n"], g["e"]

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            run_step(G, args.apps, exchange=args.exchange)
    torch.cuda.synchronize()

    # timed region: K steps, events on the library's stream, barrier + sync on both sides
    launches0 = ipr.kernel_launches()
    per_step = []
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        start.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                per_step.append(run_step(G, args.apps, exchange=args.exchange))
        stop.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = ipr.kernel_launches() - launches0
    ms_total = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([ms_total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_per_step = ms_total / args.steps

    # work per step (identical every step; counters are global, so rank-independent)
    msgs = sum(delivered_messages(st) for st in per_step[0].values())
    value = msgs / (ms_per_step * 1e-3) / 1e9

    # dominant kernel: the PageRank pull gather (+ its fixup), timed by the library's events
    peak, peak_src = measured_peak()
    apps_out = {}
    for app in args.apps:
        sts = [step[app] for step in per_step]
        t_app = float(np.mean([s["time_ms"].sum() for s in sts]))
        d = delivered_messages(sts[0])
        st0 = sts[0]
        apps_out[app] = {"gteps": d / (t_app * 1e-3) / 1e9, "ms": t_app,
                         "supersteps": int(st0["supersteps"]),
                         "modes": "".join("ilpr"[m] for m in st0["mode"]),
                         "exchange": st0.get("exchange"),
                         # per superstep (first timed step): device ms, messages sent, model bytes
                         "superstep_ms": [round(float(x), 4) for x in st0["time_ms"]],
                         "superstep_messages": [int(x) for x in st0["messages"]],
                         "superstep_model_gb": [round(float(x) / 1e9, 3) for x in st0["model_bytes"]]}
    roof = None
    if "pagerank" in args.apps:
        sts = [step["pagerank"] for step in per_step]
        k_ms = np.concatenate([s["kernel_ms"][1:] for s in sts])
        rk_ms = np.concatenate([s["part_ms"][1:] for s in sts])
        mb = np.concatenate([s["model_bytes"][1:] for s in sts]).astype(np.float64)
        t_ms = float(np.mean(k_ms))
        if world > 1:
            t = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_ms = float(t.item())
        # 12 B per edge + 24 B per vertex (per-rank bytes at N > 1); the 16 B
        # per-vertex variant leaves out the rank write a fixed-k run does in its last superstep
        # only
        achieved = float(np.mean(mb) / (t_ms * 1e-3) / 1e9)
        mb16 = 12.0 * e + 16.0 * n if world == 1 else np.mean(mb) - 8.0 * (n / world)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(),
                "kernel": "PageRank gather superstep: k_pr_flag + k_flag_fixup + "
                          "k_pr_finish (Fig. 8 update)",
                "bytes_per_launch": float(np.mean(mb)),
                "model": "SURVEY.md 8(d): 12 B/edge (4 B index + 8 B gathered f64 outbox) + "
                         "24 B/vertex (CSC offset, out-degree, rank, next outbox)",
                "avg_launch_ms": t_ms, "peak_source": peak_src,
                # attribution of the superstep (library events, same stream and clocks): the
                # range kernel + fixup, and the update pass (k_pr_finish)
                "range_kernel_ms": float(np.mean(rk_ms)),
                "update_pass_ms": float(np.mean(k_ms - rk_ms)),
                "frac_of_8TBps": achieved / 8000.0,
                "frac_16N": float(mb16 / (t_ms * 1e-3) / 1e9) / peak}
        apps_out["pagerank"]["superstep_ms_median"] = float(np.median(
            np.concatenate([s["time_ms"][1:] for s in sts])))
        apps_out["pagerank"]["gteps_per_gather_superstep"] = float(
            e / (apps_out["pagerank"]["superstep_ms_median"] * 1e-3) / 1e9)

    # device-memory footprint (the Table 3 analog): the user's graph arrays
    # (borrowed), the library's graph-side memory (range plans) and the vertex state
    gb, sb = G.memory_footprint()
    user_bytes = sum(int(t.numel()) * t.element_size() for t in
                     (part.csc_offsets, part.csc_indices, part.csc_weights, part.csr_offsets,
                      part.csr_indices, part.csr_weights) if t is not None)
    memory = {"user_graph_bytes": user_bytes, "library_graph_bytes": int(gb),
              "vertex_state_bytes": int(sb),
              "state_bytes_per_vertex": round(sb / (n / world), 2),
              "note": "vertex state is Theta(N) (single-slot mailboxes, PAPER.md:205-211, "
                      ":476-480); library graph bytes: the relabelled CSC and the derived CSR "
                      "(IPREGEL_LAYOUT_DEGREE), the range plans, and PageRank's row-end-flagged "
                      "copy of the CSC indices (4 B per edge, pr_flag.cuh); the user's arrays "
                      "are borrowed"}

    if roof is not None:
        roof["request_bound"] = request_bound(roof["range_kernel_ms"], clk.summary(),
                                              device_info(local)["sms"])
    # e2e: host buffers through the C ABI, H2D of the graph + D2H of every result in the region
    e2e = None
    G.close()   # its device state goes back to the pool for the e2e graphs
    G = None
    if not args.no_e2e:
        if use_comm:
            e2e = e2e_measure_ranks(part, n, e, args, msgs, stream, comm, world)
        else:
            part = None   # the device copy of the user's graph is not needed past this point
            e2e = e2e_measure(g, args, msgs, stream)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic",
        "config": {"workload": f"{args.config}: R-MAT scale 26 ef 28 seed 5, "
                               f"{'+'.join(args.apps)} per step",
                   "layout": "original-id CSC relabelled by out-degree by the library "
                             "(IPREGEL_LAYOUT_DEGREE, at create); results in original ids",
                   "n": n, "e": e, "parallelism": f"1D destination partition x{world}",
                   "exchange_requested": args.exchange,
                   "l2": "inputs larger than L2 (7.5 GB per adjacency array), no flush",
                   "device": device_info(local),
                   "apps": apps_out},
        "roofline": roof,
        "memory": memory,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.apps)
        line["cpu_baseline"].pop("apps", None)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm:
        comm.close()
    if use_comm:
        dist.destroy_process_group()


def e2e_measure_ranks(part, n, e, args, msgs_per_step, stream, comm, world):
    """e2e on the rank path (torchrun, N >= 1 with a communicator): every rank creates its
    partition from pinned host copies of its CSC + CSR slices (+ weights, vertex layout), runs
    the apps and reads every result back (ipregel_get_values: collective, every rank receives
    all N values).  Device time of the slowest rank; bytes summed over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2010_08781_b200 as ipr

    def pin(t):
        if t is None:
            return None, 0
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h, h.numel() * h.element_size()

    hs, h2d = {}, 0
    for k in ("csc_offsets", "csc_indices", "csc_weights", "csr_offsets", "csr_indices",
              "csr_weights", "vertex_ids"):
        hs[k], b = pin(getattr(part, k))
        h2d += b
    hpart = ipr.Partition(n, e, part.vertex_begin, part.vertex_end,
                          *[None if hs[k] is None else hs[k].numpy() for k in
                            ("csc_offsets", "csc_indices", "csr_offsets", "csr_indices",
                             "csc_weights", "csr_weights", "vertex_ids")],
                          part.degree_ordered, part.layout)
    outs = {app: torch.empty(n, dtype=torch.float64 if app == "pagerank" else torch.int32,
                             pin_memory=True) for app in args.apps}
    d2h = sum(o.numel() * o.element_size() for o in outs.values())
    steps = max(1, min(args.steps, 5))

    def one():
        G = ipr.Graph(hpart, comm=comm, stream=stream)
        lib = ipr.load()
        for app in args.apps:
            G.run(app, mode="pull" if app == "pagerank" else "auto", exchange=args.exchange)
            o = outs[app]
            assert lib.ipregel_get_values(G.handle, o.data_ptr(), o.numel() * o.element_size(),
                                          0) == 0, ipr.last_error()
        G.close()

    one()  # warm-up
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for i in range(steps):
        one()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    wall = (time.perf_counter() - t0) / steps
    each = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    t = torch.tensor([ev[0].elapsed_time(ev[steps]) / steps, float(h2d), float(d2h)],
                     device="cuda", dtype=torch.float64)
    tmax = t[:1].clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    tsum = t[1:].clone()
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    ms = float(tmax.item())
    return {"value": msgs_per_step / (ms * 1e-3) / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": int(tsum[0].item()), "d2h_bytes_per_step": int(tsum[1].item()),
            "ms_per_step": ms, "wall_ms_per_step": wall * 1e3,
            "ms_each_step": [round(x, 2) for x in each], "steps": steps, "ranks": world,
            "path": "per rank: ipregel_graph_create(IPREGEL_MEMORY_HOST, pinned CSC + CSR slices + "
                    "weights + vertex ids, communicator) + ipregel_run x apps + "
                    "ipregel_get_values(host, collective) + destroy; max over ranks, bytes "
                    "summed over ranks"}


def e2e_measure(g, args, msgs_per_step, stream):
    """Same work through ipregel_graph_create(MEMORY_HOST) from pinned host arrays.  The user's
    graph is its CSC (in-edges, weights) plus the vertex layout; the library uploads it and
    derives the out-adjacency on the device (all inside the timed region)."""
    import torch

    import paper_2010_08781_b200 as ipr
    host = {}
    h2d = 0
    for k in ("csc_off", "csc_idx", "csc_w"):
        t = g[k]
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        host[k] = h.numpy()
        h2d += h.numel() * h.element_size()
    # the user's graph lives in host memory from here on: its device copy (15 GB at cfg4, the
    # fixture's) goes back to the driver, so the library's pool has the device to itself
    for k in ("csc_off", "csc_idx", "csc_w"):
        g[k] = None
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    # the graph as the user has it: its CSC in ORIGINAL ids + weights; the library uploads it,
    # relabels it by out-degree (IPREGEL_LAYOUT_DEGREE) and derives the out-adjacency on the device
    part = ipr.full_partition(g["n"], g["e"], host["csc_off"], host["csc_idx"], None, None,
                              host["csc_w"], None, layout=ipr.LAYOUT_DEGREE)
    outs = {app: torch.empty(g["n"], dtype=torch.float64 if app == "pagerank" else torch.int32,
                             pin_memory=True) for app in args.apps}
    d2h = 0
    steps = max(1, min(args.steps, 5))

    def one():
        # each app's values are copied to pinned host memory asynchronously (the copy overlaps
        # the next app's run), all complete at ipregel_graph_sync
        nonlocal d2h
        d2h = 0
        G = ipr.Graph(part, stream=stream)
        lib = ipr.load()
        for app in args.apps:
            G.run(app, mode="pull" if app == "pagerank" else "auto")
            o = outs[app]
            st = lib.ipregel_get_values_async(G.handle, o.data_ptr(), o.numel() * o.element_size())
            assert st == 0, ipr.last_error()
            d2h += o.numel() * o.element_size()
        assert lib.ipregel_graph_sync(G.handle) == 0, ipr.last_error()
        G.close()

    # warm-up: the device pool grows to the job's high-water mark and its large blocks settle
    # (cfg4: ~60 GB of graph + state per handle, the 7.5 GB arrays landing in reused blocks)
    # and the pinned staging pages are taken, over the first graphs
    for _ in range(4):
        one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for i in range(steps):
        one()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps
    each = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    ms = ev[0].elapsed_time(ev[steps]) / steps
    return {"value": msgs_per_step / (ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "wall_ms_per_step": wall * 1e3,
            "ms_each_step": [round(x, 2) for x in each],
            "steps": steps,
            "path": "ipregel_graph_create(IPREGEL_MEMORY_HOST, pinned original-id CSC + weights, "
                    "IPREGEL_LAYOUT_DEGREE: degree relabel + CSR derived on the device) + "
                    "ipregel_run x apps, each followed by ipregel_get_values_async(pinned host) "
                    "+ ipregel_graph_sync + destroy"}


if __name__ == "__main__":
    main()
