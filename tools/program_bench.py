"""User programs vs the built-in apps, and fused vs collective exchange on loopback partitions,
on a BASELINE config (device time from the library's own per-superstep CUDA events).

    python tools/program_bench.py [--config cfg4] [--parts 1,2,4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from paper_2010_08781_b200 import programs  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--parts", default="1,2,4")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
g = config_graph_device(a.config, weighted=True, degree_order=True)
n, e = g["n"], g["e"]
progs = {k: programs.compile(k) for k in ("pagerank", "hashmin_cc", "sssp")}
out = {"config": a.config, "n": n, "e": e, "rows": []}


def timed(G, fn):
    best = None
    for _ in range(a.reps):
        fn()
        torch.cuda.synchronize()
        s = G.stats()
        t = float(np.sum(s["time_ms"]))
        best = t if best is None else min(best, t)
    return best, s


for parts in [int(x) for x in a.parts.split(",")]:
    if parts == 1:
        G = ipr.Graph(ipr.full_partition(n, e, g["csc_off"], g["csc_idx"], g["csr_off"], g["csr_idx"],
                                         g["csc_w"], g["csr_w"], g["vertex_ids"], degree_ordered=True))
        exchanges = ["auto"]
    else:
        b = ipr.edge_balanced_bounds(g["csc_off"].cpu().numpy(), parts, g["csr_off"].cpu().numpy())
        G = ipr.Graph(ipr.split_partitions(n, e, b, g["csc_off"], g["csc_idx"], g["csr_off"],
                                           g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"],
                                           degree_ordered=True))
        exchanges = ["fused", "collective"]
    for ex in exchanges:
        for app in ("pagerank", "cc", "sssp"):
            mode = "pull" if app == "pagerank" else "auto"
            t_b, s_b = timed(G, lambda: G.run(app, mode=mode, exchange=ex))
            pname = {"pagerank": "pagerank", "cc": "hashmin_cc", "sssp": "sssp"}[app]
            params = [10] if app == "pagerank" else ([0] if app == "sssp" else [])
            t_p, s_p = timed(G, lambda: G.run_program(progs[pname], params=params, mode=mode,
                                                      exchange=ex))
            row = {"parts": parts, "exchange": ex, "app": app, "builtin_ms": round(t_b, 3),
                   "program_ms": round(t_p, 3), "supersteps": int(s_b["supersteps"]),
                   "program_supersteps": int(s_p["supersteps"]),
                   "builtin_modes": "".join("ilpr"[m] for m in s_b["mode"]),
                   "program_modes": "".join("ilpr"[m] for m in s_p["mode"])}
            out["rows"].append(row)
            print(json.dumps(row), flush=True)
    G.close()
print(json.dumps(out))
