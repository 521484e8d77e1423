"""Direction-optimising superstep at cfg4: per-superstep device time of
Hash-Min CC and SSSP in forced PULL, forced PUSH and AUTO (several push fractions), on the
library-relabelled graph bench.py uses.  Values and counters are identical in every mode (the
parity tests check that), so superstep s does the same algorithmic work in each column.

    python tools/f1_table.py [--config cfg4] [--fractions 0.01,0.02,0.04,0.08,0.16] [--out f.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--fractions", default="0.005,0.01,0.02,0.04,0.08,0.16")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default=None)
a = ap.parse_args()
g = config_graph_device(a.config, weighted=True, degree_order=False)
G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], None, None,
                                 g["csc_w"], None, layout=ipr.LAYOUT_DEGREE))
res = {}
for app in ("cc", "sssp"):
    rows = {}
    runs = [("pull", "pull", 0.04), ("push", "push", 0.04)] + \
           [(f"auto@{f}", "auto", float(f)) for f in a.fractions.split(",")]
    for name, mode, frac in runs:
        best = None
        for _ in range(a.reps):
            G.run(app, mode=mode, push_fraction=frac)
            s = G.stats()
            t = np.asarray(s["time_ms"], np.float64)
            if best is None or t.sum() < best[0].sum():
                best = (t, s)
        t, s = best
        rows[name] = {"ms": [round(float(x), 3) for x in t], "total_ms": round(float(t.sum()), 3),
                      "modes": "".join("ilpr"[m] for m in s["mode"]),
                      "messages": [int(x) for x in s["messages"]]}
        print(f"{app:5s} {name:10s} total {t.sum():8.2f} ms  modes {rows[name]['modes']}  "
              f"{rows[name]['ms']}", flush=True)
    # per superstep: the better fixed mode, and each AUTO setting against it
    pull, push = np.array(rows["pull"]["ms"]), np.array(rows["push"]["ms"])
    best_fixed = np.minimum(pull, push)
    for name in rows:
        if name.startswith("auto"):
            t = np.array(rows[name]["ms"])
            rows[name]["slower_than_best_fixed_ms"] = [round(float(x), 3)
                                                       for x in np.maximum(t - best_fixed, 0)]
    rows["best_fixed_per_superstep_ms"] = [round(float(x), 3) for x in best_fixed]
    rows["best_fixed_total_ms"] = round(float(best_fixed.sum()), 3)
    res[app] = rows
G.close()
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
