"""Per-superstep device times of the built-in apps on a BASELINE config (library CUDA events).

    python tools/app_times.py [--config cfg4] [--apps cc,sssp,pagerank] [--modes auto]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2010_08781_b200 as ipr  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--apps", default="cc,sssp,pagerank")
ap.add_argument("--modes", default="auto")
ap.add_argument("--relabel", action="store_true",
                help="original-id CSC relabelled by the library (bench.py's graph)")
a = ap.parse_args()
g = config_graph_device(a.config, weighted=True, degree_order=not a.relabel)
if a.relabel:
    G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], None, None,
                                     g["csc_w"], None, layout=ipr.LAYOUT_DEGREE))
else:
    G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                     g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"],
                                     degree_ordered=True))
for app in a.apps.split(","):
    for mode in a.modes.split(","):
        m = "pull" if app == "pagerank" and mode == "auto" else mode
        G.run(app, mode=m)
        G.run(app, mode=m)
        s = G.stats()
        print(f"{app:8s} {m:5s} total {float(s['time_ms'].sum()):8.2f} ms  "
              f"{[round(float(x), 2) for x in s['time_ms']]}", flush=True)
G.close()
