"""Per-superstep device times of the paper's programs as user programs vs the built-in apps
(cfg4 by default; library CUDA events).

    python tools/program_times.py [--config cfg4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2010_08781_b200 as ipr  # noqa: E402
from paper_2010_08781_b200 import programs  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
a = ap.parse_args()
g = config_graph_device(a.config, weighted=True, degree_order=True)
G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                 g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"],
                                 degree_ordered=True))
for app, pname, params in (("cc", "hashmin_cc", []), ("sssp", "sssp", [0])):
    p = programs.compile(pname)
    for label, fn in (("builtin", lambda: G.run(app, mode="auto")),
                      ("program", lambda: G.run_program(p, params=params, mode="auto"))):
        fn()
        fn()
        s = G.stats()
        print(f"{app:5s} {label:8s} total {float(s['time_ms'].sum()):7.2f} ms modes "
              f"{''.join('ilpr'[m] for m in s['mode'])} {[round(float(x), 2) for x in s['time_ms']]}",
              flush=True)
