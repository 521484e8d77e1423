"""Run one app on one BASELINE.json config through the C ABI (for ncu / compute-sanitizer).

    python tools/run_app.py --config cfg4 --app pagerank --iterations 2 [--mode pull] [--repeat 1]
                            [--degree-order | --relabel]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--app", default="pagerank")
ap.add_argument("--iterations", type=int, default=2)
ap.add_argument("--mode", default="auto")
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--degree-order", action="store_true")
ap.add_argument("--relabel", action="store_true",
                help="original-id CSC relabelled by the library (bench.py's graph)")
a = ap.parse_args()
g = config_graph_device(a.config, weighted=True, degree_order=a.degree_order and not a.relabel)
if a.relabel:
    G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], None, None,
                                     g["csc_w"], None, layout=ipr.LAYOUT_DEGREE))
else:
    G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                     g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"],
                                     degree_ordered=a.degree_order))
for _ in range(a.repeat):
    t = time.time()
    G.run(a.app, mode=a.mode, iterations=a.iterations)
    torch.cuda.synchronize()
    s = G.stats()
    print(f"{a.app} {a.config}: {s['supersteps']} supersteps, {time.time() - t:.3f}s, "
          f"superstep ms {[round(float(x), 3) for x in s['time_ms']]}, "
          f"kernel ms {[round(float(x), 3) for x in s['kernel_ms']]}")
G.close()
