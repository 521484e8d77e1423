"""Run one of the paper's programs as an NVRTC user program on a BASELINE config (for ncu).

    python tools/run_program.py --config cfg4 --program sssp [--params 0] [--repeat 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from paper_2010_08781_b200 import programs  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--program", default="sssp")
ap.add_argument("--params", default="0")
ap.add_argument("--mode", default="auto")
ap.add_argument("--repeat", type=int, default=2)
a = ap.parse_args()
g = config_graph_device(a.config, weighted=True, degree_order=True)
G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                 g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"],
                                 degree_ordered=True))
p = programs.compile(a.program)
params = [float(x) for x in a.params.split(",")] if a.params else []
for _ in range(a.repeat):
    G.run_program(p, params=params, mode=a.mode)
    torch.cuda.synchronize()
    s = G.stats()
    print(f"{a.program}: modes {''.join('ilpr'[m] for m in s['mode'])} superstep ms "
          f"{[round(float(x), 3) for x in s['time_ms']]}", flush=True)
G.close()
