"""bench.py's end-to-end step, repeated, with the wall time of each phase (create, the three runs,
sync, destroy): which phase an outlier step spends its extra time in.  Not product code.

    python tools/e2e_steps.py [--config cfg4] [--steps 14] [--device-first]
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
ap.add_argument("--steps", type=int, default=14)
ap.add_argument("--device-first", action="store_true",
                help="create, run and close a device-resident graph first (as bench.py does)")
a = ap.parse_args()
g = config_graph_device(a.config, weighted=True, degree_order=False)
n, e = g["n"], g["e"]
if a.device_first:
    G = ipr.Graph(ipr.full_partition(n, e, g["csc_off"], g["csc_idx"], None, None, g["csc_w"],
                                     None, layout=ipr.LAYOUT_DEGREE))
    for app in ("pagerank", "cc", "sssp"):
        G.run(app, mode="pull" if app == "pagerank" else "auto")
    G.close()
host = {}
for k in ("csc_off", "csc_idx", "csc_w"):
    h = torch.empty(g[k].shape, dtype=g[k].dtype, pin_memory=True)
    h.copy_(g[k])
    host[k] = h.numpy()
del g
torch.cuda.synchronize()
torch.cuda.empty_cache()
part = ipr.full_partition(n, e, host["csc_off"], host["csc_idx"], None, None, host["csc_w"], None,
                          layout=ipr.LAYOUT_DEGREE)
outs = {app: torch.empty(n, dtype=torch.float64 if app == "pagerank" else torch.int32,
                         pin_memory=True) for app in ("pagerank", "cc", "sssp")}
lib = ipr.load()
stream = torch.cuda.Stream()
for i in range(a.steps):
    t = {}
    t0 = time.perf_counter()
    G = ipr.Graph(part, stream=stream)
    t["create"] = time.perf_counter() - t0
    for app in ("pagerank", "cc", "sssp"):
        t0 = time.perf_counter()
        G.run(app, mode="pull" if app == "pagerank" else "auto")
        o = outs[app]
        lib.ipregel_get_values_async(G.handle, o.data_ptr(), o.numel() * o.element_size())
        t[app] = time.perf_counter() - t0
    t0 = time.perf_counter()
    lib.ipregel_graph_sync(G.handle)
    t["sync"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    G.close()
    stream.synchronize()
    t["destroy"] = time.perf_counter() - t0
    free, total = torch.cuda.mem_get_info()
    print(i, {k: round(v * 1e3, 1) for k, v in t.items()}, "total",
          round(sum(t.values()) * 1e3, 1), f"free {free / 2**30:.1f} GiB", flush=True)
