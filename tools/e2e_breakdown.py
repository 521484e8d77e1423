"""Where the end-to-end step (bench.py e2e) spends its time: create (H2D + derived CSR + plans),
the three runs, get_values, destroy.  Wall clock around each synchronous C-ABI call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = config_graph_device(cfg, weighted=True, degree_order=True)
host = {}
for k in ("csc_off", "csc_idx", "csc_w", "csr_off", "csr_idx", "csr_w", "vertex_ids"):
    h = torch.empty(g[k].shape, dtype=g[k].dtype, pin_memory=True)
    h.copy_(g[k])
    host[k] = h.numpy()
n, e = g["n"], g["e"]
del g
torch.cuda.empty_cache()
out_pr = torch.empty(n, dtype=torch.float64, pin_memory=True)
out_u = torch.empty(n, dtype=torch.int32, pin_memory=True)
for derive in (True, False) + (True,) * 8:
    if derive:
        part = ipr.Partition(n, e, 0, n, host["csc_off"], host["csc_idx"], None, None,
                             host["csc_w"], None, host["vertex_ids"], True)
    else:
        part = ipr.full_partition(n, e, host["csc_off"], host["csc_idx"], host["csr_off"],
                                  host["csr_idx"], host["csc_w"], host["csr_w"],
                                  host["vertex_ids"], degree_ordered=True)
    t = {}
    t0 = time.perf_counter()
    G = ipr.Graph(part)
    torch.cuda.synchronize()
    t["create"] = time.perf_counter() - t0
    for app in ("pagerank", "cc", "sssp"):
        t0 = time.perf_counter()
        G.run(app, mode="pull" if app == "pagerank" else "auto")
        t[app] = time.perf_counter() - t0
        o = out_pr if app == "pagerank" else out_u
        t0 = time.perf_counter()
        ipr.load().ipregel_get_values(G.handle, o.data_ptr(), o.numel() * o.element_size(), 0)
        t["get_" + app] = time.perf_counter() - t0
    t0 = time.perf_counter()
    G.close()
    torch.cuda.synchronize()
    t["destroy"] = time.perf_counter() - t0
    print("derive" if derive else "given ", {k: round(v * 1e3, 1) for k, v in t.items()},
          "total", round(sum(t.values()) * 1e3, 1), flush=True)

# create from DEVICE arrays (no H2D): CSR given vs derived -> the derivation and plan costs
gd = config_graph_device(cfg, weighted=True, degree_order=True)
for derive in (False, True, False, True):
    if derive:
        part = ipr.Partition(n, e, 0, n, gd["csc_off"], gd["csc_idx"], None, None, gd["csc_w"],
                             None, gd["vertex_ids"], True)
    else:
        part = ipr.full_partition(n, e, gd["csc_off"], gd["csc_idx"], gd["csr_off"], gd["csr_idx"],
                                  gd["csc_w"], gd["csr_w"], gd["vertex_ids"], degree_ordered=True)
    t0 = time.perf_counter()
    G = ipr.Graph(part)
    torch.cuda.synchronize()
    tc = time.perf_counter() - t0
    t0 = time.perf_counter()
    G.close()
    torch.cuda.synchronize()
    print("device create", "derive" if derive else "given ", round(tc * 1e3, 1), "ms, destroy",
          round((time.perf_counter() - t0) * 1e3, 1), "ms", flush=True)
