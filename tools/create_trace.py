"""Create-phase timeline of a host-memory create at cfg4 (--relabel: from the original-id CSC
with the library degree relabel) (IPREGEL_TRACE_CREATE=1 prints the
library's CUDA-event marks), on torch's default stream and on a private stream."""
import os
import sys

os.environ.setdefault("IPREGEL_TRACE_CREATE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
relabel = "--relabel" in sys.argv   # original-id CSC, IPREGEL_LAYOUT_DEGREE (bench.py's e2e)
g = config_graph_device(cfg, weighted=True, degree_order=not relabel)
host = {}
for k in ("csc_off", "csc_idx", "csc_w") + (() if relabel else ("vertex_ids",)):
    h = torch.empty(g[k].shape, dtype=g[k].dtype, pin_memory=True)
    h.copy_(g[k])
    host[k] = h.numpy()
n, e = g["n"], g["e"]
del g
torch.cuda.empty_cache()
if relabel:
    part = ipr.full_partition(n, e, host["csc_off"], host["csc_idx"], None, None, host["csc_w"],
                              None, layout=ipr.LAYOUT_DEGREE)
else:
    part = ipr.Partition(n, e, 0, n, host["csc_off"], host["csc_idx"], None, None, host["csc_w"],
                         None, host["vertex_ids"], True)
for name, st in (("default", None), ("private", torch.cuda.Stream()), ("default", None),
                 ("private", torch.cuda.Stream())):
    print("---", name, flush=True)
    import time
    t0 = time.perf_counter()
    G = ipr.Graph(part, stream=st)
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    if "--runs" in sys.argv:   # the e2e step's runs after create: is any waiting on the CSR?
        for app in ("pagerank", "cc", "sssp"):
            G.run(app)
            torch.cuda.synchronize()
            t.append(time.perf_counter())
    print("create %.1f ms, runs %s ms" % (1e3 * (t[0] - t0), [round(1e3 * (b - a), 1) for a, b in
                                                           zip(t[:-1], t[1:])]), flush=True)
    G.close()
    torch.cuda.synchronize()
