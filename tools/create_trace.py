"""Create-phase timeline of a host-memory create at cfg4 (IPREGEL_TRACE_CREATE=1 prints the
library's CUDA-event marks), on torch's default stream and on a private stream."""
import os
import sys

os.environ.setdefault("IPREGEL_TRACE_CREATE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = config_graph_device(cfg, weighted=True, degree_order=True)
host = {}
for k in ("csc_off", "csc_idx", "csc_w", "vertex_ids"):
    h = torch.empty(g[k].shape, dtype=g[k].dtype, pin_memory=True)
    h.copy_(g[k])
    host[k] = h.numpy()
n, e = g["n"], g["e"]
del g
torch.cuda.empty_cache()
part = ipr.Partition(n, e, 0, n, host["csc_off"], host["csc_idx"], None, None, host["csc_w"], None,
                     host["vertex_ids"], True)
for name, st in (("default", None), ("private", torch.cuda.Stream()), ("default", None),
                 ("private", torch.cuda.Stream())):
    print("---", name, flush=True)
    G = ipr.Graph(part, stream=st)
    torch.cuda.synchronize()
    G.close()
    torch.cuda.synchronize()
