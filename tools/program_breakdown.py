"""Per-superstep wall (time_ms) vs delivery-kernel (kernel_ms) time of the paper's programs as
NVRTC user programs vs the built-ins at cfg4 (library events).  Not product code."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2010_08781_b200 as ipr  # noqa: E402
from paper_2010_08781_b200 import programs  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

g = config_graph_device("cfg4", weighted=True, degree_order=True)
G = ipr.Graph(ipr.full_partition(g["n"], g["e"], g["csc_off"], g["csc_idx"], g["csr_off"],
                                 g["csr_idx"], g["csc_w"], g["csr_w"], g["vertex_ids"],
                                 degree_ordered=True))
for app, pname, params in (("cc", "hashmin_cc", []), ("sssp", "sssp", [0]),
                           ("pagerank", "pagerank", [10])):
    p = programs.compile(pname)
    for label, fn in (("builtin", lambda: G.run(app, mode="pull" if app == "pagerank" else "auto")),
                      ("program", lambda: G.run_program(p, params=params,
                                                        mode="pull" if app == "pagerank" else "auto"))):
        fn()
        fn()
        s = G.stats()
        print(f"{app} {label} total {float(s['time_ms'].sum()):.2f} modes "
              f"{''.join('ilpr'[m] for m in s['mode'])}")
        print("  time  ", [round(float(x), 3) for x in s["time_ms"]])
        print("  kernel", [round(float(x), 3) for x in s["kernel_ms"]], flush=True)
