"""Small end-to-end run of every app and mode (1 and 3 partitions) for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from tests import checkers  # noqa: E402
from tests.graphs import csr_csc, make_graph  # noqa: E402

rng = np.random.default_rng(1)
n = 3000
src, dst, w = checkers.random_graph(rng, n, 20000, weighted=True)
g = csr_csc(n, src, dst, w)
for parts in (1, 3):
    G = make_graph(g, partitions=parts)
    for app in ("pagerank", "cc", "sssp"):
        for mode in ("pull", "push", "auto"):
            if app == "pagerank" and mode == "auto":
                continue
            G.run(app, mode=mode)
            v = G.values(host=True)
    G.close()
o = oracle.sssp(n, src, dst, w)
print("ok", int((o["values"] != oracle.INF).sum()))
