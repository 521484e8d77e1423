"""Small end-to-end sweep of every app, mode and exchange (1 and 3 partitions), the to-convergence
PageRank, the Hash-Min row-list pull and user programs (a quick all-paths smoke run; compute-sanitizer
is not available on the GPU pool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tests import checkers  # noqa: E402
from tests.graphs import csr_csc, make_graph  # noqa: E402

rng = np.random.default_rng(1)
n = 3000
src, dst, w = checkers.random_graph(rng, n, 20000, weighted=True)
g = csr_csc(n, src, dst, w)
progs = None
if "--programs" in sys.argv:
    from paper_2010_08781_b200 import programs
    progs = {k: programs.compile(k) for k in ("pagerank", "hashmin_cc", "sssp", "widest_path")}
for parts in (1, 3):
    G = make_graph(g, partitions=parts)
    for ex in (("auto",) if parts == 1 else ("fused", "collective")):
        for app in ("pagerank", "cc", "sssp"):
            for mode in ("pull", "push", "auto"):
                if app == "pagerank" and mode == "auto":
                    continue
                G.run(app, mode=mode, exchange=ex)
                v = G.values(host=True)
        G.run("pagerank", mode="pull", iterations=40, tolerance=1e-9, exchange=ex)
        G.run("cc", mode="pull", push_fraction=0.0, exchange=ex)   # reaches the row-list pull
        assert 3 in list(G.stats()["mode"])
        if progs:
            for name, p in progs.items():
                for mode in ("pull", "push", "auto"):
                    G.run_program(p, params=[10] if name == "pagerank" else [0], mode=mode,
                                  exchange=ex)
                    v = G.values(host=True)
    G.close()
print("ok")   # a run-everything smoke; parity against the oracle lives in tests/ only
