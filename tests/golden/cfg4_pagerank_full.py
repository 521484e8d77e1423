"""The ORACLE's full PageRank vector on BASELINE.json configs[4] (R-MAT scale 26, edgefactor
28, seed 5; Fig. 8 with k = 10), for the element-by-element cfg4 parity test
(tests/test_zz_cfg4_full_gpu.py).  Calls only oracle/ and inputs/ -- never the CUDA path.

tests/conftest.py starts it in the background when a GPU test session begins, so the ~12 min
of one host core (oracle adjacency build ~190 s + 11 supersteps of ~48 s) overlap the other GPU
tests; the test waits for it.  Writes <out>.npy (the 67,108,864 f64 values) and <out>.json
(counters, timings) atomically (rename when complete).

    python tests/golden/cfg4_pagerank_full.py --out /tmp/ipregel_cfg4_pr
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--config", default="cfg4")
    a = ap.parse_args()
    cfg = inputs.CONFIGS[a.config]
    t0 = time.time()
    src, dst, _ = inputs.rmat_coo(cfg.scale, cfg.edgefactor, cfg.seed, weighted=False)
    t_gen = time.time() - t0
    r = oracle.pagerank(cfg.n, src, dst, k=cfg.iterations)
    del src, dst
    v = r["values"]
    np.save(a.out + ".tmp.npy", v)
    meta = {"config": a.config, "n": cfg.n, "supersteps": int(r["supersteps"]),
            "changed": [int(x) for x in r["changed"]],
            "messages": [int(x) for x in r["messages"]],
            "oracle_superstep_seconds": [float(x) for x in r["seconds"]],
            "oracle_build_seconds": float(r["build_seconds"]), "generate_seconds": t_gen,
            "total_seconds": time.time() - t0, "sum": float(np.sum(v, dtype=np.float64))}
    with open(a.out + ".tmp.json", "w") as f:
        json.dump(meta, f)
    os.replace(a.out + ".tmp.npy", a.out + ".npy")
    os.replace(a.out + ".tmp.json", a.out + ".json")


if __name__ == "__main__":
    main()
