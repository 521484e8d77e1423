"""Write tests/golden/cfg4_oracle.json: the ORACLE's results on BASELINE.json
configs[4] (R-MAT scale 26, edgefactor 28, seed 5), for the full-size GPU
parity tests.  Calls only oracle/ and inputs/ -- never the CUDA path.

Stored per app: status, superstep count, per-superstep changed/messages, a
sha256 of the whole value array (CC labels / SSSP distances are compared
bit-exactly through it), and the values at a fixed sample of vertices
(PageRank is compared there within the 1e-9 gate).

Runs single-threaded in the oracle (~30 min, ~40 GB RAM):
    python tests/golden/make_cfg4_golden.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg4_oracle.json")


def sample_ids(n, count=1 << 16, seed=12345):
    """Fixed vertex sample: the 64 lowest ids (the R-MAT hubs) + uniform draws."""
    rng = np.random.default_rng(seed)
    ids = np.unique(np.concatenate([np.arange(64), rng.integers(0, n, count)]))
    return ids.astype(np.int64)


def main():
    cfg = inputs.CONFIGS["cfg4"]
    n = cfg.n
    t = time.time()
    src, dst, w = inputs.config_coo(cfg)
    print(f"generated E={len(src)} in {time.time() - t:.1f}s", flush=True)
    ids = sample_ids(n)
    out = {"config": "cfg4", "n": n, "edges": int(len(src)),
           "coo_sha256": inputs.array_digest(src, dst, w),
           "sample_ids": ids.tolist(), "apps": {}}
    for app, name in ((oracle.APP_PAGERANK, "pagerank"), (oracle.APP_HASHMIN_CC, "cc"),
                      (oracle.APP_SSSP, "sssp")):
        t = time.time()
        r = oracle.run(app, n, src, dst, w if app == oracle.APP_SSSP else None,
                       k=cfg.iterations, source=0)
        v = r["values"]
        rec = {"status": r["status"], "supersteps": r["supersteps"],
               "changed": [int(x) for x in r["changed"]],
               "messages": [int(x) for x in r["messages"]],
               "oracle_superstep_seconds": [float(x) for x in r["seconds"]],
               "oracle_build_seconds": r["build_seconds"],
               "values_sha256": inputs.array_digest(v),
               "sample_values": [float(x) for x in v[ids]] if app == oracle.APP_PAGERANK
               else [int(x) for x in v[ids]]}
        if app == oracle.APP_PAGERANK:
            rec["sum"] = float(np.sum(v, dtype=np.float64))
        else:
            key = "unreached" if app == oracle.APP_SSSP else "roots"
            rec[key] = int((v == oracle.INF).sum()) if app == oracle.APP_SSSP \
                else int((v == np.arange(n, dtype=np.uint32)).sum())
        out["apps"][name] = rec
        print(f"{name}: {r['supersteps']} supersteps in {time.time() - t:.1f}s", flush=True)
        del r, v
    with open(OUT, "w") as f:
        json.dump(out, f)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
