"""How much of the PageRank range kernel's time do short rows take?  Times a PageRank pull
superstep (library events) on the cfg4 degree-ordered CSC and on copies where every row with
in-degree <= T keeps no edges (the long rows unchanged), and reports the short rows' edge count
and the sliced-ELL (32 consecutive rows per slice) padding they would need.  Not product code.

    python tools/short_rows_lab.py [--thresholds 16,32,64,128]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--thresholds", default="16,32,64,128")
a = ap.parse_args()
g = config_graph_device("cfg4", weighted=False, degree_order=True)
n, e = g["n"], g["e"]
off = g["csc_off"].long()
deg = off[1:] - off[:-1]


def superstep_ms(csc_off, csc_idx):
    # num_edges stays E (the CSR is the full one); the CSC holds only the kept rows' edges
    G = ipr.Graph(ipr.Partition(n, e, 0, n, csc_off, csc_idx, g["csr_off"], g["csr_idx"], None,
                                None, g["vertex_ids"], True))
    G.run("pagerank", mode="pull")
    G.run("pagerank", mode="pull")
    s = G.stats()
    G.close()
    return float(np.median(s["time_ms"][1:10]))


full = superstep_ms(g["csc_off"], g["csc_idx"])
print(f"full: E={e} superstep {full:.3f} ms", flush=True)
for t in [int(x) for x in a.thresholds.split(",")]:
    short = deg <= t
    e_short = int(deg[short].sum())
    # sliced ELL over consecutive rows: width of each slice of 32 = max short degree in it
    dd = torch.where(short, deg, torch.zeros_like(deg))
    pad = torch.nn.functional.pad(dd, (0, (-n) % 32)).view(-1, 32)
    entries = int(pad.max(dim=1).values.sum()) * 32
    keep = torch.repeat_interleave(~short, deg)
    idx2 = g["csc_idx"][keep]
    off2 = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    off2[1:] = torch.cumsum(torch.where(short, torch.zeros_like(deg), deg), 0)
    ms = superstep_ms(off2.to(torch.int32), idx2)
    print(f"T={t}: short rows {int(short.sum())} hold {e_short} edges ({e_short / e:.3f} of E); "
          f"sliced ELL entries {entries} ({entries / max(e_short, 1):.2f}x); superstep without "
          f"their edges {ms:.3f} ms (full {full:.3f})", flush=True)
    del keep, idx2, off2, pad, dd
    torch.cuda.empty_cache()
