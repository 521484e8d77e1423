"""Does the PageRank gather need each CSC row's sources ascending?  Times the PageRank and Hash-Min
/ SSSP supersteps (library events) on the cfg4 degree-relabelled CSC as the fixture builds it
(rows sorted by new source) and on the same rows with their edges in the ORIGINAL-id order (what a
relabel that moves rows and renames sources without sorting them would give).  Not product code.

    python tools/unsorted_rows_lab.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402
from inputs.gpu import config_graph_device  # noqa: E402


def times(off, idx, w, n, e, tag):
    G = ipr.Graph(ipr.full_partition(n, e, off, idx, None, None, w, None, None,
                                     degree_ordered=True))
    for app in ("pagerank", "cc", "sssp"):
        G.run(app, mode="pull" if app == "pagerank" else "auto")
        G.run(app, mode="pull" if app == "pagerank" else "auto")
        t = np.asarray(G.stats()["time_ms"], np.float64)
        print(f"{tag:9s} {app:8s} total {t.sum():7.2f} ms  {[round(float(x), 2) for x in t]}",
              flush=True)
    G.close()


g = config_graph_device("cfg4", weighted=True, degree_order=False)   # original ids
n, e = g["n"], g["e"]
off = g["csc_off"].long()
idx = g["csc_idx"]
w = g["csc_w"]
deg_out = torch.bincount(idx.long(), minlength=n)
# degree order: decreasing out-degree, ties by ascending id (the library's IPREGEL_LAYOUT_DEGREE)
old_of_new = torch.sort(-deg_out, stable=True).indices
new_of_old = torch.empty_like(old_of_new)
new_of_old[old_of_new] = torch.arange(n, device="cuda")
deg_in = off[1:] - off[:-1]
nd = deg_in[old_of_new]
noff = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
noff[1:] = torch.cumsum(nd, 0)
# edge positions of the new rows in the old CSC (row blocks moved, edge order inside kept)
start_old = off[:-1][old_of_new]
row_of_e = torch.repeat_interleave(torch.arange(n, device="cuda"), nd)
pos = start_old[row_of_e] + (torch.arange(e, device="cuda") - noff[:-1][row_of_e])
del row_of_e
nidx = new_of_old[idx.long()[pos]].to(torch.int32)
nw = w[pos]
del pos, g, idx, w
torch.cuda.empty_cache()
noff32 = noff.to(torch.int32)
times(noff32, nidx, nw, n, e, "unsorted")
# partially sorted: by a monotone class of the new source (its top bit and the `sub` bits below:
# fine for the hot low ids, coarse for the cold ones), stable (original order inside a class)
for sub in (3, 6):
    s64 = nidx.long()
    hb = torch.where(s64 > 0, torch.floor(torch.log2(s64.clamp(min=1).double())).long() + 1, 0)
    cls = torch.where(hb <= sub, s64, hb * (1 << sub) + ((s64 >> (hb - 1 - sub).clamp(min=0)) &
                                                         ((1 << sub) - 1)))
    del s64, hb
    key = torch.repeat_interleave(torch.arange(n, device="cuda"), nd) * 4096 + cls
    del cls
    order = torch.sort(key, stable=True).indices
    del key
    cidx, cw = nidx[order], nw[order]
    del order
    torch.cuda.empty_cache()
    times(noff32, cidx, cw, n, e, f"class+{sub}")
    del cidx, cw
    torch.cuda.empty_cache()
# the same rows with their sources ascending (the fixture's / library's layout)
key = torch.repeat_interleave(torch.arange(n, device="cuda"), nd) * n + nidx.long()
order = torch.argsort(key)
del key
sidx = nidx[order]
sw = nw[order]
del order, nidx, nw
torch.cuda.empty_cache()
times(noff32, sidx, sw, n, e, "sorted")
