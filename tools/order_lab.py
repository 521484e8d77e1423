"""Vertex-order lab: how many L1 -> L2 gather requests would the PageRank pull issue on the cfg4
CSC under the library's degree order, and under degree order with ties broken by each vertex's
first destination (sources gathered by the same row get neighbouring ids, so that row's gathers
share 128-byte lines)?  Model: per 32 consecutive CSC edges (one warp gather instruction), the
distinct 128-byte lines (16 f64 sources) among sources >= 8192 (the hotter ones hit in L1).
Not product code.      python tools/order_lab.py [--config cfg4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs import CONFIGS  # noqa: E402
from inputs.gpu import rmat_coo_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
a = ap.parse_args()
cfg = CONFIGS[a.config]
src, dst, _ = rmat_coo_device(cfg.scale, cfg.edgefactor, cfg.seed)
n, E = cfg.n, int(src.numel())
print(f"{a.config}: N={n} E={E}", flush=True)
outdeg = torch.bincount(src.long(), minlength=n)
# edge share by source out-degree
dh = torch.bincount(outdeg, minlength=64)[:64].double()
share = dh * torch.arange(64, device="cuda", dtype=torch.float64) / E
print("edge share of sources with out-degree 1..8: " +
      " ".join(f"{d}:{float(share[d]):.4f}" for d in range(1, 9)), flush=True)


def stable_order(keys_major, keys_minor=None):
    """new id -> old id: sort by keys_major ascending, ties by keys_minor, then old id."""
    idx = torch.arange(n, device="cuda")
    if keys_minor is not None:
        o = torch.sort(keys_minor, stable=True).indices
        idx = idx[o]
        km = keys_major[o]
    else:
        km = keys_major
    o2 = torch.sort(km, stable=True).indices
    return idx[o2]


def requests(old_of_new, tag, shift=4, hot=8192):
    new_of_old = torch.empty(n, dtype=torch.int64, device="cuda")
    new_of_old[old_of_new] = torch.arange(n, device="cuda")
    ns = new_of_old[src.long()]
    nd = new_of_old[dst.long()]
    key = (nd << 26) | ns
    del nd
    key = torch.sort(key).values
    s_sorted = key & ((1 << 26) - 1)
    del key
    line = s_sorted >> shift
    cold = s_sorted >= hot
    # change points inside each 32-edge group among cold sources
    pos = torch.arange(E, device="cuda")
    first_in_group = (pos % 32) == 0
    prev_line = torch.roll(line, 1)
    # a cold edge starts a new request if it is the first cold edge of its group or its line
    # differs from the previous edge's (rows sorted ascending: lines are monotone inside a row)
    newreq = cold & (first_in_group | (line != prev_line) | ~torch.roll(cold, 1))
    r = int(newreq.sum().item())
    print(f"{tag}: modelled gather requests {r / 1e9:.3f}e9 ({r / E:.3f} per edge), "
          f"cold edges {float(cold.double().mean()):.3f}", flush=True)
    return r


deg_key = -outdeg
o0 = stable_order(deg_key)
r0 = requests(o0, "degree order (ties by original id)")
requests(o0, "degree order, u32 values (32 per line, 16384 in L1)", shift=5, hot=16384)
# first destination of every source under order 0
new0 = torch.empty(n, dtype=torch.int64, device="cuda")
new0[o0] = torch.arange(n, device="cuda")
fd = torch.full((n,), n, dtype=torch.int64, device="cuda")
fd.scatter_reduce_(0, src.long(), new0[dst.long()], reduce="amin")
o1 = stable_order(deg_key, fd)
r1 = requests(o1, "degree order, ties by first destination")
print(f"ratio {r1 / r0:.3f}", flush=True)
