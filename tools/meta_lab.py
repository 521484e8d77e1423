"""Metadata-driven row logic lab on the cfg4 degree-ordered CSC (tools/meta_lab.cu).  Not product
code.   python tools/meta_lab.py [--config cfg4] [--ctas 3] [--product]
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from inputs import CONFIGS  # noqa: E402
from inputs.gpu import degree_order_device, rmat_adjacency_device  # noqa: E402

so = os.path.join(ROOT, "tools", "libmeta_lab.so")
src = os.path.join(ROOT, "tools", "meta_lab.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, src])
lib = ctypes.CDLL(so)
P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
lib.meta_build.argtypes = [P, I64, P, P]
lib.run_meta_lab.restype = ctypes.c_float
lib.run_meta_lab.argtypes = [I, P, P, P, I64, P, I64, P, P, P, P, I, I, I]
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--ctas", default="3")
ap.add_argument("--product", action="store_true")
a = ap.parse_args()
cfg = CONFIGS[a.config]
old_of_new, new_of_old = degree_order_device(cfg.scale, cfg.edgefactor, cfg.seed)
off, idx, _ = rmat_adjacency_device(cfg.scale, cfg.edgefactor, cfg.seed, True, False, new_of_old)
del old_of_new, new_of_old
n, E = cfg.n, int(idx.shape[0])
deg = (off[1:] - off[:-1])
nz = deg > 0
nrows = int(nz.sum().item())
rs = torch.zeros(E + 1, dtype=torch.uint8, device="cuda")
rs[off[:-1][nz].long()] = 1
rs[E] = 1
nch = (E + 127) // 128
mask = torch.empty(nch, 4, dtype=torch.int32, device="cuda")
cnt = torch.empty(nch, dtype=torch.int32, device="cuda")
lib.meta_build(rs.data_ptr(), E, mask.data_ptr(), cnt.data_ptr())
ordc = (torch.cumsum(cnt.long(), 0) - cnt.long()).to(torch.int32)
assert int(cnt.long().sum().item()) == nrows
print(f"{a.config}: N={n} E={E} rows with in-edges {nrows}; chunks {nch}: "
      f"no end {int((cnt == 0).sum())}, one end {int((cnt == 1).sum())}, "
      f"more {int((cnt > 1).sum())}", flush=True)
lib.meta_bad.argtypes = [I]
lib.meta_bad(nrows)
for H in (4096, 8192, 16384, 25088, 65536):
    print(f"edges with source < {H}: {float((idx < H).sum()) / E:.4f}", flush=True)
vals = torch.rand(n, dtype=torch.float64, device="cuda")
sumc = torch.zeros(nrows, dtype=torch.float64, device="cuda")
carry = torch.zeros((nch + 31) // 32, dtype=torch.float64, device="cuda")
out = torch.empty(148 * 8 * 256, dtype=torch.float64, device="cuda")
ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
endf = rs[1:].bool()
idxf = torch.where(endf, idx | (-2 ** 31), idx)
del endf
starts = off[:-1][nz].long()
ends = off[1:][nz].long()
inside = (starts // 8192) == ((ends - 1) // 8192)
del starts, ends
ve = vals[idx.long()]
rid = torch.repeat_interleave(torch.arange(nrows, device="cuda"), deg[nz].long())
ref = torch.zeros(nrows, dtype=torch.float64, device="cuda").index_add_(0, rid, ve)
del ve, rid


def check(tag):
    rel = ((sumc - ref).abs() / ref.abs().clamp_min(1e-300))[inside]
    print(f"  {tag}: rows inside one block {int(inside.sum())}: max rel err {float(rel.max()):.3e}",
          flush=True)
    sumc.zero_()


for ctas in [int(x) for x in a.ctas.split(",")]:
    for order in (0, 1):
        for v in (0, 9, 16, 13, 14, 15):
            ms = lib.run_meta_lab(v, (idxf if v >= 8 else idx).data_ptr(), mask.data_ptr(), ordc.data_ptr(), E,
                                  vals.data_ptr(), n, sumc.data_ptr(), carry.data_ptr(),
                                  out.data_ptr(), ctr.data_ptr(), ctas, order, 5)
            print(f"v{v} {ctas} CTAs/SM order {order}: {ms:.3f} ms  bad {lib.meta_bad(nrows)}",
                  flush=True)
            if v in (9, 13, 15):
                check(f"v{v} order {order}")
# check rows held inside one 8192-edge block
check("last")
if a.product:
    import paper_2010_08781_b200 as ipr
    del sumc, ref, mask, cnt, ordc, rs
    o2n, n2o = degree_order_device(cfg.scale, cfg.edgefactor, cfg.seed)
    roff, ridx, _ = rmat_adjacency_device(cfg.scale, cfg.edgefactor, cfg.seed, False, False, n2o)
    del o2n, n2o
    G = ipr.Graph(ipr.full_partition(n, E, off, idx, roff, ridx, degree_ordered=True))
    for _ in range(2):
        G.run("pagerank", mode="pull", iterations=10)
        s = G.stats()
        print("product PR supersteps " + str([round(float(x), 3) for x in s["time_ms"]]),
              flush=True)
