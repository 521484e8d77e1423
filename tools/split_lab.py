"""Hot/cold split ceiling of the PageRank gather on the cfg4 CSC (see tools/split_lab.cu).
Not product code.

    python tools/split_lab.py [--config cfg4]
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

so = os.path.join(ROOT, "tools", "libsplit_lab.so")
src = os.path.join(ROOT, "tools", "split_lab.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, src])
lib = ctypes.CDLL(so)
lib.split_lab.restype = ctypes.c_float
lib.split_lab.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                          ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
lib.lines_per_edge.restype = ctypes.c_double
lib.lines_per_edge.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
a = ap.parse_args()
cfg = CONFIGS[a.config]
old_of_new, new_of_old = degree_order_device(cfg.scale, cfg.edgefactor, cfg.seed)
off, idx, _ = rmat_adjacency_device(cfg.scale, cfg.edgefactor, cfg.seed, True, False, new_of_old)
del old_of_new, new_of_old, off
n, e = cfg.n, int(idx.shape[0])
vals = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty(148 * 64 * 1024, dtype=torch.float64, device="cuda")
print(f"{a.config}: N={n} E={e}", flush=True)


def t(variant, ix, ee, H, blocks, threads):
    return lib.split_lab(variant, ix.data_ptr(), ee, vals.data_ptr(), H, out.data_ptr(), blocks,
                         threads, 5)


full = t(0, idx, e, 0, 148 * 12, 256)
print(f"raw full: {full:.3f} ms; lines/edge {lib.lines_per_edge(idx.data_ptr(), e, 4):.4f} "
      f"sectors/edge {lib.lines_per_edge(idx.data_ptr(), e, 2):.4f}", flush=True)
for blocks, threads in ((148 * 8, 256), (148 * 16, 256), (148 * 6, 256)):
    print(f"  raw full {blocks}x{threads}: {t(0, idx, e, 0, blocks, threads):.3f} ms", flush=True)
for H in (8192, 16384, 24576, 27648):
    m = idx >= H
    cold = torch.masked_select(idx, m)
    hot = torch.masked_select(idx, ~m)
    del m
    ec, eh = int(cold.shape[0]), int(hot.shape[0])
    tc = t(0, cold, ec, 0, 148 * 12, 256)
    lc = lib.lines_per_edge(cold.data_ptr(), ec, 4)
    lh = lib.lines_per_edge(hot.data_ptr(), eh, 4)
    hot16 = hot.to(torch.int16)
    res = []
    for blocks, threads in ((148, 1024), (148, 512), (296, 512) if H <= 12288 else (148, 768)):
        res.append((blocks, threads, t(1, hot, eh, H, blocks, threads),
                    t(2, hot16, eh, H, blocks, threads)))
    print(f"H={H}: hot fraction {eh / e:.4f}; cold raw {tc:.3f} ms (lines/edge {lc:.4f}); "
          f"hot lines/edge {lh:.4f}", flush=True)
    for blocks, threads, ti, t16 in res:
        print(f"    hot smem {blocks}x{threads}: i32 idx {ti:.3f} ms, u16 idx {t16:.3f} ms; "
              f"cold+hot(u16) {tc + t16:.3f} ms vs full {full:.3f}", flush=True)
    del cold, hot, hot16
    torch.cuda.empty_cache()
