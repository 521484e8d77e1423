"""Gather-stream lab on the cfg4 CSC (see tools/gather_lab.cu).  Not product code.

    python tools/gather_lab.py [--config cfg4] [--no-degree-order]
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from inputs.gpu import config_graph_device  # noqa: E402

so = os.path.join(ROOT, "tools", "libgather_lab.so")
src = os.path.join(ROOT, "tools", "gather_lab.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, src])
lib = ctypes.CDLL(so)
lib.gather_lab.restype = ctypes.c_float
lib.gather_lab.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
lib.count_below.restype = ctypes.c_double
lib.count_below.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--no-degree-order", action="store_true")
a = ap.parse_args()
g = config_graph_device(a.config, weighted=False, degree_order=not a.no_degree_order)
n, e = g["n"], g["e"]
idx = g["csc_idx"]
vals = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty(148 * 64 * 256, dtype=torch.float64, device="cuda")
model = 12 * e + 16 * n


def show(tag, ms):
    print(f"{tag:48s} {ms:7.3f} ms  {e / ms / 1e6:6.1f} G gathers/s  "
          f"{model / ms / 1e6:6.0f} GB/s model", flush=True)


for H in (1024, 4096, 8192, 16384, 24576, 65536, 1 << 20):
    print(f"fraction of edges with source < {H}: {lib.count_below(idx.data_ptr(), e, H):.3f}")
for blocks, threads in ((148 * 8, 256), (148 * 16, 256), (148 * 4, 512)):
    show(f"v0 baseline {blocks}x{threads}",
         lib.gather_lab(0, idx.data_ptr(), e, vals.data_ptr(), 0, out.data_ptr(), blocks, threads, 5))
for H in (2048, 8192, 16384):
    show(f"v2 L1 evict-last below {H}",
         lib.gather_lab(2, idx.data_ptr(), e, vals.data_ptr(), H, out.data_ptr(), 148 * 8, 256, 5))
for H, blocks, threads in ((4096, 148 * 4, 512), (8192, 148 * 2, 1024), (8192, 148 * 3, 512),
                           (12288, 148 * 2, 1024), (16384, 148, 1024), (16384, 148 * 2, 512),
                           (24576, 148, 1024)):
    show(f"v1 smem hot {H} ({H * 8 // 1024} KB) {blocks}x{threads}",
         lib.gather_lab(1, idx.data_ptr(), e, vals.data_ptr(), H, out.data_ptr(), blocks, threads, 5))
