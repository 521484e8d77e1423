"""DSMEM hot-cache lab on the cfg4 CSC (see tools/dsmem_lab.cu).  Not product code."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from inputs.gpu import config_graph_device  # noqa: E402

so = os.path.join(ROOT, "tools", "libdsmem_lab.so")
src = os.path.join(ROOT, "tools", "dsmem_lab.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, src])
lib = ctypes.CDLL(so)
lib.dsmem_lab.restype = ctypes.c_float
lib.dsmem_lab.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                          ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                          ctypes.c_int]
g = config_graph_device("cfg4", weighted=False, degree_order=True)
n, e = g["n"], g["e"]
idx = g["csc_idx"]
vals = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty(148 * 8 * 1024, dtype=torch.float64, device="cuda")
model = 12 * e + 16 * n
for mode, per_cta, cluster, ctas, threads in (
        (0, 0, 1, 148 * 8, 256), (0, 0, 8, 144 * 2, 1024), (0, 0, 8, 144, 1024),
        (1, 8192, 8, 144, 1024), (1, 12288, 8, 144, 1024), (1, 8192, 16, 144, 1024),
        (1, 12288, 16, 144, 1024), (1, 4096, 16, 144, 1024), (1, 8192, 8, 288, 512)):
    ms = lib.dsmem_lab(mode, idx.data_ptr(), e, vals.data_ptr(), per_cta, cluster, ctas, threads,
                       out.data_ptr(), 3)
    print(f"mode {mode} hot/cta {per_cta:6d} cluster {cluster:2d} grid {ctas}x{threads}: "
          f"{ms:7.3f} ms  {model / ms / 1e6:6.0f} GB/s model  hot set {per_cta * cluster}", flush=True)
