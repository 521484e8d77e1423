"""Raw gather ceiling on the cfg4 CSC (see tools/gather_ceiling.cu).

    python tools/gather_ceiling.py [--degree-order]
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

so = os.path.join(ROOT, "tools", "libgather_ceiling.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so,
                           os.path.join(ROOT, "tools", "gather_ceiling.cu")])
lib = ctypes.CDLL(so)
lib.gather_ceiling.restype = ctypes.c_float
lib.gather_ceiling.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                               ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
ap = argparse.ArgumentParser()
ap.add_argument("--degree-order", action="store_true")
ap.add_argument("--config", default="cfg4")
a = ap.parse_args()
g = config_graph_device(a.config, weighted=False, degree_order=a.degree_order)
n, e = g["n"], g["e"]
idx = g["csc_idx"]
for f64, name in ((1, "f64"), (0, "u32")):
    vals = torch.rand(n, dtype=torch.float64, device="cuda") if f64 else \
        torch.randint(0, 1 << 30, (n,), dtype=torch.int32, device="cuda")
    for blocks in (148 * 2, 148 * 4, 148 * 6, 148 * 8, 148 * 32):
        out = torch.empty(blocks * 256, dtype=vals.dtype, device="cuda")
        ms = lib.gather_ceiling(idx.data_ptr(), e, vals.data_ptr(), f64, out.data_ptr(), blocks, 5)
        print(f"{name} blocks={blocks}: {ms:.3f} ms  {e / ms / 1e6:.1f} G gathers/s  "
              f"model PR bytes/ms {(12 * e + 16 * n) / ms / 1e6:.0f} GB/s", flush=True)
# uniform random indices of the same length, for comparison
ridx = torch.randint(0, n, (e,), dtype=torch.int32, device="cuda")
vals = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty(148 * 16 * 256, dtype=vals.dtype, device="cuda")
ms = lib.gather_ceiling(ridx.data_ptr(), e, vals.data_ptr(), 1, out.data_ptr(), 148 * 16, 5)
print(f"f64 uniform-random indices: {ms:.3f} ms  {e / ms / 1e6:.1f} G gathers/s")
