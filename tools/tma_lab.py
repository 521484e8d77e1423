"""Memory-pipeline lab of the range kernel on the cold part of the cfg4 CSC (tools/tma_lab.cu).
Not product code.   python tools/tma_lab.py [--H 16384]"""
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

so = os.path.join(ROOT, "tools", "libtma_lab.so")
src = os.path.join(ROOT, "tools", "tma_lab.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, src])
lib = ctypes.CDLL(so)
lib.tma_lab.restype = ctypes.c_float
P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
lib.tma_lab.argtypes = [I, P, I64, P, P, P, I, I]
ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, default=16384)
a = ap.parse_args()
cfg = CONFIGS["cfg4"]
old_of_new, new_of_old = degree_order_device(cfg.scale, cfg.edgefactor, cfg.seed)
off, idx, _ = rmat_adjacency_device(cfg.scale, cfg.edgefactor, cfg.seed, True, False, new_of_old)
del old_of_new, new_of_old, off
n = cfg.n
cold = torch.masked_select(idx, idx >= a.H) if a.H > 0 else idx
del idx
torch.cuda.synchronize()
e = cold.numel()
vals = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.zeros(148 * 16 * 256, dtype=torch.float64, device="cuda")
ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
print(f"cold edges {e}", flush=True)
names = {0: "regs pipeline, warp blocks of 64 chunks", 1: "blocks of 16 chunks",
         2: "blocks of 4 chunks", 3: "blocks of 2 chunks", 4: "blocks of 256 chunks",
         5: "ring: idx 2 ahead", 6: "ring: idx 3 ahead", 7: "ring: idx 4 ahead",
         8: "ring: idx 6 ahead"}
for v in (0, 5, 6, 7, 8):
    for c in (2, 3, 4):
        ms = lib.tma_lab(v, cold.data_ptr(), e, vals.data_ptr(), out.data_ptr(), ctr.data_ptr(), c, 5)
        print(f"v{v} {names[v]:36s} {c} CTAs/SM ({8 * c} warps): {ms:.3f} ms", flush=True)
