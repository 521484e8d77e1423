"""Per-lane merge-path lab on the cold / hot parts of the cfg4 CSC (tools/mpt_lab.cu).  Not
product code.   python tools/mpt_lab.py [--H 16384]"""
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

so = os.path.join(ROOT, "tools", "libmpt_lab.so")
src = os.path.join(ROOT, "tools", "mpt_lab.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, src])
lib = ctypes.CDLL(so)
lib.mpt_lab.restype = ctypes.c_float
P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
lib.mpt_lab.argtypes = [I, P, I, I64, P, P, I, P, P, I, I, I]
ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, default=16384)
a = ap.parse_args()
cfg = CONFIGS["cfg4"]
old_of_new, new_of_old = degree_order_device(cfg.scale, cfg.edgefactor, cfg.seed)
off, idx, _ = rmat_adjacency_device(cfg.scale, cfg.edgefactor, cfg.seed, True, False, new_of_old)
del old_of_new, new_of_old
n, e = cfg.n, int(idx.shape[0])
H = a.H
flag = (idx < H).to(torch.int32)
pos = torch.zeros(e + 1, dtype=torch.int64, device="cuda")
pos[1:] = torch.cumsum(flag, 0)
hot_off = pos[off.long()].to(torch.int32)
cold_off = (off.long() - pos[off.long()]).to(torch.int32)
m = flag.bool()
hot = torch.masked_select(idx, m)
cold = torch.masked_select(idx, ~m)
del pos, flag, m
torch.cuda.synchronize()
vals = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.zeros(n, dtype=torch.float64, device="cuda")
ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
print(f"N={n} E={e} hot={hot.numel()} cold={cold.numel()}", flush=True)


def t(v, o, ix, ee, blocks, threads):
    return lib.mpt_lab(v, o.data_ptr(), n, ee, ix.data_ptr(), vals.data_ptr(), H, out.data_ptr(),
                       ctr.data_ptr(), blocks, threads, 5)


for v, name in ((0, "range 4096 batch 4"), (1, "range 4096 batch 8"), (2, "range 8192 batch 8"),
                (3, "range 2048 batch 4")):
    for blocks, threads in ((148 * 8, 256), (148 * 4, 256), (148 * 2, 1024)):
        print(f"cold mpt {name} {blocks}x{threads}: {t(v, cold_off, cold, cold.numel(), blocks, threads):.3f} ms",
              flush=True)
for v, name in ((10, "range 4096 batch 4"), (11, "range 4096 batch 8"), (12, "range 2048 batch 4")):
    for blocks, threads in ((148, 1024), (148, 512)):
        print(f"hot mpt staged {name} {blocks}x{threads}: {t(v, hot_off, hot, hot.numel(), blocks, threads):.3f} ms",
              flush=True)
