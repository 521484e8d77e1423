"""TMA gather4 lab on the cfg4 degree-ordered CSC (tools/tma_gather_lab.cu).  Not product code.
    python tools/tma_gather_lab.py [--config cfg4]"""
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

so = os.path.join(ROOT, "tools", "libtma_gather_lab.so")
src = os.path.join(ROOT, "tools", "tma_gather_lab.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, src])
lib = ctypes.CDLL(so)
P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
lib.run_tma_lab.restype = ctypes.c_float
lib.run_tma_lab.argtypes = [I, P, I64, P, I64, P, P, I, I, I]
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
a = ap.parse_args()
cfg = CONFIGS[a.config]
o2n, n2o = degree_order_device(cfg.scale, cfg.edgefactor, cfg.seed)
off, idx, _ = rmat_adjacency_device(cfg.scale, cfg.edgefactor, cfg.seed, True, False, n2o)
del o2n, n2o, off
n, E = cfg.n, int(idx.shape[0])
Ep = (E + 127) // 128 * 128
pad = Ep - E
idxp = torch.zeros(Ep, dtype=torch.int32, device="cuda")
idxp[:E] = idx
del idx
vals = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.zeros(148 * 3 * 256, dtype=torch.float64, device="cuda")
ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
print(f"{a.config}: N={n} E={E} (padded {Ep})", flush=True)
ms = lib.run_tma_lab(0, idxp.data_ptr(), E, vals.data_ptr(), n, out.data_ptr(), ctr.data_ptr(), 1, 0, 5)
ref = float(out.sum())
print(f"raw loads: {ms:.3f} ms  sum {ref:.10e}", flush=True)
for v, box, l2 in ((1, 1, 0), (2, 1, 0), (3, 1, 0), (2, 1, 2)):
    out.zero_()
    ms = lib.run_tma_lab(v, idxp.data_ptr(), Ep, vals.data_ptr(), n, out.data_ptr(), ctr.data_ptr(), box, l2, 5)
    s = float(out.sum()) - pad * float(vals[0])
    print(f"TMA gather4 stages {[0, 1, 2, 3][v]} box rows {box} l2promo {l2}: {ms:.3f} ms  "
          f"sum rel diff {abs(s - ref) / ref:.2e}", flush=True)
    if ms < 0:
        break
