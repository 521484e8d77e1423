"""Compressed-index lab on the cfg4 degree-ordered CSC (tools/compress_lab.cu).  Not product code.

    python tools/compress_lab.py [--config cfg4]
Prints the encoded sizes (bytes per edge, bit-width histogram) and the raw gather stream's time
with int32, frame-of-reference and delta-coded indices, with a checksum of the decoded ids.
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

so = os.path.join(ROOT, "tools", "libcompress_lab.so")
src = os.path.join(ROOT, "tools", "compress_lab.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-o", so, src])
lib = ctypes.CDLL(so)
P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
lib.enc_width.argtypes = [P, P, I64, I, P, P]
lib.enc_pack.argtypes = [P, I64, P, P, P, P]
lib.run_lab.restype = ctypes.c_float
lib.run_lab.argtypes = [I, P, P, P, I64, P, I64, P, P, P, I, I]
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--ctas", default="3,4")
a = ap.parse_args()
cfg = CONFIGS[a.config]
old_of_new, new_of_old = degree_order_device(cfg.scale, cfg.edgefactor, cfg.seed)
off, idx, _ = rmat_adjacency_device(cfg.scale, cfg.edgefactor, cfg.seed, True, False, new_of_old)
del old_of_new, new_of_old
n, E = cfg.n, int(idx.shape[0])
rs = torch.zeros(E, dtype=torch.uint8, device="cuda")
deg = off[1:] - off[:-1]
rs[off[:-1][deg > 0].long()] = 1
del deg
nch = (E + 127) // 128
print(f"{a.config}: N={n} E={E} chunks={nch}", flush=True)
vals = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty(148 * 8 * 256, dtype=torch.float64, device="cuda")
cks = torch.zeros(1, dtype=torch.int64, device="cuda")
ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
want = int(idx.to(torch.int64).sum().item())
encs = {}
for mode in (1, 2):
    hb = torch.empty(nch, dtype=torch.int32, device="cuda")
    words = torch.empty(nch, dtype=torch.int64, device="cuda")
    lib.enc_width(idx.data_ptr(), rs.data_ptr(), E, mode, hb.data_ptr(), words.data_ptr())
    woff = torch.cumsum(words, 0) - words
    total = int(words.sum().item())
    hdr = torch.empty(nch, 2, dtype=torch.int32, device="cuda")
    pay = torch.zeros(total + 2, dtype=torch.int32, device="cuda")
    lib.enc_pack(idx.data_ptr(), E, hb.data_ptr(), woff.data_ptr(), hdr.data_ptr(), pay.data_ptr())
    torch.cuda.synchronize()
    b = (hb & 31).long()
    hist = torch.bincount(b, minlength=33).cpu().tolist()
    kind = int((hb >> 5).sum().item())
    bpe = (4 * total + 8 * nch) / E
    print(f"mode {mode}: payload {4 * total / 1e9:.3f} GB + headers {8 * nch / 1e9:.3f} GB = "
          f"{bpe:.3f} B/edge (raw 4); delta chunks {kind} of {nch}", flush=True)
    print("  b histogram (chunks): " + " ".join(f"{i}:{c}" for i, c in enumerate(hist) if c),
          flush=True)
    encs[mode] = (hdr, pay)
    del hb, words, woff
for ctas in [int(x) for x in a.ctas.split(",")]:
    for v in (0, 1, 2):
        hdr, pay = encs.get(v, encs[1])
        ms = lib.run_lab(v, idx.data_ptr(), hdr.data_ptr(), pay.data_ptr(), E, vals.data_ptr(), n,
                         out.data_ptr(), cks.data_ptr(), ctr.data_ptr(), ctas, 5)
        ok = int(cks.item()) == want
        print(f"v{v} {ctas} CTAs/SM: {ms:.3f} ms  checksum {'ok' if ok else 'BAD'}", flush=True)
