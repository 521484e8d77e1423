"""Row-logic overhead of the pull kernel: PageRank pull on synthetic CSCs with the SAME edge
count and source distribution but different row lengths, next to the raw gather ceiling of the
same index stream (tools/gather_ceiling.cu).  Sources are uniform in [0, 2^20) (L2-resident
outbox) so the gathers themselves are cheap and the row logic shows.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2010_08781_b200 as ipr  # noqa: E402

so = os.path.join(ROOT, "tools", "libgather_ceiling.so")
lib = ctypes.CDLL(so)
lib.gather_ceiling.restype = ctypes.c_float
lib.gather_ceiling.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                               ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
E = 1 << 29
S = 1 << 20
g = torch.Generator(device="cuda").manual_seed(1)
E0 = E
for deg in (2, 8, 28, 128, 1024, 16384):
    rows = E0 // deg
    E = rows * deg
    n = max(rows, S)
    idx = torch.randint(0, S, (E,), generator=g, device="cuda", dtype=torch.int32)
    idx, _ = torch.sort(idx.view(rows, deg), dim=1)
    idx = idx.reshape(-1).contiguous()
    off = (torch.arange(n + 1, device="cuda", dtype=torch.int64) * deg).clamp(max=E).to(torch.int32)
    # CSR: every vertex out-degree 1 (contrib = rank), never read beyond offsets
    csr_off = torch.arange(n + 1, device="cuda", dtype=torch.int32)
    csr_idx = torch.zeros(n, device="cuda", dtype=torch.int32)
    G = ipr.Graph(ipr.full_partition(n, E, off, idx, csr_off, csr_idx))
    ts = []
    for _ in range(2):
        G.run("pagerank", mode="pull", iterations=3)
        ts += list(G.stats()["kernel_ms"][1:])
    vals = torch.rand(n, dtype=torch.float64, device="cuda")
    out = torch.empty(148 * 16 * 256, dtype=torch.float64, device="cuda")
    ceil = lib.gather_ceiling(idx.data_ptr(), E, vals.data_ptr(), 1, out.data_ptr(), 148 * 16, 3)
    print(f"in-degree {deg:6d}: pull {min(ts):.3f} ms   raw gather {ceil:.3f} ms   "
          f"ratio {min(ts) / ceil:.2f}", flush=True)
    G.close()
    del idx, off, csr_off, csr_idx
    torch.cuda.empty_cache()
