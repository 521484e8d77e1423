"""GPU twin of the R-MAT generator and the CSR/CSC fixture (inputs/rmat_gpu.cu).

Input generation only (see inputs/__init__.py).  Returns torch CUDA tensors.
"""
from __future__ import annotations

import ctypes
import os

from . import CONFIGS, Config, thresholds

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "librmat_gpu.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run `make`")
        lib = ctypes.CDLL(_LIB)
        P, U64, I, U32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32
        lib.rmat_gpu_count.restype = ctypes.c_int64
        lib.rmat_gpu_count.argtypes = [U64, I, U64, U32, U32, U32, P, P, P]
        lib.rmat_gpu_coo.restype = ctypes.c_int64
        lib.rmat_gpu_coo.argtypes = [U64, I, U64, U32, U32, U32, P, P, P, P]
        lib.rmat_gpu_adjacency.restype = ctypes.c_int64
        lib.rmat_gpu_adjacency.argtypes = [U64, I, U64, U32, U32, U32, I, P, P, P, P, P]
        lib.rmat_gpu_degree_order.restype = ctypes.c_int64
        lib.rmat_gpu_degree_order.argtypes = [U64, I, U64, U32, U32, U32, I, I, P, P, P]
        _lib = lib
    return _lib


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def rmat_coo_device(scale: int, edgefactor: int, seed: int, weighted: bool = False):
    import torch
    lib = _load()
    m = edgefactor << scale
    ta, tab, tabc = thresholds()
    src = torch.empty(m, dtype=torch.int32, device="cuda")
    dst = torch.empty(m, dtype=torch.int32, device="cuda")
    w = torch.empty(m, dtype=torch.int32, device="cuda") if weighted else None
    kept = lib.rmat_gpu_coo(seed, scale, m, ta, tab, tabc, src.data_ptr(), dst.data_ptr(),
                            None if w is None else w.data_ptr(), _stream())
    if kept < 0:
        raise RuntimeError("rmat_gpu_coo failed")
    return src[:kept], dst[:kept], (None if w is None else w[:kept])


def degree_order_device(scale: int, edgefactor: int, seed: int, use_out=True, use_in=False):
    """(old_of_new, new_of_old) int32 tensors: vertices sorted by descending degree."""
    import torch
    lib = _load()
    n = 1 << scale
    ta, tab, tabc = thresholds()
    old_of_new = torch.empty(n, dtype=torch.int32, device="cuda")
    new_of_old = torch.empty(n, dtype=torch.int32, device="cuda")
    r = lib.rmat_gpu_degree_order(seed, scale, edgefactor << scale, ta, tab, tabc, int(use_out),
                                  int(use_in), old_of_new.data_ptr(), new_of_old.data_ptr(),
                                  _stream())
    if r < 0:
        raise RuntimeError("rmat_gpu_degree_order failed")
    return old_of_new, new_of_old


def rmat_adjacency_device(scale: int, edgefactor: int, seed: int, by_dst: bool,
                          weighted: bool = False, remap=None):
    """(offsets int32 [N+1], indices int32 [E], weights int32-as-uint32 [E] | None).

    remap (int32 [N] device tensor, optional): relabel vertex v as remap[v]."""
    import torch
    lib = _load()
    n = 1 << scale
    m = edgefactor << scale
    ta, tab, tabc = thresholds()
    off = torch.zeros(n + 1, dtype=torch.int32, device="cuda")
    e = lib.rmat_gpu_count(seed, scale, m, ta, tab, tabc, None, None, _stream())
    if e < 0:
        raise RuntimeError("rmat_gpu_count failed")
    idx = torch.empty(max(e, 1), dtype=torch.int32, device="cuda")
    w = torch.empty(max(e, 1), dtype=torch.int32, device="cuda") if weighted else None
    e2 = lib.rmat_gpu_adjacency(seed, scale, m, ta, tab, tabc, 1 if by_dst else 0,
                                off.data_ptr(), idx.data_ptr(),
                                None if w is None else w.data_ptr(),
                                None if remap is None else remap.data_ptr(), _stream())
    if e2 != e:
        raise RuntimeError("rmat_gpu_adjacency failed")
    return off, idx[:e], (None if w is None else w[:e])


def config_graph_device(cfg: Config | str, weighted: bool | None = None, degree_order=False):
    """CSC + CSR of a BASELINE.json config on the current device.

    degree_order=True lays the graph out with vertices sorted by descending out-degree
    ("vertex_ids" maps internal id -> original id); the graph is the same up to isomorphism.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    wt = cfg.weighted if weighted is None else weighted
    old_of_new = new_of_old = None
    if degree_order:
        old_of_new, new_of_old = degree_order_device(cfg.scale, cfg.edgefactor, cfg.seed)
    csc_off, csc_idx, csc_w = rmat_adjacency_device(cfg.scale, cfg.edgefactor, cfg.seed, True, wt,
                                                    new_of_old)
    csr_off, csr_idx, csr_w = rmat_adjacency_device(cfg.scale, cfg.edgefactor, cfg.seed, False, wt,
                                                    new_of_old)
    return {"n": cfg.n, "e": int(csc_idx.shape[0]), "csc_off": csc_off, "csc_idx": csc_idx,
            "csc_w": csc_w, "csr_off": csr_off, "csr_idx": csr_idx, "csr_w": csr_w,
            "vertex_ids": old_of_new}
