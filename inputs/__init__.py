"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module generates inputs ONLY: R-MAT edge lists (CPU twin
``rmat_cpu.c``, GPU twin ``rmat_gpu.cu``) and the five BASELINE.json
configurations.  It holds none of the method's arithmetic: no superstep, no
combiner, no vertex program.  The GPU twin additionally builds the CSR/CSC
arrays that ``ipregel_graph_create`` takes (a fixture for the device path;
the oracle builds its own adjacency from the same COO).

The R-MAT definition is in the header of ``rmat_cpu.c``.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_CPU_LIB = os.path.join(_HERE, "librmat_cpu.so")
_cpu = None

A, B, C = 0.57, 0.19, 0.19


def thresholds(a: float = A, b: float = B, c: float = C):
    """Integer quadrant thresholds floor(p * 2^32) for the cumulative a, a+b, a+b+c."""
    two32 = 4294967296.0
    return (int(np.floor(a * two32)), int(np.floor((a + b) * two32)),
            int(np.floor((a + b + c) * two32)))


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration (the graph, not the timing)."""
    name: str
    app: str            # "pagerank" | "cc" | "sssp" | "all"
    scale: int
    edgefactor: int
    seed: int
    weighted: bool
    iterations: int = 10

    @property
    def n(self) -> int:
        return 1 << self.scale

    @property
    def slots(self) -> int:
        return self.edgefactor << self.scale


# BASELINE.json configs[0..4]
CONFIGS = {
    "cfg0": Config("cfg0", "pagerank", 14, 16, 1, False),
    "cfg1": Config("cfg1", "cc", 20, 16, 2, False),
    "cfg2": Config("cfg2", "sssp", 22, 16, 3, True),
    "cfg3": Config("cfg3", "pagerank", 22, 28, 4, False),
    "cfg4": Config("cfg4", "all", 26, 28, 5, True),
}


def build_cpu(force: bool = False) -> str:
    src = os.path.join(_HERE, "rmat_cpu.c")
    if force or not os.path.exists(_CPU_LIB) or os.path.getmtime(_CPU_LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-std=c99", "-pthread", "-fPIC", "-shared",
                               "-o", _CPU_LIB, src])
    return _CPU_LIB


def _load_cpu():
    global _cpu
    if _cpu is None:
        build_cpu()
        lib = ctypes.CDLL(_CPU_LIB)
        p = ctypes.c_void_p
        lib.rmat_generate.restype = ctypes.c_int64
        lib.rmat_generate.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                      ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                      p, p, p, ctypes.c_int]
        lib.rmat_slot_edge.restype = None
        lib.rmat_slot_edge.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32,
                                       ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                       p, p, p]
        lib.rmat_splitmix64.restype = ctypes.c_uint64
        lib.rmat_splitmix64.argtypes = [ctypes.c_uint64]
        _cpu = lib
    return _cpu


def splitmix64(x: int) -> int:
    return int(_load_cpu().rmat_splitmix64(x))


def rmat_coo(scale: int, edgefactor: int, seed: int, weighted: bool = False,
             threads: int | None = None, slots: int | None = None):
    """Directed R-MAT COO on the CPU: (src int32, dst int32, w uint32 | None).

    Self-loops removed, slot order and duplicates kept.  ``slots`` defaults to
    edgefactor * 2^scale.
    """
    lib = _load_cpu()
    m = (edgefactor << scale) if slots is None else int(slots)
    threads = threads or os.cpu_count() or 1
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    w = np.empty(m, np.uint32) if weighted else None
    ta, tab, tabc = thresholds()
    vp = ctypes.c_void_p
    kept = lib.rmat_generate(seed, scale, m, ta, tab, tabc,
                             src.ctypes.data_as(vp), dst.ctypes.data_as(vp),
                             None if w is None else w.ctypes.data_as(vp), threads)
    if kept < 0:
        raise ValueError("rmat_generate: bad arguments")
    src = src[:kept]
    dst = dst[:kept]
    if w is not None:
        w = w[:kept]
    return src, dst, w


def rmat_slot(scale: int, seed: int, i: int):
    """(src, dst, w) of slot i before self-loop removal (for tests)."""
    lib = _load_cpu()
    s, d, w = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
    ta, tab, tabc = thresholds()
    lib.rmat_slot_edge(seed, scale, ta, tab, tabc, i, ctypes.byref(s), ctypes.byref(d),
                       ctypes.byref(w))
    return s.value, d.value, w.value


def config_coo(cfg: Config | str, threads: int | None = None):
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return rmat_coo(cfg.scale, cfg.edgefactor, cfg.seed, cfg.weighted, threads)


def array_digest(*arrays) -> str:
    """sha256 over the raw bytes of the given arrays (None skipped)."""
    h = hashlib.sha256()
    for a in arrays:
        if a is None:
            continue
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(memoryview(a).cast("B"))
    return h.hexdigest()
