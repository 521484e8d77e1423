"""Oracle -- TEST INFRASTRUCTURE ONLY.

A plain single-threaded CPU Pregel interpreter of iPregel's three vertex
programs (Figs. 8-10), written in C (oracle/oracle.c, see its header
for the passage each step follows) and loaded here through ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2010_08781_b200``) never imports it and shares no code
with it; the only common input is the COO edge list from ``inputs``.

Parity status per function:
  run(APP_PAGERANK, tol>=0)  pinned: closed forms of the per-superstep change
                     (cycle, complete digraph, in-star), exact-rational deltas
                     and stopping superstep on random graphs.
  run(APP_PAGERANK)  pinned: worked examples W1-W3 (exact rationals), closed
                     forms (cycle, complete digraph, in-star, out-star), the
                     mass invariant, scipy sparse power iteration.
  run(APP_HASHMIN_CC) pinned: worked examples W5/W9, union-find, BFS balls
                     per superstep, scipy connected_components.
  run(APP_SSSP)      pinned: worked examples W6/W7, Dijkstra (heapq), hop-
                     bounded Bellman-Ford per superstep, BFS for w = 1.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

APP_PAGERANK = 0
APP_HASHMIN_CC = 1
APP_SSSP = 2
INF = 0xFFFFFFFF

OK = 0
INVALID = 1
NOMEM = 3
GUARD = 6

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2 -ffp-contract=off, one thread)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-D_POSIX_C_SOURCE=199309L", "-ffp-contract=off",
             "-fno-fast-math", "-fPIC", "-shared", "-o", _LIB, src])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        p = ctypes.c_void_p
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run.argtypes = [
            ctypes.c_int, ctypes.c_int64, ctypes.c_int64, p, p, p, ctypes.c_uint32,
            ctypes.c_uint32, ctypes.c_uint32, p, p, ctypes.c_uint32, p, p, p, p, p,
            ctypes.c_double, p]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def run(app: int, n: int, src, dst, w=None, k: int = 10, source: int = 0,
        max_supersteps: int = 1 << 30, cap: int = 4096, tol: float = -1.0) -> dict:
    """Run the interpreter; returns values, status and per-superstep counters.

    ``src``/``dst`` are the directed edges (int32), ``w`` optional uint32
    weights (SSSP only; None means w = 1, Fig. 10).  ``tol`` >= 0 runs
    PageRank to convergence (max per-vertex change <= tol, reading R27).  PageRank values are f64,
    CC labels and SSSP distances u32 (INF = 0xFFFFFFFF).
    """
    lib = _load()
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    if w is not None:
        w = np.ascontiguousarray(w, dtype=np.uint32)
    m = int(src.shape[0])
    assert dst.shape[0] == m and (w is None or w.shape[0] == m)
    vals = np.zeros(n, dtype=np.float64 if app == APP_PAGERANK else np.uint32)
    steps = ctypes.c_uint32(0)
    ran = np.zeros(cap, np.uint64)
    changed = np.zeros(cap, np.uint64)
    messages = np.zeros(cap, np.uint64)
    secs = np.zeros(cap, np.float64)
    build_s = ctypes.c_double(0.0)
    delta = np.zeros(cap, np.float64)
    rc = lib.oracle_run(app, n, m, _ptr(src), _ptr(dst), _ptr(w), k, source,
                        max_supersteps, _ptr(vals), ctypes.byref(steps), cap, _ptr(ran),
                        _ptr(changed), _ptr(messages), _ptr(secs), ctypes.byref(build_s),
                        float(tol), _ptr(delta))
    if rc not in (OK, GUARD):
        raise ValueError(f"oracle_run failed with status {rc}")
    s = min(steps.value, cap)
    return {
        "status": rc,
        "values": vals,
        "supersteps": steps.value,
        "ran": ran[:s].copy(),
        "changed": changed[:s].copy(),
        "messages": messages[:s].copy(),
        "seconds": secs[:s].copy(),
        "delta": delta[:s].copy(),
        "build_seconds": build_s.value,
    }


def pagerank(n, src, dst, k=10, **kw):
    return run(APP_PAGERANK, n, src, dst, None, k=k, **kw)


def hashmin_cc(n, src, dst, **kw):
    return run(APP_HASHMIN_CC, n, src, dst, None, **kw)


def sssp(n, src, dst, w=None, source=0, **kw):
    return run(APP_SSSP, n, src, dst, w, source=source, **kw)
