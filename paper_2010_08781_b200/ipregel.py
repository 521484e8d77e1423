"""Thin ctypes binding of libipregel.so (include/ipregel.h).

Argument marshalling only: every superstep runs in the library's sm_100a kernels.  PyTorch
supplies device memory (tensors whose data_ptr() are passed as borrowed device pointers),
streams and, for multi-GPU, the process group that ships the NCCL unique id.  There is no
CPU fallback: if the shared library is missing or the device is not sm_100, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IPREGEL_LIB") or os.path.join(_HERE, "libipregel.so")

APP_PAGERANK, APP_HASHMIN_CC, APP_SSSP = 0, 1, 2
COMBINE_SUM, COMBINE_MIN, COMBINE_MAX = 0, 1, 2
VALUE_U32, VALUE_F64, VALUE_F32, VALUE_I32, VALUE_U64, VALUE_I64 = 0, 1, 2, 3, 4, 5
COMBINERS = {"sum": COMBINE_SUM, "min": COMBINE_MIN, "max": COMBINE_MAX}
VALUE_TYPES = {"u32": VALUE_U32, "f64": VALUE_F64, "f32": VALUE_F32, "i32": VALUE_I32,
               "u64": VALUE_U64, "i64": VALUE_I64}
_NP_DTYPES = {"u32": np.uint32, "f64": np.float64, "f32": np.float32, "i32": np.int32,
              "u64": np.uint64, "i64": np.int64}
APP_PROGRAM = 3   # last run was a user program
MODE_AUTO, MODE_PULL, MODE_PUSH = 0, 1, 2
MEMORY_DEVICE, MEMORY_HOST = 0, 1
INF = 0xFFFFFFFF

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_INVALID_GRAPH = 2
ERR_OUT_OF_MEMORY = 3
ERR_CUDA = 4
ERR_NCCL = 5
ERR_MAX_SUPERSTEPS = 6
ERR_STATE = 7
ERR_UNSUPPORTED = 8

APPS = {"pagerank": APP_PAGERANK, "cc": APP_HASHMIN_CC, "sssp": APP_SSSP}
COMBINER_OF = {APP_PAGERANK: COMBINE_SUM, APP_HASHMIN_CC: COMBINE_MIN, APP_SSSP: COMBINE_MIN}
MODES = {"auto": MODE_AUTO, "pull": MODE_PULL, "push": MODE_PUSH}
RUN_EXCHANGE_COLLECTIVE, RUN_EXCHANGE_FUSED = 0x1, 0x2
RUN_PAGERANK_MASS = 0x4
LAYOUT_AS_GIVEN, LAYOUT_DEGREE = 0, 1
EXCHANGES = {"auto": 0, "collective": RUN_EXCHANGE_COLLECTIVE, "fused": RUN_EXCHANGE_FUSED}
EXCHANGE_NAMES = {0: "none", 1: "collective", 2: "fused"}


class IpregelError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {status_string(status)}: {detail}")
        self.status = status


class GraphDesc(ctypes.Structure):
    _fields_ = [
        ("num_vertices", ctypes.c_int64), ("num_edges", ctypes.c_int64),
        ("vertex_begin", ctypes.c_int64), ("vertex_end", ctypes.c_int64),
        ("csc_edges", ctypes.c_int64), ("csr_edges", ctypes.c_int64),
        ("csc_offsets", ctypes.c_void_p), ("csc_indices", ctypes.c_void_p),
        ("csc_weights", ctypes.c_void_p),
        ("csr_offsets", ctypes.c_void_p), ("csr_indices", ctypes.c_void_p),
        ("csr_weights", ctypes.c_void_p),
        ("memory", ctypes.c_int32), ("validate", ctypes.c_int32),
        ("vertex_ids", ctypes.c_void_p), ("degree_ordered", ctypes.c_int32),
        ("layout", ctypes.c_int32),
    ]


class RunParams(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("pagerank_iterations", ctypes.c_uint32),
                ("sssp_source", ctypes.c_uint32), ("push_fraction", ctypes.c_float),
                ("flags", ctypes.c_uint32), ("pagerank_tolerance", ctypes.c_double)]


class Stats(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_uint32), ("supersteps", ctypes.c_uint32),
                ("status", ctypes.c_int32), ("exchange", ctypes.c_int32),
                ("time_ms", ctypes.c_void_p), ("kernel_ms", ctypes.c_void_p),
                ("mode", ctypes.c_void_p), ("changed", ctypes.c_void_p),
                ("messages", ctypes.c_void_p), ("edges_scanned", ctypes.c_void_p),
                ("model_bytes", ctypes.c_void_p), ("pagerank_delta", ctypes.c_void_p),
                ("pagerank_mass", ctypes.c_void_p), ("pagerank_mass_nd", ctypes.c_void_p),
                ("part_ms", ctypes.c_void_p)]


class ProgramDesc(ctypes.Structure):
    _fields_ = [("source", ctypes.c_char_p), ("value_type", ctypes.c_int32),
                ("combiner", ctypes.c_int32), ("symmetric", ctypes.c_int32),
                ("aggregator", ctypes.c_int32), ("reserved", ctypes.c_int32)]


# every symbol include/ipregel.h declares (tests check the library exports all of them)
EXPORTS = [
    "ipregel_status_string", "ipregel_last_error", "ipregel_abi_version",
    "ipregel_kernel_launches", "ipregel_device_check",
    "ipregel_run_params_default", "ipregel_nccl_unique_id", "ipregel_comm_create",
    "ipregel_comm_destroy", "ipregel_partition", "ipregel_graph_create",
    "ipregel_graph_create_partitioned", "ipregel_graph_destroy", "ipregel_memory_footprint",
    "ipregel_run", "ipregel_get_values", "ipregel_get_values_async", "ipregel_graph_sync",
    "ipregel_get_stats",
    "ipregel_program_create", "ipregel_program_log", "ipregel_program_cubin_bytes",
    "ipregel_program_destroy", "ipregel_run_program",
]

_lib = None


def load() -> ctypes.CDLL:
    """Load libipregel.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    I = ctypes.c_int
    sig = {
        "ipregel_status_string": (ctypes.c_char_p, [I]),
        "ipregel_last_error": (ctypes.c_char_p, []),
        "ipregel_abi_version": (I, []),
        "ipregel_kernel_launches": (ctypes.c_uint64, []),
        "ipregel_device_check": (I, [I]),
        "ipregel_run_params_default": (I, [ctypes.POINTER(RunParams)]),
        "ipregel_nccl_unique_id": (I, [P]),
        "ipregel_comm_create": (I, [I, I, P, I, ctypes.POINTER(P)]),
        "ipregel_comm_destroy": (None, [P]),
        "ipregel_partition": (I, [P, ctypes.c_int64, I, P]),
        "ipregel_graph_create": (I, [ctypes.POINTER(GraphDesc), P, P, ctypes.POINTER(P)]),
        "ipregel_graph_create_partitioned": (I, [ctypes.POINTER(GraphDesc), I, P,
                                                 ctypes.POINTER(P)]),
        "ipregel_graph_destroy": (None, [P]),
        "ipregel_memory_footprint": (I, [P, ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.POINTER(ctypes.c_uint64)]),
        "ipregel_run": (I, [P, I, I, ctypes.c_uint32, ctypes.POINTER(RunParams)]),
        "ipregel_get_values": (I, [P, P, ctypes.c_size_t, I]),
        "ipregel_get_values_async": (I, [P, P, ctypes.c_size_t]),
        "ipregel_graph_sync": (I, [P]),
        "ipregel_get_stats": (I, [P, ctypes.POINTER(Stats)]),
        "ipregel_program_create": (I, [ctypes.POINTER(ProgramDesc), ctypes.POINTER(P)]),
        "ipregel_program_log": (ctypes.c_char_p, [P]),
        "ipregel_program_cubin_bytes": (ctypes.c_uint64, [P]),
        "ipregel_program_destroy": (None, [P]),
        "ipregel_run_program": (I, [P, P, ctypes.c_uint32, ctypes.POINTER(RunParams),
                                    ctypes.POINTER(ctypes.c_double), I]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def status_string(status: int) -> str:
    return load().ipregel_status_string(status).decode()


def last_error() -> str:
    return load().ipregel_last_error().decode()


def _check(status: int, where: str, allow=()):
    if status != OK and status not in allow:
        raise IpregelError(status, where, last_error())
    return status


def kernel_launches() -> int:
    """Kernels launched by libipregel.so in this process so far."""
    return int(load().ipregel_kernel_launches())


def device_check(device: int = 0) -> None:
    _check(load().ipregel_device_check(device), "ipregel_device_check")


def run_params_default() -> RunParams:
    p = RunParams()
    _check(load().ipregel_run_params_default(ctypes.byref(p)), "ipregel_run_params_default")
    return p


def partition(cost_prefix: np.ndarray, world: int) -> np.ndarray:
    """Host edge-balanced 1D partition bounds (ipregel_partition)."""
    cp = np.ascontiguousarray(cost_prefix, dtype=np.int64)
    out = np.zeros(world + 1, np.int64)
    _check(load().ipregel_partition(cp.ctypes.data, len(cp) - 1, world, out.ctypes.data),
           "ipregel_partition")
    return out


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(load().ipregel_nccl_unique_id(ctypes.addressof(buf)), "ipregel_nccl_unique_id")
    return bytes(buf)


class Comm:
    """Library-owned NCCL communicator (one process per GPU)."""

    def __init__(self, rank: int, world: int, uid: bytes, device: int):
        assert len(uid) == 128
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        _check(load().ipregel_comm_create(rank, world, ctypes.addressof(buf), device,
                                          ctypes.byref(h)), "ipregel_comm_create")
        self.handle = h
        self.rank, self.world, self.device = rank, world, device

    @classmethod
    def from_process_group(cls, device: int):
        """Bootstrap over torch.distributed: rank 0 makes the id, a broadcast ships it."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        t = torch.zeros(128, dtype=torch.uint8,
                        device=f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, src=0)
        return cls(rank, world, bytes(t.cpu().numpy().tobytes()), device)

    def close(self):
        if self.handle:
            load().ipregel_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Program:
    """A user vertex program (ipregel_program_create): CUDA C++ source defining ipr_init,
    ipr_compute and ipr_edge (include/ipregel.h), compiled by NVRTC for sm_100a."""

    def __init__(self, source: str, value_type: str = "u32", combiner: str = "min",
                 symmetric: bool = False, aggregator: str | None = None):
        d = ProgramDesc()
        self._src = source.encode()
        d.source = self._src
        d.value_type = VALUE_TYPES[value_type]
        d.combiner = COMBINERS[combiner]
        d.symmetric = 1 if symmetric else 0
        d.aggregator = 0 if aggregator is None else 1 + COMBINERS[aggregator]
        d.reserved = 0
        h = ctypes.c_void_p()
        _check(load().ipregel_program_create(ctypes.byref(d), ctypes.byref(h)),
               "ipregel_program_create")
        self.handle = h
        self.value_type = value_type
        self.combiner = combiner
        self.symmetric = symmetric

    @property
    def log(self) -> str:
        return load().ipregel_program_log(self.handle).decode()

    @property
    def cubin_bytes(self) -> int:
        return int(load().ipregel_program_cubin_bytes(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            load().ipregel_program_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


@dataclass
class Partition:
    """One owned destination range [vertex_begin, vertex_end) with rebased CSC/CSR rows.

    Arrays are torch CUDA tensors (borrowed, kept alive by this object) or numpy arrays
    (memory = HOST: copied by the library during create).
    """
    num_vertices: int
    num_edges: int
    vertex_begin: int
    vertex_end: int
    csc_offsets: object
    csc_indices: object
    csr_offsets: object            # None (with csr_indices, csr_weights): derived on the device
    csr_indices: object
    csc_weights: object = None
    csr_weights: object = None
    vertex_ids: object = None        # original id of each internal vertex (full [N]) or None
    degree_ordered: bool = False
    layout: int = 0                  # LAYOUT_DEGREE: the library relabels by out-degree

    def desc(self, validate: bool = False) -> GraphDesc:
        host = isinstance(self.csc_offsets, np.ndarray)
        d = GraphDesc()
        d.num_vertices = self.num_vertices
        d.num_edges = self.num_edges
        d.vertex_begin = self.vertex_begin
        d.vertex_end = self.vertex_end
        d.csc_edges = int(self.csc_indices.shape[0])
        d.csr_edges = 0 if self.csr_indices is None else int(self.csr_indices.shape[0])
        d.csc_offsets = _ptr(self.csc_offsets)
        d.csc_indices = _ptr(self.csc_indices)
        d.csc_weights = _ptr(self.csc_weights)
        d.csr_offsets = _ptr(self.csr_offsets)
        d.csr_indices = _ptr(self.csr_indices)
        d.csr_weights = _ptr(self.csr_weights)
        d.memory = MEMORY_HOST if host else MEMORY_DEVICE
        d.validate = 1 if validate else 0
        d.vertex_ids = _ptr(self.vertex_ids)
        d.degree_ordered = 1 if self.degree_ordered else 0
        d.layout = int(self.layout)
        return d


class Graph:
    """An ipregel_graph handle (single GPU, one rank of a Comm, or loopback partitions)."""

    def __init__(self, parts, comm: Comm | None = None, stream=None, validate: bool = False):
        import torch
        if isinstance(parts, Partition):
            parts = [parts]
        self.parts = list(parts)  # keeps borrowed tensors alive
        self.n = self.parts[0].num_vertices
        self.e = self.parts[0].num_edges
        self.comm = comm
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        sp = ctypes.c_void_p(self.stream.cuda_stream)
        h = ctypes.c_void_p()
        lib = load()
        descs = (GraphDesc * len(self.parts))(*[p.desc(validate) for p in self.parts])
        if len(self.parts) == 1:
            st = lib.ipregel_graph_create(descs, comm.handle if comm else None, sp, ctypes.byref(h))
        else:
            assert comm is None
            st = lib.ipregel_graph_create_partitioned(descs, len(self.parts), sp, ctypes.byref(h))
        _check(st, "ipregel_graph_create")
        self.handle = h
        self.last_app = None
        self._pending = []   # host tensors of values_async copies in flight

    def close(self):
        if getattr(self, "handle", None):
            load().ipregel_graph_destroy(self.handle)   # waits for the async copies
            self.handle = None
        self._pending = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, app, max_supersteps: int = 1 << 30, mode="auto", iterations: int = 10,
            source: int = 0, push_fraction: float = 0.04, combiner=None,
            allow_guard: bool = False, exchange: str = "auto", tolerance: float = -1.0,
            mass: bool = False) -> int:
        app = APPS[app] if isinstance(app, str) else int(app)
        p = run_params_default()
        p.mode = MODES[mode] if isinstance(mode, str) else int(mode)
        p.pagerank_iterations = iterations
        p.sssp_source = source
        p.push_fraction = push_fraction
        p.flags = EXCHANGES[exchange] | (RUN_PAGERANK_MASS if mass else 0)
        p.pagerank_tolerance = tolerance
        comb = COMBINER_OF.get(app, COMBINE_SUM) if combiner is None else combiner
        st = load().ipregel_run(self.handle, app, comb, max_supersteps, ctypes.byref(p))
        _check(st, "ipregel_run", allow=(ERR_MAX_SUPERSTEPS,) if allow_guard else ())
        self.last_app = app
        return st

    def run_program(self, program: "Program", params=(), max_supersteps: int = 1 << 30,
                    mode="auto", push_fraction: float = 0.04, exchange: str = "auto",
                    allow_guard: bool = False) -> int:
        """Run a user vertex program (ipregel_run_program); params: up to 8 floats."""
        p = run_params_default()
        p.mode = MODES[mode] if isinstance(mode, str) else int(mode)
        p.push_fraction = push_fraction
        p.flags = EXCHANGES[exchange]
        vals = (ctypes.c_double * 8)(*[float(x) for x in params])
        st = load().ipregel_run_program(self.handle, program.handle, max_supersteps,
                                        ctypes.byref(p), vals, len(params))
        _check(st, "ipregel_run_program", allow=(ERR_MAX_SUPERSTEPS,) if allow_guard else ())
        self.last_app = APP_PROGRAM
        self._last_vt = program.value_type
        return st

    def values_async(self, out):
        """Start copying the last run's values into `out` (a pinned, contiguous CPU torch tensor
        of N elements of the last run's value type); complete after sync().  The graph keeps a
        reference to `out` until sync() or close(), so the copy never writes freed memory."""
        import torch
        if self.last_app is None:
            raise IpregelError(ERR_STATE, "values_async", "no completed run")
        if self.last_app == APP_PROGRAM:
            want = _NP_DTYPES[self._last_vt]
        else:
            want = np.float64 if self.last_app == APP_PAGERANK else np.uint32
        esz = np.dtype(want).itemsize
        if (not isinstance(out, torch.Tensor) or out.device.type != "cpu" or not out.is_pinned()
                or not out.is_contiguous() or out.numel() != self.n or out.element_size() != esz):
            raise IpregelError(ERR_INVALID_ARGUMENT, "values_async",
                               f"out must be a pinned contiguous CPU tensor of {self.n} "
                               f"{esz}-byte elements")
        _check(load().ipregel_get_values_async(self.handle, out.data_ptr(),
                                               out.numel() * out.element_size()),
               "ipregel_get_values_async")
        self._pending.append(out)
        return out

    def sync(self):
        _check(load().ipregel_graph_sync(self.handle), "ipregel_graph_sync")
        self._pending.clear()

    def values(self, out=None, host: bool = False):
        """Full N-vector of the last run: torch CUDA tensor (default) or numpy (host=True)."""
        import torch
        if self.last_app is None:
            raise IpregelError(ERR_STATE, "values", "no completed run")
        if self.last_app == APP_PROGRAM:
            dt = _NP_DTYPES[self._last_vt]
        else:
            dt = np.float64 if self.last_app == APP_PAGERANK else np.uint32
        if host:
            out = np.empty(self.n, dt)
            _check(load().ipregel_get_values(self.handle, out.ctypes.data, out.nbytes, 0),
                   "ipregel_get_values")
            return out
        if out is None:
            tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
                   np.dtype(np.uint64): torch.int64, np.dtype(np.int64): torch.int64}.get(
                       np.dtype(dt), torch.int32)
            out = torch.empty(self.n, dtype=tdt, device="cuda")
        _check(load().ipregel_get_values(self.handle, out.data_ptr(),
                                         out.numel() * out.element_size(), 1),
               "ipregel_get_values")
        return out

    def stats(self, capacity: int = 4096) -> dict:
        arrs = {
            "time_ms": np.zeros(capacity, np.float32), "kernel_ms": np.zeros(capacity, np.float32),
            "mode": np.zeros(capacity, np.uint8), "changed": np.zeros(capacity, np.uint64),
            "messages": np.zeros(capacity, np.uint64),
            "edges_scanned": np.zeros(capacity, np.uint64),
            "model_bytes": np.zeros(capacity, np.uint64),
            "pagerank_delta": np.zeros(capacity, np.float64),
            "pagerank_mass": np.zeros(capacity, np.float64),
            "pagerank_mass_nd": np.zeros(capacity, np.float64),
            "part_ms": np.zeros(capacity, np.float32),
        }
        st = Stats()
        st.capacity = capacity
        for k, a in arrs.items():
            setattr(st, k, a.ctypes.data)
        _check(load().ipregel_get_stats(self.handle, ctypes.byref(st)), "ipregel_get_stats")
        m = min(st.supersteps, capacity)
        out = {k: a[:m].copy() for k, a in arrs.items()}
        out["supersteps"] = st.supersteps
        out["status"] = st.status
        out["exchange"] = EXCHANGE_NAMES.get(st.exchange, str(st.exchange))
        return out

    def memory_footprint(self):
        gb, sb = ctypes.c_uint64(), ctypes.c_uint64()
        _check(load().ipregel_memory_footprint(self.handle, ctypes.byref(gb), ctypes.byref(sb)),
               "ipregel_memory_footprint")
        return gb.value, sb.value


def full_partition(n: int, e: int, csc_offsets, csc_indices, csr_offsets, csr_indices,
                   csc_weights=None, csr_weights=None, vertex_ids=None,
                   degree_ordered=False, layout: int = LAYOUT_AS_GIVEN) -> Partition:
    """The whole graph as one partition (single GPU).  layout=LAYOUT_DEGREE: the library
    relabels it by out-degree during create (vertex_ids None, degree_ordered False)."""
    return Partition(n, e, 0, n, csc_offsets, csc_indices, csr_offsets, csr_indices,
                     csc_weights, csr_weights, vertex_ids, degree_ordered, layout)


def split_partitions(n: int, e: int, bounds, csc_offsets, csc_indices, csr_offsets, csr_indices,
                     csc_weights=None, csr_weights=None, vertex_ids=None, degree_ordered=False):
    """Slice a full CSC/CSR (torch CUDA tensors) into destination ranges `bounds` (rebased
    offsets; index/weight arrays are views, not copies).  Create-time plumbing only."""
    parts = []
    for r in range(len(bounds) - 1):
        vb, ve = int(bounds[r]), int(bounds[r + 1])
        cb, ce = int(csc_offsets[vb]), int(csc_offsets[ve])
        rb, re_ = int(csr_offsets[vb]), int(csr_offsets[ve])
        parts.append(Partition(
            n, e, vb, ve,
            (csc_offsets[vb:ve + 1] - cb).contiguous(), csc_indices[cb:ce],
            (csr_offsets[vb:ve + 1] - rb).contiguous(), csr_indices[rb:re_],
            None if csc_weights is None else csc_weights[cb:ce],
            None if csr_weights is None else csr_weights[rb:re_], vertex_ids, degree_ordered))
    return parts


def edge_balanced_bounds(csc_offsets_host: np.ndarray, world: int, csr_offsets_host=None,
                         vertex_cost: int = 2) -> np.ndarray:
    """Destination partition with cost(v) = indeg(v) (+ outdeg(v) for CC) + vertex_cost
    (SURVEY.md 8(e)); bounds via ipregel_partition."""
    cp = np.asarray(csc_offsets_host, np.int64).copy()
    if csr_offsets_host is not None:
        cp = cp + np.asarray(csr_offsets_host, np.int64)
    cp = cp + vertex_cost * np.arange(len(cp), dtype=np.int64)
    return partition(cp, world)
