"""Host-side logic of the multi-GPU path, exercised with world_size 2 over gloo on the CPU.

Covers what runs on the host of every rank: the deterministic edge-balanced
destination partition (identical on every rank, tiling [0, N)), the slicing of CSC/CSR into
rebased per-rank rows, and the NCCL unique-id bootstrap through torch.distributed.  The device
side of the partitioned path is covered on the GPU by the loopback-partition tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.graphs import csr_csc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2010_08781_b200 as ipr
        rng = np.random.default_rng(5)
        n = 5000
        src = rng.integers(0, n, 40000)
        dst = (src * 7 + rng.integers(0, 50, 40000)) % n
        g = csr_csc(n, src, dst)
        bounds = ipr.edge_balanced_bounds(g["csc_off"], world, g["csr_off"])
        # every rank computes the same bounds
        t = torch.tensor(bounds, dtype=torch.int64)
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        same = all(torch.equal(gathered[0], x) for x in gathered)
        # rebased slices of this rank
        T = {k: (None if v is None else torch.from_numpy(np.ascontiguousarray(v)))
             for k, v in g.items() if k in ("csc_off", "csc_idx", "csr_off", "csr_idx")}
        parts = ipr.split_partitions(n, g["e"], bounds, T["csc_off"], T["csc_idx"],
                                     T["csr_off"], T["csr_idx"])
        p = parts[rank]
        own_edges = torch.tensor([p.csc_indices.numel(), p.csr_indices.numel()])
        dist.all_reduce(own_edges)
        ok_slices = (int(p.csc_offsets[0]) == 0 and
                     int(p.csc_offsets[-1]) == p.csc_indices.numel() and
                     int(p.csr_offsets[-1]) == p.csr_indices.numel() and
                     own_edges.tolist() == [g["e"], g["e"]])
        # reconstruct this rank's edges from its slice and compare with the COO restricted to
        # its destination range
        vb, ve = p.vertex_begin, p.vertex_end
        off = p.csc_offsets.numpy()
        rows = np.repeat(np.arange(vb, ve), np.diff(off))
        mine = sorted(zip(p.csc_indices.numpy().tolist(), rows.tolist()))
        want = sorted((int(a), int(b)) for a, b in zip(src, dst) if vb <= b < ve)
        ok_edges = mine == want
        # NCCL unique id: rank 0 creates it, a gloo broadcast ships it
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(ipr.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, src=0)
        ids = [torch.zeros_like(uid) for _ in range(world)]
        dist.all_gather(ids, uid)
        ok_uid = all(torch.equal(ids[0], x) for x in ids) and int(uid.sum()) > 0
        # without a GPU the communicator cannot be created: it must fail loudly, not fall back
        try:
            ipr.Comm(rank, world, bytes(uid.numpy().tobytes()), 0)
            comm_fails = False
        except ipr.IpregelError:
            comm_fails = True
        out[rank] = (same, bounds.tolist(), ok_slices, ok_edges, ok_uid, comm_fails)
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic():
    if torch.cuda.is_available():
        pytest.skip("CPU-only test (a GPU box runs the loopback partition tests instead)")
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        same, bounds, ok_slices, ok_edges, ok_uid, comm_fails = out[r]
        assert same and ok_slices and ok_edges and ok_uid and comm_fails, out[r]
        assert bounds[0] == 0 and bounds[-1] == 5000 and bounds[0] <= bounds[1] <= bounds[2]
