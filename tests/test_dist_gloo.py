"""Multi-process (world_size 2 and 3) CPU tests of the parameter-point partition and
the chunk-pipelined gather (paper_1804_07682_b200/dist.py), on the gloo backend.

The compute step is the oracle on each rank's shard (the CUDA path runs on one
GPU only in this environment); the partition, padding, chunking, collective and
unpadding logic is exactly the code bench.py runs over NCCL.  The gathered
result must be bitwise identical to the single-process oracle on all points.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1804_07682_b200 import dist as gdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(P=11, nbins=13, nbase=2, order=4):
    g = synth.rng(77)
    pts = synth.points_uniform(g, P, dict(theta12=(0.5, 0.65), theta13=(0.1, 0.2),
                                          dm2_21=(6e-5, 9e-5), dm2_31=(2.2e-3, 2.8e-3)))
    L = np.array([52.5, 215.0][:nbase])
    om = np.array([1.0, 0.1][:nbase])
    edges = synth.uniform_edges(nbins, 1.0, 10.0)
    data = synth.pseudo_data(g, edges, om.sum())
    return pts, L, om, edges, order, data


def _worker(rank, world, port, chunks, P, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pts, L, om, edges, order, data = _case(P=P)
        nb = edges.size - 1
        sb = gdist.ShardedBatch(P, nb, world, rank, chunks=chunks).allocate("cpu")

        def compute(vlo, vhi, sp_rows, x2_rows):
            idx = np.arange(sb.lo + vlo, sb.lo + vhi)
            sp, x2 = oracle.batch(synth.subset_points(pts, idx), L, om, edges, order, data=data)
            sp_rows.copy_(torch.from_numpy(sp))
            x2_rows.copy_(torch.from_numpy(x2))

        sb.step(compute)
        s, x = sb.gathered()
        out_q.put((rank, s.numpy().copy(), x.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks,P", [(2, 1, 11), (2, 3, 11), (3, 2, 7), (2, 2, 1)])
def test_sharded_gather_bitwise_equals_single_process(world, chunks, P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, chunks, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pts, L, om, edges, order, data = _case(P=P)
    sp, x2 = oracle.batch(pts, L, om, edges, order, data=data)
    for rank, s, x in res:
        assert np.array_equal(s, sp), rank  # every rank holds the full, ordered result
        assert np.array_equal(x, x2), rank


@pytest.mark.parametrize("P,world", [(0, 1), (1, 1), (7, 2), (1000, 8), (1001, 8), (5, 8)])
def test_shard_range_partitions(P, world):
    cover = []
    counts = []
    for r in range(world):
        lo, hi = gdist.shard_range(P, world, r)
        cover += list(range(lo, hi))
        counts.append(hi - lo)
    assert cover == list(range(P))
    assert max(counts) - min(counts) <= 1
    assert max(counts) <= gdist.padded_rows(P, world)


@pytest.mark.parametrize("P,world,chunks", [(11, 2, 1), (11, 2, 3), (7, 3, 2), (1000, 8, 4),
                                            (3, 8, 2)])
def test_gather_index_is_injective_into_padded_layout(P, world, chunks):
    pos = gdist.gather_index(P, world, chunks)
    Pl = gdist.padded_rows(P, world)
    assert len(set(pos.tolist())) == P
    assert pos.min() >= 0 and pos.max() < world * Pl


def test_shard_range_rejects_bad_args():
    with pytest.raises(ValueError):
        gdist.shard_range(10, 0, 0)
    with pytest.raises(ValueError):
        gdist.shard_range(10, 2, 2)


class _FakeHandle:
    def __init__(self, rank, ptrs, mc):
        self.rank, self.buffer_ptrs, self.multicast_ptr = rank, ptrs, mc


class _FakeTensor:
    def __init__(self, p):
        self.p = p

    def data_ptr(self):
        return self.p


def test_fused_gather_window_arithmetic():
    """Row pointers of the fused-gather epilogue: tensor offset inside the symmetric buffer,
    peer (root) vs multicast base, and this rank's first row."""
    fg = gdist.FusedGather.__new__(gdist.FusedGather)
    fg.npoints, fg.nbins, fg.world, fg.rank = 11, 7, 2, 1
    fg.lo, fg.hi = gdist.shard_range(11, 2, 1)
    fg.spectra, fg.chi2 = _FakeTensor(20_064), _FakeTensor(50_016)
    fg.h_spec = _FakeHandle(1, [10_000, 20_000], 90_000)
    fg.h_chi2 = _FakeHandle(1, [40_000, 50_000], 95_000)
    for mc in (False, True):
        fg.multicast = mc
        sp, x2, flags = fg.out_ptrs()
        base_s = (90_000 if mc else 10_000) + 64
        base_c = (95_000 if mc else 40_000) + 16
        assert sp == base_s + fg.lo * 7 * 8 and x2 == base_c + fg.lo * 8
        assert flags == (2 if mc else 1)


def _probe_worker(rank, world, port, timeout, out_q):
    """Both ranks of a gloo job run bench.isolated_fused_probe: rank 0 starts the isolated
    N-rank check, the other ranks wait on the store; all must get the same verdict."""
    import sys
    from types import SimpleNamespace
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        args = SimpleNamespace(workload="cfg5", precision="fp64", probe_timeout=timeout)
        out_q.put((rank, bench.isolated_fused_probe(args, world, rank, dist)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("timeout", [0.2, 240.0])
def test_isolated_fused_probe_falls_back_and_all_ranks_agree(timeout):
    """With no GPU here the isolated check fails (its ranks cannot start NCCL) or times out;
    either way every rank of the main job gets ok = False and the same reason, so the run
    falls back to the NCCL gather instead of hanging or crashing."""
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: the probe would really run")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_probe_worker, args=(r, 2, port, timeout, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=400) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]
    assert res[0]["ok"] is False
    assert ("timed out" in res[0]["why"]) if timeout < 1 else ("rc=" in res[0]["why"])


def test_auto_chunks():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    per_point = 8 * 10_000 * 10  # cfg5
    assert bench.auto_chunks(1000, 1, per_point) == 1
    assert [bench.auto_chunks(1000, g, per_point) for g in (2, 4, 8)] == [4, 4, 4]
    assert [bench.auto_chunks(10_000, g, 10_000) for g in (2, 4, 8)] == [2, 1, 1]  # cfg4


def _shared_worker(rank, world, port, P, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        store = dist.distributed_c10d._get_default_store()
        nb = 5
        out = gdist.NodeSharedHost({"spectra": (P, nb), "chi2": (P,)}, rank, store, pin=False)
        sb = gdist.ShardedBatch(P, nb, world, rank)
        # each rank writes only its own rows (what gna_oscprob_batch_host does on the GPU)
        out.arrays["spectra"][sb.lo:sb.hi] = np.arange(sb.lo, sb.hi)[:, None] + np.arange(nb) / 10
        out.arrays["chi2"][sb.lo:sb.hi] = -np.arange(sb.lo, sb.hi, dtype=float)
        dist.barrier()
        out_q.put((rank, out.arrays["spectra"].copy(), out.arrays["chi2"].copy()))
        out.close(barrier=dist.barrier)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,P", [(2, 11), (3, 7)])
def test_node_shared_host_gathers_every_ranks_rows(world, P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shared_worker, args=(r, world, port, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.arange(P)[:, None] + np.arange(5) / 10
    for rank, s, x in res:
        assert np.array_equal(s, want) and np.array_equal(x, -np.arange(P, dtype=float)), rank
