"""Multi-GPU tests of the batch path: one process per GPU, NCCL.

They need at least two GPUs (one rank per GPU; ranks whose kernels wait on one another must
not share a GPU) and skip otherwise — gpurun and the round-end GPU tier here have one GPU,
so on this pool they document and guard the N > 1 path for a multi-GPU box:

* the chunk-pipelined NCCL all-gather (dist.ShardedBatch) of spectra and chi^2: every
  rank's gathered result equals the oracle on sampled points and equals one single-GPU batch
  bit for bit;
* the gather fused into the kernel epilogue (gna_oscprob_batch_ex with GNA_OUT_PEER, and
  GNA_OUT_MULTICAST where the fabric supports NVLS) through symmetric memory: the gathered
  result equals the oracle on sampled points and one local batch bit for bit.

The same checks run inside bench.py at N > 1 (config.gather_verified, the isolated fused
probe).  The CPU side of this logic is covered on gloo by tests/test_dist_gloo.py.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL_BIN = 1e-11
EPS = np.finfo(np.float64).eps


def _ngpus() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:  # noqa: BLE001
        return 0


needs2 = pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (one rank per GPU)")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(P=37, nbase=3, nbins=257, order=10):
    g = synth.rng(3100 + P)
    pts = synth.points_uniform(g, P, dict(theta12=(0.5, 0.65), theta13=(0.1, 0.2),
                                          dm2_21=(6e-5, 9e-5), dm2_31=(2.2e-3, 2.8e-3)))
    pts = synth.invert_ordering(g, pts)
    L = np.array([52.5, 215.0, 265.0][:nbase])
    om = (52.5 / L) ** 2
    edges = synth.uniform_edges(nbins)
    data = synth.pseudo_data(g, edges, om.sum())
    return pts, L, om, edges, order, data


def _worker(rank, world, port, mode, out_dir):
    import torch
    import torch.distributed as dist

    import paper_1804_07682_b200 as gna
    from paper_1804_07682_b200 import dist as gdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        pts, L, om, edges, order, data = _case()
        P, nb = pts["theta12"].size, edges.size - 1
        f64 = dict(dtype=torch.float64, device=dev)
        de, dd = torch.tensor(edges, **f64), torch.tensor(data, **f64)
        if mode == "nccl":
            sb = gdist.ShardedBatch(P, nb, world, rank, chunks=3).allocate(dev)
            mine = {k: torch.tensor(v[sb.lo:sb.hi], **f64) for k, v in pts.items()}
            ws = torch.empty(gna.oscprob_batch_workspace_size(sb.count, L.size, nb, order) // 8
                             + 2, **f64)

            def compute(vlo, vhi, sp_rows, x2_rows):
                gna.oscprob_batch({k: v[vlo:vhi] for k, v in mine.items()}, L, om, de, order,
                                  data=dd, spectra=sp_rows, chi2=x2_rows, workspace=ws,
                                  tables_valid=vlo > 0)

            sb.step(compute, comm_stream=torch.cuda.Stream(device=dev))
            s, x = sb.gathered()
            have = True
        else:
            fg = gdist.FusedGather(P, nb, dev, prefer_multicast=(mode == "multicast"))
            if mode == "multicast" and not fg.multicast:
                np.save(os.path.join(out_dir, "skip_%d.npy" % rank), np.zeros(1))
                return
            sp_ptr, x2_ptr, flags = fg.out_ptrs()
            mine = {k: torch.tensor(v[fg.lo:fg.hi], **f64) for k, v in pts.items()}
            fg.spectra.fill_(float("nan"))
            fg.chi2.fill_(float("nan"))
            fg.barrier(timeout_ms=20_000)
            gna.oscprob_batch_ex(mine, L, om, de, order, sp_ptr, x2_ptr, flags, data=dd)
            fg.barrier(timeout_ms=20_000)
            torch.cuda.synchronize()
            s, x = fg.result()
            have = rank == 0 or fg.multicast
        if have:
            allp = {k: torch.tensor(v, **f64) for k, v in pts.items()}
            s1, x1 = gna.oscprob_batch(allp, L, om, de, order, data=dd)
            np.save(os.path.join(out_dir, "same_%d.npy" % rank),
                    np.array([bool(torch.equal(s, s1)) and bool(torch.equal(x, x1))]))
            np.save(os.path.join(out_dir, "sp_%d.npy" % rank), s.cpu().numpy())
            np.save(os.path.join(out_dir, "x2_%d.npy" % rank), x.cpu().numpy())
        torch.cuda.synchronize()
        dist.barrier(device_ids=[rank])
    finally:
        dist.destroy_process_group()


def _run(mode, tmp_path, world=2):
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(world, _free_port(), mode, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    if any(f.startswith("skip_") for f in os.listdir(tmp_path)):
        pytest.skip("no NVLS multicast on this fabric")
    pts, L, om, edges, order, data = _case()
    idx = np.array([0, 1, 18, 19, 36])
    spr, x2r = oracle.batch(synth.subset_points(pts, idx), L, om, edges, order, data=data)
    checked = 0
    for r in range(world):
        f = os.path.join(tmp_path, "sp_%d.npy" % r)
        if not os.path.exists(f):
            continue
        sp, x2 = np.load(f), np.load(os.path.join(tmp_path, "x2_%d.npy" % r))
        assert bool(np.load(os.path.join(tmp_path, "same_%d.npy" % r))[0]), r
        assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= TOL_BIN
        d = np.abs(spr - data)  # the chi^2 bound of tests/test_gpu_parity.py::_chi2_bound
        bound = np.sum((2 * d * TOL_BIN * np.abs(spr) + d * d * 8 * EPS) / data, axis=-1)
        assert np.all(np.abs(x2[idx] - x2r) <= bound + 1e-300)
        checked += 1
    assert checked >= 1


@needs2
def test_two_rank_nccl_gather_vs_oracle_and_bitwise(tmp_path):
    _run("nccl", tmp_path)


@needs2
def test_two_rank_fused_epilogue_peer_vs_oracle_and_bitwise(tmp_path):
    _run("peer", tmp_path)


@needs2
def test_two_rank_fused_epilogue_multicast_vs_oracle_and_bitwise(tmp_path):
    _run("multicast", tmp_path)


def test_fused_probe_runs_on_one_rank():
    """bench.py's isolated start-up check of the fused epilogue (--fused-probe) as a one-rank
    torch.distributed.run job on this GPU: symmetric-memory window, gna_oscprob_batch_ex with
    peer-window stores, barrier, bitwise comparison with a local batch -> FUSED_PROBE_OK.  The
    same code runs at N > 1 before bench.py ever uses the fused path."""
    import subprocess
    import sys
    if _ngpus() < 1:
        pytest.skip("no GPU")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    for w in ("cfg5", "cfg4"):
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                            "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                            "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
                            "--fused-probe", "--gpus", "1", "--workload", w],
                           capture_output=True, text=True, timeout=300, env=env, cwd=root)
        assert r.returncode == 0, r.stderr[-3000:]
        assert "FUSED_PROBE_OK peer-to-root" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


def _ipc_writer(rank, world, q_buf, q_done, P, nb):
    """Rank r > 0: receive the root's output tensors (CUDA IPC mapping of another process's
    allocation) and write its rows through the fused epilogue (GNA_OUT_PEER)."""
    import torch

    import paper_1804_07682_b200 as gna
    from paper_1804_07682_b200 import dist as gdist
    import traceback
    try:
        torch.cuda.set_device(0)
        sp_root, x2_root = q_buf.get()
        pts, L, om, edges, order, data = _case(P=P, nbins=nb)
        lo, hi = gdist.shard_range(P, world, rank)
        f64 = dict(dtype=torch.float64, device="cuda")
        mine = {k: torch.tensor(v[lo:hi], **f64) for k, v in pts.items()}
        gna.oscprob_batch_ex(mine, L, om, torch.tensor(edges, **f64), order,
                             sp_root.data_ptr() + lo * nb * 8, x2_root.data_ptr() + lo * 8,
                             gna.GNA_OUT_PEER, data=torch.tensor(data, **f64))
        torch.cuda.synchronize()
        q_done.put(rank)
    except BaseException:  # reported to the root instead of a silent child exit
        q_done.put("rank %d: %s" % (rank, traceback.format_exc()))
        return
    q_buf.get()  # keep the mapping alive until the root has read the result


def test_peer_epilogue_writes_another_process_buffer_one_gpu(tmp_path):
    """The fused epilogue's peer stores across a process boundary, on one GPU: rank 0 owns the
    gathered spectra / chi^2 buffers, ranks 1-2 (separate processes, CUDA IPC mappings of
    rank 0's allocations) write their rows with gna_oscprob_batch_ex(GNA_OUT_PEER) while rank 0
    writes its own; no kernel waits on another process (host-side hand-off only).  The buffer
    must equal one local batch bit for bit and the oracle on sampled points.  NVLink is not
    involved (one GPU); the window arithmetic and the remote-store epilogue are."""
    import torch
    import torch.multiprocessing as mp

    import paper_1804_07682_b200 as gna
    from paper_1804_07682_b200 import dist as gdist
    if _ngpus() < 1:
        pytest.skip("no GPU")
    P, nb, world = 37, 257, 3
    pts, L, om, edges, order, data = _case(P=P, nbins=nb)
    f64 = dict(dtype=torch.float64, device="cuda")
    sp = torch.full((P, nb), float("nan"), **f64)
    x2 = torch.full((P,), float("nan"), **f64)
    ctx = mp.get_context("spawn")
    q_buf, q_done = ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_ipc_writer, args=(r, world, q_buf, q_done, P, nb))
             for r in range(1, world)]
    for p in procs:
        p.start()
    for _ in procs:
        q_buf.put((sp, x2))
    de, dd = torch.tensor(edges, **f64), torch.tensor(data, **f64)
    lo, hi = gdist.shard_range(P, world, 0)
    gna.oscprob_batch_ex({k: torch.tensor(v[lo:hi], **f64) for k, v in pts.items()}, L, om, de,
                         order, sp.data_ptr() + lo * nb * 8, x2.data_ptr() + lo * 8,
                         gna.GNA_OUT_PEER, data=dd)
    torch.cuda.synchronize()
    # collect the writers' hand-offs; a child that died (or reported an exception) fails the
    # test at once instead of after the timeout
    import queue
    import time
    done, t0 = [], time.monotonic()
    while len(done) < len(procs):
        try:
            done.append(q_done.get(timeout=5))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead, "writer exited with %s" % dead
            assert time.monotonic() - t0 < 300, "writers did not finish in 300 s"
    errs = [d for d in done if isinstance(d, str)]
    assert not errs, "\n".join(errs)
    done = sorted(done)
    assert done == list(range(1, world))
    got_sp, got_x2 = sp.cpu().numpy(), x2.cpu().numpy()
    for _ in procs:
        q_buf.put(None)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_sp, ref_x2 = gna.oscprob_batch({k: torch.tensor(v, **f64) for k, v in pts.items()}, L, om,
                                       de, order, data=dd)
    assert np.array_equal(got_sp, ref_sp.cpu().numpy()) and np.array_equal(got_x2,
                                                                           ref_x2.cpu().numpy())
    idx = np.array([0, 12, 13, 24, 25, 36])  # both sides of every shard boundary
    spr, x2r = oracle.batch(synth.subset_points(pts, idx), L, om, edges, order, data=data)
    assert np.max(np.abs(got_sp[idx] - spr) / np.abs(spr)) <= TOL_BIN
    d = np.abs(spr - data)
    bound = np.sum((2 * d * TOL_BIN * np.abs(spr) + d * d * 8 * EPS) / data, axis=-1)
    assert np.all(np.abs(got_x2[idx] - x2r) <= bound + 1e-300)


def test_sharded_step_with_nccl_capturable_in_cuda_graph_one_rank():
    """bench.py captures the N > 1 NCCL step in a CUDA graph (chunk kernels on the current
    stream, all-gathers on the communication stream); here the same dist.ShardedBatch.step is
    captured with a one-rank NCCL group — the collectives are still NCCL calls inside the
    capture — and the replayed result equals the eager one and the oracle."""
    import subprocess
    import sys
    if _ngpus() < 1:
        pytest.skip("no GPU")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r'''
import sys, socket
import numpy as np
sys.path.insert(0, %r)
sys.path.insert(0, %r)
import torch, torch.distributed as dist
import paper_1804_07682_b200 as gna
from paper_1804_07682_b200 import dist as gdist
import test_multigpu as tm
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%%d" %% port, rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
pts, L, om, edges, order, data = tm._case()
P, nb = pts["theta12"].size, edges.size - 1
f64 = dict(dtype=torch.float64, device="cuda")
de, dd = torch.tensor(edges, **f64), torch.tensor(data, **f64)
sb = gdist.ShardedBatch(P, nb, 1, 0, chunks=3).allocate("cuda")
mine = {k: torch.tensor(v, **f64) for k, v in pts.items()}
ws = torch.empty(gna.oscprob_batch_workspace_size(P, L.size, nb, order) // 8 + 2, **f64)
def compute(vlo, vhi, sp_rows, x2_rows):
    gna.oscprob_batch({k: v[vlo:vhi] for k, v in mine.items()}, L, om, de, order, data=dd,
                      spectra=sp_rows, chi2=x2_rows, workspace=ws, tables_valid=vlo > 0)
comm = torch.cuda.Stream()
# one rank: step() gathers nothing, so drive the chunk gathers explicitly as bench does at N > 1
def step():
    works = []
    for c, (lo, hi) in enumerate(sb.cb):
        compute(lo, min(hi, sb.count), sb.spectra[lo:hi], sb.chi2[lo:hi])
        ev = torch.cuda.Event(); ev.record()
        with torch.cuda.stream(comm):
            comm.wait_event(ev)
            works += sb._gather_chunk(c, lo, hi, dist)
    for w in works:
        w.wait()
    torch.cuda.current_stream().wait_stream(comm)
step(); torch.cuda.synchronize()
ref = torch.cat([gs for gs in sb.g_spectra]).clone()
for gs in sb.g_spectra: gs.zero_()
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream(); cap.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
    step()
torch.cuda.current_stream().wait_stream(cap)
g.replay(); torch.cuda.synchronize()
got = torch.cat([gs for gs in sb.g_spectra])
assert torch.equal(got, ref)
np.save(%r, got.cpu().numpy())
dist.destroy_process_group()
print("CAPTURE_OK")
''' % (root, os.path.join(root, "tests"), os.path.join(root, "build", "nccl_capture_sp.npy"))
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True,
                       timeout=300, cwd=root)
    assert r.returncode == 0 and "CAPTURE_OK" in r.stdout, r.stderr[-3000:]
    pts, L, om, edges, order, data = _case()
    sp = np.load(os.path.join(root, "build", "nccl_capture_sp.npy"))
    idx = np.array([0, 18, 36])
    spr, _ = oracle.batch(synth.subset_points(pts, idx), L, om, edges, order, data=data)
    assert np.max(np.abs(sp[idx] - spr) / np.abs(spr)) <= TOL_BIN
