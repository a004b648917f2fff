"""Multi-GPU partition of the batch path.

Parameter points are independent units (§2.3 "divide input data into
smaller independent datasets"; P:596-603 independent OscProb instances), so
rank r of G takes the contiguous block [r*P//G, (r+1)*P//G) of points; the
energy grid, GL rule, baselines and data are replicated (uploaded once per GPU,
as the paper copies E once).  The only exchange is the gather of the
per-point binned spectra and chi^2 (BASELINE.json north_star), done with NCCL
all_gather_into_tensor over NVLink, chunk-pipelined on a communication stream so
that chunk c's gather overlaps chunk c+1's kernel.

End to end (host buffers in and out), NodeSharedHost + oscprob_batch_host_sharded
gather the result into host memory shared by the node's ranks, each GPU writing its
own rows over its own PCIe link.

One point's arithmetic never depends on the other points in a call, so the
gathered result is bitwise identical for every G (tests/test_dist_gloo.py on CPU
with gloo; tests/test_gpu_parity.py split invariance on the GPU).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable

import numpy as np


def shard_range(npoints: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced block of points owned by `rank` (counts differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or npoints < 0:
        raise ValueError("bad shard request")
    return rank * npoints // world, (rank + 1) * npoints // world


def padded_rows(npoints: int, world: int) -> int:
    """Rows per rank in the gathered layout (all_gather needs equal sizes)."""
    return -(-npoints // world)


def chunk_bounds(rows: int, chunks: int) -> list[tuple[int, int]]:
    """Row ranges of the gather pipeline's chunks, tapered: chunk c gets a share proportional
    to chunks - c (4 chunks: 4:3:2:1), so that the last chunk — whose all-gather is the only
    one not hidden under a later chunk's kernel — is the smallest.  Every chunk is non-empty
    while rows >= chunks."""
    chunks = max(1, min(chunks, max(rows, 1)))
    wsum = chunks * (chunks + 1) // 2
    bounds, acc = [], 0
    for c in range(chunks):
        acc += chunks - c
        hi = rows * acc // wsum
        lo = bounds[-1][1] if bounds else 0
        hi = max(hi, min(rows, lo + 1))  # non-empty when rows allow
        bounds.append((lo, hi))
    bounds[-1] = (bounds[-1][0], rows)
    return bounds


def gather_index(npoints: int, world: int, chunks: int = 1) -> np.ndarray:
    """Position of global point p in the gathered, padded, chunk-major buffer.

    Gathered layout: for chunk c (bounds over the padded row count Pl), a block of
    world * rows_c rows, rank-major — row r * rows_c + i of chunk c holds local
    row lo_c + i of rank r.
    """
    Pl = padded_rows(npoints, world)
    cb = chunk_bounds(Pl, chunks)
    pos = np.empty(npoints, dtype=np.int64)
    base = 0
    starts = []
    for lo, hi in cb:
        starts.append(base)
        base += world * (hi - lo)
    for r in range(world):
        a, b = shard_range(npoints, world, r)
        for j in range(b - a):
            c = next(k for k, (lo, hi) in enumerate(cb) if lo <= j < hi)
            lo, hi = cb[c]
            pos[a + j] = starts[c] + r * (hi - lo) + (j - lo)
    return pos


@dataclass
class ShardedBatch:
    """Per-rank state of the sharded batch step (spectra + chi^2, gathered on every rank).

    compute(lo, hi, spectra_rows, chi2_rows) fills the local rows [lo, hi) of the
    rank's shard; by default it is the CUDA path (gna.oscprob_batch) — tests on
    CPU pass the oracle instead to exercise the partition and gather logic
    with gloo.
    """
    npoints: int
    nbins: int
    world: int
    rank: int
    chunks: int = 1
    group: object = None

    def __post_init__(self):
        self.lo, self.hi = shard_range(self.npoints, self.world, self.rank)
        self.count = self.hi - self.lo
        self.Pl = padded_rows(self.npoints, self.world)
        self.cb = chunk_bounds(self.Pl, self.chunks)

    def allocate(self, device, want_spectra=True, want_chi2=True):
        import torch
        f64 = dict(dtype=torch.float64, device=device)
        self.spectra = torch.zeros((self.Pl, self.nbins), **f64) if want_spectra else None
        self.chi2 = torch.zeros(self.Pl, **f64) if want_chi2 else None
        # chunk-major gathered buffers: chunk c -> [world * rows_c, ...] (rank-major rows)
        self.g_spectra = ([torch.empty((self.world * (hi - lo), self.nbins), **f64)
                           for lo, hi in self.cb] if want_spectra else None)
        self.g_chi2 = ([torch.empty(self.world * (hi - lo), **f64) for lo, hi in self.cb]
                       if want_chi2 else None)
        return self

    def step(self, compute: Callable, comm_stream=None):
        """Compute every chunk, gathering chunk c while chunk c+1 computes."""
        import torch
        import torch.distributed as dist
        works = []
        on_cuda = self.spectra is not None and self.spectra.is_cuda or (
            self.chi2 is not None and self.chi2.is_cuda)
        for c, (lo, hi) in enumerate(self.cb):
            vlo, vhi = min(lo, self.count), min(hi, self.count)  # valid rows of this chunk
            if vhi > vlo:
                compute(vlo, vhi,
                        self.spectra[vlo:vhi] if self.spectra is not None else None,
                        self.chi2[vlo:vhi] if self.chi2 is not None else None)
            if self.world == 1:
                continue
            if on_cuda and comm_stream is not None:
                ev = torch.cuda.Event()
                ev.record()
                with torch.cuda.stream(comm_stream):
                    comm_stream.wait_event(ev)
                    works += self._gather_chunk(c, lo, hi, dist)
            else:
                works += self._gather_chunk(c, lo, hi, dist)
        for w in works:
            w.wait()
        if on_cuda and comm_stream is not None and self.world > 1:
            torch.cuda.current_stream().wait_stream(comm_stream)

    def _gather_chunk(self, c, lo, hi, dist):
        ws = []
        if self.spectra is not None:
            ws.append(dist.all_gather_into_tensor(self.g_spectra[c], self.spectra[lo:hi],
                                                  group=self.group, async_op=True))
        if self.chi2 is not None:
            ws.append(dist.all_gather_into_tensor(self.g_chi2[c], self.chi2[lo:hi],
                                                  group=self.group, async_op=True))
        return ws

    def gathered(self):
        """(spectra [P, nbins], chi2 [P]) in global point order (copies; for checks)."""
        import torch
        if self.world == 1:
            s = self.spectra[:self.count] if self.spectra is not None else None
            x = self.chi2[:self.count] if self.chi2 is not None else None
            return s, x
        pos = torch.as_tensor(gather_index(self.npoints, self.world, len(self.cb)),
                              device=(self.spectra if self.spectra is not None else self.chi2).device)
        s = x = None
        if self.spectra is not None:
            flat = torch.cat([g.reshape(-1, self.nbins) for g in self.g_spectra])
            s = flat.index_select(0, pos)
        if self.chi2 is not None:
            flat = torch.cat([g.reshape(-1) for g in self.g_chi2])
            x = flat.index_select(0, pos)
        return s, x


class FusedGather:
    """NEXT-4: the gather fused into the batch kernel's epilogue over NVLink.

    The gathered spectra [P, nbins] and chi2 [P] live in symmetric memory
    (torch.distributed._symmetric_memory: every rank's buffer is mapped into every
    rank's address space).  Rank r's kernel writes its rows [lo_r, hi_r) directly:
      * multicast (NVLS, when the fabric supports it): multimem stores to the
        multicast address, so every rank ends with the full result (all-gather);
      * otherwise: plain stores into rank 0's buffer over NVLink (gather to root).
    A symmetric-memory barrier on the stream then orders the remote writes before any
    rank reads.  No separate collective moves the data.
    """

    def __init__(self, npoints: int, nbins: int, device, group=None, prefer_multicast=True):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.npoints, self.nbins = npoints, nbins
        self.lo, self.hi = shard_range(npoints, self.world, self.rank)
        f64 = dict(dtype=torch.float64, device=device)
        self.spectra = symm.empty((npoints, nbins), **f64)
        self.chi2 = symm.empty((npoints,), **f64)
        self.h_spec = symm.rendezvous(self.spectra, self.group)
        self.h_chi2 = symm.rendezvous(self.chi2, self.group)
        mc = False
        if prefer_multicast:
            from torch._C._autograd import DeviceType
            from torch._C._distributed_c10d import _SymmetricMemory
            dev = torch.device(device)
            idx = dev.index if dev.index is not None else torch.cuda.current_device()
            try:
                mc = bool(_SymmetricMemory.has_multicast_support(DeviceType.CUDA, idx))
            except (TypeError, RuntimeError):
                mc = False
        # the multicast window exists only if NVLS initialisation succeeded for both buffers
        self.multicast = (mc and bool(self.h_spec.multicast_ptr)
                          and bool(self.h_chi2.multicast_ptr))
        self.root_only = not self.multicast

    @staticmethod
    def _base(h, tensor, multicast: bool, target_rank: int) -> int:
        ptrs = list(h.buffer_ptrs)
        off = tensor.data_ptr() - ptrs[h.rank]  # the tensor's offset in the symmetric buffer
        return (h.multicast_ptr if multicast else ptrs[target_rank]) + off

    def out_ptrs(self):
        """(spectra rows ptr, chi2 ptr, flags) for this rank's rows."""
        from . import GNA_OUT_MULTICAST, GNA_OUT_PEER
        sb = self._base(self.h_spec, self.spectra, self.multicast, 0)
        cb = self._base(self.h_chi2, self.chi2, self.multicast, 0)
        flags = GNA_OUT_MULTICAST if self.multicast else GNA_OUT_PEER
        return sb + self.lo * self.nbins * 8, cb + self.lo * 8, flags

    def barrier(self, timeout_ms: int = 60_000):
        """Device-side barrier on the current stream: every rank's remote writes are done
        (finite timeout, so a missing rank is an error rather than a hang)."""
        self.h_spec.barrier(channel=0, timeout_ms=timeout_ms)

    def result(self):
        """The gathered (spectra, chi2) as local tensors (all ranks with multicast, rank 0 else)."""
        return self.spectra, self.chi2


class NodeSharedHost:
    """Host output arrays shared by the ranks of one node (POSIX shared memory) and
    page-locked in every rank's CUDA context, for the end-to-end multi-GPU step: each rank's
    host-buffer batch call writes its own rows of the spectra and chi^2 straight from its GPU
    over its own PCIe link, so after a barrier the node's host memory holds the whole,
    gathered result (end to end including the gather; the paper's
    transfer-inclusive timing).  Rank 0 creates the segment; the name travels
    through the process group's store.

    arrays: dict name -> numpy float64 array of the requested shape (same memory on all
    ranks).  close() unpins and detaches (rank 0 also unlinks, after a barrier).
    """

    def __init__(self, shapes: dict, rank: int, store, tag: str = "gna_node_shared",
                 pin: bool = True):
        from multiprocessing import shared_memory
        self.rank = rank
        sizes = {k: int(np.prod(s)) * 8 for k, s in shapes.items()}
        offs, total = {}, 0
        for k, n in sizes.items():
            offs[k] = total
            total += -(-n // 4096) * 4096  # page-aligned arrays
        self.nbytes = max(total, 4096)
        # Rank 0 decides and always publishes a verdict (the segment's name, or "" when it
        # cannot create it), so no rank waits forever.  A tmpfs smaller than the segment would
        # SIGBUS on first touch (or when pinning), so rank 0 refuses up front.
        if rank == 0:
            try:
                st = os.statvfs("/dev/shm")
                free = st.f_bavail * st.f_frsize
            except OSError:
                free = 0
            if free < self.nbytes + (64 << 20):
                store.set(tag, "")
                raise RuntimeError("/dev/shm has %d MB free, the node-shared buffer needs %d MB"
                                   % (free >> 20, self.nbytes >> 20))
            try:
                self.shm = shared_memory.SharedMemory(create=True, size=self.nbytes)
            except Exception:
                store.set(tag, "")
                raise
            store.set(tag, self.shm.name)
        else:
            store.wait([tag])
            name = store.get(tag).decode()
            if not name:
                raise RuntimeError("rank 0 could not create the node-shared buffer")
            self.shm = shared_memory.SharedMemory(name=name)
            try:  # the creator owns the segment's lifetime (Python 3.12 tracks attaches too)
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:  # noqa: BLE001
                pass
        self.arrays = {k: np.ndarray(s, dtype=np.float64, buffer=self.shm.buf, offset=offs[k])
                       for k, s in shapes.items()}
        self.pinned = False
        if pin:
            import torch
            addr = np.frombuffer(self.shm.buf, dtype=np.uint8).ctypes.data
            rc = torch.cuda.cudart().cudaHostRegister(addr, self.nbytes, 0)
            if int(rc) != 0:
                self.arrays = {}
                self.shm.close()
                if rank == 0:
                    self.shm.unlink()
                raise RuntimeError("cudaHostRegister of the node-shared buffer failed (%s)" % rc)
            self._addr, self.pinned = addr, True

    def close(self, barrier=None):
        if self.pinned:
            import torch
            torch.cuda.cudart().cudaHostUnregister(self._addr)
            self.pinned = False
        self.arrays = {}
        if barrier is not None:
            barrier()
        self.shm.close()
        if self.rank == 0:
            self.shm.unlink()


def oscprob_batch_host_sharded(sb: ShardedBatch, points: dict, L_km, omega, edges, order: int,
                               data, out: NodeSharedHost, barrier: Callable, spectra=True):
    """End-to-end multi-GPU batch over HOST arrays: rank r runs the host-buffer batch
    (gna_oscprob_batch_host: chunked H2D -> kernels -> D2H on three streams) on its points
    [lo, hi), writing rows [lo, hi) of the node-shared spectra / chi2, then all ranks meet at
    `barrier`; afterwards every rank sees the full result in host memory.  `points` holds the
    rank's own points (host float64 arrays of hi - lo values, pinned for full PCIe speed)."""
    from . import oscprob_batch_host
    if sb.count > 0:
        oscprob_batch_host(points, L_km, omega, edges, order, data=data,
                           spectra=out.arrays["spectra"][sb.lo:sb.hi] if spectra else False,
                           chi2=out.arrays["chi2"][sb.lo:sb.hi])
    barrier()
