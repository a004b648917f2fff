"""Host-side cost of enqueueing one chunk of the N > 1 step (gna.oscprob_batch on a cfg5 shard
chunk, and a 1-rank NCCL all_gather_into_tensor), and whether the NCCL collective can be
captured in a CUDA graph with this torch / NCCL (1-rank group on this GPU)."""
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def main():
    torch.cuda.set_device(0)
    c = synth.config("cfg5")
    f64 = dict(dtype=torch.float64, device="cuda")
    n = 31
    pts = {k: torch.tensor(v[:n], **f64) for k, v in c["points"].items()}
    edges, data = torch.tensor(c["edges"], **f64), torch.tensor(c["data"], **f64)
    nb = c["edges"].size - 1
    sp = torch.empty((n, nb), **f64)
    x2 = torch.empty(n, **f64)
    ws = torch.empty(gna.oscprob_batch_workspace_size(n, 8, nb, 10) // 8 + 2, **f64)

    def call():
        gna.oscprob_batch(pts, c["L_km"], c["omega"], edges, 10, data=data, spectra=sp, chi2=x2,
                          workspace=ws, tables_valid=True)
    call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        call()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print("host enqueue per batch call: %.1f us" % ((t1 - t0) / 50 * 1e6))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % port, rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    out = torch.empty((n, nb), **f64)
    dist.all_gather_into_tensor(out, sp, async_op=True).wait()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        w = dist.all_gather_into_tensor(out, sp, async_op=True)
    t1 = time.perf_counter()
    w.wait()
    torch.cuda.synchronize()
    print("host enqueue per NCCL all_gather_into_tensor: %.1f us" % ((t1 - t0) / 50 * 1e6))
    # capture: kernel on the current stream, gather on a side stream, joined back
    comm = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    try:
        with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
            call()
            ev = torch.cuda.Event()
            ev.record()
            with torch.cuda.stream(comm):
                comm.wait_event(ev)
                wk = dist.all_gather_into_tensor(out, sp, async_op=True)
            wk.wait()
            torch.cuda.current_stream().wait_stream(comm)
        torch.cuda.current_stream().wait_stream(cap)
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        ok = torch.equal(out, sp)
        print("graph capture of batch + NCCL all_gather: OK, replay result equal:", ok)
    except Exception as exc:  # noqa: BLE001
        print("graph capture of batch + NCCL all_gather FAILED:", repr(exc)[:300])
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
