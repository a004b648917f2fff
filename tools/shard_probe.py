"""Per-rank compute of the cfg5 strong-scaling shards, measured on one GPU: the batch kernel on
P/G points for G = 1, 2, 4, 8 (what each rank runs before the gather).  Shows whether the kernel
keeps its efficiency as the shard shrinks (tail / wave effects).  No collective is involved."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def main(precision="fp64"):
    print("# precision:", precision)
    dev = torch.device("cuda", 0)
    c = synth.config("cfg5")
    f64 = dict(dtype=torch.float64, device=dev)
    edges = torch.tensor(c["edges"], **f64)
    data = torch.tensor(c["data"], **f64)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    nb = c["edges"].size - 1
    base = None
    for G in (1, 2, 4, 8, 16):
        P = 1000 // G
        pts = {k: torch.tensor(v[:P], **f64) for k, v in c["points"].items()}
        sp = torch.empty((P, nb), **f64)
        x2 = torch.empty(P, **f64)
        ws = torch.empty(gna.oscprob_batch_workspace_size(P, 8, nb, 10) // 8 + 2, **f64)
        call = lambda: gna.oscprob_batch(pts, c["L_km"], c["omega"], edges, 10, data=data,  # noqa
                                         spectra=sp, chi2=x2, workspace=ws, precision=precision)
        call()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            call()
        torch.cuda.current_stream().wait_stream(s)
        ts = []
        for _ in range(30):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        t = np.median([x.elapsed_time(y) for x, y in ts])
        evals = P * 8 * nb * 10
        if base is None:
            base = t
        print("G=%2d  points/rank=%4d  %.4f ms  %.1f G energy points/s per GPU  "
              "compute scaling efficiency %.3f" % (G, P, t, evals / t / 1e6, base / (G * t)))


if __name__ == "__main__":
    main(*sys.argv[1:])
