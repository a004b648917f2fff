"""Fixed cost of one gna_gl_integrate step replayed from a CUDA graph, vs problem size,
with and without an L2 flush before each step (the bench flushes)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for nbins in (1, 1000, 10_000, 100_000, 1_000_000):
        edges = torch.tensor(synth.uniform_edges(nbins), dtype=torch.float64, device=dev)
        out = torch.empty(nbins, dtype=torch.float64, device=dev)
        gna.gl_integrate(synth.CANONICAL, 52.5, edges, 10, out=out)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            gna.gl_integrate(synth.CANONICAL, 52.5, edges, 10, out=out)
        torch.cuda.current_stream().wait_stream(s)
        for fl in (True, False):
            ts = []
            for _ in range(50):
                if fl:
                    flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                ts.append((a, b))
            torch.cuda.synchronize()
            t = np.median([x.elapsed_time(y) for x, y in ts]) * 1e3
            print("nbins %8d  flush %-5s  %.2f us/step  %.1f G energies/s" % (
                nbins, fl, t, nbins * 10 / t / 1e3))
    # back-to-back replays without events in between (launch-rate limit)
    edges = torch.tensor(synth.uniform_edges(100_000), dtype=torch.float64, device=dev)
    out = torch.empty(100_000, dtype=torch.float64, device=dev)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(20):
            gna.gl_integrate(synth.CANONICAL, 52.5, edges, 10, out=out)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    print("cfg2 x 20 in one graph, L2 warm: %.2f us per launch" % (a.elapsed_time(b) * 1e3 / 200))


if __name__ == "__main__":
    main()
