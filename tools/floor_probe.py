"""Where the fixed ~8 us per graph-replayed single-point step comes from.

Times (median of 100, CUDA events on the launching stream) an empty event pair, a
1-bin and a cfg2 gna_gl_integrate step replayed from a CUDA graph, each
  plain:   flush; e0; replay; e1           (the bench's pattern)
  backed:  flush; sleep(~40 us); e0; replay; e1
'backed' keeps the stream busy while the host enqueues e0/replay/e1, so e0..e1 holds
only device time; the difference between the two is host submission latency that
the GPU waited on.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def graph_of(fn):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    return g


def timeit(step, flush, backed, reps=100):
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        if backed:
            torch.cuda._sleep(80_000)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([x.elapsed_time(y) for x, y in ts]) * 1e3)


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    print("empty event pair        plain %.2f us  backed %.2f us" % (
        timeit(lambda: None, flush, False), timeit(lambda: None, flush, True)))
    # an empty kernel (torch's spin kernel with 0 cycles) and a 1-element fill, graph-replayed
    tiny = torch.empty(1, dtype=torch.float64, device=dev)
    for name, fn in (("empty kernel", lambda: torch.cuda._sleep(0)),
                     ("1-element fill", lambda: tiny.fill_(1.0))):
        fn()
        g = graph_of(fn)
        print("%-22s  graph backed %.2f us  eager backed %.2f us" % (
            name, timeit(g.replay, flush, True), timeit(fn, flush, True)))
    for nbins in (1, 100_000, 1_000_000):
        edges = torch.tensor(synth.uniform_edges(nbins), dtype=torch.float64, device=dev)
        out = torch.empty(nbins, dtype=torch.float64, device=dev)

        def call():
            gna.gl_integrate(synth.CANONICAL, 52.5, edges, 10, out=out)
        call()
        g = graph_of(call)
        for fl in (flush, None):
            p = timeit(g.replay, fl, False)
            q = timeit(g.replay, fl, True)
            e = timeit(call, fl, True)
            print("gl nbins %8d flush %-5s graph plain %.2f us  graph backed %.2f us  "
                  "eager backed %.2f us  (%.1f G energies/s backed graph)" % (
                      nbins, fl is not None, p, q, e, nbins * 10 / q / 1e3))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
