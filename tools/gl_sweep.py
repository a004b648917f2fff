"""gna_gl_integrate step time vs nbins for one library build (tuning variants of the
single-point GL kernel).  Graph-replayed steps, L2 flushed before each, the stream kept
busy while the host enqueues (device time only); median of 100.  Prints one JSON line
per (order, nbins) with the bins' checksum so variants can be compared.

usage: python tools/gl_sweep.py [--lib path] [--tag name]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--tag", default="base")
    ap.add_argument("--sizes", default="100,10000,100000,1000000,10000000")
    ap.add_argument("--orders", default="5,10")
    a = ap.parse_args()
    gna.load(a.lib)
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for order in [int(x) for x in a.orders.split(",")]:
        for nbins in [int(x) for x in a.sizes.split(",")]:
            edges = torch.tensor(synth.uniform_edges(nbins), dtype=torch.float64, device=dev)
            out = torch.empty(nbins, dtype=torch.float64, device=dev)

            def call():
                gna.gl_integrate(synth.CANONICAL, 52.5, edges, order, out=out)
            call()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
                call()
            torch.cuda.current_stream().wait_stream(s)
            ts = []
            for _ in range(100):
                flush.zero_()
                torch.cuda._sleep(80_000)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                ts.append((e0, e1))
            torch.cuda.synchronize()
            us = float(np.median([x.elapsed_time(y) for x, y in ts]) * 1e3)
            ev = nbins * order
            print(json.dumps(dict(tag=a.tag, order=order, nbins=nbins, us=round(us, 3),
                                  G_per_s=round(ev / us / 1e3, 1),
                                  fp64_frac_36=round(ev * 36 / (us * 1e-6) / 18.61248e12, 3),
                                  checksum=float(out.sum()))), flush=True)


if __name__ == "__main__":
    main()
