"""Back-to-back gna_gl_integrate launches (20 per CUDA graph, L2 warm) for one library build:
the per-launch device time of the single-point GL kernel without the per-step event
granularity (≈ 2 µs) that quantises single-step timings.

usage: python tools/gl_b2b.py [--lib path] [--tag name]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--tag", default="base")
    ap.add_argument("--mode", default="fp64", choices=["fp64", "mixed", "ab", "eval"])
    ap.add_argument("--cases", default="100:5,100000:10,1000000:10", help="nbins:order,...")
    a = ap.parse_args()
    gna.load(a.lib)
    dev = torch.device("cuda", 0)
    for nbins, order in [tuple(int(v) for v in c.split(":")) for c in a.cases.split(",")]:
        edges = torch.tensor(synth.uniform_edges(nbins), dtype=torch.float64, device=dev)
        out = torch.empty(nbins, dtype=torch.float64, device=dev)
        if a.mode == "eval":  # nbins = number of energies (elementwise P_ee), order ignored
            E = torch.linspace(1.0, 10.0, nbins, dtype=torch.float64, device=dev)

            def call():
                gna.oscprob_eval(synth.CANONICAL, 52.5, E, out=out)
            order = 1
        elif a.mode == "ab":
            def call():
                gna.gl_integrate_ab(0, 1, synth.CANONICAL, 52.5, edges, order, out=out)
        else:
            def call():
                gna.gl_integrate(synth.CANONICAL, 52.5, edges, order, out=out,
                                 precision=a.mode)
        call()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            for _ in range(20):
                call()
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            g.replay()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (50 * 20)
        print(json.dumps(dict(tag=a.tag, mode=a.mode, nbins=nbins, order=order, us_per_launch=round(us, 3),
                              G_energies_per_s=round(nbins * order / us / 1e3, 1))), flush=True)


if __name__ == "__main__":
    main()
