"""cfg4grid scan: step time with and without the 256 MiB L2 flush, with and without the
spectra (chi^2 only: stage B does no stores), graph-replayed; splits the ~29 us step into
stage-A cold start, stage A, stage B."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_07682_b200 as gna  # noqa: E402
import synth  # noqa: E402


def main():
    c = synth.config("cfg4grid")
    f64 = dict(dtype=torch.float64, device="cuda")
    grid = {k: torch.tensor(v, **f64) for k, v in c["grid"].items()}
    edges, data = torch.tensor(c["edges"], **f64), torch.tensor(c["data"], **f64)
    nmix, nmass, nb = 100, 100, 1000
    sp = torch.empty((nmass, nmix, nb), **f64)
    x2 = torch.empty((nmass, nmix), **f64)
    ws = torch.empty(gna.oscprob_scan_workspace_size(nmix, nmass, nb) // 8 + 8, **f64)
    ws = ws[(-ws.data_ptr()) % 32 // 8:]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for spectra in (True, False):
        def step():
            gna.oscprob_scan(grid, c["L_km"], c["omega"], edges, 10, data=data,
                             spectra=sp if spectra else False, chi2=x2, workspace=ws)
        step()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        for fl in (True, False):
            ts = []
            for _ in range(60):
                if fl:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts = sorted(ts[10:])
            print("spectra=%s flush=%s: median %.2f us  min %.2f us" % (spectra, fl, ts[len(ts) // 2], ts[0]))


if __name__ == "__main__":
    main()
