"""Write-bandwidth ceiling for the scan's output (80 MB of spectra): torch fill / copy of an
80 MB fp64 tensor, L2 flushed before each, device time with CUDA events."""
import json
import torch

def t(fn, reps=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    best = 1e9
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best

n = 10_000_000
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
fill_ms = t(lambda: a.fill_(1.0))
copy_ms = t(lambda: b.copy_(a))
print(json.dumps({"bytes": n * 8, "fill_us": fill_ms * 1e3, "fill_TBps": n * 8 / fill_ms / 1e9,
                  "copy_us": copy_ms * 1e3, "copy_TBps_rw": 2 * n * 8 / copy_ms / 1e9}))
