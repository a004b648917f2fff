"""Build tuning variants of libgna_b200.so (compile-time knobs of the batch kernel) and
print their register/spill counts.  Measured with bench.py --lib on the GPU box."""
from __future__ import annotations

import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1804_07682_b200 import _build  # noqa: E402

VARIANTS = {
    "ev_stg": dict(GNA_EVAL_BULK_STORE=0),
    "ev_bulk": dict(GNA_EVAL_BULK_STORE=1),
    "ev_bulk_s6m5": dict(GNA_EVAL_BULK_STORE=1, GNA_EVAL_STAGES=5, GNA_EVAL_MINB=5),
}


def main(names):
    outdir = os.path.join(ROOT, "build", "variants")
    os.makedirs(outdir, exist_ok=True)
    for name in names or VARIANTS:
        out = os.path.join(outdir, name + ".so")
        cmd_out = subprocess.run(
            [_build.nvcc(), *_build.NVCC_FLAGS, *["-D%s=%s" % kv for kv in VARIANTS[name].items()],
             "-Xptxas", "-v", "-o", out, os.path.join(_build.CSRC, "gna_b200.cu")],
            capture_output=True, text=True, check=True).stderr
        m = re.search(r"k_oscprob_eval_tmaIN3gna7PeeCoefEEvT_PKdPdl.*?\n.*?(\d+) bytes spill stores.*?\n.*?Used (\d+) registers",
                      cmd_out, re.S)
        print(name, "regs", m.group(2) if m else "?", "spills", m.group(1) if m else "?")


if __name__ == "__main__":
    main(sys.argv[1:])
