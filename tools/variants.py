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
    "base": dict(),
    "nopdl": dict(GNA_PDL=0),
    "mx_ju1": dict(GNA_MIXED_JUNROLL=1),
    "mx_n10": dict(GNA_MIXED_N10=1),
    "mx_n5": dict(GNA_MIXED_N10=0, GNA_MIXED_JUNROLL=2),
    "mx_n10_ju2": dict(GNA_MIXED_JUNROLL=2),
    "mx_n10_ju1": dict(GNA_MIXED_N10=1, GNA_MIXED_JUNROLL=1),
    "mx_ju3": dict(GNA_MIXED_JUNROLL=3),
    "mx_ju4": dict(GNA_MIXED_JUNROLL=4),
    "mx_mb16": dict(GNA_BATCH_MINB=16, GNA_BATCH_PI_MINB=1),
    "mx_mb24": dict(GNA_BATCH_MINB=24, GNA_BATCH_PI_MINB=1),
    "d7_mb20": dict(GNA_BATCH_MINB=20, GNA_BATCH_PI_MINB=1),
    "d7_mb18": dict(GNA_BATCH_MINB=18, GNA_BATCH_PI_MINB=1),
    "d7_ju2": dict(GNA_BATCH_JUNROLL=2),
    "d7_ju3": dict(GNA_BATCH_JUNROLL=3),
    "d7_ju4": dict(GNA_BATCH_JUNROLL=4),
    "d7_ju8": dict(GNA_BATCH_JUNROLL=8),
    "d7_ju2_mb20": dict(GNA_BATCH_JUNROLL=2, GNA_BATCH_MINB=20, GNA_BATCH_PI_MINB=1),
    "d7_pim20": dict(GNA_BATCH_PI_MINB=20),
    "pi_m20": dict(GNA_BATCH_PI_MINB=20),
    "pi_m18": dict(GNA_BATCH_PI_MINB=18),
    "pi_m24": dict(GNA_BATCH_PI_MINB=24),
    "pi_nt3": dict(GNA_BATCH_PI_NT=1),
    "deg8": dict(GNA_SIN2_DEG=8),
    "mb20": dict(GNA_BATCH_MINB=20, GNA_BATCH_PI_MINB=1),
    "mb20_nt3": dict(GNA_BATCH_MINB=20, GNA_BATCH_PI_MINB=1, GNA_BATCH_PI_NT=1),
    "pi_nt3_m16": dict(GNA_BATCH_PI_NT=1, GNA_BATCH_PI_MINB=16),
    "pi_m20_w240": dict(GNA_BATCH_PI_MINB=20, GNA_BATCH_PPW_WORK=240),
    "gl_nosplit": dict(GNA_GL_SPLIT=0),
    "nopdl_single": dict(GNA_PDL_SINGLE=0),
    "nopdl_single_nosplit": dict(GNA_PDL_SINGLE=0, GNA_GL_SPLIT=0),
    "gl_nosplit_tb64": dict(GNA_GL_SPLIT=0, GNA_GL_TB_THREADS=64, GNA_GL_TB_MINB=8),
    "gl_split_bw2": dict(GNA_GL_SPLIT_BW=2, GNA_GL_SPLIT_MINB=4),
    "gl_split_mb21": dict(GNA_GL_SPLIT_MINB=21),
    "gl_split_mb16": dict(GNA_GL_SPLIT_MINB=16),
    "scan_a8": dict(GNA_SCAN_A=8),
    "scan_a16": dict(GNA_SCAN_A=16),
    "scan_a8_t256": dict(GNA_SCAN_A=8, GNA_SCAN_THREADS=256),
    "scan_a16_t256": dict(GNA_SCAN_A=16, GNA_SCAN_THREADS=256),
    "pt_b23_s1": dict(GNA_BATCH_PT_BPSM=23, GNA_BATCH_PT_SUB=1),
    "pt_b23_s2": dict(GNA_BATCH_PT_BPSM=23, GNA_BATCH_PT_SUB=2),
    "pt_b24_s4": dict(GNA_BATCH_PT_BPSM=24, GNA_BATCH_PT_SUB=4),
    "pt_noshared": dict(GNA_BATCH_PT_SHARED21=0),
    "pt_n10": dict(GNA_BATCH_PT_N10=1),
    "pt_n10_mb20": dict(GNA_BATCH_PT_N10=1, GNA_BATCH_PT_MINB=20),
    "pt_s1_sh": dict(GNA_BATCH_PT_SUB=1),
    "pt_s4_sh": dict(GNA_BATCH_PT_SUB=4),
    "pt_mb20": dict(GNA_BATCH_PT_MINB=20),
    "pt_mb16": dict(GNA_BATCH_PT_MINB=16),
    "pt_mb12": dict(GNA_BATCH_PT_MINB=12),
    "pt_n10_mb16": dict(GNA_BATCH_PT_N10=1, GNA_BATCH_PT_MINB=16),
    "pt_n10_mb12": dict(GNA_BATCH_PT_N10=1, GNA_BATCH_PT_MINB=12),
    "pt_s1": dict(GNA_BATCH_PT_SUB=1),
    "pt_s4": dict(GNA_BATCH_PT_SUB=4),
    "gl_split_bw4": dict(GNA_GL_SPLIT_BW=4, GNA_GL_SPLIT_MINB=2),
    "gl_split_bw2_mb5": dict(GNA_GL_SPLIT_BW=2, GNA_GL_SPLIT_MINB=5),
    "fit_batch": dict(GNA_FIT_SCAN=0),
    "host_staged": dict(GNA_HOST_DIRECT=0),
    "sign_lop": dict(GNA_SIGN_IMAD=0),
    "pt_eh": dict(GNA_BATCH_PT_EH=1),
    "b_ju1": dict(GNA_BATCH_JUNROLL=1),
    "term_rolled": dict(GNA_PROB_TERM_UNROLL=1),
    "scan_noord": dict(GNA_SCAN_ORD10=0),
    "scan_ord_mb6": dict(GNA_SCAN_SETUP_MINB=6),

    "b_ju3": dict(GNA_BATCH_JUNROLL=3),
    "b_ju4": dict(GNA_BATCH_JUNROLL=4),
    "pt_noord": dict(GNA_BATCH_PT_ORD10=0),
    "scan_a5": dict(GNA_SCAN_A=5),
    "scan_a2": dict(GNA_SCAN_A=2),
    "scan_a3": dict(GNA_SCAN_A=3),
    "scan_t64": dict(GNA_SCAN_THREADS=64),
    "scan_noexp2": dict(GNA_SCAN_EXPAND2=0),
    "nopdl_scan": dict(GNA_PDL_SCAN=0),
    "scan_mb1": dict(GNA_SCAN_SETUP_MINB=1),
    "fit_nofold": dict(GNA_FIT_FOLD=0),
    "scan_stcs": dict(GNA_SCAN_STREAMING_STORES=1),
    "scan_ch256": dict(GNA_SCAN_BIN_CHUNK=256, GNA_SCAN_CHUNK_BPSM=64),
    "scan_ch512": dict(GNA_SCAN_BIN_CHUNK=512, GNA_SCAN_CHUNK_BPSM=64),
    "scan_ch128": dict(GNA_SCAN_BIN_CHUNK=128, GNA_SCAN_CHUNK_BPSM=64),
    "scan_mb2": dict(GNA_SCAN_SETUP_MINB=2),
    "scan_mb4": dict(GNA_SCAN_SETUP_MINB=4),
    "ev_stg": dict(GNA_EVAL_BULK_STORE=0),
    "ev_bulk": dict(GNA_EVAL_BULK_STORE=1),
    "ev_bulk_s6m5": dict(GNA_EVAL_BULK_STORE=1, GNA_EVAL_STAGES=5, GNA_EVAL_MINB=5),
}


KERNELS = [r"k_oscprob_eval_tmaIN3gna7PeeCoef", r"k_oscprob_batchILi1ELi5ELi0ELb0E",
           r"k_oscprob_batch_piILi5ELi0ELi0ELb0E", r"k_oscprob_batch_piILi5ELi0ELi3ELb0E",
           r"k_oscprob_batchILi1ELi5ELi0ELb1E", r"k_oscprob_batch_piILi5ELi0ELi3ELb1E",
           r"k_oscprob_batchILi1ELi10ELi0ELb1E", r"k_gl_integrate_splitILi10EN3gna7PeeCoef",
           r"k_gl_integrate_tbILi10EN3gna7PeeCoef", r"k_scan_expand", r"k_scan_setupILi5ELi10E", r"k_oscprob_batch_ptILi5ELi3ELi0ELb0E"]


def main(names):
    outdir = os.path.join(ROOT, "build", "variants")
    os.makedirs(outdir, exist_ok=True)
    for name in names or VARIANTS:
        out = os.path.join(outdir, name + ".so")
        cmd_out = subprocess.run(
            [_build.nvcc(), *_build.NVCC_FLAGS, *["-D%s=%s" % kv for kv in VARIANTS[name].items()],
             "-Xptxas", "-v", "-o", out, os.path.join(_build.CSRC, "gna_b200.cu")],
            capture_output=True, text=True, check=True).stderr
        for kern in KERNELS:
            m = re.search(r"Compiling entry function '[^']*" + kern + r"[^']*' for 'sm_100a'\n"
                          r"[^\n]*\n\s*\d+ bytes stack frame, (\d+) bytes spill stores[^\n]*\n"
                          r"[^\n]*Used (\d+) registers", cmd_out)
            print(name, kern, "regs", m.group(2) if m else "?", "spills", m.group(1) if m else "?")


if __name__ == "__main__":
    main(sys.argv[1:])
