"""Install the evidence of a tools/profile_round.sh run (gpurun_out/final/) under profiles/.

  python tools/install_profiles.py [--round r01] [--src gpurun_out/final]

Writes, for the round R:
  profiles/R_bench_<workload>.jsonl            the bench line of every workload (+ reference arm)
  profiles/R_final_ncu_<kernel>_summary.txt    key metrics of each ncu --set full capture, plus
                                               the executed FP64 instructions per energy point
                                               (from the SASS source page: predicated-on thread
                                               instructions of DFMA/DMUL/DADD / energy points)
  profiles/R_launches_default_cfg5.csv + _summary.txt   the default command's launch list
  profiles/ncu_traffic.json                    DRAM bytes per launch, copied by bench.py into
                                               roofline.traffic
Runs here (no GPU needed): ncu -i reads the .ncu-rep files.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

WORKLOADS = ["cfg5", "cfg4", "cfg3", "cfg2", "cfg1", "cfg4grid", "cfg3emu", "cfg5fit"]
# capture name -> (workload it was captured on, kernel label for ncu_traffic.json)
CAPTURES = {
    "batch": ("cfg5", "k_oscprob_batch"),
    "batch_pt": ("cfg4", "k_oscprob_batch_pt"),
    "batch_pt_mixed": ("cfg4_mixed", "k_oscprob_batch_pt<..., kMixed>"),
    "eval": ("cfg3", "k_oscprob_eval_tma"),
    "eval_ab": ("cfg3emu", "k_oscprob_eval_tma<PabCoef>"),
    "gl": ("cfg2", "k_gl_integrate_split"),
    "scan": ("cfg4grid", "k_scan_expand2"),
    "scan_setup": ("cfg4grid_setup", "k_scan_setup"),
    "batch_mixed": ("cfg5_mixed", "k_oscprob_batch<..., kMixed>"),
}


def last_json(path):
    for line in reversed(open(path).read().strip().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    raise ValueError("no JSON line in " + path)


def fp64_executed(rep):
    """Predicated-on thread-level DFMA + DMUL + DADD executed, from the source page."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if "Source" in r)
    i_src = hdr.index("Source")
    i_th = hdr.index("Predicated-On Thread Instructions Executed")
    tot = 0
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= i_th:
            continue
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        if op.split(".")[0] in ("DFMA", "DMUL", "DADD"):
            tot += int(float(r[i_th] or 0))
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out", "final"))
    a = ap.parse_args()
    R, src, prof = a.round, a.src, os.path.join(ROOT, "profiles")

    units = {}
    for w in WORKLOADS:
        p = os.path.join(src, "bench_%s.log" % w)
        if not os.path.exists(p):
            continue
        d = last_json(p)
        units[w] = d["config"].get("energy_points_per_step")
        with open(os.path.join(prof, "%s_bench_%s.jsonl" % (R, w)), "w") as f:
            f.write(json.dumps(d) + "\n")
        print("bench", w, "%.4g" % d["value"], d["unit"])
    for w in ("cfg5", "cfg4", "cfg3", "cfg2"):
        p = os.path.join(src, "bench_%s_mixed.log" % w)
        if os.path.exists(p):
            d = last_json(p)
            units[w + "_mixed"] = d["config"].get("energy_points_per_step")
            with open(os.path.join(prof, "%s_bench_%s_mixed.jsonl" % (R, w)), "w") as f:
                f.write(json.dumps(d) + "\n")
            print("bench", w, "mixed", "%.4g" % d["value"])
    p = os.path.join(src, "bench_reference.log")
    if os.path.exists(p):
        with open(os.path.join(prof, "%s_bench_reference_cfg5.jsonl" % R), "w") as f:
            f.write(json.dumps(last_json(p)) + "\n")

    tpath = os.path.join(prof, "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for name, (w, label) in CAPTURES.items():
        rep = os.path.join(src, "prof_%s.ncu-rep" % name)
        if not os.path.exists(rep):
            continue
        buf = io.StringIO()
        stdout, sys.stdout = sys.stdout, buf
        try:
            ncu_summary.main(rep, "final round-%s capture: %s (%s)" % (R[1:], label, w))
        finally:
            sys.stdout = stdout
        text = buf.getvalue()
        kv = {}
        for line in text.splitlines():
            parts = line.split("\t")
            if len(parts) >= 2:
                kv[parts[0]] = parts[1]
        fp = fp64_executed(rep)
        n = units.get(w)
        if n:
            text += "fp64_executed_per_energy_point\t%.2f\t(DFMA+DMUL+DADD predicated-on / %d)\n" % (
                fp / n, n)
        with open(os.path.join(prof, "%s_final_ncu_%s_summary.txt" % (R, name)), "w") as f:
            f.write(text)
        if w.endswith("_setup"):  # secondary kernel of a workload: summary only
            continue
        rd = float(kv.get("dram__bytes_read.sum", "0") or 0)
        wr = float(kv.get("dram__bytes_write.sum", "0") or 0)
        unit_r = text.split("dram__bytes_read.sum\t")[1].split("\n")[0].split("\t")[-1]
        unit_w = text.split("dram__bytes_write.sum\t")[1].split("\n")[0].split("\t")[-1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = int(rd * scale.get(unit_r, 1) + wr * scale.get(unit_w, 1))
        ent = traffic.get(w, {})
        if "algorithmic_bytes" not in ent and w.endswith("_mixed"):
            ent["algorithmic_bytes"] = traffic.get(w[:-len("_mixed")], {}).get("algorithmic_bytes")
        ent.update(kernel=label, bytes=b,
                   source="profiles/%s_final_ncu_%s_summary.txt" % (R, name))
        traffic[w] = ent
        print("ncu", name, "fp64/pt", "%.2f" % (fp / n) if n else "?", "traffic", b)
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1)

    lp = os.path.join(src, "launches_default.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(prof, "%s_launches_default_cfg5.csv" % R))
        rows = list(csv.reader(l for l in open(lp) if l.startswith('"')))
        h = rows[0]
        i_k, i_m, i_v = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
        i_u = h.index("Metric Unit")
        to_us = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
        agg = {}
        for r in rows[1:]:
            if r[i_m] != "gpu__time_duration.sum":
                continue
            v = float(r[i_v].replace(",", "")) * to_us.get(r[i_u], 1.0)
            n, t = agg.get(r[i_k], (0, 0.0))
            agg[r[i_k]] = (n + 1, t + v)
        # the live FP64 probe (build/probe_fp64, run by bench.py before its timed region) is
        # listed apart: it is neither the product nor part of a step
        probe = {k: v for k, v in agg.items() if k.startswith("k_dfma")}
        agg = {k: v for k, v in agg.items() if not k.startswith("k_dfma")}
        total = sum(t for _, t in agg.values()) or 1.0
        with open(os.path.join(prof, "%s_launches_default_cfg5_summary.txt" % R), "w") as f:
            f.write("# ncu launch list of `python bench.py --steps 20 --warmup 3` (default cfg5 "
                    "incl. e2e), B200 round %s\n" % R[1:])
            f.write("# gpu__time_duration per launch, cold-cache and serialised: compare SHARES, "
                    "not absolutes\n")
            for k, (n, t) in sorted(agg.items(), key=lambda z: -z[1][1]):
                f.write("%-60.60s n=%4d avg=%9.2fus share=%.3f\n" % (k, n, t / n, t / total))
            for k, (n, t) in probe.items():
                f.write("# not in the shares: %s n=%d avg=%.2fus (bench.py's FP64 peak probe, "
                        "before the timed region)\n" % (k[:40], n, t / n))
        print("launches", len(rows) - 1)


if __name__ == "__main__":
    main()
