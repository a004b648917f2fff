#!/usr/bin/env python
"""Benchmark of the fused fp64 P_ee + Gauss-Legendre hot path on B200 (BASELINE.json metric:
"energy points/sec (fp64 P_ee+GL) at 1/2/4/8 B200; % of HBM/FP64 roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5|cfg4|cfg2|cfg3]
                    [--impl ours|reference]

A step is one pass of the whole hot path over one batch:
default workload cfg5 = 8 baselines x 1000 parameter points x 1e5 energies
(1e4 bins x GL10), spectra + chi^2 per point, points sharded over ranks and the
spectra/chi^2 gathered with NCCL (N > 1).  An "energy point" is one (parameter
point x baseline x GL node) evaluation of P_ee.  Timing: CUDA events on the
launching stream around each step, L2 flushed (256 MiB write) between steps,
barrier + synchronize on both sides, max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "energy points/sec (fp64 P_ee+GL)"
UNIT = "energy points/s"

# Algorithmic FP64-pipe work per energy point: three sin^2
# terms x (degree + 5) FP64 instructions (rint 2, reduced argument 1, square 1, minimax
# Horner `degree`, weighted accumulate 1) = 36 at the default degree 7 (39 at degree 8);
# the degree is read from the loaded library (gna_sin2_poly_degree).  Per-node work
# (reciprocal, node position, GL weight) is amortised over baselines and not counted.
def fp64_ops_per_eval(deg):
    return 3 * (deg + 5)


# mixed tier (NEXT-3): instructions per sin^2 term (3 FP64 + F2F + 4 per chain of a packed
# FFMA2 pair), DESIGN.md §6.8
MIXED_INSTR_PER_TERM = 8
# elementwise mode adds the reciprocal of each energy: MUFU.RCP64H (1/3-rate, 3 slots)
# + 3 DFMA (tools/probe_rcp.cu)
RCP_OPS = 6
FP64_LANES_PER_SM = 64        # measured: tools/probe_fp64.cu, profiles/r01_probe_fp64.jsonl
SM_COUNT = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="cfg5", choices=["cfg5", "cfg4", "cfg3", "cfg2", "cfg1",
                                                            "cfg4grid", "cfg3emu", "cfg5fit"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chunks", type=int, default=0, help="gather pipeline chunks (0 = auto)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--lib", default=None, help="alternative libgna_b200.so (tuning variants)")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "mixed"],
                    help="fp64 (default, 1e-12 / 1e-11) or the NEXT-3 mixed tier (GNA_PREC_MIXED: "
                         "fp64 phases, fp32 polynomial; 1e-6 on P, 1e-5 on bins), cfg1-cfg5")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo only to exercise the N>1 code path on "
                         "one GPU, with GNA_BENCH_SAME_DEVICE=1; not for measurements)")
    ap.add_argument("--gather", default="auto", choices=["auto", "nccl", "fused"],
                    help="N>1 exchange: fused kernel-epilogue stores (validated) or NCCL all-gather")
    ap.add_argument("--fused-probe", action="store_true",
                    help=argparse.SUPPRESS)  # internal: the isolated start-up check (N > 1)
    ap.add_argument("--probe-timeout", type=float, default=240.0,
                    help="seconds allowed for the isolated fused-gather start-up check")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each step as a CUDA graph (auto: when N == 1)")
    a = ap.parse_args()
    if a.precision == "mixed" and (a.workload not in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")
                                   or a.impl != "ours"):
        ap.error("--precision mixed applies to cfg1-cfg5 of --impl ours")
    return a


# ----------------------------------------------------------------------------- workloads
FIT_ITERS = 50


def workload(name: str) -> dict:
    c = synth.config({"cfg3emu": "cfg3", "cfg5fit": "cfg5"}.get(name, name))
    if name == "cfg5fit":
        nb = c["edges"].size - 1
        c["evals"] = FIT_ITERS * 81 * c["L_km"].size * nb * c["order"]
        c["bins_total"] = FIT_ITERS * 81 * nb
        c["desc"] = dict(workload="cfg5fit: on-GPU chi^2 pattern-search fit (NEXT-4), %d "
                         "iterations x 81 candidate points on the cfg5 geometry (8 baselines x "
                         "%d energies), one CUDA graph per fit; the 3^4 stencil is evaluated as "
                         "a 9 x 9 separable scan (NEXT-1), so energy points = candidate x energy "
                         "evaluations delivered" % (FIT_ITERS, nb * c["order"]),
                         points=81 * FIT_ITERS, baselines=int(c["L_km"].size), bins=nb,
                         order=c["order"])
        c["name"] = name
        return c
    if name == "cfg3emu":
        c["params"] = dict(c["params"], delta_cp=1.2)
    if name in ("cfg4", "cfg5"):
        P = c["points"]["theta12"].size
        nb = c["edges"].size - 1
        c["evals"] = P * c["L_km"].size * nb * c["order"]
        c["bins_total"] = P * nb
        c["desc"] = dict(workload="%s: %d baselines x %d parameter points x %d energies "
                         "(%d bins x GL%d), spectra + chi2 per point" % (
                             name, c["L_km"].size, P, nb * c["order"], nb, c["order"]),
                         points=P, baselines=int(c["L_km"].size), bins=nb, order=c["order"])
    elif name == "cfg3emu":
        c["evals"] = c["n"]
        c["bins_total"] = 0
        c["desc"] = dict(workload="cfg3emu: NEXT-2 appearance channel nu_e -> nu_mu (general "
                         "formula P:633-636, delta_cp = 1.2, theta23 = 0.785) over %d energies "
                         "streamed from HBM" % c["n"], points=1, energies=c["n"])
    elif name == "cfg4grid":
        nmix, nmass = c["grid"]["theta12"].size, c["grid"]["dm2_21"].size
        nb = c["edges"].size - 1
        c["evals"] = nmix * nmass * c["L_km"].size * nb * c["order"]
        c["bins_total"] = nmix * nmass * nb
        c["points"] = synth.expand_grid(c["grid"])
        c["desc"] = dict(workload="cfg4grid: %d x %d (theta13 x dm2_31) grid x %d energies "
                         "(%d bins x GL%d) via the separable scan (NEXT-1); energy points = "
                         "point x energy evaluations delivered" % (nmix, nmass, nb * c["order"],
                                                                  nb, c["order"]),
                         points=nmix * nmass, baselines=int(c["L_km"].size), bins=nb,
                         order=c["order"])
    elif name == "cfg1":
        nb = c["edges"].size - 1
        c["evals"] = c["E"].size + nb * c["order"]
        c["bins_total"] = nb
        c["desc"] = dict(workload="cfg1: 1 parameter point, %d energies (eval) + %d bins x GL%d "
                         "(DESIGN.md R11)" % (c["E"].size, nb, c["order"]), points=1, bins=nb,
                         order=c["order"])
    elif name == "cfg2":
        nb = c["edges"].size - 1
        c["evals"] = nb * c["order"]
        c["bins_total"] = nb
        c["desc"] = dict(workload="cfg2: 1 parameter point, %d energies (%d bins x GL%d)" % (
            nb * c["order"], nb, c["order"]), points=1, bins=nb, order=c["order"])
    else:
        c["evals"] = c["n"]
        c["bins_total"] = 0
        c["desc"] = dict(workload="cfg3: 1 parameter point, %d energies streamed from HBM "
                         "(elementwise P_ee)" % c["n"], points=1, energies=c["n"])
    return c


class KernelTimer:
    """CUDA events around one library call on the launching (current) stream."""
    enabled = True

    def __init__(self, sink):
        self.sink = sink

    def __enter__(self):
        if KernelTimer.enabled:
            import torch
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
            self.e0.record()
        return self

    def __exit__(self, *a):
        if KernelTimer.enabled:
            self.e1.record()
            self.sink.append((self.e0, self.e1))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The oracle (plain C, fp64) on this host's cores: the base contract's reference arm."""
    if rank != 0:
        return
    import oracle
    c = workload(args.workload)
    nt = oracle.max_threads()
    times, units = [], []

    def one_step():
        t0 = time.perf_counter()
        if args.workload in ("cfg4", "cfg5", "cfg4grid"):
            idx = np.arange(ns)
            sub = synth.subset_points(c["points"], idx)
            oracle.batch(sub, c["L_km"], c["omega"], c["edges"], c["order"], data=c["data"],
                         nthreads=nt)
            u = ns * c["L_km"].size * (c["edges"].size - 1) * c["order"]
        elif args.workload == "cfg2":
            e = c["edges"][:ns + 1]
            oracle.gl_integrate(c["params"], c["L_km"], e, c["order"], nthreads=nt)
            u = ns * c["order"]
        elif args.workload == "cfg1":
            oracle.prob_array(c["params"], c["L_km"], c["E"], nthreads=nt)
            oracle.gl_integrate(c["params"], c["L_km"], c["edges"], c["order"], nthreads=nt)
            u = c["evals"]
        else:
            E = np.linspace(c["lo"], c["hi"], ns)
            ab = (0, 1) if args.workload == "cfg3emu" else (0, 0)
            oracle.prob_array(c["params"], c["L_km"], E, alpha=ab[0], beta=ab[1], nthreads=nt)
            u = ns
        return time.perf_counter() - t0, u

    # size each step to ~ (cpu_seconds / (steps+warmup)), bounded by the workload
    ns = nt if args.workload in ("cfg4", "cfg5", "cfg4grid") else 10_000
    dt, u = one_step()
    rate = u / max(dt, 1e-9)
    per_step = max(0.05, min(args.cpu_seconds, 120.0) / max(args.steps + args.warmup, 1))
    full = {"cfg4": 10_000, "cfg5": 1000, "cfg2": 100_000, "cfg3": 100_000_000,
            "cfg1": 100, "cfg4grid": 10_000, "cfg3emu": 100_000_000}[args.workload]
    unit_per = u / ns
    ns = int(max(1, min(full, rate * per_step / unit_per)))
    for _ in range(args.warmup):
        one_step()
    for _ in range(args.steps):
        dt, u = one_step()
        times.append(dt)
        units.append(u)
    value = sum(units) / sum(times)
    sample = "%d of %d %s per step (%s), oracle general complex formula, %d OpenMP threads" % (
        ns, full, "parameter points" if args.workload in ("cfg4", "cfg5", "cfg4grid") else
        ("bins" if args.workload == "cfg2" else "energies"), args.workload, nt)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            # the same label as this workload's own arm (the batch configs split a fixed set
            # of parameter points over the ranks)
            "scaling": "strong" if args.workload in ("cfg4", "cfg5") else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": c["desc"],
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nt, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(c, name, seconds):
    """The oracle as it stands, on a bounded sample of the same workload (rank 0, N=1)."""
    import oracle
    nt = oracle.max_threads()
    if name in ("cfg4", "cfg5", "cfg4grid"):
        per_point = c["L_km"].size * (c["edges"].size - 1) * c["order"]
        P = c["points"]["theta12"].size
        n = min(P, nt)  # calibrate with one point per thread (the oracle threads over points)
        t0 = time.perf_counter()
        oracle.batch(synth.subset_points(c["points"], np.arange(n)), c["L_km"], c["omega"],
                     c["edges"], c["order"], data=c["data"], nthreads=nt)
        dt = time.perf_counter() - t0
        n = int(max(1, min(P, nt * round(seconds / max(dt, 1e-9)))))
        idx = np.arange(n)
        t0 = time.perf_counter()
        oracle.batch(synth.subset_points(c["points"], idx), c["L_km"], c["omega"], c["edges"],
                     c["order"], data=c["data"], nthreads=nt)
        dt = time.perf_counter() - t0
        units = n * per_point
        sample = "first %d of %d parameter points of %s (all baselines, bins, nodes)" % (n, P, name)
    elif name == "cfg2":
        t0 = time.perf_counter()
        oracle.gl_integrate(c["params"], c["L_km"], c["edges"], c["order"], nthreads=nt)
        dt = time.perf_counter() - t0
        units = (c["edges"].size - 1) * c["order"]
        sample = "full cfg2"
    elif name == "cfg1":
        reps = 200
        t0 = time.perf_counter()
        for _ in range(reps):
            oracle.prob_array(c["params"], c["L_km"], c["E"], nthreads=1)
            oracle.gl_integrate(c["params"], c["L_km"], c["edges"], c["order"], nthreads=1)
        dt = time.perf_counter() - t0
        units = c["evals"] * reps
        nt = 1
        sample = "full cfg1 x %d repetitions, 1 thread" % reps
    else:
        n = 20_000_000
        E = np.linspace(c["lo"], c["hi"], n)
        ab = (0, 1) if name == "cfg3emu" else (0, 0)
        t0 = time.perf_counter()
        oracle.prob_array(c["params"], c["L_km"], E, alpha=ab[0], beta=ab[1], nthreads=nt)
        dt = time.perf_counter() - t0
        units = n
        sample = "%d of %d energies of cfg3 (same linspace range)" % (n, c["n"])
    out = {"value": units / dt, "unit": UNIT, "cores": nt, "kind": "oracle",
           "sample": sample, "seconds": dt, "cpu_model": _cpu_model()}
    # the oracle at 1 thread as well as on all cores (bounded sample)
    if name in ("cfg4", "cfg5", "cfg4grid"):
        t0 = time.perf_counter()
        oracle.batch(synth.subset_points(c["points"], np.arange(1)), c["L_km"], c["omega"],
                     c["edges"], c["order"], data=c["data"], nthreads=1)
        dt1 = time.perf_counter() - t0
        out["single_thread"] = {"value": per_point / dt1, "sample": "1 parameter point of %s" % name}
    elif name in ("cfg2", "cfg3", "cfg3emu"):
        E = np.linspace(1.0, 10.0, 2_000_000)
        ab = (0, 1) if name == "cfg3emu" else (0, 0)
        t0 = time.perf_counter()
        oracle.prob_array(c["params"], c["L_km"], E, alpha=ab[0], beta=ab[1], nthreads=1)
        dt1 = time.perf_counter() - t0
        out["single_thread"] = {"value": E.size / dt1, "sample": "2e6 energies, 1 thread"}
    return out


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def auto_chunks(npoints: int, world: int, evals_per_point: int) -> int:
    """Gather pipeline depth for N > 1: up to 4 chunks, each >= ~2.5e7 energy
    points of the rank's shard (>= ~60 us of kernel, several waves), so that all but the last
    chunk's all-gather hides under the next chunk's kernel; chunks after the first reuse the
    node tables (GNA_WS_TABLES_VALID), so a chunk costs only its own points."""
    if world == 1:
        return 1
    per_rank = -(-npoints // world) * evals_per_point
    return int(max(1, min(4, round(per_rank / 2.5e7))))


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def isolated_fused_probe(args, world, rank, dist):
    """Rank 0 runs the fused-epilogue start-up check (bench.py --fused-probe) as a separate
    N-rank torch.distributed.run job with a hard timeout, while the other ranks wait on the
    store (CPU side, no GPU work).  Returns {"ok": bool, "mode"/"why": str}."""
    store = dist.distributed_c10d._get_default_store()
    key = "gna_fused_probe"
    if rank == 0:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
               str(world), "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.abspath(__file__), "--fused-probe", "--gpus", str(world), "--workload",
               args.workload, "--precision", args.precision]
        env = {k: v for k, v in os.environ.items() if not k.startswith("TORCHELASTIC")
               and k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE",
                             "GROUP_RANK", "ROLE_RANK", "ROLE_WORLD_SIZE", "MASTER_ADDR",
                             "MASTER_PORT", "TORCHELASTIC_RUN_ID")}
        res = {"ok": False, "why": "probe did not run"}
        t0 = time.time()
        try:
            # own session: on a timeout the launcher AND its worker ranks (which may be stuck
            # in a device-side wait) are killed as one process group, so none keeps a GPU busy
            proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                    text=True, env=env, start_new_session=True)
            try:
                so, se = proc.communicate(timeout=args.probe_timeout)
                ok_lines = [l for l in so.splitlines() if l.startswith("FUSED_PROBE_OK")]
                if proc.returncode == 0 and ok_lines:
                    res = {"ok": True, "mode": ok_lines[-1].split()[1]}
                else:
                    tail = (so + se).strip().splitlines()[-1:] or ["no output"]
                    res = {"ok": False, "why": "probe rc=%d: %s" % (proc.returncode,
                                                                    tail[0][:160])}
            except subprocess.TimeoutExpired:
                import signal
                try:
                    os.killpg(proc.pid, signal.SIGKILL)
                except OSError:
                    pass
                proc.communicate()
                res = {"ok": False, "why": "probe timed out after %.0f s" % args.probe_timeout}
        except OSError as exc:
            res = {"ok": False, "why": "probe failed to start: %s" % exc}
        res["seconds"] = round(time.time() - t0, 1)
        store.set(key, json.dumps(res))
        return res
    store.wait([key], __import__("datetime").timedelta(seconds=args.probe_timeout + 120))
    return json.loads(store.get(key))


def fused_probe_main(args):
    """--fused-probe (one rank of the isolated check): build the symmetric-memory window, run
    the batch with the gather fused into its epilogue on a small slice of the workload (every
    baseline, bin and node; 8 points per rank) and compare the gathered result bit for bit
    with one local batch over the same points.  Prints FUSED_PROBE_OK <mode> on rank 0."""
    import torch
    import torch.distributed as dist

    import paper_1804_07682_b200 as gna
    from paper_1804_07682_b200 import dist as gdist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    try:
        gna.load(args.lib)
        c = workload(args.workload)
        f64 = dict(dtype=torch.float64, device=dev)
        P = min(c["points"]["theta12"].size, 8 * world)
        nb = c["edges"].size - 1
        allp = {k: torch.tensor(v[:P], **f64) for k, v in c["points"].items()}
        edges, data = torch.tensor(c["edges"], **f64), torch.tensor(c["data"], **f64)
        fg = gdist.FusedGather(P, nb, dev)
        sp_ptr, x2_ptr, flags = fg.out_ptrs()
        if args.precision == "mixed":
            flags |= gna.GNA_PREC_MIXED
        mine = {k: v[fg.lo:fg.hi].contiguous() for k, v in allp.items()}
        fg.spectra.fill_(float("nan"))
        fg.chi2.fill_(float("nan"))
        fg.barrier(timeout_ms=20_000)
        gna.oscprob_batch_ex(mine, c["L_km"], c["omega"], edges, c["order"], sp_ptr, x2_ptr,
                             flags, data=data)
        fg.barrier(timeout_ms=20_000)
        torch.cuda.synchronize()
        ok = torch.ones(1, device=dev)
        if rank == 0 or fg.multicast:
            sp, x2 = gna.oscprob_batch(allp, c["L_km"], c["omega"], edges, c["order"], data=data,
                                       precision=args.precision)
            ok.fill_(1.0 if torch.equal(fg.spectra, sp) and torch.equal(fg.chi2, x2) else 0.0)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        torch.cuda.synchronize()
        if float(ok) != 1.0:
            print("fused probe: gathered result differs from the local batch", file=sys.stderr)
            return 3
        if rank == 0:
            print("FUSED_PROBE_OK %s" % ("multicast" if fg.multicast else "peer-to-root"),
                  flush=True)
        return 0
    finally:
        dist.destroy_process_group()


def relaunch(n: int) -> int:
    """Re-run this command as n ranks under torch.distributed.run on 127.0.0.1 (one process
    per GPU); returns the launcher's exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # N > 1 without a launcher: start the N ranks ourselves (one process per GPU, the
        # driver's own torchrun command line); rank 0 prints the JSON line
        sys.exit(relaunch(args.gpus))
    if args.fused_probe:
        sys.exit(fused_probe_main(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:  # the launcher's world size is what runs
        print("bench.py: --gpus %d under WORLD_SIZE=%d; using %d ranks" % (args.gpus, world, world),
              file=sys.stderr)
    if args.impl == "reference":
        if args.workload == "cfg5fit":
            args.workload = "cfg5"  # the oracle has no fit loop: time its batch evaluation
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_1804_07682_b200 as gna
    from paper_1804_07682_b200 import dist as gdist

    if os.environ.get("GNA_BENCH_SAME_DEVICE") == "1":
        local = 0  # code-path test: every rank on GPU 0 (independent kernels, no device spin)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # the fused epilogue (NEXT-4): tried by default at N > 1; `--gather fused` also runs it on
    # one GPU, writing through a one-rank symmetric-memory window (the N > 1 code path,
    # probe and bitwise check included, on hardware that has only one GPU)
    batch = args.workload in ("cfg4", "cfg5")
    want_fused = batch and (args.gather == "fused" or (args.gather == "auto" and world > 1))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
            want_fused = False  # the fused epilogue needs one GPU per rank
    elif want_fused:
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % _free_port(),
                                rank=0, world_size=1, device_id=dev)
    gna.load(args.lib)
    c = workload(args.workload)
    f64 = dict(dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # ---------------- setup (configuration stage): upload once, allocate once
    if args.workload in ("cfg4", "cfg5"):
        P = c["points"]["theta12"].size
        nb = c["edges"].size - 1
        chunks = args.chunks or auto_chunks(P, world, c["L_km"].size * nb * c["order"])
        sb = gdist.ShardedBatch(P, nb, world, rank, chunks=chunks).allocate(dev)
        lo, hi = sb.lo, sb.hi
        pts = {k: torch.tensor(v[lo:hi], **f64) for k, v in c["points"].items()}
        edges = torch.tensor(c["edges"], **f64)
        data = torch.tensor(c["data"], **f64)
        ws = torch.empty(max(gna.oscprob_batch_workspace_size(
            max(hi - lo, 1), c["L_km"].size, nb, c["order"]) // 8, 2), **f64)
        comm = torch.cuda.Stream(device=dev) if world > 1 else None
        L, om = c["L_km"], c["omega"]
        kern_ev = []

        def compute(vlo, vhi, sp_rows, x2_rows):
            # chunks after a step's first reuse its node tables (1/E, h w) in `ws`
            sub = {k: v[vlo:vhi] for k, v in pts.items()}
            with KernelTimer(kern_ev):
                gna.oscprob_batch(sub, L, om, edges, c["order"], data=data, spectra=sp_rows,
                                  chi2=x2_rows, workspace=ws, precision=args.precision,
                                  tables_valid=vlo > 0)

        def step():
            sb.step(compute, comm_stream=comm)

        gather_mode = "none" if world == 1 else "%s all_gather (%d chunk%s)" % (
            args.backend, len(sb.cb), "s" if len(sb.cb) > 1 else "")
        fused_fg = None
        probe = None
        if want_fused:
            # the fused epilogue runs here only after it has passed the same check in an
            # isolated process group under a hard timeout (a stall or a fault there cannot
            # take this run down with it)
            probe = isolated_fused_probe(args, world, rank, dist)
            if not probe["ok"]:
                gather_mode += " (fused epilogue not used: %s)" % probe["why"]
        if want_fused and probe["ok"]:
            # NEXT-4: gather fused into the kernel epilogue through symmetric memory;
            # every rank must have built it before any rank runs it, and it is validated
            # bitwise against the NCCL gather before it is used
            fg, err = None, ""
            try:
                fg = gdist.FusedGather(P, nb, dev)
            except Exception as exc:  # noqa: BLE001 — reported in config.gather
                err = str(exc).splitlines()[0][:120] if str(exc) else type(exc).__name__
            built = torch.tensor([1.0 if fg is not None else 0.0], device=dev)
            dist.all_reduce(built, op=dist.ReduceOp.MIN)
            if float(built) == 1.0:
                sp_ptr, x2_ptr, fflags = fg.out_ptrs()
                if args.precision == "mixed":
                    fflags |= gna.GNA_PREC_MIXED

                def step_fused():
                    with KernelTimer(kern_ev):
                        gna.oscprob_batch_ex(pts, L, om, edges, c["order"], sp_ptr, x2_ptr,
                                             fflags, data=data, workspace=ws)
                    fg.barrier()

                step()
                s_ref, x_ref = sb.gathered()
                step_fused()
                torch.cuda.synchronize()
                ok = torch.ones(1, device=dev)
                if rank == 0 or fg.multicast:
                    same = bool(torch.equal(fg.spectra, s_ref)) and bool(torch.equal(fg.chi2, x_ref))
                    ok.fill_(1.0 if same else 0.0)
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
                if float(ok) == 1.0:
                    step = step_fused  # noqa: F811
                    fused_fg = fg
                    gather_mode = "fused-epilogue-" + ("multicast" if fg.multicast else "peer-to-root")
                else:
                    gather_mode = "nccl (fused epilogue failed bitwise validation)"
                del s_ref, x_ref
            else:
                gather_mode = "nccl (fused epilogue unavailable on some rank%s)" % (
                    ": " + err if err else "")
            kern_ev.clear()

        units_per_rank = (hi - lo) * L.size * nb * c["order"]
        calls_per_step = (1 if gather_mode.startswith("fused") else
                          len([1 for a, b in sb.cb if min(b, sb.count) > min(a, sb.count)]))
        scaling = "strong"
    elif args.workload == "cfg4grid":
        grid = {k: torch.tensor(v, **f64) for k, v in c["grid"].items()}
        edges = torch.tensor(c["edges"], **f64)
        data = torch.tensor(c["data"], **f64)
        nmix, nmass = c["grid"]["theta12"].size, c["grid"]["dm2_21"].size
        nb = c["edges"].size - 1
        sp_out = torch.empty((nmass, nmix, nb), **f64)
        x2_out = torch.empty((nmass, nmix), **f64)
        wsz = gna.oscprob_scan_workspace_size(nmix, nmass, nb) // 8 + 8
        ws_raw = torch.empty(wsz, **f64)
        ws = ws_raw[(-ws_raw.data_ptr()) % 32 // 8:]
        kern_ev = []

        def step():
            with KernelTimer(kern_ev):
                gna.oscprob_scan(grid, c["L_km"], c["omega"], edges, c["order"], data=data,
                                 spectra=sp_out, chi2=x2_out, workspace=ws)

        units_per_rank = c["evals"]
        calls_per_step = 1
        scaling = "weak"  # replicas only (one grid per GPU)
    elif args.workload == "cfg1":
        edges = torch.tensor(c["edges"], **f64)
        out = torch.empty(c["edges"].size - 1, **f64)
        E1 = torch.tensor(c["E"], **f64)
        P1 = torch.empty_like(E1)
        kern_ev = []

        def step():
            with KernelTimer(kern_ev):
                gna.oscprob_eval(c["params"], c["L_km"], E1, out=P1, precision=args.precision)
                gna.gl_integrate(c["params"], c["L_km"], edges, c["order"], out=out,
                                 precision=args.precision)

        units_per_rank = c["evals"]
        calls_per_step = 1
        scaling = "weak"  # replicas only
    elif args.workload == "cfg2":
        edges = torch.tensor(c["edges"], **f64)
        out = torch.empty(c["edges"].size - 1, **f64)
        kern_ev = []

        def step():
            with KernelTimer(kern_ev):
                gna.gl_integrate(c["params"], c["L_km"], edges, c["order"], out=out,
                                 precision=args.precision)

        units_per_rank = c["evals"]
        calls_per_step = 1
        scaling = "weak"  # replicas only
    elif args.workload == "cfg5fit":
        edges = torch.tensor(c["edges"], **f64)
        data = torch.tensor(c["data"], **f64)
        nb = c["edges"].size - 1
        start = np.array([0.5838, 0.1496, 7.53e-5, 2.52e-3, 0.01, 0.005, 2e-6, 5e-5])
        state = torch.tensor(start, **f64)
        state0 = torch.tensor(start, **f64)
        hist = torch.empty(FIT_ITERS, **f64)
        ws = torch.empty(gna.fit_workspace_size(c["L_km"].size, nb, c["order"]) // 8 + 2, **f64)
        kern_ev = []

        def step():
            state.copy_(state0)
            with KernelTimer(kern_ev):
                gna.fit_pattern_search(state, c["L_km"], c["omega"], edges, c["order"], data,
                                       FIT_ITERS, hist=hist, workspace=ws)

        units_per_rank = c["evals"]
        calls_per_step = FIT_ITERS
        scaling = "weak"  # replicas only (one fit per GPU)
    elif args.workload == "cfg3emu":
        E = torch.linspace(c["lo"], c["hi"], c["n"], **f64)
        out = torch.empty_like(E)
        kern_ev = []

        def step():
            with KernelTimer(kern_ev):
                gna.oscprob_eval_ab(0, 1, c["params"], c["L_km"], E, out=out)

        units_per_rank = c["evals"]
        calls_per_step = 1
        scaling = "weak"  # replicas only
    else:
        E = torch.linspace(c["lo"], c["hi"], c["n"], **f64)
        out = torch.empty_like(E)
        kern_ev = []

        def step():
            with KernelTimer(kern_ev):
                gna.oscprob_eval(c["params"], c["L_km"], E, out=out, precision=args.precision)

        units_per_rank = c["evals"]
        calls_per_step = 1
        scaling = "weak"  # replicas only

    def barrier():
        if world > 1:
            _barrier(dist, args, local)

    # live FP64 denominator check: DFMA issue rate of this GPU (outside the timed region)
    fp64_probe = run_fp64_probe(local) if rank == 0 else None

    # ---------------- warm-up
    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    kern_ev.clear()

    # ---------------- CUDA graph of the step (the repeated-evaluation loop of a fit):
    # one graph launch per step instead of per-call host work.  NCCL steps stay eager.
    # CUDA graph of the whole step.  At N > 1 the NCCL path is captured too (its chunk kernels
    # and all-gathers on the communication stream): eagerly, enqueueing one chunk costs ~100 us
    # of host time (34 us per batch call, 31 us per all-gather; tools/host_overhead_probe.py),
    # which at G = 8 would exceed the chunk's GPU time.  Every rank must capture successfully,
    # else all run eagerly.  The fused epilogue (symmetric-memory barrier) and gloo stay eager.
    fused_used = args.workload in ("cfg4", "cfg5") and fused_fg is not None
    use_graph = args.graph == "on" or (args.graph == "auto" and not fused_used and
                                       (world == 1 or args.backend == "nccl"))
    launches_per_step = None
    graph_note = None
    if use_graph:
        KernelTimer.enabled = False
        g = torch.cuda.CUDAGraph()
        n0 = gna.launch_count()
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(torch.cuda.current_stream())
        captured = True
        try:
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    step()
        except Exception as exc:  # noqa: BLE001 — reported; the run continues eagerly
            captured = False
            graph_note = "capture failed, eager steps: %s" % (str(exc).splitlines()[0][:120]
                                                            if str(exc) else type(exc).__name__)
        torch.cuda.current_stream().wait_stream(cap)
        torch.cuda.synchronize()
        if world > 1:
            agree = torch.tensor([1.0 if captured else 0.0], device=dev)
            dist.all_reduce(agree, op=dist.ReduceOp.MIN)
            if float(agree) != 1.0 and captured:
                graph_note = "capture failed on another rank, eager steps"
            captured = float(agree) == 1.0
        use_graph = captured
        if not captured:
            KernelTimer.enabled = True
            kern_ev.clear()
    if use_graph:
        launches_per_step = gna.launch_count() - n0
        eager_step = step

        def step():  # noqa: F811
            g.replay()
        for _ in range(3):
            step()
        torch.cuda.synchronize()

    # ---------------- timed region: K steps, per-step events, L2 flushed between steps
    barrier()
    torch.cuda.synchronize()
    n_launch0 = gna.launch_count()
    evs = []
    with ClockSampler(_smi_index(local)) as clk:
        for _ in range(args.steps):
            flush.zero_()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            step()
            s1.record()
            evs.append((s0, s1))
        torch.cuda.synchronize()
    barrier()
    launches = gna.launch_count() - n_launch0
    step_times = sorted(a.elapsed_time(b) for a, b in evs)
    total_ms = sum(step_times)
    if use_graph:
        # kernels replayed from the graph: count = per-step launches captured x steps;
        # the step is the dominant kernel plus two us-scale helpers -> step time bounds it
        launches = launches_per_step * args.steps
        kern_ms = [a.elapsed_time(b) for a, b in evs]
    else:
        kern_ms = [a.elapsed_time(b) for a, b in kern_ev]
    t = torch.tensor([total_ms, float(np.mean(kern_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_avg_ms = float(t[0]), float(t[1])
    units_total = units_per_rank if scaling == "strong" else units_per_rank * world
    if scaling == "strong":
        units_total = c["evals"]
    value = units_total * args.steps / (total_ms * 1e-3)

    # ---------------- roofline of the dominant kernel (batch / gl / eval)
    peak_ops = SM_COUNT * FP64_LANES_PER_SM * (clk.summary()["sm_max_mhz"] or 1965.0) * 1e6
    deg = gna.sin2_poly_degree()
    ops_eval = fp64_ops_per_eval(deg)
    if args.workload == "cfg4grid":
        # separable scan: the step is bound by writing the spectra (8 B per point x bin)
        out_bytes = c["bins_total"] * 8
        achieved = out_bytes / (kern_avg_ms * 1e-3) / 1e9
        peaks = _measured_peaks()
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                "peak_source": peaks["source"],
                "note": "whole gna_oscprob_scan call (stage-A sin^2 tables + rank-3 expansion "
                        "+ chi2 reduce); algorithmic bytes = spectra written"}
    elif args.workload == "cfg5fit":
        # the fit's stencil runs through the separable scan: per iteration the sin^2 work is
        # 9 mass points (not 81 candidates) x baselines x nodes x 3 terms x (degree + 5)
        nb = c["edges"].size - 1
        ops_fit = FIT_ITERS * 9 * c["L_km"].size * nb * c["order"] * fp64_ops_per_eval(deg)
        achieved = ops_fit / (kern_avg_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak_ops / 1e12,
                "unit": "T fp64-ops/s", "frac": achieved * 1e12 / peak_ops, "traffic": None,
                "ops_per_fit": ops_fit, "kernel_ms_per_launch": kern_avg_ms,
                "note": "algorithmic work of the separable evaluation (stage A of 9 mass points "
                        "per iteration); the stage-B expansion and the update are not counted"}
    elif args.workload == "cfg3emu":
        # general channel: 3 pairs x (16 + degree) FP64 + reciprocal 6 + 1 slots per energy
        # (76 at degree 7; gna_device.cuh sin2_sin_c)
        ops = 3 * (16 + deg) + RCP_OPS + 1
        achieved = units_per_rank * ops / (kern_avg_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak_ops / 1e12,
                "unit": "T fp64-ops/s", "frac": achieved * 1e12 / peak_ops, "traffic": None,
                "ops_per_energy_point": ops,
                "hbm_frac": units_per_rank * 16 / (kern_avg_ms * 1e-3) / 1e9 /
                _measured_peaks()["hbm_gbs"]}
    elif args.workload == "cfg3":
        # co-limited stream: report the HBM side (16 B per energy) and note FP64 (mixed tier:
        # 3 FP64 per term instead of degree + 5)
        launch_units = units_per_rank
        fp64_eval = (9 if args.precision == "mixed" else ops_eval) + RCP_OPS
        achieved = launch_units * 16 / (kern_avg_ms * 1e-3) / 1e9
        peaks = _measured_peaks()
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                "peak_source": peaks["source"],
                "fp64_frac": launch_units * fp64_eval / (kern_avg_ms * 1e-3) / peak_ops,
                "fp64_ops_per_energy": fp64_eval}
    else:
        # per library call, or per graph-replayed step (then the step time is the kernel time)
        launch_units = (units_per_rank / max(calls_per_step, 1)
                        if args.workload in ("cfg4", "cfg5") and not use_graph else units_per_rank)
        per_point_ops = ops_eval
        shared21 = shared_dm2_21(c, args, units_per_rank)
        if shared21:
            # the points-across-lanes kernel evaluates sin^2 Delta_21 once per warp of 32
            # points when dm2_21 (and L) is the same for all of them: the
            # algorithmic work per energy point is 2 point-specific terms + 1/32 of the third
            ops_eval = (deg + 5) * (2 + 1 / 32)
        achieved = launch_units * ops_eval / (kern_avg_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak_ops / 1e12,
                "unit": "T fp64-ops/s", "frac": achieved * 1e12 / peak_ops, "traffic": None,
                "peak_source": "148 SM x 64 FP64 lanes x sm_max clock (DESIGN.md §6; the lane "
                               "count is measured: fp64_probe below)",
                "ops_per_energy_point": ops_eval, "sin2_poly_degree": deg,
                "kernel_ms_per_launch": kern_avg_ms,
                # the same time on the other bases: every term per point (36), and SURVEY
                # §8(d)'s ~50 FP64 instructions per energy point (its estimate before the
                # 12-op sin^2 of DESIGN.md §6.1)
                "bases": {"algorithmic_%g_ops" % ops_eval: achieved * 1e12 / peak_ops,
                          "per_point_%d_ops" % per_point_ops:
                              launch_units * per_point_ops / (kern_avg_ms * 1e-3) / peak_ops,
                          "survey_50_ops": launch_units * 50 / (kern_avg_ms * 1e-3) / peak_ops}}
        if shared21:
            roof["shared_dm2_21"] = ("sin^2 Delta_21 evaluated once per warp of 32 points (same "
                                     "dm2_21 and L for every point)")
        if fp64_probe:
            roof["fp64_probe"] = fp64_probe
            roof["frac_of_probe"] = achieved * 1e3 / fp64_probe["dfma_G_per_s"]
        if args.precision == "mixed":
            # NEXT-3 mixed tier: the work spreads over the FP64, XU and FMA
            # pipes, so the roofline is instruction issue (1 warp instruction per SMSP per cycle
            # = 148 x 4 x 32 lanes x clock).  Per sin^2 term: 3 FP64 (rint of y/2, m, h) + 1 F2F
            # + half of a packed pair's FMUL2 + 6 FFMA2 + accumulating FFMA2 = 8.
            ipp = MIXED_INSTR_PER_TERM * ((2 + 1 / 32) if shared21 else 3)
            peak_issue = SM_COUNT * 4 * 32 * (clk.summary()["sm_max_mhz"] or 1965.0) * 1e6
            ach = launch_units * ipp / (kern_avg_ms * 1e-3)
            roof = {"bound": "alu", "achieved": ach / 1e12, "peak": peak_issue / 1e12,
                    "unit": "T instr/s (issue)", "frac": ach / peak_issue, "traffic": None,
                    "peak_source": "148 SM x 4 SMSP x 32 lanes x sm_max clock (one warp "
                                   "instruction per SMSP per cycle)",
                    "ops_per_energy_point": ipp,
                    "fp64_frac": launch_units * ipp * 3 / 8 / (kern_avg_ms * 1e-3) / peak_ops,
                    "kernel_ms_per_launch": kern_avg_ms}
            if shared21:
                roof["shared_dm2_21"] = ("W(h^2) of the (2,1) term evaluated once per warp of "
                                         "32 points (same dm2_21 and L for every point)")

    if args.workload in ("cfg1", "cfg2") and roof.get("bound") == "alu":
        # single-point configs: the step above carries the L2-flush recovery and launch floor
        # (DESIGN.md §6.4); report the kernel back to back as well — 20 steps per CUDA graph,
        # no flush between them (what a fit loop over one point sees), outside the timed region
        KernelTimer.enabled = False
        b2b = back_to_back_us(torch, eager_step if use_graph else step)
        roof["kernel_b2b_us"] = b2b
        roof["frac_b2b"] = units_per_rank * roof["ops_per_energy_point"] / (b2b * 1e-6) / peak_ops
        roof["frac_note"] = ("frac: per flushed step (launch + flush-recovery floor); frac_b2b: "
                             "the same work back to back")
    tr = _ncu_traffic(args.workload if args.precision == "fp64" else args.workload + "_mixed")
    if tr:
        roof["traffic"] = tr["bytes"]
        roof["traffic_source"] = tr["source"]
        roof["algorithmic_bytes"] = tr.get("algorithmic_bytes")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if scaling == "strong" else "weak",
            "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f64 phases + f32 polynomial (mixed tier)",
            "data": "synthetic",
            "config": dict(c["desc"], parallelism="dp%d over parameter points" % world
                           if scaling == "strong" else "replicas x%d" % world,
                           l2="flushed between steps (256 MiB write, untimed)",
                           energy_points_per_step=units_total),
            "bins_per_s": (c["bins_total"] * args.steps / (total_ms * 1e-3)) if c["bins_total"] else None,
            # this rank's per-step device times (median and min next to the mean)
            "step_ms": {"median": step_times[len(step_times) // 2], "min": step_times[0],
                        "max": step_times[-1]},
            "clocks": clk.summary(), "gpu_launches": launches, "roofline": roof,
            "cuda_graph": bool(use_graph)}
    if graph_note:
        line["cuda_graph_note"] = graph_note
    if args.workload in ("cfg4", "cfg5"):
        line["config"]["gather"] = gather_mode
        line["config"]["gather_chunks"] = len(sb.cb)
        if probe is not None:
            line["config"]["fused_probe"] = probe
        if world > 1 or fused_fg is not None:
            # the gathered result after the timed steps must equal a single-GPU batch of
            # all points, bit for bit (checked on rank 0, outside the timed region)
            line["config"]["gather_verified"] = _verify_gather(
                args, c, gna, torch, dist, dev, rank, sb, fused_fg if gather_mode.startswith(
                    "fused") else None)

    if args.precision == "mixed":
        line["config"]["precision"] = ("mixed (GNA_PREC_MIXED; tier tolerance 1e-6 absolute on "
                                       "P, 1e-5 relative on bins and spectra)")
        line["mixed_vs_fp64"] = (_mixed_accuracy(c, gna, torch, dev, args.workload)
                                 if rank == 0 else None)
    # ---------------- e2e: host buffers through the C ABI, copies inside the timed region
    if args.precision == "mixed":
        line["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0, "note": "host-buffer API is fp64-only"}
    elif not args.no_e2e and args.workload not in ("cfg4grid", "cfg3emu", "cfg5fit"):
        line["e2e"] = e2e(args, c, gna, torch, dist, dev, world, rank, local)
    elif args.workload in ("cfg4grid", "cfg3emu", "cfg5fit"):
        line["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0, "note": "no host-buffer variant for this NEXT row yet"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(c, "cfg5" if args.workload == "cfg5fit" else
                                            args.workload, args.cpu_seconds)
        # Table-1-style ratios: CPU time / GPU time for the same work
        cpu_v = line["cpu_baseline"]["value"]
        e2e_v = (line.get("e2e") or {}).get("value")
        line["table1_context"] = {
            "cpu_over_gpu_compute_only": value / cpu_v,
            "cpu_over_gpu_incl_transfer": (e2e_v / cpu_v) if e2e_v else None,
            "paper": {"cpu_over_gpu_compute_only": {"1e4": 20.90, "1e6": 26.46},
                      "cpu_over_gpu_incl_transfer": {"1e4": 0.017, "1e6": 1.39},
                      "hardware": "Intel Core i7-6700HQ vs NVIDIA GeForce GTX 970M, fp64",
                      "source": "PAPER.md Table 1 (P:658-689); context only"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        _barrier(dist, args, local)
    if dist.is_initialized():
        dist.destroy_process_group()


def _mixed_accuracy(c, gna, torch, dev, workload):
    """Max deviation of the mixed tier from the fp64 path on this workload (both on the GPU,
    outside the timed region; the fp64 path is itself within 1e-12 / 1e-11 of the oracle)."""
    f64 = dict(dtype=torch.float64, device=dev)
    if workload in ("cfg1", "cfg2", "cfg3"):
        out = {}
        if workload in ("cfg1", "cfg3"):
            E = (torch.tensor(c["E"], **f64) if workload == "cfg1" else
                 torch.linspace(c["lo"], c["hi"], c["n"], **f64))
            a = gna.oscprob_eval(c["params"], c["L_km"], E)
            b = gna.oscprob_eval(c["params"], c["L_km"], E, precision="mixed")
            out["P_max_abs"] = float((a - b).abs().max())
            del E, a, b
        if workload in ("cfg1", "cfg2"):
            e = torch.tensor(c["edges"], **f64)
            a = gna.gl_integrate(c["params"], c["L_km"], e, c["order"])
            b = gna.gl_integrate(c["params"], c["L_km"], e, c["order"], precision="mixed")
            out["bins_max_rel"] = float(((a - b).abs() / a.abs()).max())
        return out
    pts = {k: torch.tensor(v, **f64) for k, v in c["points"].items()}
    args = (pts, c["L_km"], c["omega"], torch.tensor(c["edges"], **f64), c["order"])
    d = torch.tensor(c["data"], **f64)
    s64, x64 = gna.oscprob_batch(*args, data=d)
    smx, xmx = gna.oscprob_batch(*args, data=d, precision="mixed")
    return {"spectra_max_rel": float(((smx - s64).abs() / s64.abs()).max()),
            "chi2_max_rel": float(((xmx - x64).abs() / x64.abs()).max())}


def _verify_gather(args, c, gna, torch, dist, dev, rank, sb, fg):
    """Rank 0: gathered spectra/chi2 == one batch over all points on this GPU (bitwise)."""
    ok = torch.ones(1, device=dev)
    if rank == 0:
        f64 = dict(dtype=torch.float64, device=dev)
        pts = {k: torch.tensor(v, **f64) for k, v in c["points"].items()}
        sp, x2 = gna.oscprob_batch(pts, c["L_km"], c["omega"], torch.tensor(c["edges"], **f64),
                                   c["order"], data=torch.tensor(c["data"], **f64),
                                   precision=args.precision)
        gs, gx = (fg.spectra, fg.chi2) if fg is not None else sb.gathered()
        ok.fill_(1.0 if (torch.equal(gs, sp) and torch.equal(gx, x2)) else 0.0)
        del pts, sp, x2
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    return bool(float(ok) == 1.0)


def back_to_back_us(torch, step, per_graph=20, reps=50) -> float:
    """Device time per step with `per_graph` steps captured back to back in one CUDA graph (no
    L2 flush in between), averaged over `reps` replays."""
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(per_graph):
            step()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * per_graph)


def shared_dm2_21(c, args, units_per_rank) -> bool:
    """True when the batch runs the points-across-lanes kernel (>= 256 points on the rank,
    <= 2 baselines; fp64 or mixed tier) and every point has the same dm2_21, so that kernel's
    shared sin^2 Delta_21 path is taken (k_batch.cuh, GNA_BATCH_PT_SHARED21)."""
    if args.workload not in ("cfg4", "cfg5"):
        return False
    pts = c["points"]
    nbase = c["L_km"].size
    per_point = nbase * (c["edges"].size - 1) * c["order"]
    p_rank = units_per_rank // per_point
    return bool(nbase <= 2 and p_rank >= 256 and np.all(pts["dm2_21"] == pts["dm2_21"][0]))


def run_fp64_probe(local: int):
    """build/probe_fp64 (tools/probe_fp64.cu, built by __graft_entry__.build()) in DFMA-only
    mode on this rank's GPU: 148 x 8 blocks x 256 threads of 8 independent DFMA chains, best
    of 5; returns its rate and the SM clock it saw, or None when the binary is absent."""
    exe = os.path.join(ROOT, "build", "probe_fp64")
    if not os.path.exists(exe):
        return None
    env = dict(os.environ, PROBE_DFMA_ONLY="1", CUDA_VISIBLE_DEVICES=str(_smi_index(local)))
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60, env=env).stdout
        rows = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
        d = next(r for r in rows if r.get("probe") == "dfma")
        dev = rows[0]
        return {"dfma_G_per_s": d["Gops_per_s"], "clock_khz": dev.get("clock_khz"),
                "source": "build/probe_fp64 (tools/probe_fp64.cu), run before the timed region"}
    except (OSError, subprocess.SubprocessError, StopIteration, ValueError, KeyError):
        return None


def _barrier(dist, args, local):
    if args.backend == "nccl":
        dist.barrier(device_ids=[local])
    else:
        dist.barrier()


def _ncu_traffic(workload: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(workload)
    except (OSError, ValueError):
        return None


def _smi_index(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    try:
        return int(vis.split(",")[local]) if vis else local
    except (ValueError, IndexError):
        return local


def _measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def e2e(args, c, gna, torch, dist, dev, world, rank, local):
    """Same metric through the host-buffer C ABI: per step H2D of the inputs from pinned
    memory and D2H of the results (overlapped in chunks inside the library)."""
    steps = max(args.e2e_steps, 1)

    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory()
        return t, t.numpy()

    host_note = None
    if args.workload in ("cfg4", "cfg5"):
        from types import SimpleNamespace

        from paper_1804_07682_b200 import dist as gdist
        P = c["points"]["theta12"].size
        nb = c["edges"].size - 1
        sb = gdist.ShardedBatch(P, nb, world, rank)
        lo, hi = sb.lo, sb.hi
        keep = []
        pts = {}
        for k, v in c["points"].items():
            t, a = pinned(v[lo:hi])
            keep.append(t)
            pts[k] = a
        te, edges = pinned(c["edges"])
        td, data = pinned(c["data"])
        keep += [te, td]
        out = None
        if world > 1:
            # the node's host memory receives every rank's rows (shared, page-locked)
            try:
                out = gdist.NodeSharedHost({"spectra": (P, nb), "chi2": (P,)}, rank,
                                           dist.distributed_c10d._get_default_store())
                host_note = "spectra + chi2 of all points gathered into one node-shared host buffer"
            except Exception as exc:  # noqa: BLE001 — e.g. a small /dev/shm
                out = None
                host_note = "per-rank pinned buffers (node-shared buffer unavailable: %s)" % (
                    str(exc).splitlines()[0][:100] if str(exc) else type(exc).__name__)
            ok = torch.tensor([1.0 if out is not None else 0.0], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if float(ok) != 1.0 and out is not None:
                out.close()
                out = None
        if out is None:
            ts, spectra = pinned(np.empty((P, nb)))
            tx, chi2 = pinned(np.empty(P))
            keep += [ts, tx]
            out = SimpleNamespace(arrays={"spectra": spectra, "chi2": chi2})

        def bar():
            if world > 1:
                _barrier(dist, args, local)

        def one():
            # the declared outputs: per step the points, edges and data go H2D, the spectra
            # and chi^2 of every point come back D2H into host memory (gathered at N > 1)
            gdist.oscprob_batch_host_sharded(sb, pts, c["L_km"], c["omega"], edges, c["order"],
                                             data, out, bar)

        def one_fit():
            # the fit step a minimiser makes: only chi^2 per point comes back (the "loss")
            gdist.oscprob_batch_host_sharded(sb, pts, c["L_km"], c["omega"], edges, c["order"],
                                             data, out, bar, spectra=False)

        # bytes summed over the ranks
        h2d = 4 * P * 8 + world * (edges.nbytes + data.nbytes)
        d2h = P * nb * 8 + P * 8
        d2h_fit = P * 8
        units = (hi - lo) * c["L_km"].size * nb * c["order"]
    elif args.workload in ("cfg1", "cfg2"):
        te, edges = pinned(c["edges"])
        ts, out = pinned(np.empty(c["edges"].size - 1))
        keep = [te, ts]
        if args.workload == "cfg1":
            tE, E1 = pinned(c["E"])
            tP, P1 = pinned(np.empty(c["E"].size))
            keep += [tE, tP]

        def one():
            if args.workload == "cfg1":
                gna.oscprob_eval_host(c["params"], c["L_km"], E1, out=P1)
            gna.gl_integrate_host(c["params"], c["L_km"], edges, c["order"], out=out)

        h2d, d2h = edges.nbytes, out.nbytes
        if args.workload == "cfg1":
            h2d += E1.nbytes
            d2h += P1.nbytes
        units = c["evals"]
    else:
        n = c["n"]
        tE, E = pinned(np.linspace(c["lo"], c["hi"], n))
        tP, Pout = pinned(np.empty(n))
        keep = [tE, tP]

        def one():
            gna.oscprob_eval_host(c["params"], c["L_km"], E, out=Pout)

        h2d, d2h = E.nbytes, Pout.nbytes
        units = n
    one()
    torch.cuda.synchronize()
    if world > 1:
        _barrier(dist, args, local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        one()
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_units = units * world if args.workload in ("cfg1", "cfg2", "cfg3") else c["evals"]
    extra = {}
    if args.workload in ("cfg4", "cfg5"):
        # second measurement: the chi^2-only fit step
        one_fit()
        torch.cuda.synchronize()
        if world > 1:
            _barrier(dist, args, local)
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(steps):
            one_fit()
        f1.record()
        torch.cuda.synchronize()
        ms2 = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms2, op=dist.ReduceOp.MAX)
        extra["fit_step"] = {"value": total_units * steps / (float(ms2[0]) * 1e-3),
                             "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h_fit),
                             "outputs": "chi2 per point only"}
        extra["outputs"] = "spectra + chi2 of every point in host memory"
        if host_note:
            extra["host_gather"] = host_note
        if world > 1 and hasattr(out, "close"):
            out.close(barrier=lambda: _barrier(dist, args, local))
    del keep
    return {"value": total_units * steps / (float(ms[0]) * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), **extra,
            "steps": steps, "api": ("dist.oscprob_batch_host_sharded -> gna_oscprob_batch_host "
                                    "per rank (H2D inputs, kernels, D2H spectra + chi2), barrier")
            if args.workload in ("cfg4", "cfg5")
            else ("gna_gl_integrate_host" if args.workload == "cfg2" else
                  ("gna_oscprob_eval_host + gna_gl_integrate_host" if args.workload == "cfg1"
                   else "gna_oscprob_eval_host"))}


if __name__ == "__main__":
    main()
