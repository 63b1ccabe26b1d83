#!/usr/bin/env python
"""bench.py -- FETI dual-operator hot path on B200 (BASELINE.json metric).

Workload (config.workload): BASELINE.json configs[3] "C4", the throughput
config: FETI-DP with corner primal DOFs, k-scaling, 64x32 modules of 64x64 Q4
elements (2048 subdomains, 8450 DOFs each), rho ~ U(0,1), SIMP p=3,
Emin=1e-9, left clamp, right-edge traction.  Seeded synthetic densities
(paper_2111_11728_b200/problems.py) stand in for the paper's TO snapshots.

A step is one application of the condensed FETI-DP dual operator
F = F_rr + F_rc Kbar_cc^{-1} F_rc^T to one multiplier vector (what every PCG
iteration does), with the operator resident in HBM.  value = bytes one apply
streams with symmetric operator storage (the packed lower block-triangle of
every F_s and of Kbar_cc^-1, A_bc in both phases, lambda + y, gather lists:
2.33 GB for C4, config.value_bytes_per_apply) / device time per apply, whole
job over all ranks.  The reference arm divides the SAME byte count by its own
apply time, so the value ratio is the apply-time ratio.  The SURVEY.md 8d
full-storage figure (8 sum n_s^2 + ..., 4.28 GB) is reported as
value_full_storage_GBps.  The operator is far larger than L2 (126 MB), so no
flush is needed between steps.

Also reported on the same line: e2e (the same metric through the C-ABI with
host buffers, H2D of lambda and D2H of F lambda inside the timed region),
the roofline of the dominant kernel, the CPU oracle baseline, build time and
per-config PCG solve times.

--impl reference: the reference's own CPU algorithm (the C++ oracle port in
oracle/; the reference itself does not compile here) on this
box's host cores, same metric, unit and config: one step is one full C4
apply (about 0.3 s on 16 cores), no extrapolation.
"""
import argparse
import ctypes as C
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

from paper_2111_11728_b200 import problems as pb  # noqa: E402

METRIC = "F-apply GB/s & FP64 TFLOP/s vs roofline; PCG solve time to 1e-6 rel. res."


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(n_gpus):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if ws > 1:
        import torch
        import torch.distributed as td
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            td.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # no GPU (e.g. the CPU reference arm): plumbing over gloo
            td.init_process_group("gloo")
        dist = td
    return ws, rank, local, dist


def barrier(dist):
    if dist is not None:
        dist.barrier()


def _dev(dist):
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(dist, v):
    """Max over ranks (device timing rule: the slowest rank defines the step)."""
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_dev(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_dev(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def replica_throughput(dist, bytes_per_step, steps, ms_per_step_local):
    """Whole-job GB/s of N independent replicas: all ranks' steps over the
    slowest rank's time (replicas only)."""
    t = max_over_ranks(dist, ms_per_step_local)
    total = sum_over_ranks(dist, float(steps))
    return bytes_per_step * total / (t * 1e-3 * steps) / 1e9, t


# ---- CPU oracle (reference algorithm) on a bounded sample -----------------
def cpu_c4(steps=3, block_k=64):
    """The oracle's implicit F-apply (per-subdomain band-Cholesky solves +
    coarse solve) on the FULL C4 configuration, all host cores:
    build time, mean of `steps` single applies after one warm-up, and the
    SURVEY 8d block slice -- `block_k` columns applied one after another (the
    oracle's simultaneous_pcg line 7), extrapolated to k = 2048 and labelled
    as such."""
    from oracle import pyoracle
    pyoracle.build()
    t0 = time.perf_counter()
    o = pyoracle.Oracle(pb.config4())
    t_build = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    x = rng.standard_normal(o.m)
    o.apply_F(x)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        o.apply_F(x)
        ts.append(time.perf_counter() - t0)
    t_apply = sum(ts) / len(ts)
    blk = None
    if block_k:
        X = rng.standard_normal((block_k, o.m))
        t0 = time.perf_counter()
        for c in range(block_k):
            o.apply_F(X[c])
        tb = time.perf_counter() - t0
        w = c4_work()
        blk = {"k": block_k, "s": tb, "tflops": w["flops_per_col"] * block_k / tb / 1e12,
               "extrapolated_k2048_s": tb * 2048 / block_k,
               "note": "oracle block apply = one implicit apply per column; k = 2048 figure extrapolated"}
    return {"t_apply_s": t_apply, "t_build_s": t_build, "cores": os.cpu_count(), "block": blk,
            "sample": f"full C4 (2048 subdomains, m = {o.m}): mean of {steps} applies after 1 warm-up"}


def cpu_applies(steps=3):
    """the oracle's build time and single F-apply time (median of
    `steps` after one warm-up, all host cores) for C1-C3 and C5."""
    from oracle import pyoracle
    out = {}
    for name, fn in (("C1", pb.config1), ("C2", pb.config2), ("C3-tfeti", lambda: pb.config3(method=0)),
                     ("C3-fetidp", lambda: pb.config3(method=1)), ("C5", pb.config5)):
        t0 = time.perf_counter()
        o = pyoracle.Oracle(fn())
        tb = time.perf_counter() - t0
        x = np.random.default_rng(0).standard_normal(o.m)
        o.apply_F(x)
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            o.apply_F(x)
            ts.append(time.perf_counter() - t0)
        out[name] = {"build_s": round(tb, 4), "apply_ms": round(statistics.median(ts) * 1e3, 3), "m": o.m}
        log("cpu apply", name, out[name])
    return out


def cpu_solves():
    """The oracle's full PCG solves (implicit per-subdomain solves, all host
    cores) for the configs whose CPU solve fits a bounded budget; the C3 T-FETI
    FO (44 s) and C5 RRS (~700 s) CPU solves are recorded in
    profiles/r01_solves_full_vs_oracle.jsonl and profiles/r01_parity_C5_full.json."""
    from oracle import pyoracle
    out = {}
    for name, fn, dirs in (("C1", pb.config1, 0), ("C2", pb.config2, 0), ("C2-fo", pb.config2, 1),
                           ("C3-fetidp", lambda: pb.config3(method=1), 1)):
        t0 = time.perf_counter()
        o = pyoracle.Oracle(fn())
        tb = time.perf_counter() - t0
        t0 = time.perf_counter()
        _, tr = o.solve(tol=1e-6, max_it=6000, directions=dirs)
        out[name] = {"build_s": tb, "solve_s": time.perf_counter() - t0, "iterations": tr["iterations"],
                     "status": ["converged", "max_iter", "breakdown"][tr["status"]],
                     "directions": ["single", "fo", "rrs"][dirs]}
        log("cpu", name, out[name])
    return out


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def c4_work(sx=64, sy=32, n=64):
    """Algorithmic work of one C4 F-apply from the partition geometry alone
    (SURVEY.md 8d / App. A): FETI-DP with every partition vertex primal and the
    left edge clamped.  n_s = 2(n-1) DOFs per shared module edge; n_c,s = the
    module's unclamped corner DOFs."""
    e = 2 * (n - 1)
    sn2 = snc = sns = 0.0
    m = 0
    for sj in range(sy):
        for si in range(sx):
            nb = (si > 0) + (si < sx - 1) + (sj > 0) + (sj < sy - 1)
            ns = e * nb
            nc = 4 if si == 0 else 8
            sn2 += ns * ns
            snc += ns * nc
            sns += ns
    m = e * ((sx - 1) * sy + sx * (sy - 1))
    Nc = 2 * (sx + 1) * (sy + 1) - 2 * (sy + 1)
    byts = 8 * sn2 + 16 * snc + 8.0 * Nc * Nc + 16.0 * m + 8 * sns
    flops = 2 * sn2 + 4 * snc + 2.0 * Nc * Nc
    # symmetric storage: lower block-triangle of 32x32 tiles of every F_s and
    # of the coarse inverse (what the packed kernels stream)
    packed = 0.0
    for sj in range(sy):
        for si in range(sx):
            nb = (si > 0) + (si < sx - 1) + (sj > 0) + (sj < sy - 1)
            t = (e * nb + 31) // 32
            packed += 8192.0 * t * (t + 1) / 2
    tc = (Nc + 31) // 32
    stream = packed + 16 * snc + 8192.0 * tc * (tc + 1) / 2 + 16.0 * m + 8 * sns
    return {"bytes": byts, "flops_per_col": flops, "main_bytes": 8 * sn2, "packed_main_bytes": packed,
            "stream_bytes": stream, "m": m, "n_c": Nc}


def c4_config(flush_l2=False):
    """config of the headline line, identical in both arms (same workload)."""
    w = c4_work()
    return {"workload": "C4 FETI-DP F-apply (single direction): 64x32 modules of 64x64 Q4 (2048 "
                        "subdomains), rho ~ U(0,1), k-scaling, Dirichlet precond, seed 1",
            "m": w["m"], "n_c": w["n_c"], "flush_l2": flush_l2,
            "l2_note": "operator (2.3 GB symmetric-packed) larger than L2 (126 MB)",
            "value_bytes_per_apply": w["stream_bytes"],
            "value_bytes": "bytes one apply must stream with symmetric operator storage (packed lower "
                           "block-triangle of each F_s and of Kbar_cc^-1, A_bc twice, lambda + y, gather "
                           "lists); the same constant in both arms, so value ratios are time ratios",
            "parallelism": "replicas"}


def run_reference(args, ws, rank, dist):
    """--impl reference: the reference's CPU algorithm (the oracle port of the
    implicit operator: per-subdomain band-Cholesky solves + coarse solve,
    SPEC.md:399) on the FULL C4 configuration, all host cores, rank 0 only;
    the other ranks exit without work.  No product code on this path.  A step
    is one full F-apply of C4 (504,000 dual rows), the same step as ours."""
    if rank != 0:
        return
    from oracle import pyoracle
    pyoracle.build()
    cores = pyoracle.lib().fo_set_threads(os.cpu_count() or 1)  # torchrun sets OMP_NUM_THREADS=1
    t0 = time.perf_counter()
    o = pyoracle.Oracle(pb.config4())
    t_build = time.perf_counter() - t0
    x = np.random.default_rng(0).standard_normal(o.m)
    for _ in range(args.warmup):
        o.apply_F(x)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.apply_F(x)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    w = c4_work()
    v = w["stream_bytes"] / t / 1e9
    sample = (f"full C4 (2048 subdomains, m = {o.m}): {args.steps} timed applies after {args.warmup} "
              f"warm-up, oracle build {t_build:.1f} s (not timed)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U(0,1) densities, C4 law)",
            "config": c4_config(),
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "port",
                             "sample": sample, "cpu_model": cpu_model(),
                             "build_s": t_build, "apply_ms_min": min(ts) * 1e3},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def apply_time_us(engine, g, reps=200):
    """Device time of one F-apply (CUDA events around each apply, after 20
    warm-up applies, no L2 flush): for C1-C3/C5 the operator fits L2."""
    L = engine.lib()
    m = g.m
    dx, dy = C.c_void_p(), C.c_void_p()
    engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dx)))
    engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dy)))
    xp, yp = C.cast(dx, C.POINTER(C.c_double)), C.cast(dy, C.POINTER(C.c_double))
    engine.check(L.fetigpu_fill_random(g.h, xp, C.c_size_t(m), C.c_ulonglong(7)))
    ms, n = (C.c_double * 3)(), C.c_int()
    engine.check(L.fetigpu_time_apply(g.h, xp, yp, 1, 20, 0, ms, C.byref(n)))
    engine.check(L.fetigpu_time_apply(g.h, xp, yp, 1, reps, 0, ms, C.byref(n)))
    L.fetigpu_device_free(g.h, dx)
    L.fetigpu_device_free(g.h, dy)
    return ms[0] * 1e3


def solve_table(engine, configs):
    out = {}
    for name, fn, kw in configs:
        prob = fn()
        g = engine.FetiSystem(prob)
        st = g.stats()
        lam, tr = g.solve(**kw)
        out[name] = {"build_ms": round(st["build_ms"], 2), "solve_ms": round(tr["solve_ms"], 2),
                     "iterations": tr["iterations"], "status": ["converged", "max_iter", "breakdown"][tr["status"]],
                     "rel_residual": tr["eps_final"] / tr["eps0"] if tr["eps0"] > 0 else 0.0,
                     "m": st["m"], "directions": ["single", "fo", "rrs"][kw.get("directions", 0)]}
        if kw.get("directions", 0) == 2:
            # FETI-DP auto store (solve_rrs.cuh): the implicit store applies F to
            # three k-column blocks per iteration, the explicit one to one
            k = st["n_sub"]
            out[name]["f_applies"] = tr["f_applies"]
            out[name]["store"] = "implicit" if tr["f_applies"] > 2 * k * tr["iterations"] + 1 else "explicit"
            out[name]["kept"] = [int(x) for x in tr["kept"][1:]]
            out[name]["phase_ms"] = {p: round(v, 1) for p, v in zip(
                ("FW", "gram", "pivchol", "compress", "update", "precond", "pack", "reorth"), tr["phase_ms"])}
        ops = g.time_ops(reps=200 if not name.startswith("C4") else 20)
        out[name]["per_iteration_ops_us"] = {k.replace("_ms", ""): round(v * 1e3, 2) for k, v in ops.items()}
        out[name]["us_per_iteration"] = round(tr["solve_ms"] * 1e3 / max(1, tr["iterations"]), 1)
        if not name.startswith("C4"):
            # C1-C3 and C5 operators are L2-resident -- time per apply and
            # effective GB/s of the formula bytes, labelled as such (no HBM-fraction claim)
            us = apply_time_us(engine, g)
            out[name]["apply_us"] = round(us, 2)
            out[name]["apply_formula_bytes"] = st["op_bytes"]
            out[name]["apply_effective_GBps_L2_resident"] = round(st["op_bytes"] / (us * 1e-6) / 1e9, 1)
        g.close()
        log(name, out[name])
    return out


class _SoloComm:
    """world size 1 without torchrun: the exchanges are identities"""

    def allreduce_sum(self, t):
        return t


def run_shard(args, ws, rank, local, dist):
    """--shard: the C4 apply sharded over the ranks by module row bands
    (paper_2111_11728_b200/shard.py): halo rows and the coarse t exchanged by
    NCCL allreduce, the coarse problem solved redundantly.  Strong scaling:
    every rank applies 1/N of the subdomains to the same multiplier vector.
    The apply synchronises the host around its exchanges, so the time is the
    host wall clock of `steps` applies after a device synchronisation, max
    over ranks."""
    import torch
    from paper_2111_11728_b200 import engine, shard
    torch.cuda.set_device(local)
    prob = pb.config4()
    g = engine.FetiSystem(prob)
    ranges = shard.row_bands(prob.sx, prob.sy, ws)
    comm = shard.TorchComm(dist, "cuda") if dist is not None else _SoloComm()
    sh = shard.ShardedSystem(g, rank, ranges, comm)
    x = torch.as_tensor(np.random.default_rng(1234).standard_normal(g.m), device="cuda")
    for _ in range(args.warmup):
        sh.apply(x)
    torch.cuda.synchronize()
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        y = sh.apply(x)
    torch.cuda.synchronize()
    t = max_over_ranks(dist, (time.perf_counter() - t0) / args.steps)
    ref = g.apply_F(x.cpu().numpy())
    tt = sh.plan.touched(rank)
    exact = bool(np.array_equal(y.cpu().numpy()[tt], ref[tt]))
    if rank == 0:
        vbytes = c4_work()["stream_bytes"]
        cfg = dict(c4_config(), parallelism=f"subdomain-sharded x{ws} (row bands)")
        print(json.dumps({"metric": METRIC, "value": vbytes / t / 1e9, "unit": "GB/s", "n_gpus": ws,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic (seeded U(0,1) densities, C4 law)", "config": cfg,
                          "sharded_equals_1gpu_bitwise": exact,
                          "timing": "host wall clock per sharded apply (exchanges synchronise), max over ranks"}),
              flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-solves", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-block", action="store_true")
    ap.add_argument("--block-k", type=int, default=2048)
    ap.add_argument("--block-reps", type=int, default=3)
    ap.add_argument("--shard", action="store_true",
                    help="strong scaling: one C4 apply sharded over the ranks (shard.py, NCCL exchanges) "
                         "instead of N replicas")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws, rank, local, dist = dist_setup(args.gpus)
    if args.impl == "reference":
        # The other ranks wait until rank 0 has measured, in a blocking gloo
        # barrier: exiting early left them polling in the process-group
        # teardown (and an NCCL barrier would spin a host thread each), which
        # halved the CPU baseline's throughput.
        cpu_group = dist.new_group(backend="gloo") if dist is not None else None
        run_reference(args, ws, rank, dist)
        if dist is not None:
            dist.barrier(group=cpu_group)
        return
    from paper_2111_11728_b200 import engine
    engine.check(engine.lib().fetigpu_set_device(local))
    L = engine.lib()
    if args.shard:
        run_shard(args, ws, rank, local, dist)
        return

    prob = pb.config4()
    t0 = time.perf_counter()
    g = engine.FetiSystem(prob)
    build_wall = time.perf_counter() - t0
    st = g.stats()
    m = g.m
    log(f"[rank {rank}] C4 built: m={m} build_ms={st['build_ms']:.1f} wall={build_wall:.1f}s "
        f"device={st['device_bytes']/1e9:.1f} GB")
    # device-resident multiplier and output
    dx, dy = C.c_void_p(), C.c_void_p()
    engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dx)))
    engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dy)))
    engine.check(L.fetigpu_fill_random(g.h, C.cast(dx, C.POINTER(C.c_double)), C.c_size_t(m),
                                       C.c_ulonglong(1234)))
    ms = (C.c_double * 3)()
    launches = C.c_int()
    xp, yp = C.cast(dx, C.POINTER(C.c_double)), C.cast(dy, C.POINTER(C.c_double))
    engine.check(L.fetigpu_time_apply(g.h, xp, yp, 1, args.warmup, 0, ms, C.byref(launches)))
    barrier(dist)
    engine.check(L.fetigpu_synchronize(g.h))
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        engine.check(L.fetigpu_time_apply(g.h, xp, yp, 1, args.steps, 0, ms, C.byref(launches)))
        engine.check(L.fetigpu_synchronize(g.h))
        # soak the same apply loop so the sampler sees >= 2 s of load
        soak = 0
        while time.perf_counter() - t_wall0 < 2.0:
            engine.check(L.fetigpu_time_apply(g.h, xp, yp, 1, 20, 0, (C.c_double * 3)(), C.byref(C.c_int())))
            soak += 20
    barrier(dist)
    # value: the bytes one apply streams with symmetric storage (same constant
    # as the reference arm); the SURVEY's full-storage figure is kept as a
    # secondary key
    vbytes = c4_work()["stream_bytes"]
    if abs(st["stream_bytes"] - vbytes) > 1e-6 * vbytes:
        log(f"note: library stream bytes {st['stream_bytes']:.0f} != geometry {vbytes:.0f}")
    value, t_apply_ms = replica_throughput(dist, vbytes, args.steps, ms[0])
    t_main_ms = max_over_ranks(dist, ms[1])
    total_steps = sum_over_ranks(dist, args.steps)
    peak, peak_kind = peaks()
    achieved = st["main_kernel_bytes"] / (t_main_ms * 1e-3) / 1e9
    traffic = None
    sym = st["main_kernel_bytes"] < 0.9 * c4_work()["main_bytes"]
    kname = {2: "k_sym_gemv_tma<1,true> (symmetric-packed F_rr tiles by TMA bulk copies into per-warp mbarrier "
                "rings, persistent grid, fused coarse pre-pass)",
             1: "k_sym_gemv_scatter<1,true> (symmetric-packed F_rr stream by LDG + fused coarse pre-pass)",
             0: "k_gather_gemv_scatter<1,true> (F_rr stream + fused coarse pre-pass)"}[st["apply_kernel"]]
    # the apply only reads its operator: the read-only stream ceiling of this
    # device, measured here, beside the copy (read + write) figure the driver
    # wrote to MEASURED_PEAKS.json, which stays the roofline's `peak`
    try:
        read_peak = engine.hbm_read_peak(2 << 30, 10)
    except Exception as e:  # noqa: BLE001
        log(f"note: hbm_read_peak failed: {e}")
        read_peak = None
    tp = os.path.join(ROOT, "profiles", {2: "traffic_sym_gemv_tma.json", 1: "traffic_sym_gemv.json",
                                         0: "traffic_gemv.json"}[st["apply_kernel"]])
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # e2e through the C-ABI with pinned host buffers (H2D lambda, D2H F lambda)
    hx, hy = C.c_void_p(), C.c_void_p()
    engine.check(L.fetigpu_host_alloc(C.c_size_t(8 * m), C.byref(hx)))
    engine.check(L.fetigpu_host_alloc(C.c_size_t(8 * m), C.byref(hy)))
    hxa = np.ctypeslib.as_array(C.cast(hx, C.POINTER(C.c_double)), shape=(m,))
    hxa[:] = np.random.default_rng(3).standard_normal(m)
    hxp, hyp = C.cast(hx, C.POINTER(C.c_double)), C.cast(hy, C.POINTER(C.c_double))
    for _ in range(args.warmup):
        engine.check(L.fetigpu_apply_F(g.h, hxp, hyp, 1, m))
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        engine.check(L.fetigpu_apply_F(g.h, hxp, hyp, 1, m))
    t_e2e = max_over_ranks(dist, (time.perf_counter() - t0) / args.steps)
    e2e = vbytes * total_steps / (t_e2e * args.steps) / 1e9
    # the same call on pageable host memory (a std::vector caller of the C++
    # adapter, include/feti_gpu.hpp)
    px = np.random.default_rng(3).standard_normal(m)
    py = np.empty(m)
    pxp, pyp = px.ctypes.data_as(C.POINTER(C.c_double)), py.ctypes.data_as(C.POINTER(C.c_double))
    for _ in range(args.warmup):
        engine.check(L.fetigpu_apply_F(g.h, pxp, pyp, 1, m))
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        engine.check(L.fetigpu_apply_F(g.h, pxp, pyp, 1, m))
    t_e2e_pg = max_over_ranks(dist, (time.perf_counter() - t0) / args.steps)

    # ---- K5 block apply (Alg. 1 line 7) at the C4 block width k = N_s = 2048
    block = None
    if not args.no_block:
        k = args.block_k
        dW, dQ = C.c_void_p(), C.c_void_p()
        engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m * k), C.byref(dW)))
        engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m * k), C.byref(dQ)))
        Wp, Qp = C.cast(dW, C.POINTER(C.c_double)), C.cast(dQ, C.POINTER(C.c_double))
        engine.check(L.fetigpu_fill_random(g.h, Wp, C.c_size_t(m * k), C.c_ulonglong(99)))
        bms = (C.c_double * 1)()
        engine.check(L.fetigpu_time_apply_block(g.h, Wp, Qp, k, 1, bms))      # warm-up
        barrier(dist)
        with ClockSampler(local) as bclk:
            engine.check(L.fetigpu_time_apply_block(g.h, Wp, Qp, k, args.block_reps, bms))
        t_blk = max_over_ranks(dist, bms[0])
        dmma, dfma = engine.fp64_peak()
        flops = st["op_flops_per_col"] * k
        tf = flops / (t_blk * 1e-3) / 1e12
        block = {"k": k, "ms": t_blk, "flops": flops, "tflops": tf * ws, "peak_dmma_tflops": dmma,
                 "peak_dfma_tflops": dfma, "frac": tf / dmma,
                 "peak_kind": "measured on this device by fetigpu_fp64_peak (independent DMMA.8x8x4 from "
                              "registers, all SMs); MEASURED_PEAKS.json has no FP64 figure; datasheet 40",
                 "clocks": bclk.summary(),
                 "kernel": "k_block_apply_dp2<64,64,16,2> (DMMA m8n8k4, fused W-row gather and Q scatter) + coarse pre-pass + DMMA GEMM (dla.cuh) for U = Kbar^-1 T"}
        L.fetigpu_device_free(g.h, dW)
        L.fetigpu_device_free(g.h, dQ)
        log("block", block)

    solves = None
    if rank == 0 and not args.no_solves:
        g.close()
        solves = solve_table(engine, [
            ("C1", pb.config1, dict(tol=1e-6, max_it=2000, directions=0)),
            ("C2", pb.config2, dict(tol=1e-6, max_it=6000, directions=0)),
            ("C2-fo", pb.config2, dict(tol=1e-6, max_it=2000, directions=1)),
            ("C3-tfeti", lambda: pb.config3(method=0), dict(tol=1e-6, max_it=2000, directions=1)),
            ("C3-fetidp", lambda: pb.config3(method=1), dict(tol=1e-6, max_it=2000, directions=1)),
            ("C5", pb.config5, dict(tol=1e-6, max_it=200, directions=2)),
            ("C4-cg", pb.config4, dict(tol=1e-6, max_it=3000, directions=0)),
            ("C4-fo", pb.config4, dict(tol=1e-6, max_it=3000, directions=1)),
            ("C4-rrs", pb.config4, dict(tol=1e-6, max_it=100, directions=2)),
        ])

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            from oracle import pyoracle
            pyoracle.build()
            pyoracle.lib().fo_set_threads(os.cpu_count() or 1)
            r = cpu_c4()
            cpu = {"value": vbytes / r["t_apply_s"] / 1e9, "unit": "GB/s",
                   "cores": r["cores"], "kind": "port", "sample": r["sample"],
                   "cpu_model": cpu_model(), "t_apply_ms": r["t_apply_s"] * 1e3,
                   "build_s": r["t_build_s"], "block_slice": r["block"]}
            if not args.no_solves:
                cpu["applies"] = cpu_applies()
                cpu["solves"] = cpu_solves()
        except Exception as e:  # the checker is optional for the GPU number
            log("cpu baseline failed:", e)

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_apply_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U(0,1) densities, C4 law)",
            "config": c4_config(),
            "value_full_storage_GBps": st["op_bytes"] * total_steps / (t_apply_ms * 1e-3 * args.steps) / 1e9,
            "us_per_apply": t_apply_ms * 1e3,
            "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": 8 * m, "d2h_bytes_per_step": 8 * m,
                    "ms_per_step": t_e2e * 1e3, "host_memory": "pinned",
                    "pageable": {"value": vbytes * total_steps / (t_e2e_pg * args.steps) / 1e9,
                                 "ms_per_step": t_e2e_pg * 1e3}},
            "gpu_launches": launches.value * args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kname,
                         "kernel_ms": t_main_ms, "kernel_share": t_main_ms / t_apply_ms,
                         "bytes_per_launch": st["main_kernel_bytes"], "peak_kind": peak_kind,
                         "peak_note": "peak = copy bandwidth (read + write bytes) from MEASURED_PEAKS.json; the "
                                      "kernel only reads, so frac can exceed 1 -- read_only_peak is the same "
                                      "device's read-only stream ceiling measured by fetigpu_hbm_read_peak",
                         "read_only_peak": read_peak,
                         "frac_read_only": (achieved / read_peak) if read_peak else None},
            "clocks": clocks,
            "build": {"ms": st["build_ms"], "nd_ms": st["nd_ms"], "slot_ms": st["slot_ms"],
                      "wall_s": build_wall},
            "cpu_baseline": cpu,
            "block_apply": block,
            "solves": solves,
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
