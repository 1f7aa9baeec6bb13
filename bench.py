#!/usr/bin/env python
"""Benchmark of the B200 zip-up hot path (BASELINE.json metric: zip-up site-contractions/sec
and FP64 TFLOP/s, 1-8 GPUs) on the batched workload configs[4] (cfg5): per GPU 512
independent zip-ups, L=40 sites of size 2, state rank 64, random rank-4 MPO, max rank 64,
eps 1e-10, fp64; weak scaling (512 members per GPU, 4096 at 8 GPUs) with one NCCL
all-reduce of the batch error budget per step.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload cfgK]

Prints ONE JSON line on rank 0.  A "step" = one qtt_zipup over this GPU's members (a1..a7)
+ the a8 summary + the cross-GPU all-reduce.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2602_20226_b200 import dist as qdist  # noqa: E402
from paper_2602_20226_b200 import gen  # noqa: E402

METRIC = "zip-up site-contractions/sec"
UNIT = "site-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "qft", "variational"],
                    help="qft: the tensorized DFT of PAPER.md:533-566 (N = 2^13, max rank 16) as a chain of "
                         "12 complex Hadamard zip-ups (SURVEY.md §8(f) f2); variational: one sweep of "
                         "qtt_variational (f3) on cfg5 members seeded by a max-rank-16 zip-up")
    ap.add_argument("--members-per-gpu", type=int, default=512)
    ap.add_argument("--strong", action="store_true",
                    help="cfg5 strong scaling: --global-members (4096) split over the N ranks (dist.strong_range) "
                         "instead of --members-per-gpu per rank (weak scaling, the default)")
    ap.add_argument("--global-members", type=int, default=4096)
    ap.add_argument("--cpu-members", type=int, default=64,
                    help="cfg5 oracle sample size (members b = stride*t of this rank's shard) for cpu_baseline")
    ap.add_argument("--cpu-budget-s", type=float, default=30.0,
                    help="cfg1-4 cpu_baseline: stop the oracle zip-up after this many seconds (bounded sample)")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"],
                    help="f32: the fp32 variant (binary32 cores; large-path contractions as 3xTF32 on tcgen05)")
    ap.add_argument("--window", type=int, default=1, choices=[1, 2],
                    help="2: QTT_WINDOW2 super-cores of two sites (SURVEY.md §8(f) f4; per-member kernel)")
    ap.add_argument("--ncores", type=int, default=1, choices=[1, 2],
                    help="--workload variational: 1 = single-site sweeps, 2 = two-site super-cores (PAPER.md:300)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------- workload

def build_workload(args, rank):
    """Returns (subscripts, kind, problems (list of gen.Problem for this rank), x_stack, op_stack, cfg dict)."""
    if args.workload == "cfg5":
        if args.strong:
            lo, hi = qdist.strong_range(rank, args.gpus, args.global_members)
            gb = args.global_members
        else:
            lo, hi = qdist.member_range(rank, args.gpus, args.members_per_gpu)
            gb = args.members_per_gpu * args.gpus
        members = list(range(lo, hi))
        probs, xs, ops = gen.cfg5_batch_arrays(members)
        cfg = {"workload": "configs[4] cfg5: batch of independent zip-ups, L=40 d=2, state rank 64 N(0,1/64), "
                           "random rank-4 MPO N(0,1/4), max rank 64, eps 1e-10",
               "members_per_gpu": hi - lo, "global_batch": gb, "L": 40, "rank": 64, "mpo_rank": 4,
               "max_rank": 64, "eps": 1e-10,
               "parallelism": f"dp{args.gpus} (members sharded, 1 all-reduce/step, "
                              f"{'strong: fixed global batch' if args.strong else 'weak: fixed members per GPU'})"}
        return "ij,j->i", "matvec", probs, xs, ops, cfg
    mk = {"cfg1": lambda: gen.cfg1(), "cfg2": lambda: gen.cfg2(), "cfg3": lambda: gen.cfg3(),
          "cfg4": lambda: gen.cfg4()}[args.workload]
    p = mk()
    xs = [c[None] for c in p.x.cores]
    ops = None if p.op is None else [c[None] for c in p.op.cores]
    subs = {"matvec": "ij,j->i", "hadamard": "i,i->i", "truncate": "i->i"}[p.kind]
    cfg = {"workload": f"{args.workload} ({p.name})", "members_per_gpu": 1, "global_batch": args.gpus,
           "max_rank": p.max_rank, "eps": p.eps, "parallelism": f"replicas x{args.gpus}"}
    return subs, p.kind, [p], xs, ops, cfg


def site_flops_w2(kind, ranks_y, xr, orr, d, dj, sweeps):
    """site_flops for the window-2 zip-up: split q is (chi_q d_q) x (d_{q+1} w r) after
    absorbing site q+1 into a carry of chi_q d_q rows (site 0 absorbed first, chi = 1)."""
    L = len(d)
    d, dj = [int(v) for v in d], [int(v) for v in dj]

    def contract(rows, s):
        w, w2 = (int(orr[s]), int(orr[s + 1])) if kind != "truncate" else (1, 1)
        r, r2 = int(xr[s]), int(xr[s + 1])
        if kind == "matvec":
            return 2 * rows * w * r * dj[s] * r2 + 2 * rows * d[s] * w2 * r2 * w * dj[s]
        if kind == "hadamard":
            return 2 * rows * w * r * d[s] * r2 + 2 * rows * d[s] * r2 * w * w2
        return 2 * rows * r * d[s] * r2

    out = [(float(contract(1, 0)), 0.0, 0.0, 0.0)]
    for q in range(L - 1):
        s = q + 1
        chi = int(ranks_y[q])
        rows = chi * d[q]
        w2 = int(orr[s + 1]) if kind != "truncate" else 1
        m, n = rows, d[s] * w2 * int(xr[s + 1])
        k = int(ranks_y[q + 1])
        p = min(m, n)
        fq = (2.0 * n * m * m - (2.0 / 3.0) * m ** 3) if m <= n else 0.0
        out.append((float(contract(rows, s)), fq, 2.0 * k * m * n, float(sweeps[q]) * p * (p - 1) / 2 * 12 * m))
    return out


def site_flops(kind, ranks_y, xr, orr, d, dj, sweeps, window=1):
    """Per-site algorithmic flops for one member:
    contract / qr / carry / jacobi (executed sweeps x p(p-1)/2 pairs x 12 m)."""
    if window == 2:
        return site_flops_w2(kind, ranks_y, xr, orr, d, dj, sweeps)
    L = len(d)
    d, dj = [int(v) for v in d], [int(v) for v in dj]
    out = []
    for q in range(L):
        chi, r, r2 = int(ranks_y[q]), int(xr[q]), int(xr[q + 1])        # Python ints: no int32 overflow
        w, w2 = (int(orr[q]), int(orr[q + 1])) if kind != "truncate" else (1, 1)
        m, n = chi * d[q], w2 * r2
        if kind == "matvec":
            fc = 2 * chi * w * r * dj[q] * r2 + 2 * chi * d[q] * w2 * r2 * w * dj[q]
        elif kind == "hadamard":
            fc = 2 * chi * w * r * d[q] * r2 + 2 * chi * d[q] * r2 * w * w2
        else:
            fc = 2 * chi * r * d[q] * r2
        if q == L - 1:
            out.append((fc, 0.0, 0.0, 0.0))
            continue
        k = int(ranks_y[q + 1])
        p = min(m, n)
        fq = (2.0 * n * m * m - (2.0 / 3.0) * m ** 3) if m <= n else 0.0
        fk = 2.0 * k * m * n
        fj = float(sweeps[q]) * p * (p - 1) / 2 * 12 * m
        out.append((float(fc), fq, fk, fj))
    return out


# ----------------------------------------------------------------------------- peaks / clocks

def fp64_peaks(torch, stream):
    """Measure DFMA and DMMA (mma.sync f64) peaks on this GPU (MEASURED_PEAKS.json has none)."""
    import ctypes
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2602_20226_b200", "lib", "libqttprobe.so"))
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    out = torch.zeros(4096, dtype=torch.float64, device="cuda")
    res = {}
    for name, fn, per in (("dfma", lib.qtt_probe_dfma, 256 * 16 * 8 * 2), ("dmma", lib.qtt_probe_dmma, 8 * 8 * 4 * 512)):
        blocks, iters = sms * 4, 2000
        fn(ctypes.c_void_p(out.data_ptr()), blocks, iters, ctypes.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(ctypes.c_void_p(out.data_ptr()), blocks, iters, ctypes.c_void_p(stream.cuda_stream))
            e1.record(stream)
            torch.cuda.synchronize()
            best = max(best, blocks * iters * per / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        res[name + "_tflops"] = round(best, 2)
    return res


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dram_traffic(workload, members):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel per launch, from the
    committed ncu --set full capture (profiles/traffic.json, bytes per member), scaled to this
    launch's member count; None when no capture exists for the workload."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f).get(workload)
    except (OSError, ValueError):
        return None
    return None if not t else round(t["bytes_per_member"] * members)


# ----------------------------------------------------------------------------- CPU oracle leg

def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"] or [1])
    except Exception:
        return None


def _cpu_member(job):
    """Pool worker (spawned, BLAS threads = 1): regenerate cfg5 member b from its seed and run
    the oracle zip-up on it, as it stands.  Returns (b, ranks, cores, seconds)."""
    b, window = job
    from oracle.zipup import zipup as ozip1, zipup_window
    p = gen.cfg5_member(b)
    t0 = time.perf_counter()
    if window == 1:
        r = ozip1(p.kind, p.op.cores, p.x.cores, p.eps, p.max_rank)
    else:
        r = zipup_window(p.kind, p.op.cores, p.x.cores, p.eps, p.max_rank, window=window)
    return b, r["ranks"], r["cores"], time.perf_counter() - t0


def _pool_init():
    pass


def cpu_baseline_cfg5(members, n_sample, window=1):
    """SURVEY.md §8(d) (line 666): the oracle, as it stands, over a deterministic member sample
    b = stride*t of this rank's shard, run by a multiprocessing pool of cpu_count workers with
    BLAS threads = 1 (one member per worker at a time).  The rate (site-steps/s) of the sample
    is the baseline; the full workload's oracle time is that rate's extrapolation (stated)."""
    import multiprocessing as mp
    n = max(1, min(n_sample, len(members)))
    stride = max(1, len(members) // n)
    sample = [members[stride * t] for t in range(n)]
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "BLIS_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in keys}
    for k in keys:
        os.environ[k] = "1"                      # inherited by the spawned workers only
    try:
        ctx = mp.get_context("spawn")
        with ctx.Pool(ncores, initializer=_pool_init) as pool:
            pool.map(abs, range(ncores))         # start every worker before the clock
            t0 = time.perf_counter()
            out = pool.map(_cpu_member, [(b, window) for b in sample], chunksize=1)
            dt = time.perf_counter() - t0
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    L = len(out[0][2])
    steps = n * L
    cpu_s = sum(o[3] for o in out)
    full = len(members) * L / (steps / dt)
    info = {"value": round(steps / dt, 3), "unit": UNIT, "cores": ncores, "kind": "oracle",
            "sample": f"{n} members b = {stride}*t (t < {n}) of the workload's {len(members)}, x {L} sites; "
                      f"multiprocessing pool of {ncores} workers, BLAS threads 1 (SURVEY.md §8(d)); "
                      f"{dt:.1f} s wall, {cpu_s:.1f} core-s; NumPy fp64 + LAPACK gesdd; "
                      f"extrapolated oracle time for all {len(members)} members: {full:.0f} s"}
    return info, {b: (rk, cores) for b, rk, cores, _ in out}


class _Budget(Exception):
    pass


def cpu_baseline_single(p, budget_s, window=1):
    """cfg1-4: one oracle zip-up with BLAS threads = host cores, stopped after
    budget_s seconds at a site boundary (bounded sample).  Returns (info, result or None)."""
    from oracle.zipup import zipup as ozip1, zipup_window
    L = len(p.x.cores)
    done = [0]
    t0 = time.perf_counter()

    marks = [t0]

    def on_site(q):
        # stop at a site boundary when the next site, predicted from the growth of the last two,
        # would overrun the budget (a site cannot be interrupted)
        done[0] = q + 1
        now = time.perf_counter()
        marks.append(now)
        last = marks[-1] - marks[-2]
        prev = marks[-2] - marks[-3] if len(marks) > 2 else last
        pred = last * min(8.0, max(1.0, last / max(prev, 1e-9)))
        if now - t0 + pred > budget_s:
            raise _Budget()

    res = None
    try:
        if window == 1:
            res = ozip1(p.kind, None if p.op is None else p.op.cores, p.x.cores, p.eps, p.max_rank, on_site=on_site)
            done[0] = L
        else:
            res = zipup_window(p.kind, None if p.op is None else p.op.cores, p.x.cores, p.eps, p.max_rank,
                               window=window)
            done[0] = L
    except _Budget:
        res = None
    dt = time.perf_counter() - t0
    whole = done[0] == L
    info = {"value": round(done[0] / dt, 4), "unit": UNIT, "cores": _blas_threads() or os.cpu_count(),
            "kind": "oracle",
            "sample": (f"one full zip-up ({L} sites), {dt:.1f} s wall" if whole else
                       f"sites 0..{done[0] - 1} of {L} (stopped at the {budget_s:.0f} s budget; the early sites are "
                       f"the small ones, so this rate is an upper bound on the oracle's), {dt:.1f} s wall")
                      + f"; one process, NumPy fp64 + LAPACK gesdd, BLAS threads {_blas_threads()}"}
    return info, res


# ----------------------------------------------------------------------------- main

def self_launch(args):
    """`bench.py --gpus N` outside torchrun: re-exec this command under torch.distributed.run with
    N ranks (one process per GPU, rendezvous on 127.0.0.1), so the line measures N GPUs."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print("bench.py: launching " + " ".join(cmd), file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        if args.gpus != 1:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        args.gpus = world
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference" and args.workload == "qft":
        return run_qft_reference(args, rank)
    if args.impl == "reference" and args.workload == "variational":
        return run_variational_reference(args, rank)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.workload == "qft":
        return run_qft(args, rank, world, local)
    if args.workload == "variational":
        return run_variational(args, rank, world, local)

    import torch
    import torch.distributed as dist
    from paper_2602_20226_b200 import qtt

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()

    subs, kind, probs, xs, ops, cfg = build_workload(args, rank)
    if args.window == 2:
        cfg = dict(cfg, window=2)
    mpo = kind == "matvec"
    npdt = np.float32 if args.dtype == "f32" else np.float64
    xd = qtt.to_device(xs, dtype=npdt)
    od = None if ops is None else qtt.to_device(ops, mpo=mpo, dtype=npdt)
    p0 = probs[0]
    wflags = qtt.WINDOW2 if args.window == 2 else 0
    plan = qtt.ZipupPlan(subs, od, xd, p0.eps, p0.max_rank, flags=wflags, sweeps=True, cycles=True)
    L = xd.n_sites
    B = xd.batch
    summary = torch.zeros(4, dtype=torch.float64, device="cuda")

    def step(events=None):
        res = plan.run(od, xd, events=events)
        s = qtt.summary(res)
        qdist.allreduce_summary(s, dist)          # the one cross-GPU exchange (a8)
        summary.copy_(s)
        return res

    peaks = fp64_peaks(torch, stream)
    for _ in range(max(args.warmup, 3)):
        res = step()
    torch.cuda.synchronize()
    assert int(res.status.item()) == 0, f"device status {int(res.status.item())}"

    # ---------------- timed region (device time, max over ranks)
    ev_sets = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for ev in ev_sets:          # torch creates the CUDA event lazily: force it before handing the handle over
        for e in ev:
            e.record(stream)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.25)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(args.steps):
        step(ev_sets[k])
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / args.steps
    ms_max = qdist.max_over_ranks(ms, "cuda", dist)

    # per-kernel device time of the dominant kernel (k_site) from the live events
    site_ms = sum(ev[2].elapsed_time(ev[3]) for ev in ev_sets)
    orth_ms = sum(ev[0].elapsed_time(ev[1]) for ev in ev_sets)
    ranks = res.ranks.cpu().numpy()
    sweeps = res.sweeps.cpu().numpy()
    cyc = res.cycles.cpu().numpy().astype(np.float64).sum(axis=(0, 1))
    phase_share = None if not cyc.sum() > 0 else {      # the large-member path has no phase counters
        k: round(float(v / cyc.sum()), 4) for k, v in
        zip(("a2_contract", "a3_qr", "a4_jacobi", "a5_a6_trunc_emit_carry"), cyc)}
    d = xd.d_out if kind != "matvec" else od.d_out
    dj = xd.d_out
    tot = np.zeros(4)
    for b in range(B):
        f = site_flops(kind, list(ranks[b]), xd.ranks, od.ranks if od is not None else None, d, dj, sweeps[b],
                       args.window)
        tot += np.sum(np.array(f), axis=0)
    flops_alg = tot[0] + tot[1] + tot[2]          # contract + QR + carry, Jacobi excluded
    site_s = site_ms * 1e-3 / args.steps
    fp64_peak = max(peaks["dfma_tflops"], peaks["dmma_tflops"])
    achieved = flops_alg / site_s / 1e12
    jac_share = phase_share["a4_jacobi"] if phase_share else None
    jacobi = {"flops_executed_per_step": tot[3], "sweeps_mean": float(sweeps[:, :-1].mean()),
              "sweeps_max": int(sweeps.max()),
              "note": "sweep-dependent work, excluded from the algorithmic rate (SURVEY.md §8(d))"}
    if jac_share:
        jt = site_s * jac_share
        jacobi.update({"time_share_of_kernel": jac_share, "ms_per_step": round(jt * 1e3, 3),
                       "fp64_tflops_executed": round(tot[3] / jt / 1e12, 3),
                       "fp64_frac_executed": round(tot[3] / jt / 1e12 / fp64_peak, 4)})
    launches_per_step = 3 + (1 if kind != "truncate" else 0)   # a1 (x[, op]), k_sweep, summary
    if args.window == 2:
        launches_per_step = 3 + (1 if kind != "truncate" else 0)   # a1 (x[, op]), k_zipup<double>, summary
    if od is not None and getattr(od, "batch", B) == 1 and B > 1:
        launches_per_step += 1                                    # shared operator: rank broadcast

    units = world * B * L
    value = units / (ms_max * 1e-3)
    traffic = dram_traffic(args.workload, B)

    # ---------------- e2e through the public API with host buffers
    # qtt.HostPipeline: every step copies its inputs host->device and its results device->host
    # inside the timed region; with two buffer sets the copies of steps k+1 / k-1 overlap the
    # zip-up of step k (copy engines vs SMs), as a streaming user of the library would run it.
    e2e = None
    if not args.no_e2e:
        depth = 2
        pipe = qtt.HostPipeline(subs, od, xd, p0.eps, p0.max_rank, depth=depth, flags=wflags)
        hx = [c.detach().cpu().pin_memory() for c in xd.cores]
        ho = [c.detach().cpu().pin_memory() for c in od.cores] if od is not None else None
        hsets = []
        for _ in range(depth):
            hsets.append(([torch.empty(c.shape, dtype=c.dtype).pin_memory() for c in plan.out.cores],
                          torch.empty(tuple(plan.ranks.shape), dtype=plan.ranks.dtype).pin_memory(),
                          torch.empty(tuple(plan.delta2.shape), dtype=torch.float64).pin_memory(),
                          torch.empty(tuple(plan.norm2.shape), dtype=torch.float64).pin_memory()))
        h2d = sum(t.numel() * t.element_size() for t in hx + (ho or []))
        hout0, hr0, hd0, hn0 = hsets[0]
        d2h = sum(t.numel() * t.element_size() for t in hout0) + hr0.numel() * 4 + hd0.numel() * 8 + hn0.numel() * 8
        kstep = [0]

        def e2e_step():
            hout, hr, hd, hn = hsets[kstep[0] % depth]
            kstep[0] += 1
            r = pipe.step(hx, ho, hout, hr, hd, hn, stream=stream)
            s = qtt.summary(r)
            qdist.allreduce_summary(s, dist)
            summary.copy_(s)

        for _ in range(depth):
            e2e_step()
        pipe.finish(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        pipe.begin(stream)
        for _ in range(args.steps):
            e2e_step()
        pipe.finish(stream)
        a1.record(stream)
        torch.cuda.synchronize()
        ems = qdist.max_over_ranks(a0.elapsed_time(a1) / args.steps, "cuda", dist)
        # the last step's host results must match the device-timed run's (same inputs)
        hout, hr, hd, hn = hsets[(kstep[0] - 1) % depth]
        assert torch.equal(hr, plan.ranks.cpu()), "e2e ranks differ from the device-resident run"
        e2e = {"value": units / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ems, 3),
               "pipeline": f"{depth} buffer sets: H2D of step k+1 and D2H of step k-1 overlap step k's zip-up"}

    # ---------------- CPU oracle baseline + sampled parity (rank 0, N=1 only)
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import tt
        worst, n_cmp, ranks_equal = 0.0, 0, True
        if args.workload == "cfg5":
            members = [int(pp.meta["member"]) for pp in probs]
            cpu, refs = cpu_baseline_cfg5(members, args.cpu_members, args.window)
            for b, (rk_ref, cores_ref) in refs.items():
                i = members.index(b)
                rk = [int(v) for v in ranks[i]]
                if rk != rk_ref:
                    ranks_equal = False
                    continue
                yg = qtt.member_cores(plan.out, rk, i)
                worst = max(worst, tt.diff_norm(yg, cores_ref) / tt.qr_norm(cores_ref))
                n_cmp += 1
        else:
            cpu, ref = cpu_baseline_single(probs[0], args.cpu_budget_s, args.window)
            if ref is not None:
                rk = [int(v) for v in ranks[0]]
                ranks_equal = rk == ref["ranks"]
                if ranks_equal:
                    yg = qtt.member_cores(plan.out, rk, 0)
                    worst = tt.diff_norm(yg, ref["cores"]) / tt.qr_norm(ref["cores"])
                    n_cmp = 1
        parity = {"members": n_cmp, "max_rel_fro": worst, "ranks_equal": ranks_equal,
                  "how": "QR-sweep norm of the exact difference train / QR-sweep norm of the oracle's (c-A29)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms_max, 3), "higher_is_better": True,
            "scaling": ("strong" if args.strong else "weak") if args.workload == "cfg5" else "replicas",
            "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded generators, BASELINE.json configs)",
            "config": dict(cfg, l2="inputs %.2f GB/GPU%s" % (
                sum(c.numel() * c.element_size() for c in xd.cores) / 1e9,
                " > 126 MB L2: no flush needed" if args.workload == "cfg5" else
                " (single zip-up; its per-site scratch exceeds L2 for cfg3/cfg4)")),
            "alg_tflops": round(world * flops_alg / (ms_max * 1e-3) / 1e12, 3),
            "alg_tflops_note": "whole step: contraction+QR+carry flops (SURVEY.md §8(d)) / ms_per_step; Jacobi excluded",
            "roofline": {"kernel": (("k_sweep (persistent a2-a7 over all sites and members)" if B * L > 0 and
                                     args.workload in ("cfg1", "cfg5") else
                                     "large-member path (per site: k_gemm_dmma, k_qr_coop, k_jacobi_coop, k_finish)")
                                    if args.window == 1 else "k_zipup<double> (window 2: one CTA per member, every step)"),
                         "bound": "fp64",
                         "achieved": round(achieved, 4), "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": round(achieved / fp64_peak, 4), "traffic": traffic,
                         "achieved_def": "SURVEY.md §8(d) algorithmic flops of the launch (sum over sites and members "
                                         "of F_contract + F_qr + F_carry; Jacobi excluded) / the launch's CUDA-event time",
                         "peak_source": "FP64 (DMMA/DFMA) measured in this run by csrc/probe/peak.cu "
                                        "(MEASURED_PEAKS.json has no FP64 entry)",
                         "alg_flops_per_step": flops_alg, "kernel_ms_per_step": round(site_ms / args.steps, 3),
                         "share_of_step": round(site_ms / args.steps / ms, 4),
                         "flop_split": {"contract": tot[0], "qr": tot[1], "carry": tot[2]},
                         "prepass_ms_per_step": round(orth_ms / args.steps, 3)},
            "jacobi": jacobi,
            "fp64_peaks": peaks, "site_kernel_phase_share": phase_share,
            "cpu_baseline": cpu, "parity_sample": parity, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps, "clocks": clk,
            "summary": qdist.summary_dict(summary.cpu().tolist()),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


QFT_BASES = [2] * 13
QFT_RANK = 16


def _qft_cfg(world):
    return {"workload": "f2: tensorized DFT N=2^13 (PAPER.md:533-566) as a chain of 12 complex128 Hadamard "
                        "zip-ups of the rank-2 factor trains, max rank 16, eps 0",
            "N": 2 ** 13, "sites": 13, "max_rank": QFT_RANK, "members_per_gpu": 1, "global_batch": max(world, 1),
            "parallelism": f"replicas x{max(world, 1)}",
            "l2": "working set < L2 (a latency-bound chain of 12 dependent calls): no flush"}


def run_qft(args, rank, world, local):
    """--workload qft: one step = the whole 12-call chain Y_q = zip-up(T_q o Y_{q-1}); the
    output ranks of each call are read on the host to size the next (member_view), so the
    timed region includes those 12 small device->host reads.  ZipupPlans (outputs + workspace)
    are cached per call and input ranks, as a repeated user would hold them."""
    import torch
    import torch.distributed as dist
    from paper_2602_20226_b200 import qtt
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    T = [t.cores for t in gen.qft_trains(QFT_BASES)]
    dev = [qtt.to_device(t, dtype=np.complex128) for t in T]
    n = len(QFT_BASES)

    plans = {}                                          # ZipupPlan per (call, input ranks): reused

    def chain(inputs, sweeps_out=None):
        y = inputs[0]
        keep = []
        for q in range(1, n):
            key = (q, tuple(y.ranks), sweeps_out is not None)
            plan = plans.get(key)
            if plan is None:
                plan = plans[key] = qtt.ZipupPlan("i,i->i", inputs[q], y, 0.0, QFT_RANK, sweeps=sweeps_out is not None)
            res = plan.run(inputs[q], y)
            ranks = res.ranks[0].cpu().tolist()            # host sizes for the next call
            if sweeps_out is not None:
                sweeps_out.append((list(ranks), res.sweeps[0].cpu().tolist(), list(y.ranks), list(inputs[q].ranks)))
            y = qtt.member_view(res.out, ranks, 0)
            keep.append(plan)
        return y, keep

    for _ in range(max(args.warmup, 3)):
        y, keep = chain(dev)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    clocks.start()
    time.sleep(0.25)
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        y, keep = chain(dev)
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = qdist.max_over_ranks(t0.elapsed_time(t1) / args.steps, "cuda", dist)
    units = max(world, 1) * (n - 1) * n                 # site steps per chain, all replicas
    value = units / (ms * 1e-3)
    # algorithmic flops (complex: 4 real flops per complex multiply-add pair -> x4 the real model)
    info = []
    chain(dev, info)
    torch.cuda.synchronize()
    fl = 0.0
    for ranks, sw, yr, tr in info:
        f = site_flops("hadamard", ranks, yr, tr, [4] * n, [4] * n, sw)
        fl += 4.0 * sum(sum(v) for v in f)
    # e2e: factor trains copied from pinned host memory, result cores copied back, every step
    hT = [[torch.from_numpy(np.ascontiguousarray(c[None])).pin_memory() for c in t] for t in T]
    h2d = sum(c.numel() * c.element_size() for t in hT for c in t)

    def e2e_step():
        for dt_, ht in zip(dev, hT):
            for dst, src in zip(dt_.cores, ht):
                dst.copy_(src, non_blocking=True)
        yy, kk = chain(dev)
        outs = [c.cpu() for c in yy.cores]
        return sum(c.numel() * c.element_size() for c in outs)

    e2e_step()
    torch.cuda.synchronize()
    a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    d2h = 0
    for _ in range(args.steps):
        d2h = e2e_step()
    a1.record(stream)
    torch.cuda.synchronize()
    ems = qdist.max_over_ranks(a0.elapsed_time(a1) / args.steps, "cuda", dist)
    peaks = fp64_peaks(torch, stream)
    per_sm = max(peaks["dfma_tflops"], peaks["dmma_tflops"]) / torch.cuda.get_device_properties(local).multi_processor_count
    achieved = fl / (ms * 1e-3) / 1e12
    cpu = None
    dist_err = None
    if rank == 0 and world == 1:
        from oracle import qft as oqft
        ycores = qtt.member_cores(y, y.ranks, 0)
        dist_err = float(np.linalg.norm(oqft.to_matrix(ycores, QFT_BASES) - oqft.dft_matrix(2 ** 13))) / math.sqrt(2 ** 13)
        if not args.no_cpu_baseline:
            c0 = time.perf_counter()
            oqft.chain(T, QFT_RANK)
            cdt = time.perf_counter() - c0
            cpu = {"value": (n - 1) * n / cdt, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"one full chain (12 zip-ups) with NumPy complex128 + LAPACK zgesdd, {cdt:.2f} s wall"}
    if rank == 0:
        line = {"metric": METRIC + " (f2 Fourier chain)", "value": round(value, 3), "unit": UNIT, "n_gpus": max(world, 1),
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
                "scaling": "replicas", "vs_baseline": None, "dtype": "c128",
                "data": "the paper's closed-form DFT factor trains (gen.qft_trains)", "config": _qft_cfg(world),
                "roofline": {"kernel": "k_zipup<complex> (one CTA per member: the chain has one member)", "bound": "alu",
                             "achieved": round(achieved, 6), "peak": round(per_sm, 4), "unit": "TFLOP/s",
                             "frac": round(achieved / per_sm, 5), "traffic": None,
                             "peak_source": "measured FP64 peak / SM count (one CTA runs the member)"},
                "distance_over_sqrtN": dist_err, "paper_distance": 9.3e-11,
                "jacobi_sweeps": {"mean": float(np.mean([v for _, sw, _, _ in info for v in sw[:-1]])),
                                  "max": int(max(v for _, sw, _, _ in info for v in sw))},
                "cpu_baseline": cpu,
                "e2e": {"value": units / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ems, 3)},
                "gpu_launches": (n - 1) * args.steps, "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def variational_flops(kind, L, d, dj, xr, orr, cr, ncores):
    """Algorithmic flops of one variational sweep of one member (contractions + QR/LQ centre
    moves; the two-site split's Jacobi excluded, as for the zip-up) from the
    final ranks cr of C (two-site ranks adapt during the sweep: an estimate at the final ranks)."""
    f = 0.0
    for q in range(L):
        c, c2, r, r2 = cr[q], cr[q + 1], xr[q], xr[q + 1]
        w, w2 = (orr[q], orr[q + 1]) if kind != "truncate" else (1, 1)
        left = 2.0 * c * w * r * dj[q] * r2 + 2.0 * c * d[q] * w2 * r2 * w * dj[q]      # X1, X2 (env_apply_left)
        if ncores == 1:
            upd = left + 2.0 * c * d[q] * w2 * r2 * c2                                    # C_q = X2 Re^T
            move = 2.0 * (c * d[q]) * c2 * c2 - (2.0 / 3.0) * c2 ** 3                      # QR / LQ
            env = 2.0 * c2 * w2 * r2 * c * d[q] + (2.0 * c * d[q] * c2 * w2 * r2 + 2.0 * c * w * dj[q] * r2 * d[q] * w2
                                                   + 2.0 * c * w * r * dj[q] * r2)          # Le / Re updates
            f += 2 * (upd + move) + env
        elif q < L - 1:
            c3, r3 = cr[q + 2], xr[q + 2]
            w3 = orr[q + 2] if kind != "truncate" else 1
            m, n = c * d[q], d[q + 1] * c3
            second = 2.0 * m * w2 * r2 * dj[q + 1] * r3 + 2.0 * m * d[q + 1] * w3 * r3 * w2 * dj[q + 1]
            split = 2.0 * m * d[q + 1] * w3 * r3 * c3                                        # S = Z Re^T
            qr = (2.0 * n * m * m - (2.0 / 3.0) * m ** 3) if m <= n else (2.0 * m * n * n - (2.0 / 3.0) * n ** 3)
            carry = 2.0 * c2 * m * n
            env = 2.0 * c2 * w2 * r2 * c * d[q] + (2.0 * c * d[q] * c2 * w2 * r2 + 2.0 * c * w * dj[q] * r2 * d[q] * w2
                                                   + 2.0 * c * w * r * dj[q] * r2)
            f += 2 * (left + second + split + qr + carry) + env
    return f


def run_variational(args, rank, world, local):
    """--workload variational (f3): cfg5 members (this rank's shard) seeded by a max-rank-16
    zip-up (untimed); one step = one qtt_variational sweep (right and back) over every member.
    Unit: site updates per second (2 L per member per sweep)."""
    import torch
    import torch.distributed as dist
    from paper_2602_20226_b200 import qtt
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    M = args.members_per_gpu
    lo, hi = qdist.member_range(rank, max(world, 1), M)
    probs, xs, ops = gen.cfg5_batch_arrays(list(range(lo, hi)))
    xd, od = qtt.to_device(xs), qtt.to_device(ops, mpo=True)
    seed = qtt.ZipupPlan("ij,j->i", od, xd, 1e-10, 16).run(od, xd)
    L, B = xd.n_sites, xd.batch
    nc = args.ncores
    vkw = dict(ncores=nc, eps=0.0, max_rank=16) if nc == 2 else {}
    for _ in range(max(args.warmup, 3)):
        v = qtt.variational("ij,j->i", od, xd, seed, 1, **vkw)
    torch.cuda.synchronize()
    assert int(v.status.item()) == 0
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    clocks.start()
    time.sleep(0.25)
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        v = qtt.variational("ij,j->i", od, xd, seed, 1, **vkw)
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = qdist.max_over_ranks(t0.elapsed_time(t1) / args.steps, "cuda", dist)
    units = max(world, 1) * B * (2 * L if nc == 1 else 2 * (L - 1))
    value = units / (ms * 1e-3)
    vr = v.ranks.cpu().numpy()
    d5 = [2] * L
    flops = sum(variational_flops("matvec", L, d5, d5, xd.ranks, od.ranks, [int(t) for t in vr[b]], nc)
                for b in range(B))
    peaks = fp64_peaks(torch, stream)
    fp64_peak = max(peaks["dfma_tflops"], peaks["dmma_tflops"])
    achieved = flops / (ms * 1e-3) / 1e12
    cpu = None
    gain = None
    if rank == 0 and world == 1:
        from oracle import tt
        from oracle.variational import variational as ovar
        b = 0
        sd = qtt.member_cores(seed.out, seed.ranks[b].cpu().tolist(), b)
        got = qtt.member_cores(v.out, v.ranks[b].cpu().tolist(), b)
        ex = tt.exact_matvec(probs[b].op.cores, probs[b].x.cores)
        gain = {"member": b, "dist_seed": tt.diff_norm(sd, ex), "dist_after_1_sweep": tt.diff_norm(got, ex)}
        if not args.no_cpu_baseline:
            c0 = time.perf_counter()
            ref = ovar("matvec", probs[b].op.cores, probs[b].x.cores, sd, 1, ncores=nc, eps=0.0,
                       max_rank=16 if nc == 2 else 0)
            cdt = time.perf_counter() - c0
            gain["parity_vs_oracle"] = tt.diff_norm(got, ref["cores"]) / tt.qr_norm(ref["cores"])
            cpu = {"value": (units / max(world, 1) / B) / cdt, "unit": "site-updates/s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"one member, one sweep, NumPy einsum + LAPACK QR, {cdt:.2f} s wall"}
    if rank == 0:
        line = {"metric": "variational site updates/sec (f3)", "value": round(value, 3), "unit": "site-updates/s",
                "n_gpus": max(world, 1), "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (cfg5 members, seeded generators)",
                "config": {"workload": ("f3: one single-site variational sweep" if nc == 1 else
                                        "f3: one two-site (ncores=2, max_rank 16, cutoff 0) variational sweep")
                                       + " (PAPER.md:277-301) on cfg5 members seeded by a max-rank-16 zip-up",
                           "members_per_gpu": M, "ncores": nc,
                           "global_batch": M * max(world, 1), "L": L, "seed_max_rank": 16,
                           "parallelism": f"dp{max(world, 1)} (members sharded)"},
                "roofline": {"kernel": "k_variational (one CTA per member, environments in global memory)",
                             "bound": "fp64", "achieved": round(achieved, 4), "peak": fp64_peak, "unit": "TFLOP/s",
                             "frac": round(achieved / fp64_peak, 5), "traffic": None,
                             "achieved_def": "bench.variational_flops (contractions + centre-move QR; the two-site "
                                             "split's Jacobi excluded) at the final ranks / sweep time",
                             "peak_source": "FP64 measured in this run by csrc/probe/peak.cu"},
                "distance": gain, "cpu_baseline": cpu, "e2e": None,
                "gpu_launches": args.steps, "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_variational_reference(args, rank):
    """--impl reference for --workload variational: the oracle's sweep on one member (bounded
    sample) with the GPU arm's config and unit."""
    if rank != 0:
        return
    from oracle.zipup import zipup as ozip
    from oracle.variational import variational as ovar
    probs, xs, ops = gen.cfg5_batch_arrays([0])
    p = probs[0]
    seed = ozip("matvec", p.op.cores, p.x.cores, 1e-10, 16)["cores"]
    L = len(p.x.cores)
    nc = args.ncores
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ovar("matvec", p.op.cores, p.x.cores, seed, 1, ncores=nc, eps=0.0, max_rank=16 if nc == 2 else 0)
    dt = (time.perf_counter() - t0) / args.steps
    value = (2 * L if nc == 1 else 2 * (L - 1)) / dt
    line = {"metric": "variational site updates/sec (f3)", "value": round(value, 3), "unit": "site-updates/s",
            "n_gpus": 1, "steps": args.steps, "warmup": 0, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
            "data": "synthetic (cfg5 members, seeded generators)",
            "config": {"workload": "f3: one single-site variational sweep (PAPER.md:277-301) on cfg5 members "
                                   "seeded by a max-rank-16 zip-up", "members_per_gpu": args.members_per_gpu,
                       "global_batch": args.members_per_gpu, "L": L, "seed_max_rank": 16, "parallelism": "dp1"},
            "cpu_baseline": {"value": round(value, 3), "unit": "site-updates/s", "cores": os.cpu_count(),
                             "kind": "oracle", "sample": "each step: one member, one sweep (oracle)"},
            "e2e": {"value": round(value, 3), "unit": "site-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_qft_reference(args, rank):
    if rank != 0:
        return
    from oracle import qft as oqft
    T = [t.cores for t in gen.qft_trains(QFT_BASES)]
    n = len(QFT_BASES)
    for _ in range(args.warmup):
        oqft.chain(T, QFT_RANK)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oqft.chain(T, QFT_RANK)
    dt = (time.perf_counter() - t0) / args.steps
    value = (n - 1) * n / dt
    line = {"metric": METRIC + " (f2 Fourier chain)", "value": round(value, 3), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
            "scaling": "replicas", "vs_baseline": None, "dtype": "c128", "impl": "reference",
            "data": "the paper's closed-form DFT factor trains (gen.qft_trains)", "config": _qft_cfg(1),
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                             "sample": "each step: one full chain (oracle)"},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (as it stands) on the host cores, on this arm's config,
    metric and unit.  Each step is a bounded sample of the workload: cfg5 -- one member per host
    core (members b = stride*t of rank 0's shard), a spawned pool with BLAS threads 1 (SURVEY.md
    §8(d)); cfg1-4 -- one oracle zip-up stopped at a per-step time budget.  Rank 0 only."""
    if rank != 0:
        return
    subs, kind, probs, xs, ops, cfg = build_workload(args, 0)
    if args.window == 2:
        cfg = dict(cfg, window=2)
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    vals, info = [], None
    budget = max(2.0, min(args.cpu_budget_s, 150.0 / max(1, args.steps + args.warmup)))
    t0 = None
    for it in range(args.warmup + args.steps):
        if it == args.warmup:
            t0 = time.perf_counter()
        if args.workload == "cfg5":
            members = [int(pp.meta["member"]) for pp in probs]
            info, _ = cpu_baseline_cfg5(members, ncores, args.window)
        else:
            info, _ = cpu_baseline_single(probs[0], budget, args.window)
        if it >= args.warmup:
            vals.append(info["value"])
    dt = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": ("strong" if args.strong else "weak") if args.workload == "cfg5" else "replicas",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, BASELINE.json configs)", "impl": "reference",
            "config": cfg,
            "cpu_baseline": dict(info, value=round(value, 4),
                                 sample="each step: " + info["sample"] + f"; median of {args.steps} steps"),
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
