#!/usr/bin/env python
"""Benchmark of the B200 SR-FMG solve (BASELINE.json metric: fine-grid cells solved/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C3] [--dtype f64|f32]

A step is one complete FMG+SR solve (sr_fmg_solve) of the workload: f-pyramid, coarsest
solve, conventional FMG below the transition level, K SR levels, output gather.  Prints one
JSON line on rank 0.  Default workload C3 (BASELINE.json configs[2]): 512^3 cells, fp64,
manufactured f + N(0, 1e-3) noise, 8^3 segments of 64^3, buffer 2, 4 SR levels, M = 8 --
the largest single-GPU configuration (configs[0]/[1] are the small parity cases).

`--impl reference` times the CPU oracle (oracle/, the test reference implementation) on a
bounded sample of the same workload on the host cores.
"""
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

import workloads as W  # noqa: E402

WORKLOADS = {
    # name: (n, M, seg, buffer, K, rhs)
    "C1": ((32, 32, 32), 4, 16, 2, 2, "manufactured"),
    "C2": ((128, 128, 128), 6, 32, 2, 3, "manufactured"),
    "C3": ((512, 512, 512), 8, 64, 2, 4, "manufactured+noise"),
    "C5": ((1024, 1024, 1024), 9, 128, 2, 4, "bumps"),
    "C5-s32": ((1024, 1024, 1024), 9, 32, 2, 4, "bumps"),  # C5's other segment size
    # the paper's own model problem: Omega = [0,2]x[0,1]^2, 27-point operator
    # (use with --stencil 27pt), 64^3 segments, J = 2, K = 4, pN0V = 4
    "P27": ((1024, 512, 512), 8, 64, 2, 4, "manufactured"),
}
# bounded CPU sample of C3 for the oracle: the same 8^3 segment grid, K = 4, J = 2, at
# 128^3 (1/64 of the cells); about 7 s of numpy per solve on one core
ORACLE_SAMPLE = dict(n=(128, 128, 128), M=6, seg=16, buffer=2, K=4, rhs="manufactured+noise")
PGRID = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
# kernel classes (sr_fmg_kernel_name) that can dominate the finest level: the roofline line
# reports the one with the largest device time per solve
KC_CANDIDATES = (1, 3, 7, 8, 10)  # k_restrict, k_prolong, k_cheb2, entry (Pi + S^1), up pass


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(WORKLOADS) + ["C4"],
                    help="default: C3 on 1 GPU, C4 (weak scaling, 512^3 per GPU) on N > 1")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--stencil", default="7pt", choices=["7pt", "27pt"],
                    help="27pt: the paper's operator (SURVEY f1; unfused kernels)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true")
    return ap.parse_args()


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms; started before the warm-up so
    that it is already sampling when the (short) timed region begins, and reduced to the
    samples that arrived inside that region (window(t0, t1), monotonic host clock)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.win = None

    def window(self, t0, t1):
        self.win = (t0, t1)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        if not self.rows:
            return None
        inside = True
        rows = self.rows
        if self.win:  # samples arriving inside the region (+ one period of lag)
            t0, t1 = self.win
            rows = [r for t, r in self.rows if t0 <= t <= t1 + 0.06]
            if not rows:  # region shorter than the sampling period: the nearest samples
                inside = False
                rows = [r for t, r in self.rows if t0 - 0.3 <= t <= t1 + 0.3]
        else:
            rows = [r for _, r in self.rows]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > i + 2 and r[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "in_timed_region": inside}


def oracle_sample_solve():
    import oracle as O
    s = ORACLE_SAMPLE
    f = W.make_rhs(s["rhs"], s["n"])
    cfg = O.Config(n=s["n"], M=s["M"], seg=s["seg"], buffer=s["buffer"], K=s["K"])
    t0 = time.perf_counter()
    O.solve(f, cfg)
    return time.perf_counter() - t0, float(np.prod(s["n"]))


def sample_desc():
    s = ORACLE_SAMPLE
    return (f"oracle (numpy fp64) FMG+SR solve of {s['n'][0]}^3 cells, M={s['M']}, "
            f"seg={s['seg']} (8^3 segments), buffer={s['buffer']}, K={s['K']}, "
            f"{s['rhs']} rhs: the C3 segment grid/K/J at 1/64 of the cells")


def mem_available_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 1e6
    except Exception:
        pass
    return 0.0


def oracle_full_solve(n, M, seg, buf, K, rhs, h):
    """The oracle, as it stands, on the bench workload itself: one solve of
    the same f on the host; returns (seconds, cells, cores used = CPU time / wall time)."""
    import resource

    import oracle as O
    f = W.make_rhs(rhs, n, h=h)
    cfg = O.Config(n=n, M=M, seg=seg, buffer=buf, K=K, h=h)
    r0 = resource.getrusage(resource.RUSAGE_SELF)
    t0 = time.perf_counter()
    O.solve(f, cfg)
    t = time.perf_counter() - t0
    r1 = resource.getrusage(resource.RUSAGE_SELF)
    cpu = (r1.ru_utime - r0.ru_utime) + (r1.ru_stime - r0.ru_stime)
    return t, float(np.prod(n)), max(1, round(cpu / t))


def accuracy(solver_args, n, M, seg, buf, K, h, dtype, f_bench, u_bench):
    """Accuracy of the measured configuration (north_star: the GPU must match the error-to-
    discretisation-error ratios; PAPER.md:262-264 defines e_r = ||e_SR||_inf/||e_FMG||_inf).
    * the manufactured f alone (no noise): e_SR = ||u_SR - u||_inf and e_FMG (K = 0) against the
      exact u, e_disc = ||u_h* - u||_inf with u_h* = A^-1 f by DST (tests/pins.py), e_r;
    * the bench's own f: the algebraic error ||u - u_h*||_inf against u_h* of that f."""
    import torch

    from paper_1406_7808_b200 import Solver
    from tests import pins
    npd = np.float64 if dtype == "f64" else np.float32
    fm = W.manufactured_f(n, h)
    ue = W.manufactured_u(n, h)
    out = {"rhs": "manufactured f (no noise) for e_r; the bench f for e_alg",
           "norm": "max norm over the fine grid"}
    ft = torch.from_numpy(fm.astype(npd)).cuda()
    u_sr = solver_args["solver"].solve(ft).double().cpu().numpy()
    with Solver(n, M, seg=seg, buffer=buf, K=0, dtype=dtype, h=h) as s0:
        u_fmg = s0.solve(ft).double().cpu().numpy()
    del ft
    ustar = pins.dst_solve(fm, h)
    e_sr = float(np.abs(u_sr - ue).max())
    e_fmg = float(np.abs(u_fmg - ue).max())
    e_disc = float(np.abs(ustar - ue).max())
    out.update({"e_sr_inf": e_sr, "e_fmg_inf": e_fmg, "e_disc_inf": e_disc,
                "e_r": e_sr / e_fmg,
                "e_sr_alg_over_disc": float(np.abs(u_sr - ustar).max()) / e_disc,
                "e_fmg_alg_over_disc": float(np.abs(u_fmg - ustar).max()) / e_disc})
    if f_bench is not None:
        ub = pins.dst_solve(np.asarray(f_bench, dtype=np.float64), h)
        out["bench_f_e_alg_inf"] = float(np.abs(np.asarray(u_bench, np.float64) - ub).max())
        out["bench_f_e_alg_rel_l2"] = float(np.linalg.norm(u_bench - ub) / np.linalg.norm(ub))
    return out


def ref_workload():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1:
        return ("C3: global 512x512x512 cells (134217728 per GPU), M=8, seg=64, buffer=2, K=4 SR "
                "levels, F(1,2,2), rhs manufactured+noise, 7pt operator")
    P = PGRID.get(world, (world, 1, 1))
    n = (512 * P[0], 512 * P[1], 512 * P[2])
    return (f"C4: global {n[0]}x{n[1]}x{n[2]} cells (134217728 per GPU), M=8, seg=64, buffer=2, "
            "K=4 SR levels, F(1,2,2), rhs manufactured, 7pt operator")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        oracle_sample_solve()
    ts, cells = [], 0.0
    for _ in range(args.steps):
        t, cells = oracle_sample_solve()
        ts.append(t)
    tot = sum(ts)
    value = cells * len(ts) / tot
    line = {
        "impl": "reference", "metric": "fine-grid cells solved/s (FMG+SR, fp64)", "value": value,
        "unit": "cells/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(ts), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic ({ORACLE_SAMPLE['rhs']}, seed {W.SEED})",
        # our arm's workload (C3 on one GPU, C4 weak scaling on N); every step is a bounded
        # sample of it on this host (same segment grid, K, J)
        "config": {"workload": ref_workload(), "sample": sample_desc()},
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": 1, "kind": "oracle",
                         "sample": sample_desc()},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1406_7808_b200 import Solver, nccl_unique_id

    config = args.config or ("C3" if world == 1 else "C4")
    npd = np.float64 if args.dtype == "f64" else np.float32
    if config == "C4":
        # weak scaling (BASELINE configs[3]): 512^3 cells per GPU on the global grid
        # (512 P1, 512 P2, 512 P3), h = 1/512, R = pgrid, manufactured f, M = 8 (coarsest 2R)
        P = PGRID.get(world, (world, 1, 1))
        n = (512 * P[0], 512 * P[1], 512 * P[2])
        M, seg, buf, K, rhs, h = 8, 64, 2, 4, "manufactured", 1.0 / 512
    else:
        # one global problem; on N GPUs its segment grid is split into pgrid blocks (strong
        # scaling, BASELINE configs[4] for C5)
        P = PGRID.get(world, (world, 1, 1)) if world > 1 else (1, 1, 1)
        n, M, seg, buf, K, rhs = WORKLOADS[config]
        h = 1.0 / n[0] if config != "P27" else 2.0 / n[0]
    nccl_id = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    solver = Solver(n, M, seg=seg, buffer=buf, K=K, dtype=args.dtype, h=h, world=world,
                    rank=rank, pgrid=P, nccl_id=nccl_id, stencil=args.stencil)
    if world == 1 and config != "C4":
        f_host = W.make_rhs(rhs, n, h=h).astype(npd)
    else:
        # this rank's haloed block (evaluated on the block for the analytic kinds)
        lo = [solver.block_lo[d] - solver.f_halo for d in range(3)]
        dims = [solver.block_n[d] + 2 * solver.f_halo for d in range(3)]
        f_host = W.rhs_block(rhs, n, h, lo, dims).astype(npd)
    f = torch.from_numpy(f_host).cuda()
    u = torch.empty(solver.shape, dtype=f.dtype, device=f.device)
    cells = float(np.prod(solver.block_n))  # this rank's fine cells
    stream = torch.cuda.current_stream()

    for _ in range(max(args.warmup, 3)):
        solver.solve(f, u)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    # ---- dominant finest-level kernel class (untimed probe solves, events in the graph)
    from paper_1406_7808_b200 import kernel_names
    names = kernel_names()
    best, best_ms = KC_CANDIDATES[0], -1.0
    for c in KC_CANDIDATES:
        solver.profile_select(c, solver.M)
        solver.solve(f, u)
        torch.cuda.synchronize()
        solver.solve(f, u)
        torch.cuda.synchronize()
        pm, _, pn = solver.profile_read()
        if pn > 0 and pm > best_ms:
            best, best_ms = c, pm
    # ---- timed region: K solves back to back; CUDA events around every launch of that
    # class, one event set per step (the library's profiling ring swaps them into the
    # captured graph), read after the region -- no host synchronisation between steps
    solver.profile_select(best, solver.M)
    solver.solve(f, u)  # re-capture the graph with the profiling events (untimed)
    torch.cuda.synchronize()
    solver.profile_ring(args.steps)
    kms, kbytes, klaunch = 0.0, 0.0, 0
    for _ in range(3):  # keep the GPU loaded until the sampler is running
        solver.solve(f, u)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tw0 = time.monotonic()
    ev0.record(stream)
    for _ in range(args.steps):
        solver.solve(f, u)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.window(tw0, time.monotonic())
    if world > 1:
        dist.barrier()
    for i in range(args.steps):
        a, b, c = solver.profile_read_slot(i)
        kms, kbytes, klaunch = kms + a, kbytes + b, klaunch + c
    solver.profile_ring(0)
    ms = ev0.elapsed_time(ev1) / args.steps
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = cells * world / (ms / 1e3)

    # ---- end-to-end through the public API from pinned host buffers
    solver.profile_select(-1, -1)
    fh = torch.from_numpy(f_host).pin_memory()
    uh = torch.empty(solver.shape, dtype=fh.dtype).pin_memory()
    # the public host-buffer API, pipelined (sr_fmg_solve_host_async): every step copies its
    # f in and its u out; consecutive steps overlap the two PCIe directions and the solve
    for _ in range(2):
        solver.solve_host_async(fh, uh)
    solver.synchronize()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        solver.solve_host_async(fh, uh)
    solver.synchronize()  # every copy and solve of the K steps has completed
    e1.record(stream)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ems], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    nbytes_in = f_host.nbytes
    nbytes_out = int(np.prod(solver.shape)) * f_host.itemsize

    peak, peak_src = measured_peak()
    achieved = (kbytes / (kms / 1e3)) / 1e9 if kms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"{config}_{args.dtype}")
        except Exception:
            traffic = None
    line = {
        "metric": "fine-grid cells solved/s (FMG+SR, fp64)" if args.dtype == "f64"
        else "fine-grid cells solved/s (FMG+SR, fp32)",
        "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 and config != "C4" else "weak",
        "vs_baseline": None, "dtype": args.dtype,
        "data": f"synthetic ({rhs}" + (f", seed {W.SEED})" if "noise" in rhs else ")"),
        "config": {"workload": f"{config}: global {n[0]}x{n[1]}x{n[2]} cells "
                               f"({int(cells)} per GPU), M={M}, seg={seg}, buffer={buf}, "
                               f"K={K} SR levels, F(1,2,2), rhs {rhs}, {args.stencil} operator",
                   "global_cells": cells * world, "pgrid": list(P),
                   "parallelism": (f"segment blocks pgrid {P}: SR levels without communication; "
                                   f"conventional levels {solver.level_A + 1}..{solver.T} "
                                   "domain-decomposed (halo exchange, grouped ncclSend/ncclRecv), "
                                   f"level {solver.level_A} and below gathered (ncclAllGather) and "
                                   f"solved redundantly; {solver.exchanges_per_solve} collective "
                                   "calls per solve")
                   if world > 1 else "1 GPU",
                   "l2": "inputs larger than L2 (f %.2f GB, workspace %.2f GB)"
                         % (nbytes_in / 1e9, solver.workspace_bytes / 1e9)},
        "roofline": {"bound": "hbm", "kernel": f"{names[best]} @ finest level (largest device "
                                               "time per solve among the finest-level kernels)",
                     "achieved": achieved, "peak": peak, "peak_source": peak_src,
                     "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic,
                     "launches_per_step": klaunch / max(args.steps, 1),
                     "alg_bytes_per_launch": kbytes / max(klaunch, 1),
                     "avg_launch_ms": kms / max(klaunch, 1),
                     "share_of_step": (kms / args.steps) / ms if ms > 0 else None},
        "e2e": {"value": cells * world / (ems / 1e3), "unit": "cells/s",
                "h2d_bytes_per_step": nbytes_in, "d2h_bytes_per_step": nbytes_out,
                "ms_per_step": ems},
        "gpu_launches": int(solver.launches_per_solve * args.steps),
        "solve_alg_bytes": solver.alg_bytes_per_solve,
        "solve_roofline_frac": (solver.alg_bytes_per_solve / (ms / 1e3)) / (peak * 1e9),
        "clocks": clk,
    }
    if rank == 0 and world == 1 and args.stencil == "7pt" and max(n) <= 512 and not args.no_accuracy:
        try:
            line["accuracy"] = accuracy({"solver": solver}, n, M, seg, buf, K, h, args.dtype,
                                        f_host, u.double().cpu().numpy())
        except Exception as e:  # reported, never fatal for the bench line
            line["accuracy"] = {"error": repr(e)[:200]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpus = len(os.sched_getaffinity(0))
        if config == "C3" and args.stencil == "7pt" and mem_available_gb() >= 24:
            # the oracle on the bench workload itself: one full-size 512^3 C3 solve (~75 s)
            t1, c1, used = oracle_full_solve(n, M, seg, buf, K, rhs, h)
            line["cpu_baseline"] = {
                "value": c1 / t1, "unit": "cells/s", "cores": used, "kind": "oracle",
                "host_cpus": cpus, "seconds": t1,
                "sample": f"the full C3 workload: one oracle (numpy fp64) solve of the same "
                          f"512^3 manufactured+noise f, M=8, seg=64, buffer=2, K=4"}
        else:
            t1, c1 = oracle_sample_solve()
            t2, c2 = oracle_sample_solve()
            line["cpu_baseline"] = {"value": (c1 + c2) / (t1 + t2), "unit": "cells/s",
                                    "cores": 1, "kind": "oracle", "host_cpus": cpus,
                                    "sample": sample_desc() + " (2 solves)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
