#!/usr/bin/env python
"""bench.py — driver benchmark contract for the GS(p) + Krylov hot path on B200.

A *step* is one pass of the whole hot path over one synthetic
system: GS(2) of A and b (a2), the SELL value refresh of the plan (a3), the
Bi-CGSTAB solve (a4-a7) and the GMRES(m) solve (a4-a6, a8-a9) to the config's
tolerance, each ending in its true-residual check (a10); all control runs on the
device (a11).  At N=1 the workload is BASELINE.json configs[3] (C4: 256^3, 7-point
upwind, 5 slabs, SELL-C-32-256; the headline roofline config), generated with the
seeded recipe of DESIGN.md §3 and resident in HBM before timing.

The GMRES(30) leg runs a fixed budget of 300 iterations (--gmres-maxit).

value  = solver iterations per second (Bi-CGSTAB + GMRES iterations of the step,
         summed over ranks, / max-over-ranks device time); unit "iters/s".
e2e    = the same through the public API with the system copied from pinned host
         memory every step (plan rebuilt) and x read back (summed over ranks).
roofline: the probed kernel with the largest share of the step (per-launch CUDA-event
         time inside the captured graphs x its launches per step; at C4 with the
         row-class dictionary the GMRES MGS projection pass, 4*8n bytes per launch;
         on plain SELL slots the Bi-CGSTAB pass v = A p, <r^,v>, 12 nnz + 4(n+1) +
         3*8n); every probed kernel is listed in extra.roofline_all; traffic from the
         committed ncu captures (profiles/r02_ncu_traffic*.json).
layout:  the plan is SELL-C-32-256 built on the device; by default (--sell-index
         classes) its passes read the row-class dictionary (a uint16
         class id per row and one 128-byte line per distinct row instead of 12 bytes
         per nonzero — lossless, bit-identical) where the matrix's rows repeat (C1, C3,
         C4), else the slots; extra.sell_plain holds the same solves on the slots.
extra  = SpMV and GS(2) rooflines, per-pass probes and time_to_tol (time to 1e-8 of
         Bi-CGSTAB and of GMRES(30) without scaling, with GS(1), GS(2) and two-sided
         scaling).
--impl reference: the CPU oracle (oracle/) on a bounded sample of the same work.
--shards P: one system in P row blocks: emulated on one GPU, or one
         shard per rank over NCCL under torchrun ("scaling": "strong").
Multi-GPU: under torchrun with N > 1 ranks the default step is the
         row-block sharded solve of ONE C4 system, one shard per rank, halos and the
         reduction partials over NCCL ("scaling": "strong"; the residual history is
         bit-identical at every N, its SHA-256 is in extra.history).  --weak: weak
         scaling instead — C4's 256^3 block stacked N times in z (C4w), one block per
         rank, each rank generating and holding only its own rows.  --replicas runs N
         independent single-GPU replicas (no data-path collective).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
# one metric string for every arm and mode (the driver divides the arms' values only
# when the strings match); the workload and the grid live in "config"
METRIC = "solver iters/s (GS(2)+Bi-CGSTAB+GMRES(30) step)"
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gsk", choices=["gsk", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--N", type=int, default=None, help="override grid size (debug only)")
    ap.add_argument("--gmres-maxit", type=int, default=300,
                    help="GMRES(30) iteration budget per step (10 restart cycles; DESIGN.md §7)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-time-to-tol", action="store_true",
                    help="skip the time-to-tolerance runs (Bi-CGSTAB and GMRES(30): none / GS(1) / GS(2) / "
                         "two-sided, ~40 s at C4)")
    ap.add_argument("--schedule", default="auto", choices=["auto", "fused", "split", "split4"])
    ap.add_argument("--orth", default="mgs", choices=["mgs", "cgs2"],
                    help="GMRES orthogonalisation (MGS: north star; CGS2: the paper's AZTEC)")
    ap.add_argument("--sell-index", default="classes", choices=["plain", "dict", "uniform", "classes"],
                    help="SELL plan encoding: the row-class dictionary (classes, the default: a 2-byte class id per "
                         "row instead of slot data where the rows repeat, else plain), int32 columns per slot "
                         "(plain), the SELL-D per-chunk delta dictionary, or SELL-U chunk-uniform deltas "
                         "(DESIGN.md §5); all bit-identical")
    ap.add_argument("--no-plain-compare", action="store_true",
                    help="skip the extra.sell_plain comparison run (one step on plain SELL-C-32-256 slots)")
    ap.add_argument("--fmt", default="sell", choices=["csr", "sell"],
                    help="plan layout built on the device from the CSR input (SELL-C-32-256 is faster "
                         "on every config: DESIGN.md §7)")
    ap.add_argument("--replicas", action="store_true",
                    help="with N > 1 ranks: N independent single-GPU replicas (weak scaling) instead of the "
                         "sharded solve of one system")
    ap.add_argument("--weak", action="store_true",
                    help="with N > 1 ranks: weak scaling — C4's 256^3 block stacked N times in z (C4w), one "
                         "block per rank, each rank generating and holding only its own rows")
    ap.add_argument("--peer", action="store_true",
                    help="sharded modes: reductions by device-initiated peer stores over CUDA IPC / NVLink "
                         "(gsk_shard_opts.peer_reduce) instead of ncclAllGather")
    ap.add_argument("--shards", type=int, default=0,
                    help="row-block sharded solve (DESIGN.md §8): with one process, P shards emulated on "
                         "one GPU (the cost of sharding); under torchrun, one shard per rank over NCCL "
                         "(strong scaling).  0 = the default replicated step")
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, idx):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(idx), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for nm, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def byte_model(n, nnz, rcd=False):
    """Algorithmic bytes per launch; B_A = 12 nnz + 4(n+1),
    or 2 n with the row-class dictionary (a uint16 class id per row; the class lines
    stay in L1)."""
    BA = 2 * n if rcd else 12 * nnz + 4 * (n + 1)
    return {"spmv": BA + 16 * n, "gs": 16 * nnz + 4 * (n + 1) + 24 * n,
            # fused schedule: P1 gathers r, p, v and writes p, v (+ r^ own row); P2 r, v -> t
            "bicg_p1": BA + 48 * n, "bicg_p2": BA + 24 * n,
            # split schedule: S1 v = A p (p gather, r^, v), S3 t = A s (s gather, t)
            "bicg_s1": BA + 24 * n, "bicg_s3": BA + 16 * n,
            # four-pass schedule: S1q gathers q, r (p = r + beta q), reads r^, writes p, v
            "bicg_s1q": BA + 40 * n,
            "bicg_s4": 56 * n, "bicg_p3": 64 * n,
            "bicg_iter": 2 * BA + 17 * 8 * n, "bicg_iter_split": 2 * BA + 19 * 8 * n,
            # GMRES S_j: w = A v_j as a plain SpMV pass (its h_1j dot is a separate pass)
            "gmres_mgs": 32 * n, "gmres_arnoldi": BA + 16 * n}


def oracle_sample(sys_, cfg, m, kb=8, kg=8):
    """Bounded oracle sample of the step: GS(2), kb Bi-CGSTAB iterations, kg GMRES steps."""
    import oracle
    t = time.perf_counter()
    vo, bo, _ = oracle.gs_scale(sys_["row_ptr"], sys_["val"], sys_["b"], 2)
    _, _, rb = oracle.bicgstab(sys_["row_ptr"], sys_["col"], vo, bo, cfg.tol, kb)
    _, _, rg = oracle.gmres(sys_["row_ptr"], sys_["col"], vo, bo, m, cfg.tol, kg)
    dt = time.perf_counter() - t
    its = rb["iterations"] + rg["iterations"]
    return its / dt, its, dt, oracle.num_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = workloads.CONFIGS[args.config]
    s = workloads.generate(args.config, N=args.N)
    m = 30
    vals = []
    for i in range(args.warmup + args.steps):
        v, its, dt, cores = oracle_sample(s, cfg, m)
        if i >= args.warmup:
            vals.append((v, its, dt))
    value = float(np.mean([v for v, _, _ in vals]))
    ms = float(np.mean([dt for _, _, dt in vals]) * 1e3)
    sample = "GS(2) + 8 Bi-CGSTAB iterations + 8 GMRES(30) steps of the full system"
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "iters/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_desc(args, cfg, s),
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` (a short name or its prefix before
    the engine's variant arguments, e.g. pass_kernel<2,1,OpS1) from the committed ncu
    --set full captures (profiles/r02_ncu_traffic.json: SELL slots; r02_ncu_traffic_rcd.json:
    row-class plans), or None."""
    ks = {}
    for name in ("r02_ncu_traffic.json", "r02_ncu_traffic_rcd.json"):  # SELL slots; row classes
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                ks.update(json.load(f)["kernels"])
        except (OSError, ValueError, KeyError):
            pass
    if not ks:
        return None
    for name, k in ks.items():
        if name == kernel or name.startswith(kernel.rstrip(">") + ","):
            return k["bytes_per_launch"]
    return None


def plan_schedule(args, n=None, nnz=None):
    """Bi-CGSTAB schedule the plan runs (auto: four-pass when the matrix and eight
    vectors fit in 64 MB, else split)."""
    if args.schedule != "auto":
        return args.schedule
    if n is not None and 12 * nnz + 4 * n + 64 * n <= 64e6:
        return "split4"
    return "split"


def reduce_over_ranks(ms, its, dist, device):
    """Whole-job timing over ranks: the step time is the MAX over ranks, the work
    (solver iterations) is the SUM (each rank solves its own replica)."""
    import torch
    t = torch.tensor([ms, float(its)], device=device, dtype=torch.float64)
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(tmax[0]), float(t[1])


def config_desc(args, cfg, s, ncls=None):
    """The `config` object — the same in both arms (it depends on the arguments and the
    workload only; what the plan detected is in extra.encoding)."""
    N = cfg.N if args.N is None else args.N
    if cfg.name == "C4w":
        G = int(s["n"]) // N ** 3
        wl, grid = (f"C4w: BASELINE.json configs[3] stacked {G}x in z (one 256^3 block of C4's layered "
                    f"medium per GPU; weak scaling, DESIGN.md §8)", f"{N}x{N}x{N * G}")
    else:
        wl, grid = f"{cfg.name}: BASELINE.json configs[{int(cfg.name[1]) - 1}]", f"{N}^{3 if cfg.cfg in (3, 4) else 2}"
    sell = getattr(args, "fmt", "sell") == "sell"
    fmt = ("SELL-C-32-256" if sell else "CSR") + " (built on the device from the CSR input)"
    if sell and getattr(args, "sell_index", "classes") == "classes":
        fmt += ("; where the matrix's rows repeat the passes read the plan's row-class dictionary (a uint16 class "
                "id per row + 128-byte class lines instead of the slot data; lossless, bit-identical results; "
                "DESIGN.md §5; extra.encoding says whether it applied)")
    return {"workload": wl, "n": int(s["n"]), "nnz": int(s["nnz"]), "grid": grid, "format": fmt, "scaling": "GS(2)",
            "solvers": ["Bi-CGSTAB to tol (maxit %d)" % cfg.maxit,
                        "GMRES(30) for %d iterations (or to tol)" % args.gmres_maxit],
            "tol": cfg.tol, "seed": cfg.seed,
            "l2": ("inputs larger than L2 (126 MB): matrix %.2f GB, 8 solver vectors of %.0f MB per Bi-CGSTAB "
                   "iteration, a %.2f GB GMRES basis" % ((12 * s["nnz"] + 4 * s["n"]) / 1e9, 8 * s["n"] / 1e6,
                                                        31 * 8 * s["n"] / 1e9))}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    if args.shards or (world > 1 and not args.replicas):
        run_sharded(args, rank, world, local)
        return

    import torch
    import paper_0812_2769_b200 as gsk

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workloads.CONFIGS[args.config]
    m = 30
    gmaxit = args.gmres_maxit
    s = workloads.generate(args.config, N=args.N)
    n, nnz = s["n"], s["nnz"]
    A0 = gsk.CSR.from_system(s)
    b0 = torch.tensor(s["b"], device="cuda")
    vbuf = torch.empty_like(A0.val)
    bbuf = torch.empty_like(b0)
    dbuf = torch.empty_like(b0)
    As, bs, _ = gsk.gs_scale(A0, b0, 2, out=(vbuf, bbuf, dbuf))
    fmt = args.fmt
    sidx = args.sell_index if fmt == "sell" else "plain"
    plan = gsk.Plan(As, fmt=fmt, schedule=args.schedule, orth=args.orth, sell_index=sidx)
    x1 = torch.empty(n, dtype=torch.float64, device="cuda")
    x2 = torch.empty(n, dtype=torch.float64, device="cuda")

    def step():
        gsk.gs_scale(A0, b0, 2, out=(vbuf, bbuf, dbuf))
        plan.refresh()
        _, _, r1 = plan.bicgstab(bbuf, tol=cfg.tol, maxit=cfg.maxit, x=x1, hist=False)
        _, _, r2 = plan.gmres(bbuf, m=m, tol=cfg.tol, maxit=gmaxit, x=x2, hist=False)
        return r1, r2

    for _ in range(args.warmup):
        step()
    probes0 = [plan.probe(k) for k in range(5)]
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = Clocks(local) if os.environ.get("GSK_BENCH_NO_CLOCKS") != "1" else None
    launches0 = gsk.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    reps = []
    sev = []
    for _ in range(args.steps):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        sev.append(e)
        reps.append(step())
    ev1.record()
    torch.cuda.synchronize()
    sev.append(ev1)
    step_ms = [sev[k].elapsed_time(sev[k + 1]) for k in range(args.steps)]
    launches = gsk.launch_count() - launches0
    clk = clocks.stop() if clocks else None
    ms = ev0.elapsed_time(ev1)
    its = sum(r1["iterations"] + r2["iterations"] for r1, r2 in reps)
    if dist:
        ms, its = reduce_over_ranks(ms, its, dist, "cuda")
    value = its / (ms / 1e3)

    # dominant kernel: per-launch times from the CUDA-event probes inside the timed steps;
    # the roofline object reports the probed kernel with the largest share of the step
    NP = 5
    probes = []
    for k in range(NP):
        tot, cnt = plan.probe(k)
        t0, c0 = probes0[k]
        dc = cnt - c0
        probes.append(((tot * cnt - t0 * c0) / dc) if dc > 0 else None)
    try:
        ncls = plan.num_classes() if fmt == "sell" else -1
    except Exception:
        ncls = -1
    rcd = ncls > 0
    bm = byte_model(n, nnz, rcd)
    hbm, src = peaks()
    sched = plan_schedule(args, n, nnz)
    try:
        nsl = plan.num_slots() if rcd else -1
    except Exception:
        nsl = -1
    # pass_kernel format argument: 1 CSR, 2 SELL slots, 5 class lines, 6 / 7 classes with a 7- / 5-delta stencil
    F = ({7: 6, 5: 7}.get(nsl, 5)) if rcd else (2 if fmt == "sell" else 1)
    r1l, r2l = reps[-1]
    its_b, its_g = r1l["iterations"], r2l["iterations"]
    # MGS projection passes of a GMRES(m) run of its_g steps: step j of a cycle has j - 1
    full, rest = divmod(its_g, m)
    n_mgs = full * (m * (m - 1) // 2) + rest * (rest - 1) // 2
    vkey, vname, vshort = {
        "split": ("bicg_s1", f"pass_kernel<{F},1,OpS1> (v = A p, <r^,v>)", f"pass_kernel<{F},1,OpS1>"),
        "split4": ("bicg_s1q", f"pass_kernel<{F},1,OpS1q> (p = r + beta q at the gather, v = A p, <r^,v>)",
                   f"pass_kernel<{F},1,OpS1q>"),
        "fused": ("bicg_p1", f"pass_kernel<{F},1,OpP1> (p update at the gather, v = A p, <r^,v>)",
                  f"pass_kernel<{F},1,OpP1>")}[sched]
    ukey, uname, ushort = {
        "split": ("bicg_s4", "pass_kernel<0,4,OpS4> (x, r update, 3 dots)", "pass_kernel<0,4,OpS4>"),
        "split4": ("bicg_s4", "pass_kernel<0,4,OpS4q> (x, r, q update, 3 dots)", "pass_kernel<0,4,OpS4q>"),
        "fused": ("bicg_p3", "pass_kernel<0,4,OpP3> (x, r update, 3 dots)", "pass_kernel<0,4,OpP3>")}[sched]
    cands = [
        (vkey, vname, vshort, probes[0], its_b),
        ("bicg_p2" if sched == "fused" else "bicg_s3",
         f"pass_kernel<{F},1,{'OpP2' if sched == 'fused' else 'OpS3'}> (t = A s, <t,s>, <t,t>)",
         f"pass_kernel<{F},1,{'OpP2' if sched == 'fused' else 'OpS3'}>", probes[1], its_b),
        (ukey, uname, ushort, probes[4], its_b),
        ("gmres_arnoldi", f"pass_kernel<{F},1,OpCgsS> (GMRES w = A v_j)", f"pass_kernel<{F},1,OpCgsS>", probes[3], its_g),
    ]
    if args.orth == "mgs":
        cands.append(("gmres_mgs", "pass_kernel<0,4,OpMgs> (GMRES MGS: w -= h v_i, <w,v_{i+1}>)",
                      "pass_kernel<0,8,OpMgs>", probes[2], n_mgs))
    step_ms_last = step_ms[-1]
    roofs = []
    for key, kname, kshort, p_ms, count in cands:
        if not p_ms:
            continue
        ach = bm[key] / (p_ms / 1e3) / 1e9
        roofs.append({"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                      "traffic": ncu_traffic(kshort), "kernel": kname, "bytes_per_launch": bm[key],
                      "ms_per_launch": p_ms, "launches_per_step": count,
                      "share_of_step": p_ms * count / step_ms_last, "peak_source": src,
                      "frac_of_8TBps": ach / 8000.0})
    for r in roofs:
        if r["frac"] > 1.0:  # algorithmic bytes / time above the copy peak: part of them never reach DRAM
            r["note"] = ("achieved > peak: consecutive passes alternate their row order, so a pass starts on the "
                         "rows the previous one left in the 126 MB L2 (DESIGN.md §5); compare `traffic` (ncu DRAM "
                         "bytes per launch) with bytes_per_launch")
    roofs.sort(key=lambda r: -r["share_of_step"])
    roof = roofs[0] if roofs else None
    p1_ms = probes[0]

    # SpMV standalone roofline (same plan, 50 back-to-back launches)
    x = torch.tensor(workloads.uniform(n, 9, 9), device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        plan.spmv(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        plan.spmv(x, y)
    e1.record()
    torch.cuda.synchronize()
    spmv_ms = e0.elapsed_time(e1) / 50
    spmv_gbps = bm["spmv"] / (spmv_ms / 1e3) / 1e9

    # GS(2) standalone roofline (row a2): each call is flag reset + gs_kernel + flag
    # read + stream sync; events bracket one call, best of 10
    gs_times = []
    for _ in range(10):
        e0.record()
        gsk.gs_scale(A0, b0, 2, out=(vbuf, bbuf, dbuf))
        e1.record()
        torch.cuda.synchronize()
        gs_times.append(e0.elapsed_time(e1))
    gs_ms = min(gs_times)
    gs_gbps = bm["gs"] / (gs_ms / 1e3) / 1e9

    r1, r2 = reps[-1]
    extra = {
        "bicgstab": {"iterations": r1["iterations"], "status": gsk.STATUS[r1["status"]],
                     "relres": r1["relres"], "true_relres": r1["true_relres"], "solve_ms": r1["solve_ms"],
                     "iters_per_s": r1["iterations"] / (r1["solve_ms"] / 1e3) if r1["solve_ms"] else None,
                     "gbps_model": bm["bicg_iter" if sched == "fused" else "bicg_iter_split"] * r1["iterations"]
                     / (r1["solve_ms"] / 1e3) / 1e9 if r1["solve_ms"] else None,
                     "gbps_17vector_model": bm["bicg_iter"] * r1["iterations"] / (r1["solve_ms"] / 1e3) / 1e9
                     if r1["solve_ms"] else None, "schedule": sched},
        "gmres": {"m": m, "orth": args.orth, "iterations": r2["iterations"], "status": gsk.STATUS[r2["status"]],
                  "relres": r2["relres"], "true_relres": r2["true_relres"], "solve_ms": r2["solve_ms"],
                  "iters_per_s": r2["iterations"] / (r2["solve_ms"] / 1e3) if r2["solve_ms"] else None},
        "steps_ms": [{"step": round(t, 2), "bicgstab": round(r1["solve_ms"], 2), "gmres": round(r2["solve_ms"], 2),
                      "rest": round(t - r1["solve_ms"] - r2["solve_ms"], 2)} for t, (r1, r2) in zip(step_ms, reps)],
        "spmv": {"ms": spmv_ms, "gbps": spmv_gbps, "frac_of_hbm": spmv_gbps / hbm,
                 "frac_of_8TBps": spmv_gbps / 8000.0},
        "gs2": {"ms": gs_ms, "gbps": gs_gbps, "bytes": bm["gs"], "frac_of_hbm": gs_gbps / hbm,
                "frac_of_8TBps": gs_gbps / 8000.0},
        "probe_ms": {"bicg_v_pass": probes[0], "bicg_t_pass": probes[1], "gmres_mgs": probes[2],
                     "gmres_arnoldi_spmv": probes[3], "bicg_update_pass": probes[4]},
        "roofline_all": roofs,
        "encoding": {"sell_index": args.sell_index, "row_classes": ncls if rcd else None,
                     "stencil_slots": nsl if nsl > 0 else None,
                     "matrix_bytes_per_spmv": bm["spmv"] - 16 * n},
        "probe_gbps": {"bicg_v_pass": bm[{"split": "bicg_s1", "split4": "bicg_s1q", "fused": "bicg_p1"}[sched]]
                       / (probes[0] / 1e3) / 1e9
                       if probes[0] else None,
                       "bicg_t_pass": bm["bicg_p2" if sched == "fused" else "bicg_s3"] / (probes[1] / 1e3) / 1e9
                       if probes[1] else None,
                       "gmres_mgs": bm["gmres_mgs"] / (probes[2] / 1e3) / 1e9 if probes[2] else None,
                       "gmres_arnoldi_spmv": bm["gmres_arnoldi"] / (probes[3] / 1e3) / 1e9
                       if probes[3] else None},
    }

    if rcd and not args.no_plain_compare:
        # the same two solves on the plain SELL-C-32-256 slots (one warm-up, one timed)
        pp = gsk.Plan(As, fmt=fmt, schedule=args.schedule, orth=args.orth, sell_index="plain")
        for _ in range(2):
            _, _, q1 = pp.bicgstab(bbuf, tol=cfg.tol, maxit=cfg.maxit, x=x1, hist=False)
            _, _, q2 = pp.gmres(bbuf, m=m, tol=cfg.tol, maxit=gmaxit, x=x2, hist=False)
        bmp = byte_model(n, nnz, False)
        pv = pp.probe(0)[0]
        extra["sell_plain"] = {
            "iters_per_s": (q1["iterations"] + q2["iterations"]) / ((q1["solve_ms"] + q2["solve_ms"]) / 1e3),
            "bicgstab_iters_per_s": q1["iterations"] / (q1["solve_ms"] / 1e3),
            "gmres_iters_per_s": q2["iterations"] / (q2["solve_ms"] / 1e3),
            "bicgstab_iterations": q1["iterations"], "gmres_iterations": q2["iterations"],
            "bicg_v_pass_ms": pv, "bicg_v_pass_gbps": bmp[vkey] / (pv / 1e3) / 1e9 if pv else None,
            "bicg_v_pass_frac_of_hbm": bmp[vkey] / (pv / 1e3) / 1e9 / hbm if pv else None,
            "same_iterations": q1["iterations"] == r1["iterations"] and q2["iterations"] == r2["iterations"]}
        pp.close()
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(gsk, torch, s, cfg, m, gmaxit, fmt, args, dist)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, its_c, dt, cores = oracle_sample(s, cfg, m)
        cpu = {"value": v, "unit": "iters/s", "cores": cores, "kind": "oracle",
               "sample": f"GS(2) + 8 Bi-CGSTAB its + 8 GMRES(30) steps of {cfg.name} ({dt:.1f} s)"}
    if not args.no_time_to_tol and rank == 0:
        extra["time_to_tol"] = time_to_tol(gsk, torch, s, cfg, fmt, sidx=sidx)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value,
            "unit": "iters/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_desc(args, cfg, s, ncls if rcd else None),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_sharded(args, rank, world, local):
    """--shards: ONE system split into row blocks.  world == 1: all
    shards on this GPU (halo exchange by device copies); world > 1: one shard per rank,
    halos and reductions over NCCL, timing max over ranks, value = iterations of the one
    solve per second ("scaling": "strong")."""
    import torch
    import paper_0812_2769_b200 as gsk

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P = world if world > 1 else args.shards
    cfg = workloads.CONFIGS[args.config]
    m, gmaxit = 30, args.gmres_maxit
    weak = args.weak and world > 1
    fmt = args.fmt
    comm = gsk.NcclComm() if world > 1 else None
    if weak:
        # C4w: one 256^3 block of C4's layered medium per rank, stacked in z; each rank
        # generates and holds only its own rows (gsk_shard_opts.local_input)
        cfg = workloads.STACKED
        n_glob, nnz_glob = workloads.dims(cfg.cfg, args.N or cfg.N, world)
        lo, hi = gsk.shard_rows(n_glob, world, rank)
        s = workloads.generate_rows("C4w", lo, hi, N=args.N, param=world)
        s_desc = {"n": n_glob, "nnz": nnz_glob}
    else:
        s = workloads.generate(args.config, N=args.N)
        s_desc = s
    A0 = gsk.CSR.from_system(s)
    b0 = torch.tensor(s["b"], device="cuda")
    vbuf, bbuf, dbuf = torch.empty_like(A0.val), torch.empty_like(b0), torch.empty_like(b0)
    As, bs, _ = gsk.gs_scale(A0, b0, 2, out=(vbuf, bbuf, dbuf))
    sidx = args.sell_index if fmt == "sell" else "plain"
    if weak:
        SP = gsk.ShardedPlan(As, fmt=fmt, comm=comm, n_global=n_glob, peer_reduce=args.peer, sell_index=sidx)
        bl = bbuf
    else:
        SP = gsk.ShardedPlan(As, shards=P, fmt=fmt, comm=comm, peer_reduce=args.peer, sell_index=sidx)
        lo, hi = SP.rows
        bl = bbuf[lo:hi]
    x1 = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
    x2 = torch.empty(hi - lo, dtype=torch.float64, device="cuda")

    def step():
        gsk.gs_scale(A0, b0, 2, out=(vbuf, bbuf, dbuf))
        SP.refresh()
        _, _, r1 = SP.bicgstab(bl, tol=cfg.tol, maxit=cfg.maxit, x=x1, hist=False)
        _, _, r2 = SP.gmres(bl, m=m, tol=cfg.tol, maxit=gmaxit, x=x2, hist=False)
        return r1["iterations"] + r2["iterations"], r1, r2

    for _ in range(args.warmup):
        step()
    probes0 = [SP.probe(k) for k in range(4)]
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = Clocks(local) if os.environ.get("GSK_BENCH_NO_CLOCKS") != "1" else None
    launches0 = gsk.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its, reps = 0, []
    for _ in range(args.steps):
        k, r1, r2 = step()
        its += k
        reps.append((r1, r2))
    e1.record()
    torch.cuda.synchronize()
    launches = gsk.launch_count() - launches0
    clk = clocks.stop() if clocks else None
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    # the residual histories (global, identical on every rank) of one more untimed
    # step: bit-identical at every N, compared across SCALE lines
    import hashlib
    _, h1, q1 = SP.bicgstab(bl, tol=cfg.tol, maxit=cfg.maxit, x=x1)
    _, h2, q2 = SP.gmres(bl, m=m, tol=cfg.tol, maxit=gmaxit, x=x2)
    history = {"bicgstab_iterations": q1["iterations"], "gmres_iterations": q2["iterations"],
               "bicgstab_sha256": hashlib.sha256(np.ascontiguousarray(h1, "<f8").tobytes()).hexdigest(),
               "gmres_sha256": hashlib.sha256(np.ascontiguousarray(h2, "<f8").tobytes()).hexdigest()}
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e_sharded(gsk, torch, s, cfg, m, gmaxit, fmt, args, P, comm, dist,
                                  n_global=n_glob if weak else None)
    # roofline: this rank's (or emulated shard 0's) v = A p pass (probe 0) against its
    # own rows' bytes
    if weak:
        l0, h0, nnz0 = lo, hi, int(s["nnz"])
    else:
        l0, h0 = gsk.shard_rows(s["n"], P, rank if world > 1 else 0)
        nnz0 = int(s["row_ptr"][h0] - s["row_ptr"][l0])
    tot, cnt = SP.probe(0)
    t0, c0 = probes0[0]
    p_ms = (tot * cnt - t0 * c0) / (cnt - c0) if cnt > c0 else None
    try:
        ncls = SP.num_classes() if fmt == "sell" else -1
    except Exception:
        ncls = -1
    bm = byte_model(h0 - l0, nnz0, ncls > 0)
    hbm, src = peaks()
    roof = None
    if p_ms:
        ach = bm["bicg_s1"] / (p_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": None,
                "kernel": "pass_kernel<SELL, OpS1> of one shard (v = A p, <r^,v>)", "bytes_per_launch": bm["bicg_s1"],
                "ms_per_launch": p_ms, "peak_source": src}
    if rank == 0:
        r1, r2 = reps[-1]
        line = {
            "metric": METRIC, "value": its / (ms / 1e3), "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if weak else ("strong" if world > 1 else "none (emulated shards on one GPU)"),
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**config_desc(args, cfg, s_desc, ncls if ncls > 0 else None), "parallelism": f"rows/{P}",
                       "shards": P,
                       "placement": (f"{world} GPUs, NCCL halos + all-gathers" if world > 1
                                     else "all shards on one GPU (device-copy halos)")
                       + ("; each rank generates and holds only its own 256^3 block (local input)"
                          if weak else "")},
            "roofline": roof, "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "comm": {"backend": "nccl" if world > 1 else "none (one process)", "nranks": world,
                     "reductions": "device-initiated peer stores + epoch flags (CUDA IPC)" if args.peer
                     else ("ncclAllGather" if world > 1 else "in place"),
                     "shards": P, "nranks_ok": (comm.world == world) if comm else world == 1},
            "extra": {"bicgstab": {"iterations": r1["iterations"], "status": gsk.STATUS[r1["status"]],
                                   "solve_ms": r1["solve_ms"]},
                      "gmres": {"iterations": r2["iterations"], "status": gsk.STATUS[r2["status"]],
                                "solve_ms": r2["solve_ms"]},
                      "history": history},
        }
        print(json.dumps(line), flush=True)
    SP.close()
    if comm:
        comm.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def measure_e2e(gsk, torch, s, cfg, m, gmaxit, fmt, args, dist=None):
    """Every step: pinned host -> device copy of the system, GS(2), plan build (SELL),
    both solves, x read back; timed with CUDA events on the current stream."""
    pin = {k: torch.from_numpy(np.ascontiguousarray(s[k])).pin_memory() for k in ("row_ptr", "col", "val", "b")}
    h2d = sum(t.numel() * t.element_size() for t in pin.values())
    n = s["n"]
    xo1 = torch.empty(n, dtype=torch.float64).pin_memory()
    xo2 = torch.empty(n, dtype=torch.float64).pin_memory()
    d2h = 2 * n * 8

    def step():
        dev = {k: v.to("cuda", non_blocking=True) for k, v in pin.items()}
        A = gsk.CSR(dev["row_ptr"], dev["col"], dev["val"])
        As, bs, _ = gsk.gs_scale(A, dev["b"], 2, inplace=True)
        P = gsk.Plan(As, fmt=fmt, sell_index=args.sell_index if fmt == "sell" else "plain")
        x1, _, r1 = P.bicgstab(bs, tol=cfg.tol, maxit=cfg.maxit, hist=False)
        x2, _, r2 = P.gmres(bs, m=m, tol=cfg.tol, maxit=gmaxit, hist=False)
        xo1.copy_(x1, non_blocking=True)
        xo2.copy_(x2, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        P.close()
        return r1["iterations"] + r2["iterations"]

    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = 0
    k = max(1, min(args.steps, 2))
    for _ in range(k):
        its += step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist:  # whole job: every rank's replica, slowest rank's time
        ms, its = reduce_over_ranks(ms, its, dist, "cuda")
        h2d *= dist.get_world_size()
        d2h *= dist.get_world_size()
    return {"value": its / (ms / 1e3), "unit": "iters/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms / k, "steps": k}


def measure_e2e_sharded(gsk, torch, s, cfg, m, gmaxit, fmt, args, P, comm, dist, n_global=None):
    """e2e of the sharded step: every step each rank copies the system from pinned host
    memory (the sharded plan reads its rows and halo from the global arrays; with
    n_global, the rank's own rows only), scales it, builds its shard plan, runs both
    solves and reads its rows of x back.  Whole-job value: the one system's iterations
    / the slowest rank's time."""
    pin = {k: torch.from_numpy(np.ascontiguousarray(s[k])).pin_memory() for k in ("row_ptr", "col", "val", "b")}
    h2d = sum(t.numel() * t.element_size() for t in pin.values())
    if n_global is not None:
        lo, hi = 0, s["hi"] - s["lo"]
    elif comm:
        lo, hi = gsk.shard_rows(s["n"], P, comm.rank)
    else:
        lo, hi = 0, s["n"]
    xo1 = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
    xo2 = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
    d2h = 2 * (hi - lo) * 8

    def step():
        dev = {k: v.to("cuda", non_blocking=True) for k, v in pin.items()}
        A = gsk.CSR(dev["row_ptr"], dev["col"], dev["val"])
        As, bs, _ = gsk.gs_scale(A, dev["b"], 2, inplace=True)
        SP = gsk.ShardedPlan(As, shards=P, fmt=fmt, comm=comm, n_global=n_global, peer_reduce=args.peer,
                             sell_index=args.sell_index if fmt == "sell" else "plain")
        x1, _, r1 = SP.bicgstab(bs[lo:hi], tol=cfg.tol, maxit=cfg.maxit, hist=False)
        x2, _, r2 = SP.gmres(bs[lo:hi], m=m, tol=cfg.tol, maxit=gmaxit, hist=False)
        xo1.copy_(x1, non_blocking=True)
        xo2.copy_(x2, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        SP.close()
        return r1["iterations"] + r2["iterations"]

    step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = 0
    k = max(1, min(args.steps, 2))
    for _ in range(k):
        its += step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist:  # one system: iterations once, the slowest rank's time; bytes of every rank
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        if n_global is None:
            h2d *= dist.get_world_size()
            d2h = 2 * s["n"] * 8
        else:  # each rank copied its own rows
            t = torch.tensor([float(h2d), float(d2h)], device="cuda", dtype=torch.float64)
            dist.all_reduce(t)
            h2d, d2h = int(t[0].item()), int(t[1].item())
    return {"value": its / (ms / 1e3), "unit": "iters/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms / k, "steps": k}


def time_to_tol(gsk, torch, s, cfg, fmt, m=30, sidx="plain"):
    """Time to cfg.tol with and without GS (north-star metric; the paper times both
    solvers): Bi-CGSTAB and GMRES(m) from the device-resident
    unscaled system — scaling + plan (SELL build) + solve, CUDA events — for no
    scaling, GS(1), GS(2) and two-sided D^1/2 A D^1/2.  Every variant stops in the GS(2)
    frame: Bi-CGSTAB through the plan's frame weights, GMRES on the
    GS(2)-scaled system on its least-squares estimate and on the other systems on the
    weighted true residual at cycle ends (reading B2w)."""
    return {"bicgstab": _time_to_tol(gsk, torch, s, cfg, fmt, None, sidx),
            f"gmres({m})": _time_to_tol(gsk, torch, s, cfg, fmt, m, sidx)}


def _time_to_tol(gsk, torch, s, cfg, fmt, m, sidx="plain"):
    out = {}
    A0 = gsk.CSR.from_system(s)
    b0 = torch.tensor(s["b"], device="cuda")
    _, _, d2 = gsk.gs_scale(A0, b0, 2)
    for name, p in (("none", None), ("GS1", 1), ("GS2", 2), ("two-sided GS2", "sym")):
        A = gsk.CSR(A0.row_ptr, A0.col, A0.val.clone())
        b = b0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        w = d2
        if p == "sym":
            A, b, w = gsk.gs_scale_sym(A, b, 2)  # GS(2) frame: D r = D^1/2 r_sym
        elif p is not None:
            A, b, dp = gsk.gs_scale(A, b, p, inplace=True)
            w = None if p == 2 else d2 / dp
        # GMRES on a system that is not the GS(2)-scaled one stops on the GS(2)-frame true
        # residual at cycle ends (gsk_opts.gmres_wstop, reading B2w), as Bi-CGSTAB does
        # through its frame weights
        wstop = m is not None and w is not None
        P = gsk.Plan(A, fmt=fmt, weights=w, sell_index=sidx, gmres_wstop=wstop)
        if m is None:
            _, h, r = P.bicgstab(b, tol=cfg.tol, maxit=cfg.maxit, hist=False)
        else:
            _, h, r = P.gmres(b, m=m, tol=cfg.tol, maxit=cfg.maxit, hist=False)
        e1.record()
        torch.cuda.synchronize()
        out[name] = {"ms": e0.elapsed_time(e1), "iterations": r["iterations"],
                     "status": gsk.STATUS[r["status"]], "best_relres": r["best_relres"],
                     "true_relres_gs2_frame": r["true_relres_w"] if w is not None else r["true_relres"]}
        if m is not None:
            out[name]["stopping_frame"] = ("GS(2) frame: weighted true residual at cycle ends (gmres_wstop)" if wstop
                                           else "solved = GS(2) frame (least-squares estimate)")
        P.close()
    return out


if __name__ == "__main__":
    main()
