#!/usr/bin/env python
"""Benchmark of the ComBo Lippmann-Schwinger hot path on B200.

Metric (BASELINE.json): ComBo boxel-iterations/s (fp64) and % of the HBM
roofline. One boxel-iteration = one boxel through one LS iteration, i.e. one
Green-operator application in the reference control flow
(/root/reference/proj/src/solver.cpp:94,134,180,209).

Workload: C5 (RSA spheres, r in [8,24] voxels, phi 0.3, seed 1, condensed
4x4x4, Neo-Hookean contrast 100, Newton-CG, rotated Gamma, tol 1e-8). One
bench step = the complete Newton-CG solve of C5's first load increment
(Fbar = I + 0.02 e1(x)e1, step 1 of 5) from the reference state with reset
warm starts: residual evaluations, CG iterations and line-search trials in
the reference's own mix.
  --gpus 1: the 1-GPU variant, 2048^3 image -> 512^3 grid.
  --gpus P (weak scaling, default): the SURVEY 8d ladder, P x 512^3 boxels
    (1024x512^2, 1024^2x512, 1024^3 from 4096^3), one rank per GPU over
    NCCL, each rank generating / coarsening only its slab of the image.
  --mode strong: the 512^3 grid split over P GPUs; --check then re-solves on
    one GPU and asserts the P-rank reports are bitwise identical.
Fields (9.7 GB each at 512^3) exceed the 126 MB L2, so no flush is needed.

--impl reference: the CPU restatement of the reference (oracle/; the
reference itself needs Eigen3 / FFTW3, absent from the image) on all host
cores, on the same workload (2048^3 image -> 512^3 grid built on the CPU):
one oracle solve of the first increment with an LS budget of W + K; a step
is one LS iteration, the K after the W warm-up ones are timed (the oracle
records the end of every LS iteration).
"""
import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ComBo boxel-iterations/sec (fp64)"
UNIT = "boxel-iterations/s"
LS_MODEL = {  # algorithmic bytes per boxel per LS iteration
    "basic": lambda phi: 792 + 5 + 80 * phi,
    "residual": lambda phi: 720 + 5 + 80 * phi,
    "cg": lambda phi: 1368 + 5 + 56 * phi,
    "trial": lambda phi: 792 + 5 + 80 * phi,
}
GREEN = {"continuous": 0, "rotated": 1, "staggered": 2}


def ncu_traffic(kernel, grid):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
    `kernel` from the committed ncu --set full capture, when it was taken on
    this grid (profiles/ncu_traffic.json); None otherwise."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get(kernel)
    if not d or list(d.get("grid", [])) != list(grid):
        return None
    return d


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def host_facts():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    mem = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal:"):
                mem = round(int(line.split()[1]) / 2**20, 1)
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "ram_gb": mem}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, device=0):
        self.samples = []
        self.device = device
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and
                          s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def workload(gpus, mode):
    from paper_2204_13624_b200.configs import CONFIGS, c5_ladder

    return c5_ladder(gpus) if mode == "weak" else CONFIGS["C5"]


def first_increment(cfg, k=1):
    """macroscopic F after the first k of the config's load increments"""
    return np.eye(3) + k * (cfg.fbar - np.eye(3)) / cfg.load_steps


def ls_counts(report):
    c = {"basic": 0, "residual": 0, "cg": 0, "trial": 0}
    for s in report["steps"]:
        c["basic"] += s["ls_basic"]
        c["residual"] += s["ls_residual"]
        c["cg"] += s["ls_cg"]
        c["trial"] += s["ls_trial"]
    return c


def config_dict(cfg, world, mode):
    return {"workload": f"{cfg.name}: {'x'.join(map(str, cfg.fine))} image -> {'x'.join(map(str, cfg.grid))} "
                        f"ComBo grid, Newton-CG first load increment",
            "grid": list(cfg.grid), "green": cfg.green,
            "l2": "inputs (>= 9.7 GB per field) exceed the 126 MB L2; no flush needed",
            "parallelism": (f"{world} slabs along axis 0, one GPU each (NCCL all-to-all transposes), "
                            f"{mode} scaling") if world > 1 else "single GPU"}


# ------------------------------------------------------------ CPU (oracle)
def oracle_run(kind, cp, nrm, cfg, warm, timed, threads):
    """One oracle solve of the workload's first increment with an LS budget
    of warm + timed; returns boxel-iterations/s over the timed LS window."""
    import oracle as O

    os.environ["ORACLE_LEAN_TANGENTS"] = "1"  # composite tangents only: fits the box's host RAM at 512^3
    dims = cfg.grid
    cm = O.CellMaterials(dims, kind, cp, nrm, O.neo_hookean(*cfg.matrix), O.neo_hookean(*cfg.inclusion),
                         lengths=cfg.lengths)
    r = cm.solve(first_increment(cfg), scheme=1 if cfg.scheme == "newton_cg" else 0, green=GREEN[cfg.green],
                 tol=cfg.tol, max_outer=cfg.max_outer, load_steps=1, max_ls_iterations=warm + timed,
                 want_fields=False)
    clk = r["report"]["ls_clock"]
    n = int(np.prod(dims))
    t0 = clk[warm - 1] if warm > 0 else 0.0
    dt = clk[warm + timed - 1] - t0
    return {"value": n * timed / dt, "seconds": dt, "ls_timed": timed, "ls_warm": warm, "cells": n,
            "grid": list(dims), "first_ls_s": clk[0], "threads": threads}


def cpu_leg_main(args):
    """subprocess entry (bench.py --cpu-leg FILE): the oracle on the grid in
    FILE (kind / c+ / normals built on the GPU, bit-identical to the oracle's
    own preprocessing: tests/test_gpu_fullsize.py)"""
    from paper_2204_13624_b200.configs import CONFIGS

    threads = os.cpu_count() or 1
    d = np.load(args.cpu_leg)
    cfg = CONFIGS["C5"]
    out = oracle_run(d["kind"], d["cp"], d["nrm"], cfg, 1, args.cpu_ls, threads)
    print(json.dumps(out), flush=True)


def run_reference(args, rank, world):
    """--impl reference: the oracle on the host cores on the same workload."""
    if rank != 0:
        return
    from paper_2204_13624_b200.configs import CONFIGS

    import oracle as O

    threads = os.cpu_count() or 1
    cfg = workload(world, args.mode) if world == 1 else CONFIGS["C5"]
    t0 = time.perf_counter()
    img = O.generate(cfg.shape, cfg.fine, cfg.lengths, *cfg.params)
    kind, cp, _ = O.coarsen(img, cfg.factors, cfg.lengths)
    nrm, _, _ = O.normals(img, cfg.factors, cfg.lengths)
    del img
    gc.collect()
    t_pre = time.perf_counter() - t0
    s = oracle_run(kind, cp, nrm, cfg, args.warmup, args.steps, threads)
    v = s["value"]
    desc = (f"oracle (C++/OpenMP restatement of the reference; Eigen/FFTW absent) on {cfg.name} "
            f"{'x'.join(map(str, s['grid']))}: one solve of the first increment, LS budget "
            f"{args.warmup + args.steps}; {args.steps} LS iterations after {args.warmup} warm-up ones timed by the "
            f"oracle's per-iteration clock ({s['seconds']:.1f} s); grid built on the CPU in {t_pre:.0f} s")
    cfgd = config_dict(cfg, 1, "weak")
    if world > 1:
        cfgd["note"] = f"CPU arm runs the 1-GPU rung ({cfg.name}); the {world}-GPU rung needs ~1 TB of host RAM"
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * s["seconds"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded RSA spheres)",
            "impl": "reference", "config": cfgd,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc,
                             "host": host_facts(), "omp_proc_bind": os.environ.get("OMP_PROC_BIND")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(kind_h, cp_h, nrm_h, ls):
    """the oracle in a subprocess (its ~140 GB at 512^3 are freed on exit)"""
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "grid.npz")
        np.savez(path, kind=kind_h, cp=cp_h, nrm=nrm_h)
        env = dict(os.environ, OMP_NUM_THREADS=str(os.cpu_count() or 1), OMP_PROC_BIND="close")
        p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--cpu-leg", path, "--cpu-ls", str(ls)],
                           capture_output=True, text=True, env=env, timeout=1500)
        for line in p.stdout.splitlines():
            if line.startswith("{"):
                return json.loads(line)
        raise RuntimeError(p.stderr[-2000:])


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="weak", choices=["weak", "strong"])
    ap.add_argument("--check", action="store_true", help="strong mode: bitwise check against one GPU")
    ap.add_argument("--cpu-ls", type=int, default=2, help="timed LS iterations of the cpu_baseline leg")
    ap.add_argument("--cpu-leg", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--increments", type=int, default=1,
                    help="load increments of the config per bench step (default: the first; C5 has 5)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.cpu_leg:
        cpu_leg_main(args)
        return

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    from paper_2204_13624_b200 import CellMaterials, Context, neo_hookean
    from paper_2204_13624_b200.configs import build_slab_grid

    cfg = workload(world, args.mode)
    ctx = Context(local)
    if dist:
        # one rank per GPU: slabs along axis 0 over NCCL; the id travels over gloo
        uid = [ctx.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.set_ranks(world, rank, uid[0])
    t_pre = time.perf_counter()
    kind, cp, nrm, nstats = build_slab_grid(ctx, cfg, world, rank)
    t_pre = time.perf_counter() - t_pre
    dims = cfg.grid
    N = int(np.prod(dims))
    N_local = N // world

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # cpu_baseline first, while host memory is free (the oracle needs ~140 GB at 512^3)
        try:
            s = cpu_baseline_leg(kind.cpu().numpy(), cp.cpu().numpy(), nrm.cpu().numpy(), args.cpu_ls)
            cpu = {"value": s["value"], "unit": UNIT, "cores": s["threads"], "kind": "port",
                   "sample": (f"oracle (C++/OpenMP restatement of the reference) on this grid "
                              f"({'x'.join(map(str, s['grid']))}), first increment: {s['ls_timed']} LS iterations "
                              f"after the first (the tangent sweep from reset warm starts, {s['first_ls_s']:.1f} s), "
                              f"timed by the oracle's per-iteration clock ({s['seconds']:.1f} s)"),
                   "host": host_facts()}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}

    def bind(k, c, n):
        return CellMaterials(ctx, dims, k, c, n, neo_hookean(*cfg.matrix), neo_hookean(*cfg.inclusion),
                             lengths=cfg.lengths, local=True)

    cm = bind(kind, cp, nrm)
    ncomp = float(cm.composites)
    if dist:
        t = torch.tensor([ncomp], dtype=torch.float64)
        dist.all_reduce(t)
        ncomp = float(t.item())
    phi = ncomp / N
    fbar = first_increment(cfg, args.increments)
    kw = dict(scheme=cfg.scheme, green=cfg.green, tol_equilibrium=cfg.tol, max_outer=cfg.max_outer,
              load_steps=args.increments)

    def step():
        cm.reset_warm_starts()
        return cm.solve(fbar, want_fields=False, **kw)

    for _ in range(args.warmup):
        r = step()
    ext = torch.cuda.ExternalStream(ctx.stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches
    ctx.profile(True)
    counts = {"basic": 0, "residual": 0, "cg": 0, "trial": 0}
    ls_total = 0
    reports = []
    with ClockSampler(local) as clk:
        ev0.record(ext)
        for _ in range(args.steps):
            r = step()
            reports.append(r["report"])
            for k, v in ls_counts(r["report"]).items():
                counts[k] += v
            ls_total += r["report"]["ls_total"]
        ev1.record(ext)
        ev1.synchronize()
    torch.cuda.synchronize()
    prof = ctx.profile_report()
    ctx.profile(False)
    launches = ctx.kernel_launches - launches0
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # every rank runs the same LS iterations on its slab of the one grid
    value = N * float(ls_total) / (ms / 1000.0)  # whole-job boxel-iterations/s

    peak, peak_kind = measured_peaks()
    dom = max((kv for kv in prof.items() if kv[0] != "exchange"), key=lambda kv: kv[1]["ms"])
    dname, d = dom
    per_launch_bytes = d["bytes"] / d["launches"]
    avg_s = d["ms"] / d["launches"] / 1000.0
    achieved = per_launch_bytes / avg_s / 1e9
    model_bytes = sum(counts[k] * LS_MODEL[k](phi) for k in counts) * N_local
    ls_achieved = model_bytes / (ms / 1000.0) / 1e9  # per GPU (this rank's slab)

    # e2e: through the C-ABI with host buffers (bind + solve + F, P read back)
    e2e = None
    if not args.no_e2e:
        kind_h = torch.empty(N_local, dtype=torch.uint8, pin_memory=True)
        cp_h = torch.empty(N_local, dtype=torch.float64, pin_memory=True)
        nrm_h = torch.empty(3 * N_local, dtype=torch.float64, pin_memory=True)
        kind_h.copy_(kind.cpu())
        cp_h.copy_(cp.cpu())
        nrm_h.copy_(nrm.reshape(-1).cpu())
        # SolveResult{f, p, pbar} (solver.hpp:57-62): both fields come back to
        # pinned host buffers of this rank's slab
        f_h = torch.empty(9 * N_local, dtype=torch.float64, pin_memory=True)
        p_h = torch.empty(9 * N_local, dtype=torch.float64, pin_memory=True)
        del cm
        e_ms = []
        ls_e = 0
        for _ in range(max(1, args.steps)):
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            cm2 = bind(kind_h, cp_h, nrm_h)
            r2 = cm2.solve(fbar, f_out=f_h, p_out=p_h, **kw)
            ctx.synchronize()
            e_ms.append((time.perf_counter() - t0) * 1000.0)
            ls_e += r2["report"]["ls_total"]
            del cm2
        e_tot = sum(e_ms)
        if dist:
            t = torch.tensor([e_tot], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_tot = float(t.item())
        e2e = {"value": N * ls_e / (e_tot / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": N_local * (1 + 8 + 24), "d2h_bytes_per_step": 2 * 9 * N_local * 8 + 72,
               "ms_per_step": e_tot / len(e_ms)}
        del f_h, p_h, kind_h, cp_h, nrm_h

    check = None
    if args.check and world > 1 and args.mode == "strong":
        check = bitwise_check(ctx, cfg, reports[-1], rank, dist, kw, fbar)

    if rank == 0:
        rep0 = reports[-1]
        cfgd = config_dict(cfg, world, args.mode)
        if args.increments > 1:
            cfgd["workload"] = cfgd["workload"].replace("first load increment",
                                                        f"first {args.increments} load increments")
            cfgd["ls_per_increment"] = [s["ls_residual"] + s["ls_cg"] + s["ls_trial"] + s["ls_basic"]
                                        for s in rep0["steps"]]
        cfgd.update({"composite_fraction": phi, "ls_per_step": ls_total / args.steps, "ls_mix": counts,
                     "newton_per_step": sum(s["outer_iters"] for s in rep0["steps"]), "preprocess_s": t_pre,
                     "preprocess": "per-slab device generation / coarsening / normals" if world > 1
                     else "device generation / coarsening / normals"})
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": args.mode, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded RSA spheres, random-free analytic materials)",
            "config": cfgd,
            "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": (ncu_traffic(dname, dims) or {}).get("traffic_bytes_per_launch"),
                         "traffic_source": (ncu_traffic(dname, dims) or {}).get("source"),
                         "peak_kind": peak_kind, "bytes_per_launch": per_launch_bytes, "avg_ms": avg_s * 1000.0},
            "ls_roofline": {"model_bytes_per_boxel_iter": model_bytes / (N_local * ls_total) if ls_total else None,
                            "achieved": ls_achieved, "peak": peak, "unit": "GB/s", "frac": ls_achieved / peak},
            "kernels": prof,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if check is not None:
            line["check"] = check
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def bitwise_check(ctx, cfg, rep_dist, rank, dist, kw, fbar):
    """--check (strong mode): rank 0 re-solves the same grid on its GPU alone
    and compares the P-rank run's report bitwise (reductions are combined
    in global chunk order, so every scalar is decomposition invariant)."""
    import torch

    from paper_2204_13624_b200 import CellMaterials, Context, neo_hookean
    from paper_2204_13624_b200.configs import build_slab_grid

    ctx.close()
    torch.cuda.empty_cache()
    ok = None
    if rank == 0:
        c1 = Context(torch.cuda.current_device())
        k, c, n, _ = build_slab_grid(c1, cfg, 1, 0)
        cm = CellMaterials(c1, cfg.grid, k, c, n, neo_hookean(*cfg.matrix), neo_hookean(*cfg.inclusion),
                           lengths=cfg.lengths)
        r1 = cm.solve(fbar, want_fields=False, **kw)["report"]
        keys = ("outer_iters", "cg_iters", "line_search_cuts", "residuals", "pbar_history")
        ok = all(a[k] == b[k] for a, b in zip(r1["steps"], rep_dist["steps"]) for k in keys) and \
            len(r1["steps"]) == len(rep_dist["steps"])
        c1.close()
    dist.barrier()
    return {"against": "the same solve on 1 GPU", "bitwise_equal_histories": ok}


if __name__ == "__main__":
    main()
