"""Throughput of the BASELINE parity configs C1-C4 on the GPU (not bench
lines: bench.py measures C5). One JSON line per config: the config's whole
load path (C4 with an LS budget), wall time of solve() with a device sync,
boxel-iterations/s = cells x LS iterations / seconds. C1 (32^3, basic
scheme) is launch-latency bound: its per-iteration time is reported too.
Usage: python tools/bench_configs.py [C1 C2 C3 C4] [--reps N] [--max-ls N]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

from paper_2204_13624_b200 import CellMaterials, Context, neo_hookean  # noqa: E402
from paper_2204_13624_b200.configs import CONFIGS, build_slab_grid  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3", "C4"])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--max-ls", type=int, default=0, help="LS budget for C4 (0: whole path)")
a = ap.parse_args()
ctx = Context(0)
for name in a.configs:
    cfg = CONFIGS[name]
    kind, cp, nrm, _ = build_slab_grid(ctx, cfg)
    cm = CellMaterials(ctx, cfg.grid, kind, cp, nrm, neo_hookean(*cfg.matrix), neo_hookean(*cfg.inclusion))
    n = int(np.prod(cfg.grid))
    budget = a.max_ls if name == "C4" else 0
    best = None
    for rep in range(a.reps if name == "C1" else 1):
        cm.reset_warm_starts()
        ctx.synchronize()
        l0 = ctx.kernel_launches
        t0 = time.perf_counter()
        r = cm.solve(cfg.fbar, want_fields=False, scheme=cfg.scheme, green=cfg.green, eval=cfg.eval,
                     tol_equilibrium=cfg.tol, max_outer=cfg.max_outer, load_steps=cfg.load_steps,
                     max_ls_iterations=budget)
        ctx.synchronize()
        dt = time.perf_counter() - t0
        rep_ = r["report"]
        rec = {"config": name, "grid": list(cfg.grid), "scheme": cfg.scheme, "eval": cfg.eval,
               "steps": len(rep_["steps"]), "success": rep_["success"], "error": rep_["error"],
               "ls_total": rep_["ls_total"], "seconds": dt, "boxel_iterations_per_s": n * rep_["ls_total"] / dt,
               "us_per_ls_iteration": 1e6 * dt / max(rep_["ls_total"], 1),
               "launches_per_ls_iteration": (ctx.kernel_launches - l0) / max(rep_["ls_total"], 1)}
        if best is None or rec["seconds"] < best["seconds"]:
            best = rec
    print(json.dumps(best), flush=True)
    del cm
ctx.close()
