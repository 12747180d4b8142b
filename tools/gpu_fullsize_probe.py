"""Full-size GPU runs of the parity cases (tests/fullsize_common.py) without a
fixture: prints the report shape (per-step Newton / CG / line-search counts,
LS iterations) and timings, to choose LS budgets. Usage:
  python tools/gpu_fullsize_probe.py [case ...] [--max-ls N]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from fullsize_common import CASES, case_fbar  # noqa: E402
from paper_2204_13624_b200 import CellMaterials, Context, neo_hookean  # noqa: E402
from paper_2204_13624_b200.configs import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cases", nargs="*", default=list(CASES))
ap.add_argument("--max-ls", type=int, default=-1)
a = ap.parse_args()
ctx = Context(0)
for name in a.cases:
    case = CASES[name]
    cfg = CONFIGS[case["config"]]
    t0 = time.perf_counter()
    img = torch.empty(int(np.prod(cfg.fine)), dtype=torch.uint8, device="cuda")
    ctx.generate(cfg.shape, cfg.fine, (1.0, 1.0, 1.0), *cfg.params, out=img)
    kind, cp, cnt = ctx.coarsen(img, cfg.factors, dims=cfg.fine)
    nrm, flags, st = ctx.compute_normals(img, cfg.factors, kind, dims=cfg.fine)
    ctx.synchronize()
    del img
    torch.cuda.empty_cache()
    t_pre = time.perf_counter() - t0
    cm = CellMaterials(ctx, cfg.grid, kind, cp, nrm, neo_hookean(*cfg.matrix), neo_hookean(*cfg.inclusion))
    fbar, steps = case_fbar(cfg, case)
    gold = os.path.join(ROOT, "tests", "golden", f"full_{name}.json")
    doc = json.load(open(gold)) if os.path.exists(gold) else None
    budget = (doc["max_ls"] if doc else case["max_ls"]) if a.max_ls < 0 else a.max_ls
    t1 = time.perf_counter()
    r = cm.solve(fbar, scheme=cfg.scheme, green=cfg.green, eval=cfg.eval, tol_equilibrium=cfg.tol,
                 max_outer=cfg.max_outer, load_steps=steps, max_ls_iterations=budget, want_fields=False)
    t_s = time.perf_counter() - t1
    rep = r["report"]
    print(json.dumps({"case": name, "grid": cfg.grid, "composites": cm.composites, "preprocess_s": round(t_pre, 2),
                      "solve_s": round(t_s, 2), "ls_total": rep["ls_total"], "success": rep["success"],
                      "error": rep["error"], "bisections": rep["bisections"]}), flush=True)
    for i, s in enumerate(rep["steps"]):
        print(f"  step {i}: newton {s['outer_iters']} cg {s['cg_iters']} cuts {s['line_search_cuts']} "
              f"ls r/c/t {s['ls_residual']}/{s['ls_cg']}/{s['ls_trial']} resid {s['residuals'][-1]:.3e} "
              f"sweep {s['sweep']}", flush=True)
    if doc and budget == doc["max_ls"]:
        # deviation of every recorded P-bar / residual from the oracle fixture
        for i, (sa, sb) in enumerate(zip(rep["steps"], doc["report"]["steps"])):
            dev = [float(np.linalg.norm(np.subtract(x, y)) / np.linalg.norm(y))
                   for x, y in zip(sa["pbar_history"], sb["pbar_history"])]
            rdev = [abs(x - y) / sb["residuals"][0] for x, y in zip(sa["residuals"], sb["residuals"])]
            print(f"  step {i}: oracle newton {sb['outer_iters']} cg {sb['cg_iters']}; pbar history deviations "
                  f"{['%.1e' % d for d in dev]}; residual deviations {['%.1e' % d for d in rdev]}", flush=True)
ctx.close()
