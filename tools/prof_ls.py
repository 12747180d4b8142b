"""Short driver for ncu captures: builds a config's grid on the GPU and runs a
solve bounded to a few LS iterations (residual + CG)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2204_13624_b200 import CellMaterials, Context, neo_hookean  # noqa: E402
from paper_2204_13624_b200.configs import CONFIGS, build_slab_grid, scaled  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--scale", type=int, default=1)
ap.add_argument("--ls", type=int, default=4)
a = ap.parse_args()
cfg = scaled(CONFIGS[a.config], a.scale)
ctx = Context(0)
kind, cp, nrm, _ = build_slab_grid(ctx, cfg)
cm = CellMaterials(ctx, cfg.grid, kind, cp, nrm, neo_hookean(*cfg.matrix), neo_hookean(*cfg.inclusion))
r = cm.solve(bench.first_increment(cfg), want_fields=False, scheme=cfg.scheme, green=cfg.green,
             tol_equilibrium=cfg.tol, load_steps=1, max_ls_iterations=a.ls)
print("ls", r["report"]["ls_total"], r["report"]["error"])
