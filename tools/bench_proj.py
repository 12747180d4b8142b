"""Projection-only microbenchmark: combo_project on a random 9-component
field resident on the device; per-pass CUDA-event times from the library
profiler. Tuning knobs are read from the environment (COMBO_XW, COMBO_YW,
COMBO_ZLINES). Usage: python tools/bench_proj.py N [reps] [kind] [ranks]
(ranks > 1: that many emulated slab ranks on the one device, with the
slab <-> pencil transposes as device copies; COMBO_OVERLAP=0/1 selects the
serial / row-group pipelined schedule)"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2204_13624_b200 import Context  # noqa: E402
from paper_2204_13624_b200.combo import MEM_DEVICE, _ptr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kind = sys.argv[3] if len(sys.argv) > 3 else "rotated"
ranks = int(sys.argv[4]) if len(sys.argv) > 4 else 1
ctx = Context(0)
if ranks > 1:
    ctx.set_virtual_ranks(ranks)
ctx.set_grid((n, n, n))
N = n ** 3
a = torch.rand(9 * N, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
L = ctx.L
g = {"continuous": 0, "rotated": 1, "staggered": 2}[kind]
ctx._check(L.combo_project(ctx.h, g, _ptr(a), _ptr(b), MEM_DEVICE))
import time  # noqa: E402

ctx.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    ctx._check(L.combo_project(ctx.h, g, _ptr(a), _ptr(b), MEM_DEVICE))
ctx.synchronize()
elapsed_ms = (time.perf_counter() - t0) * 1000.0 / reps  # wall time per projection (overlapped streams included)
ctx.profile(True)
for _ in range(reps):
    ctx._check(L.combo_project(ctx.h, g, _ptr(a), _ptr(b), MEM_DEVICE))
prof = ctx.profile_report()
tot = sum(v["ms"] for v in prof.values()) / reps
knobs = {k: v for k, v in os.environ.items() if k.startswith("COMBO_")}
print(json.dumps({"n": n, "ranks": ranks, "knobs": knobs, "ms_per_projection": round(tot, 3), "elapsed_ms_per_projection": round(elapsed_ms, 3),
                  "passes": {k: [round(v["ms"] / v["launches"], 3), round(v["bytes"] / v["ms"] / 1e6, 1)]
                             for k, v in prof.items()}}))
