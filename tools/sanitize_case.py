"""Small-grid driver for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the hot path once, on 16^3 / 32^3 grids
(SURVEY.md section 5). Usage (GPU box):
  compute-sanitizer --tool racecheck python tools/sanitize_case.py [n]
Prints one line per stage; the sanitizer's summary follows on exit."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402

import paper_2204_13624_b200 as pkg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
what = sys.argv[2] if len(sys.argv) > 2 else "all"
ctx = pkg.Context(0)
fine = (4 * n, 4 * n, 4 * n)
r = (0.2 * 3 / (4 * np.pi)) ** (1.0 / 3.0)
img = ctx.generate("sphere", fine, (1, 1, 1), r)
kind, cp, cnt = ctx.coarsen(img, (4, 4, 4))
nrm, flags, st = ctx.compute_normals(img, (4, 4, 4), kind)
w = ctx.laplace_weights(ctx.generate("sphere", (n, n, n), (1, 1, 1), r))
print("preprocess ok: composites", int((kind == 2).sum()), flush=True)
dims = (n, n, n)
N = n ** 3
laws = pkg.neo_hookean(2.0, 1.0), pkg.neo_hookean(20.0, 10.0)
rng = np.random.default_rng(5)
F = (np.eye(3).reshape(9, 1) + 0.03 * rng.uniform(-1, 1, (9, N))).ravel()
x = rng.uniform(-1, 1, 9 * N)
if what in ("all", "fft"):
    for g in ("continuous", "rotated", "staggered"):
        ctx.project(x.copy(), g, dims=dims)
    ctx.fft_forward(dims, x[:N].copy())
    # odd / nonequiaxed grid through the generic FFT
    ctx.project(rng.uniform(-1, 1, 9 * 12 * 10 * 18), "rotated", dims=(12, 10, 18))
    print("projection ok", flush=True)
cm = pkg.CellMaterials(ctx, dims, kind, cp, nrm, *laws)
if what in ("all", "point"):
    cm.stress_sweep(F)
    cm.tangent_matvec(F, x)
    t45 = cm.tangent45(F)
    cm.tangent45_matvec(t45, x)
    cm.phase_averages(F)
    cm.recover_composites(F)
    print("material point ok", flush=True)
fbar = np.eye(3)
fbar[0, 0] += 0.05
if what in ("all", "solve"):
    rr = cm.solve(fbar, scheme="newton_cg", green="rotated", tol_equilibrium=1e-8, load_steps=1, max_ls_iterations=12)
    print("newton-cg ok", rr["report"]["ls_total"], flush=True)
    cm.reset_warm_starts()
    rr = cm.solve(fbar, scheme="basic", green="continuous", tol_equilibrium=1e-4, load_steps=1, max_ls_iterations=6)
    print("basic ok", rr["report"]["ls_total"], flush=True)
if what in ("all", "dfmg"):
    img2 = ctx.generate("sphere", (2 * n, 2 * n, 2 * n), (1, 1, 1), r)
    k2, c2, _ = ctx.coarsen(img2, (2, 2, 2))
    n2, _, _ = ctx.compute_normals(img2, (2, 2, 2), k2)
    cm2 = pkg.CellMaterials(ctx, dims, k2, c2, n2, *laws)
    cm2.dfmg_stress(F)
    cm2.dfmg_tangent_matvec(F, x)
    rr = cm2.solve(fbar, green="staggered", eval="dfmg", tol_equilibrium=1e-8, load_steps=1, max_ls_iterations=8)
    print("dfmg ok", rr["report"]["ls_total"], flush=True)
if what in ("all", "ranks"):
    ctx.set_virtual_ranks(2)
    cm3 = pkg.CellMaterials(ctx, dims, kind, cp, nrm, *laws)
    rr = cm3.solve(fbar, scheme="newton_cg", green="rotated", tol_equilibrium=1e-8, load_steps=1, max_ls_iterations=6)
    print("2 emulated ranks ok", rr["report"]["ls_total"], flush=True)
    ctx.set_virtual_ranks(1)
ctx.close()
print("done", flush=True)
