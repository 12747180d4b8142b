"""Full-size parity: BASELINE configs C2-C5 at their real sizes on the GPU
against committed CPU-oracle fixtures (tests/golden/full_*.json, made by
tools/fullsize_fixtures.py on the B200 box's host cores).

Per case: the device-built grid (2048^3 image for C5) is bit-exact with the
oracle's (sha256 of kind / c+ / count / normals / flags); the solve along
the config's load path (solver.cpp:286-346; C4 with an LS budget, C5 = the
bench workload) reproduces the oracle's report -- every step's fbar and t
bitwise, Newton iterations and CG iterations per Newton iteration within +-1
and equal line-search cuts, P-bar after every LS iteration within 1e-9
relative, residual histories within 1e-6 of the step's first residual -- and
F: per-component sums within 1e-9 of sum|F|, and per voxel within 1e-7
relative at the seeded sample cells. C4 (DFMG, contrast 1000, stopped by its
LS budget mid-Newton after CG solves of 57 + 136 iterations) compares the
inexact-Newton iterates after the first at 1e-6 (tests/fullsize_common.py).
"""
import glob
import json
import os

import numpy as np
import pytest

from fullsize_common import CASES, case_fbar, grid_digests

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIXTURES = sorted(os.path.basename(p)[5:-5] for p in glob.glob(os.path.join(GOLDEN, "full_C*.json")))


def compare_reports(a, b, pbar_tol=1e-9, res_tol=1e-6, its=1, mid_tol=None):
    """mid_tol: tolerance of the P-bar entries after the first of a step
    that did not converge (LS budget): inexact-Newton iterates, which inherit
    the rounding amplification of the CG solves before them."""
    assert a["success"] == b["success"] and a["error"] == b["error"], (a["error"], b["error"])
    assert a["bisections"] == b["bisections"]
    assert len(a["steps"]) == len(b["steps"])
    worst = 0.0
    for k, (sa, sb) in enumerate(zip(a["steps"], b["steps"])):
        assert sa["fbar"] == sb["fbar"] and sa["t_start"] == sb["t_start"] and sa["t_end"] == sb["t_end"], k
        assert sa["converged"] == sb["converged"], k
        assert abs(sa["outer_iters"] - sb["outer_iters"]) <= its, (k, sa["outer_iters"], sb["outer_iters"])
        same_newton = sa["outer_iters"] == sb["outer_iters"]
        if same_newton:
            assert sa["line_search_cuts"] == sb["line_search_cuts"], k
        ca, cb = sa["cg_iters"], sb["cg_iters"]
        assert all(abs(x - y) <= its for x, y in zip(ca, cb)), (k, ca, cb)
        r0 = sb["residuals"][0]
        for x, y in zip(sa["residuals"], sb["residuals"]):
            assert abs(x - y) <= res_tol * r0, (k, x, y)
        for i, (pa, pb) in enumerate(zip(sa["pbar_history"], sb["pbar_history"])):
            d = np.linalg.norm(np.subtract(pa, pb)) / np.linalg.norm(pb)
            tol = mid_tol if (mid_tol and i > 0 and not sb["converged"]) else pbar_tol
            assert d <= tol, (k, i, d, tol)
            worst = max(worst, d)
    return worst


@pytest.mark.parametrize("name", FIXTURES)
def test_fullsize_vs_oracle_fixture(ctx, name):
    import torch

    from paper_2204_13624_b200 import CellMaterials, neo_hookean
    from paper_2204_13624_b200.configs import CONFIGS

    doc = json.load(open(os.path.join(GOLDEN, f"full_{name}.json")))
    samp = np.load(os.path.join(GOLDEN, f"full_{name}_F.npy"))
    case = CASES[name]
    cfg = CONFIGS[case["config"]]
    assert list(doc["grid"]) == list(cfg.grid)
    max_ls = int(doc["max_ls"])  # the LS budget the fixture was generated with
    # preprocessing on the device, bit-exact with the oracle at full size
    img = torch.empty(int(np.prod(cfg.fine)), dtype=torch.uint8, device="cuda")
    ctx.generate(cfg.shape, cfg.fine, (1.0, 1.0, 1.0), *cfg.params, out=img)
    kind, cp, cnt = ctx.coarsen(img, cfg.factors, dims=cfg.fine)
    nrm, flags, nstats = ctx.compute_normals(img, cfg.factors, kind, dims=cfg.fine)
    ctx.synchronize()
    del img
    torch.cuda.empty_cache()
    assert grid_digests(kind, cp, cnt, nrm, flags) == doc["grid_digests"]
    assert [int(x) for x in nstats] == doc["normal_stats"]
    del cnt, flags
    # the solve
    dims = cfg.grid
    n = int(np.prod(dims))
    cm = CellMaterials(ctx, dims, kind, cp, nrm, neo_hookean(*cfg.matrix), neo_hookean(*cfg.inclusion))
    assert cm.composites == doc["composites"]
    fbar, steps = case_fbar(cfg, case)
    F = torch.empty(9 * n, dtype=torch.float64, device="cuda")
    r = cm.solve(fbar, want_fields=False, scheme=cfg.scheme, green=cfg.green, eval=cfg.eval, tol_equilibrium=cfg.tol,
                 max_outer=cfg.max_outer, load_steps=steps, max_ls_iterations=max_ls, f_out=F)
    rep, ref = r["report"], doc["report"]
    truncated = not ref["success"]  # the LS budget ended the last step mid-Newton
    mid = case.get("mid_tol")
    compare_reports(rep, ref, mid_tol=mid)
    assert abs(rep["ls_total"] - ref["ls_total"]) <= max(4, ref["ls_total"] // 100)
    pb = np.asarray(doc["pbar"])
    assert np.linalg.norm(r["pbar"].ravel() - pb) <= (mid if truncated and mid else 1e-9) * np.linalg.norm(pb)
    F = F.view(9, n)
    s = doc["f_sums"]
    assert np.all(np.abs(F.sum(dim=1).cpu().numpy() - np.asarray(s["sum"])) <= 1e-9 * np.asarray(s["sumabs"]))
    cells = torch.as_tensor(doc["sample_cells"], dtype=torch.int64, device="cuda")
    got = F[:, cells].T.cpu().numpy()
    rel = np.linalg.norm(got - samp, axis=1) / np.linalg.norm(samp, axis=1)
    assert rel.max() <= (10 * mid if truncated and mid else 1e-7), rel.max()
