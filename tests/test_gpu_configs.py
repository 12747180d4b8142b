"""GPU parity on all five BASELINE.json configurations (C1..C5).

Each config runs end to end -- seeded image generation, coarsening, normals,
the solve with the config's scheme / Green operator / evaluation -- on the GPU
through the C-ABI and in the CPU oracle, at a resolution the oracle finishes
in under a minute (a cropped fine image, CASES below). C1 runs at full size
(test_gpu_parity.py::test_c1_basic_vs_oracle). Bars
(BASELINE.json north_star): boxel volume fractions and normals bit-exact,
P-bar per load step within 1e-9 relative, F per voxel within 1e-7 relative,
iteration counts within +-1.

Oracle solves are the reference's control flow (solver.cpp:286-346); config
parameters follow SURVEY.md §8(d).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GREEN = {"continuous": 0, "rotated": 1, "staggered": 2}

# (config, fine image, load steps used here). The fine image is cropped, not
# rescaled: radii stay in voxel units and the factors are the config's own, so
# the composite fractions match the full-size configs (C2 0.50, C3 0.11,
# C4 0.127, C5 0.295) while each oracle solve stays under a minute. The load
# path is the first `steps` increments of the config's ramp.
CASES = [
    ("C2", (128, 128, 128), 3),   # -> 32^3 grid, simple shear, contrast 100
    ("C3", (256, 256, 128), 2),   # -> 128x128x16 (2,2,8) non-equiaxed boxels, z-fibres
    ("C4", (64, 64, 64), 2),      # -> 32^3, DFMG + staggered, contrast 1000
    ("C5", (192, 192, 192), 2),   # -> 48^3, RSA r in [8,24] vox
]


def _grids(ctx, oracle, cfg):
    img = ctx.generate(cfg.shape, cfg.fine, (1.0, 1.0, 1.0), *cfg.params)
    kind, cp, cnt = ctx.coarsen(img, cfg.factors)
    nrm, flags, _ = ctx.compute_normals(img, cfg.factors, kind)
    img_o = oracle.generate(cfg.shape, cfg.fine, (1.0, 1.0, 1.0), *cfg.params)
    assert np.array_equal(np.asarray(img).ravel(), np.asarray(img_o).ravel())
    k2, cp2, cnt2 = oracle.coarsen(img_o, cfg.factors)
    n2, f2, _ = oracle.normals(img_o, cfg.factors)
    assert np.array_equal(kind, k2)
    assert np.array_equal(np.asarray(cnt).ravel(), np.asarray(cnt2).ravel())
    assert np.array_equal(cp.view(np.uint64), cp2.view(np.uint64))
    assert np.array_equal(nrm.view(np.uint64), n2.view(np.uint64))
    assert np.array_equal(np.asarray(flags).ravel(), np.asarray(f2).ravel())
    return kind, cp, nrm


def _compare(r, ro, pbar_tol=1e-9, f_tol=1e-7, its=1):
    assert r["report"]["success"] == ro["report"]["success"]
    sg, so = r["report"]["steps"], ro["report"]["steps"]
    assert len(sg) == len(so)
    for a, b in zip(sg, so):
        assert abs(a["outer_iters"] - b["outer_iters"]) <= its, (a["outer_iters"], b["outer_iters"])
        if len(a["cg_iters"]) == len(b["cg_iters"]):  # CG iterations per Newton iteration
            assert all(abs(x - y) <= its for x, y in zip(a["cg_iters"], b["cg_iters"])), (a["cg_iters"],
                                                                                         b["cg_iters"])
        pa, pb = np.array(a["pbar_history"][-1]), np.array(b["pbar_history"][-1])
        assert np.linalg.norm(pa - pb) <= pbar_tol * np.linalg.norm(pb)
    assert np.linalg.norm(r["pbar"] - ro["pbar"]) <= pbar_tol * np.linalg.norm(ro["pbar"])
    Fg, Fo = r["f"].reshape(9, -1), ro["f"].reshape(9, -1)
    rel = np.linalg.norm(Fg - Fo, axis=0) / np.linalg.norm(Fo, axis=0)
    assert rel.max() <= f_tol, rel.max()


@pytest.mark.parametrize("name,fine,steps", CASES, ids=[c for c, _, _ in CASES])
def test_config_vs_oracle(ctx, oracle, name, fine, steps):
    import dataclasses

    from paper_2204_13624_b200 import CellMaterials, neo_hookean
    from paper_2204_13624_b200.configs import CONFIGS

    cfg = dataclasses.replace(CONFIGS[name], fine=fine)
    kind, cp, nrm = _grids(ctx, oracle, cfg)
    dims = cfg.grid
    # the partial load path: the first `steps` increments of the config's ramp
    fbar = np.eye(3) + (cfg.fbar - np.eye(3)) * steps / cfg.load_steps
    cm = CellMaterials(ctx, dims, kind, cp, nrm, neo_hookean(*cfg.matrix), neo_hookean(*cfg.inclusion))
    r = cm.solve(fbar, scheme=cfg.scheme, green=cfg.green, eval=cfg.eval, tol_equilibrium=cfg.tol,
                 max_outer=cfg.max_outer, load_steps=steps)
    cmo = oracle.CellMaterials(dims, kind, cp, nrm, oracle.neo_hookean(*cfg.matrix),
                               oracle.neo_hookean(*cfg.inclusion))
    ro = cmo.solve(fbar, scheme=1 if cfg.scheme == "newton_cg" else 0, green=GREEN[cfg.green],
                   eval=1 if cfg.eval == "dfmg" else 0, tol=cfg.tol, max_outer=cfg.max_outer, load_steps=steps)
    assert ro["report"]["success"]
    _compare(r, ro)
