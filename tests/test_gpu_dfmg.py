"""DFMG (doubly-fine material grid, reference src/dfmg.cpp) on the GPU vs the
CPU oracle: stress sweep, exact linearization, and staggered + DFMG solves
(the C4 scheme) including the reference's own DFMG test geometries."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _grid(ctx, shape, fine, fac, *params):
    img = ctx.generate(shape, fine, (1, 1, 1), *params)
    kind, cp, _ = ctx.coarsen(img, fac)
    n, _, _ = ctx.compute_normals(img, fac, kind)
    return tuple(f // k for f, k in zip(fine, fac)), kind, cp, n


def _laws(mod, contrast=10.0):
    return mod.neo_hookean(2.0, 1.0), mod.neo_hookean(2.0 * contrast, contrast)


@pytest.mark.parametrize("fine,fac", [((16, 16, 16), (2, 2, 2)), ((16, 8, 24), (2, 2, 4))])
def test_dfmg_stress_and_tangent_vs_oracle(ctx, oracle, fine, fac):
    from paper_2204_13624_b200 import CellMaterials, neo_hookean

    dims, kind, cp, nrm = _grid(ctx, "boolean_ellipsoids", fine, fac, 3, 1.0, 3.0, 0.25)
    assert (kind == 2).sum() > 0
    n = int(np.prod(dims))
    rng = np.random.default_rng(97)
    F = (np.eye(3).reshape(9, 1) + 0.05 * rng.uniform(-1, 1, (9, n))).ravel()
    cm = CellMaterials(ctx, dims, kind, cp, nrm, *_laws(__import__("paper_2204_13624_b200")))
    cmo = oracle.CellMaterials(dims, kind, cp, nrm, *_laws(oracle))
    P, st = cm.dfmg_stress(F)
    Po, sto = cmo.dfmg_stress(F)
    assert np.abs(P - Po).max() <= 1e-12 * np.abs(Po).max()
    assert st[0] == sto[0] and st[1] == sto[1]
    # exact linearization (dfmg_tangent_pass + dfmg_tangent_matvec)
    x = rng.uniform(-1, 1, 9 * n)
    cm2 = CellMaterials(ctx, dims, kind, cp, nrm, *_laws(__import__("paper_2204_13624_b200")))
    cmo2 = oracle.CellMaterials(dims, kind, cp, nrm, *_laws(oracle))
    y = cm2.dfmg_tangent_matvec(F, x)
    yo = cmo2.dfmg_tangent_matvec(F, x)
    assert np.abs(y - yo).max() <= 1e-10 * np.abs(yo).max()


def test_dfmg_homogeneous_constant_field(ctx):
    # test_kernels.cpp: constant F on a homogeneous grid -> P(F) everywhere
    from paper_2204_13624_b200 import CellMaterials, neo_hookean_enu

    n = 64
    cm = CellMaterials(ctx, (4, 4, 4), np.ones(n, np.uint8), np.ones(n), None, neo_hookean_enu(1.0, 0.0),
                       neo_hookean_enu(10.0, 0.3))
    f = np.eye(3)
    f[0, 1] = 0.37
    f[2, 0] = -0.12
    F = np.repeat(f.reshape(9, 1), n, axis=1).ravel()
    P, st = cm.dfmg_stress(F)
    import oracle as O

    ok, pref, _ = O.law_eval(O.neo_hookean_enu(10.0, 0.3), f)
    assert np.abs(P.reshape(9, n) - pref.reshape(9, 1)).max() <= 1e-13 * np.linalg.norm(pref)


def test_dfmg_solve_vs_oracle(ctx, oracle):
    # C4 scheme (Newton-CG + staggered + DFMG) on a small ellipsoid grid
    import paper_2204_13624_b200 as pkg

    dims, kind, cp, nrm = _grid(ctx, "boolean_ellipsoids", (32, 32, 32), (2, 2, 2), 1, 1.0, 3.0, 0.25)
    fbar = np.eye(3) + 0.05 * np.diag([1.0, -0.5, -0.5])
    cm = pkg.CellMaterials(ctx, dims, kind, cp, nrm, *_laws(pkg, 100.0))
    r = cm.solve(fbar, green="staggered", eval="dfmg", tol_equilibrium=1e-8, load_steps=2)
    cmo = oracle.CellMaterials(dims, kind, cp, nrm, *_laws(oracle, 100.0))
    ro = cmo.solve(fbar, scheme=1, green=2, eval=1, tol=1e-8, load_steps=2)
    assert r["report"]["success"] and ro["report"]["success"]
    for a, b in zip(r["report"]["steps"], ro["report"]["steps"]):
        assert abs(a["outer_iters"] - b["outer_iters"]) <= 1
    assert np.linalg.norm(r["pbar"] - ro["pbar"]) <= 1e-9 * np.linalg.norm(ro["pbar"])
    Fg, Fo = r["f"].reshape(9, -1), ro["f"].reshape(9, -1)
    assert (np.linalg.norm(Fg - Fo, axis=0) / np.linalg.norm(Fo, axis=0)).max() <= 1e-7


def test_dfmg_laminate_slab_within_one_percent(ctx):
    # test_solver.cpp:266-289: slab laminate, dfmg vs continuous <= 1%
    import paper_2204_13624_b200 as pkg

    img = ctx.generate("slab", (128, 2, 2), (1, 1, 1), 0, 0.5)
    kind, cp, _ = ctx.coarsen(img, (1, 1, 1))
    f = np.eye(3)
    f[0, 1] = 0.5
    soft, stiff = pkg.neo_hookean_enu(1.0, 0.0), pkg.neo_hookean_enu(10.0, 0.3)
    ref = pkg.CellMaterials(ctx, (128, 2, 2), kind, cp, None, soft, stiff, combo=False).solve(
        f, green="continuous", tol_equilibrium=1e-10)
    d = pkg.CellMaterials(ctx, (128, 2, 2), kind, cp, None, soft, stiff, combo=False).solve(
        f, green="staggered", eval="dfmg", tol_equilibrium=1e-10)
    assert ref["report"]["success"] and d["report"]["success"]
    assert np.linalg.norm(d["pbar"] - ref["pbar"]) / np.linalg.norm(ref["pbar"]) <= 0.01


def test_dfmg_requires_staggered(ctx):
    import paper_2204_13624_b200 as pkg

    n = 8
    cm = pkg.CellMaterials(ctx, (2, 2, 2), np.zeros(n, np.uint8), np.zeros(n), None, pkg.neo_hookean(2, 1),
                           pkg.neo_hookean(20, 10))
    with pytest.raises(pkg.ComboError) as e:
        cm.solve(np.eye(3), green="rotated", eval="dfmg")
    assert e.value.type == "ConfigInvalid"
