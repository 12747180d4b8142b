"""The reference's solver tests (/root/reference/proj/tests/test_solver.cpp)
on the GPU, each run through the C-ABI and also compared with the CPU
oracle on the same inputs: the reference's own assertion on the GPU result,
plus P-bar within 1e-9, F within 1e-7 and equal iteration counts (+-1)
against the oracle.

Also the solver's failure branches (solver.cpp:182-185, 232-234, 313-338):
CG breakdown, step cuts, bisection and LoadPathFailed with the final P of
the last evaluated state, and the packed-tangent exports.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STIFF = (10.0, 0.3)
SOFT = (1.0, 0.0)
GREEN = {"continuous": 0, "rotated": 1, "staggered": 2}


def shear(g):
    f = np.eye(3)
    f[0, 1] = g
    return f


def sphere_grid(ctx, fine, fac):
    img = ctx.generate("sphere", (fine,) * 3, (1, 1, 1), 0.4)
    kind, cp, _ = ctx.coarsen(img, (fac,) * 3)
    nrm, _, _ = ctx.compute_normals(img, (fac,) * 3, kind)
    return (fine // fac,) * 3, kind, cp, nrm


def both(ctx, oracle, grid, laws_g, laws_o, fbar, combo=True, opts=None, oopts=None, **kw):
    """the same solve on the GPU and in the oracle"""
    from paper_2204_13624_b200 import CellMaterials

    dims, kind, cp, nrm = grid
    cm = CellMaterials(ctx, dims, kind, cp, nrm, *laws_g, combo=combo, opts=opts)
    r = cm.solve(fbar, **kw)
    okw = dict(scheme={"basic": 0, "newton_cg": 1}[kw.get("scheme", "newton_cg")],
               green=GREEN[kw.get("green", "rotated")], tol=kw.get("tol_equilibrium", 1e-8))
    for k in ("max_outer", "cg_tol", "load_steps", "max_bisections", "cg_max"):
        if k in kw:
            okw[k] = kw[k]
    cmo = oracle.CellMaterials(dims, kind, cp, nrm, *laws_o, combo=combo, opts=oopts)
    ro = cmo.solve(fbar, **okw)
    return r, ro, cm, cmo


def agree(r, ro, pbar_tol=1e-9, f_tol=1e-7, its=1):
    a, b = r["report"], ro["report"]
    assert a["success"] == b["success"] and a["bisections"] == b["bisections"], (a["error"], b["error"])
    assert a["error"] == b["error"]
    assert len(a["steps"]) == len(b["steps"])
    for sa, sb in zip(a["steps"], b["steps"]):
        assert sa["t_start"] == sb["t_start"] and sa["t_end"] == sb["t_end"]
        assert abs(sa["outer_iters"] - sb["outer_iters"]) <= its
        assert sa["cg_breakdowns"] == sb["cg_breakdowns"]
        if sa["outer_iters"] == sb["outer_iters"]:
            assert sa["line_search_cuts"] == sb["line_search_cuts"]
            assert all(abs(x - y) <= its for x, y in zip(sa["cg_iters"], sb["cg_iters"]))
        for pa, pb in zip(sa["pbar_history"], sb["pbar_history"]):
            assert np.linalg.norm(np.subtract(pa, pb)) <= pbar_tol * max(np.linalg.norm(pb), 1e-300)
    den = max(np.linalg.norm(ro["pbar"]), 1e-300)
    assert np.linalg.norm(r["pbar"] - ro["pbar"]) <= pbar_tol * den
    Fg, Fo = r["f"].reshape(9, -1), ro["f"].reshape(9, -1)
    rel = np.linalg.norm(Fg - Fo, axis=0) / np.linalg.norm(Fo, axis=0)
    assert rel.max() <= f_tol, rel.max()


def nh(mod):
    return mod.neo_hookean_enu(*SOFT), mod.neo_hookean_enu(*STIFF)


def test_linear_problem_one_productive_newton_step(ctx, oracle):
    # test_solver.cpp:171-190
    from paper_2204_13624_b200 import iso_mandel, linear

    g = sphere_grid(ctx, 16, 2)
    lg = (linear(iso_mandel(1.0, 0.5)), linear(iso_mandel(3.0, 2.0)))
    lo = (oracle.linear(oracle.iso_mandel(1.0, 0.5)), oracle.linear(oracle.iso_mandel(3.0, 2.0)))
    r, ro, _, _ = both(ctx, oracle, g, lg, lo, np.eye(3) + 1e-3 * shear(1.0), green="continuous",
                       tol_equilibrium=1e-7, cg_tol=1e-12)
    s = r["report"]["steps"][0]
    assert r["report"]["success"] and s["outer_iters"] == 2 and s["cg_iters"][-1] == 0
    agree(r, ro)


def test_path_independence(ctx, oracle):
    # test_solver.cpp:192-211
    import paper_2204_13624_b200 as P

    g = sphere_grid(ctx, 16, 2)
    r1, ro1, _, _ = both(ctx, oracle, g, nh(P), nh(oracle), shear(0.4), tol_equilibrium=1e-10, load_steps=1)
    r3, ro3, _, _ = both(ctx, oracle, g, nh(P), nh(oracle), shear(0.4), tol_equilibrium=1e-10, load_steps=3)
    assert r1["report"]["success"] and r3["report"]["success"] and len(r3["report"]["steps"]) == 3
    assert np.linalg.norm(r3["pbar"] - r1["pbar"]) <= 1e-8 * np.linalg.norm(r1["pbar"])
    agree(r1, ro1)
    agree(r3, ro3)


def test_newton_residual_history_monotone(ctx, oracle):
    # test_solver.cpp:213-223; the histories themselves against the oracle
    import paper_2204_13624_b200 as P

    g = sphere_grid(ctx, 16, 2)
    r, ro, _, _ = both(ctx, oracle, g, nh(P), nh(oracle), shear(0.5), tol_equilibrium=1e-10)
    assert r["report"]["success"]
    for st, so in zip(r["report"]["steps"], ro["report"]["steps"]):
        res = st["residuals"]
        assert all(res[i] <= res[i - 1] * (1.0 + 1e-10) for i in range(1, len(res)))
        # same history: relative to the step's first residual (rounding of
        # the FFT summation order enters at ~1e-13 of it)
        for x, y in zip(res, so["residuals"]):
            assert abs(x - y) <= 1e-7 * so["residuals"][0]
    agree(r, ro)


def test_rerun_bitwise(ctx):
    # test_solver.cpp:225-240
    import paper_2204_13624_b200 as P

    g = sphere_grid(ctx, 16, 2)
    out = []
    for _ in range(2):
        cm = P.CellMaterials(ctx, *g, *nh(P))
        out.append(cm.solve(shear(0.5), tol_equilibrium=1e-9))
    a, b = out
    assert np.array_equal(a["pbar"], b["pbar"])
    assert [s["residuals"] for s in a["report"]["steps"]] == [s["residuals"] for s in b["report"]["steps"]]
    assert np.array_equal(a["f"].view(np.uint64), b["f"].view(np.uint64))


def test_combo_switch_exact_vs_majority(ctx, oracle):
    # test_solver.cpp:242-252: represented c+ (phase averages' c+ at any F)
    import paper_2204_13624_b200 as P

    img = ctx.generate("sphere", (32, 32, 32), (1, 1, 1), 0.4)
    kind, cp, _ = ctx.coarsen(img, (4, 4, 4))
    nrm, _, _ = ctx.compute_normals(img, (4, 4, 4), kind)
    exact = float(np.mean(cp))
    F = np.tile(np.eye(3).reshape(9, 1), (1, 512)).ravel()
    got = {}
    for combo in (True, False):
        cm = P.CellMaterials(ctx, (8, 8, 8), kind, cp, nrm, *nh(P), combo=combo)
        got[combo] = cm.phase_averages(F)["c_plus"]
        cmo = oracle.CellMaterials((8, 8, 8), kind, cp, nrm, *nh(oracle), combo=combo)
        assert abs(got[combo] - cmo.represented_c_plus) <= 1e-13
        assert cm.composites == cmo.composites
    assert abs(got[True] - exact) <= 1e-13
    assert abs(got[False] - exact) > 1e-4


def test_bisection_recovers_aggressive_step(ctx, oracle):
    # test_solver.cpp:254-264
    import paper_2204_13624_b200 as P

    g = sphere_grid(ctx, 16, 2)
    r, ro, _, _ = both(ctx, oracle, g, nh(P), nh(oracle), shear(0.8), tol_equilibrium=1e-8, load_steps=1,
                       max_outer=5)
    assert r["report"]["success"] and r["report"]["bisections"] >= 1
    agree(r, ro)


def test_c_min_ablation(ctx, oracle):
    # test_solver.cpp:291-302
    import paper_2204_13624_b200 as P

    img = ctx.generate("sphere", (32, 32, 32), (1, 1, 1), 0.4)
    kind, cp, _ = ctx.coarsen(img, (4, 4, 4))
    nrm, _, _ = ctx.compute_normals(img, (4, 4, 4), kind)
    n = {}
    for c_min in (0.0, 0.25):
        cm = P.CellMaterials(ctx, (8, 8, 8), kind, cp, nrm, *nh(P), opts=P.LaminateOptions(c_min=c_min))
        cmo = oracle.CellMaterials((8, 8, 8), kind, cp, nrm, *nh(oracle), opts=oracle.lam_opts(c_min=c_min))
        n[c_min] = cm.composites
        assert n[c_min] == cmo.composites
    assert 0 < n[0.25] < n[0.0]


def test_basic_scheme_voxel_pair(ctx, oracle):
    # test_solver.cpp:304-324
    import paper_2204_13624_b200 as P

    img = np.array([1, 0], np.uint8).reshape(2, 1, 1)
    kind, cp, _ = ctx.coarsen(img, (1, 1, 1))
    g = ((2, 1, 1), kind, cp, np.zeros((2, 3)))
    r, ro, _, _ = both(ctx, oracle, g, nh(P), nh(oracle), shear(0.5), scheme="basic", green="rotated",
                       tol_equilibrium=1e-11, max_outer=20000)
    assert r["report"]["success"]
    lam = oracle.laminate_solve(shear(0.5), oracle.neo_hookean_enu(*STIFF), oracle.neo_hookean_enu(*SOFT),
                                [1, 0, 0], 0.5, opts=oracle.lam_opts(tol_rel=1e-13))
    assert np.linalg.norm(r["pbar"] - lam["p_box"]) <= 1e-8 * np.linalg.norm(lam["p_box"])
    agree(r, ro)


def _negative_linear(mod, lam, mu):
    return mod.linear(-np.asarray(mod.iso_mandel(lam, mu)))


def test_cg_breakdown_and_load_path_failed(ctx, oracle):
    """Negative-definite tangents: pT A p < 0 at the first CG iteration
    (solver.cpp:182-185) -> cut step with 0 CG iterations (:232-234) ->
    bisection until the budget is spent -> LoadPathFailed reported, not
    thrown (:332-336); P of the solve is the stress of the last evaluated F
    (:343)."""
    import paper_2204_13624_b200 as P

    g = sphere_grid(ctx, 16, 2)
    lg = (_negative_linear(P, 1.0, 0.5), _negative_linear(P, 3.0, 2.0))
    lo = (_negative_linear(oracle, 1.0, 0.5), _negative_linear(oracle, 3.0, 2.0))
    r, ro, _, _ = both(ctx, oracle, g, lg, lo, np.eye(3) + 1e-3 * shear(1.0), green="continuous",
                       tol_equilibrium=1e-8, load_steps=2, max_bisections=3)
    rep = r["report"]
    assert not rep["success"] and rep["error"].startswith("LoadPathFailed")
    assert rep["bisections"] == 4 and rep["steps"][-1]["cg_breakdowns"] == 1
    assert rep["steps"][-1]["cg_iters"] == [0]
    agree(r, ro)
    pg, po = r["p"].reshape(9, -1), ro["p"].reshape(9, -1)
    assert np.abs(pg - po).max() <= 1e-12 * np.abs(po).max()


def test_cg_breakdown_indefinite_mixture(ctx, oracle):
    """indefinite tangent field (one phase negative definite): whatever the
    breakdown / cut / bisection sequence, GPU and oracle take the same one"""
    import paper_2204_13624_b200 as P

    g = sphere_grid(ctx, 16, 2)
    lg = (P.linear(P.iso_mandel(1.0, 0.5)), _negative_linear(P, 3.0, 2.0))
    lo = (oracle.linear(oracle.iso_mandel(1.0, 0.5)), _negative_linear(oracle, 3.0, 2.0))
    r, ro, _, _ = both(ctx, oracle, g, lg, lo, np.eye(3) + 1e-3 * shear(1.0), green="continuous",
                       tol_equilibrium=1e-8, load_steps=1, max_bisections=2)
    agree(r, ro)
    pg, po = r["p"].reshape(9, -1), ro["p"].reshape(9, -1)
    assert np.abs(pg - po).max() <= 1e-9 * max(np.abs(po).max(), 1e-300)


def test_packed_tangent_exports(ctx, oracle):
    """combo_tangent45 / combo_tangent45_matvec (pack45 / tangent_matvec,
    cell_material.cpp:86-102, 170-194) against the oracle's sweep tangents"""
    import paper_2204_13624_b200 as P

    dims, kind, cp, nrm = sphere_grid(ctx, 32, 4)
    n = int(np.prod(dims))
    rng = np.random.default_rng(5)
    F = (np.eye(3).reshape(9, 1) + 0.05 * rng.standard_normal((9, n))).ravel()
    cm = P.CellMaterials(ctx, dims, kind, cp, nrm, *nh(P))
    cmo = oracle.CellMaterials(dims, kind, cp, nrm, *nh(oracle))
    cm.stress_sweep(F)  # laminate warm starts -> the converged jump vectors
    t45 = cm.tangent45(F)
    _, _, to = cmo.stress_sweep(F, tangents=True)
    # layout [cell][45] as pack45 (upper triangle, symmetrized)
    assert np.abs(t45 - to).max() <= 1e-10 * np.abs(to).max()
    x = rng.standard_normal(9 * n)
    y = cm.tangent45_matvec(to, x)
    yo = oracle.tangent_matvec(to, dims, x)
    assert np.abs(y - yo).max() <= 1e-13 * np.abs(yo).max()
