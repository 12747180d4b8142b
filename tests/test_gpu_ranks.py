"""Slab decomposition on one GPU: R ranks emulated in one
context (combo_ctx_set_virtual_ranks) run the same per-rank kernels, the
slab <-> pencil spectrum transpose and the rank-ordered reductions as the
NCCL path. Every result must be bitwise identical for R = 1, 2, 4 -- the
P-invariance bar of the scope table -- and R = 1 stays on the oracle."""
import numpy as np
import pytest

from paper_2204_13624_b200 import CellMaterials, Context, neo_hookean_enu

pytestmark = pytest.mark.gpu


def shear(g):
    f = np.eye(3)
    f[0, 1] = g
    return f


@pytest.fixture()
def fresh():
    ctxs = []

    def make(R):
        c = Context(0)
        c.set_virtual_ranks(R)
        ctxs.append(c)
        return c

    yield make
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("kind", ["continuous", "rotated", "staggered"])
@pytest.mark.parametrize("dims,ranks", [((8, 8, 8), (2, 4)), ((16, 32, 64), (2, 4, 8)), ((6, 4, 5), (2,)),
                                        ((64, 64, 64), (2, 4))])
def test_project_rank_invariant(fresh, kind, dims, ranks):
    rng = np.random.default_rng(5)
    tau = rng.uniform(-1, 1, 9 * int(np.prod(dims)))
    ref = fresh(1).project(tau, kind, dims)
    for R in ranks:
        got = fresh(R).project(tau, kind, dims)
        assert np.array_equal(got, ref), f"R={R}"


def test_project_ranks_vs_oracle(fresh, oracle):
    dims = (16, 8, 8)
    rng = np.random.default_rng(9)
    tau = rng.uniform(-1, 1, 9 * 1024)
    got = fresh(4).project(tau, "rotated", dims)
    ref = oracle.project(dims, (1, 1, 1), 1, tau)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def _sphere_problem(ctx):
    img = ctx.generate("sphere", (32, 32, 32), (1, 1, 1), 0.4)
    kind, cp, _ = ctx.coarsen(img, (2, 2, 2))
    n, _, _ = ctx.compute_normals(img, (2, 2, 2), kind)
    return kind, cp, n


@pytest.mark.parametrize("scheme", ["newton_cg", "basic"])
def test_solve_rank_invariant(fresh, scheme):
    soft, stiff = neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3)
    base = fresh(1)
    kind, cp, n = _sphere_problem(base)
    kw = dict(scheme=scheme, green="rotated", tol_equilibrium=1e-8 if scheme == "newton_cg" else 1e-6, load_steps=2,
              max_outer=5000)
    r1 = CellMaterials(base, (16, 16, 16), kind, cp, n, soft, stiff).solve(shear(0.4), **kw)
    assert r1["report"]["success"]
    for R in (2, 4):
        c = fresh(R)
        rr = CellMaterials(c, (16, 16, 16), kind, cp, n, soft, stiff).solve(shear(0.4), **kw)
        assert np.array_equal(rr["pbar"], r1["pbar"]), f"R={R}"
        assert np.array_equal(rr["f"], r1["f"]), f"R={R}"
        assert np.array_equal(rr["p"], r1["p"]), f"R={R}"
        for s1, s2 in zip(r1["report"]["steps"], rr["report"]["steps"]):
            assert s1["cg_iters"] == s2["cg_iters"] and s1["residuals"] == s2["residuals"]


def test_solve_ranks_staggered_continuous(fresh):
    soft, stiff = neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3)
    base = fresh(1)
    kind, cp, n = _sphere_problem(base)
    for green in ("staggered", "continuous"):
        kw = dict(green=green, tol_equilibrium=1e-8)
        r1 = CellMaterials(base, (16, 16, 16), kind, cp, n, soft, stiff).solve(shear(0.3), **kw)
        r2 = CellMaterials(fresh(2), (16, 16, 16), kind, cp, n, soft, stiff).solve(shear(0.3), **kw)
        assert np.array_equal(r2["f"], r1["f"]) and np.array_equal(r2["pbar"], r1["pbar"])


def test_rank_shape_errors(fresh):
    from paper_2204_13624_b200.combo import ComboError

    c = fresh(3)
    with pytest.raises(ComboError):
        c.project(np.zeros(9 * 512), "rotated", (8, 8, 8))  # 3 does not divide 8
    c2 = fresh(2)
    c2.set_grid((8, 8, 8))
    with pytest.raises(ComboError):
        c2.fft_forward((8, 8, 8), np.zeros((9, 8, 8, 8)))  # operator-level entry points: one slab


@pytest.mark.parametrize("R", [2, 4])
def test_dfmg_solve_rank_invariant(fresh, oracle, R):
    """DFMG on R slabs: one-plane axis-0 halos of F / pdir (gather_dfc reads
    i + 1) and of the per-dfc stresses (the assembly reads i - 1,
    dfmg.cpp:27-47, 148-156); bitwise equal to one slab, which matches the
    oracle"""
    soft, stiff = neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3)
    base = fresh(1)
    img = base.generate("boolean_ellipsoids", (32, 32, 32), (1, 1, 1), 3, 2.0, 4.0, 0.25)
    kind, cp, _ = base.coarsen(img, (2, 2, 2))
    n, _, _ = base.compute_normals(img, (2, 2, 2), kind)
    kw = dict(green="staggered", eval="dfmg", tol_equilibrium=1e-8, load_steps=2)
    r1 = CellMaterials(base, (16, 16, 16), kind, cp, n, soft, stiff).solve(shear(0.3), **kw)
    assert r1["report"]["success"]
    rr = CellMaterials(fresh(R), (16, 16, 16), kind, cp, n, soft, stiff).solve(shear(0.3), **kw)
    assert np.array_equal(rr["pbar"], r1["pbar"]) and np.array_equal(rr["f"], r1["f"])
    assert np.array_equal(rr["p"], r1["p"])
    for s1, s2 in zip(r1["report"]["steps"], rr["report"]["steps"]):
        assert s1["cg_iters"] == s2["cg_iters"] and s1["residuals"] == s2["residuals"]
    cmo = oracle.CellMaterials((16, 16, 16), kind, cp, n, oracle.neo_hookean_enu(1.0, 0.0),
                               oracle.neo_hookean_enu(10.0, 0.3))
    ro = cmo.solve(shear(0.3), scheme=1, green=2, eval=1, tol=1e-8, load_steps=2)
    assert np.linalg.norm(rr["pbar"] - ro["pbar"]) <= 1e-9 * np.linalg.norm(ro["pbar"])


def test_multi_gpu_context_single_device(oracle):
    """combo_ctx_create_multi (one process, R GPUs, ranks on host threads):
    with the one GPU available the same threaded path runs one rank; the
    solve equals the plain context's bit for bit (a clique of R > 1 GPUs
    needs as many devices)"""
    import torch

    soft, stiff = neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3)
    plain = Context(0)
    kind, cp, n = _sphere_problem(plain)
    kw = dict(tol_equilibrium=1e-8, load_steps=2)
    r1 = CellMaterials(plain, (16, 16, 16), kind, cp, n, soft, stiff).solve(shear(0.4), **kw)
    multi = Context(devices=[0])
    assert multi.ranks()["nranks"] == 1
    r2 = CellMaterials(multi, (16, 16, 16), kind, cp, n, soft, stiff).solve(shear(0.4), **kw)
    assert np.array_equal(r1["f"], r2["f"]) and np.array_equal(r1["pbar"], r2["pbar"])
    tau = np.random.default_rng(3).uniform(-1, 1, 9 * 512)
    assert np.array_equal(multi.project(tau, "rotated", (8, 8, 8)), plain.project(tau, "rotated", (8, 8, 8)))
    if torch.cuda.device_count() > 1:
        m2 = Context(devices=[0, 1])
        r3 = CellMaterials(m2, (16, 16, 16), kind, cp, n, soft, stiff).solve(shear(0.4), **kw)
        assert np.array_equal(r1["f"], r3["f"]) and np.array_equal(r1["pbar"], r3["pbar"])
        m2.close()
    multi.close()
    plain.close()
