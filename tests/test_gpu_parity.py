"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star): P-bar per step within 1e-9 relative, F per
voxel within 1e-7 relative, iteration counts identical (+-1), volume
fractions and normals bit-exact. Operator-level checks use tighter bars.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STIFF = (10.0, 0.3)
SOFT = (1.0, 0.0)


def shear(g):
    f = np.eye(3)
    f[0, 1] = g
    return f


def laws(mod):
    return mod.neo_hookean_enu(*SOFT), mod.neo_hookean_enu(*STIFF)


# ------------------------------------------------------------------ FFT / Gamma
@pytest.mark.parametrize("dims", [(8, 8, 8), (6, 5, 4), (2, 1, 1), (16, 32, 64), (32, 32, 32), (64, 16, 128),
                                  (4, 4, 1), (12, 10, 7), (128, 4, 512)])
def test_fft_forward_vs_numpy(ctx, dims):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((9,) + dims)
    got = ctx.fft_forward(dims, x)
    ref = np.fft.rfftn(x, axes=(1, 2, 3))
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("kind", ["continuous", "rotated", "staggered"])
@pytest.mark.parametrize("dims,lengths", [((6, 5, 4), (1.0, 0.8, 1.2)), ((8, 8, 8), (1, 1, 1)),
                                          ((32, 16, 8), (1, 1, 1)), ((2, 1, 1), (1, 1, 1)),
                                          ((64, 64, 64), (1, 1, 1))])
def test_project_vs_oracle(ctx, oracle, kind, dims, lengths):
    rng = np.random.default_rng(2)
    n = int(np.prod(dims))
    tau = rng.uniform(-1, 1, 9 * n)
    got = ctx.project(tau, kind, dims, lengths)
    ref = oracle.project(dims, lengths, {"continuous": 0, "rotated": 1, "staggered": 2}[kind], tau)
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("kind", ["continuous", "rotated", "staggered"])
def test_green_identities_gpu(ctx, kind):
    # test_green.cpp:62-103
    dims, lengths = (6, 5, 4), (1.0, 0.8, 1.2)
    n = 120
    rng = np.random.default_rng(71)
    const = np.repeat(rng.uniform(-1, 1, 9), n)
    assert np.abs(ctx.project(const, kind, dims, lengths)).max() <= 1e-13
    tau = rng.uniform(-1, 1, 9 * n)
    once = ctx.project(tau, kind, dims, lengths)
    assert np.abs(once.reshape(9, n).mean(axis=1)).max() <= 1e-12
    twice = ctx.project(once, kind, dims, lengths)
    assert np.abs(twice - once).max() <= 1e-10 * np.abs(once).max()


def test_continuous_reproduces_compatible_field(ctx):
    # test_green.cpp:45-60
    dims, L = (6, 5, 4), (1.0, 0.8, 1.2)
    i, j, k = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
    x = 2 * np.pi * (i + 0.5) / dims[0]
    y = 2 * np.pi * (j + 0.5) / dims[1]
    z = 2 * np.pi * (k + 0.5) / dims[2]
    kx, ky, kz = (2 * np.pi / l for l in L)
    g = np.zeros((9,) + dims)
    g[0] = kx * np.cos(x) * np.cos(y)
    g[1] = -ky * np.sin(x) * np.sin(y)
    g[4] = -ky * np.sin(y) * np.sin(z)
    g[5] = kz * np.cos(y) * np.cos(z)
    g[8] = kz * np.cos(z)
    out = ctx.project(g.ravel(), "continuous", dims, L)
    assert np.abs(out - g.ravel()).max() <= 1e-10 * np.abs(g).max()


# --------------------------------------------------------------- preprocessing
@pytest.mark.parametrize("shape,fine,fac,params", [
    ("sphere", (256, 256, 256), (8, 8, 8), (0.4,)),
    ("sphere", (128, 128, 128), (4, 4, 4), ((0.15 / math.pi) ** (1 / 3),)),
    ("octahedron", (64, 64, 64), (8, 16, 2), (0.35,)),
    ("slab", (48, 16, 16), (6, 2, 4), (0, 0.4375)),
])
def test_generate_coarsen_normals_bit_exact(ctx, oracle, shape, fine, fac, params):
    img = ctx.generate(shape, fine, (1, 1, 1), *params)
    ref = oracle.generate(shape, fine, (1, 1, 1), *params)
    assert np.array_equal(img, ref)
    kind, cp, cnt = ctx.coarsen(img, fac)
    k2, cp2, cnt2 = oracle.coarsen(img, fac)
    assert np.array_equal(kind, k2) and np.array_equal(cnt, cnt2)
    assert np.array_equal(cp.view(np.uint64), cp2.view(np.uint64))
    if shape == "sphere" and fac == (8, 8, 8):
        assert int((kind == 2).sum()) == 2624
    for method in ("barycenter", "second_moment"):
        n, fl, st = ctx.compute_normals(img, fac, kind, method=method)
        n2, fl2, st2 = oracle.normals(img, fac, method={"barycenter": 0, "second_moment": 1}[method])
        assert np.array_equal(fl, fl2)
        assert np.array_equal(n.view(np.uint64), n2.view(np.uint64))
        assert tuple(st) == tuple(st2)


def test_plane_boxel_normals_bit_exact(ctx, oracle):
    th = 12.0 * np.pi / 180.0
    n0 = np.array([math.sin(th), math.cos(th), 0.0])
    i, j = np.meshgrid(np.arange(48), np.arange(18), indexing="ij")
    img = ((((i + 0.5) - 24.0) * n0[0] + ((j + 0.5) - 9.0) * n0[1] + 0.0) + 0.75 < 0).astype(np.uint8)
    img = img.reshape(48, 18, 1)
    L = (48.0, 18.0, 1.0)
    kind, _, _ = ctx.coarsen(img, (16, 6, 1))
    n, fl, _ = ctx.compute_normals(img, (16, 6, 1), kind, lengths=L)
    n2, fl2, _ = oracle.normals(img, (16, 6, 1), L, method=1)
    assert np.array_equal(n.view(np.uint64), n2.view(np.uint64))
    assert round(float(n[4] @ n0), 6) == 0.999983


def test_laplace_weights_bit_exact(ctx, oracle):
    img = oracle.generate("fiber_pack", (24, 20, 16), (1.0, 0.8, 1.2), 9, 10, 0.1, 0.5, 0.4)
    w = ctx.laplace_weights(img, (1.0, 0.8, 1.2))
    w2 = oracle.laplace_weights(img, (1.0, 0.8, 1.2))
    assert np.array_equal(w.view(np.uint64), w2.view(np.uint64))


def test_config_generators_volume_fraction(ctx):
    for shape, params, phi in [("rsa_spheres", (1, 3.0, 5.0, 0.3), 0.3), ("rsa_fibers_z", (1, 4.0, 0.35), 0.35),
                               ("boolean_ellipsoids", (1, 2.0, 6.0, 0.25), 0.25)]:
        img = ctx.generate(shape, (128, 128, 128), (1, 1, 1), *params)
        assert abs(img.mean() - phi) < 0.05, (shape, img.mean())
        assert np.array_equal(img, ctx.generate(shape, (128, 128, 128), (1, 1, 1), *params))


# --------------------------------------------------------------- material point
def _c1_grid(ctx, fine=128, fac=4):
    r = (0.15 / math.pi) ** (1 / 3)
    img = ctx.generate("sphere", (fine,) * 3, (1, 1, 1), r)
    kind, cp, _ = ctx.coarsen(img, (fac,) * 3)
    n, _, _ = ctx.compute_normals(img, (fac,) * 3, kind)
    return (fine // fac,) * 3, kind, cp, n


def test_laminate_back_projection_gpu(ctx):
    from paper_2204_13624_b200 import LaminateOptions, neo_hookean_enu

    stiff, soft = neo_hookean_enu(*STIFF), neo_hookean_enu(*SOFT)
    n = np.array([-1.0, 1.0, 1.0]) / math.sqrt(3.0)
    r = ctx.laminate_solve(shear(0.5), stiff, soft, n, 0.99625,
                           opts=LaminateOptions(tol_rel=1e-10, stress_floor=1e-12 * stiff.mu))
    assert r["converged"] and r["iterations"] == 5 and r["back_projections"] >= 1


def test_stress_sweep_and_tangent_vs_oracle(ctx, oracle):
    from paper_2204_13624_b200 import CellMaterials, neo_hookean

    dims, kind, cp, nrm = _c1_grid(ctx)
    m, i = neo_hookean(2.0, 1.0), neo_hookean(20.0, 10.0)
    cm = CellMaterials(ctx, dims, kind, cp, nrm, m, i)
    cmo = oracle.CellMaterials(dims, kind, cp, nrm, oracle.neo_hookean(2.0, 1.0), oracle.neo_hookean(20.0, 10.0))
    assert cm.composites == cmo.composites == int((kind == 2).sum())
    n = int(np.prod(dims))
    rng = np.random.default_rng(3)
    F = (np.eye(3).reshape(9, 1) + 0.1 * rng.uniform(-1, 1, (9, n))).ravel()
    P, st = cm.stress_sweep(F)
    Po, sto, t45 = cmo.stress_sweep(F, tangents=True)
    scale = np.abs(Po).max()
    assert np.abs(P - Po).max() <= 1e-12 * scale
    assert st[0] == sto[0] and st[1] == sto[1]
    assert np.abs(cm.warm() - cmo.warm()).max() <= 1e-12
    x = rng.uniform(-1, 1, 9 * n)
    y = cm.tangent_matvec(F, x)
    yo = oracle.tangent_matvec(t45, dims, x)
    assert np.abs(y - yo).max() <= 1e-10 * np.abs(yo).max()


# ----------------------------------------------------------------------- solver
def _compare_solves(r, ro, pbar_tol=1e-9, f_tol=1e-7, its=1):
    assert r["report"]["success"] == ro["report"]["success"]
    sg, so = r["report"]["steps"], ro["report"]["steps"]
    assert len(sg) == len(so)
    for a, b in zip(sg, so):
        assert abs(a["outer_iters"] - b["outer_iters"]) <= its, (a["outer_iters"], b["outer_iters"])
        assert a["line_search_cuts"] == b["line_search_cuts"]
        pa = np.array(a["pbar_history"][-1])
        pb = np.array(b["pbar_history"][-1])
        assert np.linalg.norm(pa - pb) <= pbar_tol * np.linalg.norm(pb)
    assert np.linalg.norm(r["pbar"] - ro["pbar"]) <= pbar_tol * np.linalg.norm(ro["pbar"])
    if r["f"] is not None and ro["f"] is not None:
        Fg = r["f"].reshape(9, -1)
        Fo = ro["f"].reshape(9, -1)
        rel = np.linalg.norm(Fg - Fo, axis=0) / np.linalg.norm(Fo, axis=0)
        assert rel.max() <= f_tol


def test_homogeneous_one_iteration_gpu(ctx):
    from paper_2204_13624_b200 import CellMaterials, neo_hookean_enu

    soft, stiff = neo_hookean_enu(*SOFT), neo_hookean_enu(*STIFF)
    n = 512
    for scheme, green in [("basic", "continuous"), ("basic", "rotated"), ("basic", "staggered"),
                          ("newton_cg", "continuous"), ("newton_cg", "rotated"), ("newton_cg", "staggered")]:
        cm = CellMaterials(ctx, (8, 8, 8), np.zeros(n, np.uint8), np.zeros(n), None, soft, stiff)
        r = cm.solve(shear(0.5), scheme=scheme, green=green)
        assert r["report"]["success"] and r["report"]["steps"][0]["outer_iters"] == 1
        assert np.abs(r["f"].reshape(9, -1) - shear(0.5).reshape(9, 1)).max() <= 1e-12


def test_laminate_rve_gpu(ctx, oracle):
    from paper_2204_13624_b200 import CellMaterials, neo_hookean_enu

    soft, stiff = neo_hookean_enu(*SOFT), neo_hookean_enu(*STIFF)
    img = np.array([1, 0], np.uint8).reshape(2, 1, 1)
    kind, cp, _ = ctx.coarsen(img, (1, 1, 1))
    lam = oracle.laminate_solve(shear(0.5), oracle.neo_hookean_enu(*STIFF), oracle.neo_hookean_enu(*SOFT),
                                [1, 0, 0], 0.5, opts=oracle.lam_opts(tol_rel=1e-13))
    for green in ("rotated", "staggered"):
        cm = CellMaterials(ctx, (2, 1, 1), kind, cp, np.zeros((2, 3)), soft, stiff)
        r = cm.solve(shear(0.5), green=green, tol_equilibrium=1e-12)
        assert r["report"]["success"]
        assert np.linalg.norm(r["pbar"] - lam["p_box"]) <= 1e-9 * np.linalg.norm(lam["p_box"])
        F = r["f"].reshape(9, 2)
        assert np.linalg.norm(F[:, 0] - lam["f_plus"].ravel()) <= 1e-8


def test_sphere_newton_vs_oracle(ctx, oracle):
    from paper_2204_13624_b200 import CellMaterials, neo_hookean_enu

    img = ctx.generate("sphere", (32, 32, 32), (1, 1, 1), 0.4)
    kind, cp, _ = ctx.coarsen(img, (2, 2, 2))
    n, _, _ = ctx.compute_normals(img, (2, 2, 2), kind)
    soft, stiff = neo_hookean_enu(*SOFT), neo_hookean_enu(*STIFF)
    for green in ("continuous", "rotated", "staggered"):
        cm = CellMaterials(ctx, (16, 16, 16), kind, cp, n, soft, stiff)
        r = cm.solve(shear(0.5), green=green, tol_equilibrium=1e-10, load_steps=2)
        cmo = oracle.CellMaterials((16, 16, 16), kind, cp, n, *laws(oracle))
        ro = cmo.solve(shear(0.5), scheme=1, green={"continuous": 0, "rotated": 1, "staggered": 2}[green],
                       tol=1e-10, load_steps=2)
        _compare_solves(r, ro)


def test_c1_basic_vs_oracle(ctx, oracle):
    # C1 exactly (32^3 grid, basic scheme, 10 load steps, tol 1e-6)
    from paper_2204_13624_b200 import CellMaterials, neo_hookean

    dims, kind, cp, nrm = _c1_grid(ctx)
    fbar = np.eye(3)
    fbar[0, 0] += 0.1
    cm = CellMaterials(ctx, dims, kind, cp, nrm, neo_hookean(2.0, 1.0), neo_hookean(20.0, 10.0))
    r = cm.solve(fbar, scheme="basic", green="rotated", tol_equilibrium=1e-6, load_steps=10, max_outer=5000)
    cmo = oracle.CellMaterials(dims, kind, cp, nrm, oracle.neo_hookean(2.0, 1.0), oracle.neo_hookean(20.0, 10.0))
    ro = cmo.solve(fbar, scheme=0, green=1, tol=1e-6, load_steps=10, max_outer=5000)
    assert r["report"]["success"] and ro["report"]["success"]
    _compare_solves(r, ro)
