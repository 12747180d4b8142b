"""Per-slab preprocessing for the multi-GPU decomposition (SURVEY.md 8e,
BASELINE C5 at 4096^3: every rank builds only its planes): plane windows of
the generators, slab coarsening and slab normals with one halo plane each
side are bit-identical to the whole-image results; the 64-bit generator
seed is exact; a CellMaterials handle retired by a later binding refuses to
run."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    ("rsa_spheres", (64, 48, 40), (4, 4, 4), (1, 3.0, 6.0, 0.3)),
    ("boolean_ellipsoids", (48, 48, 48), (2, 2, 2), (3, 2.0, 5.0, 0.25)),
    ("rsa_fibers_z", (64, 64, 32), (2, 2, 8), (5, 4.0, 0.35)),
    ("sphere", (32, 32, 32), (4, 4, 4), (0.3,)),
    ("fiber_pack", (48, 48, 48), (4, 4, 4), (7, 12, 0.05, 0.5, 0.25)),
]


@pytest.mark.parametrize("shape,fine,fac,params", CASES, ids=[c[0] for c in CASES])
def test_plane_windows_bit_identical(ctx, shape, fine, fac, params):
    whole = np.asarray(ctx.generate(shape, fine, (1, 1, 1), *params))
    n1 = fine[0]
    for plane0, nplanes in ((0, n1), (-1, 10), (n1 - 3, 7), (5, 1), (17, n1 // 2)):
        got = np.asarray(ctx.generate(shape, fine, (1, 1, 1), *params, planes=(plane0, nplanes)))
        idx = [(plane0 + t) % n1 for t in range(nplanes)]
        assert np.array_equal(got, whole[idx]), (plane0, nplanes)


@pytest.mark.parametrize("shape,fine,fac,params", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("R", [2, 4])
def test_slab_coarsen_and_normals(ctx, shape, fine, fac, params, R):
    whole = np.asarray(ctx.generate(shape, fine, (1, 1, 1), *params))
    kind, cp, cnt = ctx.coarsen(whole, fac)
    nrm, flags, st = ctx.compute_normals(whole, fac, kind)
    b1 = fine[0] // fac[0]
    if b1 % R:
        pytest.skip("R must divide the boxel planes")
    nbp = b1 // R
    nb_plane = (fine[1] // fac[1]) * (fine[2] // fac[2])
    tot = np.zeros(3, np.int64)
    for q in range(R):
        bp0 = q * nbp
        f0, nf = bp0 * fac[0], nbp * fac[0]
        win = np.asarray(ctx.generate(shape, fine, (1, 1, 1), *params, planes=(f0 - 1, nf + 2)))
        k, c, n = ctx.coarsen(np.ascontiguousarray(win[1:1 + nf]), fac)
        sl = slice(bp0 * nb_plane, (bp0 + nbp) * nb_plane)
        assert np.array_equal(k, kind[sl]) and np.array_equal(n, cnt.ravel()[sl])
        assert np.array_equal(c.view(np.uint64), cp[sl].view(np.uint64))
        nn, ff, s = ctx.compute_normals_slab(win, f0 - 1, fine, fac, bp0, nbp, k)
        assert np.array_equal(nn.view(np.uint64), nrm[sl].view(np.uint64))
        assert np.array_equal(ff, flags[sl])
        tot += np.asarray(s)
    assert tuple(tot) == tuple(st)


def test_normals_slab_window_check(ctx):
    from paper_2204_13624_b200 import ComboError

    fine, fac = (32, 32, 32), (4, 4, 4)
    win = np.asarray(ctx.generate("sphere", fine, (1, 1, 1), 0.3, planes=(8, 8)))  # no halo
    k, _, _ = ctx.coarsen(win, fac)
    with pytest.raises(ComboError):
        ctx.compute_normals_slab(win, 8, fine, fac, 2, 2, k)


def test_seed_is_64_bit_exact(ctx, oracle):
    # seeds above 2^53 used to pass through a double
    a = np.asarray(ctx.generate("rsa_spheres", (32, 32, 32), (1, 1, 1), 2**60, 2.0, 5.0, 0.2))
    b = np.asarray(ctx.generate("rsa_spheres", (32, 32, 32), (1, 1, 1), 2**60 + 1, 2.0, 5.0, 0.2))
    assert not np.array_equal(a, b)
    c = np.asarray(ctx.generate("rsa_spheres", (32, 32, 32), (1, 1, 1), 0, 2.0, 5.0, 0.2, seed=2**60 + 1))
    assert np.array_equal(b, c)
    # small seeds: unchanged and equal to the oracle's generator
    d = np.asarray(ctx.generate("rsa_spheres", (32, 32, 32), (1, 1, 1), 12345, 2.0, 5.0, 0.2))
    e = oracle.generate("rsa_spheres", (32, 32, 32), (1, 1, 1), 12345, 2.0, 5.0, 0.2)
    assert np.array_equal(d.ravel(), np.asarray(e).ravel())


def test_retired_cell_materials_refuse(ctx):
    from paper_2204_13624_b200 import CellMaterials, ComboError, neo_hookean

    kind = np.zeros(64, np.uint8)
    a = CellMaterials(ctx, (4, 4, 4), kind, np.zeros(64), None, neo_hookean(2, 1), neo_hookean(20, 10))
    b = CellMaterials(ctx, (4, 4, 4), kind, np.zeros(64), None, neo_hookean(2, 1), neo_hookean(20, 10), local=True)
    with pytest.raises(ComboError) as e:
        a.solve(np.eye(3))
    assert e.value.type == "BadState"
    r = b.solve(np.eye(3) + 0.01)
    assert r["report"]["success"]
