"""Post-solve phase recovery and phase averages on the GPU (SURVEY.md §8f #1,
postprocess.cpp:13-106) against the oracle at the same converged F and warm
starts, plus the reference's own identities (test_postprocess.cpp:31-84)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_phase_averages_vs_oracle(ctx, oracle):
    from paper_2204_13624_b200 import CellMaterials, neo_hookean_enu

    img = ctx.generate("sphere", (32, 32, 32), (1, 1, 1), 0.4)
    kind, cp, _ = ctx.coarsen(img, (4, 4, 4))
    nrm, _, _ = ctx.compute_normals(img, (4, 4, 4), kind)
    soft, stiff = neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3)
    cm = CellMaterials(ctx, (8, 8, 8), kind, cp, nrm, soft, stiff)
    f = np.eye(3)
    f[0, 1] = 0.3
    r = cm.solve(f, green="rotated", tol_equilibrium=1e-9)
    assert r["report"]["success"]
    pa = cm.phase_averages(r["f"])
    assert pa["max_resolve_iterations"] <= 1
    assert pa["has_plus"] and pa["has_minus"]
    rec = pa["c_plus"] * pa["pbar_plus"] + (1.0 - pa["c_plus"]) * pa["pbar_minus"]
    assert np.linalg.norm(rec - pa["pbar"]) <= 1e-12 * np.linalg.norm(pa["pbar"])
    assert np.linalg.norm(pa["pbar"] - r["pbar"]) <= 1e-10 * np.linalg.norm(r["pbar"])
    # oracle at the GPU's converged F and warm starts
    cmo = oracle.CellMaterials((8, 8, 8), kind, cp, nrm, oracle.neo_hookean_enu(1.0, 0.0),
                               oracle.neo_hookean_enu(10.0, 0.3))
    cmo.warm(cm.warm())
    po = cmo.phase_averages(r["f"])
    assert pa["max_resolve_iterations"] == po["max_resolve_iterations"]
    assert abs(pa["c_plus"] - po["c_plus"]) <= 1e-15
    for k in ("pbar", "pbar_plus", "pbar_minus"):
        assert np.linalg.norm(pa[k] - po[k]) <= 1e-12 * np.linalg.norm(po[k]), k


def test_phase_averages_all_matrix_gpu(ctx):
    from paper_2204_13624_b200 import CellMaterials, neo_hookean_enu

    kind = np.zeros(64, np.uint8)
    cm = CellMaterials(ctx, (4, 4, 4), kind, np.zeros(64), np.zeros(3 * 64), neo_hookean_enu(1.0, 0.0),
                       neo_hookean_enu(10.0, 0.3))
    f = np.eye(3)
    f[0, 1] = 0.2
    r = cm.solve(f, tol_equilibrium=1e-8)
    assert r["report"]["success"]
    pa = cm.phase_averages(r["f"])
    assert not pa["has_plus"] and pa["has_minus"]
    assert np.linalg.norm(pa["pbar_minus"] - pa["pbar"]) <= 1e-14 * np.linalg.norm(pa["pbar"])
