"""Interface tractions on laminate boxels: the device
recovery (`combo_recover_composites`) feeding facet_export /
interface_tractions, against the oracle's laminate solve; mirrors
test_postprocess.cpp:113-159 ("interface tractions on a single laminate
boxel") on a 4x4x4 grid of identical laminate boxels."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_interface_tractions_homogeneous_laminates(ctx, oracle, tmp_path):
    from paper_2204_13624_b200 import CellMaterials, neo_hookean_enu
    from paper_2204_13624_b200 import facets as fx

    dims = (4, 4, 4)
    n = int(np.prod(dims))
    kind = np.full(n, 2, np.uint8)
    cp = np.full(n, 0.5)
    nrm = np.tile([1.0, 0.0, 0.0], (n, 1))
    cm = CellMaterials(ctx, dims, kind, cp, nrm, neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3))
    fbar = np.eye(3)
    fbar[0, 1] = 0.4
    F = np.repeat(fbar.reshape(9, 1), n, axis=1).ravel()
    rec = cm.recover_composites(F)
    assert rec["cell"].shape == (n,) and sorted(rec["cell"].tolist()) == list(range(n))

    stiff, soft = oracle.neo_hookean_enu(10.0, 0.3), oracle.neo_hookean_enu(1.0, 0.0)
    lam = oracle.laminate_solve(fbar, stiff, soft, (1.0, 0.0, 0.0), 0.5, want_tangent=False)
    assert lam["converged"]
    ok, pp, _ = oracle.law_eval(stiff, lam["f_plus"])
    assert ok
    t_ref = pp @ np.array([1.0, 0.0, 0.0])
    for q in range(n):
        assert np.linalg.norm(rec["f_plus"][q] - lam["f_plus"]) <= 1e-12 * np.linalg.norm(lam["f_plus"])
        assert np.linalg.norm(rec["f_minus"][q] - lam["f_minus"]) <= 1e-12 * np.linalg.norm(lam["f_minus"])
        assert np.linalg.norm(rec["traction"][q] - t_ref) <= 1e-10 * np.linalg.norm(t_ref)

    facets = fx.facet_export(dims, (1.0, 1.0, 1.0), kind, cp, nrm)
    assert len(facets) == n
    s = fx.interface_tractions(rec, facets, dims)
    assert len(s) == n
    fmid = 0.5 * (lam["f_plus"] + lam["f_minus"])
    stretch = np.linalg.norm(np.linalg.det(fmid) * np.linalg.inv(fmid).T @ np.array([1.0, 0.0, 0.0]))
    for row in s:
        assert abs(row["area"] - 1.0 / 16.0) <= 1e-9
        assert abs(row["area_spatial"] - stretch * row["area"]) <= 1e-10 * stretch * row["area"]
        assert np.linalg.norm(row["traction_spatial"] * stretch - row["traction"]) <= 1e-12
    fx.write_traction_csv(s, tmp_path / "tractions.csv")

    # stress-free state: zero traction (test_postprocess.cpp:153-158)
    rec0 = cm.recover_composites(np.repeat(np.eye(3).reshape(9, 1), n, axis=1).ravel())
    assert np.abs(rec0["traction"]).max() <= 1e-12
