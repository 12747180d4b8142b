"""Staged pipeline on the GPU: generate -> condense on the
device, save_grid / load_grid (io.cpp:69-124), solve from the loaded grid,
save_field / load_field of the device F (io.cpp:126-150), report_to_json
(io.cpp:216-243). Files must carry the oracle's bytes, and the solve from
the reloaded grid must be bitwise the solve from the in-memory grid."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_staged_pipeline_round_trip(ctx, oracle, tmp_path):
    import torch

    from paper_2204_13624_b200 import CellMaterials, neo_hookean_enu
    from paper_2204_13624_b200 import io as cio

    dims, fac = (32, 32, 32), (4, 4, 4)
    img_d = torch.empty(int(np.prod(dims)), dtype=torch.uint8, device="cuda")
    ctx.generate("sphere", dims, (1, 1, 1), 0.4, out=img_d)
    img = cio.Image(img_d.view(dims))
    cio.save_image(img, tmp_path / "img.json")
    assert np.array_equal(cio.load_image(tmp_path / "img.json").data, oracle.generate("sphere", dims, (1, 1, 1), 0.4))

    kind, cp, cnt = ctx.coarsen(img_d, fac, dims=dims)
    nrm, flags, _ = ctx.compute_normals(img_d, fac, kind, dims=dims)
    grid = cio.Grid((8, 8, 8), fac, (1, 1, 1), kind, cp, nrm, count_plus=cnt, normal_flag=flags)
    cio.save_grid(grid, tmp_path / "grid.json")
    g2 = cio.load_grid(tmp_path / "grid.json")
    ko, cpo, cnto = oracle.coarsen(img.data, fac)
    no, _, _ = oracle.normals(img.data, fac)
    assert np.array_equal(g2.kind, ko) and np.array_equal(g2.c_plus, cpo) and np.array_equal(g2.count_plus, cnto)
    assert np.array_equal(g2.normal, no)

    f = np.eye(3)
    f[0, 1] = 0.2
    soft, stiff = neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3)
    r1 = CellMaterials(ctx, grid.dims, grid.kind, grid.c_plus, grid.normal, soft, stiff).solve(f, tol_equilibrium=1e-9)
    r2 = CellMaterials(ctx, g2.dims, g2.kind, g2.c_plus, g2.normal, soft, stiff).solve(f, tol_equilibrium=1e-9)
    assert r1["report"]["success"] and r2["report"]["success"]
    F1 = np.asarray(r1["f"], dtype=np.float64)
    assert np.array_equal(F1, np.asarray(r2["f"], dtype=np.float64))

    cio.save_field(r1["f"], grid.dims, tmp_path / "f.json")
    F2, d2, _ = cio.load_field(tmp_path / "f.json")
    assert d2 == grid.dims and np.array_equal(F2.ravel(), F1.ravel())

    j1 = cio.report_to_json(r1["report"])
    j2 = cio.report_to_json(r2["report"])
    strip = lambda j: {k: v for k, v in j.items() if k != "timings"}  # noqa: E731
    assert strip(j1) == strip(j2)
