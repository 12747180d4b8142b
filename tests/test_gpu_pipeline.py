"""Staged pipeline generate -> coarsen -> normals -> solve -> post on the
device (runconfig.py, tools/combo_main.cpp:84-245): artifacts equal the
oracle's bit for bit (image, grid), the solve from the staged files equals a
direct CellMaterials solve bitwise, the phase averages of `post` at the
dumped F equal those of `solve`."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_pipeline_stages(ctx, oracle, tmp_path):
    from paper_2204_13624_b200 import CellMaterials, neo_hookean_enu
    from paper_2204_13624_b200 import io as cio
    from paper_2204_13624_b200 import runconfig as rc

    cfg = rc.RunConfig.from_json({
        "geometry": {"shape": "sphere", "radius": 0.3}, "dims": [32, 32, 32], "coarsen": [4, 4, 4],
        "loading": [[1.0, 0.2, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]],
        "solver": {"scheme": "newton_cg", "green": "rotated", "tol_equilibrium": 1e-9, "load_steps": 2},
        "output": {"dir": str(tmp_path), "dump_fields": True, "slices": [{"component": 1, "axis": 2, "index": 3}]},
    })
    img = rc.stage_generate(ctx, cfg)
    assert np.array_equal(img.data, oracle.generate("sphere", (32, 32, 32), (1, 1, 1), 0.3))
    rc.stage_coarsen(ctx, cfg)
    assert cio.read_json(tmp_path / "coarsen_report.json")["volume_fraction_exact"]
    grid = rc.stage_normals(ctx, cfg)
    ko, cpo, _ = oracle.coarsen(img.data, (4, 4, 4))
    no, fo, _ = oracle.normals(img.data, (4, 4, 4))
    g2 = cio.load_grid(tmp_path / "grid.json")
    assert np.array_equal(g2.kind, ko) and np.array_equal(g2.c_plus, cpo) and np.array_equal(g2.normal, no)
    assert np.array_equal(grid.normal_flag, fo)

    r, rep = rc.stage_solve(ctx, cfg)
    assert rep["report"]["success"] and len(rep["report"]["steps"]) == 2
    direct = CellMaterials(ctx, g2.dims, ko, cpo, no, neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3))
    rd = direct.solve(cfg.loading, cfg.solver_config())
    assert np.array_equal(np.asarray(rd["f"]), np.asarray(r["f"]))
    assert np.allclose(rep["averages"]["pbar"], rd["pbar"], rtol=1e-9, atol=1e-14)
    F, dims, _ = cio.load_field(tmp_path / "F.json")
    assert dims == (8, 8, 8) and np.array_equal(F.ravel(), np.asarray(r["f"]).ravel())

    rc.stage_post(ctx, cfg)
    av = cio.read_json(tmp_path / "averages.json")
    assert np.allclose(av["pbar"], rep["averages"]["pbar"], rtol=1e-8, atol=1e-14)  # re-solved from cold warm starts
    assert (tmp_path / "slice_0.raw").stat().st_size == 8 * 8 * 8
    rows = (tmp_path / "tractions.csv").read_text().splitlines()
    assert len(rows) - 1 == int(np.count_nonzero((g2.kind == 2) & (np.linalg.norm(g2.normal, axis=1) > 0)))
    for s in ("generate", "coarsen", "normals", "solve", "post"):
        assert (tmp_path / f"config_effective.{s}.json").exists()


def test_cli_stage_chain(tmp_path):
    """python -m paper_2204_13624_b200 generate/coarsen/normals/solve/post
    (combo_main.cpp; test_cli.cpp:32-73): each stage exits 0, reports
    reproduce modulo "timings"."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"geometry": {"shape": "sphere", "radius": 0.3}, "dims": [16, 16, 16],
                               "coarsen": [2, 2, 2], "loading": [[1.0, 0.1, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]],
                               "solver": {"scheme": "newton_cg", "tol_equilibrium": 1e-8},
                               "output": {"dump_fields": True}}))
    out = tmp_path / "o"

    def run(stage):
        r = subprocess.run([sys.executable, "-m", "paper_2204_13624_b200", stage, "--config", str(cfg), "--out",
                            str(out)], cwd=root, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr

    for s in ("generate", "coarsen", "normals", "solve"):
        run(s)
    rep1 = json.loads((out / "solve_report.json").read_text())
    run("solve")
    rep2 = json.loads((out / "solve_report.json").read_text())
    strip = lambda j: {k: v for k, v in j["report"].items() if k != "timings"}  # noqa: E731
    assert strip(rep1) == strip(rep2) and rep1["averages"] == rep2["averages"]
    assert rep1["report"]["success"]
    run("post")
    assert (out / "averages.json").exists() and (out / "tractions.csv").exists()
    assert json.loads((out / "coarsen_report.json").read_text())["volume_fraction_exact"]
