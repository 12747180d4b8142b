"""CLI `bench --suite sphere-desk` on the device (combo_main.cpp:295-340)
against the reference's acceptance criterion 7 as recorded in
test_output.txt:48-50 and pinned in tests/golden/c7_oracle.json: the fine
128^3 reference P-bar and the ComBo errors of the 16^3 and 8x16x32 grids."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_sphere_desk_matches_acceptance_c7(ctx, tmp_path):
    from paper_2204_13624_b200 import runconfig as rc

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c7_oracle.json")))
    cfg = rc.RunConfig.from_json({"output": {"dir": str(tmp_path)}})
    rows = rc.stage_bench(ctx, cfg, "sphere-desk")
    assert [r["label"] for r in rows] == ["ref 128^3 (no combo)", "combo 16x16x16 barycenter",
                                          "combo 16x16x16 second-moment", "combo 8x16x32 barycenter",
                                          "combo 8x16x32 second-moment"]
    ref = np.asarray(gold["ref_pbar"]).reshape(3, 3)
    assert np.linalg.norm(rows[0]["pbar"] - ref) <= 1e-9 * np.linalg.norm(ref)
    rec = gold["recorded_reference_run"]
    p = rows[0]["pbar"]
    assert (round(p[0, 0], 4), round(p[0, 1], 4), round(p[1, 0], 4), round(p[1, 1], 4)) == (
        rec["XX"], rec["XY"], rec["YX"], rec["YY"])
    err = lambda r: np.linalg.norm(r["pbar"] - p) / np.linalg.norm(p)  # noqa: E731
    for row, key in zip(rows[1:], (("combo_8_8_8", "barycenter"), ("combo_8_8_8", "second_moment"),
                                   ("combo_16_8_4", "barycenter"), ("combo_16_8_4", "second_moment"))):
        assert abs(err(row) - gold[key[0]][key[1]]) <= 1e-8, row["label"]
    # printed digits of test_output.txt:49-50
    assert [round(100 * err(r), 4) for r in rows[1:]] == [0.066, 0.0525, 1.5736, 0.1624]
    lines = (tmp_path / "bench_sphere_desk.csv").read_text().splitlines()
    assert lines[0].startswith("label,XX,XY,YX,YY,err_pbar_pct") and len(lines) == 6
