"""Staged-pipeline file formats (paper_2204_13624_b200/io.py), CPU only.

Mirrors the reference's own I/O tests:
  "image, grid and field files round trip"      test_config.cpp:84-119
  "slice of a constant field is constant; bad index throws"
                                                test_postprocess.cpp:180-198
  "report json isolates timings"                test_config.cpp:121+
plus byte-level checks of the header/raw layout io.cpp writes.
"""
import json
import os

import numpy as np
import pytest

from paper_2204_13624_b200 import io as cio


def _grid_from_oracle(oracle, img, factors, lengths):
    kind, cp, cnt = oracle.coarsen(img.data, factors, lengths)
    n3, flags, _ = oracle.normals(img.data, factors, lengths, method=1)
    dims = tuple(d // f for d, f in zip(img.dims, factors))
    return cio.Grid(dims, factors, lengths, kind, cp, n3, count_plus=cnt, normal_flag=flags)


def test_image_grid_field_round_trip(tmp_path, oracle):
    # test_config.cpp:84-119
    lengths = (1.0, 0.9, 1.1)
    img = cio.Image(oracle.generate("fiber_pack", (12, 10, 8), lengths, 3, 5, 0.1, 0.5, 0.2), lengths)
    cio.save_image(img, tmp_path / "img.json")
    img2 = cio.load_image(tmp_path / "img.json")
    assert img2.dims == img.dims
    assert img2.lengths == img.lengths
    assert np.array_equal(img2.data, img.data)

    grid = _grid_from_oracle(oracle, img, (4, 5, 2), lengths)
    cio.save_grid(grid, tmp_path / "grid.json")
    grid2 = cio.load_grid(tmp_path / "grid.json")
    assert grid2.dims == grid.dims
    assert np.array_equal(grid2.kind, grid.kind)
    assert np.array_equal(grid2.c_plus, grid.c_plus)
    assert np.array_equal(grid2.count_plus, grid.count_plus)  # recovered via llround
    assert np.array_equal(grid2.normal, grid.normal)
    assert grid2.global_count_plus() == img.inclusion_count()
    assert np.all(grid2.normal_flag == 0)  # io.cpp:123

    rng = np.random.default_rng(99)
    f = rng.uniform(-1.0, 1.0, size=(9, 5, 4, 3))
    cio.save_field(f, (5, 4, 3), tmp_path / "f.json")
    f2, dims, lengths2 = cio.load_field(tmp_path / "f.json")
    assert dims == (5, 4, 3) and lengths2 == (1.0, 1.0, 1.0)
    assert np.array_equal(f2, f)

    with pytest.raises(cio.IOFailure):
        cio.load_image(tmp_path / "missing.json")


def test_file_layout_matches_reference(tmp_path, oracle):
    """io.cpp:41-96 / 126-138: header keys, sibling names and raw bytes."""
    lengths = (1.0, 1.0, 1.0)
    img = cio.Image(oracle.generate("sphere", (8, 8, 8), lengths, 0.3), lengths)
    cio.save_image(img, tmp_path / "im.json")
    h = json.loads((tmp_path / "im.json").read_text())
    assert h == {"data": "im.raw", "dims": [8, 8, 8], "dtype": "u8", "endianness": "little",
                 "lengths": [1.0, 1.0, 1.0], "order": "C, k fastest"}
    assert (tmp_path / "im.raw").read_bytes() == img.data.tobytes()
    # nlohmann dump(2): sorted keys, two-space indent, trailing newline
    text = (tmp_path / "im.json").read_text()
    assert text.endswith("}\n") and text.startswith('{\n  "data": "im.raw",\n  "dims": [\n    8,')

    grid = _grid_from_oracle(oracle, img, (2, 2, 2), lengths)
    cio.save_grid(grid, tmp_path / "g.json")
    h = json.loads((tmp_path / "g.json").read_text())
    assert h["arrays"] == {"kind": "g.kind.raw", "c_plus": "g.c_plus.raw", "normals": "g.normals.raw"}
    assert h["fine_voxels"] == 512 and h["global_count_plus"] == img.inclusion_count()
    assert h["composite_count"] == int(np.count_nonzero(grid.kind == 2))
    assert (tmp_path / "g.normals.raw").read_bytes() == grid.normal.astype("<f8").tobytes()
    assert (tmp_path / "g.c_plus.raw").read_bytes() == grid.c_plus.astype("<f8").tobytes()

    f = np.arange(9 * 2 * 3 * 4, dtype=np.float64)
    cio.save_field(f, (2, 3, 4), tmp_path / "x.json")
    assert (tmp_path / "x.raw").read_bytes() == f.astype("<f8").tobytes()
    assert json.loads((tmp_path / "x.json").read_text())["components"] == 9


def test_short_read_and_bad_dtype(tmp_path):
    img = cio.Image(np.ones((4, 4, 4), np.uint8))
    cio.save_image(img, tmp_path / "a.json")
    raw = tmp_path / "a.raw"
    raw.write_bytes(raw.read_bytes()[:-1])
    with pytest.raises(cio.IOFailure, match="short read"):
        cio.load_image(tmp_path / "a.json")
    h = json.loads((tmp_path / "a.json").read_text())
    h["dtype"] = "f32"
    (tmp_path / "a.json").write_text(json.dumps(h))
    with pytest.raises(cio.IOFailure, match="unsupported dtype"):
        cio.load_image(tmp_path / "a.json")
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(cio.IOFailure, match="bad JSON"):
        cio.read_json(tmp_path / "bad.json")


def test_slice_constant_field_and_bad_index(tmp_path):
    # test_postprocess.cpp:180-198
    dims = (4, 5, 6)
    f = np.zeros((9,) + dims)
    for c in (0, 4, 8):
        f[c] = 2.5
    cio.save_slice(f, dims, 0, 2, 3, tmp_path / "slice.json")
    h = cio.read_json(tmp_path / "slice.json")
    assert h["dims"] == [4, 5]
    vals = np.frombuffer((tmp_path / "slice.raw").read_bytes(), "<f8")
    assert vals.size == 20 and np.all(vals == 2.5)
    with pytest.raises(cio.IOFailure):
        cio.save_slice(f, dims, 0, 2, 6, tmp_path / "bad.json")
    with pytest.raises(cio.IOFailure):
        cio.save_slice(f, dims, 0, 3, 0, tmp_path / "bad.json")


def test_slice_orientation():
    dims = (3, 4, 5)
    f = np.random.default_rng(1).standard_normal((9,) + dims)
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        for axis, idx, shape, ref in ((0, 1, [4, 5], f[2][1, :, :]), (1, 2, [3, 5], f[2][:, 2, :]),
                                      (2, 4, [3, 4], f[2][:, :, 4])):
            p = os.path.join(d, f"s{axis}.json")
            cio.save_slice(f, dims, 2, axis, idx, p)
            assert cio.read_json(p)["dims"] == shape
            got = np.frombuffer(open(os.path.join(d, f"s{axis}.raw"), "rb").read(), "<f8")
            assert np.array_equal(got, ref.ravel())


def test_report_json_isolates_timings(tmp_path):
    # test_config.cpp:121+ / test_cli.cpp:55-60: reports equal modulo "timings"
    step = {"t_start": 0.0, "t_end": 0.5, "fbar": [1.1, 0, 0, 0, 1, 0, 0, 0, 1], "converged": True, "outer_iters": 3,
            "residuals": [1e-2, 1e-5, 1e-9], "cg_iters": [0, 4, 6], "cg_breakdowns": 0, "line_search_cuts": 0,
            "seconds": 0.25, "sweep": {"failures": 0, "back_projections": 2, "iter_max": 4}}
    rep = {"steps": [step], "success": True, "error": "", "bisections": 0, "seconds_total": 0.3}
    j1 = cio.report_to_json(rep)
    j2 = cio.report_to_json({**rep, "seconds_total": 9.0, "steps": [{**step, "seconds": 7.0}]})
    assert j1 != j2
    strip = lambda j: {k: v for k, v in j.items() if k != "timings"}  # noqa: E731
    assert strip(j1) == strip(j2)
    assert j1["steps"][0]["fbar"] == [[1.1, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]
    assert j1["steps"][0]["laminate"] == {"failures": 0, "back_projections": 2, "iter_max": 4}
    assert j1["timings"] == {"per_step_seconds": [0.25], "total_seconds": 0.3}
    cio.write_json(j1, tmp_path / "r.json")
    assert cio.read_json(tmp_path / "r.json") == j1
    pa = cio.phase_averages_to_json({"pbar": np.eye(3), "c_plus": 0.2, "pbar_plus": 2 * np.eye(3),
                                     "pbar_minus": np.eye(3), "has_plus": True, "has_minus": False})
    assert set(pa) == {"pbar", "c_plus", "pbar_plus"}
