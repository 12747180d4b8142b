"""RunConfig / make_material / apply_override (paper_2204_13624_b200/runconfig.py),
CPU only; mirrors test_config.cpp:11-78 of the reference."""
import pytest

from paper_2204_13624_b200 import runconfig as rc


def test_defaults_and_echo_round_trip():
    # test_config.cpp:11-24
    c = rc.RunConfig.from_json({})
    assert c.solver["scheme"] == "newton_cg"
    assert c.solver["green"] == "rotated"
    assert c.loading[0, 1] == 0.5
    assert c.laminate["tol_rel"] == 1e-10
    assert c.solver["tol_equilibrium"] == 1e-8
    echo = c.to_json()
    assert rc.RunConfig.from_json(echo).to_json() == echo


def test_unknown_keys_rejected_everywhere():
    # test_config.cpp:26-37
    for j in ({"bogus": 1}, {"solver": {"schem": "basic"}}, {"normals": {"methodd": "barycenter"}},
              {"geometry": {"shape": "sphere", "r": 1}}, {"laminate": {"tol": 1}}, {"output": {"dirr": "x"}},
              {"materials": {"fiber": {}}}):
        with pytest.raises(rc.ConfigInvalid):
            rc.RunConfig.from_json(j)


def test_invalid_values_rejected():
    # test_config.cpp:39-49 and SolverConfig::validate (solver.cpp:277-284)
    for j in ({"loading": [[-1, 0, 0], [0, 1, 0], [0, 0, 1]]},
              {"solver": {"material_eval": "dfmg", "green": "rotated"}}, {"solver": {"scheme": "x"}},
              {"solver": {"load_steps": 0}}, {"solver": {"tol_equilibrium": 0.0}}, {"normals": {"conv": "x"}},
              {"geometry": {"radius": 0.3}}):
        with pytest.raises(rc.ConfigInvalid):
            rc.RunConfig.from_json(j)
    with pytest.raises(rc.BadShapeSpec):
        rc.RunConfig.from_json({"geometry": {"shape": "moebius"}})
    c = rc.RunConfig.from_json({"solver": {"material_eval": "dfmg", "green": "staggered"}})
    assert c.solver["material_eval"] == "dfmg"


def test_material_factory():
    # test_config.cpp:51-62 (law structs of the C-ABI; no GPU needed)
    nh = rc.make_material({"model": "neo_hookean", "E": 10.0, "nu": 0.3})
    assert nh.kind == 0 and abs(nh.mu - 10.0 / 2.6) < 1e-15
    lin = rc.make_material({"model": "linear", "E": 1.0, "nu": 0.0})
    assert lin.kind == 1 and lin.c6[0] == 1.0
    with pytest.raises(rc.ConfigInvalid):
        rc.make_material({"model": "thermal", "kappa": [[1, 0, 0], [0, 1, 0], [0, 0, 1]]})
    with pytest.raises(rc.ConfigInvalid):
        rc.make_material({"model": "squishy"})
    with pytest.raises(rc.ConfigInvalid):
        rc.make_material({"model": "neo_hookean", "E": 1.0, "nu": 0.2, "G": 3})


def test_overrides_with_dot_paths():
    # test_config.cpp:64-74
    j = {}
    rc.apply_override(j, "solver.scheme=basic")
    rc.apply_override(j, "solver.tol_equilibrium=1e-6")
    rc.apply_override(j, "dims=[8,8,8]")
    c = rc.RunConfig.from_json(j)
    assert c.solver["scheme"] == "basic"
    assert c.solver["tol_equilibrium"] == 1e-6
    assert c.dims[0] == 8
    with pytest.raises(rc.ConfigInvalid):
        rc.apply_override(j, "no_equals_sign")
    with pytest.raises(rc.ConfigInvalid):
        rc.apply_override(j, "solver..x=1")


def test_missing_upstream_artifacts(tmp_path):
    # combo_main.cpp: stages fail with UpstreamArtifactMissing before touching the device
    c = rc.RunConfig.from_json({"output": {"dir": str(tmp_path / "o")}})
    with pytest.raises(rc.UpstreamArtifactMissing):
        rc.stage_solve(None, c)
    with pytest.raises(rc.UpstreamArtifactMissing):
        rc.stage_post(None, c)
    with pytest.raises(rc.UpstreamArtifactMissing):
        rc.stage_normals(None, c)
    assert (tmp_path / "o" / "config_effective.solve.json").exists()


def test_cli_failures_exit_nonzero_with_json(tmp_path):
    # test_cli.cpp:75-93
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2204_13624_b200", *a], cwd=root,  # noqa: E731
                                    capture_output=True, text=True, timeout=120)
    r = run("post", "--out", str(tmp_path / "o"))
    assert r.returncode != 0
    err = json.loads(r.stderr.strip().splitlines()[-1])
    assert err["error"]["type"] == "UpstreamArtifactMissing" and err["error"]["message"]
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"bogus_key": 1}))
    r = run("generate", "--config", str(bad))
    assert r.returncode != 0
    assert json.loads(r.stderr.strip().splitlines()[-1])["error"]["type"] == "ConfigInvalid"
    r = run("solve", "--out", str(tmp_path / "o"), "--override", "solver.scheme=nope")
    assert json.loads(r.stderr.strip().splitlines()[-1])["error"]["type"] == "ConfigInvalid"


def test_fft_laplace_weights_refused():
    # normals.conv = "fft" (normals.cpp:54-84) has no device path: refused,
    # never silently replaced by the direct stencil
    with pytest.raises(rc.ConfigInvalid):
        rc.RunConfig.from_json({"normals": {"conv": "fft"}})
    assert rc.RunConfig.from_json({"normals": {"conv": "direct"}}).to_json()["normals"]["conv"] == "direct"


def test_cli_error_types_follow_the_reference():
    # error_type (combo_main.cpp:395-407)
    from paper_2204_13624_b200.__main__ import error_type
    from paper_2204_13624_b200.combo import ComboError

    assert error_type(ComboError(-1, "x")) == "ConfigInvalid"
    assert error_type(ComboError(-2, "x")) == "InadmissibleMacroState"
    assert error_type(ComboError(-3, "x")) == "LoadPathFailed"
    assert error_type(ComboError(-5, "x")) == "NonDividingFactor"
    assert error_type(ComboError(-6, "x")) == "BadShapeSpec"
    assert error_type(ComboError(-4, "x")) == "SolverFailed"  # SingularMatrix is a combo::Error
    for code in (-10, -11, -12, -13, -14):
        assert error_type(ComboError(code, "x")) == "InternalError"
    assert error_type(ValueError("x")) == "InternalError"
