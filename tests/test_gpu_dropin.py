"""The C++ drop-in layer (include/combo_b200.hpp) driving the GPU: the
reference's acceptance criterion 9 (2x1x1 laminate RVE vs the laminate
kernel, acceptance.cpp:407-434) checked against the oracle."""
import json
import subprocess

import numpy as np
import pytest

from test_capi import build_dropin_example

pytestmark = pytest.mark.gpu


def test_cpp_dropin_rve(tmp_path, oracle):
    exe = build_dropin_example(str(tmp_path / "dropin"))
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    f = np.eye(3)
    f[0, 1] = 0.5
    lam = oracle.laminate_solve(f, oracle.neo_hookean_enu(10.0, 0.3), oracle.neo_hookean_enu(1.0, 0.0), [1, 0, 0],
                                0.5, opts=oracle.lam_opts(tol_rel=1e-13))
    p = lam["p_box"]
    ref = np.array([p[0, 0], p[0, 1], p[1, 0], p[1, 1]])
    got = np.array(r["pbar"])
    assert r["success"]
    assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(p)
