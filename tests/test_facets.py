"""Facet geometry (paper_2204_13624_b200/facets.py), CPU only; mirrors
test_normals.cpp:158-211 ("box cut fraction and facet placement", "facets
recover c_plus for random planes") and the traction CSV schema (io.cpp:276-290)."""
import math

import numpy as np

from paper_2204_13624_b200 import facets as fx


def test_box_cut_fraction():
    lo, hi = (0, 0, 0), (1, 1, 1)
    assert abs(fx.box_cut_fraction(lo, hi, (1, 0, 0), 0.5) - 0.5) <= 1e-12
    assert fx.box_cut_fraction(lo, hi, (1, 0, 0), -0.1) == 0.0
    assert fx.box_cut_fraction(lo, hi, (1, 0, 0), 1.1) == 1.0
    # corner tetrahedron of side s: s^3 / 6
    n = np.ones(3) / math.sqrt(3.0)
    s = 0.4
    assert abs(fx.box_cut_fraction(lo, hi, n, s / math.sqrt(3.0)) - s ** 3 / 6.0) <= 1e-10 * s ** 3 / 6.0


def test_facets_recover_c_plus_random_planes():
    rng = np.random.default_rng(61)
    for _ in range(25):
        cp = 0.05 + 0.9 * rng.random()
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        fs = fx.facet_export((1, 1, 1), (1.0, 0.8, 1.3), [2], [cp], [n])
        assert len(fs) == 1
        frac = fx.box_cut_fraction((0, 0, 0), (1.0, 0.8, 1.3), fs[0].normal, fs[0].plane_offset)
        assert abs(frac - cp) <= 1e-8
        assert fs[0].area > 0.0
    fs = fx.facet_export((1, 1, 1), (1, 1, 1), [2], [0.5], [(1.0, 0.0, 0.0)])
    assert len(fs) == 1
    assert abs(fs[0].plane_offset - 0.5) <= 1e-9 and abs(fs[0].area - 1.0) <= 1e-9
    assert np.allclose(fs[0].centroid, (0.5, 0.5, 0.5))


def test_facets_skip_pure_and_zero_normal_boxels():
    kind = [0, 2, 1, 2]
    nrm = [(0, 0, 0), (0, 0, 1), (1, 0, 0), (0, 0, 0)]
    fs = fx.facet_export((1, 1, 4), (1, 1, 1), kind, [0, 0.25, 1, 0.5], nrm)
    assert [f.boxel for f in fs] == [(0, 0, 1)]
    # z-normal plane cutting a quarter of the boxel [0.25, 0.5] in z
    assert abs(fs[0].plane_offset - (0.25 + 0.25 * 0.25)) <= 1e-9


def test_tractions_nanson_and_csv(tmp_path):
    fs = fx.facet_export((1, 1, 1), (1, 1, 1), [2], [0.5], [(1.0, 0.0, 0.0)])
    f_plus = np.eye(3)
    f_plus[0, 0] = 1.2
    f_minus = np.eye(3)
    f_minus[0, 0] = 1.1
    rec = dict(cell=np.array([0]), f_plus=f_plus[None], f_minus=f_minus[None], traction=np.array([[2.0, 0.0, 0.0]]))
    s = fx.interface_tractions(rec, fs, (1, 1, 1))
    assert len(s) == 1
    fmid = 0.5 * (f_plus + f_minus)
    stretch = np.linalg.norm(np.linalg.det(fmid) * np.linalg.inv(fmid).T @ np.array([1.0, 0.0, 0.0]))
    assert abs(s[0]["area_spatial"] - stretch * s[0]["area"]) <= 1e-12
    assert np.linalg.norm(s[0]["traction_spatial"] * stretch - s[0]["traction"]) <= 1e-12
    fx.write_traction_csv(s, tmp_path / "t.csv")
    lines = (tmp_path / "t.csv").read_text().splitlines()
    assert lines[0] == "bi,bj,bk,cx,cy,cz,nx,ny,nz,Tx,Ty,Tz,Tnorm,tx,ty,tz,tnorm,area,area_spatial"
    assert len(lines) == 2 and len(lines[1].split(",")) == 19
