"""Facet export and interface tractions, host side.

  box_cut_fraction     normals.cpp:404-413
  facet_export         normals.cpp:415-469 (cut plane per composite boxel,
                       offset bisected so the inclusion side holds c_plus)
  interface_tractions  postprocess.cpp:114-141 (Nanson push-forward with
                       the midpoint deformation gradient)
  write_traction_csv   io.cpp:276-290

Facet geometry is per-boxel host arithmetic (a few hundred flops per
composite boxel, run once after a solve); the laminate states it consumes
come from the device (`CellMaterials.recover_composites`, one kernel).

The clipper follows the reference's polyhedron conventions: faces are
outward vertex loops, a vertex is kept when s = x.n - d <= eps, an edge is
split only where it strictly crosses (|s| > eps at both ends), vertices
closer than eps are merged, and the cap polygon is the set of distinct
crossing points ordered by angle around their mean in the plane basis
(u = (e_x or e_y) x n, w = n x u).
"""
from __future__ import annotations

import math

import numpy as np

__all__ = ["Facet", "box_cut_fraction", "facet_export", "interface_tractions", "write_traction_csv"]

_BOX_FACES = ((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (2, 3, 7, 6), (1, 2, 6, 5), (0, 4, 7, 3))


class Facet:
    """Facet (normals.hpp:72-79)"""

    def __init__(self, boxel, normal, plane_offset, polygon, centroid, area):
        self.boxel = boxel
        self.normal = normal
        self.plane_offset = plane_offset
        self.polygon = polygon
        self.centroid = centroid
        self.area = area


def _box(lo, hi):
    x0, y0, z0 = lo
    x1, y1, z1 = hi
    verts = [np.array(v, dtype=np.float64) for v in (
        (x0, y0, z0), (x1, y0, z0), (x1, y1, z0), (x0, y1, z0),
        (x0, y0, z1), (x1, y0, z1), (x1, y1, z1), (x0, y1, z1))]
    return verts, [list(f) for f in _BOX_FACES]


def _volume(verts, faces):
    v = 0.0
    for f in faces:
        a = verts[f[0]]
        for t in range(1, len(f) - 1):
            v += float(np.dot(a, np.cross(verts[f[t]], verts[f[t + 1]])))
    return v / 6.0


def _clip(verts, faces, n, d, eps):
    """Keep {x.n <= d}; returns (verts, faces, cap polygon)."""
    s = [float(np.dot(v, n)) - d for v in verts]
    nverts, nfaces, cap = [], [], []

    def vid(x):
        for i, u in enumerate(nverts):
            if np.linalg.norm(u - x) <= eps:
                return i
        nverts.append(x)
        return len(nverts) - 1

    for f in faces:
        loop = []
        m = len(f)
        for a in range(m):
            ia, ib = f[a], f[(a + 1) % m]
            sa, sb = s[ia], s[ib]
            if sa <= eps:
                loop.append(vid(verts[ia]))
            if (sa < -eps and sb > eps) or (sa > eps and sb < -eps):
                x = verts[ia] + (sa / (sa - sb)) * (verts[ib] - verts[ia])
                loop.append(vid(x))
                cap.append(x)
        clean = []
        for a, i in enumerate(loop):
            if not clean or (clean[-1] != i and not (a + 1 == len(loop) and i == clean[0])):
                clean.append(i)
        if len(clean) >= 3:
            nfaces.append(clean)
    uniq = []
    for x in cap:
        if all(np.linalg.norm(u - x) > eps for u in uniq):
            uniq.append(x)
    if len(uniq) >= 3:
        c = sum(uniq) / float(len(uniq))
        u = np.cross(np.array([1.0, 0.0, 0.0]) if abs(n[0]) < 0.9 else np.array([0.0, 1.0, 0.0]), n)
        u = u / np.linalg.norm(u)
        w = np.cross(n, u)
        uniq.sort(key=lambda x: math.atan2(float(np.dot(x - c, w)), float(np.dot(x - c, u))))
        nfaces.append([vid(x) for x in uniq])  # outward (+n) cap face
    return nverts, nfaces, uniq


def box_cut_fraction(lo, hi, n, d):
    """Volume fraction of the box [lo, hi] on the side x.n <= d."""
    lo, hi, n = (np.asarray(a, dtype=np.float64) for a in (lo, hi, n))
    verts, faces = _box(lo, hi)
    eps = 1e-12 * float(np.linalg.norm(hi - lo))
    nv, nf, _ = _clip(verts, faces, n, float(d), eps)
    if not nf:
        return 0.0
    return min(max(_volume(nv, nf) / float(np.prod(hi - lo)), 0.0), 1.0)


def facet_export(dims, lengths, kind, c_plus, normal):
    """One planar facet per composite boxel with a nonzero normal; the plane
    offset is bisected (<= 200 halvings, |fraction - c_plus| <= 1e-10)."""
    dims = tuple(int(x) for x in dims)
    bl = np.array([float(lengths[a]) / dims[a] for a in range(3)])
    kind = np.asarray(kind).reshape(-1)
    c_plus = np.asarray(c_plus, dtype=np.float64).reshape(-1)
    normal = np.asarray(normal, dtype=np.float64).reshape(-1, 3)
    out = []
    for ib in np.flatnonzero(kind == 2):
        n = normal[ib]
        if float(np.linalg.norm(n)) == 0.0:
            continue
        bi, bj, bk = (int(x) for x in np.unravel_index(int(ib), dims))
        lo = np.array([bi, bj, bk], dtype=np.float64) * bl
        hi = lo + bl
        corners = [np.dot(np.where([cx, cy, cz], hi, lo), n) for cx in (0, 1) for cy in (0, 1) for cz in (0, 1)]
        a, b = float(min(corners)), float(max(corners))
        target = float(c_plus[ib])
        d = 0.5 * (a + b)
        for _ in range(200):
            d = 0.5 * (a + b)
            frac = box_cut_fraction(lo, hi, n, d)
            if abs(frac - target) <= 1e-10:
                break
            if frac < target:
                a = d
            else:
                b = d
        verts, faces = _box(lo, hi)
        _, _, poly = _clip(verts, faces, n, d, 1e-12 * float(np.linalg.norm(hi - lo)))
        if len(poly) < 3:
            continue
        cen = sum(poly) / float(len(poly))
        area = sum(0.5 * float(np.linalg.norm(np.cross(poly[t] - poly[0], poly[t + 1] - poly[0])))
                   for t in range(1, len(poly) - 1))
        out.append(Facet((bi, bj, bk), n.copy(), d, poly, cen, area))
    return out


def interface_tractions(recovered, facets, dims):
    """interface_tractions (postprocess.cpp:114-141) from
    `CellMaterials.recover_composites(F)`: per facet the material traction
    T, its spatial push-forward t = T / |J F_mid^-T N| and the spatial area."""
    dims = tuple(int(x) for x in dims)
    by_cell = {int(c): q for q, c in enumerate(np.asarray(recovered["cell"]).tolist())}
    rows = []
    for f in facets:
        q = by_cell.get(int(np.ravel_multi_index(f.boxel, dims)))
        if q is None:
            continue
        t = np.asarray(recovered["traction"][q], dtype=np.float64)
        fmid = 0.5 * (recovered["f_plus"][q] + recovered["f_minus"][q])
        nanson = np.linalg.det(fmid) * np.linalg.inv(fmid).T @ f.normal
        stretch = float(np.linalg.norm(nanson))
        rows.append(dict(boxel=f.boxel, centroid=f.centroid, normal=f.normal, traction=t,
                         traction_spatial=t / stretch if stretch > 0.0 else np.zeros(3), area=f.area,
                         area_spatial=f.area * stretch))
    return rows


def write_traction_csv(samples, path):
    """write_traction_csv (io.cpp:276-290): fixed column schema, 17 digits."""
    g = lambda x: format(float(x), ".17g")  # noqa: E731
    with open(path, "w") as fh:
        fh.write("bi,bj,bk,cx,cy,cz,nx,ny,nz,Tx,Ty,Tz,Tnorm,tx,ty,tz,tnorm,area,area_spatial\n")
        for s in samples:
            t, ts = s["traction"], s["traction_spatial"]
            vals = [str(int(v)) for v in s["boxel"]] + [g(v) for v in s["centroid"]] + [g(v) for v in s["normal"]]
            vals += [g(v) for v in t] + [g(np.linalg.norm(t))] + [g(v) for v in ts] + [g(np.linalg.norm(ts))]
            vals += [g(s["area"]), g(s["area_spatial"])]
            fh.write(",".join(vals) + "\n")
