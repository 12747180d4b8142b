"""TEST INFRASTRUCTURE ONLY -- ctypes bindings of the CPU oracle (liboracle.so).

The oracle restates the reference ComBo solver (/root/reference/proj/src) in
plain C++/OpenMP (see oracle.hpp). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module, and
only as the checker or the CPU baseline -- never as the product path.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_U8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_I64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class Law(C.Structure):
    _fields_ = [("kind", C.c_int), ("lam", C.c_double), ("mu", C.c_double), ("c6", C.c_double * 36)]


class LamOpts(C.Structure):
    _fields_ = [("tol_abs", C.c_double), ("tol_rel", C.c_double), ("stress_floor", C.c_double),
                ("max_iter", C.c_int), ("back_projection", C.c_int), ("c_min", C.c_double)]


class SolverCfg(C.Structure):
    _fields_ = [("scheme", C.c_int), ("green", C.c_int), ("eval", C.c_int),
                ("tol_equilibrium", C.c_double), ("max_outer", C.c_int), ("cg_tol", C.c_double),
                ("cg_max", C.c_int), ("load_steps", C.c_int), ("max_bisections", C.c_int),
                ("threads", C.c_int), ("verbose", C.c_int), ("max_ls_iterations", C.c_longlong)]


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_generate.argtypes = [C.c_int, _I64, _D, _D, _U8]
        L.oracle_mirror.argtypes = [_U8, _I64, C.c_int, _U8]
        L.oracle_coarsen.argtypes = [_U8, _I64, _D, _I64, _U8, _D, _I64]
        L.oracle_laplace_weights.argtypes = [_U8, _I64, _D, _D]
        L.oracle_normals.argtypes = [_U8, _I64, _D, _I64, C.c_int, C.c_int, C.c_int, _D, _U8, _I64]
        L.oracle_sym_eig3.argtypes = [_D, _D, _D]
        L.oracle_law_eval.argtypes = [C.POINTER(Law), _D, _D, C.c_void_p]
        L.oracle_spectrum_bounds.argtypes = [C.POINTER(Law), _D, _D]
        L.oracle_laminate_solve.argtypes = [_D, C.POINTER(Law), C.POINTER(Law), _D, C.c_double, _D,
                                            C.POINTER(LamOpts), C.c_int, _D, _D, _D, C.c_void_p, _D,
                                            np.ctypeslib.ndpointer(dtype=np.int32), _D]
        L.oracle_cm_create.restype = C.c_void_p
        L.oracle_cm_create.argtypes = [_I64, _D, _U8, _D, _D, C.POINTER(Law), C.POINTER(Law),
                                       C.c_int, C.c_void_p]
        L.oracle_cm_destroy.argtypes = [C.c_void_p]
        L.oracle_cm_composites.argtypes = [C.c_void_p]
        L.oracle_cm_composites.restype = C.c_longlong
        L.oracle_cm_represented_c_plus.argtypes = [C.c_void_p]
        L.oracle_cm_represented_c_plus.restype = C.c_double
        L.oracle_cm_stress_floor.argtypes = [C.c_void_p]
        L.oracle_cm_stress_floor.restype = C.c_double
        L.oracle_cm_warm.argtypes = [C.c_void_p, _D, C.c_int]
        L.oracle_stress_sweep.argtypes = [C.c_void_p, _D, _D, C.c_void_p, _I64]
        L.oracle_phase_averages.argtypes = [C.c_void_p, _D, _D]
        L.oracle_tangent_matvec.argtypes = [_D, _I64, _D, _D]
        L.oracle_dfmg_stress.argtypes = [C.c_void_p, _D, _D, _I64]
        L.oracle_dfmg_tangent.argtypes = [C.c_void_p, _D, _D, _D]
        L.oracle_dfmg_warm.argtypes = [C.c_void_p, _D, C.c_int]
        L.oracle_project.argtypes = [_I64, _D, C.c_int, _D, _D]
        L.oracle_fft_forward.argtypes = [_I64, C.c_int, _D, _D]
        L.oracle_solve.restype = C.c_void_p
        L.oracle_solve.argtypes = [C.c_void_p, _D, C.POINTER(SolverCfg), C.c_void_p, C.c_void_p, _D]
        L.oracle_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _i64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _err():
    return lib().oracle_last_error().decode()


# ------------------------------------------------------------------ laws
def neo_hookean(lam, mu):
    return Law(0, float(lam), float(mu))


def neo_hookean_enu(e, nu):
    """materials.cpp:11-20"""
    return neo_hookean(e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), e / (2.0 * (1.0 + nu)))


def iso_mandel(lam, mu):
    """materials.cpp:22-30"""
    c = np.zeros((6, 6))
    c[:3, :3] = lam
    for i in range(3):
        c[i, i] += 2.0 * mu
        c[i + 3, i + 3] = 2.0 * mu
    return c


def linear(c6):
    law = Law(1, 0.0, 0.0)
    for i, v in enumerate(np.asarray(c6, dtype=np.float64).ravel()):
        law.c6[i] = v
    return law


def lam_opts(tol_abs=0.0, tol_rel=1e-10, stress_floor=0.0, max_iter=50, back_projection=True, c_min=0.0):
    return LamOpts(tol_abs, tol_rel, stress_floor, max_iter, int(back_projection), c_min)


# ------------------------------------------------------------ generators
SHAPES = {"sphere": 0, "octahedron": 1, "fiber": 2, "cross_ply": 3, "fiber_pack": 4, "slab": 5,
          "rsa_spheres": 10, "rsa_fibers_z": 11, "boolean_ellipsoids": 12}


def generate(shape, dims, lengths=(1.0, 1.0, 1.0), *params):
    out = np.zeros(int(np.prod(dims)), dtype=np.uint8)
    p = _f64(list(params) + [0.0] * (6 - len(params)))
    rc = lib().oracle_generate(SHAPES[shape], _i64(dims), _f64(lengths), p, out)
    if rc:
        raise ValueError(_err())
    return out.reshape(tuple(dims))


def mirrored(img, axis):
    out = np.zeros(img.size, dtype=np.uint8)
    lib().oracle_mirror(np.ascontiguousarray(img.ravel()), _i64(img.shape), int(axis), out)
    return out.reshape(img.shape)


def coarsen(img, factors, lengths=(1.0, 1.0, 1.0)):
    dims = np.array(img.shape, dtype=np.int64)
    f = _i64(factors)
    if np.any(f < 1) or np.any(dims % np.maximum(f, 1)):
        raise ValueError("NonDividingFactor")
    nb = int(np.prod(dims // f))
    kind = np.zeros(nb, np.uint8)
    cp = np.zeros(nb)
    cnt = np.zeros(nb, np.int64)
    rc = lib().oracle_coarsen(np.ascontiguousarray(img.ravel()), dims, _f64(lengths), f, kind, cp, cnt)
    if rc:
        raise ValueError(_err())
    return kind, cp, cnt


def laplace_weights(img, lengths=(1.0, 1.0, 1.0)):
    w = np.zeros(img.size)
    lib().oracle_laplace_weights(np.ascontiguousarray(img.ravel()), _i64(img.shape), _f64(lengths), w)
    return w.reshape(img.shape)


def normals(img, factors, lengths=(1.0, 1.0, 1.0), method=1, centering=0, min_support=3):
    dims = _i64(img.shape)
    nb = int(np.prod(dims // _i64(factors)))
    n3 = np.zeros(3 * nb)
    flags = np.zeros(nb, np.uint8)
    stats = np.zeros(3, np.int64)
    rc = lib().oracle_normals(np.ascontiguousarray(img.ravel()), dims, _f64(lengths), _i64(factors),
                              method, centering, min_support, n3, flags, stats)
    if rc:
        raise ValueError(_err())
    return n3.reshape(nb, 3), flags, stats


def sym_eig3(m):
    lam = np.zeros(3)
    vec = np.zeros(9)
    lib().oracle_sym_eig3(_f64(np.asarray(m).ravel()), lam, vec)
    return lam, vec.reshape(3, 3)


# ------------------------------------------------------------- materials
def law_eval(law, f, tangent=False):
    p = np.zeros(9)
    a = np.zeros(81) if tangent else None
    ok = lib().oracle_law_eval(C.byref(law), _f64(np.asarray(f).ravel()), p,
                               a.ctypes.data_as(C.c_void_p) if tangent else None)
    return ok == 0, p.reshape(3, 3), (a.reshape(9, 9) if tangent else None)


def spectrum_bounds(law, f):
    out = np.zeros(2)
    lib().oracle_spectrum_bounds(C.byref(law), _f64(np.asarray(f).ravel()), out)
    return out[0], out[1]


def laminate_solve(fbox, plus, minus, normal, c_plus, a0=(0, 0, 0), opts=None, want_tangent=True):
    opts = opts or lam_opts()
    p, fp, fm, a3 = np.zeros(9), np.zeros(9), np.zeros(9), np.zeros(3)
    a81 = np.zeros(81)
    ist = np.zeros(4, np.int32)
    dst = np.zeros(2)
    rc = lib().oracle_laminate_solve(_f64(np.asarray(fbox).ravel()), C.byref(plus), C.byref(minus),
                                     _f64(normal), float(c_plus), _f64(a0), C.byref(opts),
                                     int(want_tangent), p, fp, fm, a81.ctypes.data_as(C.c_void_p), a3, ist, dst)
    if rc == -2:
        raise ArithmeticError("InadmissibleMacroState: " + _err())
    if rc:
        raise ValueError(_err())
    return dict(p_box=p.reshape(3, 3), f_plus=fp.reshape(3, 3), f_minus=fm.reshape(3, 3),
                a_box=a81.reshape(9, 9), a=a3, converged=bool(ist[0]), iterations=int(ist[1]),
                back_projections=int(ist[2]), first_inadmissible_iter=int(ist[3]),
                residual=float(dst[0]), residual_rel=float(dst[1]))


# --------------------------------------------------------- cell materials
class CellMaterials:
    """CellMaterials (cell_material.hpp:19-74) over a coarse grid."""

    def __init__(self, dims, kind, c_plus, normal, matrix, inclusion, combo=True, opts=None,
                 lengths=(1.0, 1.0, 1.0)):
        self.dims = tuple(int(d) for d in dims)
        self.lengths = tuple(float(x) for x in lengths)
        self.n = int(np.prod(self.dims))
        normal = np.ascontiguousarray(np.asarray(normal, dtype=np.float64).reshape(-1))
        self._h = lib().oracle_cm_create(_i64(self.dims), _f64(self.lengths),
                                         np.ascontiguousarray(kind, dtype=np.uint8).ravel(),
                                         _f64(c_plus).ravel(), normal, C.byref(matrix), C.byref(inclusion),
                                         int(combo), C.byref(opts) if opts is not None else None)
        if not self._h:
            raise ValueError(_err())

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oracle_cm_destroy(self._h)
            self._h = None

    @property
    def composites(self):
        return int(lib().oracle_cm_composites(self._h))

    @property
    def represented_c_plus(self):
        return float(lib().oracle_cm_represented_c_plus(self._h))

    @property
    def stress_floor(self):
        return float(lib().oracle_cm_stress_floor(self._h))

    def warm(self, value=None):
        buf = np.zeros(3 * self.composites)
        if value is None:
            lib().oracle_cm_warm(self._h, buf, 0)
            return buf.reshape(-1, 3)
        buf[:] = np.asarray(value, dtype=np.float64).ravel()
        lib().oracle_cm_warm(self._h, buf, 1)

    def stress_sweep(self, F, tangents=False):
        F = _f64(F).ravel()
        P = np.zeros_like(F)
        st = np.zeros(4, np.int64)
        t = np.zeros(45 * self.n) if tangents else None
        lib().oracle_stress_sweep(self._h, F, P, t.ctypes.data_as(C.c_void_p) if tangents else None, st)
        return P, st, t

    def phase_averages(self, F):
        """recover_phase_fields + phase_averages (postprocess.cpp:13-106)."""
        out = np.zeros(31)
        if lib().oracle_phase_averages(self._h, _f64(F).ravel(), out) != 0:
            raise RuntimeError(_err())
        return dict(pbar=out[0:9].reshape(3, 3), pbar_plus=out[9:18].reshape(3, 3),
                    pbar_minus=out[18:27].reshape(3, 3), c_plus=out[27], has_plus=bool(out[28]),
                    has_minus=bool(out[29]), max_resolve_iterations=int(out[30]))

    def dfmg_stress(self, F):
        F = _f64(F).ravel()
        P = np.zeros_like(F)
        st = np.zeros(4, np.int64)
        lib().oracle_dfmg_stress(self._h, F, P, st)
        return P, st

    def dfmg_tangent_matvec(self, F, x):
        y = np.zeros(9 * self.n)
        lib().oracle_dfmg_tangent(self._h, _f64(F).ravel(), _f64(x).ravel(), y)
        return y

    def solve(self, fbar, scheme=1, green=1, eval=0, tol=1e-8, max_outer=200, cg_tol=1e-2, cg_max=2000,
              load_steps=1, max_bisections=5, max_ls_iterations=0, want_fields=True, want_p=None):
        cfg = SolverCfg(scheme, green, eval, tol, max_outer, cg_tol, cg_max, load_steps, max_bisections,
                        0, 0, max_ls_iterations)
        want_p = want_fields if want_p is None else want_p
        F = np.zeros(9 * self.n) if want_fields else None
        P = np.zeros(9 * self.n) if want_p else None
        pbar = np.zeros(9)
        ptr = lib().oracle_solve(self._h, _f64(np.asarray(fbar).ravel()), C.byref(cfg),
                                 F.ctypes.data_as(C.c_void_p) if want_fields else None,
                                 P.ctypes.data_as(C.c_void_p) if want_p else None, pbar)
        rep = json.loads(C.string_at(ptr).decode())
        lib().oracle_free(ptr)
        return dict(f=F, p=P, pbar=pbar.reshape(3, 3), report=rep)


def tangent_matvec(t45, dims, x):
    y = np.zeros(9 * int(np.prod(dims)))
    lib().oracle_tangent_matvec(_f64(t45), _i64(dims), _f64(x).ravel(), y)
    return y


def project(dims, lengths, kind, field):
    f = _f64(field).ravel()
    out = np.zeros_like(f)
    lib().oracle_project(_i64(dims), _f64(lengths), int(kind), f, out)
    return out


def fft_forward(dims, ncomp, field):
    n1, n2, n3 = dims
    nc = n1 * n2 * (n3 // 2 + 1)
    out = np.zeros(2 * ncomp * nc)
    lib().oracle_fft_forward(_i64(dims), int(ncomp), _f64(field).ravel(), out)
    return out.view(np.complex128).reshape(ncomp, n1, n2, n3 // 2 + 1)
