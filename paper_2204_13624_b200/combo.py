"""ctypes bindings of libcombo_cuda.so mirroring the reference API.

Reference interfaces mirrored (/root/reference/proj/include/combo):
  solve(CellMaterials&, fbar, SolverConfig)      solver.hpp:68-69
  CellMaterials(grid, matrix, inclusion, combo)  cell_material.hpp:22-23
  stress_sweep / tangent_matvec                  cell_material.hpp:90-96
  GreenOperator::project                         green.hpp:40
  coarsen / compute_normals / laplace_weights    combo_grid.hpp:62, normals.hpp:26-61
  generate_*                                     image.hpp:47-88
Error codes map onto the reference exception types (errors.hpp:11-55).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

GREEN = {"continuous": 0, "rotated": 1, "staggered": 2}
SCHEME = {"basic": 0, "newton_cg": 1}
EVAL = {"per_cell": 0, "dfmg": 1}
MEM_HOST, MEM_DEVICE = 0, 1

_ERRORS = {
    -1: "ConfigInvalid", -2: "InadmissibleMacroState", -3: "LoadPathFailed", -4: "SingularMatrix",
    -5: "NonDividingFactor", -6: "BadShapeSpec", -10: "CudaError", -11: "NcclError", -12: "OutOfMemory",
    -13: "BadArgument", -14: "BadState",
}


class ComboError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        self.type = _ERRORS.get(code, "Error")
        super().__init__(f"{self.type} ({code}): {msg}")


class Law(C.Structure):  # combo_law
    _fields_ = [("kind", C.c_int), ("lam", C.c_double), ("mu", C.c_double), ("c6", C.c_double * 36)]


class LamOpts(C.Structure):  # combo_laminate_opts
    _fields_ = [("tol_abs", C.c_double), ("tol_rel", C.c_double), ("stress_floor", C.c_double),
                ("max_iter", C.c_int), ("back_projection", C.c_int), ("c_min", C.c_double)]


class SolverCfg(C.Structure):  # combo_solver_cfg
    _fields_ = [("scheme", C.c_int), ("green", C.c_int), ("eval", C.c_int), ("tol_equilibrium", C.c_double),
                ("max_outer", C.c_int), ("cg_tol", C.c_double), ("cg_max", C.c_int), ("load_steps", C.c_int),
                ("max_bisections", C.c_int), ("threads", C.c_int), ("verbose", C.c_int),
                ("max_ls_iterations", C.c_longlong)]


class SweepStats(C.Structure):
    _fields_ = [("inadmissible_cells", C.c_int64), ("laminate_failures", C.c_int64),
                ("back_projections", C.c_int64), ("laminate_iter_max", C.c_int64)]


class PhaseAvg(C.Structure):  # combo_phase_avg (postprocess.hpp:27-35)
    _fields_ = [("pbar", C.c_double * 9), ("pbar_plus", C.c_double * 9), ("pbar_minus", C.c_double * 9),
                ("c_plus", C.c_double), ("has_plus", C.c_int32), ("has_minus", C.c_int32),
                ("max_resolve_iterations", C.c_int32)]


class NormalStats(C.Structure):
    _fields_ = [("composite", C.c_int64), ("degenerate_fallbacks", C.c_int64), ("too_few_fallbacks", C.c_int64)]


def lib_path():
    return os.path.join(_HERE, "libcombo_cuda.so")


_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_U8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_I64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_VP = C.c_void_p

# symbol -> (restype, argtypes); every function of include/combo_cuda.h
SIGNATURES = {
    "combo_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "combo_ctx_create_multi": (C.c_int, [C.c_int, _VP, C.POINTER(C.c_void_p)]),
    "combo_ctx_destroy": (C.c_int, [_VP]),
    "combo_last_error": (C.c_char_p, [_VP]),
    "combo_version": (C.c_char_p, []),
    "combo_kernel_launches": (C.c_int, [_VP, C.POINTER(C.c_int64)]),
    "combo_synchronize": (C.c_int, [_VP]),
    "combo_profile_enable": (C.c_int, [_VP, C.c_int]),
    "combo_profile_json": (C.c_char_p, [_VP]),
    "combo_reset_warm_starts": (C.c_int, [_VP]),
    "combo_get_stream": (C.c_int, [_VP, C.POINTER(C.c_void_p)]),
    "combo_generate": (C.c_int, [_VP, C.c_int, _I64, _D, _D, C.c_int, _VP, C.c_int]),
    "combo_coarsen": (C.c_int, [_VP, _VP, _I64, _I64, _VP, _VP, _VP, C.c_int]),
    "combo_laplace_weights": (C.c_int, [_VP, _VP, _I64, _D, _VP, C.c_int]),
    "combo_normals": (C.c_int, [_VP, _VP, _I64, _D, _I64, _VP, C.c_int, C.c_int, C.c_int, _VP, _VP,
                                C.POINTER(NormalStats), C.c_int]),
    "combo_generate_planes": (C.c_int, [_VP, C.c_int, _I64, _D, _D, C.c_int, C.c_uint64, C.c_int64, C.c_int64,
                                        _VP, C.c_int]),
    "combo_normals_slab": (C.c_int, [_VP, _VP, C.c_int64, C.c_int64, _I64, _D, _I64, C.c_int64, C.c_int64, _VP,
                                     C.c_int, C.c_int, C.c_int, _VP, _VP, C.POINTER(NormalStats), C.c_int]),
    "combo_bind_materials_slab": (C.c_int, [_VP, _I64, _D, _VP, _VP, _VP, C.POINTER(Law), C.POINTER(Law),
                                            C.c_int, C.POINTER(LamOpts), C.c_int]),
    "combo_bind_generation": (C.c_int, [_VP, C.POINTER(C.c_int64)]),
    "combo_set_grid": (C.c_int, [_VP, _I64, _D]),
    "combo_nccl_unique_id": (C.c_int, [_VP]),
    "combo_ctx_set_virtual_ranks": (C.c_int, [_VP, C.c_int]),
    "combo_ctx_set_ranks": (C.c_int, [_VP, C.c_int, C.c_int, _VP]),
    "combo_ctx_ranks": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "combo_slab_row": (C.c_int, [_I64, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, _VP]),
    "combo_chunk_range": (C.c_int, [_I64, C.c_int64, C.c_int64, _VP, _VP, _VP]),
    "combo_bind_materials": (C.c_int, [_VP, _I64, _D, _VP, _VP, _VP, C.POINTER(Law), C.POINTER(Law), C.c_int,
                                       C.POINTER(LamOpts), C.c_int]),
    "combo_composite_cells": (C.c_int, [_VP, C.POINTER(C.c_int64)]),
    "combo_stress_floor": (C.c_int, [_VP, C.POINTER(C.c_double)]),
    "combo_get_warm_starts": (C.c_int, [_VP, _VP, C.c_int]),
    "combo_set_warm_starts": (C.c_int, [_VP, _VP, C.c_int]),
    "combo_spectrum_bounds": (C.c_int, [_VP, _D, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "combo_stress_sweep": (C.c_int, [_VP, _VP, _VP, C.POINTER(SweepStats), C.c_int]),
    "combo_phase_averages": (C.c_int, [_VP, _VP, C.POINTER(PhaseAvg), C.c_int]),
    "combo_recover_composites": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, C.c_int]),
    "combo_tangent_matvec": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int]),
    "combo_tangent45": (C.c_int, [_VP, _VP, _VP, C.c_int]),
    "combo_tangent45_matvec": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int]),
    "combo_project": (C.c_int, [_VP, C.c_int, _VP, _VP, C.c_int]),
    "combo_fft_forward": (C.c_int, [_VP, _I64, C.c_int, _VP, _VP, C.c_int]),
    "combo_dfmg_stress": (C.c_int, [_VP, _VP, _VP, C.POINTER(SweepStats), C.c_int]),
    "combo_dfmg_tangent_matvec": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int]),
    "combo_dfmg_get_warm_starts": (C.c_int, [_VP, _VP, C.c_int]),
    "combo_laminate_solve": (C.c_int, [_VP, _D, C.POINTER(Law), C.POINTER(Law), _D, C.c_double, _D,
                                       C.POINTER(LamOpts), _D, _D, np.ctypeslib.ndpointer(dtype=np.int32)]),
    "combo_solve": (C.c_int, [_VP, _D, C.POINTER(SolverCfg), _VP, _VP, _D, C.POINTER(C.c_void_p), C.c_int]),
    "combo_report_summary": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "combo_report_step": (C.c_int, [_VP, C.c_int, _VP]),
    "combo_report_step_history": (C.c_int, [_VP, C.c_int, _VP, _VP, _VP]),
    "combo_report_json": (C.c_char_p, [_VP]),
    "combo_report_free": (C.c_int, [_VP]),
}


def load_library(path=None):
    """Load libcombo_cuda.so (no fallback: raises if it is missing)."""
    global _LIB
    if _LIB is None:
        p = path or lib_path()
        if not os.path.exists(p):
            raise ComboError(-14, f"{p} missing: build it with __graft_entry__.build()")
        L = C.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _is_dev(a):
    return hasattr(a, "data_ptr") and getattr(a, "is_cuda", False)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, int):
        return C.c_void_p(a)
    if hasattr(a, "data_ptr"):  # torch tensor (device memory or pinned host)
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _mem(*arrays):
    dev = [_is_dev(a) for a in arrays if a is not None]
    if any(dev) and not all(dev):
        raise ComboError(-13, "mixing host and device arrays in one call")
    return MEM_DEVICE if dev and dev[0] else MEM_HOST


def neo_hookean(lam, mu):
    """NeoHookeanParams given as (lambda, mu) (materials.hpp:14-21)."""
    return Law(0, float(lam), float(mu))


def neo_hookean_enu(e, nu):
    """NeoHookeanParams::from_enu (materials.cpp:11-20)."""
    return neo_hookean(e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), e / (2.0 * (1.0 + nu)))


def iso_mandel(lam, mu):
    """LinearElasticParams::isotropic (materials.cpp:22-30)."""
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


@dataclass
class LaminateOptions:  # laminate.hpp:72-79
    tol_abs: float = 0.0
    tol_rel: float = 1e-10
    stress_floor: float = 0.0
    max_iter: int = 50
    back_projection: bool = True
    c_min: float = 0.0

    def c(self):
        return LamOpts(self.tol_abs, self.tol_rel, self.stress_floor, self.max_iter, int(self.back_projection),
                       self.c_min)


@dataclass
class SolverConfig:  # solver.hpp:18-32
    scheme: str = "newton_cg"
    green: str = "rotated"
    eval: str = "per_cell"
    tol_equilibrium: float = 1e-8
    max_outer: int = 200
    cg_tol: float = 1e-2
    cg_max: int = 2000
    load_steps: int = 1
    max_bisections: int = 5
    verbose: bool = False
    max_ls_iterations: int = 0

    def c(self):
        return SolverCfg(SCHEME[self.scheme], GREEN[self.green], EVAL[self.eval], self.tol_equilibrium,
                         self.max_outer, self.cg_tol, self.cg_max, self.load_steps, self.max_bisections, 0,
                         int(self.verbose), self.max_ls_iterations)


def _i64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def slab_row(dims, nranks, rank, side, c, i, j):
    """Spectrum row offset (complex units) of (c, i, j) in the slab-side
    (side 0) or pencil-side (side 1) buffer of `rank` (combo_slab_row)."""
    off = C.c_int64()
    rc = load_library().combo_slab_row(_i64(dims), int(nranks), int(rank), int(side), int(c), int(i), int(j),
                                       C.byref(off))
    if rc:
        raise ComboError(rc, "combo_slab_row")
    return off.value


def chunk_range(dims, nplanes, block):
    """(beg, end, nblocks) of reduction chunk `block` of a slab of `nplanes`
    planes (combo_chunk_range)."""
    b, e, n = C.c_int64(), C.c_int64(), C.c_int64()
    rc = load_library().combo_chunk_range(_i64(dims), int(nplanes), int(block), C.byref(b), C.byref(e), C.byref(n))
    if rc:
        raise ComboError(rc, "combo_chunk_range")
    return b.value, e.value, n.value


class Context:
    """One device + stream (combo_ctx); devices=[...]: one process driving
    several GPUs as an axis-0 slab decomposition (combo_ctx_create_multi)."""

    def __init__(self, device=0, devices=None):
        self.L = load_library()
        h = C.c_void_p()
        if devices is None:
            self._check(self.L.combo_ctx_create(int(device), C.byref(h)), ctx=None)
        else:
            devs = (C.c_int * len(devices))(*[int(d) for d in devices])
            self._check(self.L.combo_ctx_create_multi(len(devices), devs, C.byref(h)), ctx=None)
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.combo_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, ctx="self"):
        if rc != 0:
            msg = self.L.combo_last_error(self.h if ctx == "self" else None)
            raise ComboError(rc, msg.decode() if msg else "")

    @property
    def kernel_launches(self):
        v = C.c_int64()
        self._check(self.L.combo_kernel_launches(self.h, C.byref(v)))
        return int(v.value)

    @property
    def stream(self):
        s = C.c_void_p()
        self._check(self.L.combo_get_stream(self.h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        self._check(self.L.combo_synchronize(self.h))

    def profile(self, enable=True):
        self._check(self.L.combo_profile_enable(self.h, int(enable)))

    def profile_report(self):
        return json.loads(self.L.combo_profile_json(self.h).decode())

    # ------------------------------------------------------------ images
    SHAPES = {"sphere": 0, "octahedron": 1, "fiber": 2, "cross_ply": 3, "fiber_pack": 4, "slab": 5,
              "rsa_spheres": 10, "rsa_fibers_z": 11, "boolean_ellipsoids": 12}
    SEEDED = ("fiber_pack", "rsa_spheres", "rsa_fibers_z", "boolean_ellipsoids")

    def generate(self, shape, dims, lengths=(1.0, 1.0, 1.0), *params, out=None, seed=None, planes=None):
        """generate_* (image.cpp:57-227) and the seeded config generators;
        `out` may be a CUDA uint8 tensor (device result). Seeded shapes take
        their seed as params[0] (a Python int is exact to 64 bits) or
        `seed`; planes = (plane0, nplanes) generates that window of fine
        planes (mod dims[0]) only, bit-identical to the whole image's."""
        dims = tuple(int(d) for d in dims)
        plane0, nplanes = (0, dims[0]) if planes is None else (int(planes[0]), int(planes[1]))
        if seed is None:
            seed = int(params[0]) if shape in self.SEEDED and params else 0
        if out is None:
            out = np.zeros(nplanes * dims[1] * dims[2], dtype=np.uint8)
        p = _f64([float(x) for x in params] + [0.0] * (8 - len(params)))
        self._check(self.L.combo_generate_planes(self.h, self.SHAPES[shape], _i64(dims), _f64(lengths), p,
                                                 len(params), C.c_uint64(int(seed) & (2**64 - 1)), plane0, nplanes,
                                                 _ptr(out), _mem(out)))
        return out.reshape((nplanes,) + dims[1:])

    def coarsen(self, img, factors, dims=None):
        """coarsen (combo_grid.cpp:28-71) -> kind, c_plus, count_plus (device
        tensors when img is a CUDA tensor)"""
        if _is_dev(img):
            import torch

            dims = _i64(dims if dims is not None else img.shape)
            f = _i64(factors)
            nb = int(np.prod(dims // np.maximum(f, 1)))
            kind = torch.empty(nb, dtype=torch.uint8, device=img.device)
            cp = torch.empty(nb, dtype=torch.float64, device=img.device)
            cnt = torch.empty(nb, dtype=torch.int64, device=img.device)
        else:
            img = np.ascontiguousarray(img, dtype=np.uint8)
            dims = _i64(img.shape)
            f = _i64(factors)
            nb = int(np.prod(dims // np.maximum(f, 1)))
            kind = np.zeros(nb, np.uint8)
            cp = np.zeros(nb)
            cnt = np.zeros(nb, np.int64)
        self._check(self.L.combo_coarsen(self.h, _ptr(img), dims, f, _ptr(kind), _ptr(cp), _ptr(cnt), _mem(img)))
        return kind, cp, cnt

    def laplace_weights(self, img, lengths=(1.0, 1.0, 1.0)):
        img = np.ascontiguousarray(img, dtype=np.uint8)
        w = np.zeros(img.size)
        self._check(self.L.combo_laplace_weights(self.h, _ptr(img), _i64(img.shape), _f64(lengths), _ptr(w),
                                                 MEM_HOST))
        return w.reshape(img.shape)

    def compute_normals(self, img, factors, kind, lengths=(1.0, 1.0, 1.0), method="second_moment",
                        centering="weighted_centroid", min_interface_voxels=3, dims=None):
        """compute_normals (normals.cpp:211-256) -> normals (nb,3), flags, stats"""
        if _is_dev(img):
            import torch

            dims = dims if dims is not None else img.shape
            nb = kind.numel()
            n3 = torch.empty(3 * nb, dtype=torch.float64, device=img.device)
            flags = torch.empty(nb, dtype=torch.uint8, device=img.device)
        else:
            img = np.ascontiguousarray(img, dtype=np.uint8)
            dims = img.shape
            kind = np.ascontiguousarray(kind, dtype=np.uint8)
            nb = kind.size
            n3 = np.zeros(3 * nb)
            flags = np.zeros(nb, np.uint8)
        st = NormalStats()
        m = {"barycenter": 0, "second_moment": 1}[method]
        cen = {"weighted_centroid": 0, "boxel_center": 1}[centering]
        self._check(self.L.combo_normals(self.h, _ptr(img), _i64(dims), _f64(lengths), _i64(factors),
                                         _ptr(kind), m, cen, int(min_interface_voxels), _ptr(n3), _ptr(flags),
                                         C.byref(st), _mem(img, kind)))
        return n3.reshape(nb, 3), flags, (st.composite, st.degenerate_fallbacks, st.too_few_fallbacks)

    def compute_normals_slab(self, img, img0, dims, factors, bp0, nbp, kind, lengths=(1.0, 1.0, 1.0),
                             method="second_moment", centering="weighted_centroid", min_interface_voxels=3):
        """compute_normals for boxel planes [bp0, bp0 + nbp) from the image
        window of fine planes starting at global plane img0 (mod dims[0])
        that holds them plus one halo plane each side -> (nbp*b2*b3, 3),
        flags, stats"""
        dims = tuple(int(d) for d in dims)
        nb = int(kind.numel() if _is_dev(kind) else np.asarray(kind).size)
        img_planes = (int(img.numel()) if _is_dev(img) else int(np.asarray(img).size)) // (dims[1] * dims[2])
        if _is_dev(img):
            import torch

            n3 = torch.empty(3 * nb, dtype=torch.float64, device=img.device)
            flags = torch.empty(nb, dtype=torch.uint8, device=img.device)
        else:
            img = np.ascontiguousarray(img, dtype=np.uint8)
            kind = np.ascontiguousarray(kind, dtype=np.uint8)
            n3 = np.zeros(3 * nb)
            flags = np.zeros(nb, np.uint8)
        st = NormalStats()
        m = {"barycenter": 0, "second_moment": 1}[method]
        cen = {"weighted_centroid": 0, "boxel_center": 1}[centering]
        self._check(self.L.combo_normals_slab(self.h, _ptr(img), int(img0), img_planes, _i64(dims), _f64(lengths),
                                              _i64(factors), int(bp0), int(nbp), _ptr(kind), m, cen,
                                              int(min_interface_voxels), _ptr(n3), _ptr(flags), C.byref(st),
                                              _mem(img, kind)))
        return n3.reshape(nb, 3), flags, (st.composite, st.degenerate_fallbacks, st.too_few_fallbacks)

    @property
    def bind_generation(self):
        v = C.c_int64()
        self._check(self.L.combo_bind_generation(self.h, C.byref(v)))
        return int(v.value)

    # ------------------------------------------------ slab decomposition
    def set_virtual_ranks(self, nranks):
        """Host `nranks` slab ranks on this context's device;
        bind / solve / project keep whole-grid arrays and are bitwise
        independent of the rank count."""
        self._check(self.L.combo_ctx_set_virtual_ranks(self.h, int(nranks)))

    def nccl_unique_id(self):
        buf = (C.c_char * 128)()
        self._check(self.L.combo_nccl_unique_id(buf), ctx=None)
        return bytes(buf)

    def set_ranks(self, nranks, rank, nccl_id=None):
        """One rank per process (NCCL): nccl_id from rank 0's nccl_unique_id(),
        broadcast by the caller (e.g. torch.distributed.broadcast_object_list)."""
        buf = None
        if nccl_id is not None:
            buf = (C.c_char * 128).from_buffer_copy(bytes(nccl_id))
        self._check(self.L.combo_ctx_set_ranks(self.h, int(nranks), int(rank), buf))

    def ranks(self):
        n, r, loc = C.c_int(), C.c_int(), C.c_int()
        i0, ni = C.c_int64(), C.c_int64()
        self._check(self.L.combo_ctx_ranks(self.h, C.byref(n), C.byref(r), C.byref(loc), C.byref(i0), C.byref(ni)))
        return {"nranks": n.value, "rank": r.value, "local_ranks": loc.value, "i0": i0.value, "ni": ni.value}

    def _out_fraction(self):
        rk = self.ranks()
        return rk["local_ranks"] / rk["nranks"]

    # --------------------------------------------------------- operators
    def set_grid(self, dims, lengths=(1.0, 1.0, 1.0)):
        self._check(self.L.combo_set_grid(self.h, _i64(dims), _f64(lengths)))

    def project(self, field, kind="rotated", dims=None, lengths=(1.0, 1.0, 1.0)):
        """GreenOperator::project (green.cpp:133-151) on a 9 x N field"""
        if dims is not None:
            self.set_grid(dims, lengths)
        f = _f64(field).ravel()
        out = np.zeros(int(round(f.size * self._out_fraction())))
        self._check(self.L.combo_project(self.h, GREEN[kind] if isinstance(kind, str) else int(kind), _ptr(f),
                                         _ptr(out), MEM_HOST))
        return out

    def fft_forward(self, dims, field):
        n1, n2, n3 = dims
        ncomp = int(np.asarray(field).size // (n1 * n2 * n3))
        out = np.zeros(2 * ncomp * n1 * n2 * (n3 // 2 + 1))
        self._check(self.L.combo_fft_forward(self.h, _i64(dims), ncomp, _ptr(_f64(field).ravel()), _ptr(out),
                                             MEM_HOST))
        return out.view(np.complex128).reshape(ncomp, n1, n2, n3 // 2 + 1)

    def laminate_solve(self, fbox, plus, minus, normal, c_plus, a0=(0, 0, 0), opts=None):
        opts = opts or LaminateOptions()
        p = np.zeros(9)
        a = np.zeros(3)
        ist = np.zeros(4, np.int32)
        oc = opts.c()
        self._check(self.L.combo_laminate_solve(self.h, _f64(np.asarray(fbox).ravel()), C.byref(plus),
                                                C.byref(minus), _f64(normal), float(c_plus), _f64(a0),
                                                C.byref(oc), p, a, ist))
        return dict(p_box=p.reshape(3, 3), a=a, converged=bool(ist[0]), iterations=int(ist[1]),
                    back_projections=int(ist[2]))


class CellMaterials:
    """CellMaterials (cell_material.hpp:19-74) bound on the device."""

    def __init__(self, ctx, dims, kind, c_plus, normal, matrix, inclusion, combo=True, opts=None,
                 lengths=(1.0, 1.0, 1.0), local=False):
        """kind / c_plus / normal describe the whole grid, or with local=True
        this process's slabs only (combo_bind_materials_slab). The materials
        live in the context: binding another CellMaterials on the same
        context retires this one (its calls then raise BadState)."""
        self.ctx = ctx
        self.dims = tuple(int(d) for d in dims)
        self.lengths = tuple(float(x) for x in lengths)
        self.n = int(np.prod(self.dims))
        if not _is_dev(kind):
            kind = np.ascontiguousarray(kind, dtype=np.uint8).ravel()
            c_plus = _f64(c_plus).ravel()
            normal = None if normal is None else _f64(normal).ravel()
        oc = (opts or LaminateOptions()).c()
        bind = ctx.L.combo_bind_materials_slab if local else ctx.L.combo_bind_materials
        ctx._check(bind(ctx.h, _i64(self.dims), _f64(self.lengths), _ptr(kind), _ptr(c_plus), _ptr(normal),
                        C.byref(matrix), C.byref(inclusion), int(combo), C.byref(oc), _mem(kind, c_plus, normal)))
        self._gen = ctx.bind_generation

    def _h(self):
        if self.ctx.bind_generation != self._gen:
            raise ComboError(-14, "CellMaterials: the context has been re-bound to other materials")
        return self.ctx.h

    def reset_warm_starts(self):
        """CellMaterials::reset_warm_starts (cell_material.cpp:64-66)"""
        self.ctx._check(self.ctx.L.combo_reset_warm_starts(self._h()))

    @property
    def composites(self):
        v = C.c_int64()
        self.ctx._check(self.ctx.L.combo_composite_cells(self._h(), C.byref(v)))
        return int(v.value)

    @property
    def stress_floor(self):
        v = C.c_double()
        self.ctx._check(self.ctx.L.combo_stress_floor(self._h(), C.byref(v)))
        return float(v.value)

    def warm(self, value=None):
        buf = np.zeros(3 * self.composites)
        if value is None:
            self.ctx._check(self.ctx.L.combo_get_warm_starts(self._h(), _ptr(buf), MEM_HOST))
            return buf.reshape(-1, 3)
        buf[:] = np.asarray(value, dtype=np.float64).ravel()
        self.ctx._check(self.ctx.L.combo_set_warm_starts(self._h(), _ptr(buf), MEM_HOST))

    def stress_sweep(self, F):
        F = _f64(F).ravel()
        P = np.zeros_like(F)
        st = SweepStats()
        self.ctx._check(self.ctx.L.combo_stress_sweep(self._h(), _ptr(F), _ptr(P), C.byref(st), MEM_HOST))
        return P, (st.inadmissible_cells, st.laminate_failures, st.back_projections, st.laminate_iter_max)

    def phase_averages(self, F):
        """recover_phase_fields + phase_averages (postprocess.cpp:13-106) at the
        converged F: composite laminates re-solved from the warm starts."""
        o = PhaseAvg()
        mem = _mem(F)
        if mem == MEM_HOST:
            F = _f64(F).ravel()
        self.ctx._check(self.ctx.L.combo_phase_averages(self._h(), _ptr(F), C.byref(o), mem))
        m = lambda a: np.array(a[:]).reshape(3, 3)  # noqa: E731
        return dict(pbar=m(o.pbar), pbar_plus=m(o.pbar_plus), pbar_minus=m(o.pbar_minus), c_plus=o.c_plus,
                    has_plus=bool(o.has_plus), has_minus=bool(o.has_minus),
                    max_resolve_iterations=int(o.max_resolve_iterations))

    def recover_composites(self, F):
        """recover_phase_fields per composite (postprocess.cpp:13-36) ->
        dict(cell (nc,), f_plus / f_minus (nc, 3, 3), traction (nc, 3))"""
        nc = self.composites
        mem = _mem(F)
        if mem == MEM_HOST:
            F = _f64(F).ravel()
        cell = np.zeros(max(nc, 1), np.int64)
        fp, fm, tr = np.zeros(9 * max(nc, 1)), np.zeros(9 * max(nc, 1)), np.zeros(3 * max(nc, 1))
        if mem != MEM_HOST:
            import torch

            dev = F.device
            cell = torch.from_numpy(cell).to(dev)
            fp, fm, tr = (torch.from_numpy(a).to(dev) for a in (fp, fm, tr))
        self.ctx._check(self.ctx.L.combo_recover_composites(self._h(), _ptr(F), _ptr(cell), _ptr(fp), _ptr(fm),
                                                            _ptr(tr), mem))
        if mem != MEM_HOST:
            cell, fp, fm, tr = (a.cpu().numpy() for a in (cell, fp, fm, tr))
        sl = max(nc, 1)
        return dict(cell=cell[:nc], f_plus=fp.reshape(9, sl)[:, :nc].T.reshape(nc, 3, 3),
                    f_minus=fm.reshape(9, sl)[:, :nc].T.reshape(nc, 3, 3), traction=tr.reshape(3, sl)[:, :nc].T)

    def tangent_matvec(self, F, x):
        y = np.zeros(9 * self.n)
        self.ctx._check(self.ctx.L.combo_tangent_matvec(self._h(), _ptr(_f64(F).ravel()), _ptr(_f64(x).ravel()),
                                                        _ptr(y), MEM_HOST))
        return y

    def tangent45(self, F):
        t = np.zeros(45 * self.n)
        self.ctx._check(self.ctx.L.combo_tangent45(self._h(), _ptr(_f64(F).ravel()), _ptr(t), MEM_HOST))
        return t

    def tangent45_matvec(self, t45, x):
        """tangent_matvec (cell_material.cpp:170-194) with caller-packed
        tangents [cell][45] (pack45, cell_material.cpp:86-102)"""
        y = np.zeros(9 * self.n)
        self.ctx._check(self.ctx.L.combo_tangent45_matvec(self._h(), _ptr(_f64(t45).ravel()),
                                                          _ptr(_f64(x).ravel()), _ptr(y), MEM_HOST))
        return y

    def dfmg_stress(self, F):
        F = _f64(F).ravel()
        P = np.zeros_like(F)
        st = SweepStats()
        self.ctx._check(self.ctx.L.combo_dfmg_stress(self._h(), _ptr(F), _ptr(P), C.byref(st), MEM_HOST))
        return P, (st.inadmissible_cells, st.laminate_failures, st.back_projections, st.laminate_iter_max)

    def dfmg_tangent_matvec(self, F, x):
        y = np.zeros(9 * self.n)
        self.ctx._check(self.ctx.L.combo_dfmg_tangent_matvec(self._h(), _ptr(_f64(F).ravel()),
                                                             _ptr(_f64(x).ravel()), _ptr(y), MEM_HOST))
        return y

    def solve(self, fbar, cfg=None, want_fields=True, f_out=None, p_out=None, **kw):
        """solve (solver.cpp:286-346) -> dict(f, p, pbar, report). f_out /
        p_out may be caller buffers (numpy / pinned or CUDA tensors)."""
        cfg = cfg or SolverConfig(**kw)
        nloc = int(round(self.n * self.ctx._out_fraction()))  # this process's slabs
        F = f_out if f_out is not None else (np.zeros(9 * nloc) if want_fields else None)
        P = p_out if p_out is not None else (np.zeros(9 * nloc) if want_fields else None)
        pbar = np.zeros(9)
        rep = C.c_void_p()
        cc = cfg.c()
        L = self.ctx.L
        self.ctx._check(L.combo_solve(self._h(), _f64(np.asarray(fbar).ravel()), C.byref(cc), _ptr(F), _ptr(P),
                                      pbar, C.byref(rep), _mem(F, P)))
        report = json.loads(L.combo_report_json(rep).decode())
        L.combo_report_free(rep)
        return dict(f=F, p=P, pbar=pbar.reshape(3, 3), report=report)
