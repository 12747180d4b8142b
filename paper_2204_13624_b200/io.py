"""Staged-pipeline artifacts: image / grid / field / slice files and report JSON.

Host-side mirror of the reference's I/O layer, so the GPU
path can consume and produce the same files as the reference's staged CLI
(`combo generate` -> `combo condense` -> `combo solve`):

  save_image / load_image      io.cpp:41-67   (io.hpp:20-23)
  save_grid  / load_grid       io.cpp:69-124  (io.hpp:25-28)
  save_field / load_field      io.cpp:126-150 (io.hpp:30-32)
  save_slice                   io.cpp:152-193 (io.hpp:34-36)
  mat3_to_json / report_to_json / phase_averages_to_json
                               io.cpp:195-256 (io.hpp:38-45)
  write_json / read_json       io.cpp:258-274 (nlohmann `dump(2)` + "\\n")

File layout (identical bytes to the reference): a JSON header with sorted keys
(nlohmann::json objects are std::map) indented by 2, and sibling little-endian
raw arrays named after the header (`x.json` -> `x.raw`, `x.kind.raw`, ...).
Errors raise `IOFailure` where the reference throws `combo::IOFailure`
(errors.hpp:45-47).

Arrays may be numpy arrays or torch tensors (CUDA tensors are copied to the
host first); loads return numpy arrays, ready to hand to `Context` /
`CellMaterials` (host buffers) or to upload.
"""
from __future__ import annotations

import json
import math
import os

import numpy as np

__all__ = [
    "IOFailure", "Image", "Grid", "save_image", "load_image", "save_grid", "load_grid", "save_field",
    "load_field", "save_slice", "mat3_to_json", "report_to_json", "phase_averages_to_json", "write_json",
    "read_json",
]


class IOFailure(RuntimeError):
    """combo::IOFailure (errors.hpp:45-47)."""


class Image:
    """PhaseImage (image.hpp:17-44): u8 phase labels, C order, k fastest."""

    def __init__(self, data, lengths=(1.0, 1.0, 1.0)):
        self.data = np.ascontiguousarray(_host(data), dtype=np.uint8)
        if self.data.ndim != 3:
            raise IOFailure("image: data must be 3-D")
        self.dims = tuple(int(d) for d in self.data.shape)
        self.lengths = tuple(float(x) for x in lengths)

    def inclusion_count(self):
        return int(np.count_nonzero(self.data))


class Grid:
    """ComboGrid (combo_grid.hpp:29-59): per boxel kind u8, c_plus f64,
    count_plus i64, normal (nb, 3) f64, normal_flag u8."""

    def __init__(self, dims, factors, lengths, kind, c_plus, normal, count_plus=None, normal_flag=None):
        self.dims = tuple(int(d) for d in dims)
        self.factors = tuple(int(f) for f in factors)
        self.lengths = tuple(float(x) for x in lengths)
        nb = int(np.prod(self.dims))
        self.kind = np.ascontiguousarray(_host(kind), dtype=np.uint8).reshape(nb)
        self.c_plus = np.ascontiguousarray(_host(c_plus), dtype=np.float64).reshape(nb)
        self.normal = np.ascontiguousarray(_host(normal), dtype=np.float64).reshape(nb, 3)
        if count_plus is None:
            # integer counts are exactly recoverable from the rational c_plus
            # (io.cpp:118-122): llround(c_plus * fine_per_boxel)
            count_plus = _llround(self.c_plus * float(self.fine_per_boxel()))
        self.count_plus = np.ascontiguousarray(_host(count_plus), dtype=np.int64).reshape(nb)
        # load_grid resets the flags to normal_none (io.cpp:123)
        self.normal_flag = (np.zeros(nb, np.uint8) if normal_flag is None
                            else np.ascontiguousarray(_host(normal_flag), dtype=np.uint8).reshape(nb))

    def boxel_count(self):
        return int(np.prod(self.dims))

    def fine_per_boxel(self):
        return int(np.prod(self.factors))

    def global_count_plus(self):
        return int(self.count_plus.sum())

    def composite_count(self):
        return int(np.count_nonzero(self.kind == 2))  # BoxelKind::composite (combo_grid.hpp:20)


def _host(a):
    if hasattr(a, "detach"):  # torch tensor (possibly on the device)
        a = a.detach().cpu().numpy()
    return np.asarray(a)


def _llround(x):
    # std::llround: half away from zero
    return (np.sign(x) * np.floor(np.abs(x) + 0.5)).astype(np.int64)


def _sibling(json_path, suffix):
    """io.cpp:33-38: replace the extension of the JSON path by `suffix`."""
    root, _ = os.path.splitext(os.fspath(json_path))
    return root + suffix


def _write_raw(path, arr):
    """io.cpp:16-23"""
    try:
        with open(path, "wb") as f:
            f.write(np.ascontiguousarray(arr).astype(np.asarray(arr).dtype.newbyteorder("<"), copy=False).tobytes())
    except OSError as e:
        raise IOFailure(f"cannot open for writing: {path}") from e


def _read_raw(path, dtype, count):
    """io.cpp:25-31: a short read is an error."""
    dt = np.dtype(dtype).newbyteorder("<")
    try:
        with open(path, "rb") as f:
            buf = f.read(count * dt.itemsize)
    except OSError as e:
        raise IOFailure(f"cannot open for reading: {path}") from e
    if len(buf) != count * dt.itemsize:
        raise IOFailure(f"short read: {path}")
    return np.frombuffer(buf, dtype=dt).astype(np.dtype(dtype), copy=True)


def _clean(v):
    """nlohmann writes non-finite doubles as null."""
    if isinstance(v, dict):
        return {str(k): _clean(x) for k, x in v.items()}
    if isinstance(v, (list, tuple)):
        return [_clean(x) for x in v]
    if isinstance(v, (np.integer,)):
        return int(v)
    if isinstance(v, (float, np.floating)):
        v = float(v)
        return v if math.isfinite(v) else None
    if isinstance(v, np.bool_):
        return bool(v)
    if isinstance(v, np.ndarray):
        return _clean(v.tolist())
    return v


def write_json(obj, path):
    """write_json (io.cpp:258-263): `j.dump(2)` + newline, keys sorted."""
    try:
        with open(path, "w") as f:
            f.write(json.dumps(_clean(obj), indent=2, sort_keys=True, ensure_ascii=False) + "\n")
    except OSError as e:
        raise IOFailure(f"cannot open for writing: {path}") from e


def read_json(path):
    """read_json (io.cpp:265-274)"""
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise IOFailure(f"cannot open for reading: {path}") from e
    try:
        return json.loads(text)
    except json.JSONDecodeError as e:
        raise IOFailure(f"bad JSON in {path}: {e}") from e


def _field(j, key):
    try:
        return j[key]
    except (KeyError, TypeError) as e:
        raise IOFailure(f"missing key '{key}'") from e


# ---------------------------------------------------------------- images
def save_image(img, json_path):
    """save_image (io.cpp:41-52)"""
    raw = _sibling(json_path, ".raw")
    write_json({"dims": list(img.dims), "lengths": list(img.lengths), "dtype": "u8", "order": "C, k fastest",
                "endianness": "little", "data": os.path.basename(raw)}, json_path)
    _write_raw(raw, img.data)


def load_image(json_path):
    """load_image (io.cpp:54-65)"""
    j = read_json(json_path)
    dims = tuple(int(d) for d in _field(j, "dims"))
    lengths = tuple(float(x) for x in _field(j, "lengths"))
    if _field(j, "dtype") != "u8":
        raise IOFailure("image: unsupported dtype")
    data = _read_raw(os.path.join(os.path.dirname(os.fspath(json_path)), _field(j, "data")), np.uint8,
                     int(np.prod(dims)))
    return Image(data.reshape(dims), lengths)


# ----------------------------------------------------------------- grids
def save_grid(grid, json_path):
    """save_grid (io.cpp:69-96): header + kind u8 / c_plus f64 / normals f64x3"""
    names = {"kind": ".kind.raw", "c_plus": ".c_plus.raw", "normals": ".normals.raw"}
    write_json({"dims": list(grid.dims), "factors": list(grid.factors), "lengths": list(grid.lengths),
                "global_count_plus": grid.global_count_plus(),
                "fine_voxels": grid.boxel_count() * grid.fine_per_boxel(),
                "composite_count": grid.composite_count(),
                "arrays": {k: os.path.basename(_sibling(json_path, s)) for k, s in names.items()}}, json_path)
    _write_raw(_sibling(json_path, ".kind.raw"), grid.kind)
    _write_raw(_sibling(json_path, ".c_plus.raw"), grid.c_plus)
    _write_raw(_sibling(json_path, ".normals.raw"), grid.normal)


def load_grid(json_path):
    """load_grid (io.cpp:98-124); count_plus recovered from c_plus, flags reset"""
    j = read_json(json_path)
    dims = tuple(int(d) for d in _field(j, "dims"))
    n = int(np.prod(dims))
    d = os.path.dirname(os.fspath(json_path))
    arrays = _field(j, "arrays")
    kind = _read_raw(os.path.join(d, _field(arrays, "kind")), np.uint8, n)
    cp = _read_raw(os.path.join(d, _field(arrays, "c_plus")), np.float64, n)
    nrm = _read_raw(os.path.join(d, _field(arrays, "normals")), np.float64, 3 * n)
    return Grid(dims, _field(j, "factors"), _field(j, "lengths"), kind, cp, nrm.reshape(n, 3))


# ---------------------------------------------------------------- fields
def save_field(f, dims, json_path, lengths=(1.0, 1.0, 1.0)):
    """save_field (io.cpp:126-138): 9 components, component-major, each C
    order with k fastest -- the (9, n1, n2, n3) SoA layout the GPU path
    keeps in HBM, so a device field is written without reordering."""
    data = np.ascontiguousarray(_host(f), dtype=np.float64)
    if data.size != 9 * int(np.prod(dims)):
        raise IOFailure("field: size does not match 9 x dims")
    raw = _sibling(json_path, ".raw")
    write_json({"dims": [int(x) for x in dims], "lengths": [float(x) for x in lengths], "dtype": "f64",
                "components": 9, "order": "component-major; per component C, k fastest", "endianness": "little",
                "data": os.path.basename(raw)}, json_path)
    _write_raw(raw, data)


def load_field(json_path):
    """load_field (io.cpp:140-150) -> (field (9, n1, n2, n3) f64, dims, lengths)"""
    j = read_json(json_path)
    dims = tuple(int(d) for d in _field(j, "dims"))
    lengths = tuple(float(x) for x in _field(j, "lengths"))
    data = _read_raw(os.path.join(os.path.dirname(os.fspath(json_path)), _field(j, "data")), np.float64,
                     9 * int(np.prod(dims)))
    return data.reshape((9,) + dims), dims, lengths


def save_slice(f, dims, comp, axis, index, json_path):
    """save_slice (io.cpp:152-193): one component's plane at `index` along
    `axis`, row-major over the two remaining axes."""
    dims = tuple(int(d) for d in dims)
    if axis < 0 or axis > 2 or index < 0 or index >= dims[axis]:
        raise IOFailure("slice: axis/index out of range")
    a = np.asarray(_host(f), dtype=np.float64).reshape((9,) + dims)[comp]
    plane = np.ascontiguousarray(np.take(a, index, axis=axis))
    raw = _sibling(json_path, ".raw")
    write_json({"dims": list(plane.shape), "dtype": "f64", "component": int(comp), "axis": int(axis),
                "index": int(index), "endianness": "little", "data": os.path.basename(raw)}, json_path)
    _write_raw(raw, plane)


# --------------------------------------------------------------- reports
def mat3_to_json(m):
    """mat3_to_json (io.cpp:195-203): row-major list of rows"""
    m = np.asarray(_host(m), dtype=np.float64).reshape(3, 3)
    return [[float(m[i, j]) for j in range(3)] for i in range(3)]


def report_to_json(report):
    """report_to_json (io.cpp:216-243) from the report dict `Solver.solve`
    returns (`combo_report_json`); wall-clock values only under "timings"."""
    steps, timings = [], []
    for s in report["steps"]:
        sw = s.get("sweep", {})
        steps.append({
            "t_start": s["t_start"], "t_end": s["t_end"], "fbar": mat3_to_json(s["fbar"]),
            "converged": bool(s["converged"]), "outer_iters": int(s["outer_iters"]),
            "residuals": [float(r) for r in s["residuals"]], "cg_iters": [int(c) for c in s["cg_iters"]],
            "cg_breakdowns": int(s["cg_breakdowns"]), "line_search_cuts": int(s["line_search_cuts"]),
            "laminate": {"failures": int(sw.get("failures", 0)), "back_projections": int(sw.get("back_projections", 0)),
                         "iter_max": int(sw.get("iter_max", 0))},
        })
        timings.append(float(s.get("seconds", 0.0)))
    return {"steps": steps, "success": bool(report["success"]), "error": report.get("error", ""),
            "bisections": int(report.get("bisections", 0)),
            "timings": {"per_step_seconds": timings, "total_seconds": float(report.get("seconds_total", 0.0))}}


def phase_averages_to_json(pa):
    """phase_averages_to_json (io.cpp:245-252) from the dict
    `CellMaterials.phase_averages` returns."""
    j = {"pbar": mat3_to_json(pa["pbar"]), "c_plus": float(pa["c_plus"])}
    if pa.get("has_plus", True) and pa.get("pbar_plus") is not None:
        j["pbar_plus"] = mat3_to_json(pa["pbar_plus"])
    if pa.get("has_minus", True) and pa.get("pbar_minus") is not None:
        j["pbar_minus"] = mat3_to_json(pa["pbar_minus"])
    return j
