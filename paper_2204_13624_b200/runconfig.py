"""Run configuration and the staged pipeline around the GPU solve.

Mirrors the reference's caller side of the hot path:

  RunConfig.from_json / to_json      config.cpp:46-227 (config.hpp:17-44)
  make_material                      config.cpp:229-246
  apply_override                     config.cpp:277-302
  stage_generate / _coarsen / _normals / _solve / _post
                                     tools/combo_main.cpp:84-250 (cmd_*)

Artifacts are the reference's (`image.json`, `grid.json`, `solve_report.json`,
`F.json`, `P.json`, `averages.json`, `slice_<n>.json`,
`config_effective.<stage>.json`) in the same formats (io.py). Every stage
runs on the device through the C-ABI: generation, coarsening and normals
(`Context.generate/coarsen/compute_normals`), the solve and the phase
averages and the per-composite laminate recovery behind the traction CSV
(facet geometry is host arithmetic, facets.py). Out of scope: `bench` tables,
and the argv front end.
"""
from __future__ import annotations

import copy
import json
import os

import numpy as np

from . import io as cio

__all__ = ["ConfigInvalid", "BadShapeSpec", "UpstreamArtifactMissing", "RunConfig", "make_material",
           "apply_override", "stage_generate", "stage_coarsen", "stage_normals", "stage_solve", "stage_post"]


class ConfigInvalid(ValueError):
    """combo::ConfigInvalid (errors.hpp)"""


class BadShapeSpec(ValueError):
    """combo::BadShapeSpec (errors.hpp)"""


class UpstreamArtifactMissing(RuntimeError):
    """combo_main.cpp: a stage's input artifact does not exist"""


_SHAPES = {  # config.cpp:58-66
    "sphere": {"shape", "radius"},
    "octahedron": {"shape", "radius"},
    "fiber": {"shape", "axis", "radius", "length"},
    "cross_ply": {"shape", "radius", "pitch", "layers"},
    "fiber_pack": {"shape", "count", "radius", "length", "orientation_spread"},
    "slab": {"shape", "axis", "fraction"},
}
_GREEN = ("continuous", "rotated", "staggered")


def _reject_unknown(j, known, where):
    """config.cpp:13-21"""
    if not isinstance(j, dict):
        raise ConfigInvalid(f"config: {where} must be an object")
    for k in j:
        if k not in known:
            raise ConfigInvalid(f"config: unknown key \"{k}\" in {where}")


def _get(j, key, fallback):
    return j[key] if key in j else fallback


def _det3(m):
    m = np.asarray(m, dtype=np.float64)
    return float(np.linalg.det(m))


class RunConfig:
    """RunConfig (config.hpp:17-44) with the reference's defaults."""

    def __init__(self):
        self.geometry = None
        self.dims = [64, 64, 64]
        self.lengths = [1.0, 1.0, 1.0]
        self.coarsen_factors = [4, 4, 4]
        self.normal_method = "second_moment"
        self.centering = "weighted_centroid"
        self.min_interface_voxels = 3
        self.conv = "direct"
        self.materials = None
        self.loading = np.eye(3)
        self.loading[0, 1] = 0.5  # 50 % shear default (config.cpp:104-106)
        self.combo = True
        self.solver = dict(scheme="newton_cg", green="rotated", material_eval="per_cell", tol_equilibrium=1e-8,
                           max_outer=200, cg_tol=1e-2, cg_max=2000, load_steps=1, max_bisections=5, verbose=False)
        self.laminate = dict(tol_rel=1e-10, tol_abs=0.0, max_iter=50, back_projection=True, c_min=0.0)
        self.out_dir = "out"
        self.dump_fields = False
        self.slices = []
        self.seed = 0
        self.threads = 0

    @staticmethod
    def from_json(j):
        """RunConfig::from_json (config.cpp:46-183): unknown keys rejected
        at every level, enumerations checked, SolverConfig::validate."""
        _reject_unknown(j, {"geometry", "dims", "lengths", "coarsen", "normals", "materials", "loading", "solver",
                            "laminate", "output", "seed", "threads"}, "top level")
        c = RunConfig()
        g = j.get("geometry")
        if g:
            if "image" in g:
                _reject_unknown(g, {"image"}, "geometry")
            else:
                if "shape" not in g:
                    raise ConfigInvalid("config: geometry needs \"shape\" or \"image\"")
                if g["shape"] not in _SHAPES:
                    raise BadShapeSpec(f"config: unknown shape \"{g['shape']}\"")
                _reject_unknown(g, _SHAPES[g["shape"]], "geometry")
            c.geometry = copy.deepcopy(g)
        c.dims = [int(x) for x in _get(j, "dims", c.dims)]
        c.lengths = [float(x) for x in _get(j, "lengths", c.lengths)]
        c.coarsen_factors = [int(x) for x in _get(j, "coarsen", c.coarsen_factors)]
        if "normals" in j:
            n = j["normals"]
            _reject_unknown(n, {"method", "centering", "min_interface_voxels", "conv"}, "normals")
            c.normal_method = _get(n, "method", "second_moment")
            if c.normal_method not in ("barycenter", "second_moment"):
                raise ConfigInvalid(f"config: unknown normal method \"{c.normal_method}\"")
            c.centering = _get(n, "centering", "weighted_centroid")
            if c.centering not in ("weighted_centroid", "boxel_center"):
                raise ConfigInvalid(f"config: unknown centering \"{c.centering}\"")
            c.min_interface_voxels = int(_get(n, "min_interface_voxels", 3))
            c.conv = _get(n, "conv", "direct")
            if c.conv not in ("direct", "fft"):
                raise ConfigInvalid(f"config: unknown conv \"{c.conv}\"")
            if c.conv == "fft":
                # normals.cpp:54-84 (FFT Laplace weights) is not on the device
                # path; refuse it rather than silently using the direct stencil
                raise ConfigInvalid("config: normals.conv \"fft\" is not supported (use \"direct\")")
        if "materials" in j:
            _reject_unknown(j["materials"], {"matrix", "inclusion"}, "materials")
            c.materials = copy.deepcopy(j["materials"])
        if "loading" in j:
            c.loading = np.array(j["loading"], dtype=np.float64).reshape(3, 3)
            if not (_det3(c.loading) > 0.0):
                raise ConfigInvalid("config: loading must have positive determinant")
        if "solver" in j:
            s = j["solver"]
            _reject_unknown(s, {"scheme", "green", "material_eval", "tol_equilibrium", "max_outer", "cg_tol", "cg_max",
                                "load_steps", "combo", "max_bisections", "verbose"}, "solver")
            sv = c.solver
            sv["scheme"] = _get(s, "scheme", "newton_cg")
            if sv["scheme"] not in ("basic", "newton_cg"):
                raise ConfigInvalid(f"config: unknown scheme \"{sv['scheme']}\"")
            sv["green"] = _get(s, "green", "rotated")
            if sv["green"] not in _GREEN:
                raise ConfigInvalid(f"config: unknown green operator \"{sv['green']}\"")
            sv["material_eval"] = _get(s, "material_eval", "per_cell")
            if sv["material_eval"] not in ("per_cell", "dfmg"):
                raise ConfigInvalid(f"config: unknown material_eval \"{sv['material_eval']}\"")
            sv["tol_equilibrium"] = float(_get(s, "tol_equilibrium", 1e-8))
            sv["max_outer"] = int(_get(s, "max_outer", 200))
            sv["cg_tol"] = float(_get(s, "cg_tol", 1e-2))
            sv["cg_max"] = int(_get(s, "cg_max", 2000))
            sv["load_steps"] = int(_get(s, "load_steps", 1))
            sv["max_bisections"] = int(_get(s, "max_bisections", 5))
            sv["verbose"] = bool(_get(s, "verbose", False))
            c.combo = bool(_get(s, "combo", True))
        if "laminate" in j:
            lam = j["laminate"]
            _reject_unknown(lam, {"tol_rel", "tol_abs", "max_iter", "back_projection", "c_min"}, "laminate")
            c.laminate = dict(tol_rel=float(_get(lam, "tol_rel", 1e-10)), tol_abs=float(_get(lam, "tol_abs", 0.0)),
                              max_iter=int(_get(lam, "max_iter", 50)),
                              back_projection=bool(_get(lam, "back_projection", True)),
                              c_min=float(_get(lam, "c_min", 0.0)))
        if "output" in j:
            o = j["output"]
            _reject_unknown(o, {"dir", "dump_fields", "slices"}, "output")
            c.out_dir = str(_get(o, "dir", "out"))
            c.dump_fields = bool(_get(o, "dump_fields", False))
            c.slices = copy.deepcopy(o.get("slices", []))
        c.seed = int(_get(j, "seed", 0))
        c.threads = int(_get(j, "threads", 0))
        c.validate()
        return c

    def validate(self):
        """SolverConfig::validate (solver.cpp:277-284)"""
        s = self.solver
        if s["material_eval"] == "dfmg" and s["green"] != "staggered":
            raise ConfigInvalid("solver: dfmg material evaluation requires the staggered Green operator")
        if s["load_steps"] < 1:
            raise ConfigInvalid("solver: load_steps must be >= 1")
        if not (s["tol_equilibrium"] > 0.0):
            raise ConfigInvalid("solver: tol_equilibrium must be positive")

    def to_json(self):
        """RunConfig::to_json (config.cpp:185-227): the effective config."""
        return {
            "geometry": self.geometry if self.geometry is not None else {},
            "dims": list(self.dims), "lengths": list(self.lengths), "coarsen": list(self.coarsen_factors),
            "normals": {"method": self.normal_method, "centering": self.centering,
                        "min_interface_voxels": self.min_interface_voxels, "conv": self.conv},
            "materials": self.materials if self.materials is not None else {},
            "loading": cio.mat3_to_json(self.loading),
            "solver": {**{k: self.solver[k] for k in ("scheme", "green", "material_eval", "tol_equilibrium",
                                                      "max_outer", "cg_tol", "cg_max", "load_steps",
                                                      "max_bisections")},
                       "combo": self.combo, "verbose": self.solver["verbose"]},
            "laminate": dict(self.laminate),
            "output": {"dir": self.out_dir, "dump_fields": self.dump_fields, "slices": self.slices},
            "seed": self.seed, "threads": self.threads,
        }

    # --- handles for the device path
    def solver_config(self):
        from .combo import SolverConfig

        s = self.solver
        return SolverConfig(scheme=s["scheme"], green=s["green"], eval=s["material_eval"],
                            tol_equilibrium=s["tol_equilibrium"], max_outer=s["max_outer"], cg_tol=s["cg_tol"],
                            cg_max=s["cg_max"], load_steps=s["load_steps"], max_bisections=s["max_bisections"],
                            verbose=s["verbose"])

    def laminate_options(self):
        from .combo import LaminateOptions

        return LaminateOptions(**self.laminate)


def make_material(spec):
    """make_material (config.cpp:229-246) -> the C-ABI law struct."""
    from .combo import iso_mandel, linear, neo_hookean_enu

    model = spec.get("model")
    if model == "neo_hookean":
        _reject_unknown(spec, {"model", "E", "nu"}, "material")
        return neo_hookean_enu(float(spec["E"]), float(spec["nu"]))
    if model == "linear":
        _reject_unknown(spec, {"model", "E", "nu"}, "material")
        e, nu = float(spec["E"]), float(spec["nu"])
        # LinearElasticParams::from_enu -> isotropic (materials.cpp:22-39)
        return linear(iso_mandel(e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), e / (2.0 * (1.0 + nu))))
    if model == "thermal":
        raise ConfigInvalid("material: thermal conductivities parameterize the laminate ops, not the mechanical solver")
    raise ConfigInvalid(f"material: unknown model \"{model}\"")


def apply_override(config, assignment):
    """apply_override (config.cpp:277-302): key.path=value, value parsed as
    JSON when possible, else kept as a string."""
    if "=" not in assignment:
        raise ConfigInvalid("override must look like key.path=value")
    path, value = assignment.split("=", 1)
    keys = path.split(".")
    node = config
    for i, key in enumerate(keys):
        if not key:
            raise ConfigInvalid("override: empty key in path")
        if i == len(keys) - 1:
            try:
                node[key] = json.loads(value)
            except json.JSONDecodeError:
                node[key] = value
            return
        if not isinstance(node.get(key), dict):
            node[key] = {}
        node = node[key]


# ------------------------------------------------------------------ stages
def _artifact(cfg, name):
    return os.path.join(cfg.out_dir, name)


def _echo(cfg, stage):
    """load_config (combo_main.cpp:50-60): the effective config next to the outputs"""
    os.makedirs(cfg.out_dir, exist_ok=True)
    cio.write_json(cfg.to_json(), _artifact(cfg, f"config_effective.{stage}.json"))


def _material(cfg, key, e_default, nu_default):
    """material_or_default (combo_main.cpp:75-82)"""
    from .combo import neo_hookean_enu

    if cfg.materials and key in cfg.materials:
        return make_material(cfg.materials[key])
    return neo_hookean_enu(e_default, nu_default)


def _image(cfg):
    """obtain_image (combo_main.cpp:66-73)"""
    if cfg.geometry and "image" in cfg.geometry:
        return cio.load_image(cfg.geometry["image"])
    p = _artifact(cfg, "image.json")
    if os.path.exists(p):
        return cio.load_image(p)
    raise UpstreamArtifactMissing("no image found; run `generate` first or set geometry.image")


def stage_generate(ctx, cfg):
    """cmd_generate (combo_main.cpp:84-98) on the device generators."""
    _echo(cfg, "generate")
    g = cfg.geometry
    if not g or "shape" not in g:
        raise ConfigInvalid("generate: config needs geometry.shape")
    shape = g["shape"]
    if shape in ("sphere", "octahedron"):
        params = (float(g["radius"]),)
    elif shape == "slab":
        params = (float(int(g["axis"])), float(g["fraction"]))
    elif shape == "fiber":
        params = (float(int(g["axis"])), float(g["radius"]), float(g["length"]))
    elif shape == "cross_ply":
        params = (float(g["radius"]), float(g["pitch"]), float(int(g["layers"])))
    elif shape == "fiber_pack":
        params = (int(cfg.seed), float(int(g["count"])), float(g["radius"]), float(g["length"]),
                  float(g["orientation_spread"]))
    else:
        raise ConfigInvalid(f"generate: shape \"{shape}\" is not generated on the device path")
    img = cio.Image(ctx.generate(shape, tuple(cfg.dims), tuple(cfg.lengths), *params), cfg.lengths)
    cio.save_image(img, _artifact(cfg, "image.json"))
    cnt = img.inclusion_count()
    cio.write_json({"dims": list(img.dims), "inclusion_count": cnt,
                    "inclusion_fraction": cnt / float(img.data.size)}, _artifact(cfg, "generate_report.json"))
    return img


def stage_coarsen(ctx, cfg):
    """cmd_coarsen (combo_main.cpp:100-118)"""
    _echo(cfg, "coarsen")
    img = _image(cfg)
    kind, cp, cnt = ctx.coarsen(img.data, cfg.coarsen_factors)
    dims = tuple(d // f for d, f in zip(img.dims, cfg.coarsen_factors))
    grid = cio.Grid(dims, cfg.coarsen_factors, img.lengths, kind, cp, np.zeros((kind.size, 3)), count_plus=cnt)
    cio.save_grid(grid, _artifact(cfg, "grid.json"))
    fine = img.inclusion_count()
    cio.write_json({"dims": list(dims), "composite_boxels": grid.composite_count(),
                    "global_count_plus": grid.global_count_plus(),
                    "global_c_plus": grid.global_count_plus() / float(grid.boxel_count() * grid.fine_per_boxel()),
                    "fine_count_plus": fine, "volume_fraction_exact": grid.global_count_plus() == fine},
                   _artifact(cfg, "coarsen_report.json"))
    return grid


def stage_normals(ctx, cfg):
    """cmd_normals (combo_main.cpp:120-176; the analytic colinearity block
    of the report is omitted)"""
    _echo(cfg, "normals")
    gp = _artifact(cfg, "grid.json")
    if not os.path.exists(gp):
        raise UpstreamArtifactMissing("no grid.json; run `coarsen` first")
    img = _image(cfg)
    grid = cio.load_grid(gp)
    nrm, flags, st = ctx.compute_normals(img.data, grid.factors, grid.kind, img.lengths, method=cfg.normal_method,
                                         centering=cfg.centering, min_interface_voxels=cfg.min_interface_voxels)
    grid.normal = np.ascontiguousarray(nrm, dtype=np.float64)
    grid.normal_flag = np.asarray(flags, dtype=np.uint8)
    cio.save_grid(grid, gp)
    cio.write_json({"composite": int(st[0]), "degenerate_fallbacks": int(st[1]), "too_few_fallbacks": int(st[2])},
                   _artifact(cfg, "normals_report.json"))
    return grid


def _cell_materials(ctx, cfg, grid):
    from .combo import CellMaterials

    return CellMaterials(ctx, grid.dims, grid.kind, grid.c_plus, grid.normal, _material(cfg, "matrix", 1.0, 0.0),
                         _material(cfg, "inclusion", 10.0, 0.3), combo=cfg.combo, opts=cfg.laminate_options(),
                         lengths=grid.lengths)


def stage_solve(ctx, cfg):
    """cmd_solve + run_solve (combo_main.cpp:178-210): solve, phase averages,
    solve_report.json, optional F/P dumps."""
    _echo(cfg, "solve")
    gp = _artifact(cfg, "grid.json")
    if not os.path.exists(gp):
        raise UpstreamArtifactMissing("no grid.json; run `coarsen`/`normals` first")
    grid = cio.load_grid(gp)
    cm = _cell_materials(ctx, cfg, grid)
    r = cm.solve(cfg.loading, cfg.solver_config())
    if not r["report"]["success"]:
        raise RuntimeError("SolverFailed: " + r["report"].get("error", ""))
    pa = cm.phase_averages(r["f"])
    rep = {"averages": cio.phase_averages_to_json(pa), "report": cio.report_to_json(r["report"])}
    cio.write_json(rep, _artifact(cfg, "solve_report.json"))
    if cfg.dump_fields:
        cio.save_field(r["f"], grid.dims, _artifact(cfg, "F.json"), grid.lengths)
        cio.save_field(r["p"], grid.dims, _artifact(cfg, "P.json"), grid.lengths)
    return r, rep


def stage_post(ctx, cfg):
    """cmd_post (combo_main.cpp:212-245): phase averages at the dumped F,
    facet export + interface tractions (tractions.csv), configured slices."""
    _echo(cfg, "post")
    gp, fp = _artifact(cfg, "grid.json"), _artifact(cfg, "F.json")
    if not os.path.exists(gp):
        raise UpstreamArtifactMissing("no grid.json; run the pipeline first")
    if not os.path.exists(fp):
        raise UpstreamArtifactMissing("no F.json; run `solve` with output.dump_fields=true")
    grid = cio.load_grid(gp)
    f, dims, _ = cio.load_field(fp)
    cm = _cell_materials(ctx, cfg, grid)
    pa = cm.phase_averages(f.ravel())
    cio.write_json(cio.phase_averages_to_json(pa), _artifact(cfg, "averages.json"))
    from . import facets as fx

    facets = fx.facet_export(grid.dims, grid.lengths, grid.kind, grid.c_plus, grid.normal)
    samples = fx.interface_tractions(cm.recover_composites(f.ravel()), facets, grid.dims)
    fx.write_traction_csv(samples, _artifact(cfg, "tractions.csv"))
    for n, s in enumerate(cfg.slices):
        cio.save_slice(f, dims, int(s.get("component", 1)), int(s.get("axis", 2)), int(s.get("index", 0)),
                       _artifact(cfg, f"slice_{n}.json"))
    return pa


# ------------------------------------------------------------------- bench
def _error_norm(p, ref):
    """error_norm (postprocess.cpp:108-112)"""
    d = float(np.linalg.norm(ref))
    if not d > 0.0:
        raise ValueError("error_norm: zero reference")
    return float(np.linalg.norm(np.asarray(p) - np.asarray(ref))) / d


def _bench_run(ctx, label, dims, kind, cp, nrm, combo, loading, scfg):
    """bench_run (combo_main.cpp:277-293)"""
    from .combo import CellMaterials, neo_hookean_enu

    cm = CellMaterials(ctx, dims, kind, cp, nrm, neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3), combo=combo)
    r = cm.solve(loading, scfg)
    if not r["report"]["success"]:
        raise RuntimeError("SolverFailed in bench: " + label)
    pa = cm.phase_averages(r["f"])
    z = np.zeros((3, 3))
    return dict(label=label, pbar=pa["pbar"], pbar_plus=pa["pbar_plus"] if pa["has_plus"] else z,
                pbar_minus=pa["pbar_minus"] if pa["has_minus"] else z,
                seconds=float(r["report"].get("seconds_total", 0.0)))


def _emit_table(rows, path):
    """emit_table (combo_main.cpp:256-275): CSV against row 0 + console table"""
    ref = rows[0]
    with open(path, "w") as f:
        f.write("label,XX,XY,YX,YY,err_pbar_pct,err_plus_pct,err_minus_pct,seconds\n")
        g = lambda x: format(float(x), ".10g")  # noqa: E731
        print("\n  label                          P_XX     P_XY     P_YX     P_YY   err%")
        for r in rows:
            e = _error_norm(r["pbar"], ref["pbar"]) * 100.0
            ep = _error_norm(r["pbar_plus"], ref["pbar_plus"]) * 100.0
            em = _error_norm(r["pbar_minus"], ref["pbar_minus"]) * 100.0
            p = r["pbar"]
            f.write(",".join([r["label"], g(p[0, 0]), g(p[0, 1]), g(p[1, 0]), g(p[1, 1]), g(e), g(ep), g(em),
                              g(r["seconds"])]) + "\n")
            print(f"  {r['label']:<28s} {p[0, 0]:8.4f} {p[0, 1]:8.4f} {p[1, 0]:8.4f} {p[1, 1]:8.4f} {e:6.3f}")
        print()


def stage_bench(ctx, cfg, suite="sphere-smoke"):
    """cmd_bench (combo_main.cpp:295-393): desk-scale ComBo vs fine-grid
    comparison tables (sphere-desk / sphere-smoke / octahedron-desk /
    crossply-desk / fiber-desk), every solve on the device."""
    from .combo import SolverConfig

    _echo(cfg, "bench")
    loading = np.eye(3)
    loading[0, 1] = 0.5
    scfg = SolverConfig(scheme="newton_cg", green="rotated", tol_equilibrium=1e-7, load_steps=2)
    out = cfg.out_dir

    def grid(img, fac, method="second_moment"):
        kind, cp, _ = ctx.coarsen(img, fac)
        dims = tuple(d // f for d, f in zip(img.shape, fac))
        nrm = None
        if method is not None:
            nrm, _, _ = ctx.compute_normals(img, fac, kind, method=method)
        return dims, kind, cp, nrm

    def ref_row(img, label):
        dims, kind, cp, _ = grid(img, (1, 1, 1), None)
        return _bench_run(ctx, label, dims, kind, cp, np.zeros((kind.size, 3)), False, loading, scfg)

    def combo_row(label, g, combo=True):
        dims, kind, cp, nrm = g
        return _bench_run(ctx, label, dims, kind, cp, nrm, combo, loading, scfg)

    if suite in ("sphere-desk", "sphere-smoke"):
        fine, tag = (128, "desk") if suite == "sphere-desk" else (64, "smoke")
        img = ctx.generate("sphere", (fine,) * 3, (1.0, 1.0, 1.0), 0.4)
        rows = [ref_row(img, f"ref {fine}^3 (no combo)")]
        for fac in ((fine // 16,) * 3, (fine // 8, fine // 16, fine // 32)):
            for method, m in (("barycenter", "barycenter"), ("second_moment", "second-moment")):
                g = grid(img, fac, method)
                res = "x".join(str(d) for d in g[0])
                rows.append(combo_row(f"combo {res} {m}", g))
        _emit_table(rows, os.path.join(out, f"bench_sphere_{tag}.csv"))
    elif suite == "octahedron-desk":
        img = ctx.generate("octahedron", (128,) * 3, (1.0, 1.0, 1.0), 0.4)
        g = grid(img, (8, 8, 8))
        rows = [ref_row(img, "ref 128^3 (no combo)"), combo_row("combo 16^3", g),
                combo_row("staircase 16^3 (combo off)", g, combo=False)]
        _emit_table(rows, os.path.join(out, "bench_octahedron.csv"))
    elif suite == "crossply-desk":
        img = ctx.generate("cross_ply", (100,) * 3, (1.0, 1.0, 1.0), 0.1, 0.25, 4)
        rows = [ref_row(img, "ref 100^3 (no combo)"), combo_row("combo 25^3", grid(img, (4, 4, 4)))]
        _emit_table(rows, os.path.join(out, "bench_crossply.csv"))
    elif suite == "fiber-desk":
        img = ctx.generate("fiber_pack", (126,) * 3, (1.0, 1.0, 1.0), int(cfg.seed), 30, 0.03, 0.5, 0.25)
        rows = [ref_row(img, "ref 126^3 (no combo)")]
        for fac in ((6, 6, 6), (9, 3, 3)):
            g = grid(img, fac)
            rows.append(combo_row("combo " + "x".join(str(d) for d in g[0]), g))
        _emit_table(rows, os.path.join(out, "bench_fiber.csv"))
    else:
        raise ConfigInvalid(f"unknown bench suite \"{suite}\"")
    return rows
