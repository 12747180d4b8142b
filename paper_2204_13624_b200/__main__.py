"""Staged command line (tools/combo_main.cpp:395-452) over the device path:

  python -m paper_2204_13624_b200 {generate,coarsen,normals,solve,post,bench}
      [--config cfg.json] [--out DIR] [--threads N] [--seed S] [--override key.path=value ...]

Failures exit 1 with {"error": {"type": ..., "message": ...}} on stderr
(test_cli.cpp:75-93). The device context is opened only when a stage first
touches the GPU, so configuration and missing-artifact errors are reported
without one. `bench --suite` writes the desk-scale comparison tables.
"""
from __future__ import annotations

import argparse
import json
import sys

from . import io as cio
from . import runconfig as rc


class _LazyContext:
    def __init__(self):
        self._ctx = None

    def __getattr__(self, name):
        if self._ctx is None:
            from .combo import Context

            self._ctx = Context(0)
        return getattr(self._ctx, name)


def error_type(e):
    """error_type (combo_main.cpp:395-407)"""
    from .combo import ComboError

    for cls, name in ((rc.ConfigInvalid, "ConfigInvalid"), (rc.UpstreamArtifactMissing, "UpstreamArtifactMissing"),
                      (rc.BadShapeSpec, "BadShapeSpec"), (cio.IOFailure, "IOFailure")):
        if isinstance(e, cls):
            return name
    if isinstance(e, ComboError):
        # combo::Error subclasses by name, any other combo::Error ->
        # SolverFailed; device / NCCL / allocation / API-misuse failures are
        # not combo::Error in the reference -> InternalError
        if e.type in ("ConfigInvalid", "BadShapeSpec", "NonDividingFactor", "LoadPathFailed",
                      "InadmissibleMacroState"):
            return e.type
        if e.type in ("CudaError", "NcclError", "OutOfMemory", "BadArgument", "BadState"):
            return "InternalError"
        return "SolverFailed"
    if isinstance(e, RuntimeError) and str(e).startswith("SolverFailed"):
        return "SolverFailed"
    return "InternalError"


def load_config(a):
    """load_config (combo_main.cpp:48-60)"""
    j = cio.read_json(a.config) if a.config else {}
    for ov in a.override or []:
        rc.apply_override(j, ov)
    if a.out:
        j.setdefault("output", {})["dir"] = a.out
    if a.threads is not None and a.threads >= 0:
        j["threads"] = a.threads
    if a.seed is not None and a.seed >= 0:
        j["seed"] = a.seed
    return rc.RunConfig.from_json(j)


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2204_13624_b200")
    sub = ap.add_subparsers(dest="stage", required=True)
    for name in ("generate", "coarsen", "normals", "solve", "post", "bench"):
        p = sub.add_parser(name)
        p.add_argument("--config")
        p.add_argument("--out")
        p.add_argument("--threads", type=int)
        p.add_argument("--seed", type=int)
        p.add_argument("--override", action="append")
        if name == "bench":
            p.add_argument("--suite", default="sphere-smoke")
    a = ap.parse_args(argv)
    stages = {"generate": rc.stage_generate, "coarsen": rc.stage_coarsen, "normals": rc.stage_normals,
              "solve": rc.stage_solve, "post": rc.stage_post}
    try:
        cfg = load_config(a)
        if a.stage == "bench":
            rc.stage_bench(_LazyContext(), cfg, a.suite)
        else:
            stages[a.stage](_LazyContext(), cfg)
    except Exception as e:  # noqa: BLE001 -- every failure becomes the JSON error record
        sys.stderr.write(json.dumps({"error": {"type": error_type(e), "message": str(e)}}) + "\n")
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
