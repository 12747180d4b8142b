"""TEST INFRASTRUCTURE ONLY: full-size oracle fixtures for tests/test_gpu_fullsize.py.

Runs the CPU oracle (oracle/, the C++/OpenMP restatement of the reference)
on BASELINE configs C2-C5 at their real sizes -- seeded image generation,
coarsening, normals, then the solve along the config's load path
(/root/reference/proj/src/solver.cpp:286-346), with the LS budgets of
tests/fullsize_common.py::CASES -- and writes

  tests/golden/full_<case>.json    grid digests, the full report, F sums,
                                   the run's CPU facts (cores, seconds)
  tests/golden/full_<case>_F.npy   F at the seeded sample cells [n, 9]

Needs the host RAM of the B200 box for C4 / C5 (DFMG tangents 48 GB at
256^3; about 170 GB at 512^3), so it runs there:
  gpurun -- 'python tools/fullsize_fixtures.py C5 --out gpurun_out/golden'
Usage: python tools/fullsize_fixtures.py [case ...] [--out DIR]
"""
import argparse
import json
import os
import platform
import resource
import sys
import threading
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from fullsize_common import CASES, case_fbar, field_summary, grid_digests, sample_cells  # noqa: E402
from paper_2204_13624_b200.configs import CONFIGS  # noqa: E402

GREEN = {"continuous": 0, "rotated": 1, "staggered": 2}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def mem_guard(min_avail_gb=10.0):
    """exit before the host runs out of memory (the box must survive)"""
    def watch():
        while True:
            try:
                for line in open("/proc/meminfo"):
                    if line.startswith("MemAvailable:"):
                        if int(line.split()[1]) / 2**20 < min_avail_gb:
                            print("mem_guard: MemAvailable below %.0f GB, aborting" % min_avail_gb, flush=True)
                            os._exit(3)
            except OSError:
                return
            time.sleep(0.5)

    threading.Thread(target=watch, daemon=True).start()


def run_case(name, out_dir, max_ls=None):
    case = dict(CASES[name])
    if max_ls is not None:
        case["max_ls"] = max_ls
    cfg = CONFIGS[case["config"]]
    t0 = time.perf_counter()
    img = O.generate(cfg.shape, cfg.fine, (1.0, 1.0, 1.0), *cfg.params)
    t_gen = time.perf_counter() - t0
    kind, cp, cnt = O.coarsen(img, cfg.factors)
    nrm, flags, nstats = O.normals(img, cfg.factors)
    t_pre = time.perf_counter() - t0
    del img
    dig = grid_digests(kind, cp, cnt, nrm, flags)
    dims = cfg.grid
    n = int(np.prod(dims))
    cm = O.CellMaterials(dims, kind, cp, nrm, O.neo_hookean(*cfg.matrix), O.neo_hookean(*cfg.inclusion))
    ncomp = int(cm.composites) if hasattr(cm, "composites") else int((kind == 2).sum())
    cells = sample_cells(kind)
    fbar, steps = case_fbar(cfg, case)
    print(f"[{name}] grid {dims} composites {ncomp} preprocess {t_pre:.1f} s (generate {t_gen:.1f} s)", flush=True)
    t1 = time.perf_counter()
    r = cm.solve(fbar, scheme=1 if cfg.scheme == "newton_cg" else 0, green=GREEN[cfg.green],
                 eval=1 if cfg.eval == "dfmg" else 0, tol=cfg.tol, max_outer=cfg.max_outer, load_steps=steps,
                 max_ls_iterations=case["max_ls"], want_fields=True, want_p=False)
    t_solve = time.perf_counter() - t1
    rep = r["report"]
    sums, samp = field_summary(r["f"], n, cells)
    print(f"[{name}] solve {t_solve:.1f} s, {rep['ls_total']} LS iterations, success {rep['success']} "
          f"({rep.get('error', '')}), {len(rep['steps'])} steps", flush=True)
    doc = {
        "case": name, "config": cfg.name, "fine": list(cfg.fine), "grid": list(dims), "factors": list(cfg.factors),
        "fbar": np.asarray(fbar).ravel().tolist(), "load_steps": steps, "max_ls": case["max_ls"],
        "scheme": cfg.scheme, "green": cfg.green, "eval": cfg.eval, "tol": cfg.tol, "max_outer": cfg.max_outer,
        "grid_digests": dig, "composites": int((kind == 2).sum()),
        "normal_stats": [int(x) for x in nstats],
        "report": rep, "pbar": r["pbar"].ravel().tolist(), "f_sums": sums, "sample_cells": cells.tolist(),
        "cpu": {"cores": os.cpu_count(), "model": cpu_model(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS"),
                "preprocess_s": t_pre, "solve_s": t_solve,
                "boxel_iterations_per_s": n * rep["ls_total"] / t_solve if t_solve > 0 else None,
                "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20},
        "generator": "tools/fullsize_fixtures.py (CPU oracle)",
    }
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, f"full_{name}.json"), "w") as fh:
        json.dump(doc, fh)
    np.save(os.path.join(out_dir, f"full_{name}_F.npy"), samp)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=list(CASES))
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    ap.add_argument("--max-ls", type=int, default=None, help="LS budget (default: tests/fullsize_common.py)")
    a = ap.parse_args()
    os.environ.setdefault("OMP_PROC_BIND", "close")
    mem_guard()
    for name in a.cases:
        run_case(name, a.out, a.max_ls)


if __name__ == "__main__":
    main()
