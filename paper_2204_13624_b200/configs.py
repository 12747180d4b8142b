"""The five BASELINE.json configurations as concrete seeded inputs.

SURVEY.md §8(d) restatement (no public dataset is involved; every image is a
seeded synthetic microstructure):
  C1  centred sphere, phi 0.2, 128^3 -> 32^3 (4,4,4), NH (1,2)/(10,20),
      Fbar = I + 0.1 e1(x)e1 in 10 steps, basic scheme, tol 1e-6
  C2  RSA spheres r in [6,10] vox, phi 0.3, 512^3 -> 128^3, contrast 100,
      Fbar = I + 0.2 e1(x)e2 in 20 steps, Newton-CG, tol 1e-8
  C3  RSA z-fibres r = 8 vox, phi 0.35, 512^3 -> 256x256x64 (2,2,8),
      fibre (50,50) / matrix (1,4), Fbar = I + 0.15 e3(x)e3 in 15 steps
  C4  Boolean ellipsoids a in [4,12] vox, phi 0.25, 512^3 -> 256^3 (2,2,2),
      contrast 1000, DFMG + staggered, 10 steps
  C5  RSA spheres r in [8,24] vox, phi 0.3, 4096^3 -> 1024^3 (8 GPUs);
      1 GPU: 2048^3 -> 512^3; contrast 100, Fbar = I + 0.1 e1(x)e1, 5 steps
Materials are (mu, lambda); "contrast c" = inclusion (c mu_m, c lambda_m)
with matrix (1, 2). Green operator: the reference default `rotated`
(solver.hpp:20) unless DFMG requires `staggered` (solver.cpp:277-280).
Normals: second moment, weighted centroid, >= 3 support voxels
(normals.hpp:33-37). `scale` divides the fine image (and hence the grid)
for the small parity cases; voxel-unit radii are scaled along.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np


@dataclass
class Config:
    name: str
    fine: tuple
    factors: tuple
    shape: str
    params: tuple  # generator parameters (seed first for seeded shapes)
    matrix: tuple  # (lambda, mu)
    inclusion: tuple
    fbar: np.ndarray
    load_steps: int
    scheme: str
    green: str
    eval: str
    tol: float
    max_outer: int = 200
    voxel_params: tuple = field(default_factory=tuple)  # indices of params in voxel units
    lengths: tuple = (1.0, 1.0, 1.0)

    @property
    def grid(self):
        return tuple(f // k for f, k in zip(self.fine, self.factors))


def _fb(entries):
    f = np.eye(3)
    for (i, j), v in entries.items():
        f[i, j] += v
    return f


R_C1 = (0.15 / math.pi) ** (1.0 / 3.0)  # sphere of volume fraction 0.2

CONFIGS = {
    "C1": Config("C1", (128, 128, 128), (4, 4, 4), "sphere", (R_C1,), (2.0, 1.0), (20.0, 10.0),
                 _fb({(0, 0): 0.1}), 10, "basic", "rotated", "per_cell", 1e-6, max_outer=5000),
    "C2": Config("C2", (512, 512, 512), (4, 4, 4), "rsa_spheres", (1, 6.0, 10.0, 0.30), (2.0, 1.0),
                 (200.0, 100.0), _fb({(0, 1): 0.2}), 20, "newton_cg", "rotated", "per_cell", 1e-8,
                 voxel_params=(1, 2)),
    "C3": Config("C3", (512, 512, 512), (2, 2, 8), "rsa_fibers_z", (1, 8.0, 0.35), (4.0, 1.0), (50.0, 50.0),
                 _fb({(2, 2): 0.15}), 15, "newton_cg", "rotated", "per_cell", 1e-8, voxel_params=(1,)),
    "C4": Config("C4", (512, 512, 512), (2, 2, 2), "boolean_ellipsoids", (1, 4.0, 12.0, 0.25), (2.0, 1.0),
                 (2000.0, 1000.0), _fb({(0, 0): 0.1, (1, 1): -0.05, (2, 2): -0.05}), 10, "newton_cg",
                 "staggered", "dfmg", 1e-8, voxel_params=(1, 2)),
    "C5": Config("C5", (2048, 2048, 2048), (4, 4, 4), "rsa_spheres", (1, 8.0, 24.0, 0.30), (2.0, 1.0),
                 (200.0, 100.0), _fb({(0, 0): 0.1}), 5, "newton_cg", "rotated", "per_cell", 1e-8,
                 voxel_params=(1, 2)),
}


def scaled(cfg: Config, scale: int) -> Config:
    """cfg with the fine image divided by `scale` (voxel radii scaled along)."""
    if scale == 1:
        return cfg
    p = list(cfg.params)
    for i in cfg.voxel_params:
        p[i] = p[i] / scale
    fine = tuple(max(f // scale, k) for f, k in zip(cfg.fine, cfg.factors))
    return Config(cfg.name + f"/{scale}", fine, cfg.factors, cfg.shape, tuple(p), cfg.matrix, cfg.inclusion,
                  cfg.fbar, cfg.load_steps, cfg.scheme, cfg.green, cfg.eval, cfg.tol, cfg.max_outer,
                  cfg.voxel_params, cfg.lengths)


# C5 weak-scaling ladder: P GPUs carry P x 512^3 boxels --
# 512^3, 1024 x 512^2, 1024^2 x 512, 1024^3 (the 4096^3 -> 1024^3 scaling
# config) -- with lengths proportional to the dims, so the voxel size, the
# voxel-unit radii and the cubic boxels are those of the 1-GPU 512^3 case.
LADDER = {1: (512, 512, 512), 2: (1024, 512, 512), 4: (1024, 1024, 512), 8: (1024, 1024, 1024)}


def c5_ladder(P: int) -> Config:
    if P not in LADDER:
        raise ValueError(f"C5 ladder: no rung for {P} GPUs (1, 2, 4, 8)")
    g = LADDER[P]
    base = CONFIGS["C5"]
    fine = tuple(4 * n for n in g)
    lengths = tuple(n / 512.0 for n in g)
    name = "C5" if P == 1 else f"C5x{P}"
    return replace(base, name=name, fine=fine, lengths=lengths)


def build_slab_grid(ctx, cfg: Config, nranks: int = 1, rank: int = 0):
    """Device preprocessing of rank `rank`'s slab of boxel planes: the fine
    planes of the slab plus one halo plane each side are generated
    (combo_generate_planes), coarsened and given normals
    (combo_normals_slab); nothing outside the window is built. Returns
    (kind, c_plus, normals, normal stats) of the slab as CUDA tensors."""
    import torch

    f1, f2, f3 = cfg.fine
    a1 = cfg.factors[0]
    b1 = f1 // a1
    if b1 % nranks:
        raise ValueError("slab decomposition: the rank count must divide the boxel planes")
    nbp = b1 // nranks
    bp0 = rank * nbp
    plane = f2 * f3
    if nranks == 1:
        img = torch.empty(f1 * plane, dtype=torch.uint8, device="cuda")
        ctx.generate(cfg.shape, cfg.fine, cfg.lengths, *cfg.params, out=img)
        kind, cp, cnt = ctx.coarsen(img, cfg.factors, dims=cfg.fine)
        nrm, flags, st = ctx.compute_normals(img, cfg.factors, kind, lengths=cfg.lengths, dims=cfg.fine)
    else:
        f0, nf = bp0 * a1, nbp * a1
        img = torch.empty((nf + 2) * plane, dtype=torch.uint8, device="cuda")
        ctx.generate(cfg.shape, cfg.fine, cfg.lengths, *cfg.params, out=img, planes=(f0 - 1, nf + 2))
        kind, cp, cnt = ctx.coarsen(img[plane:(nf + 1) * plane], cfg.factors, dims=(nf, f2, f3))
        nrm, flags, st = ctx.compute_normals_slab(img, f0 - 1, cfg.fine, cfg.factors, bp0, nbp, kind,
                                                  lengths=cfg.lengths)
    ctx.synchronize()
    del img, cnt, flags
    torch.cuda.empty_cache()
    return kind, cp, nrm, st


def build_grid(ctx, cfg: Config):
    """image -> (kind, c_plus, count, normals, flags, image) on the GPU."""
    img = ctx.generate(cfg.shape, cfg.fine, (1.0, 1.0, 1.0), *cfg.params)
    kind, cp, cnt = ctx.coarsen(img, cfg.factors)
    nrm, flags, _ = ctx.compute_normals(img, cfg.factors, kind)
    return dict(image=img, kind=kind, c_plus=cp, count=cnt, normals=nrm, flags=flags)
