"""Multi-process host logic of the slab decomposition on CPU:
world_size 2 over gloo. Each rank holds its slab of a seeded 9-component
field, transforms z and y with numpy, scatters the rows into the slab-side
buffer at the offsets the library computes (combo_slab_row -- the same
SpecView arithmetic the kernels use), runs the all-to-all of equal blocks,
reads the pencil side back through the library's offsets and finishes the x
transform; the result must equal numpy's rfftn of the whole field, and the
inverse path must return the slab. Rank-ordered chunk partials
(combo_chunk_range) must reproduce the single-process sum bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

DIMS = (8, 6, 10)
WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _offsets(side, rank, ni_or_n1, nj_or_n2):
    from paper_2204_13624_b200 import slab_row

    off = np.zeros((9, ni_or_n1, nj_or_n2), np.int64)
    for c in range(9):
        for i in range(ni_or_n1):
            for j in range(nj_or_n2):
                off[c, i, j] = slab_row(DIMS, WORLD, rank, side, c, i, j)
    return off


def _chunk_partials(field_sq, nplanes):
    from paper_2204_13624_b200 import chunk_range

    _, _, nb = chunk_range(DIMS, nplanes, 0)
    out = []
    for b in range(nb):
        beg, end, _ = chunk_range(DIMS, nplanes, b)
        s = 0.0
        for v in field_sq[beg:end]:
            s += v
        out.append(s)
    return out


def _worker(rank, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        n1, n2, n3 = DIMS
        ni, nj = n1 // WORLD, n2 // WORLD
        n3c = n3 // 2 + 1
        n3p = (n3c + 7) // 8 * 8
        blk = 9 * ni * nj * n3p
        rng = np.random.default_rng(3)
        x = rng.standard_normal((9,) + DIMS)
        i0, j0 = rank * ni, rank * nj
        slab = x[:, i0:i0 + ni]
        # slab side: z r2c + y c2c, rows scattered to the blocked layout
        Y = np.fft.fft(np.fft.rfft(slab, axis=3), axis=2)
        A = np.zeros(WORLD * blk, np.complex128)
        offA = _offsets(0, rank, ni, n2)
        for c in range(9):
            for il in range(ni):
                for j in range(n2):
                    A[offA[c, il, j]:offA[c, il, j] + n3c] = Y[c, il, j]
        B = np.zeros_like(A)
        tb = torch.from_numpy(B.view(np.float64))
        dist.all_to_all_single(tb, torch.from_numpy(A.view(np.float64)))
        offB = _offsets(1, rank, n1, nj)
        Z = np.zeros((9, n1, nj, n3c), np.complex128)
        for c in range(9):
            for i in range(n1):
                for jl in range(nj):
                    Z[c, i, jl] = B[offB[c, i, jl]:offB[c, i, jl] + n3c]
        X = np.fft.fft(Z, axis=1)
        ref = np.fft.rfftn(x, axes=(1, 2, 3))[:, :, j0:j0 + nj]
        fwd_err = float(np.abs(X - ref).max() / np.abs(ref).max())
        # inverse: x back on the pencils, transpose back, y and z on the slab
        Zi = np.fft.ifft(X, axis=1)
        B2 = np.zeros_like(B)
        for c in range(9):
            for i in range(n1):
                for jl in range(nj):
                    B2[offB[c, i, jl]:offB[c, i, jl] + n3c] = Zi[c, i, jl]
        A2 = np.zeros_like(A)
        dist.all_to_all_single(torch.from_numpy(A2.view(np.float64)), torch.from_numpy(B2.view(np.float64)))
        Yi = np.zeros((9, ni, n2, n3c), np.complex128)
        for c in range(9):
            for il in range(ni):
                for j in range(n2):
                    Yi[c, il, j] = A2[offA[c, il, j]:offA[c, il, j] + n3c]
        back = np.fft.irfft(np.fft.ifft(Yi, axis=2), n=n3, axis=3)
        inv_err = float(np.abs(back - slab).max())
        # rank-ordered chunk partials of sum(x^2) over the slab cells
        parts = _chunk_partials((slab[0] ** 2).reshape(-1), ni)
        allp = [None] * WORLD
        dist.all_gather_object(allp, parts)
        total = 0.0
        for p in (v for r in allp for v in r):
            total += p
        single = 0.0
        for p in _chunk_partials((x[0] ** 2).reshape(-1), n1):
            single += p
        q.put((rank, fwd_err, inv_err, total, single))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e), None, None, None))


def test_slab_pencil_transpose_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for rank, fwd, inv, total, single in res:
        assert not isinstance(fwd, str), fwd
        assert fwd <= 1e-13 and inv <= 1e-13
        assert total == single  # bitwise: chunk partials combined in global order


def test_layout_single_rank_is_j_major():
    # one slab: rows j-major (x lines contiguous, the x + Gamma pass's order)
    from paper_2204_13624_b200 import slab_row

    n3p = (DIMS[2] // 2 + 1 + 7) // 8 * 8
    for c, i, j in [(0, 0, 0), (3, 5, 2), (8, 7, 5)]:
        want = ((c * DIMS[1] + j) * DIMS[0] + i) * n3p
        assert slab_row(DIMS, 1, 0, 0, c, i, j) == want == slab_row(DIMS, 1, 0, 1, c, i, j)


def test_layout_blocks_are_j_major():
    # R slabs: block s of rank q's slab side is block q of rank s's pencil
    # side, rows j-major inside a block
    from paper_2204_13624_b200 import slab_row

    R = 2
    n3p = (DIMS[2] // 2 + 1 + 7) // 8 * 8
    ni, nj = DIMS[0] // R, DIMS[1] // R
    blk = 9 * ni * nj * n3p
    for q in range(R):
        for s in range(R):
            for c, il, jl in [(0, 0, 0), (2, 1, 1), (8, ni - 1, nj - 1)]:
                a = slab_row(DIMS, R, q, 0, c, il, s * nj + jl)
                b = slab_row(DIMS, R, s, 1, c, q * ni + il, jl)
                assert a - s * blk == b - q * blk == c * ni * nj * n3p + (jl * ni + il) * n3p


def test_chunks_never_straddle_planes():
    from paper_2204_13624_b200 import chunk_range

    plane = DIMS[1] * DIMS[2]
    _, _, nb = chunk_range(DIMS, DIMS[0], 0)
    covered = 0
    for b in range(nb):
        beg, end, _ = chunk_range(DIMS, DIMS[0], b)
        assert beg // plane == (end - 1) // plane
        assert beg == covered
        covered = end
    assert covered == int(np.prod(DIMS))
