"""Pins the oracle's DFMG against a brute-force transliteration of the printed
doubly-fine assembly tables -- the reference's own DfmgTablesOracle
(/root/reference/proj/tests/test_kernels.cpp:160-309), same geometries, same
seeded field (oracle::Rng = splitmix64, tests/oracles.hpp:23-43)."""
import numpy as np
import pytest

M64 = (1 << 64) - 1


class Rng:  # tests/oracles.hpp:23-43
    def __init__(self, seed):
        self.s = seed

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def unit(self):
        return (self.next() >> 11) * 2.0 ** -53

    def sym(self):
        return 2.0 * self.unit() - 1.0


@pytest.mark.parametrize("dims", [(4, 4, 4), (4, 2, 6)])
def test_dfmg_matches_table_transliteration(oracle, dims):
    lengths = (1.0, 0.9, 1.2)
    img = oracle.generate("fiber_pack", dims, lengths, 23, 4, 0.25, 0.8, 0.4)
    kind, cp, _ = oracle.coarsen(img, (1, 1, 1), lengths)
    soft, stiff = oracle.neo_hookean_enu(1.0, 0.0), oracle.neo_hookean_enu(10.0, 0.3)
    n = int(np.prod(dims))
    cm = oracle.CellMaterials(dims, kind, cp, np.zeros((n, 3)), soft, stiff, lengths=lengths)
    rng = Rng(97)
    fbar = np.eye(3)
    fbar[0, 1] = 0.2
    F = np.repeat(fbar.reshape(9, 1), n, axis=1)
    flat = F.reshape(-1)
    for i in range(flat.size):  # `for (auto& v : f.data) v += 0.05 * rng.sym()`
        flat[i] += 0.05 * rng.sym()
    P, _ = cm.dfmg_stress(F.ravel())
    P = P.reshape(9, n)
    n1, n2, n3 = dims

    def comp(c, i, j, k):
        return F[c, ((i % n1) * n2 + (j % n2)) * n3 + (k % n3)]

    def law(i, j, k, fd):
        cell = ((i % n1) * n2 + (j % n2)) * n3 + (k % n3)
        ok, p, _ = oracle.law_eval(stiff if kind[cell] == 1 else soft, fd)
        assert ok
        return p

    worst = scale = 0.0
    for i in range(n1):
        for j in range(n2):
            for k in range(n3):
                out = np.zeros((3, 3))
                for l1 in range(2):
                    for l2 in range(2):
                        for l3 in range(2):
                            fd = np.array([[comp(0, i, j, k), comp(1, i + l1, j + l2, k), comp(2, i + l1, j, k + l3)],
                                           [comp(3, i + l1, j + l2, k), comp(4, i, j, k), comp(5, i, j + l2, k + l3)],
                                           [comp(6, i + l1, j, k + l3), comp(7, i, j + l2, k + l3), comp(8, i, j, k)]])
                            p = law(i, j, k, fd)
                            out[0, 0] += p[0, 0]
                            out[1, 1] += p[1, 1]
                            out[2, 2] += p[2, 2]
                            fd = np.array([[comp(0, i - l1, j - l2, k), comp(1, i, j, k), comp(2, i, j - l2, k + l3)],
                                           [comp(3, i, j, k), comp(4, i - l1, j - l2, k), comp(5, i - l1, j, k + l3)],
                                           [comp(6, i, j - l2, k + l3), comp(7, i - l1, j, k + l3),
                                            comp(8, i - l1, j - l2, k)]])
                            p = law(i - l1, j - l2, k, fd)
                            out[0, 1] += p[0, 1]
                            out[1, 0] += p[1, 0]
                            fd = np.array([[comp(0, i - l1, j, k - l3), comp(1, i, j + l2, k - l3), comp(2, i, j, k)],
                                           [comp(3, i, j + l2, k - l3), comp(4, i - l1, j, k - l3),
                                            comp(5, i - l1, j + l2, k)],
                                           [comp(6, i, j, k), comp(7, i - l1, j + l2, k), comp(8, i - l1, j, k - l3)]])
                            p = law(i - l1, j, k - l3, fd)
                            out[0, 2] += p[0, 2]
                            out[2, 0] += p[2, 0]
                            fd = np.array([[comp(0, i, j - l2, k - l3), comp(1, i + l1, j, k - l3),
                                            comp(2, i + l1, j - l2, k)],
                                           [comp(3, i + l1, j, k - l3), comp(4, i, j - l2, k - l3), comp(5, i, j, k)],
                                           [comp(6, i + l1, j - l2, k), comp(7, i, j, k), comp(8, i, j - l2, k - l3)]])
                            p = law(i, j - l2, k - l3, fd)
                            out[1, 2] += p[1, 2]
                            out[2, 1] += p[2, 1]
                ref = out / 8.0
                got = P[:, (i * n2 + j) * n3 + k].reshape(3, 3)
                worst = max(worst, np.linalg.norm(ref - got))
                scale = max(scale, np.linalg.norm(ref))
    assert worst <= 1e-13 * scale
