"""Checks of the synthetic input generators (inputs only; no method arithmetic)."""
import numpy as np
import pytest

import synth as S
from synth.mesh import _faces, PERMS


def test_splitmix64_vector():
    # SplitMix64 seeded with 0: first output 0xE220A8397B1DCDAF (Steele et al. reference)
    assert int(S.splitmix64(0, np.array([0]))[0]) == 0xE220A8397B1DCDAF
    u = S.uniform01(5, np.arange(10000))
    assert 0 <= u.min() and u.max() < 1 and abs(u.mean() - 0.5) < 0.02
    p = S.random_permutation(9, 1000)
    assert sorted(p.tolist()) == list(range(1000))


def _faces_bruteforce(N):
    """Interior faces by matching sorted vertex triples of every tet (generic method)."""
    ncell = 6 * N ** 3
    cell = np.arange(ncell)
    q, c = cell % 6, cell // 6
    corner = np.stack([c % N, (c // N) % N, c // (N * N)], axis=1)
    eye = np.eye(3, dtype=np.int64)
    pi = PERMS[q]
    v = [corner]
    for j in range(3):
        v.append(v[-1] + eye[pi[:, j]])
    gid = [(x[:, 2] * (N + 1) + x[:, 1]) * (N + 1) + x[:, 0] for x in v]
    faces = {}
    pairs = set()
    for t in range(ncell):
        for skip in range(4):
            key = tuple(sorted(gid[i][t] for i in range(4) if i != skip))
            if key in faces:
                pairs.add((min(faces[key], t), max(faces[key], t)))
            else:
                faces[key] = t
    return pairs


def test_analytic_adjacency_matches_face_matching():
    for N in (1, 2, 3):
        a, b, _ = _faces(N)
        assert set(zip(np.minimum(a, b).tolist(), np.maximum(a, b).tolist())) == _faces_bruteforce(N)
        assert len(a) == len(set(zip(a.tolist(), b.tolist())))


def test_mesh_geometry():
    M = S.kuhn_mesh(nbox=4, relabel=True, seed=3)
    assert M.n == 6 * 64
    assert np.all(M.edges[:, 0] < M.edges[:, 1])
    assert np.all(np.diff(M.edges[:, 0].astype(np.int64) * M.n + M.edges[:, 1]) > 0)
    # closed tets: outward area-normals sum to zero
    acc = np.zeros((M.n, 3))
    np.add.at(acc, M.edges[:, 0], M.normals)
    np.add.at(acc, M.edges[:, 1], -M.normals)
    deg = np.bincount(M.edges.ravel(), minlength=M.n)
    assert np.abs(acc[deg == 4]).max() < 1e-7
    # Kuhn faces are right triangles with legs (h, h) or (h, h*sqrt2): areas h^2/2, h^2/sqrt2
    area = np.linalg.norm(M.normals.astype(np.float64), axis=1) / M.h ** 2
    assert np.all(np.isclose(area, 0.5, rtol=1e-6) | np.isclose(area, 0.5 * np.sqrt(2), rtol=1e-6))


def test_config_sizes():
    M1 = S.config_mesh("c1")
    assert (M1.n, M1.m) == (97_046, 190_245)
    M2 = S.config_mesh("c2")
    assert (M2.n, M2.m) == (232_536, 458_168)
    assert np.bincount(M2.edges.ravel()).max() <= 4
    U = S.cfd_state(M2.n)
    p = 0.4 * (U[:, 4] - 0.5 * (U[:, 1:4] ** 2).sum(1) / U[:, 0])
    assert p.min() > 0.8


@pytest.mark.parametrize("g", [1, 2, 3, 7, 40])
def test_stencil_spmv_brute_force(g):
    """The SpMV input (C5): the 2D 5-point Laplacian on a g x g grid as a bipartite COO graph in
    row-major order -- compared with a dense construction, for every chunk size."""
    N = g * g
    A = np.zeros((N, N), np.float32)
    for i in range(N):
        r, c = divmod(i, g)
        A[i, i] = 4.0
        for dr, dc in ((-1, 0), (0, -1), (0, 1), (1, 0)):
            if 0 <= r + dr < g and 0 <= c + dc < g:
                A[i, (r + dr) * g + (c + dc)] = -1.0
    rows, cols = np.nonzero(A)                       # row-major, columns ascending
    for chunk in (1, 5, 1 << 22):
        n, e, w = S.stencil2d_spmv(g, chunk_rows=chunk)
        assert n == 2 * N
        assert np.array_equal(e[:, 0], cols) and np.array_equal(e[:, 1], N + rows)
        assert np.array_equal(w, A[rows, cols])
    if g == 40:
        assert len(e) == 5 * N - 4 * g             # 499,960,000 at g = 10,000
