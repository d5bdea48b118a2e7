"""Synthetic cfd-shaped tetrahedral meshes (SURVEY.md §8(d) "Concrete synthetic inputs").

The paper's cfd inputs (Rodinia fvcorr.domn.097K / missile.domn.0.2M)
are unstructured tetrahedral meshes whose cells interact across faces ("at most 4
neighbour particles"). We synthesise meshes of the same shape:

* a Kuhn (Freudenthal) triangulation of an N^3 box: every unit cube is split into
  6 tetrahedra, one per permutation pi of the axes, with vertices
  v0 = corner, v1 = v0 + e_pi0, v2 = v1 + e_pi1, v3 = v2 + e_pi2;
* cells are numbered ((z*N + y)*N + x)*6 + q (q = index of pi) and the first
  `n_keep` cells are kept ("truncation to exact cell counts");
* a seeded random relabel of the kept cells (Rodinia-like poor locality);
* the data-affinity graph D (Def. 1) has one vertex per cell and one
  edge per interior face, listed sorted by (min id, max id) -- the default task order;
  each edge carries the face's area-normal oriented from its first to its second cell.

This module draws inputs only; it contains none of the method's arithmetic.
Face adjacency is analytic (see `_faces`) and is cross-checked against a brute-force
face-matching construction in tests/test_synth.py.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .splitmix import random_permutation, uniform

PERMS = np.array([(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)], dtype=np.int64)
_PIDX = {tuple(p): i for i, p in enumerate(PERMS.tolist())}
SW01 = np.array([_PIDX[(p[1], p[0], p[2])] for p in PERMS.tolist()])  # face opposite v1
SW12 = np.array([_PIDX[(p[0], p[2], p[1])] for p in PERMS.tolist()])  # face opposite v2
ROT = np.array([_PIDX[(p[1], p[2], p[0])] for p in PERMS.tolist()])   # face opposite v0 (next cube)

# Named configurations.
CONFIGS = {
    "c1": dict(nbox=26, n_keep=97_046),      # fvcorr.domn.097K-shaped
    "c2": dict(nbox=34, n_keep=232_536),     # missile.domn.0.2M-shaped
    "c3": dict(nbox=221, n_keep=64_000_000),  # 64M cells, working set >> L2
}


@dataclass
class Mesh:
    n: int                 # vertices of D (cells)
    m: int                 # edges of D (interior faces)
    edges: np.ndarray      # int32 [m][2], a < b, sorted lexicographically
    normals: np.ndarray    # float32 [m][3], area-normal oriented edges[e,0] -> edges[e,1]
    volume: np.ndarray     # float64 [n]
    h: float               # cube edge length
    seed: int


def _tet_vertices(cell: np.ndarray, N: int, h: float):
    """Vertex coordinates v0..v3 (each [len(cell), 3], float64) of Kuhn tets `cell`."""
    q = cell % 6
    c = cell // 6
    corner = np.stack([c % N, (c // N) % N, c // (N * N)], axis=1).astype(np.float64)
    pi = PERMS[q]
    eye = np.eye(3)
    v0 = corner * h
    v1 = v0 + h * eye[pi[:, 0]]
    v2 = v1 + h * eye[pi[:, 1]]
    v3 = v2 + h * eye[pi[:, 2]]
    return v0, v1, v2, v3


def _faces(N: int, c0: int = 0, c1: int | None = None):
    """Interior faces of the N^3 Kuhn box with first cell in [c0, c1), as (cell_a, cell_b, kind).

    kind 1: face opposite v1 of a (shared with the tet of the same cube, pi0<->pi1);
    kind 2: face opposite v2 of a (same cube, pi1<->pi2);
    kind 0: face opposite v0 of a (tet (pi1,pi2,pi0) of the cube at corner + e_pi0).
    Intra-cube pairs are emitted once (q < q'); cross-cube faces once, from the v0 side.
    """
    ncell = 6 * N ** 3
    c1 = ncell if c1 is None else c1
    cell = np.arange(c0, c1, dtype=np.int64)
    q = cell % 6
    base = cell - q
    out_a, out_b, out_k = [], [], []
    for kind, tab in ((1, SW01), (2, SW12)):
        q2 = tab[q]
        sel = q < q2
        out_a.append(cell[sel]); out_b.append((base + q2)[sel]); out_k.append(np.full(int(sel.sum()), kind, np.int8))
    c = cell // 6
    ax = PERMS[q, 0]
    stride = np.array([1, N, N * N], dtype=np.int64)
    coord_ax = (c // stride[ax]) % N
    ok = coord_ax < N - 1
    nb = (c + stride[ax]) * 6 + ROT[q]
    out_a.append(cell[ok]); out_b.append(nb[ok]); out_k.append(np.zeros(int(ok.sum()), np.int8))
    return np.concatenate(out_a), np.concatenate(out_b), np.concatenate(out_k)


def _normals(a, kind, N, h):
    """Area-normal of the face `kind` of cells a, oriented out of a (float64 [len, 3])."""
    v0, v1, v2, v3 = _tet_vertices(a, N, h)
    k0 = (kind == 0)[:, None]
    k1 = (kind == 1)[:, None]
    f0 = np.where(k0, v1, v0)
    f1 = np.where(k0, v2, np.where(k1, v2, v1))
    opp = np.where(k0, v0, np.where(k1, v1, v2))
    nrm = 0.5 * np.cross(f1 - f0, v3 - f0)
    flip = np.einsum("ij,ij->i", nrm, f0 - opp) < 0
    nrm[flip] *= -1.0
    return nrm


def _normal_table(N, h):
    """Area-normals of the three face kinds of the six Kuhn tets, out of the tet (float64
    [18, 3], row 3q + kind). Every tet of permutation q is a translate of tet q of the
    cube at the origin, so its faces have these normals (computed once, from the exact
    corner at the origin, instead of per cell from rounded absolute coordinates)."""
    q = np.repeat(np.arange(6, dtype=np.int64), 3)
    kind = np.tile(np.array([0, 1, 2], dtype=np.int8), 6)
    return _normals(q, kind, N, h)


def _argsort_unique(keys: np.ndarray) -> np.ndarray:
    """argsort of distinct int64 keys (any correct sort gives the same order): on the GPU
    when one is present (the 64M-cell C3 mesh), else numpy."""
    try:
        import torch
        if torch.cuda.is_available() and keys.size > (1 << 22):
            return torch.sort(torch.from_numpy(keys).cuda(), stable=True)[1].cpu().numpy()
    except ImportError:
        pass
    return np.argsort(keys, kind="stable")


def kuhn_mesh(nbox: int, n_keep: int | None = None, seed: int = 1605, relabel: bool = True,
              chunk: int = 1 << 23) -> Mesh:
    N = int(nbox)
    ncell = 6 * N ** 3
    n = ncell if n_keep is None else int(n_keep)
    if not (1 <= n <= ncell):
        raise ValueError(f"n_keep must be in [1, {ncell}]")
    h = 1.0 / N
    if relabel:
        order = random_permutation(seed, n)          # order[j] = old id of new id j
        new = np.empty(n, dtype=np.int64)
        new[order] = np.arange(n, dtype=np.int64)
        del order
    table = _normal_table(N, h)
    los, his, nrms = [], [], []
    # faces are emitted from their first cell, which is < n when both cells are kept
    for c0 in range(0, n, chunk):
        a, b, kind = _faces(N, c0, min(n, c0 + chunk))
        keep = b < n
        a, b, kind = a[keep], b[keep], kind[keep]
        nrm = table[(a % 6) * 3 + kind]
        if relabel:
            a, b = new[a], new[b]
        swap = a > b
        nrm[swap] *= -1.0
        los.append(np.where(swap, b, a).astype(np.int32))
        his.append(np.where(swap, a, b).astype(np.int32))
        nrms.append(nrm.astype(np.float32))
        del a, b, kind, nrm, swap
    lo = np.concatenate(los); del los
    hi = np.concatenate(his); del his
    nrm = np.concatenate(nrms); del nrms
    idx = _argsort_unique(lo.astype(np.int64) * n + hi)
    edges = np.empty((lo.size, 2), dtype=np.int32)
    edges[:, 0] = lo[idx]
    edges[:, 1] = hi[idx]
    del lo, hi
    normals = nrm[idx]
    del nrm, idx
    volume = np.full(n, h ** 3 / 6.0)
    return Mesh(n=n, m=int(edges.shape[0]), edges=edges, normals=normals, volume=volume, h=h, seed=seed)


def config_mesh(name: str, seed: int = 1605) -> Mesh:
    return kuhn_mesh(seed=seed, **CONFIGS[name])


def cfd_state(n: int, seed: int = 1606) -> np.ndarray:
    """Initial conserved state U_v = (rho, m_x, m_y, m_z, E), float32 [n][5] (AoS rows).

    rho in U[0.9, 1.1], velocity u in U[-0.1, 0.1]^3 (m = rho*u), E in U[2.25, 2.75]
    (keeps pressure (gamma-1)(E - rho|u|^2/2) > 0.89 for gamma = 1.4)."""
    ctr = np.arange(n, dtype=np.uint64) * np.uint64(5)
    rho = uniform(seed, ctr, 0.9, 1.1)
    u = np.stack([uniform(seed, ctr + np.uint64(1 + j), -0.1, 0.1) for j in range(3)], axis=1)
    E = uniform(seed, ctr + np.uint64(4), 2.25, 2.75)
    U = np.empty((n, 5), dtype=np.float64)
    U[:, 0] = rho
    U[:, 1:4] = rho[:, None] * u
    U[:, 4] = E
    return U.astype(np.float32)


def cfd_dt(volume: np.ndarray, cfl: float = 0.1) -> np.ndarray:
    """Per-vertex update coefficient dt_v = cfl * vol^(1/3) / vol (local time step over
    cell volume), float32 [n]. Makes dt*|F|/|U| ~ 1e-2, so one step is not vacuous."""
    return (cfl * np.cbrt(volume) / volume).astype(np.float32)
