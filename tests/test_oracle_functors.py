"""Pins for the oracle's edge functors and time step (O8/O9; reading Z9 in DESIGN.md)."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
import synth as S

GAMMA = 1.4


def _rest_state(n, rho, E):
    U = np.zeros((n, 5), np.float32)
    U[:, 0] = rho
    U[:, 4] = E
    return U


def test_pressure_force_at_rest():
    """A fluid at rest pushes on a face with force p*n: the momentum residual of the
    cell the normal points out of is -p n, of the other +p n; no mass/energy flux."""
    e = np.array([[0, 1]], np.int32)
    nrm = np.array([[0.25, -0.5, 0.125]], np.float32)
    U = _rest_state(2, 1.0, 2.5)
    F = O.cfd_flux(e, 2, nrm, U)
    p = (GAMMA - 1.0) * 2.5
    assert np.allclose(F[0], [0, -p * 0.25, p * 0.5, -p * 0.125, 0], atol=1e-15)
    assert np.allclose(F[1], -F[0], atol=1e-15)


def test_dissipation_direction():
    """At rest, mass and energy diffuse from the denser/hotter cell to the other."""
    e = np.array([[0, 1]], np.int32)
    nrm = np.array([[1.0, 0.0, 0.0]], np.float32)
    U = _rest_state(2, 1.0, 2.5)
    U[0, 0], U[0, 4] = 1.2, 3.0
    F = O.cfd_flux(e, 2, nrm, U)
    assert F[0, 0] < 0 and F[1, 0] > 0 and F[0, 4] < 0


def test_free_stream_and_conservation(small_mesh):
    M = small_mesh
    # uniform moving state: every closed (degree-4) cell has zero residual
    U = np.tile(np.array([[1.05, 0.03, -0.02, 0.05, 2.6]], np.float32), (M.n, 1))
    F = O.cfd_flux(M.edges, M.n, M.normals, U)
    deg = np.bincount(M.edges.ravel(), minlength=M.n)
    scale = np.abs(M.normals).max() * 4.0
    assert np.abs(F[deg == 4]).max() < 1e-6 * scale
    assert np.abs(F[deg < 4]).max() > 1e-3 * scale          # open cells do see a residual
    # random state: global conservation, sum_v F_v = 0
    U = S.cfd_state(M.n)
    F = O.cfd_flux(M.edges, M.n, M.normals, U)
    assert np.all(np.abs(F.sum(axis=0)) <= 1e-12 * np.abs(F).sum(axis=0))


def test_antisymmetry_and_relabel(small_mesh):
    M = small_mesh
    U = S.cfd_state(M.n, seed=7)
    F = O.cfd_flux(M.edges, M.n, M.normals, U)
    F2 = O.cfd_flux(M.edges[:, ::-1].copy(), M.n, -M.normals, U)
    assert np.allclose(F, F2, rtol=0, atol=1e-15)
    rng = np.random.default_rng(1)
    vp = rng.permutation(M.n)
    ep = rng.permutation(M.m)
    F3 = O.cfd_flux(vp[M.edges[ep]].astype(np.int32), M.n, M.normals[ep], U[np.argsort(vp)])
    assert np.allclose(F3[vp], F, rtol=0, atol=1e-14)


def test_step_updates_touched_only():
    e = np.array([[0, 1], [1, 2]], np.int32)
    nrm = np.array([[1, 0, 0], [0, 1, 0]], np.float32)
    U = S.cfd_state(4)
    dt = np.full(4, 0.5, np.float32)
    Uo, F = O.cfd_step(e, 4, nrm, U, dt)
    assert np.array_equal(Uo[3], U[3].astype(np.float64))
    assert np.allclose(Uo[:3], U[:3] + 0.5 * F[:3], rtol=0, atol=1e-15)


def test_gather_scatter():
    n, e = S.random_multigraph(11, 500, 120)
    deg = np.bincount(e.ravel(), minlength=n)
    assert np.array_equal(O.gather_scatter(e, n, np.ones(n, np.float32)), deg.astype(np.float64))
    x = S.int_vector(12, n, 0, 7)
    A = sp.coo_matrix((np.ones(500), (e[:, 0], e[:, 1])), shape=(n, n)).tocsr()
    assert np.array_equal(O.gather_scatter(e, n, x), (A + A.T) @ x.astype(np.float64))


def test_spmv_stencil():
    """SpMV on the bipartite data-affinity graph of a 2D 5-point Laplacian."""
    g = 13
    rows, cols, vals = [], [], []
    for i in range(g):
        for j in range(g):
            r = i * g + j
            for di, dj, a in ((0, 0, 4.0), (-1, 0, -1.0), (1, 0, -1.0), (0, -1, -1.0), (0, 1, -1.0)):
                if 0 <= i + di < g and 0 <= j + dj < g:
                    rows.append(r); cols.append((i + di) * g + j + dj); vals.append(a)
    N = g * g
    edges = np.stack([np.array(cols), N + np.array(rows)], axis=1).astype(np.int32)
    w = np.array(vals, np.float32)
    x = np.concatenate([S.int_vector(3, N, -8, 8), np.zeros(N, np.float32)])
    y = O.spmv(edges, 2 * N, w, x)
    A = sp.coo_matrix((vals, (rows, cols)), shape=(N, N)).tocsr()
    assert np.array_equal(y[N:], A @ x[:N].astype(np.float64))
    assert np.all(y[:N] == 0)


def test_wrappers_keep_converted_inputs_alive():
    """Regression: inputs converted to float32 by the ctypes wrappers must outlive the C
    call (a temporary's buffer was freed before it, and reads returned garbage once the
    allocator reused it). float64 inputs must give the float32 results exactly."""
    import synth as S
    n, e = S.random_multigraph(3, 4000, 700)
    x64 = S.int_vector(4, n, 0, 7).astype(np.float64)
    ref = O.gather_scatter(e, n, x64.astype(np.float32))
    for i in range(30):
        junk = [np.full(n + 7 * i, 1e30, np.float32) for _ in range(4)]   # churn the allocator
        assert np.array_equal(O.gather_scatter(e, n, x64), ref)
        assert np.array_equal(O.spmv(e, n, np.ones(len(e)), x64), O.spmv(e, n, np.ones(len(e), np.float32),
                                                                          x64.astype(np.float32)))
        del junk
