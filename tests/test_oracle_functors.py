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


def _one_face(Ua, Ub, n):
    e = np.array([[0, 1]], np.int32)
    U = np.array([Ua, Ub], np.float32)
    return O.cfd_flux(e, 2, np.array([n], np.float32), U)


def test_uniform_flow_along_normal_is_textbook_euler_flux():
    """A uniform state (U_a = U_b, so the dissipation f (U_a - U_b) vanishes) moving along
    the face normal: Phi = -n.(G(U) + G(U))/2 = -n.G(U), the textbook Euler flux.
    rho = 1, u = (0.3, 0, 0), p = 1, gamma = 1.4:
      E = p/(gamma-1) + rho|u|^2/2 = 2.5 + 0.045 = 2.545,  m = rho u = (0.3, 0, 0);
      n = (1, 0, 0):  G.n = (rho u_x, rho u_x^2 + p, 0, 0, u_x (E + p))
                          = (0.3, 0.09 + 1 = 1.09, 0, 0, 0.3 * 3.545 = 1.0635).
    F_a = -G.n (the flux leaves a through n), F_b = +G.n. Fails for G_E = E u (0.7635),
    a dropped m_x (u.n) (1.0 instead of 1.09) or a dropped p (0.09)."""
    U = [1.0, 0.3, 0.0, 0.0, 2.545]
    F = _one_face(U, U, [1.0, 0.0, 0.0])
    Gn = np.array([0.3, 1.09, 0.0, 0.0, 1.0635])
    assert np.allclose(F[0], -Gn, rtol=1e-6, atol=1e-7)
    assert np.allclose(F[1], Gn, rtol=1e-6, atol=1e-7)


def test_uniform_flow_general_direction():
    """Uniform state, velocity and normal in general position (every component of the
    momentum flux m (u.n) + p n is exercised with a different value).
    rho = 2, u = (0.1, -0.2, 0.3), p = 1.5:  m = (0.2, -0.4, 0.6), |u|^2 = 0.14,
      E = 1.5/0.4 + 0.5 * 2 * 0.14 = 3.75 + 0.14 = 3.89.
    n = (0.5, 1, -2):  u.n = 0.05 - 0.2 - 0.6 = -0.75,  m.n = 0.1 - 0.4 - 1.2 = -1.5;
      (G.n)_rho = m.n = -1.5
      (G.n)_mx  = m_x (u.n) + p n_x = -0.15 + 0.75 =  0.6
      (G.n)_my  = m_y (u.n) + p n_y =  0.3  + 1.5  =  1.8
      (G.n)_mz  = m_z (u.n) + p n_z = -0.45 - 3.0  = -3.45
      (G.n)_E   = (E + p)(u.n) = 5.39 * -0.75      = -4.0425
    F_a = -G.n."""
    U = [2.0, 0.2, -0.4, 0.6, 3.89]
    F = _one_face(U, U, [0.5, 1.0, -2.0])
    assert np.allclose(F[0], [1.5, -0.6, -1.8, 3.45, 4.0425], rtol=1e-6, atol=1e-6)
    assert np.allclose(F[1], -F[0], rtol=0, atol=1e-12)


def test_dissipation_magnitude_at_rest():
    """Two fluids at rest (u = 0: no convective flux; only the pressure and the
    dissipation act). gamma = 1.4, sigma = 0.2, n = (2, 0, 0), |n| = 2:
      a: rho = 1.2, E = 2.5 -> p = 0.4 * 2.5 = 1.0, c_a = sqrt(1.4 * 1.0 / 1.2) = 1.0801234497346435
      b: rho = 1.0, E = 2.0 -> p = 0.4 * 2.0 = 0.8, c_b = sqrt(1.4 * 0.8 / 1.0) = 1.0583005244258363
      f = -|n| sigma (|u_a| + |u_b| + c_a + c_b)/2 = -0.2 (c_a + c_b) = -0.427684794832096
      Phi_rho = f (1.2 - 1.0)                 = -0.0855369589664192
      Phi_mx  = f * 0 - (p_a + p_b) n_x / 2   = -1.8
      Phi_E   = f (2.5 - 2.0)                 = -0.213842397416048
    Fails for c = sqrt(p/rho), a missing 1/2 or sigma, or |n| dropped from f."""
    F = _one_face([1.2, 0, 0, 0, 2.5], [1.0, 0, 0, 0, 2.0], [2.0, 0.0, 0.0])
    want = [-0.0855369589664192, -1.8, 0.0, 0.0, -0.213842397416048]
    assert np.allclose(F[0], want, rtol=1e-6, atol=1e-12)
    assert np.allclose(F[1], -F[0], rtol=0, atol=1e-15)


def test_dissipation_speed_includes_velocity():
    """The dissipation speed is |u| + c of both sides. a moves across the face
    (u_a = (0, 0.4, 0), u_a.n = 0: no convective flux through n = (1, 0, 0)), b is at rest;
    rho = 1, p = 1 on both sides: E_a = 2.5 + 0.16/2 = 2.58, E_b = 2.5, c = sqrt(1.4) =
    1.1832159566199232 on both sides.
      f = -1 * 0.2 * (0.4 + 2c)/2 = -0.2766431913239846
      U_a - U_b = (0, 0, 0.4, 0, 0.08)
      n.G_a = n.G_b = (0, p, 0, 0, 0) = (0, 1, 0, 0, 0)
      Phi = (0, -1, 0.4 f, 0, 0.08 f) = (0, -1, -0.11065727652959385, 0, -0.02213145530591877)."""
    F = _one_face([1.0, 0.0, 0.4, 0.0, 2.58], [1.0, 0.0, 0.0, 0.0, 2.5], [1.0, 0.0, 0.0])
    want = [0.0, -1.0, -0.11065727652959385, 0.0, -0.02213145530591877]
    assert np.allclose(F[0], want, rtol=1e-6, atol=1e-7)


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


def test_flux_abs_scale(small_mesh):
    """S_v = sum_e |Phi_e| (the componentwise scale of Z14) bounds |F_v| and equals it for
    a vertex with a single edge; for one face S_a = S_b = |Phi| (hand value of
    test_dissipation_magnitude_at_rest)."""
    M = small_mesh
    U = S.cfd_state(M.n, seed=3)
    F = O.cfd_flux(M.edges, M.n, M.normals, U)
    Sv = O.cfd_flux_abs(M.edges, M.n, M.normals, U)
    assert np.all(np.abs(F) <= Sv * (1 + 1e-12))
    e = np.array([[0, 1]], np.int32)
    Sab = O.cfd_flux_abs(e, 2, np.array([[2.0, 0, 0]], np.float32),
                         np.array([[1.2, 0, 0, 0, 2.5], [1.0, 0, 0, 0, 2.0]], np.float32))
    want = [0.0855369589664192, 1.8, 0.0, 0.0, 0.213842397416048]
    assert np.allclose(Sab[0], want, rtol=1e-6) and np.allclose(Sab[1], want, rtol=1e-6)


def test_cfd_step_omp_matches_sequential(small_mesh):
    """The all-core timing variant (vertex-centric incidence sums, CPU baseline only) adds each
    vertex's terms in orc_cfd_flux's order, so it equals the sequential step bit for bit --
    also on a random multigraph with self-loops and parallel edges."""
    M = small_mesh
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    ref, F = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    got, F2, th = O.cfd_step_omp(M.edges, M.n, M.normals, U, dt)
    assert th >= 1
    assert np.array_equal(F2, F) and np.array_equal(got, ref)
    n, e = S.random_multigraph(77, 3000, 900)
    rng = np.random.default_rng(5)
    nrm = rng.uniform(-1, 1, (len(e), 3)).astype(np.float32)
    U2, dt2 = S.cfd_state(n), rng.uniform(0.01, 0.1, n).astype(np.float32)
    ref, F = O.cfd_step(e, n, nrm, U2, dt2)
    got, F2, _ = O.cfd_step_omp(e, n, nrm, U2, dt2)
    assert np.array_equal(F2, F) and np.array_equal(got, ref)
