"""Pins of the Newton-Raphson oracle (oracle/newton.py)
against what the mathematics fixes: closed-form linear solves, the symmetric
elimination's definition, a homogeneous uniaxial-tension solution obtained by
1-D root finding on an independently written Mooney-Rivlin stress, a
stress-free reference at zero load, and the quadratic convergence of Newton on
the twist cube."""
import math

import numpy as np
import pytest
import scipy.optimize as so
import scipy.sparse as sp

import oracle
from oracle import newton as on
from synth import twist


# ---- CG-Jacobi -------------------------------------------------------------------
def test_cg_identity_one_iteration():
    b = np.arange(1.0, 6.0)
    x, it = on.cg_jacobi(sp.identity(5), b)
    assert it == 1 and np.array_equal(x, b)


def test_cg_diagonal_closed_form():
    x, it = on.cg_jacobi(sp.diags([2.0, 4.0, 8.0]), np.array([2.0, 4.0, 8.0]))
    assert it == 1 and np.allclose(x, 1.0, rtol=0, atol=1e-15)


def test_cg_random_spd_matches_dense_solve():
    rng = np.random.default_rng(5)
    M = rng.normal(size=(50, 50))
    A = M @ M.T + 50 * np.eye(50)
    b = rng.normal(size=50)
    x, it = on.cg_jacobi(sp.csr_matrix(A), b, rtol=1e-13)
    xd = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)
    assert it <= 50


def test_block_cg_block_diagonal_one_iteration():
    """A block-diagonal SPD matrix of 3x3 blocks is its own block-Jacobi preconditioner:
    PCG converges in one iteration to the exact solution."""
    rng = np.random.default_rng(7)
    blocks = []
    for _ in range(4):
        M = rng.normal(size=(3, 3))
        blocks.append(M @ M.T + 3 * np.eye(3))
    A = sp.block_diag(blocks, format="csr")
    b = rng.normal(size=12)
    x, it = on.cg_jacobi(A, b, rtol=1e-14, block=True)
    assert it == 1 and np.allclose(x, np.linalg.solve(A.toarray(), b), rtol=0, atol=1e-13)
    _, it_j = on.cg_jacobi(A, b, rtol=1e-14)
    assert it_j > 1  # the scalar Jacobi preconditioner does not invert the blocks


def test_block_cg_random_spd_matches_dense_solve():
    rng = np.random.default_rng(6)
    M = rng.normal(size=(48, 48))
    A = M @ M.T + 48 * np.eye(48)
    b = rng.normal(size=48)
    x, it = on.cg_jacobi(sp.csr_matrix(A), b, rtol=1e-13, block=True)
    xd = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd) and it <= 48


# ---- symmetric elimination -------------------------------------------------------
def test_eliminate_definition():
    rng = np.random.default_rng(3)
    A = rng.normal(size=(9, 9))
    A = A + A.T + 20 * np.eye(9)
    Acsr = sp.csr_matrix(A)
    mask = np.zeros(9, bool)
    mask[[1, 4, 8]] = True
    r = rng.normal(size=9)
    vals, r2 = on.eliminate(Acsr.indptr.astype(np.int64), Acsr.indices.astype(np.int32), Acsr.data, r, mask)
    E = sp.csr_matrix((vals, Acsr.indices, Acsr.indptr), shape=(9, 9)).toarray()
    free = ~mask
    assert np.array_equal(E[np.ix_(free, free)], A[np.ix_(free, free)])
    assert np.array_equal(E[np.ix_(mask, mask)], np.eye(3))
    assert not E[np.ix_(mask, free)].any() and not E[np.ix_(free, mask)].any()
    assert np.array_equal(r2[free], r[free]) and not r2[mask].any()


# ---- homogeneous uniaxial tension: closed form by 1-D root finding ---------------
def mooney_rivlin_ncm(c1, c2, kappa, width=8):
    z = np.zeros
    return dict(width=width, n_hidden=2, W1=z((width, 3)), W=z((1, width, width)), b=z((2, width)), a=z(width),
                skip_out=np.array([c1, c2, -(2 * c1 + 4 * c2)]), skip_hidden=None, kappa=kappa, ref_shift=0.0)


def mr_lateral_stress(mu, lam, c1, c2, kappa):
    """S_11 of W = c1 (I1-3) + c2 (I2-3) - (2c1+4c2)(J-1) + kappa (J-1)^2 at
    F = diag(mu, mu, lam): S = 2 c1 I + 2 c2 (I1 I - C) + p J C^-1,
    p = -(2 c1 + 4 c2) + 2 kappa (J - 1) (textbook compressible Mooney-Rivlin)."""
    J = mu * mu * lam
    I1 = 2 * mu * mu + lam * lam
    p = -(2 * c1 + 4 * c2) + 2 * kappa * (J - 1.0)
    return 2 * c1 + 2 * c2 * (I1 - mu * mu) + p * J / (mu * mu)


@pytest.mark.parametrize("lam", [1.1, 1.6, 0.8])
def test_uniaxial_tension_matches_closed_form(lam):
    c1, c2, kappa = 0.7, 0.2, 3.0
    ncm = mooney_rivlin_ncm(c1, c2, kappa)
    mesh, dofs, vals = twist.uniaxial_problem(lam)
    rp, ci = oracle.pattern(mesh["n_nodes"], mesh["conn"])
    u, norms, ok = on.newton_step(ncm, mesh, rp, ci, np.zeros(3 * mesh["n_nodes"]), dofs, vals, atol=1e-13,
                                  rtol=1e-14)
    assert ok and norms[-1] < 1e-12
    mu = so.brentq(lambda m: mr_lateral_stress(m, lam, c1, c2, kappa), 0.3, 1.7, xtol=1e-15)
    X = mesh["X"]
    exact = np.stack([(mu - 1) * X[:, 0], (mu - 1) * X[:, 1], (lam - 1) * X[:, 2]], axis=1).reshape(-1)
    assert np.abs(u - exact).max() <= 1e-11


# ---- zero load, twist cube -----------------------------------------------------------
def _twist(n):
    mesh = twist.twist_mesh(n)
    ncm = twist.stable_ncm()
    ncm["ref_shift"] = on.reference_shift(ncm)
    rp, ci = oracle.pattern(mesh["n_nodes"], mesh["conn"])
    dofs, _, _ = twist.twist_bc(mesh["X"])
    return mesh, ncm, rp, ci, dofs


def test_zero_load_is_converged_at_once():
    mesh, ncm, rp, ci, dofs = _twist(3)
    u, norms, ok = on.newton_step(ncm, mesh, rp, ci, np.zeros(3 * mesh["n_nodes"]), dofs, np.zeros(dofs.size))
    assert ok and len(norms) == 1 and norms[0] < 1e-13
    assert not u.any()


def test_twist_cube_converges_quadratically():
    mesh, ncm, rp, ci, dofs = _twist(4)
    u = np.zeros(3 * mesh["n_nodes"])
    orders = []
    for s in range(1, 11):
        u, norms, ok = on.newton_step(ncm, mesh, rp, ci, u, dofs, twist.twist_values(mesh["X"], dofs, s / 10),
                                      atol=1e-13, rtol=1e-14)
        assert ok, (s, norms)
        assert len(norms) <= 8
        # convergence order estimated from the last three norms above the round-off floor
        nz = [x for x in norms if x > 1e-11 * norms[0]]
        orders.append(math.log(nz[-1] / nz[-2]) / math.log(nz[-2] / nz[-3]))
    assert min(orders) >= 1.7, orders
    # the top face turned by pi and moved up by 1: the deformed top corners
    x = mesh["X"].reshape(-1) + u
    top = np.nonzero(np.abs(mesh["X"][:, 2] - 1) < 1e-12)[0]
    xt = x.reshape(-1, 3)[top]
    assert np.allclose(xt[:, 2], 2.0) and np.allclose(xt[:, :2], 1.0 - mesh["X"][top, :2], atol=1e-12)
    assert on.max_trace_C(mesh, u) > 6.0
