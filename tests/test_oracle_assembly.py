"""Pins of the oracle's pattern and assembly: closed-form
counts, brute-force patterns, energy finite differences, equilibrium, rigid
modes, patch tests, objectivity and serial/parallel agreement."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from synth import gen
from synth.gen import HEX8, TET10

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def mesh_case(kind="hex", n=2, jitter=0.1, w=16, L=2, seed=4, amp=0.05):
    if kind == "hex":
        X, conn = gen.hex_mesh(n, jitter, seed)
        et = HEX8
    else:
        X, conn = gen.tet10_mesh(n, jitter, seed)
        et = TET10
    gN, qw = gen.shape_gradients(X, conn, et)
    m = gen.ncm_weights(w, L, 0.3, seed + 1, 10.0)
    rng = np.random.default_rng(seed + 2)
    u = gen.smooth_field(X, amp, rng).reshape(-1)
    return dict(X=X, conn=conn, gN=gN, qw=qw, m=m, u=u, n_nodes=X.shape[0])


def assemble(c, u=None, m=None, mode=0):
    rp, ci = oracle.pattern(c["n_nodes"], c["conn"])
    r, v, bad = oracle.assemble(c["m"] if m is None else m, c["n_nodes"], c["conn"], c["gN"],
                                c["qw"], c["u"] if u is None else u, rp, ci, mode=mode)
    return rp, ci, r, v, bad


def dense(rp, ci, v, n):
    K = np.zeros((len(rp) - 1, n))
    for row in range(len(rp) - 1):
        K[row, ci[rp[row]:rp[row + 1]]] = v[rp[row]:rp[row + 1]]
    return K


# ------------------------------------------------------------------ pattern
def test_hex_nnz_closed_form_and_paper_dofs():
    g = json.load(open(os.path.join(GOLD, "paper_counts.json")))
    for n in (1, 2, 3, 4):
        X, conn = gen.hex_mesh(n)
        rp, ci = oracle.pattern(X.shape[0], conn)
        assert ci.size == 9 * (3 * n + 1) ** 3
    assert [x["nnz"] for x in g["hex_nnz"] if x["n"] == 4] == [19773]
    for case in g["cube_dofs"]:
        assert 3 * (case["n"] + 1) ** 3 == case["dofs"]


@pytest.mark.parametrize("kind,n", [("hex", 3), ("tet", 2)])
def test_pattern_brute_force(kind, n):
    X, conn = (gen.hex_mesh(n, 0.1) if kind == "hex" else gen.tet10_mesh(n, 0.1))
    nn = X.shape[0]
    rp, ci = oracle.pattern(nn, conn)
    pairs = set()
    for e in conn:
        for a, b in itertools.product(e, e):
            pairs.add((int(a), int(b)))
    ref = sorted((3 * a + i, 3 * b + k) for a, b in pairs for i in range(3) for k in range(3))
    got = [(row, int(c)) for row in range(3 * nn) for c in ci[rp[row]:rp[row + 1]]]
    assert got == ref
    Kp = np.zeros((3 * nn, 3 * nn), bool)
    for row, c in got:
        Kp[row, c] = True
    assert (Kp == Kp.T).all()


def test_owned_rows_slice():
    X, conn = gen.hex_mesh(3)
    nn = X.shape[0]
    rp, ci = oracle.pattern(nn, conn)
    rp2, ci2 = oracle.pattern(nn, conn, 16, 40)
    assert np.array_equal(ci2, ci[rp[48]:rp[120]])
    assert np.array_equal(rp2, rp[48:121] - rp[48])


def test_tet10_c4_counts():
    """c4 (48^3 x 6 tet10): 912,673 nodes, 231,797,385 nnz, <= 65 nodes/row
    (from an independent brute-force unique-pairs count)."""
    X, conn = gen.tet10_mesh(48, 0.0)
    assert X.shape[0] == 912673 and conn.shape == (663552, 10)
    rp, ci = oracle.pattern(X.shape[0], conn)
    assert ci.size == 231797385
    assert np.max(np.diff(rp)) == 3 * 65


# -------------------------------------------------------------- generator
@pytest.mark.parametrize("kind", ["hex", "tet"])
def test_generator_shape_gradients(kind):
    c = mesh_case(kind, n=3)
    assert np.max(np.abs(c["gN"].sum(axis=2))) < 1e-13        # partition of unity
    assert abs(c["qw"].sum() - 1.0) < 1e-14                    # unit-cube volume
    H = np.array([[0.1, -0.2, 0.05], [0.03, 0.2, -0.1], [0.0, 0.15, -0.05]])
    u = (c["X"] @ H.T).reshape(-1)
    F = oracle.qp_F(c["conn"], c["gN"], u)                      # patch: F = I + H exactly
    assert np.max(np.abs(F - (np.eye(3) + H))) < 1e-14


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_configs_valid(name):
    """Generated displacements keep min det F > 0.2 (SURVEY.md s8(d) validity)."""
    c = gen.make_config(name)
    F = oracle.qp_F(c["conn"], c["gradN"], c["u"])
    assert np.linalg.det(F).min() > 0.2


@pytest.mark.slow
def test_config_c4_valid():
    c = gen.make_config("c4")
    F = oracle.qp_F(c["conn"], c["gradN"], c["u"])
    assert np.linalg.det(F).min() > 0.2


# ------------------------------------------------------------- assembly
@pytest.mark.parametrize("kind", ["hex", "tet"])
def test_residual_is_energy_gradient(kind):
    c = mesh_case(kind, n=2 if kind == "hex" else 1, w=8)
    _, _, r, _, bad = assemble(c)
    assert bad == -1
    rng = np.random.default_rng(0)
    h = 1e-6
    for dof in rng.choice(c["u"].size, 12, replace=False):
        up, um = c["u"].copy(), c["u"].copy()
        up[dof] += h
        um[dof] -= h
        fd = (oracle.energy(c["m"], c["conn"], c["gN"], c["qw"], up)
              - oracle.energy(c["m"], c["conn"], c["gN"], c["qw"], um)) / (2 * h)
        assert abs(fd - r[dof]) < 1e-7 * np.abs(r).max()


@pytest.mark.parametrize("kind", ["hex", "tet"])
def test_stiffness_is_residual_jacobian(kind):
    c = mesh_case(kind, n=2 if kind == "hex" else 1, w=8)
    rp, ci, r, v, _ = assemble(c)
    K = dense(rp, ci, v, c["u"].size)
    rng = np.random.default_rng(1)
    h = 1e-6
    for col in rng.choice(c["u"].size, 10, replace=False):
        up, um = c["u"].copy(), c["u"].copy()
        up[col] += h
        um[col] -= h
        fd = (assemble(c, up)[2] - assemble(c, um)[2]) / (2 * h)
        assert np.max(np.abs(fd - K[:, col])) < 1e-7 * np.abs(K).max()


@pytest.mark.parametrize("kind", ["hex", "tet"])
def test_equilibrium_rigid_modes_symmetry(kind):
    c = mesh_case(kind, n=3 if kind == "hex" else 2)
    rp, ci, r, v, _ = assemble(c)
    K = dense(rp, ci, v, c["u"].size)
    # sum of internal forces vanishes for any u (translation invariance of Pi)
    assert np.max(np.abs(r.reshape(-1, 3).sum(axis=0))) < 1e-13 * np.abs(r).max()
    # K t = 0 for rigid translations
    for i in range(3):
        t = np.zeros(c["u"].size)
        t[i::3] = 1.0
        assert np.max(np.abs(K @ t)) < 1e-12 * np.abs(K).max()
    assert np.max(np.abs(K - K.T)) < 1e-13 * np.abs(K).max()


def _interior_dofs(X):
    inside = np.all((X > 1e-9) & (X < 1 - 1e-9), axis=1)
    return np.repeat(inside, 3)


@pytest.mark.parametrize("kind", ["hex", "tet"])
def test_patch_test(kind):
    """Affine u -> homogeneous F -> interior residual vanishes."""
    c = mesh_case(kind, n=3 if kind == "hex" else 2)
    H = np.array([[0.1, -0.05, 0.02], [0.04, 0.15, -0.03], [0.01, 0.02, -0.08]])
    u = (c["X"] @ H.T).reshape(-1)
    _, _, r, _, _ = assemble(c, u)
    inner = _interior_dofs(c["X"])
    assert inner.any()
    assert np.max(np.abs(r[inner])) < 1e-13 * np.abs(r).max()


def test_zero_displacement_residual():
    """Reading R11: raw NCM -> interior r(0) = 0 (constant stress is
    self-equilibrated) and boundary r != 0; with ref_shift -> r(0) = 0."""
    c = mesh_case("hex", n=3)
    u0 = np.zeros_like(c["u"])
    _, _, r, _, _ = assemble(c, u0)
    inner = _interior_dofs(c["X"])
    assert np.max(np.abs(r[inner])) < 1e-15 and np.max(np.abs(r)) > 1e-4
    g = oracle.material_point(c["m"], np.eye(3))["g"]
    m = dict(c["m"], ref_shift=2 * g[0] + 4 * g[1] + g[2])
    _, _, r, _, _ = assemble(c, u0, m)
    assert np.max(np.abs(r)) < 1e-15


def test_objectivity():
    """x' = Q x: r_a(u') = Q r_a(u), K_ab(u') = Q K_ab Q^T."""
    c = mesh_case("hex", n=2)
    Q, R = np.linalg.qr(np.random.default_rng(7).normal(size=(3, 3)))
    if np.linalg.det(Q) < 0:
        Q[:, 0] *= -1
    x = c["X"] + c["u"].reshape(-1, 3)
    u2 = (x @ Q.T - c["X"]).reshape(-1)
    rp, ci, r, v, _ = assemble(c)
    _, _, r2, v2, _ = assemble(c, u2)
    assert np.max(np.abs(r2.reshape(-1, 3) - r.reshape(-1, 3) @ Q.T)) < 1e-13 * np.abs(r).max()
    n = c["n_nodes"]
    K = dense(rp, ci, v, 3 * n).reshape(n, 3, n, 3)
    K2 = dense(rp, ci, v2, 3 * n).reshape(n, 3, n, 3)
    KQ = np.einsum("ij,ajbk,lk->aibl", Q, K, Q)
    assert np.max(np.abs(K2 - KQ)) < 1e-12 * np.abs(K).max()


@pytest.mark.parametrize("kind", ["hex", "tet"])
def test_serial_equals_coloured_parallel(kind):
    c = mesh_case(kind, n=3 if kind == "hex" else 2)
    rp, ci, r0, v0, _ = assemble(c, mode=0)
    _, _, r1, v1, _ = assemble(c, mode=1)
    assert np.max(np.abs(r0 - r1)) <= 1e-14 * np.abs(r0).max()
    assert np.max(np.abs(v0 - v1)) <= 1e-14 * np.abs(v0).max()


def test_domain_error_flag():
    """Reading R10: det F <= 0 is reported as the lowest flat e*n_q+q."""
    c = mesh_case("hex", n=2, jitter=0.0)
    u = c["u"].copy()
    # push node 13 (the centre) through its neighbours: inverts elements
    u[3 * 13 + 0] += 0.9
    _, _, _, _, bad = assemble(c, u)
    F = oracle.qp_F(c["conn"], c["gN"], u)
    J = np.linalg.det(F).reshape(-1)
    assert bad == int(np.flatnonzero(J <= 0)[0])
