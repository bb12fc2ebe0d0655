"""Pins of the oracle's material-point arithmetic (SURVEY.md s8(c) "What pins
each part"): every check compares oracle/ against something that is NOT the
oracle -- closed forms, an independent hyper-dual derivation of W(F), an
independent Jacobian+adjoint implementation of the inner network, the paper's
spatial G-tensor formulas, finite differences, symmetries and objectivity."""
import json
import os

import numpy as np
import pytest

import oracle
from synth.gen import ncm_weights
from tests import hyperdual

GOLD = os.path.join(os.path.dirname(__file__), "golden")
I3 = np.eye(3)


def rand_F(rng, amp=0.25):
    while True:
        F = I3 + rng.uniform(-amp, amp, (3, 3))
        if np.linalg.det(F) > 0.3:
            return F


def rot(rng):
    Q, R = np.linalg.qr(rng.normal(size=(3, 3)))
    Q = Q * np.sign(np.diag(R))
    if np.linalg.det(Q) < 0:
        Q[:, 0] *= -1
    return Q


def small_ncm(w=8, L=2, seed=5, skips=False, kappa=10.0):
    m = ncm_weights(w, L, 0.3, seed, kappa)
    if skips:
        rng = np.random.default_rng(seed + 100)
        m["skip_out"] = rng.normal(0, 0.3, 3)
        m["skip_hidden"] = rng.normal(0, 0.3, (L - 1, w, 3))
    return m


# ---------------------------------------------------------------- kinematics
def test_invariants_golden():
    """SPEC.md:116-117 closed forms (tests/golden/kinematics.json)."""
    g = json.load(open(os.path.join(GOLD, "kinematics.json")))
    m = small_ncm()
    for case in g["cases"]:
        out = oracle.material_point(m, np.array(case["F"], float))
        k = out["k"]
        assert abs(k[0] + 3 - case["I1"]) < 1e-14
        assert abs(k[1] + 3 - case["I2"]) < 1e-14
        assert abs(k[2] + 1 - case["J"]) < 1e-14
        assert abs(out["J"] ** 2 - case["I3"]) < 1e-14


def test_invariants_objective():
    rng = np.random.default_rng(0)
    m = small_ncm()
    for _ in range(5):
        F, Q = rand_F(rng), rot(rng)
        a, b = oracle.material_point(m, F), oracle.material_point(m, Q @ F)
        assert np.allclose(a["k"], b["k"], atol=1e-14)
        assert np.allclose(a["S"], b["S"], atol=1e-13)          # S is material: invariant
        assert np.allclose(Q @ a["P"], b["P"], atol=1e-13)      # P -> Q P


# ------------------------------------------------------------- inner network
def jac_adjoint_ncm(m, k):
    """Independent exact derivatives of the ICNN: forward Jacobians J_l,
    reverse adjoints lambda_l, H = sum_l J_l^T diag(lambda_l s''(y_l)) J_l
    (a different derivation from Alg. 4)."""
    sig = lambda y: 1.0 / (1.0 + np.exp(-y))
    sp = lambda y: np.logaddexp(0.0, y)
    L = m["n_hidden"]
    ys, Js = [], []
    y = m["W1"] @ k + m["b"][0]
    Jm = m["W1"].copy()
    ys.append(y); Js.append(Jm)
    z = sp(y)
    for l in range(1, L):
        Bl = np.zeros((m["width"], 3)) if m.get("skip_hidden") is None else m["skip_hidden"][l - 1]
        y = m["W"][l - 1] @ z + Bl @ k + m["b"][l]
        Jm = m["W"][l - 1] @ (sig(ys[-1])[:, None] * Js[-1]) + Bl
        ys.append(y); Js.append(Jm)
        z = sp(y)
    s_out = np.zeros(3) if m.get("skip_out") is None else m["skip_out"]
    N = m["a"] @ z + s_out @ k
    lam = m["a"].copy()
    g = s_out.copy()
    H = np.zeros((3, 3))
    for l in range(L - 1, -1, -1):
        s = sig(ys[l])
        H += Js[l].T @ ((lam * s * (1 - s))[:, None] * Js[l])
        mu = lam * s
        if l >= 1:
            if m.get("skip_hidden") is not None:
                g += m["skip_hidden"][l - 1].T @ mu
            lam = m["W"][l - 1].T @ mu
        else:
            g += m["W1"].T @ mu
    return N, g, H


@pytest.mark.parametrize("w,L,skips", [(8, 1, False), (8, 2, False), (16, 3, False), (8, 3, True)])
def test_alg4_equals_jacobian_adjoint(w, L, skips):
    m = small_ncm(w, L, seed=3 + w + L, skips=skips)
    rng = np.random.default_rng(1)
    for _ in range(5):
        k = rng.uniform(-0.5, 0.5, 3)
        N, g, H = oracle.ncm_eval(m, k)
        N2, g2, H2 = jac_adjoint_ncm(m, k)
        assert abs(N - N2) <= 1e-13 * max(1, abs(N2))
        assert np.max(np.abs(g - g2)) <= 1e-13 * max(1, np.max(np.abs(g2)))
        assert np.max(np.abs(H - H2)) <= 1e-13 * max(1, np.max(np.abs(H2)))
        assert np.array_equal(H, H.T) or np.max(np.abs(H - H.T)) < 1e-15


def test_ncm_finite_difference():
    """Central FD (SPEC.md:188, 221 tolerances 1e-6 / 1e-4 loosened to 1e-7/1e-5 rel here)."""
    m = small_ncm(16, 3, seed=11)
    k = np.array([0.2, -0.1, 0.05])
    N, g, H = oracle.ncm_eval(m, k)
    h = 1e-5
    for i in range(3):
        e = np.zeros(3); e[i] = h
        Np, gp, _ = oracle.ncm_eval(m, k + e)
        Nm, gm, _ = oracle.ncm_eval(m, k - e)
        assert abs((Np - Nm) / (2 * h) - g[i]) < 1e-7 * max(1, np.abs(g).max())
        assert np.max(np.abs((gp - gm) / (2 * h) - H[:, i])) < 1e-5 * max(1, np.abs(H).max())


def test_ncm_special_cases():
    """All weights 0 -> N = g = H = 0; a = 0 -> g = skip, H = 0."""
    m = small_ncm(8, 2)
    z = {k: (np.zeros_like(v) if isinstance(v, np.ndarray) else v) for k, v in m.items()}
    N, g, H = oracle.ncm_eval(z, np.array([0.3, -0.2, 0.1]))
    assert N == 0 and not g.any() and not H.any()
    m2 = dict(m, a=np.zeros(8), skip_out=np.array([1.5, -0.25, 0.75]))
    N, g, H = oracle.ncm_eval(m2, np.array([0.3, -0.2, 0.1]))
    assert np.array_equal(g, m2["skip_out"]) and not H.any()
    assert abs(N - m2["skip_out"] @ [0.3, -0.2, 0.1]) < 1e-15


# ------------------------------------------------------ stress and tangent
@pytest.mark.parametrize("skips,shift", [(False, 0.0), (True, 0.0), (False, 0.37)])
def test_hyperdual_P_and_A(skips, shift):
    """P = dW/dF and A = d2W/dFdF straight from W(F) with hyper-dual numbers
    (exact to rounding) pin steps a3-a7 of the oracle (kinematics, NCM
    derivatives, material G-tensors, push to P and A)."""
    m = small_ncm(8, 2, seed=7, skips=skips)
    m["ref_shift"] = shift
    rng = np.random.default_rng(2)
    for _ in range(3):
        F = rand_F(rng)
        W, P, A = hyperdual.derivatives(F, m)
        o = oracle.material_point(m, F)
        assert abs(o["W"] - W) < 1e-13 * max(1, abs(W))
        assert np.max(np.abs(o["P"] - P)) < 1e-12 * np.abs(P).max()
        assert np.max(np.abs(o["A"] - A)) < 1e-12 * np.abs(A).max()


def mooney_rivlin_closed_form(F, c1, c2, kappa):
    """W = c1(I1-3) + c2(I2-3) - (2c1+4c2)(J-1) + kappa (J-1)^2.
    S = 2c1 I + 2c2(I1 I - C) + p J C^-1,
    CC = 4c2 (I(x)I - II) + (2 kappa J^2 + p J) C^-1(x)C^-1 - 2 p J II_{C^-1},
    p = -(2c1+4c2) + 2 kappa (J-1)."""
    C = F.T @ F
    Ci = np.linalg.inv(C)
    J = np.linalg.det(F)
    I1 = np.trace(C)
    p = -(2 * c1 + 4 * c2) + 2 * kappa * (J - 1)
    S = 2 * c1 * I3 + 2 * c2 * (I1 * I3 - C) + p * J * Ci
    II = 0.5 * (np.einsum("ik,jl->ijkl", I3, I3) + np.einsum("il,jk->ijkl", I3, I3))
    IIc = 0.5 * (np.einsum("ik,jl->ijkl", Ci, Ci) + np.einsum("il,jk->ijkl", Ci, Ci))
    CC = (4 * c2 * (np.einsum("ij,kl->ijkl", I3, I3) - II)
          + (2 * kappa * J * J + p * J) * np.einsum("ij,kl->ijkl", Ci, Ci) - 2 * p * J * IIc)
    return S, CC


def test_mooney_rivlin_closed_form():
    c1, c2, kappa = 0.8, 0.35, 10.0
    m = small_ncm(8, 2, kappa=kappa)
    m["a"] = np.zeros(8)
    m["skip_out"] = np.array([c1, c2, -(2 * c1 + 4 * c2)])
    rng = np.random.default_rng(3)
    for F in [I3, np.diag([1.2, 0.9, 1.05])] + [rand_F(rng) for _ in range(4)]:
        o = oracle.material_point(m, F)
        S, CC = mooney_rivlin_closed_form(F, c1, c2, kappa)
        assert np.max(np.abs(o["S"] - S)) < 1e-13 * max(1, np.abs(S).max())
        assert np.max(np.abs(o["CC"] - CC)) < 1e-13 * np.abs(CC).max()
    # F = I: stress free, CC = lambda I(x)I + 2 mu II (linear elasticity)
    o = oracle.material_point(m, I3)
    lam, mu = 2 * kappa - 2 * c1, 2 * c1 + 2 * c2
    II = 0.5 * (np.einsum("ik,jl->ijkl", I3, I3) + np.einsum("il,jk->ijkl", I3, I3))
    assert np.max(np.abs(o["S"])) < 1e-14
    assert np.max(np.abs(o["CC"] - (lam * np.einsum("ij,kl->ijkl", I3, I3) + 2 * mu * II))) < 1e-13


def test_tangent_symmetries():
    m = small_ncm(16, 3, seed=9)
    rng = np.random.default_rng(4)
    for _ in range(4):
        o = oracle.material_point(m, rand_F(rng))
        CC, A = o["CC"], o["A"]
        sc = np.abs(CC).max()
        assert np.max(np.abs(CC - CC.transpose(1, 0, 2, 3))) < 1e-14 * sc   # minor
        assert np.max(np.abs(CC - CC.transpose(0, 1, 3, 2))) < 1e-14 * sc   # minor
        assert np.max(np.abs(CC - CC.transpose(2, 3, 0, 1))) < 1e-14 * sc   # major
        assert np.max(np.abs(A - A.transpose(2, 3, 0, 1))) < 1e-13 * np.abs(A).max()
        assert np.max(np.abs(o["S"] - o["S"].T)) < 1e-15 * max(1, np.abs(o["S"]).max())


def _obox(A, B):
    """(A (x)bar B)_ijkl = 1/2 (A_ik B_jl + A_il B_jk) (reading R5)."""
    return 0.5 * (np.einsum("ik,jl->ijkl", A, B) + np.einsum("il,jk->ijkl", A, B))


def test_spatial_G_tensors_match_material_form():
    """The paper's SPATIAL formulas -- G-tensors of App. A.2 (PAPER.md:812-814,
    862) in Eq. stress-cgo / stiffnes-cgo and the push of
    Eq. hyper-stress-stiffness -- evaluated here from the
    oracle's g, H must equal the push-forward of the oracle's S, CC, A
    (reading R1: material form is exactly equal)."""
    m = small_ncm(16, 2, seed=13)
    rng = np.random.default_rng(5)
    for _ in range(4):
        F = rand_F(rng)
        o = oracle.material_point(m, F)
        g, H = o["g"], o["H"]
        B = F @ F.T
        J = np.linalg.det(F)
        G = [B, B * np.trace(B) - B @ B, 0.5 * J * I3]
        GG = [np.zeros((3, 3, 3, 3)),
              np.einsum("ij,kl->ijkl", B, B) - _obox(B, B),
              0.25 * J * (np.einsum("ij,kl->ijkl", I3, I3) - 2 * _obox(I3, I3))]
        tau = 2 * sum(g[i] * G[i] for i in range(3))
        c = 4 * sum(H[i, j] * np.einsum("ij,kl->ijkl", G[i], G[j]) for i in range(3) for j in range(3))
        c = c + 4 * sum(g[i] * GG[i] for i in range(3))
        tau_o = F @ o["S"] @ F.T
        c_o = np.einsum("iI,jJ,kK,lL,IJKL->ijkl", F, F, F, F, o["CC"])
        assert np.max(np.abs(tau - tau_o)) < 1e-13 * np.abs(tau).max()
        assert np.max(np.abs(c - c_o)) < 1e-13 * np.abs(c).max()
        # Eq. hyper-stress-stiffness: c_ijkl = F_jJ A_iJkL F_lL - d_ik tau_jl
        c_h = np.einsum("jJ,iJkL,lL->ijkl", F, o["A"], F) - np.einsum("ik,jl->ijkl", I3, tau_o)
        assert np.max(np.abs(c_h - c_o)) < 1e-13 * np.abs(c).max()
        # tau = P F^T
        assert np.max(np.abs(o["P"] @ F.T - tau_o)) < 1e-13 * np.abs(tau).max()


def test_ref_shift_makes_identity_stress_free():
    """Reading R11: s0 = 2 g1(0) + 4 g2(0) + g3(0) gives S(I) = 0."""
    m = small_ncm(16, 2, seed=21)
    o = oracle.material_point(m, I3)
    g = o["g"]  # includes the penalty derivative, 0 at J = 1
    assert np.max(np.abs(o["S"])) > 1e-3      # raw seeded NCM is not stress-free
    m["ref_shift"] = 2 * g[0] + 4 * g[1] + g[2]
    o2 = oracle.material_point(m, I3)
    assert np.max(np.abs(o2["S"])) < 1e-14
