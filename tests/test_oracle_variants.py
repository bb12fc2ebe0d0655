"""Pins of the oracle's kinematic and inner-network variants (SURVEY.md s8(f)
rank 2): isochoric invariants + J (App. A.2.2, written in the
paper's spatial G-tensor form and pulled back), CANN (Eq. cann-def /
cann-chain-rule) and the Gent-Thomas reference model (App. C,
PAPER.md:1075-1079).  Each is checked against hyper-dual derivatives of W(F)
written from the definitions (tests/hyperdual.py), closed forms and the values
SPEC.md fixes."""
import numpy as np
import pytest

import oracle
from synth.gen import (A_FIBRE, A_SHEET, anisotropic, cann_params, gent_thomas_params, hex_mesh, ickan_params, ncm_weights,
                       shape_gradients)
from tests import hyperdual
from tests.test_oracle_material import I3, rand_F, rot


def isochoric_icnn():
    m = ncm_weights(8, 2, 0.3, 11, 10.0)
    m["kinematics"] = "isochoric"
    return m


VARIANTS = {
    "gent_thomas": lambda: gent_thomas_params(),
    "cann_standard": lambda: cann_params(4, seed=3),
    "cann_isochoric": lambda: cann_params(5, seed=4, kinematics="isochoric"),
    "icnn_isochoric": isochoric_icnn,
    "ickan": lambda: ickan_params(),
    "ickan_isochoric": lambda: ickan_params((3, 5, 1), nb=7, seed=5, kinematics="isochoric"),
    "cann_anisotropic": lambda: anisotropic(cann_params(4, seed=6, n_in=5)),
    "ickan_anisotropic": lambda: anisotropic(ickan_params((5, 4, 1), nb=7, seed=7)),
    "icnn_anisotropic": lambda: anisotropic(ncm_weights(8, 2, 0.3, 13, 10.0, n_in=5)),
    # two structural vectors (fibre + sheet; pairs 00, 01, 11: 9 inputs), and a non-orthogonal pair
    "cann_two_vectors": lambda: anisotropic(cann_params(3, seed=8, n_in=9), A_FIBRE, A_SHEET),
    "ickan_two_vectors": lambda: anisotropic(ickan_params((9, 4, 1), nb=7, seed=9), A_FIBRE, A_SHEET),
    "icnn_two_vectors": lambda: anisotropic(ncm_weights(8, 2, 0.3, 17, 10.0, n_in=9), A_FIBRE, (0.0, 0.6, 0.8)),
    # isochoric anisotropic inputs Ibar1, Ibar2, J, Ibar4,ij, Ibar5,ij (App. A.2.2, reading R29)
    "icnn_iso_anisotropic": lambda: anisotropic(ncm_weights(8, 2, 0.3, 19, 10.0, n_in=5), isochoric=True),
    "cann_iso_anisotropic": lambda: anisotropic(cann_params(4, seed=10, n_in=5), isochoric=True),
    "cann_iso_two_vectors": lambda: anisotropic(cann_params(3, seed=12, n_in=9), A_FIBRE, (0.0, 0.6, 0.8),
                                                isochoric=True),
    "ickan_iso_two_vectors": lambda: anisotropic(ickan_params((9, 4, 1), nb=7, seed=13), A_FIBRE, A_SHEET,
                                                 isochoric=True),
}


# ---- Gent-Thomas values the paper / SPEC fix ------------------------------------------
def test_gent_thomas_reference_values():
    m = gent_thomas_params()
    o = oracle.material_point(m, I3)
    assert o["W"] == 0.0 and np.abs(o["S"]).max() < 1e-15          # Psi(I) = 0, tau(I) = 0
    o = oracle.material_point(m, 2.0 * I3)
    assert abs(o["W"] - 49.0) < 1e-12                               # Psi(diag(2,2,2)) = (8-1)^2
    assert np.allclose(o["k"], [0.0, 0.0, 7.0], atol=1e-13)         # Ibar1 = 3, J = 8


def test_isochoric_invariance_and_objectivity():
    rng = np.random.default_rng(8)
    m = isochoric_icnn()
    for _ in range(4):
        F = rand_F(rng)
        k = oracle.material_point(m, F)["k"]
        for c in (0.7, 1.9):
            kc = oracle.material_point(m, c * F)["k"]
            assert np.abs(kc[:2] - k[:2]).max() < 1e-13            # Ibar_m(cF) = Ibar_m(F)
        kq = oracle.material_point(m, rot(rng) @ F)["k"]
        assert np.abs(kq - k).max() < 1e-13


def _isochoric_only(m, nk):
    """The same model with no dependence on J: the network's J column (W1[:, 2] / the CANN's
    branch weights of input 3) zeroed and kappa = 0, so W = N(Ibar...) depends on Cbar = J^-2/3 C only."""
    m = dict(m, kappa=0.0)
    if m.get("network", "icnn") == "cann":
        w2 = np.array(m["cann_w2"], float)
        w2[2] = 0.0
        m["cann_w2"] = w2
    else:
        W1 = np.array(m["W1"], float)
        W1[:, 2] = 0.0
        m["W1"] = W1
    return m


@pytest.mark.parametrize("name,nk", [("icnn_iso_anisotropic", 5), ("cann_iso_anisotropic", 5),
                                     ("cann_iso_two_vectors", 9)])
def test_isochoric_anisotropic_deviatoric_stress(name, nk):
    """An energy of the isochoric invariants alone is invariant under F -> cF, so the Kirchhoff
    stress is deviatoric: P : F = tr(tau) = 0 for every F; differentiating P(F) : F = 0 once more
    gives A : F + P = 0 (sum over iJ of F_iJ A_iJkL = -P_kL) -- a pin of the whole isochoric
    G / GG table (App. A.2.2) independent of the hyper-dual derivatives."""
    m = _isochoric_only(VARIANTS[name](), nk)
    rng = np.random.default_rng(31)
    for _ in range(4):
        F = rand_F(rng)
        o = oracle.material_point(m, F)
        P, A = o["P"], o["A"]
        assert abs(np.sum(P * F)) < 1e-13 * np.abs(P).max()
        assert np.abs(np.einsum("ij,ijkl->kl", F, A) + P).max() < 1e-13 * np.abs(A).max()
        # and the inputs are scale-invariant (except J - 1, input 3)
        k1 = oracle.material_point(m, 1.37 * F)["k"]
        assert np.abs(k1[:2] - o["k"][:2]).max() < 1e-13


def test_isochoric_anisotropic_inputs_closed_form():
    """Ibar4 = J^-2/3 A0.C A0 and Ibar5 = J^-4/3 A0.C^2 A0 (App. A.2.2 with e = -1/3, -2/3), checked
    through the CANN's linear branch: a one-branch identity / x^1 / linear CANN gives
    N = sum_m w2 w1 K_m, so W - kappa (J-1)^2 recovers sum_m c_m K_m."""
    c = np.array([0.3, 0.2, 0.0, 0.5, 0.7])
    m = dict(network="cann", kinematics="isochoric_anisotropic", width=8, n_hidden=1, W1=None, W=None, b=None,
             a=None, skip_out=None, skip_hidden=None, cann_f=np.tile(np.array([0, 1, 0], np.int32), (5, 1, 1)),
             cann_w1=np.ones((5, 1)), cann_w2=c[:, None].copy(), kappa=0.0, ref_shift=0.0,
             a0=np.array([0.6, 0.8, 0.0]))
    rng = np.random.default_rng(5)
    A0 = m["a0"]
    for _ in range(3):
        F = rand_F(rng)
        C = F.T @ F
        J = np.linalg.det(F)
        I1, I2 = np.trace(C), 0.5 * (np.trace(C) ** 2 - np.trace(C @ C))
        K = [J ** (-2 / 3) * I1 - 3, J ** (-4 / 3) * I2 - 3, J - 1,
             J ** (-2 / 3) * A0 @ C @ A0 - 1, J ** (-4 / 3) * A0 @ C @ C @ A0 - 1]
        assert abs(oracle.material_point(m, F)["W"] - c @ K) < 1e-14


# ---- CANN -------------------------------------------------------------------------
def test_cann_hessian_is_diagonal():
    m = cann_params(6, seed=2)
    rng = np.random.default_rng(1)
    for _ in range(5):
        _, g, H = oracle.ncm_eval(m, rng.uniform(-0.4, 0.4, 3))
        assert not (H - np.diag(np.diag(H))).any()


def test_cann_single_branch_closed_forms():
    base = dict(network="cann", kinematics="standard", width=8, n_hidden=1, W1=None, W=None, b=None, a=None,
                skip_out=None, skip_hidden=None, kappa=0.0, ref_shift=0.0)
    K = np.array([0.3, -0.2, 0.15])
    w1 = np.full((3, 1), 0.2)
    w2 = np.array([[1.5], [0.5], [2.0]])
    # identity, x^1, linear: N = sum_m w2 w1 K_m
    m = dict(base, cann_f=np.tile(np.array([0, 1, 0], np.int32), (3, 1, 1)), cann_w1=w1, cann_w2=w2)
    N, g, H = oracle.ncm_eval(m, K)
    assert np.allclose(g, (w2 * w1)[:, 0], rtol=0, atol=1e-16) and not H.any()
    # Macaulay, x^2, exp: N = sum_m w2 (exp(w1 <K_m>^2) - 1)
    m = dict(base, cann_f=np.tile(np.array([1, 2, 1], np.int32), (3, 1, 1)), cann_w1=w1, cann_w2=w2)
    N, g, H = oracle.ncm_eval(m, K)
    Kp = np.maximum(K, 0)
    e = np.exp(0.2 * Kp ** 2)
    assert abs(N - np.sum(w2[:, 0] * (e - 1))) < 1e-15
    assert np.allclose(g, w2[:, 0] * e * 0.4 * Kp, rtol=1e-14, atol=0)
    assert np.allclose(np.diag(H), w2[:, 0] * (e * 0.4 + e * (0.4 * Kp) ** 2) * (K > 0), rtol=1e-14, atol=0)
    # abs, x^3, -ln(1 - w1 x): second derivative w1^2/(1 - w1 x)^2 f1'^2 + ... (reading R22)
    m = dict(base, cann_f=np.tile(np.array([2, 3, 2], np.int32), (3, 1, 1)), cann_w1=w1, cann_w2=w2)
    N, g, H = oracle.ncm_eval(m, K)
    x = np.abs(K) ** 3
    d1, dd1 = 3 * K ** 2 * np.sign(K), 6 * np.abs(K)
    q = 1 - 0.2 * x
    assert np.allclose(g, w2[:, 0] * 0.2 / q * d1, rtol=1e-14, atol=0)
    assert np.allclose(np.diag(H), w2[:, 0] * (0.04 / q ** 2 * d1 ** 2 + 0.2 / q * dd1), rtol=1e-14, atol=0)


# ---- every variant: P and A exact from W(F) ------------------------------------------------
@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_hyperdual_P_and_A_variants(name):
    m = VARIANTS[name]()
    rng = np.random.default_rng(21)
    for F in [I3 + 1e-3 * rng.normal(size=(3, 3))] + [rand_F(rng) for _ in range(3)]:
        W, P, A = hyperdual.derivatives(F, m)
        o = oracle.material_point(m, F)
        assert abs(o["W"] - W) < 1e-13 * max(1, abs(W))
        assert np.max(np.abs(o["P"] - P)) < 1e-12 * max(1e-3, np.abs(P).max())
        assert np.max(np.abs(o["A"] - A)) < 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_assembly_residual_is_energy_gradient(name):
    """r = dPi/du by central differences of the oracle energy on a 2^3 mesh."""
    m = VARIANTS[name]()
    X, conn = hex_mesh(2, 0.1, seed=3)
    gN, w = shape_gradients(X, conn, 0)
    rng = np.random.default_rng(6)
    u = rng.uniform(-0.03, 0.03, size=X.size)
    rp, ci = oracle.pattern(X.shape[0], conn)
    r, vals, bad = oracle.assemble(m, X.shape[0], conn, gN, w, u, rp, ci)
    assert bad == -1
    h = 1e-6
    for i in rng.choice(u.size, 6, replace=False):
        up, um = u.copy(), u.copy()
        up[i] += h
        um[i] -= h
        fd = (oracle.energy(m, conn, gN, w, up) - oracle.energy(m, conn, gN, w, um)) / (2 * h)
        assert abs(fd - r[i]) <= 1e-7 * max(1e-3, np.abs(r).max())


# ---- ICKAN -----------------------------------------------------------------------------
def test_ickan_linear_spline_closed_form():
    """Control points on a line reproduce it exactly (B-spline partition of unity and
    linear precision): N = sum_j w_j (a_j + b_j k_j) for a one-layer ICKAN, inside and
    outside the knot interval (linear continuation), so g = w b and H = 0."""
    nb, k = 7, 3
    xmin, xmax = -1.0, 1.0
    h = (xmax - xmin) / (nb - k)
    # Greville abscissae of uniform cubic knots: xi_i = xmin + (i - 1) h
    xi = xmin + (np.arange(nb) - 1.0) * h
    a = np.array([0.3, -0.1, 0.2])
    b = np.array([1.5, 0.5, 2.0])
    c = np.stack([a[j] + b[j] * xi for j in range(3)])
    w = np.array([0.7, 1.1, 0.4])
    m = dict(network="ickan", kinematics="standard", width=8, n_hidden=1, W1=None, W=None, b=None, a=None,
             skip_out=None, skip_hidden=None, kan_width=np.array([3, 1], np.int32), kan_nb=nb, kan_k=k,
             kan_grid=np.array([[xmin, xmax]]), kan_w=w, kan_c=c, kappa=0.0, ref_shift=0.0)
    for K in ([0.1, -0.3, 0.7], [1.4, -1.8, 0.0]):
        N, g, H = oracle.ncm_eval(m, np.array(K))
        assert abs(N - np.sum(w * (a + b * np.array(K)))) < 1e-14
        assert np.allclose(g, w * b, rtol=0, atol=1e-14) and np.abs(H).max() < 1e-13


def test_ickan_convex_in_inputs():
    """Monotone convex splines with positive weights: H positive semi-definite (App. B.3)."""
    m = ickan_params()
    rng = np.random.default_rng(3)
    for _ in range(20):
        _, g, H = oracle.ncm_eval(m, rng.uniform(-0.8, 0.8, 3))
        assert np.linalg.eigvalsh(H).min() >= -1e-14 and (g >= 0).all()


# ---- anisotropic I4 / I5 -----------------------------------------------------------------
def test_anisotropic_invariants_values():
    """I4 = A0.C A0 and I5 = A0.C^2 A0 (App. A.2.1) on closed forms: a stretch lambda along A0
    gives I4 = lambda^2, I5 = lambda^4; a rotation leaves both at 1 (k4 = k5 = 0)."""
    a0 = np.array([0.6, 0.8, 0.0])
    m = anisotropic(cann_params(3, seed=1, n_in=5), a0)
    lam = 1.3
    F = np.eye(3) + (lam - 1.0) * np.outer(a0, a0)
    k5 = np.array([np.trace(F.T @ F) - 3.0, 0.0, np.linalg.det(F) - 1.0, lam ** 2 - 1.0, lam ** 4 - 1.0])
    C = F.T @ F
    k5[1] = 0.5 * (np.trace(C) ** 2 - np.trace(C @ C)) - 3.0
    _, g_ref, _ = oracle.ncm_eval_n(m, k5)
    o = oracle.material_point(dict(m, kappa=0.0), F)
    # S from the definition: S = 2 sum_m g_m dK_m/dC, dI4/dC = A0 A0, dI5/dC = A0 (C A0) + (C A0) A0
    Ci = np.linalg.inv(C)
    h = [np.eye(3), np.trace(C) * np.eye(3) - C, 0.5 * np.linalg.det(F) * Ci, np.outer(a0, a0),
         np.outer(a0, C @ a0) + np.outer(C @ a0, a0)]
    S = 2 * sum(g_ref[i] * h[i] for i in range(5))
    assert np.abs(o["S"] - S).max() < 1e-13 * np.abs(S).max()
    Q, _ = np.linalg.qr(np.random.default_rng(2).normal(size=(3, 3)))
    Q *= np.sign(np.linalg.det(Q))
    o = oracle.material_point(dict(m, kappa=0.0), Q)
    assert np.abs(o["k"]).max() < 1e-14


@pytest.mark.parametrize("bad", ["gt_on_5_inputs", "icnn_skips_on_5_inputs", "unknown_network"])
def test_unsupported_network_kinematics_raise(bad):
    """The checker fails loudly: a network / kinematics combination the inner network cannot
    evaluate raises (material point, energy and assembly) instead of using uninitialised
    derivatives."""
    if bad == "gt_on_5_inputs":
        m = anisotropic(gent_thomas_params())
    elif bad == "icnn_skips_on_5_inputs":
        m = anisotropic(ncm_weights(8, 2, n_in=5))
        m["skip_hidden"] = np.zeros((1, 8, 3))
    else:
        m = dict(gent_thomas_params(), network=7)
    F = I3 + 0.05 * np.arange(9).reshape(3, 3) / 9
    with pytest.raises(oracle.OracleError):
        oracle.material_point(m, F)
    X, conn = hex_mesh(1)
    gN, w = shape_gradients(X, conn, 0)
    u = np.zeros(X.size)
    with pytest.raises(oracle.OracleError):
        oracle.energy(m, conn, gN, w, u)
    rp, ci = oracle.pattern(X.shape[0], conn)
    for mode in (0, 1):
        with pytest.raises(oracle.OracleError, match="inner network"):
            oracle.assemble(m, X.shape[0], conn, gN, w, u, rp, ci, mode=mode)



def test_two_vector_invariants_closed_form():
    """Eq. standard-inv-II for i != j on a closed form: the simple shear F = I + gamma
    e1 (x) e2 with A0 = e1, A1 = e2 gives C = [[1, g, 0], [g, 1 + g^2, 0], [0, 0, 1]], so
    I4,01 = C_12 = gamma and I5,01 = (C^2)_12 = 2 gamma + gamma^3 (and I4,00 = 1, I5,00 = 1 +
    gamma^2, I4,11 = 1 + gamma^2, I5,11 = gamma^2 + (1 + gamma^2)^2); S from the definition
    S = 2 sum_m g_m dK_m/dC with dI4,ij/dC = sym(A_i (x) A_j), dI5,ij/dC = sym(A_i (x) C A_j +
    C A_i (x) A_j)."""
    e1, e2 = np.array([1.0, 0, 0]), np.array([0, 1.0, 0])
    m = anisotropic(cann_params(3, seed=10, n_in=9), e1, e2)
    gam = 0.3
    F = np.eye(3) + gam * np.outer(e1, e2)
    C = F.T @ F
    C2 = C @ C
    k = np.array([np.trace(C) - 3.0, 0.5 * (np.trace(C) ** 2 - np.trace(C2)) - 3.0, np.linalg.det(F) - 1.0,
                  0.0, gam ** 2, gam, 2 * gam + gam ** 3, gam ** 2, gam ** 2 + (1 + gam ** 2) ** 2 - 1.0])
    assert abs(C[0, 1] - gam) < 1e-15 and abs(C2[0, 1] - (2 * gam + gam ** 3)) < 1e-15
    _, g_ref, _ = oracle.ncm_eval_n(m, k)
    o = oracle.material_point(dict(m, kappa=0.0), F)
    sym = lambda X: 0.5 * (X + X.T)
    Ci = np.linalg.inv(C)
    h = [np.eye(3), np.trace(C) * np.eye(3) - C, 0.5 * np.linalg.det(F) * Ci]
    for a, b in ((e1, e1), (e1, e2), (e2, e2)):
        h += [sym(np.outer(a, b)), sym(np.outer(a, C @ b) + np.outer(C @ a, b))]
    S = 2 * sum(g_ref[i] * h[i] for i in range(9))
    assert np.abs(o["S"] - S).max() < 1e-13 * np.abs(S).max()
    # objectivity: a rotation leaves every input at 0
    Q, _ = np.linalg.qr(np.random.default_rng(3).normal(size=(3, 3)))
    Q *= np.sign(np.linalg.det(Q))
    assert np.abs(oracle.material_point(dict(m, kappa=0.0), Q)["k"]).max() < 1e-14


def test_two_vectors_reduce_to_one():
    """With A1 = A0 every pair repeats the single-vector invariants: a CANN whose branches on the
    01 and 11 inputs have zero output weights gives the one-vector model exactly."""
    m1 = anisotropic(cann_params(3, seed=11, n_in=5), A_FIBRE)
    m2 = anisotropic(cann_params(3, seed=11, n_in=9), A_FIBRE, A_FIBRE)
    for key in ("cann_f", "cann_w1", "cann_w2"):
        m2[key] = np.concatenate([m1[key], m1[key][3:5], m1[key][3:5]])
    m2["cann_w2"][5:] = 0.0
    F = I3 + 0.08 * np.random.default_rng(4).normal(size=(3, 3))
    o1, o2 = oracle.material_point(m1, F), oracle.material_point(m2, F)
    assert abs(o1["W"] - o2["W"]) < 1e-14 * abs(o1["W"])
    assert np.abs(o1["A"] - o2["A"]).max() < 1e-13 * np.abs(o1["A"]).max()
