"""GPU parity of the material-point batch call (the
paper's material point benchmarks PAPER.md:509-557): (Psi, tau, c) tables from
the fused kernel's network stages against the oracle's material point, batch /
point equivalence and the six loading paths of App. C
(PAPER.md:1092-1127)."""
import numpy as np
import pytest

import oracle
from synth.gen import A_FIBRE, A_SHEET, anisotropic, cann_params, gent_thomas_params, ickan_params, ncm_weights
from tests.test_oracle_material import rand_F
from tests.test_oracle_variants import isochoric_icnn

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

VOIGT = [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)]
PAIRS = [(v, w) for v in range(6) for w in range(v, 6)]


def spatial(o, F):
    """tau = F S F^T, c_ijkl = F_iI F_jJ F_kK F_lL CC_IJKL (App. A.1 push-forward), Voigt-packed."""
    tau = F @ o["S"] @ F.T
    c = np.einsum("iI,jJ,kK,lL,IJKL->ijkl", F, F, F, F, o["CC"])
    return (np.array([tau[i, j] for i, j in VOIGT]),
            np.array([c[VOIGT[v][0], VOIGT[v][1], VOIGT[w][0], VOIGT[w][1]] for v, w in PAIRS]))


@pytest.fixture(scope="module")
def pc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_00884_b200 as pc
    return pc


MODELS = {
    "icnn_64x3": lambda: ncm_weights(64, 3, 0.3, 1, 10.0),
    "icnn_16x1": lambda: ncm_weights(16, 1, 0.3, 2, 10.0),
    "icnn_128x3": lambda: ncm_weights(128, 3, 0.3, 5, 10.0),  # forward sweep, L = 3
    "icnn_128x2": lambda: ncm_weights(128, 2, 0.3, 6, 10.0),  # forward sweep, L = 2
    "icnn_iso_16x2": isochoric_icnn,
    "cann": lambda: cann_params(4, seed=3),
    "gent_thomas": gent_thomas_params,
    "ickan": lambda: ickan_params(),
    "cann_anisotropic": lambda: anisotropic(cann_params(4, seed=6, n_in=5)),
    "icnn_anisotropic_32x2": lambda: anisotropic(ncm_weights(32, 2, 0.3, 15, 10.0, n_in=5)),
    "cann_two_vectors": lambda: anisotropic(cann_params(3, seed=8, n_in=9), A_FIBRE, A_SHEET),
    "icnn_isochoric_anisotropic_32x2": lambda: anisotropic(ncm_weights(32, 2, 0.3, 23, 10.0, n_in=5), isochoric=True),
    # (seed 6: every -ln(1 - w1 x) branch stays inside its domain x < 1/w1 at the 53 random F below;
    # seeds 21 / 24 leave it at one point and both sides return NaN there)
    "cann_isochoric_two_vectors": lambda: anisotropic(cann_params(3, seed=6, n_in=9), A_FIBRE, A_SHEET,
                                                      isochoric=True),
}


@pytest.mark.parametrize("name", sorted(MODELS))
def test_material_eval_matches_oracle(pc, name):
    ncm = MODELS[name]()
    lib = pc.Commet(None, ncm)
    rng = np.random.default_rng(4)
    n = 53  # several batches and a ragged tail
    F = np.stack([rand_F(rng) for _ in range(n)])
    W, tau, c = lib.material_eval(torch.from_numpy(F).cuda())
    assert lib.check() == -1
    W, tau, c = W.cpu().numpy(), tau.cpu().numpy(), c.cpu().numpy()
    Wo, to, co = np.zeros(n), np.zeros((n, 6)), np.zeros((n, 21))
    for p in range(n):
        o = oracle.material_point(ncm, F[p])
        Wo[p] = o["W"]
        to[p], co[p] = spatial(o, F[p])
    assert np.abs(W - Wo).max() <= 1e-12 * np.abs(Wo).max()
    assert np.abs(tau - to).max() <= 1e-12 * np.abs(to).max()
    assert np.abs(c - co).max() <= 1e-12 * np.abs(co).max()


def test_batch_point_equivalence_bitwise(pc):
    ncm = MODELS["icnn_64x3"]()
    lib = pc.Commet(None, ncm)
    rng = np.random.default_rng(9)
    F = torch.from_numpy(np.stack([rand_F(rng) for _ in range(1000)])).cuda()
    Wb, tb, cb = lib.material_eval(F)
    for n in (1, 7, 64):
        for s0 in (0, 333):
            W, t, c = lib.material_eval(F[s0:s0 + n])
            assert torch.equal(W, Wb[s0:s0 + n]) and torch.equal(t, tb[s0:s0 + n]) and torch.equal(c, cb[s0:s0 + n])


def test_loading_paths_gent_thomas(pc):
    """App. C paths; Gent-Thomas Psi in closed form along each (0.5(Ibar1-3) + ln(Ibar2/3) + (J-1)^2)."""
    lib = pc.Commet(None, gent_thomas_params())
    g = np.linspace(0.0, 0.5, 11)
    paths = {
        "UT": lambda x: np.diag([1 + x, 1, 1]), "UC": lambda x: np.diag([1 / (1 + x), 1, 1]),
        "BT": lambda x: np.diag([1 + x, 1 + x, 1]), "BC": lambda x: np.diag([1 / (1 + x), 1 / (1 + x), 1]),
        "SS": lambda x: np.array([[1, x, 0], [0, 1, 0], [0, 0, 1.0]]), "PS": lambda x: np.diag([1 + x, 1 / (1 + x), 1]),
    }
    for name, Fp in paths.items():
        F = np.stack([Fp(x) for x in g]).astype(np.float64)
        W, _, _ = lib.material_eval(torch.from_numpy(F).cuda(), want_c=False)
        for p in range(g.size):
            C = F[p].T @ F[p]
            J = np.linalg.det(F[p])
            I1 = np.trace(C)
            I2 = 0.5 * (I1 ** 2 - np.trace(C @ C))
            ref = 0.5 * (J ** (-2 / 3) * I1 - 3) + np.log(J ** (-4 / 3) * I2 / 3) + (J - 1) ** 2
            assert abs(W[p].item() - ref) <= 1e-13 * max(1.0, abs(ref)), (name, g[p])
    assert W[0].item() == 0.0


def test_material_domain_error_index(pc):
    lib = pc.Commet(None, MODELS["icnn_16x1"]())
    F = np.tile(np.eye(3), (40, 1, 1))
    F[17] = np.diag([1.0, 1.0, -0.5])
    F[29] = np.diag([-1.0, 1.0, 1.0])
    lib.material_eval(torch.from_numpy(F).cuda())
    assert lib.check() == 17
