"""GPU parity of the Newton-Raphson path through the C
ABI: symmetric Dirichlet elimination (bit-exact), CG-Jacobi against a direct
solve, the material-point NCM call and the stress-free normalisation against
the oracle, max tr C, and whole Newton load steps against oracle/newton.py."""
import numpy as np
import pytest
import scipy.optimize as so
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
from oracle import newton as on
from synth import twist
from synth.gen import make_config

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_00884_b200 as pc
    return pc


def _ctx(pc, mesh, ncm):
    return pc.Commet(dict(elem_type=mesh["elem_type"], n_nodes=mesh["n_nodes"], conn=mesh["conn"],
                          gradN=mesh["gradN"], qp_w=mesh["qp_w"]), ncm)


def _twist_setup(pc, n):
    mesh = twist.twist_mesh(n)
    ncm = twist.stable_ncm()
    lib = _ctx(pc, mesh, ncm)
    s0 = lib.normalize_reference()
    ncm["ref_shift"] = on.reference_shift(ncm)
    dofs, _, _ = twist.twist_bc(mesh["X"])
    lib.set_dirichlet(dofs)
    return mesh, ncm, lib, dofs, s0


def test_normalize_reference_matches_oracle(pc):
    mesh, ncm, lib, dofs, s0 = _twist_setup(pc, 2)
    assert abs(s0 - ncm["ref_shift"]) <= 1e-13 * abs(ncm["ref_shift"])


def test_ncm_eval_matches_oracle(pc):
    cfg = make_config("c2", n=2)
    lib = pc.from_config(cfg)
    rng = np.random.default_rng(4)
    k = rng.uniform(-0.3, 0.3, size=(37, 3))
    g, H = lib.ncm_eval(torch.from_numpy(k).cuda())
    g, H = g.cpu().numpy(), H.cpu().numpy()
    for i in range(k.shape[0]):
        _, go, Ho = oracle.ncm_eval(dict(cfg["ncm"], kappa=0.0), k[i])
        assert np.abs(g[i] - go).max() <= 1e-13 * np.abs(go).max()
        Hu = Ho[np.triu_indices(3)]
        assert np.abs(H[i] - Hu).max() <= 1e-13 * np.abs(Hu).max()


def test_max_trace_C_matches_oracle(pc):
    cfg = make_config("c2", n=6)
    lib = pc.from_config(cfg)
    lib.assemble(torch.from_numpy(cfg["u"]).cuda())
    ref = on.max_trace_C(cfg, cfg["u"])
    assert abs(lib.max_trace_C() - ref) <= 1e-14 * ref


def test_dirichlet_elimination_bit_exact(pc):
    cfg = make_config("c2", n=5)
    lib = pc.from_config(cfg)
    r, v = lib.assemble(torch.from_numpy(cfg["u"]).cuda())
    r0, v0 = r.cpu().numpy(), v.cpu().numpy()
    rng = np.random.default_rng(9)
    dofs = np.unique(rng.integers(0, 3 * cfg["n_nodes"], size=60))
    lib.set_dirichlet(dofs)
    lib.apply_dirichlet(r, v)
    rp, ci = lib.pattern()
    mask = np.zeros(3 * cfg["n_nodes"], bool)
    mask[dofs] = True
    ve, re = on.eliminate(rp, ci, v0, r0, mask)
    assert np.array_equal(v.cpu().numpy(), ve) and np.array_equal(r.cpu().numpy(), re)


def test_cg_jacobi_matches_direct_solve(pc):
    mesh, ncm, lib, dofs, _ = _twist_setup(pc, 5)
    rp, ci = oracle.pattern(mesh["n_nodes"], mesh["conn"])
    u = np.zeros(3 * mesh["n_nodes"])
    for s in (1, 2):  # a deformed state: two oracle load steps of 10
        u, _, ok = on.newton_step(ncm, mesh, rp, ci, u, dofs, twist.twist_values(mesh["X"], dofs, s / 10))
        assert ok
    r, v = lib.assemble(torch.from_numpy(u).cuda())
    lib.apply_dirichlet(r, v)
    x, it, rel = lib.cg_jacobi(v, r, rtol=1e-12)
    n = r.numel()
    K = sp.csr_matrix((v.cpu().numpy(), ci, rp), shape=(n, n))
    xd = spla.spsolve(K.tocsc(), r.cpu().numpy())
    assert rel <= 1e-12
    assert np.linalg.norm(x.cpu().numpy() - xd) <= 1e-9 * np.linalg.norm(xd)
    _, it_o = on.cg_jacobi(K, r.cpu().numpy(), rtol=1e-12)
    assert abs(it - it_o) <= 3, (it, it_o)


def test_block_jacobi_cg_matches_direct_solve(pc):
    """3x3 block-Jacobi PCG on an eliminated twist tangent: the direct solution, and the
    oracle's block PCG iteration count (fewer iterations than scalar Jacobi)."""
    mesh, ncm, lib, dofs, _ = _twist_setup(pc, 5)
    rp, ci = oracle.pattern(mesh["n_nodes"], mesh["conn"])
    u = np.zeros(3 * mesh["n_nodes"])
    for s in (1, 2):
        u, _, ok = on.newton_step(ncm, mesh, rp, ci, u, dofs, twist.twist_values(mesh["X"], dofs, s / 10))
        assert ok
    r, v = lib.assemble(torch.from_numpy(u).cuda())
    lib.apply_dirichlet(r, v)
    _, it_j, _ = lib.cg_jacobi(v, r, rtol=1e-12)
    lib.set_preconditioner("block_jacobi")
    x, it, rel = lib.cg_jacobi(v, r, rtol=1e-12)
    n = r.numel()
    K = sp.csr_matrix((v.cpu().numpy(), ci, rp), shape=(n, n))
    xd = spla.spsolve(K.tocsc(), r.cpu().numpy())
    assert rel <= 1e-12
    assert np.linalg.norm(x.cpu().numpy() - xd) <= 1e-9 * np.linalg.norm(xd)
    _, it_o = on.cg_jacobi(K, r.cpu().numpy(), rtol=1e-12, block=True)
    assert abs(it - it_o) <= 3, (it, it_o)
    assert it < it_j, (it, it_j)
    with pytest.raises(pc.CommetError):  # the C ABI refuses an unknown kind
        pc._check(pc._lib.commet_set_preconditioner(lib.ctx, 7), lib.ctx)


@pytest.mark.parametrize("kind", ["jacobi", "block_jacobi"])
def test_cg_refuses_indefinite_preconditioner(pc, kind):
    """A non-positive diagonal entry (Jacobi) / a 3x3 diagonal block that is not positive
    definite (block Jacobi) is a domain error naming the first offending row."""
    cfg = make_config("c2", n=3)
    lib = pc.from_config(cfg)
    r, v = lib.assemble(torch.from_numpy(cfg["u"]).cuda())
    rp, ci = lib.pattern()
    row = 3 * 5 + 1  # node 5, component 1
    d = rp[row] + int(np.nonzero(ci[rp[row]:rp[row + 1]] == row)[0][0])
    v[d] = -abs(float(v[d]))
    lib.set_preconditioner(kind)
    with pytest.raises(pc.CommetError, match=str(row if kind == "jacobi" else 15)):
        lib.cg_jacobi(v, r, rtol=1e-8)


def test_block_jacobi_newton_twist_matches_oracle(pc):
    n, steps = 3, 5
    mesh, ncm, lib, dofs, _ = _twist_setup(pc, n)
    lib.set_preconditioner("block_jacobi")
    rp, ci = oracle.pattern(mesh["n_nodes"], mesh["conn"])
    uo = np.zeros(3 * mesh["n_nodes"])
    ug = torch.zeros(3 * mesh["n_nodes"], dtype=torch.float64, device="cuda")
    for s in range(1, steps + 1):
        vals = twist.twist_values(mesh["X"], dofs, s / steps)
        uo, norms, ok = on.newton_step(ncm, mesh, rp, ci, uo, dofs, vals, atol=1e-11, rtol=1e-12)
        rep = lib.newton_step(ug, vals, atol=1e-11, rtol=1e-12, cg_rtol=1e-13)
        assert ok and rep["converged"], (s, norms, rep["res_norm"])
        d = np.abs(ug.cpu().numpy() - uo).max() / np.abs(uo).max()
        assert d <= 1e-9, (s, d)


def test_newton_zero_load(pc):
    mesh, ncm, lib, dofs, _ = _twist_setup(pc, 3)
    u = torch.zeros(3 * mesh["n_nodes"], dtype=torch.float64, device="cuda")
    rep = lib.newton_step(u, np.zeros(dofs.size))
    assert rep["converged"] and rep["iters"] == 0 and rep["res_norm"][0] < 1e-13
    assert not u.any()


@pytest.mark.parametrize("precond", ["jacobi", "block_jacobi"])
def test_newton_uniaxial_closed_form(pc, precond):
    """Partially constrained nodes (one or two components fixed): the block-Jacobi blocks mix
    eliminated unit rows with free ones and must stay SPD."""
    from tests.test_oracle_newton import mooney_rivlin_ncm, mr_lateral_stress
    c1, c2, kappa, lam = 0.7, 0.2, 3.0, 1.6
    mesh, dofs, vals = twist.uniaxial_problem(lam)
    lib = _ctx(pc, mesh, mooney_rivlin_ncm(c1, c2, kappa))
    lib.set_preconditioner(precond)
    lib.set_dirichlet(dofs)
    u = torch.zeros(3 * mesh["n_nodes"], dtype=torch.float64, device="cuda")
    rep = lib.newton_step(u, vals, atol=1e-13, rtol=1e-14, cg_rtol=1e-14)
    assert rep["converged"]
    mu = so.brentq(lambda m: mr_lateral_stress(m, lam, c1, c2, kappa), 0.3, 1.7, xtol=1e-15)
    X = mesh["X"]
    exact = np.stack([(mu - 1) * X[:, 0], (mu - 1) * X[:, 1], (lam - 1) * X[:, 2]], axis=1).reshape(-1)
    assert np.abs(u.cpu().numpy() - exact).max() <= 1e-10


def test_newton_twist_matches_oracle(pc):
    n, steps = 4, 10
    mesh, ncm, lib, dofs, _ = _twist_setup(pc, n)
    rp, ci = oracle.pattern(mesh["n_nodes"], mesh["conn"])
    uo = np.zeros(3 * mesh["n_nodes"])
    ug = torch.zeros(3 * mesh["n_nodes"], dtype=torch.float64, device="cuda")
    for s in range(1, steps + 1):
        vals = twist.twist_values(mesh["X"], dofs, s / steps)
        uo, norms, ok = on.newton_step(ncm, mesh, rp, ci, uo, dofs, vals, atol=1e-11, rtol=1e-12)
        rep = lib.newton_step(ug, vals, atol=1e-11, rtol=1e-12, cg_rtol=1e-13)
        assert ok and rep["converged"], (s, norms, rep["res_norm"])
        assert rep["iters"] == len(norms) - 1, (s, norms, rep["res_norm"])
        d = np.abs(ug.cpu().numpy() - uo).max() / np.abs(uo).max()
        assert d <= 1e-9, (s, d)
    assert abs(rep["max_trC"] - on.max_trace_C(mesh, uo)) <= 1e-8 * rep["max_trC"]


def test_newton_solve_step_halving(pc):
    """Two load steps for the whole twist: the first fails (inverted elements) and is
    halved; the converged end state equals the oracle's 10-step solution."""
    n = 4
    mesh, ncm, lib, dofs, _ = _twist_setup(pc, n)
    rp, ci = oracle.pattern(mesh["n_nodes"], mesh["conn"])
    uo = np.zeros(3 * mesh["n_nodes"])
    for s in range(1, 11):
        uo, norms, ok = on.newton_step(ncm, mesh, rp, ci, uo, dofs, twist.twist_values(mesh["X"], dofs, s / 10),
                                       atol=1e-11, rtol=1e-12)
        assert ok
    ug = torch.zeros(3 * mesh["n_nodes"], dtype=torch.float64, device="cuda")
    reps = lib.newton_solve(ug, lambda t: twist.twist_values(mesh["X"], dofs, t), n_steps=1, max_halvings=6,
                            atol=1e-11, rtol=1e-12, cg_rtol=1e-13)
    assert abs(reps[-1]["t"] - 1.0) < 1e-12 and reps[-1]["converged"]
    assert any("error" in r or not r["converged"] for r in reps)  # at least one halving happened
    d = np.abs(ug.cpu().numpy() - uo).max() / np.abs(uo).max()
    assert d <= 1e-8, d
