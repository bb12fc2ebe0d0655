"""Edge cases of the CUDA path through the C ABI: an element set that is empty,
a single element and ragged batches (element counts that do not fill the per-CTA
batch of 2 hex8 / 4 tet10 elements), the stress-free reference (u = 0 gives r = 0
after the R11 normalisation), and an empty material-point batch."""
import numpy as np
import pytest

import oracle
from synth import gen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_00884_b200 as pc
    return pc


def _mesh(et, n, n_el=None, seed=3):
    X, conn = gen.hex_mesh(n, 0.1, seed) if et == gen.HEX8 else gen.tet10_mesh(n, 0.1, seed)
    if n_el is not None:
        conn = np.ascontiguousarray(conn[:n_el])
    gN, w = gen.shape_gradients(X, conn, et)
    u = gen.smooth_field(X, 0.05, np.random.default_rng(seed)).reshape(-1)
    return dict(elem_type=et, n_nodes=X.shape[0], conn=conn, gradN=gN, qp_w=w), u


def test_empty_element_set(pc):
    mesh, u = _mesh(gen.HEX8, 2, n_el=0)
    mesh["gradN"] = np.zeros((0, 8, 8, 3))
    mesh["qp_w"] = np.zeros((0, 8))
    lib = pc.Commet(mesh, gen.ncm_weights(16, 2))
    assert lib.nnz == 0
    r, v = lib.assemble(torch.from_numpy(u).cuda())
    assert lib.check() == -1 and not r.any() and v.numel() == 0


@pytest.mark.parametrize("et,n,n_el", [(gen.HEX8, 2, 1), (gen.HEX8, 3, 7), (gen.TET10, 1, 1), (gen.TET10, 2, 5),
                                        (gen.TET10, 2, 47)])
@pytest.mark.parametrize("w,L", [(16, 2), (64, 3), (128, 3)])
def test_single_and_ragged(pc, et, n, n_el, w, L):
    mesh, u = _mesh(et, n, n_el)
    ncm = gen.ncm_weights(w, L, 0.3, 9, 10.0)
    lib = pc.Commet(mesh, ncm)
    r, v = lib.assemble(torch.from_numpy(u).cuda())
    assert lib.check() == -1
    rp, ci = lib.pattern()
    orp, oci = oracle.pattern(mesh["n_nodes"], mesh["conn"])
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    ro, vo, bad = oracle.assemble(ncm, mesh["n_nodes"], mesh["conn"], mesh["gradN"], mesh["qp_w"], u, orp, oci)
    assert np.abs(r.cpu().numpy() - ro).max() <= 1e-10 * np.abs(ro).max()
    assert np.abs(v.cpu().numpy() - vo).max() <= 1e-10 * np.abs(vo).max()


@pytest.mark.parametrize("et", [gen.HEX8, gen.TET10])
def test_stress_free_reference(pc, et):
    """u = 0 with s0 from commet_normalize_reference: r = 0 to round-off (reading R11),
    while the tangent is the (non-zero) linearised stiffness."""
    mesh, _ = _mesh(et, 2)
    lib = pc.Commet(mesh, gen.ncm_weights(32, 2, 0.3, 4, 10.0))
    lib.normalize_reference()
    r, v = lib.assemble(torch.zeros(3 * mesh["n_nodes"], dtype=torch.float64, device="cuda"))
    assert np.abs(r.cpu().numpy()).max() <= 1e-13 * np.abs(v.cpu().numpy()).max()
    assert np.abs(v.cpu().numpy()).max() > 0


def test_empty_material_batch(pc):
    lib = pc.Commet(None, gen.ncm_weights(16, 2))
    W, tau, c = lib.material_eval(torch.zeros((0, 3, 3), dtype=torch.float64, device="cuda"))
    assert W.numel() == 0 and lib.check() == -1
