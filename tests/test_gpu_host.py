"""commet_assemble_host / commet_host_wait (the end-to-end call on host buffers, include/commet.h):
the host outputs equal the device call's outputs bit for bit (same kernels, same colour order),
for a chain of calls with different u (the two staging sets alternate, so call s must not see
call s-1's or s-2's u), on pinned and on pageable host memory, and against the oracle
(Eq. r-quad / k-quad).  Argument errors come back as COMMET_ERR_ARG."""
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


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_host_call_equals_device_call(pc, name, pinned):
    cfg = gen.make_config(name)
    lib = pc.from_config(cfg, device=0)
    rng = np.random.default_rng(11)
    us = [cfg["u"] * s + 1e-3 * rng.standard_normal(cfg["u"].shape) for s in (1.0, 0.5, 1.5, 0.8, 1.2)]
    outs = []
    r_host = torch.empty(lib.n_rows, dtype=torch.float64)
    v_host = torch.empty(lib.nnz, dtype=torch.float64)
    if pinned:
        r_host, v_host = r_host.pin_memory(), v_host.pin_memory()
    for uu in us:
        u_host = torch.from_numpy(uu)
        u_host = u_host.pin_memory() if pinned else u_host
        lib.assemble_host(u_host, r_host, v_host)
        lib.host_wait()
        outs.append((r_host.clone(), v_host.clone()))
    assert lib.check() == -1
    for uu, (rh, vh) in zip(us, outs):
        r, v = lib.assemble(torch.from_numpy(uu).cuda())
        torch.cuda.synchronize()
        assert torch.equal(rh, r.cpu()) and torch.equal(vh, v.cpu())
    # the last one against the oracle
    rp, ci = lib.pattern()
    ro, vo, bad = oracle.assemble(cfg["ncm"], cfg["n_nodes"], cfg["conn"], cfg["gradN"], cfg["qp_w"],
                                  us[-1], rp, ci)
    rh, vh = outs[-1]
    assert np.abs(rh.numpy() - ro).max() <= 1e-10 * np.abs(ro).max()
    assert np.abs(vh.numpy() - vo).max() <= 1e-10 * np.abs(vo).max()


def test_host_calls_pipelined(pc):
    """Several calls in flight before one wait (the bench's pattern): the outputs are the last call's."""
    cfg = gen.make_config("c2")
    lib = pc.from_config(cfg, device=0)
    u_host = torch.from_numpy(cfg["u"]).pin_memory()
    r_host = torch.empty(lib.n_rows, dtype=torch.float64).pin_memory()
    v_host = torch.empty(lib.nnz, dtype=torch.float64).pin_memory()
    st = torch.cuda.current_stream()
    for _ in range(4):
        lib.assemble_host(u_host, r_host, v_host, st)
    lib.host_wait(st)
    st.synchronize()
    r, v = lib.assemble(u_host.cuda())
    torch.cuda.synchronize()
    assert torch.equal(r_host, r.cpu()) and torch.equal(v_host, v.cpu())


def test_host_call_argument_errors(pc):
    cfg = gen.make_config("c1")
    lib = pc.from_config(cfg, device=0)
    lib.host_wait()  # no call yet: OK
    u_host = torch.from_numpy(cfg["u"])
    r_host = torch.empty(lib.n_rows, dtype=torch.float64)
    with pytest.raises(ValueError):
        lib.assemble_host(u_host, r_host, torch.empty(lib.nnz - 1, dtype=torch.float64))
    with pytest.raises(TypeError):
        lib.assemble_host(u_host.cuda(), r_host, torch.empty(lib.nnz, dtype=torch.float64))
    L = pc._lib
    assert L.commet_assemble_host(lib.ctx, None, r_host.data_ptr(), None, None) == pc.COMMET_ERR_ARG
    mat = pc.Commet(None, gen.ncm_weights(16, 2))
    assert L.commet_assemble_host(mat.ctx, u_host.data_ptr(), r_host.data_ptr(), r_host.data_ptr(),
                                  None) == pc.COMMET_ERR_ARG
    assert b"material" in L.commet_last_error(mat.ctx)


def test_destroy_with_copies_in_flight(pc):
    """commet_destroy right after commet_assemble_host (no host_wait): the staging sets are freed only
    after their copies finish, and a new ctx on the same device assembles correctly."""
    cfg = gen.make_config("c2")
    u_host = torch.from_numpy(cfg["u"]).pin_memory()
    for _ in range(2):
        lib = pc.from_config(cfg, device=0)
        r_host = torch.empty(lib.n_rows, dtype=torch.float64).pin_memory()
        v_host = torch.empty(lib.nnz, dtype=torch.float64).pin_memory()
        for _ in range(3):
            lib.assemble_host(u_host, r_host, v_host)
        lib.close()
    torch.cuda.synchronize()
    lib = pc.from_config(cfg, device=0)
    r_host = torch.empty(lib.n_rows, dtype=torch.float64).pin_memory()
    v_host = torch.empty(lib.nnz, dtype=torch.float64).pin_memory()
    lib.assemble_host(u_host, r_host, v_host)
    lib.host_wait()
    r, v = lib.assemble(u_host.cuda())
    torch.cuda.synchronize()
    assert torch.equal(r_host, r.cpu()) and torch.equal(v_host, v.cpu())
