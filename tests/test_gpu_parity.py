"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle,
element by element, on the same seeded inputs.  Bar (BASELINE north_star):
normwise relative error <= 1e-10 on residual and CSR values (R13),
CSR row_ptr / col_idx bit-exact."""
import numpy as np
import pytest

import oracle
from synth import gen

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def rel(g, o):
    return np.abs(g - o).max() / max(np.abs(o).max(), 1e-300)


def per_entry(g, o, floor=1e-6):
    """SURVEY R13's second number: max |g_i - o_i| / |o_i| over the entries with
    |o_i| >= floor * max|o| (entries that cancel to ~0 are excluded)."""
    a = np.abs(o)
    mask = a >= floor * a.max()
    return float((np.abs(g - o)[mask] / a[mask]).max()) if mask.any() else 0.0


def small_case(kind, n, w, L, skips=False, shift=False, jitter=0.1, amp=0.05, seed=3):
    et = gen.HEX8 if kind == "hex" else gen.TET10
    X, conn = gen.hex_mesh(n, jitter, seed) if kind == "hex" else gen.tet10_mesh(n, jitter, seed)
    gN, qw = gen.shape_gradients(X, conn, et)
    m = gen.ncm_weights(w, L, 0.3, seed + 1, 10.0)
    if skips:
        rng = np.random.default_rng(seed + 7)
        m["skip_out"] = rng.normal(0, 0.3, 3)
        m["skip_hidden"] = rng.normal(0, 0.3, (L - 1, w, 3))
    if shift:
        m["ref_shift"] = 0.123
    u = gen.smooth_field(X, amp, np.random.default_rng(seed + 2)).reshape(-1)
    return dict(elem_type=et, n_nodes=X.shape[0], conn=conn, gradN=gN, qp_w=qw, ncm=m, u=u, X=X)


def run_gpu(case, kernel=None, order=0):
    torch = _torch()
    import paper_2510_00884_b200 as pc
    lib = pc.from_config(case, scatter_order=order)
    if kernel is not None:
        lib.set_kernel(kernel)
    u = torch.from_numpy(case["u"]).cuda()
    r, v = lib.assemble(u)
    torch.cuda.synchronize()
    rp, ci = lib.pattern()
    return lib, r.cpu().numpy(), v.cpu().numpy(), rp, ci


def run_oracle(case):
    rp, ci = oracle.pattern(case["n_nodes"], case["conn"])
    r, v, bad = oracle.assemble(case["ncm"], case["n_nodes"], case["conn"], case["gradN"],
                                case["qp_w"], case["u"], rp, ci)
    return r, v, rp, ci, bad


CASES = [
    ("hex", 3, 8, 2, False, False),
    ("hex", 3, 16, 2, False, False),
    ("hex", 5, 32, 2, False, False),
    ("hex", 5, 64, 3, False, False),
    ("hex", 3, 128, 3, False, False),
    ("hex", 3, 64, 1, False, False),
    ("hex", 4, 64, 4, True, True),
    ("tet", 2, 16, 2, False, False),
    ("tet", 3, 64, 3, False, False),
    ("tet", 2, 128, 3, True, False),
    ("tet", 2, 32, 3, False, True),
    # w = 128: the forward sweep with L = 2 (the last layer right after layer 1), the three-pass
    # fallback at L = 4 and L = 1
    ("hex", 3, 128, 2, False, True),
    ("tet", 2, 128, 4, False, False),
    ("hex", 2, 128, 1, False, False),
]


@pytest.mark.parametrize("kind,n,w,L,skips,shift", CASES)
@pytest.mark.parametrize("kernel", [0, 1])
def test_parity_small(kind, n, w, L, skips, shift, kernel):
    case = small_case(kind, n, w, L, skips, shift)
    lib, r, v, rp, ci = run_gpu(case, kernel)
    ro, vo, orp, oci, bad = run_oracle(case)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    assert lib.check() == bad == -1
    assert rel(r, ro) <= TOL, rel(r, ro)
    assert rel(v, vo) <= TOL, rel(v, vo)


@pytest.mark.parametrize("kind,n,w,L,skips,shift", [CASES[3], CASES[8], CASES[6]])
def test_parity_element_order(kind, n, w, L, skips, shift):
    """COMMET_ORDER_ELEMENT: one launch, concurrent RED updates (non-deterministic
    summation order) -- same parity bar."""
    case = small_case(kind, n, w, L, skips, shift)
    lib, r, v, rp, ci = run_gpu(case, order=1)
    ro, vo, orp, oci, bad = run_oracle(case)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    assert lib.info()["n_colours"] == 1
    assert rel(r, ro) <= TOL and rel(v, vo) <= TOL, (rel(r, ro), rel(v, vo))


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_parity_configs(name):
    cfg = gen.make_config(name)
    lib, r, v, rp, ci = run_gpu(cfg)
    ro, vo, orp, oci, bad = run_oracle(cfg)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    assert rel(r, ro) <= TOL and rel(v, vo) <= TOL, (rel(r, ro), rel(v, vo))


def test_domain_flag_matches_oracle():
    case = small_case("hex", 2, 16, 2, jitter=0.0)
    case["u"] = case["u"].copy()
    case["u"][3 * 13] += 0.9
    lib, r, v, rp, ci = run_gpu(case)
    ro, vo, _, _, bad = run_oracle(case)
    assert bad >= 0 and lib.check() == bad
    assert rel(r, ro) <= TOL and rel(v, vo) <= TOL


def test_deterministic():
    case = small_case("hex", 4, 64, 3)
    _, r1, v1, _, _ = run_gpu(case)
    _, r2, v2, _, _ = run_gpu(case)
    assert np.array_equal(r1, r2) and np.array_equal(v1, v2)


@pytest.mark.parametrize("table_bits", [6, 8])
def test_activation_table_accuracy(table_bits):
    """The fused kernel's branch-free softplus/sigmoid (qp_math.cuh) against
    numpy's logaddexp / exp on a sweep of y, incl. the extremes -- both table sizes;
    the sigmoid-only form must equal the softplus+sigmoid one bit for bit."""
    torch = _torch()
    import paper_2510_00884_b200 as pc
    rng = np.random.default_rng(0)
    y = np.concatenate([np.linspace(-40, 40, 200001), rng.normal(0, 3, 100000), rng.uniform(-800, 800, 10000),
                        np.array([0.0, -0.0, 1e-300, -1e-300, 708.0, -708.0, 750.0, -750.0, 1e-8, -1e-8])])
    z, s = pc.activation(torch.from_numpy(y).cuda(), table_bits)
    z, s = z.cpu().numpy(), s.cpu().numpy()
    zr = np.logaddexp(0.0, y)
    sr = np.where(y >= 0, 1.0 / (1.0 + np.exp(-np.abs(y))), np.exp(-np.abs(y)) / (1.0 + np.exp(-np.abs(y))))
    mask = np.abs(y) < 700
    assert np.max(np.abs(z - zr)[mask] / np.maximum(zr[mask], 1e-300)) < 1e-15
    assert np.max(np.abs(s - sr)[mask] / np.maximum(sr[mask], 1e-300)) < 1e-15
    assert np.max(np.abs(z - zr)) < 1e-300 + 1e-15 * np.abs(zr).max()
    assert np.all(np.isfinite(z)) and np.all(np.isfinite(s))


@pytest.mark.parametrize("name,n,P", [("c1", 4, 2), ("c2", 8, 4), ("c4", 3, 3)])
def test_slabs_on_one_device(name, n, P):
    """The multi-GPU slab path on one device: P contexts (ranks) assemble their
    slabs; halo segments move between them with commet_halo_send/unpack (the
    same buffers and maps NCCL uses), no kernel waits on another.  The
    concatenated owned rows must equal the global oracle."""
    torch = _torch()
    import paper_2510_00884_b200 as pc
    g = gen.make_config(name, n=n)
    grp, gci = oracle.pattern(g["n_nodes"], g["conn"])
    gr, gv, _ = oracle.assemble(g["ncm"], g["n_nodes"], g["conn"], g["gradN"], g["qp_w"], g["u"], grp, gci)
    u = torch.from_numpy(g["u"]).cuda()
    libs, outs, parts = [], [], []
    for r in range(P):
        c = gen.slab_partition(name, P, r, n=n)
        lib = pc.Commet(c, c["ncm"])
        outs.append(lib.assemble(u))
        libs.append(lib)
        parts.append(c)
    torch.cuda.synchronize()
    for r in range(P):   # receivers unpack what their senders hold
        ns, nr = libs[r].halo_info()
        for k in range(nr):
            peer, nv, nres = libs[r].halo_recv(k)
            sender = libs[peer]
            for ks in range(sender.halo_info()[0]):
                dst, vp, snv, rp_, snr = sender.halo_send(ks)
                if dst == r:
                    assert (snv, snr) == (nv, nres)
                    libs[r].halo_unpack(k, vp, rp_, *outs[r])
    torch.cuda.synchronize()
    r_all = np.concatenate([o[0].cpu().numpy() for o in outs])
    v_all = np.concatenate([o[1].cpu().numpy() for o in outs])
    rp_all = [libs[r].pattern() for r in range(P)]
    ci_all = np.concatenate([x[1] for x in rp_all])
    assert np.array_equal(ci_all, gci)
    assert rel(r_all, gr) <= TOL and rel(v_all, gv) <= TOL, (rel(r_all, gr), rel(v_all, gv))


@pytest.mark.parametrize("name,n,P", [("c1", 4, 2), ("c2", 8, 4), ("c4", 3, 3)])
def test_slabs_peer_mode_on_one_device(name, n, P):
    """Peer mode (the fused interface reduction): each rank's kernels add their halo rows
    straight into the owner's output buffers through the owner's receive maps -- no halo
    buffers, no unpack.  P contexts on one device, outputs zeroed first, assembled one after
    the other (no kernel waits on another); the concatenated rows equal the global oracle."""
    torch = _torch()
    import paper_2510_00884_b200 as pc
    g = gen.make_config(name, n=n)
    grp, gci = oracle.pattern(g["n_nodes"], g["conn"])
    gr, gv, _ = oracle.assemble(g["ncm"], g["n_nodes"], g["conn"], g["gradN"], g["qp_w"], g["u"], grp, gci)
    u = torch.from_numpy(g["u"]).cuda()
    libs = [pc.Commet(c, c["ncm"]) for c in (gen.slab_partition(name, P, r, n=n) for r in range(P))]
    outs = [lib.alloc_outputs() for lib in libs]
    for r, lib in enumerate(libs):
        for k in range(lib.halo_info()[0]):
            owner = lib.halo_send(k)[0]
            maps = {}
            for kr in range(libs[owner].halo_info()[1]):
                sender, vm, rm = libs[owner].halo_recv_maps(kr)
                maps[sender] = (vm, rm)
            vm, rm = maps[r]
            lib.set_peer(k, outs[owner][0].data_ptr(), outs[owner][1].data_ptr(), vm, rm)
        lib.set_peer_mode(True)
    for lib, (res, val) in zip(libs, outs):
        lib.zero_outputs(res, val)
    for lib, (res, val) in zip(libs, outs):
        lib.assemble(u, res, val)
    torch.cuda.synchronize()
    r_all = np.concatenate([o[0].cpu().numpy() for o in outs])
    v_all = np.concatenate([o[1].cpu().numpy() for o in outs])
    ci_all = np.concatenate([lib.pattern()[1] for lib in libs])
    assert np.array_equal(ci_all, gci)
    assert rel(r_all, gr) <= TOL and rel(v_all, gv) <= TOL, (rel(r_all, gr), rel(v_all, gv))


def _elements_of(conn, a):
    return np.nonzero((conn == a).any(axis=1))[0]


def sampled_rows_check(name, n_samples=12, seed=0, ncm=None):
    """Full BASELINE size, the bench's launch configuration: the GPU's CSR rows of
    sampled nodes (interior, faces, edges, corners) against the oracle assembling
    only the elements that touch each node (those rows are then complete).
    ncm: another NCM on the config's mesh and displacement (the variants)."""
    torch = _torch()
    import paper_2510_00884_b200 as pc
    cfg = gen.make_config(name)
    if ncm is not None:
        cfg["ncm"] = ncm
    lib = pc.from_config(cfg)
    u = torch.from_numpy(cfg["u"]).cuda()
    r, v = lib.assemble(u)
    assert lib.check() == -1
    rp_d, ci_d = lib.pattern(device=True)
    rng = np.random.default_rng(seed)
    nn = cfg["n_nodes"]
    nodes = list(rng.choice(nn, n_samples, replace=False)) + [0, nn - 1, nn // 2]
    errs_v, errs_r, scale_v, scale_r = [], [], 0.0, 0.0
    for a in nodes:
        els = _elements_of(cfg["conn"], a)
        sub = np.ascontiguousarray(cfg["conn"][els])
        orp, oci = oracle.pattern(nn, sub, node_begin=a, node_end=a + 1)
        ro, vo, bad = oracle.assemble(cfg["ncm"], nn, sub, cfg["gradN"][els], cfg["qp_w"][els], cfg["u"], orp, oci,
                                      node_begin=a, node_end=a + 1, mode=0)
        assert bad == -1
        s0, s1 = int(rp_d[3 * a].item()), int(rp_d[3 * a + 3].item())
        assert np.array_equal(ci_d[s0:s1].cpu().numpy(), oci)
        gv = v[s0:s1].cpu().numpy()
        gr = r[3 * a:3 * a + 3].cpu().numpy()
        errs_v.append(np.abs(gv - vo).max())
        errs_r.append(np.abs(gr - ro).max())
        scale_v = max(scale_v, np.abs(vo).max())
        scale_r = max(scale_r, np.abs(ro).max())
    assert max(errs_v) <= TOL * scale_v, (max(errs_v), scale_v)
    assert max(errs_r) <= TOL * scale_r, (max(errs_r), scale_r)
    return max(errs_v) / scale_v, max(errs_r) / scale_r


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_parity_full_size_sampled(name):
    sampled_rows_check(name)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_parity_full_size(name):
    """Every output of the BASELINE-size c3 (64.7M nonzeros) and c4 (231.8M) assembly, in the
    bench's launch configuration (persistent grid, many batches per CTA and colour, register
    prefetch of the next batch) against the full oracle (OpenMP over colours): pattern bit-exact,
    residual and CSR values <= 1e-10 normwise; the per-entry relative error is reported."""
    torch = _torch()
    import paper_2510_00884_b200 as pc
    cfg = gen.make_config(name)
    lib = pc.from_config(cfg)
    u = torch.from_numpy(cfg["u"]).cuda()
    r, v = lib.assemble(u)
    assert lib.check() == -1
    rp, ci = lib.pattern()
    r, v = r.cpu().numpy(), v.cpu().numpy()
    del lib
    orp, oci = oracle.pattern(cfg["n_nodes"], cfg["conn"])
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    del rp, ci
    ro, vo, bad = oracle.assemble(cfg["ncm"], cfg["n_nodes"], cfg["conn"], cfg["gradN"], cfg["qp_w"], cfg["u"],
                                  orp, oci)
    assert bad == -1
    er, ev = rel(r, ro), rel(v, vo)
    pr, pv = per_entry(r, ro), per_entry(v, vo)
    print(f"{name} full: residual {er:.2e} normwise / {pr:.2e} per entry; CSR values {ev:.2e} / {pv:.2e} "
          f"({v.size} nonzeros)")
    assert er <= TOL and ev <= TOL, (er, ev)


def test_parity_c5_sampled():
    """c5: 4.09e9 nonzeros (> 2^31: int64 row starts), 256^3 hex8 -- sampled rows."""
    ev, er = sampled_rows_check("c5", n_samples=10)
    print(f"c5 sampled rows: values rel err {ev:.2e}, residual rel err {er:.2e}")


@pytest.mark.parametrize("variant", ["icnn_isochoric", "icnn_anisotropic", "cann_anisotropic", "ickan",
                                     "cann_two_vectors", "icnn_isochoric_anisotropic", "cann_isochoric_two_vectors"])
def test_parity_full_size_sampled_variants(variant):
    """The variants' instantiations at the c3 size (2.1M qp, the persistent grid of the bench):
    sampled complete rows against the oracle."""
    ncm = {"icnn_isochoric": lambda: dict(gen.ncm_weights(64, 3, 0.3, 11, 10.0), kinematics="isochoric"),
           "icnn_anisotropic": lambda: gen.anisotropic(gen.ncm_weights(64, 3, 0.3, 14, 10.0, n_in=5)),
           "cann_anisotropic": lambda: gen.anisotropic(gen.cann_params(4, seed=6, n_in=5)),
           "ickan": lambda: gen.ickan_params(),
           "cann_two_vectors": lambda: gen.anisotropic(gen.cann_params(3, seed=8, n_in=9), gen.A_FIBRE,
                                                       gen.A_SHEET),
           "icnn_isochoric_anisotropic": lambda: gen.anisotropic(gen.ncm_weights(64, 3, 0.3, 20, 10.0, n_in=5),
                                                                 isochoric=True),
           "cann_isochoric_two_vectors": lambda: gen.anisotropic(gen.cann_params(3, seed=21, n_in=9), gen.A_FIBRE,
                                                                 (0.0, 0.6, 0.8), isochoric=True)}[variant]()
    sampled_rows_check("c3", n_samples=8, ncm=ncm)


@pytest.mark.parametrize("kind,n,w", [("hex", 3, 64), ("hex", 2, 128), ("tet", 2, 64)])
def test_forward_sweep_saturated_inner_layer(kind, n, w):
    """Forward sweep with half of layer 2 saturated (biases -800: sigma_2 underflows to ~1e-308) and
    large adjoints (output weights x 20, |lambda_2| >> 6): the inner layer's Hessian term
    lambda (1 - s)/s P P^T must stay finite (1/s of s clamped at 2^-500) and match
    the oracle."""
    case = small_case(kind, n, w, 3)
    m = case["ncm"]
    m["b"] = m["b"].copy()
    m["b"][1, ::2] = -800.0
    m["a"] = m["a"] * 20.0
    lib, r, v, rp, ci = run_gpu(case)
    ro, vo, orp, oci, bad = run_oracle(case)
    assert np.isfinite(r).all() and np.isfinite(v).all()
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    assert rel(r, ro) <= TOL and rel(v, vo) <= TOL, (rel(r, ro), rel(v, vo))
