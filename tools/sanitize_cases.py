#!/usr/bin/env python
"""Small runs of every fused-kernel instantiation (and the other kernels of the
library) for compute-sanitizer: racecheck / synccheck / memcheck / initcheck,
one tool per gpurun call:

  compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py

Covers: ICNN w = 16 (3-pass), 64 (forward sweep, and the 3-pass fallback with
hidden skips / L = 4), 128 (forward sweep); hex8 and tet10; NET = 1 (CANN,
Gent-Thomas, ICKAN); KIN = 1 (isochoric) and 2 (anisotropic: CANN, ICNN);
MODE = 1 (material points); the one-thread-per-element cross-check kernel; peer
mode with two contexts on one device (outputs zeroed first, no kernel waits on
another); the Newton / CG kernels; the activation self-test.  c1/c2-sized
meshes (one or a few batches per CTA and colour).  Prints one line per case.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_00884_b200 as pc  # noqa: E402
from synth import gen  # noqa: E402


def mesh(et, n, jitter=0.1, seed=5, amp=0.05):
    X, conn = gen.hex_mesh(n, jitter, seed) if et == gen.HEX8 else gen.tet10_mesh(n, jitter, seed)
    gN, w = gen.shape_gradients(X, conn, et)
    u = gen.smooth_field(X, amp, np.random.default_rng(seed + 2)).reshape(-1)
    return dict(elem_type=et, n_nodes=X.shape[0], conn=np.ascontiguousarray(conn), gradN=gN, qp_w=w), u


def assemble(name, et, n, ncm, kernel=None):
    m, u = mesh(et, n)
    lib = pc.Commet(m, ncm)
    if kernel is not None:
        lib.set_kernel(kernel)
    r, v = lib.assemble(torch.from_numpy(u).cuda())
    torch.cuda.synchronize()
    bad = lib.check()
    print(f"{name:34s} nnz {lib.nnz:8d}  |r| {float(r.abs().max()):.3e}  bad {bad}", flush=True)
    lib.close()


def main():
    w = gen.ncm_weights
    skips = w(64, 3, 0.3, 3, 10.0)
    rng = np.random.default_rng(9)
    skips["skip_out"] = rng.normal(0, 0.3, 3)
    skips["skip_hidden"] = rng.normal(0, 0.3, (2, 64, 3))
    iso = dict(w(64, 3, 0.3, 11, 10.0), kinematics="isochoric")
    cases = [
        ("icnn16x2 hex8 (3-pass)", gen.HEX8, 3, w(16, 2)),
        ("icnn64x3 hex8 (fwd sweep)", gen.HEX8, 3, w(64, 3)),
        ("icnn64x3 tet10 (fwd sweep)", gen.TET10, 2, w(64, 3)),
        ("icnn64x3 hex8 skips (3-pass)", gen.HEX8, 3, skips),
        ("icnn64x4 hex8 (3-pass)", gen.HEX8, 2, w(64, 4)),
        ("icnn64x1 hex8", gen.HEX8, 2, w(64, 1)),
        ("icnn128x3 hex8 (fwd sweep)", gen.HEX8, 2, w(128, 3)),
        ("icnn128x3 tet10 (fwd sweep)", gen.TET10, 2, w(128, 3)),
        ("icnn64x3 isochoric hex8", gen.HEX8, 2, iso),
        ("icnn64x3 anisotropic hex8", gen.HEX8, 2, gen.anisotropic(w(64, 3, 0.3, 14, 10.0, n_in=5))),
        ("cann hex8", gen.HEX8, 3, gen.cann_params(4, seed=3)),
        ("cann anisotropic tet10", gen.TET10, 2, gen.anisotropic(gen.cann_params(4, seed=6, n_in=5))),
        ("gent-thomas tet10", gen.TET10, 2, gen.gent_thomas_params()),
        ("ickan hex8", gen.HEX8, 3, gen.ickan_params()),
        ("ickan anisotropic hex8", gen.HEX8, 2, gen.anisotropic(gen.ickan_params((5, 4, 1), nb=7, seed=7))),
    ]
    for name, et, n, ncm in cases:
        assemble(name, et, n, ncm)
    assemble("simple kernel icnn64x3 hex8", gen.HEX8, 2, w(64, 3), kernel=pc.KERNEL_SIMPLE)

    # material points (MODE 1): ICNN forward sweep, 3-pass, analytic
    for name, ncm in [("material icnn64x3", w(64, 3)), ("material icnn16x2", w(16, 2)),
                      ("material icnn128x3", w(128, 3)), ("material cann", gen.cann_params(4, seed=3))]:
        lib = pc.Commet(None, ncm)
        F = np.eye(3)[None] + 0.05 * np.random.default_rng(1).normal(size=(37, 3, 3))
        W, tau, c = lib.material_eval(torch.from_numpy(F.reshape(-1, 9)).cuda())
        torch.cuda.synchronize()
        print(f"{name:34s} points 37  |c| {float(c.abs().max()):.3e}", flush=True)
        lib.close()

    # peer mode: two slab contexts on one device, halo rows added into the owner's buffers
    name, n, P = "c2", 6, 2
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
    g = gen.make_config(name, n=n)
    u = torch.from_numpy(g["u"]).cuda()
    for lib, (res, val) in zip(libs, outs):
        lib.zero_outputs(res, val)
    torch.cuda.synchronize()
    for lib, (res, val) in zip(libs, outs):
        lib.assemble(u, res, val)
    torch.cuda.synchronize()
    print(f"{'peer mode c2 n=6 P=2':34s} |r| {max(float(o[0].abs().max()) for o in outs):.3e}", flush=True)
    for lib in libs:
        lib.close()

    # Newton + CG (solver kernels) on a small twist-free stretch, and the activation self-test
    m, u0 = mesh(gen.HEX8, 3, jitter=0.0)
    ncm = w(16, 2)
    lib = pc.Commet(m, ncm)
    lib.normalize_reference()
    X = gen.hex_mesh(3)[0]
    fixed = np.nonzero(X[:, 2] < 1e-12)[0]
    top = np.nonzero(X[:, 2] > 1 - 1e-12)[0]
    dofs = np.concatenate([3 * fixed + c for c in range(3)] + [3 * top + 2])
    lib.set_dirichlet(dofs)
    u = torch.zeros(3 * m["n_nodes"], dtype=torch.float64, device="cuda")
    bc = np.concatenate([np.zeros(3 * fixed.size), 0.05 * np.ones(top.size)])
    rep = lib.newton_step(u, bc)
    print(f"{'newton + cg (jacobi)':34s} iters {rep['iters']} converged {rep['converged']}", flush=True)
    lib.set_preconditioner("block_jacobi")
    rep = lib.newton_step(u, bc * 2)
    print(f"{'newton + cg (block jacobi)':34s} iters {rep['iters']} converged {rep['converged']}", flush=True)
    lib.close()
    y = torch.linspace(-50, 50, 4097, dtype=torch.float64, device="cuda")
    for tb in (6, 8):
        z, s = pc.activation(y, tb)
    torch.cuda.synchronize()
    print("activation self-test ok", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
