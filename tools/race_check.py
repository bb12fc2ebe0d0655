#!/usr/bin/env python
"""Race / stale-read / out-of-range check of the CUDA path without compute-sanitizer
(closed on this GPU pool): a debug build of the library (COMMET_DEBUG_CHECKS, see
kernel_fused.cu) poisons every shared buffer with NaN before each batch, so a read
not ordered after this batch's write of the same word returns NaN, and traps on
any scatter address outside its buffer.  Every instantiation runs on small meshes
(several batches per CTA and colour, ragged tails) and is checked for
  * finite outputs,
  * parity with the oracle (normwise <= 1e-10, pattern bit-exact),
  * bitwise determinism over repeated runs (the coloured scatter fixes the
    summation order, so a race shows as run-to-run differences).
The planted-race builds (COMMET_DEBUG_DROP=1: no barrier between stages 7a and 7b;
=2: none after stage 1) must FAIL this check -- that is the check's sensitivity.

  python tools/race_check.py [--lib tools/ab/libcommet_debug.so] [--repeats 5] [--expect-fail]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cases():
    import numpy as np
    from synth import gen
    w = gen.ncm_weights
    skips = w(64, 3, 0.3, 3, 10.0)
    rng = np.random.default_rng(9)
    skips["skip_out"] = rng.normal(0, 0.3, 3)
    skips["skip_hidden"] = rng.normal(0, 0.3, (2, 64, 3))
    iso = dict(w(64, 3, 0.3, 11, 10.0), kinematics="isochoric")
    return [
        ("icnn16x2 hex8 (3-pass)", gen.HEX8, 4, w(16, 2)),
        ("icnn32x2 tet10 (3-pass)", gen.TET10, 3, w(32, 2)),
        ("icnn64x3 hex8 (fwd sweep)", gen.HEX8, 5, w(64, 3)),
        ("icnn64x3 tet10 (fwd sweep)", gen.TET10, 3, w(64, 3)),
        ("icnn64x2 hex8 (fwd sweep, L=2)", gen.HEX8, 4, w(64, 2)),
        ("icnn64x3 hex8 skips (3-pass)", gen.HEX8, 4, skips),
        ("icnn64x4 hex8 (3-pass)", gen.HEX8, 3, w(64, 4)),
        ("icnn64x1 hex8", gen.HEX8, 3, w(64, 1)),
        ("icnn128x3 hex8 (fwd sweep)", gen.HEX8, 3, w(128, 3)),
        ("icnn128x3 tet10 (fwd sweep)", gen.TET10, 2, w(128, 3)),
        ("icnn64x3 isochoric hex8", gen.HEX8, 3, iso),
        ("icnn64x3 anisotropic hex8", gen.HEX8, 3, gen.anisotropic(w(64, 3, 0.3, 14, 10.0, n_in=5))),
        ("cann hex8", gen.HEX8, 4, gen.cann_params(4, seed=3)),
        ("cann anisotropic tet10", gen.TET10, 2, gen.anisotropic(gen.cann_params(4, seed=6, n_in=5))),
        ("gent-thomas tet10", gen.TET10, 3, gen.gent_thomas_params()),
        ("ickan hex8", gen.HEX8, 3, gen.ickan_params()),
        ("cann two vectors hex8", gen.HEX8, 3, gen.anisotropic(gen.cann_params(3, seed=8, n_in=9), gen.A_FIBRE,
                                                                gen.A_SHEET)),
        ("icnn64x3 isochoric anisotropic hex8", gen.HEX8, 3,
         gen.anisotropic(w(64, 3, 0.3, 20, 10.0, n_in=5), isochoric=True)),
        ("cann isochoric two vectors tet10", gen.TET10, 2,
         gen.anisotropic(gen.cann_params(3, seed=21, n_in=9), gen.A_FIBRE, (0.0, 0.6, 0.8), isochoric=True)),
    ]


def run(lib_path, repeats):
    import numpy as np
    import torch
    import oracle
    import paper_2510_00884_b200 as pc
    from synth import gen
    assert os.path.samefile(pc.LIB_PATH, lib_path), (pc.LIB_PATH, lib_path)
    out = []
    for name, et, n, ncm in cases():
        X, conn = gen.hex_mesh(n, 0.1, 5) if et == gen.HEX8 else gen.tet10_mesh(n, 0.1, 5)
        gN, qw = gen.shape_gradients(X, conn, et)
        u = gen.smooth_field(X, 0.05, np.random.default_rng(7)).reshape(-1)
        m = dict(elem_type=et, n_nodes=X.shape[0], conn=np.ascontiguousarray(conn), gradN=gN, qp_w=qw)
        lib = pc.Commet(m, ncm)
        ud = torch.from_numpy(u).cuda()
        res = []
        for _ in range(repeats):
            r, v = lib.assemble(ud)
            torch.cuda.synchronize()
            res.append((r.cpu().numpy(), v.cpu().numpy()))
        bad = lib.check()
        finite = all(np.isfinite(a).all() and np.isfinite(b).all() for a, b in res)
        determ = all(np.array_equal(res[0][0], a) and np.array_equal(res[0][1], b) for a, b in res[1:])
        rp, ci = lib.pattern()
        orp, oci = oracle.pattern(m["n_nodes"], m["conn"])
        ro, vo, obad = oracle.assemble(ncm, m["n_nodes"], m["conn"], gN, qw, u, orp, oci)
        er = float(np.abs(res[0][0] - ro).max() / np.abs(ro).max()) if finite else float("nan")
        ev = float(np.abs(res[0][1] - vo).max() / np.abs(vo).max()) if finite else float("nan")
        ok = bool(finite and determ and bad == obad == -1 and np.array_equal(rp, orp) and np.array_equal(ci, oci)
                  and er <= 1e-10 and ev <= 1e-10)
        out.append(dict(case=name, elements=int(conn.shape[0]), finite=bool(finite), deterministic=bool(determ),
                        residual_rel=er, values_rel=ev, ok=ok))
        print(json.dumps(out[-1]), flush=True)
        lib.close()
    # material points (MODE 1)
    for name, ncm in [("material icnn64x3", gen.ncm_weights(64, 3)), ("material icnn16x2", gen.ncm_weights(16, 2)),
                      ("material icnn128x3", gen.ncm_weights(128, 3))]:
        lib = pc.Commet(None, ncm)
        F = np.eye(3)[None] + 0.05 * np.random.default_rng(1).normal(size=(77, 3, 3))
        Fd = torch.from_numpy(F.reshape(-1, 9)).cuda()
        outs = [tuple(t.cpu().numpy() for t in lib.material_eval(Fd)) for _ in range(repeats)]
        finite = all(all(np.isfinite(t).all() for t in o) for o in outs)
        determ = all(all(np.array_equal(a, b) for a, b in zip(outs[0], o)) for o in outs[1:])
        Wo = np.array([oracle.material_point(ncm, Fi)["W"] for Fi in F])
        ew = float(np.abs(outs[0][0] - Wo).max() / np.abs(Wo).max()) if finite else float("nan")
        ok = bool(finite and determ and ew <= 1e-10)
        out.append(dict(case=name, points=77, finite=bool(finite), deterministic=bool(determ), psi_rel=ew, ok=ok))
        print(json.dumps(out[-1]), flush=True)
        lib.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "tools", "ab", "libcommet_debug.so"))
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--expect-fail", action="store_true", help="planted-race build: some case must fail")
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    lib = os.path.abspath(args.lib)
    if not args.child:  # the library path must be set before the package is imported
        env = dict(os.environ, COMMET_LIB=lib)
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "--lib", lib, "--repeats", str(args.repeats),
                            "--child"], env=env, cwd=ROOT)
        if args.expect_fail:
            print(f"planted race: {'detected' if p.returncode != 0 else 'NOT detected'} (rc {p.returncode})")
            return 0 if p.returncode != 0 else 1
        return p.returncode
    sys.path.insert(0, ROOT)
    res = run(lib, args.repeats)
    bad = [r["case"] for r in res if not r["ok"]]
    print(json.dumps(dict(lib=os.path.basename(lib), cases=len(res), failed=bad)))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
