#!/usr/bin/env python
"""Full-array GPU-vs-oracle parity at the BASELINE sizes.

  python tools/full_parity.py [--configs c3,c4,c5] [--slabs 16] [--out FILE]

c3 / c4: the whole residual and CSR value arrays against one full oracle run.
c5 (4.09e9 nonzeros): node-range slabs -- for rows [3a, 3b) the oracle assembles
only the elements that touch nodes [a, b) (those rows are then complete), so
every row of the GPU's single full-mesh assembly is compared, one slab at a
time.  One JSON line per config (and per c5 slab with --verbose): pattern
bit-exactness, normwise max|g-o|/max|o| and the per-entry relative error over
|o| >= 1e-6 max|o|, and the oracle's wall time.

Test infrastructure (calls oracle/); the GPU path runs through the C ABI.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import gen  # noqa: E402


def stats(g, o, floor=1e-6):
    a = np.abs(o)
    mx = float(a.max()) if a.size else 0.0
    err = np.abs(g - o)
    mask = a >= floor * mx
    return dict(normwise=float(err.max() / max(mx, 1e-300)) if a.size else 0.0,
                per_entry=float((err[mask] / a[mask]).max()) if mask.any() else 0.0,
                max_abs_err=float(err.max()) if a.size else 0.0, scale=mx)


def merge(acc, s, n):
    """Combine slab stats into whole-array stats (normwise needs the global max|o|)."""
    if acc is None:
        return dict(max_abs_err=s["max_abs_err"], scale=s["scale"], per_entry=s["per_entry"], n=n)
    acc["max_abs_err"] = max(acc["max_abs_err"], s["max_abs_err"])
    acc["scale"] = max(acc["scale"], s["scale"])
    acc["per_entry"] = max(acc["per_entry"], s["per_entry"])
    acc["n"] += n
    return acc


def run(name, slabs, verbose, out):
    import torch
    import paper_2510_00884_b200 as pc
    t0 = time.perf_counter()
    cfg = gen.make_config(name)
    lib = pc.from_config(cfg)
    u = torch.from_numpy(cfg["u"]).cuda()
    r, v = lib.assemble(u)
    bad = lib.check()
    torch.cuda.synchronize()
    rp_d, ci_d = lib.pattern(device=True)
    nn = cfg["n_nodes"]
    bounds = np.linspace(0, nn, slabs + 1).astype(np.int64) if slabs > 1 else np.array([0, nn])
    acc_r = acc_v = None
    pattern_ok = True
    t_or = 0.0
    for s in range(len(bounds) - 1):
        a, b = int(bounds[s]), int(bounds[s + 1])
        if slabs > 1:
            els = np.nonzero(((cfg["conn"] >= a) & (cfg["conn"] < b)).any(axis=1))[0]
            sub = np.ascontiguousarray(cfg["conn"][els])
            gN, qw = cfg["gradN"][els], cfg["qp_w"][els]
        else:
            sub, gN, qw = cfg["conn"], cfg["gradN"], cfg["qp_w"]
        t1 = time.perf_counter()
        orp, oci = oracle.pattern(nn, sub, node_begin=a, node_end=b)
        ro, vo, obad = oracle.assemble(cfg["ncm"], nn, sub, gN, qw, cfg["u"], orp, oci, node_begin=a,
                                       node_end=b, mode=1)
        t_or += time.perf_counter() - t1
        s0, s1 = int(rp_d[3 * a].item()), int(rp_d[3 * b].item())
        grp = (rp_d[3 * a:3 * b + 1] - s0).cpu().numpy()
        gci = ci_d[s0:s1].cpu().numpy()
        ok = bool(np.array_equal(grp, orp) and np.array_equal(gci, oci))
        pattern_ok &= ok
        gv = v[s0:s1].cpu().numpy()
        gr = r[3 * a:3 * b].cpu().numpy()
        sr, sv = stats(gr, ro), stats(gv, vo)
        acc_r, acc_v = merge(acc_r, sr, gr.size), merge(acc_v, sv, gv.size)
        if verbose:
            print(json.dumps(dict(config=name, slab=s, nodes=[a, b], elements=int(sub.shape[0]), pattern_exact=ok,
                                  residual=sr, csr_values=sv, oracle_bad=obad)), file=out, flush=True)
        del orp, oci, ro, vo, gv, gr, grp, gci
    for acc in (acc_r, acc_v):
        acc["normwise"] = acc["max_abs_err"] / max(acc["scale"], 1e-300)
    line = dict(config=name, n_nodes=nn, elements=int(cfg["conn"].shape[0]), nnz=int(lib.nnz),
                slabs=len(bounds) - 1, pattern_exact=pattern_ok, det_f_ok=bad == -1,
                residual=acc_r, csr_values=acc_v, oracle_s=t_or, oracle_threads=oracle.max_threads(),
                wall_s=time.perf_counter() - t0,
                passed=bool(pattern_ok and bad == -1 and acc_r["normwise"] <= 1e-10 and acc_v["normwise"] <= 1e-10))
    print(json.dumps(line), file=out, flush=True)
    del lib, r, v, rp_d, ci_d
    torch.cuda.empty_cache()
    return line["passed"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c3,c4,c5")
    ap.add_argument("--slabs", type=int, default=16, help="node-range slabs for c5 (c3/c4: one full run)")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    out = open(args.out, "a") if args.out else sys.stdout
    ok = True
    for name in args.configs.split(","):
        ok &= run(name, args.slabs if name == "c5" else 1, args.verbose, out)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
