#!/usr/bin/env python
"""Twist-cube Newton benchmark on one GPU (PAPER.md:601-665,
Fig. 7 and the assembly-vs-solve comparison of Fig. 9): load steps of Newton-
Raphson with GPU assembly and GPU CG-Jacobi, reporting device times of both
phases, iteration counts, max tr C, and the CG iteration's achieved HBM
bandwidth against the measured peak.

  python tools/newton_bench.py [--n 32] [--steps 10] [--width 16] [--layers 2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import twist  # noqa: E402

HBM_PEAK_GBS = 6549.1  # MEASURED_PEAKS.json hbm_gbs (copy bandwidth)


def cg_bytes_per_iter(n_rows: int, nnz: int) -> float:
    """Algorithmic HBM bytes of one CG-Jacobi iteration: the spmv
    reads vals (8 B/nnz) and col_idx once per node-row triple (4/3 B/nnz), gathers
    p and writes q; update_xr reads x, r, p, q, dinv and writes x, r, z; update_p
    reads z, p and writes p: 9.33 B/nnz + 15 vectors of 8 B."""
    return nnz * (8.0 + 4.0 / 3.0) + 15 * 8.0 * n_rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--width", type=int, default=16)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--cg-rtol", type=float, default=1e-8)
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--precond", default="jacobi", choices=["jacobi", "block_jacobi"])
    args = ap.parse_args()
    import torch
    import paper_2510_00884_b200 as pc

    t0 = time.time()
    mesh = twist.twist_mesh(args.n)
    ncm = twist.stable_ncm(args.width, args.layers)
    lib = pc.Commet(dict(elem_type=mesh["elem_type"], n_nodes=mesh["n_nodes"], conn=mesh["conn"],
                         gradN=mesh["gradN"], qp_w=mesh["qp_w"]), ncm)
    lib.set_preconditioner(args.precond)
    s0 = lib.normalize_reference()
    dofs, _, _ = twist.twist_bc(mesh["X"])
    lib.set_dirichlet(dofs)
    setup_s = time.time() - t0
    u = torch.zeros(3 * mesh["n_nodes"], dtype=torch.float64, device="cuda")
    steps = []
    ms_a = ms_s = 0.0
    cg_total = 0
    w0 = time.time()
    reps = lib.newton_solve(u, lambda t: twist.twist_values(mesh["X"], dofs, t), n_steps=args.steps,
                            atol=1e-12, rtol=args.rtol, max_iter=40, cg_rtol=args.cg_rtol)
    for s, rep in enumerate(reps, 1):
        if "error" in rep:
            steps.append(dict(step=s, t=rep["t"], failed=rep["error"]))
            continue
        steps.append(dict(step=s, t=rep["t"], iters=rep["iters"], converged=rep["converged"],
                          cg_iters=rep["cg_iters"], res=[float("%.3e" % x) for x in rep["res_norm"]]))
        ms_a += rep["ms_assemble"]
        ms_s += rep["ms_solve"]
        cg_total += rep["cg_iters_total"]
    rep = [r for r in reps if "error" not in r][-1]
    torch.cuda.synchronize()
    wall = time.time() - w0
    max_trc = rep["max_trC"]
    # CG iteration time on the final tangent, timed alone
    r, v = lib.assemble(u)
    lib.apply_dirichlet(r, v)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    x, it, rel = lib.cg_jacobi(v, r, rtol=1e-6, max_iter=200000)
    e1.record()
    torch.cuda.synchronize()
    ms_cg = e0.elapsed_time(e1)
    per_it = ms_cg / max(it, 1)
    gbs = cg_bytes_per_iter(lib.n_rows, lib.nnz) / (per_it * 1e-3) / 1e9
    line = dict(what="twist-cube Newton (GPU assembly + GPU CG-Jacobi)", n=args.n, dofs=lib.n_rows, nnz=lib.nnz,
                elements=int(mesh["conn"].shape[0]), ncm=f"{args.width}x{args.layers} convex ICNN, s0={s0:.6f}",
                precond=args.precond, load_steps=args.steps, steps_taken=len(steps),
                newton_iters=sum(x.get("iters", 0) for x in steps), cg_iters_total=int(cg_total),
                converged=bool(steps) and abs(steps[-1]["t"] - 1.0) < 1e-12 and steps[-1].get("converged", False),
                max_trC=max_trc,
                ms_assemble_total=ms_a, ms_solve_total=ms_s, solve_over_assemble=ms_s / max(ms_a, 1e-9),
                wall_s=wall, setup_s=setup_s,
                cg=dict(iters=it, rel_res=rel, ms=ms_cg, ms_per_iter=per_it,
                        bytes_per_iter=cg_bytes_per_iter(lib.n_rows, lib.nnz), achieved_gbs=gbs,
                        peak_gbs=HBM_PEAK_GBS, frac=gbs / HBM_PEAK_GBS),
                steps=steps)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
