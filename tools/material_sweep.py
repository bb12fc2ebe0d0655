#!/usr/bin/env python
"""GPU version of the paper's material point benchmarks (PAPER.md:509-557,
Figs. 4-5): constitutive updates (Psi, tau, c) of n_pts material points issued
in batches of a given size (one commet_material_eval call per batch), timed with
CUDA events.  Reports points/s per (n_pts, batch) and the fp64 roofline
fraction of the large-batch runs (network flops only: NCM_min of SURVEY s8(d)).

  python tools/material_sweep.py [--width 64] [--layers 3]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth.gen import ncm_weights  # noqa: E402

FP64_PEAK = 36.9  # TF/s, profiles/r01_fp64_peak.json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=64)
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--npts", default="16384,262144,4194304")
    ap.add_argument("--batches", default="1,16,256,4096,65536,1048576,4194304")
    args = ap.parse_args()
    import torch
    import paper_2510_00884_b200 as pc

    w, L = args.width, args.layers
    lib = pc.Commet(None, ncm_weights(w, L, 0.3, 1, 10.0))
    rng = np.random.default_rng(0)
    nmax = max(int(x) for x in args.npts.split(","))
    F = torch.from_numpy(np.eye(3)[None] + rng.uniform(-0.2, 0.2, size=(nmax, 3, 3))).cuda()
    W = torch.empty(nmax, dtype=torch.float64, device="cuda")
    tau = torch.empty((nmax, 6), dtype=torch.float64, device="cuda")
    c = torch.empty((nmax, 21), dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    ncm_flops = 10 * w * w * (L - 1) + 20 * w * L + 8 * w
    rows = []
    for n in (int(x) for x in args.npts.split(",")):
        for b in (int(x) for x in args.batches.split(",")):
            if b > n or n // b > 20000:
                continue
            nb = n // b

            def run():
                for k in range(nb):
                    s0 = k * b
                    pc._check(pc._lib.commet_material_eval(lib.ctx, F[s0].data_ptr(), b, W[s0:].data_ptr(),
                                                           tau[s0].data_ptr(), c[s0].data_ptr(), st.cuda_stream),
                              lib.ctx)
            run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(1, min(20, int(2e6 // n)))
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            pts = nb * b / (ms * 1e-3)
            rows.append(dict(n_pts=nb * b, batch=b, launches=nb, ms=ms, pts_per_s=pts,
                             ncm_tflops=pts * ncm_flops / 1e12, frac_fp64=pts * ncm_flops / 1e12 / FP64_PEAK))
            print(json.dumps(rows[-1]), flush=True)
    best = max(rows, key=lambda r: r["pts_per_s"])
    print(json.dumps(dict(what="material point sweep (Psi, tau, c per point)", ncm=f"{w}x{L}",
                          ncm_flops_per_pt=ncm_flops, best=best)), flush=True)


if __name__ == "__main__":
    main()
