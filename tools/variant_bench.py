#!/usr/bin/env python
"""Assembly throughput of the NCM variants on the c3 mesh
(64^3 hex8, 2.1M qp): kernel milliseconds per assembly (CUDA events around the colour
launches) and qp/s for each kinematics x network combination."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import gen  # noqa: E402


def main():
    import torch
    import paper_2510_00884_b200 as pc
    cfg = gen.make_config("c3")
    iso = lambda m: dict(m, kinematics="isochoric")  # noqa: E731
    models = {
        "icnn 64x3 (c3)": cfg["ncm"],
        "icnn 64x3 isochoric": iso(cfg["ncm"]),
        "gent-thomas": gen.gent_thomas_params(),
        "cann 4 branches": gen.cann_params(4),
        "cann anisotropic": gen.anisotropic(gen.cann_params(4, n_in=5)),
        "ickan 3-6-6-1": gen.ickan_params(),
        "ickan anisotropic 5-4-1": gen.anisotropic(gen.ickan_params((5, 4, 1), nb=7, seed=7)),
        "icnn 64x3 anisotropic": gen.anisotropic(gen.ncm_weights(64, 3, 0.3, 14, 10.0, n_in=5)),
        "cann two vectors (9 inputs)": gen.anisotropic(gen.cann_params(3, seed=8, n_in=9), gen.A_FIBRE, gen.A_SHEET),
        "ickan two vectors 9-4-1": gen.anisotropic(gen.ickan_params((9, 4, 1), nb=7, seed=9), gen.A_FIBRE,
                                                   gen.A_SHEET),
        "icnn 64x3 isochoric anisotropic": gen.anisotropic(gen.ncm_weights(64, 3, 0.3, 20, 10.0, n_in=5),
                                                           isochoric=True),
        "cann isochoric two vectors (9 inputs)": gen.anisotropic(gen.cann_params(3, seed=21, n_in=9), gen.A_FIBRE,
                                                                 (0.0, 0.6, 0.8), isochoric=True),
    }
    u = torch.from_numpy(cfg["u"]).cuda()
    nq = cfg["conn"].shape[0] * 8
    for name, m in models.items():
        lib = pc.Commet(dict(elem_type=cfg["elem_type"], n_nodes=cfg["n_nodes"], conn=cfg["conn"],
                             gradN=cfg["gradN"], qp_w=cfg["qp_w"]), m)
        r, v = lib.alloc_outputs()
        for _ in range(3):
            lib.assemble(u, r, v)
        lib.set_timing(10)
        for _ in range(10):
            lib.assemble(u, r, v)
        ms = float(np.median(lib.kernel_times(10)))
        print(json.dumps(dict(model=name, kernel_ms=ms, qp_per_s=nq / (ms * 1e-3), det_ok=lib.check() == -1,
                              launch=lib.kernel_info())), flush=True)
        lib.close()


if __name__ == "__main__":
    main()
