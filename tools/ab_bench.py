#!/usr/bin/env python
"""A/B timing of libcommet builds (tuning tool): assemble a config with each
given .so through the minimal C ABI and print kernel ms / qp/s.
usage: ab_bench.py c3 lib1.so lib2.so ..."""
import ctypes as C
import sys
import os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import gen


from paper_2510_00884_b200 import MeshDesc, NcmDesc  # noqa: E402  (struct layouts of include/commet.h)


def run(path, cfg, steps=20):
    lib = C.CDLL(path)
    conn = np.ascontiguousarray(cfg["conn"], np.int32)
    md = MeshDesc(cfg["elem_type"], cfg["n_nodes"], conn.shape[0], conn.ctypes.data, cfg["gradN"].ctypes.data,
                  cfg["qp_w"].ctypes.data, 0, cfg["n_nodes"], 1, 0, None, 0, None, None,
                  int(os.environ.get("AB_ORDER", "0")))
    m = cfg["ncm"]
    net = os.environ.get("AB_NET")  # variants: gt | cann | ickan | cann5 | ickan5 | icnn5 | icnnwWxL
    if net == "gt":
        m = gen.gent_thomas_params()
    elif net == "cann":
        m = gen.cann_params(4)
    elif net == "ickan":
        m = gen.ickan_params()
    elif net == "cann5":
        m = gen.anisotropic(gen.cann_params(4, n_in=5))
    elif net == "ickan5":
        m = gen.anisotropic(gen.ickan_params((5, 4, 1), nb=7, seed=7))
    elif net and net.startswith("icnnw"):  # e.g. icnnw32x2: the 3-pass ICNN instantiations (w <= 32)
        w_, l_ = net[5:].split("x")
        m = gen.ncm_weights(int(w_), int(l_), 0.3, 12, 10.0)
    elif net == "icnn5":
        m = gen.anisotropic(gen.ncm_weights(64, 3, 0.3, 14, 10.0, n_in=5))
    import paper_2510_00884_b200 as pc
    nd, keep = pc.ncm_desc(m)
    ctx = C.c_void_p()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.commet_setup(C.byref(md), C.byref(nd), 0, C.c_void_p(st), None, C.byref(ctx)) == 0
    nr, nnz = C.c_int64(), C.c_int64()
    lib.commet_csr_pattern(ctx, C.byref(nr), C.byref(nnz), None, None)
    u = torch.from_numpy(cfg["u"]).cuda()
    r = torch.empty(nr.value, dtype=torch.float64, device="cuda")
    v = torch.empty(nnz.value, dtype=torch.float64, device="cuda")
    lib.commet_set_timing(ctx, steps)
    for _ in range(3):
        lib.commet_assemble(ctx, C.c_void_p(u.data_ptr()), C.c_void_p(r.data_ptr()), C.c_void_p(v.data_ptr()), C.c_void_p(st))
    torch.cuda.synchronize()
    for _ in range(steps):
        lib.commet_assemble(ctx, C.c_void_p(u.data_ptr()), C.c_void_p(r.data_ptr()), C.c_void_p(v.data_ptr()), C.c_void_p(st))
    ms = (C.c_float * steps)()
    lib.commet_kernel_times(ctx, ms, steps)
    torch.cuda.synchronize()
    t = float(np.median(list(ms)))
    if hasattr(lib, "commet_debug_stage_cycles") and os.environ.get("AB_STAGES"):
        cyc = (C.c_ulonglong * 11)()
        lib.commet_debug_stage_cycles(cyc, 1)
        tot = sum(cyc)
        names = ["0 stage-in", "1 kinem", "2 layer1", "3 value", "4 adjoint", "5 g/H1", "6 jacobian",
                 "7a post", "7b A_q", "8a X", "8b K/scatter"]
        print("  stage cycles (thread 0, summed over CTAs, %d steps + 3 warm-ups):" % steps)
        for n_, c_ in zip(names, cyc):
            print(f"    {n_:14s} {100.0 * c_ / tot:6.2f} %")
    res = (r.cpu().numpy(), v.cpu().numpy())
    lib.commet_destroy(ctx)
    return t, res


if __name__ == "__main__":
    cfg = gen.make_config(sys.argv[1])
    nq = cfg["gradN"].shape[1] * cfg["conn"].shape[0]
    ref = None
    for p in sys.argv[2:]:
        t, res = run(p, cfg)
        d = "" if ref is None else " dv %.2e dr %.2e" % (np.abs(res[1] - ref[1]).max() / np.abs(ref[1]).max(),
                                                        np.abs(res[0] - ref[0]).max() / np.abs(ref[0]).max())
        ref = ref or res
        print(f"{os.path.basename(p):28s} {sys.argv[1]} kernel {t:8.3f} ms  {nq / t * 1e3:.4e} qp/s{d}", flush=True)
