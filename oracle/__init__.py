"""ctypes wrapper around the plain-C fp64 oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs -- never by the product
package ``paper_2510_00884_b200``.  Shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc -O2 (no -ffast-math, no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Ncm(C.Structure):
    _fields_ = [("n_hidden", C.c_int32), ("width", C.c_int32),
                ("W1", C.c_void_p), ("W", C.c_void_p), ("b", C.c_void_p), ("a", C.c_void_p),
                ("skip_out", C.c_void_p), ("skip_hidden", C.c_void_p),
                ("kappa", C.c_double), ("ref_shift", C.c_double),
                ("kinematics", C.c_int32), ("network", C.c_int32), ("cann_n", C.c_int32),
                ("cann_f", C.c_void_p), ("cann_w1", C.c_void_p), ("cann_w2", C.c_void_p),
                ("gt", C.c_double * 3), ("kan_layers", C.c_int32), ("kan_width", C.c_void_p),
                ("kan_nb", C.c_int32), ("kan_k", C.c_int32), ("kan_grid", C.c_void_p), ("kan_w", C.c_void_p),
                ("kan_c", C.c_void_p), ("a0", C.c_double * 3), ("n_sv", C.c_int32), ("a1", C.c_double * 3)]

KIN = {"standard": 0, "isochoric": 1, "anisotropic": 2, "isochoric_anisotropic": 3}
NET = {"icnn": 0, "cann": 1, "gent_thomas": 2, "ickan": 3}


_lib = None


class OracleError(RuntimeError):
    """The checker could not compute a trustworthy result (it fails loudly, never silently)."""


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i64, i32, vp = C.c_double, C.c_int64, C.c_int, C.c_void_p
        _lib.oracle_ncm_eval.argtypes = [vp, vp, vp, vp, vp]
        _lib.oracle_ncm_eval_n.argtypes = [vp, i32, vp, vp, vp, vp]
        _lib.oracle_ncm_eval_n.restype = i32
        _lib.oracle_ncm_eval.restype = i32
        _lib.oracle_material_point.argtypes = [vp] * 10
        _lib.oracle_material_point.restype = d
        _lib.oracle_qp_F.argtypes = [i64, i32, i32, vp, vp, vp, vp]
        _lib.oracle_energy.argtypes = [vp, i64, i32, i32, vp, vp, vp, vp]
        _lib.oracle_energy.restype = d
        _lib.oracle_pattern.argtypes = [i64, i64, i32, vp, i64, i64, vp, vp, vp]
        _lib.oracle_pattern.restype = i32
        _lib.oracle_assemble.argtypes = [vp, i64, i64, i32, i32, vp, vp, vp, vp, i64, i64,
                                         vp, vp, vp, vp, vp, i32, i32]
        _lib.oracle_assemble.restype = i64
        _lib.oracle_max_threads.restype = i32
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


class Ncm:
    """Holds contiguous fp64 copies of the NCM parameters and the C struct."""

    def __init__(self, ncm: dict):
        f = lambda x: None if x is None else np.ascontiguousarray(x, dtype=np.float64)
        self.arrays = {k: f(ncm.get(k)) for k in ("W1", "W", "b", "a", "skip_out", "skip_hidden")}
        if self.arrays["W"] is None or self.arrays["W"].size == 0:
            self.arrays["W"] = np.zeros(1)
        kin = ncm.get("kinematics", "standard")
        net = ncm.get("network", "icnn")
        self.cann_f = None if ncm.get("cann_f") is None else np.ascontiguousarray(ncm["cann_f"], dtype=np.int32)
        for k in ("cann_w1", "cann_w2"):
            self.arrays[k] = f(ncm.get(k))
        gt = (C.c_double * 3)(*(ncm.get("gt") if ncm.get("gt") is not None else (0.0, 0.0, 0.0)))
        self.kan_width = None if ncm.get("kan_width") is None else np.ascontiguousarray(ncm["kan_width"], np.int32)
        for k in ("kan_grid", "kan_w", "kan_c"):
            self.arrays[k] = f(ncm.get(k))
        self.s = _Ncm(int(ncm.get("n_hidden", 1)), int(ncm.get("width", 8)),
                      *[_p(self.arrays[k]) for k in ("W1", "W", "b", "a", "skip_out", "skip_hidden")],
                      float(ncm.get("kappa", 0.0)), float(ncm.get("ref_shift", 0.0)),
                      KIN[kin] if isinstance(kin, str) else int(kin), NET[net] if isinstance(net, str) else int(net),
                      0 if self.cann_f is None else self.cann_f.shape[1], _p(self.cann_f),
                      _p(self.arrays["cann_w1"]), _p(self.arrays["cann_w2"]), gt,
                      0 if self.kan_width is None else self.kan_width.size - 1, _p(self.kan_width),
                      int(ncm.get("kan_nb", 0)), int(ncm.get("kan_k", 3)), _p(self.arrays["kan_grid"]),
                      _p(self.arrays["kan_w"]), _p(self.arrays["kan_c"]),
                      (C.c_double * 3)(*(ncm.get("a0") if ncm.get("a0") is not None else (0.0, 0.0, 0.0))),
                      2 if ncm.get("a1") is not None else 1,
                      (C.c_double * 3)(*(ncm.get("a1") if ncm.get("a1") is not None else (0.0, 0.0, 0.0))))

    @property
    def ptr(self):
        return C.addressof(self.s)


def ncm_eval(ncm: dict, k):
    m = Ncm(ncm)
    k = np.ascontiguousarray(k, dtype=np.float64)
    N, g, H = np.zeros(1), np.zeros(3), np.zeros(9)
    rc = lib().oracle_ncm_eval(m.ptr, _p(k), _p(N), _p(g), _p(H))
    if rc != 0:
        raise OracleError(f"oracle: inner network evaluation failed (status {rc})")
    return N[0], g, H.reshape(3, 3)


def ncm_eval_n(ncm: dict, k):
    """Inner network on nin = len(k) inputs (3, or 5 for CANN / ICKAN on anisotropic inputs)."""
    m = Ncm(ncm)
    k = np.ascontiguousarray(k, dtype=np.float64)
    n = k.size
    N, g, H = np.zeros(1), np.zeros(n), np.zeros(n * n)
    rc = lib().oracle_ncm_eval_n(m.ptr, n, _p(k), _p(N), _p(g), _p(H))
    if rc != 0:
        raise OracleError(f"oracle: inner network evaluation on {n} inputs failed (status {rc})")
    return N[0], g, H.reshape(n, n)


def material_point(ncm: dict, F):
    """-> dict(J, k, W, g, H, S, CC, P, A) at one F (3x3)."""
    m = Ncm(ncm)
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(9)
    k, W, g, H = np.zeros(3), np.zeros(1), np.zeros(3), np.zeros(9)
    S, CC, P, A = np.zeros(9), np.zeros(81), np.zeros(9), np.zeros(81)
    J = lib().oracle_material_point(m.ptr, _p(F), _p(k), _p(W), _p(g), _p(H), _p(S), _p(CC),
                                    _p(P), _p(A))
    if np.isnan(J):
        raise OracleError("oracle: the inner network rejected this network / kinematics combination (or F is "
                          "not finite)")
    return dict(J=J, k=k, W=W[0], g=g, H=H.reshape(3, 3), S=S.reshape(3, 3),
                CC=CC.reshape(3, 3, 3, 3), P=P.reshape(3, 3), A=A.reshape(3, 3, 3, 3))


def qp_F(conn, gradN, u):
    n_el, n_en = conn.shape
    n_q = gradN.shape[1]
    out = np.zeros((n_el, n_q, 3, 3))
    lib().oracle_qp_F(n_el, n_en, n_q, _p(np.ascontiguousarray(conn, np.int32)),
                      _p(np.ascontiguousarray(gradN)), _p(np.ascontiguousarray(u)), _p(out))
    return out


def energy(ncm: dict, conn, gradN, qp_w, u):
    m = Ncm(ncm)
    n_el, n_en = conn.shape
    Pi = lib().oracle_energy(m.ptr, n_el, n_en, gradN.shape[1],
                             _p(np.ascontiguousarray(conn, np.int32)),
                             _p(np.ascontiguousarray(gradN)), _p(np.ascontiguousarray(qp_w)),
                             _p(np.ascontiguousarray(u, np.float64)))
    if np.isnan(Pi):
        raise OracleError("oracle: energy is NaN (inner network evaluation failed or non-finite input)")
    return Pi


def pattern(n_nodes, conn, node_begin=0, node_end=None):
    """-> (row_ptr int64, col_idx int32) for owned rows [3 node_begin, 3 node_end)."""
    node_end = n_nodes if node_end is None else node_end
    conn = np.ascontiguousarray(conn, np.int32)
    n_el, n_en = conn.shape
    nr = 3 * (node_end - node_begin)
    row_ptr = np.zeros(nr + 1, np.int64)
    nnz = np.zeros(1, np.int64)
    lib().oracle_pattern(n_nodes, n_el, n_en, _p(conn), node_begin, node_end, _p(row_ptr), None,
                         _p(nnz))
    col_idx = np.zeros(int(nnz[0]), np.int32)
    lib().oracle_pattern(n_nodes, n_el, n_en, _p(conn), node_begin, node_end, _p(row_ptr),
                         _p(col_idx), _p(nnz))
    return row_ptr, col_idx


def assemble(ncm: dict, n_nodes, conn, gradN, qp_w, u, row_ptr, col_idx, node_begin=0,
             node_end=None, mode=1, n_threads=0):
    """Alg. 1 assembly.  -> (r, vals, bad).  mode 0 serial, 1 OpenMP/colours."""
    node_end = n_nodes if node_end is None else node_end
    m = Ncm(ncm)
    conn = np.ascontiguousarray(conn, np.int32)
    n_el, n_en = conn.shape
    r = np.zeros(3 * (node_end - node_begin))
    vals = np.zeros(col_idx.size)
    bad = np.zeros(1, np.int64)
    miss = lib().oracle_assemble(m.ptr, n_nodes, n_el, n_en, gradN.shape[1], _p(conn),
                                 _p(np.ascontiguousarray(gradN)), _p(np.ascontiguousarray(qp_w)),
                                 _p(np.ascontiguousarray(u, np.float64)), node_begin, node_end,
                                 _p(row_ptr), _p(col_idx), _p(r), _p(vals), _p(bad), mode,
                                 n_threads)
    if miss == -2:
        raise OracleError("oracle: inner network evaluation failed (unsupported network / kinematics "
                          "combination)")
    if miss == -1:
        raise OracleError("oracle: element colouring needs more than 64 colours")
    if miss != 0:
        raise OracleError("oracle: %d stiffness entries outside the pattern" % miss)
    return r, vals, int(bad[0])


def max_threads() -> int:
    return lib().oracle_max_threads()
