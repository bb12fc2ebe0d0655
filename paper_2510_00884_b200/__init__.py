"""Thin Python binding of libcommet.so (the C ABI in include/commet.h).

Argument marshalling only: every step of the assembly runs in the CUDA
kernels of ``csrc/``.  PyTorch supplies device memory and streams.  There is
no CPU fallback -- importing this package raises if the shared library is
missing (build it with ``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_2510_00884_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcommet.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `make -C {os.path.join(_HERE, 'csrc')}` "
                      "(the CUDA extension is required; there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)

COMMET_OK, COMMET_ERR_ARG, COMMET_ERR_CUDA, COMMET_ERR_NCCL, COMMET_ERR_OOM, COMMET_ERR_DOMAIN = range(6)
HEX8, TET10 = 0, 1
KERNEL_FUSED, KERNEL_SIMPLE = 0, 1
SYMBOLS = ("commet_setup", "commet_csr_pattern", "commet_csr_pattern_copy", "commet_assemble",
           "commet_check", "commet_set_kernel", "commet_info", "commet_set_timing",
           "commet_kernel_times", "commet_last_error", "commet_destroy")


class MeshDesc(C.Structure):
    _fields_ = [("elem_type", C.c_int32), ("n_nodes", C.c_int64), ("n_elems", C.c_int64),
                ("conn", C.c_void_p), ("grad_N", C.c_void_p), ("qp_w", C.c_void_p),
                ("owned_node_begin", C.c_int64), ("owned_node_end", C.c_int64)]


class NcmDesc(C.Structure):
    _fields_ = [("n_hidden", C.c_int32), ("width", C.c_int32), ("W1", C.c_void_p), ("W", C.c_void_p),
                ("b", C.c_void_p), ("a", C.c_void_p), ("skip_out", C.c_void_p),
                ("skip_hidden", C.c_void_p), ("kappa", C.c_double), ("ref_shift", C.c_double)]


_vp, _i64, _i32 = C.c_void_p, C.c_int64, C.c_int32
_lib.commet_setup.argtypes = [C.POINTER(MeshDesc), C.POINTER(NcmDesc), C.c_int, _vp, _vp, C.POINTER(_vp)]
_lib.commet_setup.restype = C.c_int
_lib.commet_csr_pattern.argtypes = [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_vp), C.POINTER(_vp)]
_lib.commet_csr_pattern.restype = C.c_int
_lib.commet_csr_pattern_copy.argtypes = [_vp, _vp, _vp]
_lib.commet_csr_pattern_copy.restype = C.c_int
_lib.commet_assemble.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.commet_assemble.restype = C.c_int
_lib.commet_check.argtypes = [_vp, C.POINTER(_i64)]
_lib.commet_check.restype = C.c_int
_lib.commet_set_kernel.argtypes = [_vp, _i32]
_lib.commet_set_kernel.restype = C.c_int
_lib.commet_info.argtypes = [_vp] + [C.POINTER(_i32)] * 4
_lib.commet_info.restype = C.c_int
_lib.commet_set_timing.argtypes = [_vp, _i32]
_lib.commet_set_timing.restype = C.c_int
_lib.commet_kernel_times.argtypes = [_vp, _vp, _i32]
_lib.commet_kernel_times.restype = C.c_int
_lib.commet_last_error.argtypes = [_vp]
_lib.commet_last_error.restype = C.c_char_p
_lib.commet_destroy.argtypes = [_vp]
_lib.commet_destroy.restype = None


class CommetError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"commet status {status}: {msg}")
        self.status = status


def _check(status, ctx=None):
    if status != COMMET_OK:
        raise CommetError(status, _lib.commet_last_error(ctx).decode())


def _f64(x):
    return None if x is None else np.ascontiguousarray(x, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data


class Commet:
    """One library context: ``Commet(mesh, ncm).assemble(u) -> (r, vals)``.

    mesh: dict with elem_type, n_nodes, conn [n_el, n_en] int32, gradN
    [n_el, n_q, n_en, 3] fp64, qp_w [n_el, n_q] fp64 and optional
    owned_node_begin / owned_node_end.  ncm: dict with width, n_hidden, W1,
    W, b, a, optional skip_out, skip_hidden, kappa, ref_shift.
    """

    def __init__(self, mesh: dict, ncm: dict, device: int = 0, stream=None, nccl_comm=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        conn = np.ascontiguousarray(mesh["conn"], dtype=np.int32)
        gradN = _f64(mesh["gradN"])
        qp_w = _f64(mesh["qp_w"])
        n_nodes = int(mesh["n_nodes"])
        nb = int(mesh.get("owned_node_begin", 0))
        ne = int(mesh.get("owned_node_end", n_nodes))
        md = MeshDesc(int(mesh["elem_type"]), n_nodes, conn.shape[0], _ptr(conn), _ptr(gradN),
                      _ptr(qp_w), nb, ne)
        arrs = {k: _f64(ncm.get(k)) for k in ("W1", "W", "b", "a", "skip_out", "skip_hidden")}
        if arrs["W"] is not None and arrs["W"].size == 0:
            arrs["W"] = None
        nd = NcmDesc(int(ncm["n_hidden"]), int(ncm["width"]), *[_ptr(arrs[k]) for k in
                     ("W1", "W", "b", "a", "skip_out", "skip_hidden")],
                     float(ncm.get("kappa", 0.0)), float(ncm.get("ref_shift", 0.0)))
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            status = _lib.commet_setup(C.byref(md), C.byref(nd), device, st.cuda_stream,
                                       nccl_comm, C.byref(ctx))
        if status != COMMET_OK:
            raise CommetError(status, _lib.commet_last_error(None).decode())
        self.ctx = ctx
        nr, nnz = _i64(), _i64()
        _check(_lib.commet_csr_pattern(ctx, C.byref(nr), C.byref(nnz), None, None), ctx)
        self.n_rows, self.nnz = nr.value, nnz.value
        self.n_nodes = n_nodes
        self.owned = (nb, ne)

    # -- pattern --------------------------------------------------------------------
    def pattern(self, device: bool = False):
        """(row_ptr int64, col_idx int32) as numpy arrays (or cuda tensors)."""
        t = self.torch
        if device:
            rp = t.empty(self.n_rows + 1, dtype=t.int64, device=self.device)
            ci = t.empty(self.nnz, dtype=t.int32, device=self.device)
            _check(_lib.commet_csr_pattern_copy(self.ctx, rp.data_ptr(), ci.data_ptr()), self.ctx)
            return rp, ci
        rp = np.empty(self.n_rows + 1, np.int64)
        ci = np.empty(self.nnz, np.int32)
        _check(_lib.commet_csr_pattern_copy(self.ctx, _ptr(rp), _ptr(ci)), self.ctx)
        return rp, ci

    def info(self):
        v = [_i32() for _ in range(4)]
        _check(_lib.commet_info(self.ctx, *[C.byref(x) for x in v]), self.ctx)
        return dict(n_colours=v[0].value, n_q=v[1].value, n_en=v[2].value, launches=v[3].value)

    def set_kernel(self, variant: int):
        _check(_lib.commet_set_kernel(self.ctx, variant), self.ctx)

    # -- assemble -------------------------------------------------------------------
    def alloc_outputs(self):
        t = self.torch
        return (t.empty(self.n_rows, dtype=t.float64, device=self.device),
                t.empty(self.nnz, dtype=t.float64, device=self.device))

    def assemble(self, u, residual=None, values=None, stream=None):
        """u: cuda fp64 tensor [3 n_nodes]. Returns (residual, values) (asynchronous)."""
        t = self.torch
        if not (isinstance(u, t.Tensor) and u.is_cuda and u.dtype == t.float64 and u.is_contiguous()):
            raise TypeError("u must be a contiguous cuda float64 tensor")
        if u.numel() != 3 * self.n_nodes:
            raise ValueError(f"u has {u.numel()} entries, expected {3 * self.n_nodes}")
        if residual is None or values is None:
            residual, values = self.alloc_outputs()
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(_lib.commet_assemble(self.ctx, u.data_ptr(), residual.data_ptr(), values.data_ptr(),
                                    st.cuda_stream), self.ctx)
        return residual, values

    def set_timing(self, n_slots: int):
        _check(_lib.commet_set_timing(self.ctx, n_slots), self.ctx)

    def kernel_times(self, n: int):
        """Kernel-only milliseconds of the last n assembles (see commet_set_timing)."""
        out = np.zeros(n, np.float32)
        _check(_lib.commet_kernel_times(self.ctx, _ptr(out), n), self.ctx)
        return out

    def check(self) -> int:
        """-1 if every det F > 0, else the lowest flat e*n_q+q with det F <= 0."""
        bad = _i64()
        s = _lib.commet_check(self.ctx, C.byref(bad))
        if s not in (COMMET_OK, COMMET_ERR_DOMAIN):
            _check(s, self.ctx)
        return bad.value

    def close(self):
        if getattr(self, "ctx", None):
            _lib.commet_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def from_config(cfg: dict, device: int = 0, **kw) -> Commet:
    """Convenience: a context for a ``synth.gen.make_config`` dict."""
    return Commet(dict(elem_type=cfg["elem_type"], n_nodes=cfg["n_nodes"], conn=cfg["conn"],
                       gradN=cfg["gradN"], qp_w=cfg["qp_w"]), cfg["ncm"], device=device, **kw)
