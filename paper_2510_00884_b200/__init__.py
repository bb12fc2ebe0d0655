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
# COMMET_LIB: another build of the library (A/B tuning tools); default: the in-tree build
LIB_PATH = os.environ.get("COMMET_LIB") or os.path.join(_HERE, "libcommet.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `make -C {os.path.join(_HERE, 'csrc')}` "
                      "(the CUDA extension is required; there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)

COMMET_OK, COMMET_ERR_ARG, COMMET_ERR_CUDA, COMMET_ERR_NCCL, COMMET_ERR_OOM, COMMET_ERR_DOMAIN = range(6)
HEX8, TET10 = 0, 1
KERNEL_FUSED, KERNEL_SIMPLE = 0, 1
ORDER_COLOURED, ORDER_ELEMENT = 0, 1
SYMBOLS = ("commet_setup", "commet_csr_pattern", "commet_csr_pattern_copy", "commet_assemble",
           "commet_check", "commet_set_kernel", "commet_info", "commet_set_timing",
           "commet_kernel_times", "commet_selftest_activation", "commet_last_error", "commet_destroy",
           "commet_nccl_unique_id", "commet_nccl_comm_init", "commet_nccl_comm_destroy",
           "commet_halo_info", "commet_halo_send", "commet_halo_recv", "commet_halo_unpack",
           "commet_plan_create", "commet_plan_info", "commet_plan_csr", "commet_plan_halo",
           "commet_plan_send", "commet_plan_recv", "commet_plan_colours", "commet_plan_destroy",
           "commet_kernel_info", "commet_max_trace_C", "commet_set_dirichlet", "commet_apply_dirichlet",
           "commet_cg_jacobi", "commet_newton_step", "commet_ncm_eval", "commet_normalize_reference",
           "commet_material_eval", "commet_halo_recv_maps", "commet_set_peer", "commet_set_peer_mode",
           "commet_zero_outputs", "commet_set_preconditioner", "commet_check_ranks", "commet_plan_colour_iface",
           "commet_selftest_activation_tab", "commet_kernel_config", "commet_kernel_batch",
           "commet_assemble_host", "commet_host_wait")
NEWTON_MAX_LOG = 64


class MeshDesc(C.Structure):
    _fields_ = [("elem_type", C.c_int32), ("n_nodes", C.c_int64), ("n_elems", C.c_int64),
                ("conn", C.c_void_p), ("grad_N", C.c_void_p), ("qp_w", C.c_void_p),
                ("owned_node_begin", C.c_int64), ("owned_node_end", C.c_int64),
                ("n_ranks", C.c_int32), ("rank", C.c_int32), ("rank_node_begin", C.c_void_p),
                ("n_ghost", C.c_int64), ("ghost_conn", C.c_void_p), ("ghost_rank", C.c_void_p),
                ("scatter_order", C.c_int32)]


class NcmDesc(C.Structure):
    _fields_ = [("n_hidden", C.c_int32), ("width", C.c_int32), ("W1", C.c_void_p), ("W", C.c_void_p),
                ("b", C.c_void_p), ("a", C.c_void_p), ("skip_out", C.c_void_p),
                ("skip_hidden", C.c_void_p), ("kappa", C.c_double), ("ref_shift", C.c_double),
                ("kinematics", C.c_int32), ("network", C.c_int32), ("cann_n", C.c_int32),
                ("cann_f", C.c_void_p), ("cann_w1", C.c_void_p), ("cann_w2", C.c_void_p),
                ("gt", C.c_double * 3), ("kan_layers", C.c_int32), ("kan_width", C.c_void_p),
                ("kan_nb", C.c_int32), ("kan_k", C.c_int32), ("kan_grid", C.c_void_p), ("kan_w", C.c_void_p),
                ("kan_c", C.c_void_p), ("a0", C.c_double * 3), ("n_sv", C.c_int32), ("a1", C.c_double * 3)]


KIN_STANDARD, KIN_ISOCHORIC, KIN_ANISOTROPIC, KIN_ISOCHORIC_ANISOTROPIC = 0, 1, 2, 3
NET_ICNN, NET_CANN, NET_GENT_THOMAS, NET_ICKAN = 0, 1, 2, 3
_KIN = {"standard": KIN_STANDARD, "isochoric": KIN_ISOCHORIC, "anisotropic": KIN_ANISOTROPIC,
        "isochoric_anisotropic": KIN_ISOCHORIC_ANISOTROPIC}
_NET = {"icnn": NET_ICNN, "cann": NET_CANN, "gent_thomas": NET_GENT_THOMAS, "ickan": NET_ICKAN}


def ncm_desc(ncm: dict):
    """-> (NcmDesc, keepalive).  ncm keys: width, n_hidden, W1, W, b, a, optional skip_out,
    skip_hidden, kappa, ref_shift, kinematics ("standard" | "isochoric" | "anisotropic" |
    "isochoric_anisotropic"), network ("icnn" |
    "cann" | "gent_thomas"), cann_f [3, n, 3] int, cann_w1 / cann_w2 [3, n], gt [3]."""
    arrs = {k: _f64(ncm.get(k)) for k in ("W1", "W", "b", "a", "skip_out", "skip_hidden", "cann_w1", "cann_w2",
                                          "kan_grid", "kan_w", "kan_c")}
    if arrs["W"] is not None and arrs["W"].size == 0:
        arrs["W"] = None
    cf = None if ncm.get("cann_f") is None else np.ascontiguousarray(ncm["cann_f"], dtype=np.int32)
    kw = None if ncm.get("kan_width") is None else np.ascontiguousarray(ncm["kan_width"], dtype=np.int32)
    kin, net = ncm.get("kinematics", "standard"), ncm.get("network", "icnn")
    gt = ncm.get("gt")
    nd = NcmDesc(int(ncm.get("n_hidden", 1)), int(ncm.get("width", 16)),
                 *[_ptr(arrs[k]) for k in ("W1", "W", "b", "a", "skip_out", "skip_hidden")],
                 float(ncm.get("kappa", 0.0)), float(ncm.get("ref_shift", 0.0)),
                 _KIN[kin] if isinstance(kin, str) else int(kin), _NET[net] if isinstance(net, str) else int(net),
                 0 if cf is None else cf.shape[1], _ptr(cf), _ptr(arrs["cann_w1"]), _ptr(arrs["cann_w2"]),
                 (C.c_double * 3)(*(gt if gt is not None else (0.0, 0.0, 0.0))),
                 0 if kw is None else kw.size - 1, _ptr(kw), int(ncm.get("kan_nb", 0)), int(ncm.get("kan_k", 3)),
                 _ptr(arrs["kan_grid"]), _ptr(arrs["kan_w"]), _ptr(arrs["kan_c"]),
                 (C.c_double * 3)(*(ncm.get("a0") if ncm.get("a0") is not None else (0.0, 0.0, 0.0))),
                 2 if ncm.get("a1") is not None else 1,
                 (C.c_double * 3)(*(ncm.get("a1") if ncm.get("a1") is not None else (0.0, 0.0, 0.0))))
    return nd, [arrs, cf, kw]


class NewtonCfg(C.Structure):
    _fields_ = [("atol", C.c_double), ("rtol", C.c_double), ("max_iter", C.c_int32), ("cg_rtol", C.c_double),
                ("cg_max_iter", C.c_int32)]


class NewtonReport(C.Structure):
    _fields_ = [("iters", C.c_int32), ("converged", C.c_int32), ("n_assemble", C.c_int32),
                ("cg_iters_total", C.c_int64), ("res_norm", C.c_double * NEWTON_MAX_LOG),
                ("cg_iters", C.c_int32 * NEWTON_MAX_LOG), ("max_trC", C.c_double), ("ms_assemble", C.c_double),
                ("ms_solve", C.c_double)]


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
_lib.commet_check_ranks.argtypes = [_vp, C.POINTER(_i32), C.POINTER(_i64)]
_lib.commet_check_ranks.restype = C.c_int
_lib.commet_set_kernel.argtypes = [_vp, _i32]
_lib.commet_set_kernel.restype = C.c_int
_lib.commet_info.argtypes = [_vp] + [C.POINTER(_i32)] * 4
_lib.commet_info.restype = C.c_int
_lib.commet_set_timing.argtypes = [_vp, _i32]
_lib.commet_set_timing.restype = C.c_int
_lib.commet_kernel_times.argtypes = [_vp, _vp, _i32]
_lib.commet_kernel_times.restype = C.c_int
_lib.commet_selftest_activation.argtypes = [_vp, _vp, _vp, _i64, _vp]
_lib.commet_selftest_activation.restype = C.c_int
_lib.commet_selftest_activation_tab.argtypes = [_vp, _vp, _vp, _i64, _i32, _vp]
_lib.commet_selftest_activation_tab.restype = C.c_int
_P = C.POINTER
_lib.commet_nccl_unique_id.argtypes = [_vp]
_lib.commet_nccl_comm_init.argtypes = [_vp, _i32, _i32, C.c_int, _P(_vp)]
_lib.commet_nccl_comm_destroy.argtypes = [_vp]
_lib.commet_halo_info.argtypes = [_vp, _P(_i32), _P(_i32)]
_lib.commet_halo_send.argtypes = [_vp, _i32, _P(_i32), _P(_vp), _P(_i64), _P(_vp), _P(_i64)]
_lib.commet_halo_recv.argtypes = [_vp, _i32, _P(_i32), _P(_i64), _P(_i64)]
_lib.commet_halo_unpack.argtypes = [_vp, _i32, _vp, _vp, _vp, _vp, _vp]
_lib.commet_plan_create.argtypes = [_P(MeshDesc), _P(_vp)]
_lib.commet_plan_info.argtypes = [_vp, _P(_i64), _P(_i64), _P(_i64), _P(_i64), _P(_i32), _P(_i32), _P(_i32)]
_lib.commet_plan_csr.argtypes = [_vp, _P(_vp), _P(_vp)]
_lib.commet_plan_halo.argtypes = [_vp, _P(_vp), _P(_vp), _P(_vp)]
_lib.commet_plan_send.argtypes = [_vp, _i32, _P(_i32), _P(_i64), _P(_i64), _P(_i64), _P(_i64)]
_lib.commet_plan_recv.argtypes = [_vp, _i32, _P(_i32), _P(_i64), _P(_vp), _P(_i64), _P(_vp)]
_lib.commet_plan_colours.argtypes = [_vp, _P(_vp), _P(_vp)]
_lib.commet_plan_colour_iface.argtypes = [_vp, _P(_vp)]
_lib.commet_plan_destroy.argtypes = [_vp]
_lib.commet_plan_destroy.restype = None
for _f in ("commet_nccl_unique_id", "commet_nccl_comm_init", "commet_nccl_comm_destroy", "commet_halo_info",
           "commet_halo_send", "commet_halo_recv", "commet_halo_unpack", "commet_plan_create",
           "commet_plan_info", "commet_plan_csr", "commet_plan_halo", "commet_plan_send", "commet_plan_recv",
           "commet_plan_colours", "commet_plan_colour_iface"):
    getattr(_lib, _f).restype = C.c_int
_lib.commet_kernel_info.argtypes = [_vp, _P(_i32), _P(_i32), _P(_i32)]
_lib.commet_kernel_info.restype = C.c_int
_lib.commet_kernel_config.argtypes = [_vp, _P(_i32), _P(_i32)]
_lib.commet_kernel_config.restype = C.c_int
_lib.commet_kernel_batch.argtypes = [_vp, _P(_i32), _P(_i32)]
_lib.commet_kernel_batch.restype = C.c_int
_lib.commet_max_trace_C.argtypes = [_vp, _P(C.c_double)]
_lib.commet_set_dirichlet.argtypes = [_vp, _vp, _i64]
_lib.commet_apply_dirichlet.argtypes = [_vp, _vp, _vp, _vp]
_lib.commet_cg_jacobi.argtypes = [_vp, _vp, _vp, _vp, C.c_double, _i32, _P(_i32), _P(C.c_double), _vp]
_lib.commet_newton_step.argtypes = [_vp, _vp, _P(NewtonCfg), _vp, _P(NewtonReport), _vp]
_lib.commet_ncm_eval.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp]
_lib.commet_normalize_reference.argtypes = [_vp, _P(C.c_double)]
_lib.commet_assemble_host.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.commet_assemble_host.restype = C.c_int
_lib.commet_host_wait.argtypes = [_vp, _vp]
_lib.commet_host_wait.restype = C.c_int
_lib.commet_material_eval.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp, _vp]
_lib.commet_material_eval.restype = C.c_int
_lib.commet_halo_recv_maps.argtypes = [_vp, _i32, _P(_vp), _P(_vp)]
_lib.commet_set_peer.argtypes = [_vp, _i32, _vp, _vp, _vp, _i64, _vp, _i64]
_lib.commet_set_peer_mode.argtypes = [_vp, _i32]
_lib.commet_zero_outputs.argtypes = [_vp, _vp, _vp, _vp]
_lib.commet_set_preconditioner.argtypes = [_vp, _i32]
for _f in ("commet_halo_recv_maps", "commet_set_peer", "commet_set_peer_mode", "commet_zero_outputs",
           "commet_set_preconditioner"):
    getattr(_lib, _f).restype = C.c_int
for _f in ("commet_ncm_eval", "commet_normalize_reference", "commet_max_trace_C", "commet_set_dirichlet", "commet_apply_dirichlet", "commet_cg_jacobi",
           "commet_newton_step"):
    getattr(_lib, _f).restype = C.c_int
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


def _mesh_desc(mesh: dict):
    """-> (MeshDesc, keepalive list).  mesh keys: elem_type, n_nodes, conn, gradN, qp_w,
    optional owned_node_begin/_end, n_ranks, rank, rank_node_begin, ghost_conn, ghost_rank."""
    conn = np.ascontiguousarray(mesh["conn"], dtype=np.int32)
    gradN = _f64(mesh["gradN"]) if mesh.get("gradN") is not None else np.zeros(1)
    qp_w = _f64(mesh["qp_w"])
    n_nodes = int(mesh["n_nodes"])
    nb = int(mesh.get("owned_node_begin", 0))
    ne = int(mesh.get("owned_node_end", n_nodes))
    n_ranks = int(mesh.get("n_ranks", 1))
    rnb = None if mesh.get("rank_node_begin") is None else np.ascontiguousarray(mesh["rank_node_begin"], np.int64)
    gc = None if mesh.get("ghost_conn") is None else np.ascontiguousarray(mesh["ghost_conn"], np.int32)
    gr = None if mesh.get("ghost_rank") is None else np.ascontiguousarray(mesh["ghost_rank"], np.int32)
    md = MeshDesc(int(mesh["elem_type"]), n_nodes, conn.shape[0], _ptr(conn), _ptr(gradN), _ptr(qp_w), nb, ne,
                  n_ranks, int(mesh.get("rank", 0)), _ptr(rnb), 0 if gc is None else gc.shape[0], _ptr(gc), _ptr(gr),
                  int(mesh.get("scatter_order", ORDER_COLOURED)))
    return md, [conn, gradN, qp_w, rnb, gc, gr]


class Commet:
    """One library context: ``Commet(mesh, ncm).assemble(u) -> (r, vals)``.

    mesh: dict with elem_type, n_nodes, conn [n_el, n_en] int32, gradN
    [n_el, n_q, n_en, 3] fp64, qp_w [n_el, n_q] fp64 and optional
    owned_node_begin / owned_node_end.  ncm: dict with width, n_hidden, W1,
    W, b, a, optional skip_out, skip_hidden, kappa, ref_shift.
    """

    def __init__(self, mesh: dict | None, ncm: dict, device: int = 0, stream=None, nccl_comm=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        if mesh is None:  # material-point calls only
            md, _keep, n_nodes, nb, ne = None, None, 0, 0, 0
        else:
            md, _keep = _mesh_desc(mesh)
            n_nodes, nb, ne = md.n_nodes, md.owned_node_begin, md.owned_node_end
        nd, _keep_ncm = ncm_desc(ncm)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            status = _lib.commet_setup(None if md is None else C.byref(md), C.byref(nd), device, st.cuda_stream,
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

    def kernel_info(self):
        v = [_i32() for _ in range(7)]
        _check(_lib.commet_kernel_info(self.ctx, *[C.byref(x) for x in v[:3]]), self.ctx)
        _check(_lib.commet_kernel_config(self.ctx, *[C.byref(x) for x in v[3:5]]), self.ctx)
        _check(_lib.commet_kernel_batch(self.ctx, *[C.byref(x) for x in v[5:]]), self.ctx)
        return dict(smem_bytes=v[0].value, ctas_per_sm=v[1].value, regs_per_thread=v[2].value,
                    threads_per_cta=v[3].value, warp_specialised=bool(v[4].value), qps_network_batch=v[5].value,
                    qps_element_batch=v[6].value)

    def set_kernel(self, variant: int):
        _check(_lib.commet_set_kernel(self.ctx, variant), self.ctx)

    # -- assemble -------------------------------------------------------------------
    def alloc_outputs(self):
        t = self.torch
        return (t.empty(self.n_rows, dtype=t.float64, device=self.device),
                t.empty(self.nnz, dtype=t.float64, device=self.device))

    def _dev_f64(self, x, n, name):
        """The library reads / writes n doubles at x on this ctx's device: refuse anything else."""
        t = self.torch
        if not (isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float64 and x.is_contiguous()):
            raise TypeError(f"{name} must be a contiguous cuda float64 tensor")
        if x.device != self.device:
            raise ValueError(f"{name} is on {x.device}, the ctx on {self.device}")
        if x.numel() != n:
            raise ValueError(f"{name} has {x.numel()} entries, expected {n}")

    def assemble(self, u, residual=None, values=None, stream=None):
        """u: cuda fp64 tensor [3 n_nodes]. Returns (residual, values) (asynchronous)."""
        t = self.torch
        self._dev_f64(u, 3 * self.n_nodes, "u")
        if residual is None or values is None:
            residual, values = self.alloc_outputs()
        self._dev_f64(residual, self.n_rows, "residual")
        self._dev_f64(values, self.nnz, "values")
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(_lib.commet_assemble(self.ctx, u.data_ptr(), residual.data_ptr(), values.data_ptr(),
                                    st.cuda_stream), self.ctx)
        return residual, values

    def _host_f64(self, x, n, name):
        t = self.torch
        if not (isinstance(x, t.Tensor) and x.device.type == "cpu" and x.dtype == t.float64
                and x.is_contiguous()):
            raise TypeError(f"{name} must be a contiguous cpu float64 tensor (pinned for asynchronous copies)")
        if x.numel() != n:
            raise ValueError(f"{name} has {x.numel()} entries, expected {n}")

    def assemble_host(self, u_host, residual_host, values_host, stream=None):
        """commet_assemble_host: host u in, host residual / CSR values out (asynchronous: the
        outputs are valid after host_wait).  The library uploads, assembles and reads back."""
        t = self.torch
        self._host_f64(u_host, 3 * self.n_nodes, "u_host")
        self._host_f64(residual_host, self.n_rows, "residual_host")
        self._host_f64(values_host, self.nnz, "values_host")
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(_lib.commet_assemble_host(self.ctx, u_host.data_ptr(), residual_host.data_ptr(),
                                         values_host.data_ptr(), st.cuda_stream), self.ctx)
        return residual_host, values_host

    def host_wait(self, stream=None):
        """commet_host_wait: stream waits for every issued assemble_host read-back (None: the host blocks)."""
        _check(_lib.commet_host_wait(self.ctx, stream.cuda_stream if stream is not None else None), self.ctx)

    def set_timing(self, n_slots: int):
        _check(_lib.commet_set_timing(self.ctx, n_slots), self.ctx)

    def kernel_times(self, n: int):
        """Kernel-only milliseconds of the last n assembles (see commet_set_timing)."""
        out = np.zeros(n, np.float32)
        _check(_lib.commet_kernel_times(self.ctx, _ptr(out), n), self.ctx)
        return out

    # -- caller-driven halo exchange (multi-rank without NCCL) --------------------------
    def halo_info(self):
        ns, nr = _i32(), _i32()
        _check(_lib.commet_halo_info(self.ctx, C.byref(ns), C.byref(nr)), self.ctx)
        return ns.value, nr.value

    def halo_send(self, k: int):
        """-> (peer, vals_ptr, n_vals, res_ptr, n_res) device pointers into this ctx."""
        peer, vp, nv, rp, nr = _i32(), _vp(), _i64(), _vp(), _i64()
        _check(_lib.commet_halo_send(self.ctx, k, C.byref(peer), C.byref(vp), C.byref(nv), C.byref(rp),
                                     C.byref(nr)), self.ctx)
        return peer.value, vp.value, nv.value, rp.value, nr.value

    def halo_recv(self, k: int):
        peer, nv, nr = _i32(), _i64(), _i64()
        _check(_lib.commet_halo_recv(self.ctx, k, C.byref(peer), C.byref(nv), C.byref(nr)), self.ctx)
        return peer.value, nv.value, nr.value

    def halo_recv_maps(self, k: int):
        """(sender rank, val_map, row_map) of receive segment k (host int64 copies)."""
        peer, nv, nr = self.halo_recv(k)
        vp, rp = _vp(), _vp()
        _check(_lib.commet_halo_recv_maps(self.ctx, k, C.byref(vp), C.byref(rp)), self.ctx)
        return peer, Plan._arr(vp, nv, np.int64), Plan._arr(rp, nr, np.int64)

    def set_peer(self, k: int, peer_residual_ptr: int, peer_values_ptr: int, val_map, row_map):
        vm = np.ascontiguousarray(val_map, np.int64)
        rm = np.ascontiguousarray(row_map, np.int64)
        _check(_lib.commet_set_peer(self.ctx, k, peer_residual_ptr, peer_values_ptr, _ptr(vm), vm.size, _ptr(rm),
                                    rm.size), self.ctx)

    def set_peer_mode(self, on: bool = True):
        _check(_lib.commet_set_peer_mode(self.ctx, 1 if on else 0), self.ctx)

    def zero_outputs(self, residual, values, stream=None):
        t = self.torch
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(_lib.commet_zero_outputs(self.ctx, residual.data_ptr(), values.data_ptr(), st.cuda_stream), self.ctx)

    def halo_unpack(self, k: int, vals_ptr: int, res_ptr: int, residual, values, stream=None):
        t = self.torch
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(_lib.commet_halo_unpack(self.ctx, k, vals_ptr, res_ptr, residual.data_ptr(), values.data_ptr(),
                                       st.cuda_stream), self.ctx)

    def max_trace_C(self) -> float:
        """max over qps of tr C at the last assemble (synchronises)."""
        v = C.c_double()
        _check(_lib.commet_max_trace_C(self.ctx, C.byref(v)), self.ctx)
        return v.value

    # -- material-point calls ----------------------------------------------------------
    def ncm_eval(self, k, stream=None):
        """Inner-network gradient [n,3] and Hessian [n,6] at invariant inputs k (cuda [n,3])."""
        t = self.torch
        k = k.contiguous()
        n, nk = k.shape[0], k.shape[1]
        g = t.empty((n, nk), dtype=t.float64, device=k.device)
        H = t.empty((n, nk * (nk + 1) // 2), dtype=t.float64, device=k.device)
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(_lib.commet_ncm_eval(self.ctx, k.data_ptr(), g.data_ptr(), H.data_ptr(), n, st.cuda_stream),
               self.ctx)
        return g, H

    def material_eval(self, F, want_c=True, stream=None):
        """Psi [n], tau [n,6] (Voigt 00,11,22,12,02,01), c [n,21] (upper 6x6 Voigt) at F (cuda [n,3,3])."""
        t = self.torch
        F = F.contiguous()
        n = F.shape[0]
        W = t.empty(n, dtype=t.float64, device=F.device)
        tau = t.empty((n, 6), dtype=t.float64, device=F.device)
        c = t.empty((n, 21), dtype=t.float64, device=F.device) if want_c else None
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(_lib.commet_material_eval(self.ctx, F.data_ptr(), n, W.data_ptr(), tau.data_ptr(),
                                         None if c is None else c.data_ptr(), st.cuda_stream), self.ctx)
        return W, tau, c

    def normalize_reference(self) -> float:
        """Make F = I stress-free (sets ref_shift); returns s0."""
        v = C.c_double()
        _check(_lib.commet_normalize_reference(self.ctx, C.byref(v)), self.ctx)
        return v.value

    # -- Newton-Raphson around the assembly (single GPU) -----------------------------
    def set_dirichlet(self, dofs):
        """Constrained global dofs (host int array)."""
        d = np.ascontiguousarray(dofs, dtype=np.int64)
        _check(_lib.commet_set_dirichlet(self.ctx, _ptr(d), d.size), self.ctx)
        self.n_dirichlet = d.size

    def apply_dirichlet(self, residual, values, stream=None):
        t = self.torch
        self._dev_f64(values, self.nnz, "values")
        if residual is not None:
            self._dev_f64(residual, self.n_rows, "residual")
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(_lib.commet_apply_dirichlet(self.ctx, None if residual is None else residual.data_ptr(),
                                           values.data_ptr(), st.cuda_stream), self.ctx)

    PRECONDITIONERS = {"jacobi": 0, "block_jacobi": 1}

    def set_preconditioner(self, kind="jacobi"):
        """CG preconditioner of cg_jacobi / newton_step: "jacobi" (the paper's) or "block_jacobi"
        (3x3 nodal diagonal blocks)."""
        _check(_lib.commet_set_preconditioner(self.ctx, self.PRECONDITIONERS[kind]), self.ctx)

    def cg_jacobi(self, values, b, rtol=1e-10, max_iter=100000, x=None, stream=None):
        """Solve K x = b on this ctx's pattern (device tensors). -> (x, iters, rel_res)."""
        t = self.torch
        if x is None:
            x = t.empty_like(b)
        self._dev_f64(values, self.nnz, "values")
        self._dev_f64(b, self.n_rows, "b")
        self._dev_f64(x, self.n_rows, "x")
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        it, rel = _i32(), C.c_double()
        _check(_lib.commet_cg_jacobi(self.ctx, values.data_ptr(), b.data_ptr(), x.data_ptr(), rtol, max_iter,
                                     C.byref(it), C.byref(rel), st.cuda_stream), self.ctx)
        return x, it.value, rel.value

    def newton_step(self, u, bc_values, atol=1e-10, rtol=1e-10, max_iter=30, cg_rtol=1e-10,
                    cg_max_iter=200000, stream=None):
        """One load step: u[dirichlet] = bc_values, Newton iterations until converged.
        u: cuda fp64 tensor [3 n_nodes] (in/out).  -> report dict."""
        t = self.torch
        bv = np.ascontiguousarray(bc_values, dtype=np.float64).reshape(-1)
        if bv.size != getattr(self, "n_dirichlet", 0):
            raise ValueError(f"bc_values has {bv.size} entries, set_dirichlet gave {getattr(self, 'n_dirichlet', 0)} dofs")
        self._dev_f64(u, 3 * self.n_nodes, "u")
        cfg = NewtonCfg(atol, rtol, max_iter, cg_rtol, cg_max_iter)
        rep = NewtonReport()
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        _check(_lib.commet_newton_step(self.ctx, _ptr(bv), C.byref(cfg), u.data_ptr(), C.byref(rep),
                                       st.cuda_stream), self.ctx)
        n = rep.iters
        return dict(iters=n, converged=bool(rep.converged), res_norm=list(rep.res_norm[:n + 1]),
                    cg_iters=list(rep.cg_iters[:n]), cg_iters_total=rep.cg_iters_total, max_trC=rep.max_trC,
                    ms_assemble=rep.ms_assemble, ms_solve=rep.ms_solve)

    def newton_solve(self, u, bc_values_at, n_steps=10, max_halvings=4, **kw):
        """Load stepping around newton_step (host loop, no compute): t = k / n_steps,
        u[dirichlet] = bc_values_at(t).  A step that fails (det F <= 0, CG or Newton
        non-convergence) is retried from the last converged u with half the increment,
        up to max_halvings times (SPEC's step-halving).  -> list of per-step reports."""
        t_done, dt, reports = 0.0, 1.0 / n_steps, []
        u_ok = u.clone()
        while t_done < 1.0 - 1e-12:
            t = min(1.0, t_done + dt)
            try:
                rep = self.newton_step(u, bc_values_at(t), **kw)
                ok = rep["converged"]
            except CommetError as e:
                if e.status != COMMET_ERR_DOMAIN:
                    raise
                rep, ok = dict(error=str(e)), False
            rep["t"] = t
            reports.append(rep)
            if ok:
                t_done = t
                u_ok.copy_(u)
                continue
            u.copy_(u_ok)
            dt *= 0.5
            if dt < 1.0 / n_steps / 2 ** max_halvings:
                raise CommetError(COMMET_ERR_DOMAIN, f"load step at t = {t:.6g} failed after {max_halvings} halvings")
        return reports

    def check(self) -> int:
        """-1 if every det F > 0 on this rank, else its lowest flat e*n_q+q with det F <= 0
        (collective with an NCCL partition: see check_ranks)."""
        bad = _i64()
        s = _lib.commet_check(self.ctx, C.byref(bad))
        if s not in (COMMET_OK, COMMET_ERR_DOMAIN):
            _check(s, self.ctx)
        return bad.value

    def check_ranks(self):
        """(rank, qp) of the lowest rank with a det F <= 0 point and its lowest local flat index,
        (-1, -1) if none; one MIN all-reduce over the NCCL communicator (every rank calls it)."""
        rk, q = _i32(), _i64()
        s = _lib.commet_check_ranks(self.ctx, C.byref(rk), C.byref(q))
        if s not in (COMMET_OK, COMMET_ERR_DOMAIN):
            _check(s, self.ctx)
        return rk.value, q.value

    def close(self):
        if getattr(self, "ctx", None):
            _lib.commet_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """Host-only view of what commet_setup builds for a (rank-local) mesh: owned
    CSR pattern, halo rows, colouring and the per-peer interface maps.  Needs
    no GPU (used by the CPU tests of the multi-rank path)."""

    def __init__(self, mesh: dict):
        md, _keep = _mesh_desc(mesh)
        h = _vp()
        st = _lib.commet_plan_create(C.byref(md), C.byref(h))
        if st != COMMET_OK:
            raise CommetError(st, _lib.commet_last_error(None).decode())
        self.h = h
        v64 = [_i64() for _ in range(4)]
        v32 = [_i32() for _ in range(3)]
        _check(_lib.commet_plan_info(h, *[C.byref(x) for x in v64 + v32]))
        self.n_rows, self.nnz, self.n_halo, self.nnz_halo = [x.value for x in v64]
        self.n_colours, self.n_send, self.n_recv = [x.value for x in v32]

    @staticmethod
    def _arr(ptr, n, dt):
        if n == 0:
            return np.zeros(0, dt)
        ct = {np.int64: C.c_int64, np.int32: C.c_int32}[dt]
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy()

    def csr(self):
        rp, ci = _vp(), _vp()
        _check(_lib.commet_plan_csr(self.h, C.byref(rp), C.byref(ci)))
        return self._arr(rp, self.n_rows + 1, np.int64), self._arr(ci, self.nnz, np.int32)

    def halo(self):
        hn, rp, ci = _vp(), _vp(), _vp()
        _check(_lib.commet_plan_halo(self.h, C.byref(hn), C.byref(rp), C.byref(ci)))
        return (self._arr(hn, self.n_halo, np.int64), self._arr(rp, 3 * self.n_halo + 1, np.int64),
                self._arr(ci, self.nnz_halo, np.int32))

    def send(self, k: int):
        peer, v0, v1, r0, r1 = _i32(), _i64(), _i64(), _i64(), _i64()
        _check(_lib.commet_plan_send(self.h, k, *[C.byref(x) for x in (peer, v0, v1, r0, r1)]))
        return peer.value, (v0.value, v1.value), (r0.value, r1.value)

    def recv(self, k: int):
        peer, nv, vm, nr, rm = _i32(), _i64(), _vp(), _i64(), _vp()
        _check(_lib.commet_plan_recv(self.h, k, *[C.byref(x) for x in (peer, nv, vm, nr, rm)]))
        return peer.value, self._arr(vm, nv.value, np.int64), self._arr(rm, nr.value, np.int64)

    def colours(self, n_el: int):
        cs, pm = _vp(), _vp()
        _check(_lib.commet_plan_colours(self.h, C.byref(cs), C.byref(pm)))
        return self._arr(cs, self.n_colours + 1, np.int64), self._arr(pm, n_el, np.int64)

    def colour_iface(self):
        """[n_colours]: the interface elements at the start of each colour (launched first)."""
        ci = _vp()
        _check(_lib.commet_plan_colour_iface(self.h, C.byref(ci)))
        return self._arr(ci, self.n_colours, np.int64)

    def __del__(self):
        try:
            _lib.commet_plan_destroy(self.h)
        except Exception:
            pass


def nccl_comm_from_process_group(rank: int, world_size: int, device: int):
    """ncclComm_t for the library: unique id from rank 0, broadcast over the
    default torch.distributed process group (plumbing only)."""
    import torch
    import torch.distributed as dist
    idb = (C.c_char * 128)()
    if rank == 0:
        _check(_lib.commet_nccl_unique_id(idb))
    obj = [bytes(idb)]
    dist.broadcast_object_list(obj, src=0)
    idb = (C.c_char * 128).from_buffer_copy(obj[0])
    comm = _vp()
    with torch.cuda.device(device):
        _check(_lib.commet_nccl_comm_init(idb, world_size, rank, device, C.byref(comm)))
    return comm.value


def setup_peer_exchange(lib: "Commet", residual, values, rank: int, world_size: int):
    """Peer mode over torch.distributed (plumbing only): every rank shares its output tensors
    through CUDA IPC (torch.multiprocessing reductions) and the receive maps it holds for
    each sender; each rank then points its send segments at the owners' buffers."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor
    n_send, n_recv = lib.halo_info()
    maps = {}
    for k in range(n_recv):
        sender, vm, rm = lib.halo_recv_maps(k)
        maps[sender] = (vm, rm)
    mine = dict(rank=rank, r=reduce_tensor(residual), v=reduce_tensor(values), maps=maps)
    everyone = [None] * world_size
    dist.all_gather_object(everyone, mine)
    keep = []
    for k in range(n_send):
        peer = lib.halo_send(k)[0]
        owner = everyone[peer]
        fr, ar = owner["r"]
        fv, av = owner["v"]
        r_peer, v_peer = fr(*ar), fv(*av)
        vm, rm = owner["maps"][rank]
        lib.set_peer(k, r_peer.data_ptr(), v_peer.data_ptr(), vm, rm)
        keep += [r_peer, v_peer]
    lib.set_peer_mode(True)
    lib._peer_keepalive = keep
    return keep


def nccl_comm_destroy(comm):
    if comm:
        _check(_lib.commet_nccl_comm_destroy(comm))


def activation(y, table_bits: int = 6):
    """The fused kernel's softplus and sigmoid on a cuda fp64 tensor (diagnostic); table_bits 6
    (64-entry tables, 3-pass kernels) or 8 (256 entries, forward-sweep kernels)."""
    import torch
    y = y.contiguous()
    z, s = torch.empty_like(y), torch.empty_like(y)
    _check(_lib.commet_selftest_activation_tab(y.data_ptr(), z.data_ptr(), s.data_ptr(), y.numel(), table_bits,
                                               torch.cuda.current_stream(y.device).cuda_stream))
    return z, s


def from_config(cfg: dict, device: int = 0, scatter_order: int = ORDER_COLOURED, **kw) -> Commet:
    """Convenience: a context for a ``synth.gen.make_config`` dict."""
    return Commet(dict(elem_type=cfg["elem_type"], n_nodes=cfg["n_nodes"], conn=cfg["conn"],
                       gradN=cfg["gradN"], qp_w=cfg["qp_w"], scatter_order=scatter_order), cfg["ncm"],
                  device=device, **kw)
