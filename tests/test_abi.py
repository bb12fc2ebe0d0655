"""CPU-side checks of the C-ABI library: it loads, exports every function the
header declares, and rejects bad arguments (host validation, no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "commet.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(commet_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2510_00884_b200 as pc
    lib = C.CDLL(pc.LIB_PATH)
    names = header_functions()
    assert "commet_setup" in names and "commet_assemble" in names
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/commet.h but not exported"
    assert set(pc.SYMBOLS) <= set(names)


def _desc(conn, gN, w, n_nodes, elem_type=0):
    import paper_2510_00884_b200 as pc
    return pc.MeshDesc(elem_type, n_nodes, conn.shape[0], conn.ctypes.data, gN.ctypes.data,
                       w.ctypes.data, 0, n_nodes)


def _ncm(width=16, L=2):
    from synth.gen import ncm_weights
    import paper_2510_00884_b200 as pc
    m = ncm_weights(width, L)
    keep = [m["W1"], m["W"], m["b"], m["a"]]
    return pc.NcmDesc(L, width, keep[0].ctypes.data, keep[1].ctypes.data, keep[2].ctypes.data,
                      keep[3].ctypes.data, None, None, 10.0, 0.0), keep


@pytest.mark.parametrize("bad", ["conn", "weight", "width", "layers", "owned", "etype"])
def test_setup_rejects_bad_arguments(bad):
    import paper_2510_00884_b200 as pc
    from synth.gen import hex_mesh, shape_gradients
    X, conn = hex_mesh(2)
    gN, w = shape_gradients(X, conn, 0)
    conn = conn.copy()
    n_nodes = X.shape[0]
    nd, keep = _ncm(16, 2)
    md = _desc(conn, gN, w, n_nodes)
    expect = {"conn": "conn[3][5]", "weight": "qp_w[1][2]", "width": "width 24", "layers": "n_hidden 9",
              "owned": "owned node range", "etype": "elem_type 7"}[bad]
    if bad == "conn":
        conn[3, 5] = n_nodes + 4
    elif bad == "weight":
        w[1, 2] = -1.0
    elif bad == "width":
        nd.width = 24
    elif bad == "layers":
        nd.n_hidden = 9
    elif bad == "owned":
        md.owned_node_end = n_nodes + 1
    elif bad == "etype":
        md.elem_type = 7
    ctx = C.c_void_p()
    st = pc._lib.commet_setup(C.byref(md), C.byref(nd), 0, None, None, C.byref(ctx))
    assert st == pc.COMMET_ERR_ARG
    assert not ctx.value
    assert expect in pc._lib.commet_last_error(None).decode()


def test_null_context_calls_fail_cleanly():
    import paper_2510_00884_b200 as pc
    assert pc._lib.commet_assemble(None, None, None, None, None) == pc.COMMET_ERR_ARG
    assert pc._lib.commet_check(None, None) == pc.COMMET_ERR_ARG
    pc._lib.commet_destroy(None)


@pytest.mark.parametrize("kin,n_sv,net,expect", [
    (7, 0, 0, "kinematics 7 unknown"),
    (3, 3, 0, "n_sv 3 not in 0..2"),                       # isochoric anisotropic, too many vectors
    (3, 1, 2, "anisotropic kinematics need an ICNN, CANN or ICKAN"),  # Gent-Thomas on 5 inputs
    (3, 2, 0, "two structural vectors (9 inputs): CANN or ICKAN"),   # ICNN on 9 inputs
])
def test_setup_rejects_bad_kinematics(kin, n_sv, net, expect):
    """Host validation of the kinematics ids (commet.h COMMET_KIN_*; 3 = isochoric anisotropic,
    App. A.2.2 / DESIGN R29) before any CUDA call."""
    import paper_2510_00884_b200 as pc
    from synth.gen import hex_mesh, shape_gradients
    X, conn = hex_mesh(2)
    gN, w = shape_gradients(X, conn, 0)
    nd, keep = _ncm(16, 2)
    nd.kinematics, nd.n_sv, nd.network = kin, n_sv, net
    md = _desc(conn, gN, w, X.shape[0])
    ctx = C.c_void_p()
    st = pc._lib.commet_setup(C.byref(md), C.byref(nd), 0, None, None, C.byref(ctx))
    assert st == pc.COMMET_ERR_ARG and not ctx.value
    assert expect in pc._lib.commet_last_error(None).decode()


def test_binding_kinematics_names():
    """The binding's names map onto the header's ids (no GPU needed)."""
    import paper_2510_00884_b200 as pc
    from synth.gen import anisotropic, cann_params, A_FIBRE, A_SHEET
    src = open(os.path.join(ROOT, "include", "commet.h")).read()
    ids = dict(re.findall(r"(COMMET_KIN_[A-Z_]+) = (\d+)", src))
    assert int(ids["COMMET_KIN_ISOCHORIC_ANISOTROPIC"]) == pc.KIN_ISOCHORIC_ANISOTROPIC == 3
    nd, _ = pc.ncm_desc(anisotropic(cann_params(3, n_in=9), A_FIBRE, A_SHEET, isochoric=True))
    assert nd.kinematics == 3 and nd.n_sv == 2 and list(nd.a1) == list(A_SHEET)
