"""Seeded synthetic inputs for the NCM-assembly hot path (configs c1-c5).

This module is shared by BOTH sides of the parity check (the CPU oracle under
``oracle/`` and the CUDA library under ``paper_2510_00884_b200/``) and by
``bench.py``.  It holds none of the method's arithmetic: it only produces the
*inputs* the boundary takes (paper Eq. r-quad/k-quad, and
Alg. 1 line 3):

* a mesh (node coordinates, hex8 or tet10 connectivity, z-major numbering),
* the per-(element, qp) reference shape-function gradients dN_a/dX and the
  quadrature "volume" weights w^{e,q} = Gauss weight * det(dX/dxi) (the
  isoparametric map of the generated geometry -- input preparation, not the
  assembled operation),
* seeded NCM weights (ICNN/MLP parameterisation),
* a seeded nodal displacement u.

Recipes follow SURVEY.md s8(d) and BASELINE.json configs; every reading is
listed in DESIGN.md ("Input recipe").  Seeds: mesh jitter 0, weights 1,
displacement 2 (numpy.random.default_rng).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

HEX8 = 0
TET10 = 1

# hex8, 2x2x2 Gauss rule (+-1/sqrt(3), weight 1), VTK node order
_HEX_XI = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                    [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=np.float64)
_G = 1.0 / math.sqrt(3.0)
_HEX_QP = np.array([[x, y, z] for z in (-_G, _G) for y in (-_G, _G) for x in (-_G, _G)])

# tet10, 4-point degree-2 rule, weight 1/24 (reference volume 1/6)
_TA, _TB = 0.5854101966249685, 0.1381966011250105
_TET_QP_BARY = np.array([[_TA, _TB, _TB, _TB], [_TB, _TA, _TB, _TB],
                         [_TB, _TB, _TA, _TB], [_TB, _TB, _TB, _TA]])
_TET_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    elem_type: int
    n: int              # cells per edge
    jitter: float       # fraction of h, interior nodes, uniform +-jitter*h
    width: int
    n_hidden: int
    u_kind: str         # "uniform" | "smooth" | "stretch+smooth"
    u_amp: float
    kappa: float = 10.0
    weight_std: float = 0.3


CONFIGS = {
    "c1": ConfigSpec("c1", HEX8, 4, 0.0, 16, 2, "uniform", 0.02),
    "c2": ConfigSpec("c2", HEX8, 16, 0.1, 32, 2, "smooth", 0.05),
    "c3": ConfigSpec("c3", HEX8, 64, 0.0, 64, 3, "stretch+smooth", 0.01),
    "c4": ConfigSpec("c4", TET10, 48, 0.1, 128, 3, "smooth", 0.1),
    "c5": ConfigSpec("c5", HEX8, 256, 0.0, 64, 3, "smooth", 0.05),
}

SEED_MESH, SEED_W, SEED_U = 0, 1, 2


# --------------------------------------------------------------------------
# meshes
# --------------------------------------------------------------------------
def _lattice(n: int, jitter: float, rng) -> np.ndarray:
    """(n+1)^3 nodes of [0,1]^3, node id = i + (n+1)(j + (n+1)k).  Interior
    coordinates jittered uniformly by +-jitter*h; a boundary node moves only
    tangentially (its coordinate on the boundary plane is kept)."""
    t = np.linspace(0.0, 1.0, n + 1)
    z, y, x = np.meshgrid(t, t, t, indexing="ij")
    X = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)
    if jitter > 0.0:
        h = 1.0 / n
        d = rng.uniform(-jitter * h, jitter * h, size=X.shape)
        on_bnd = (np.abs(X) < 1e-12) | (np.abs(X - 1.0) < 1e-12)
        d[on_bnd] = 0.0
        X = X + d
    return X


def hex_mesh(n: int, jitter: float = 0.0, seed: int = SEED_MESH, z_range=None):
    """Structured hex8 mesh of the unit cube; element id = i + n(j + n k).
    ``z_range=(k0,k1)`` returns only element layers k0..k1-1 (slab), with
    GLOBAL node ids."""
    rng = np.random.default_rng(seed)
    X = _lattice(n, jitter, rng)
    k0, k1 = (0, n) if z_range is None else z_range
    m = n + 1
    k, j, i = np.meshgrid(np.arange(k0, k1), np.arange(n), np.arange(n), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    base = i + m * (j + m * k)
    off = np.array([0, 1, 1 + m, m, m * m, 1 + m * m, 1 + m + m * m, m + m * m])
    conn = (base[:, None] + off[None, :]).astype(np.int32)
    return X, conn


def _kuhn_cell_tets():
    """6 Kuhn tets of the unit cell, as corner-offset triples (positively
    oriented): v0=(0,0,0) -> +e_p0 -> +e_p1 -> (1,1,1)."""
    tets = []
    for perm in [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]:
        v = [np.zeros(3, dtype=np.int64)]
        for p in perm:
            nv = v[-1].copy()
            nv[p] += 1
            v.append(nv)
        d = np.array([v[1] - v[0], v[2] - v[0], v[3] - v[0]], dtype=np.float64)
        if np.linalg.det(d) < 0:
            v[1], v[2] = v[2], v[1]
        tets.append(v)
    return tets


def tet10_mesh(n: int, jitter: float = 0.1, seed: int = SEED_MESH, z_range=None):
    """6 Kuhn tets per cell of an n^3 grid, straight-sided tet10 (edge nodes at
    the midpoints of the jittered vertices).  Nodes are numbered z-major on the
    doubled lattice (2i, 2j, 2k) so a z-slab owns a contiguous node range.
    Node order within an element: vertices 0-3, then edges 01,02,03,12,13,23."""
    rng = np.random.default_rng(seed)
    Xv = _lattice(n, jitter, rng)
    m = n + 1
    M = 2 * n + 1
    tets = _kuhn_cell_tets()
    k0, k1 = (0, n) if z_range is None else z_range
    # doubled-lattice codes of every node of every (global) tet; used to number
    # nodes identically whatever slab is requested
    kk, jj, ii = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    cell = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1)  # (n^3, 3) (i,j,k)
    codes = []
    for t in tets:
        vv = [2 * (cell + tv[None, :]) for tv in t]  # doubled coords of vertices
        nodes = vv + [(vv[a] + vv[b]) // 2 for a, b in _TET_EDGES]
        codes.append(np.stack([c[:, 0] + M * (c[:, 1] + M * c[:, 2]) for c in nodes], axis=1))
    codes = np.stack(codes, axis=1).reshape(-1, 10)  # element = 6*cell + t
    used = np.unique(codes)                          # sorted = z-major on doubled lattice
    node_of_code = np.full(M * M * M, -1, dtype=np.int64)
    node_of_code[used] = np.arange(used.size)
    # coordinates: vertices from the jittered lattice, edge nodes at midpoints
    cz, cy, cx = used // (M * M), (used // M) % M, used % M
    X = np.empty((used.size, 3))
    even = (cx % 2 == 0) & (cy % 2 == 0) & (cz % 2 == 0)
    X[even] = Xv[(cx[even] // 2) + m * ((cy[even] // 2) + m * (cz[even] // 2))]
    # midpoint of edge: endpoints are (c - d) and (c + d) with d in {0, 1} per axis
    odd = ~even
    lo = np.stack([cx[odd] // 2, cy[odd] // 2, cz[odd] // 2], axis=1)
    hi = np.stack([(cx[odd] + 1) // 2, (cy[odd] + 1) // 2, (cz[odd] + 1) // 2], axis=1)
    ilo = lo[:, 0] + m * (lo[:, 1] + m * lo[:, 2])
    ihi = hi[:, 0] + m * (hi[:, 1] + m * hi[:, 2])
    X[odd] = 0.5 * (Xv[ilo] + Xv[ihi])
    conn = node_of_code[codes].astype(np.int32)
    e0, e1 = 6 * n * n * k0, 6 * n * n * k1
    return X, conn[e0:e1]


def tet10_plane_bounds(n: int):
    """First node id of each doubled-lattice z plane (length 2n+2) for tet10
    meshes built by ``tet10_mesh`` (for slab ownership ranges)."""
    X, conn = tet10_mesh(n, 0.0)
    z2 = np.rint(X[:, 2] * 2 * n).astype(np.int64)
    return np.searchsorted(z2, np.arange(2 * n + 2))


# --------------------------------------------------------------------------
# reference shape gradients and quadrature weights (input preparation)
# --------------------------------------------------------------------------
def _hex_dN_dxi():
    """dN_a/dxi at the 8 Gauss points: (8 qp, 8 nodes, 3)."""
    q = _HEX_QP[:, None, :]
    s = _HEX_XI[None, :, :]
    f = 1.0 + s * q  # (8,8,3)
    d = np.empty((8, 8, 3))
    d[..., 0] = 0.125 * s[..., 0] * f[..., 1] * f[..., 2]
    d[..., 1] = 0.125 * s[..., 1] * f[..., 0] * f[..., 2]
    d[..., 2] = 0.125 * s[..., 2] * f[..., 0] * f[..., 1]
    return d


def _tet10_dN_dxi():
    """dN_a/dxi (xi = barycentric L1, L2, L3) at the 4 qp: (4, 10, 3)."""
    out = np.empty((4, 10, 3))
    dL = np.array([[-1.0, -1.0, -1.0], [1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0]])
    for q in range(4):
        L = _TET_QP_BARY[q]
        for a in range(4):  # N_a = L_a(2L_a - 1)
            out[q, a] = (4.0 * L[a] - 1.0) * dL[a]
        for e, (a, b) in enumerate(_TET_EDGES):  # N_ab = 4 L_a L_b
            out[q, 4 + e] = 4.0 * (L[a] * dL[b] + L[b] * dL[a])
    return out


def shape_gradients(X: np.ndarray, conn: np.ndarray, elem_type: int, chunk: int = 1 << 17):
    """Per (element, qp): dN_a/dX (n_el, n_q, n_en, 3) and w (n_el, n_q)."""
    if elem_type == HEX8:
        dxi, gw = _hex_dN_dxi(), 1.0
    else:
        dxi, gw = _tet10_dN_dxi(), 1.0 / 24.0
    n_el, n_en = conn.shape
    n_q = dxi.shape[0]
    gradN = np.empty((n_el, n_q, n_en, 3))
    w = np.empty((n_el, n_q))
    def one(s):
        e = min(n_el, s + chunk)
        Xe = X[conn[s:e]]                                   # (b, n_en, 3)
        Jm = np.matmul(Xe.transpose(0, 2, 1)[:, None], dxi[None])   # (b, q, 3, 3): dX_i/dxi_j
        a, b_, c = Jm[..., 0, 0], Jm[..., 0, 1], Jm[..., 0, 2]
        d, e_, f = Jm[..., 1, 0], Jm[..., 1, 1], Jm[..., 1, 2]
        g, h, k = Jm[..., 2, 0], Jm[..., 2, 1], Jm[..., 2, 2]
        cof = np.stack([e_ * k - f * h, f * g - d * k, d * h - e_ * g,
                        c * h - b_ * k, a * k - c * g, b_ * g - a * h,
                        b_ * f - c * e_, c * d - a * f, a * e_ - b_ * d], axis=-1).reshape(Jm.shape)
        det = a * cof[..., 0, 0] + b_ * cof[..., 0, 1] + c * cof[..., 0, 2]
        if np.any(det <= 0):
            raise ValueError("generator produced an inverted element")
        # dN/dX = dN/dxi J^-1, J^-1 = cof^T / det
        gradN[s:e] = np.matmul(dxi[None], cof.transpose(0, 1, 3, 2) / det[..., None, None])
        w[s:e] = gw * det

    for s in range(0, n_el, chunk):
        one(s)
    return gradN, w


# --------------------------------------------------------------------------
# NCM weights and displacements
# --------------------------------------------------------------------------
def ncm_weights(width: int, n_hidden: int, std: float = 0.3, seed: int = SEED_W, kappa: float = 10.0,
                n_in: int = 3):
    """ICNN/MLP parameters drawn N(0, std^2) in the order W1, b1, W2, b2, ...,
    a (SURVEY s8(c) reading 8).  W1: (w,3); W: (L-1,w,w) row-major (out,in);
    b: (L,w); a: (w,)."""
    rng = np.random.default_rng(seed)
    w, L = width, n_hidden
    W1 = rng.normal(0.0, std, size=(w, n_in))
    b = np.empty((L, w))
    W = np.empty((max(L - 1, 0), w, w))
    b[0] = rng.normal(0.0, std, size=w)
    for l in range(1, L):
        W[l - 1] = rng.normal(0.0, std, size=(w, w))
        b[l] = rng.normal(0.0, std, size=w)
    a = rng.normal(0.0, std, size=w)
    return dict(width=w, n_hidden=L, W1=W1, W=W, b=b, a=a, skip_out=None,
                skip_hidden=None, kappa=float(kappa), ref_shift=0.0)


def cann_params(n_branch: int = 4, seed: int = SEED_W, kinematics: str = "standard", kappa: float = 10.0,
                std: float = 0.3, n_in: int = 3) -> dict:
    """CANN (Eq. cann-def) parameters: per kinematic input m and branch b the
    activation triple (f0, f1 power, f2) cycles through the paper's menus
    (f0: identity, Macaulay, abs; f1: powers 1..3; f2: linear, exp - 1, -ln(1 - .))
    with a seeded offset; w1 ~ U(0.05, 0.3) (keeps 1 - w1 x > 0 on the benchmark
    ranges), w2 ~ |N(0, std^2)|."""
    rng = np.random.default_rng(seed)
    f = np.empty((n_in, n_branch, 3), np.int32)
    off = rng.integers(0, 3, size=3)
    for m in range(n_in):
        for b in range(n_branch):
            f[m, b] = ((b + off[0] + m) % 3, 1 + (b + off[1]) % 3, (b + off[2] + 2 * m) % 3)
    w1 = rng.uniform(0.05, 0.3, size=(n_in, n_branch))
    w2 = np.abs(rng.normal(0.0, std, size=(n_in, n_branch)))
    return dict(network="cann", kinematics=kinematics, width=8, n_hidden=1, W1=None, W=None, b=None, a=None,
                skip_out=None, skip_hidden=None, cann_f=f, cann_w1=w1, cann_w2=w2, kappa=float(kappa), ref_shift=0.0)


def anisotropic(ncm: dict, a0=(0.6, 0.8, 0.0), a1=None, isochoric: bool = False) -> dict:
    """The same network on anisotropic inputs K = (I1-3, I2-3, J-1, then per pair i <= j of the
    structural vectors I4,ij - A_i.A_j, I5,ij - A_i.A_j): one vector A0 (unit: I4-1, I5-1, 5
    inputs), or two (A0, A1: pairs 00, 01, 11, 9 inputs; e.g. a fibre and a sheet direction).
    isochoric=True: the isochoric versions Ibar1, Ibar2, Ibar4,ij, Ibar5,ij (App. A.2.2)."""
    d = dict(ncm, kinematics="isochoric_anisotropic" if isochoric else "anisotropic", a0=np.array(a0, np.float64))
    if a1 is not None:
        d["a1"] = np.array(a1, np.float64)
    return d


# fibre / sheet directions of the two-vector (orthotropic) tests: unit and orthogonal
A_FIBRE, A_SHEET = (0.6, 0.8, 0.0), (0.0, 0.0, 1.0)


def gent_thomas_params(coef=(0.5, 1.0, 1.0), kappa: float = 0.0) -> dict:
    """Gent-Thomas reference model of App. C on isochoric
    kinematics: Psi = 0.5 (Ibar1 - 3) + ln(Ibar2 / 3) + (J - 1)^2."""
    return dict(network="gent_thomas", kinematics="isochoric", width=8, n_hidden=1, W1=None, W=None, b=None,
                a=None, skip_out=None, skip_hidden=None, gt=np.array(coef, np.float64), kappa=float(kappa),
                ref_shift=0.0)


def ickan_params(widths=(3, 6, 6, 1), nb: int = 8, k: int = 3, seed: int = SEED_W, kinematics: str = "standard",
                 kappa: float = 10.0, std: float = 0.3) -> dict:
    """ICKAN (App. B.3) parameters: per edge a weight |N(0, std^2)| and nb control points that
    increase with nondecreasing steps (convex, monotone: the paper's c_{i+2}-c_{i+1} >= c_{i+1}-c_i
    >= 0); knot intervals [-1, 1] for layer 0 (the invariant inputs) and [-2, 2] after it."""
    rng = np.random.default_rng(seed)
    widths = tuple(int(x) for x in widths)
    n_edges = sum(widths[r] * widths[r + 1] for r in range(len(widths) - 1))
    w = np.abs(rng.normal(0.0, std, size=n_edges))
    d0 = rng.uniform(0.0, 0.2, size=(n_edges, 1))
    steps = np.concatenate([d0, rng.uniform(0.0, 0.15, size=(n_edges, nb - 2))], axis=1).cumsum(axis=1)
    c = np.concatenate([rng.normal(0.0, std, size=(n_edges, 1)), steps], axis=1).cumsum(axis=1)
    grid = np.array([[-1.0, 1.0]] + [[-2.0, 2.0]] * (len(widths) - 2), dtype=np.float64)
    return dict(network="ickan", kinematics=kinematics, width=8, n_hidden=1, W1=None, W=None, b=None, a=None,
                skip_out=None, skip_hidden=None, kan_width=np.array(widths, np.int32), kan_nb=nb, kan_k=k,
                kan_grid=grid, kan_w=w, kan_c=np.ascontiguousarray(c), kappa=float(kappa), ref_shift=0.0)


def smooth_field(X: np.ndarray, amp: float, rng) -> np.ndarray:
    """u_i = amp * phi_i / max|phi_i|, phi_i = sum_{m<4} c sin(2 pi k.X + th),
    k uniform on {0,1}^3 minus 0, c ~ N(0,1), th ~ U[0, 2pi)."""
    ks = np.array([[a, b, c] for a in (0, 1) for b in (0, 1) for c in (0, 1)][1:], dtype=np.float64)
    u = np.empty_like(X)
    for i in range(3):
        kk = ks[rng.integers(0, 7, size=4)]
        c = rng.normal(0.0, 1.0, size=4)
        th = rng.uniform(0.0, 2.0 * math.pi, size=4)
        phi = np.zeros(X.shape[0])
        for m in range(4):
            phi += c[m] * np.sin(2.0 * math.pi * (X @ kk[m]) + th[m])
        u[:, i] = amp * phi / np.max(np.abs(phi))
    return u


def displacement(spec: ConfigSpec, X: np.ndarray, seed: int = SEED_U) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if spec.u_kind == "uniform":
        u = rng.uniform(-spec.u_amp, spec.u_amp, size=X.shape)
    elif spec.u_kind == "smooth":
        u = smooth_field(X, spec.u_amp, rng)
    elif spec.u_kind == "stretch+smooth":
        u = smooth_field(X, spec.u_amp, rng)
        u[:, 0] += 0.2 * X[:, 0]   # uniaxial stretch lambda = 1.2
    else:
        raise ValueError(spec.u_kind)
    return np.ascontiguousarray(u.reshape(-1))


# --------------------------------------------------------------------------
# one call per config
# --------------------------------------------------------------------------
def make_mesh(spec: ConfigSpec, n: int | None = None, z_range=None):
    n = spec.n if n is None else n
    if spec.elem_type == HEX8:
        return hex_mesh(n, spec.jitter, SEED_MESH, z_range)
    return tet10_mesh(n, spec.jitter, SEED_MESH, z_range)


def make_config(name: str, n: int | None = None, z_range=None, with_gradients: bool = True,
                jitter: float | None = None) -> dict:
    """Everything the boundary needs for config ``name`` (optionally resized to
    ``n`` cells per edge, or restricted to element layers ``z_range``; ``jitter``
    overrides the config's node jitter, e.g. a jittered c3 / c5 to show that the
    kernel does not depend on the regular lattice's identical element gradients)."""
    spec = CONFIGS[name]
    if jitter is not None:
        import dataclasses
        spec = dataclasses.replace(spec, jitter=float(jitter))
    X, conn = make_mesh(spec, n, z_range)
    cfg = dict(name=name, spec=spec, elem_type=spec.elem_type, n=n or spec.n,
               X=X, conn=np.ascontiguousarray(conn), n_nodes=X.shape[0],
               ncm=ncm_weights(spec.width, spec.n_hidden, spec.weight_std, SEED_W, spec.kappa),
               u=displacement(spec, X, SEED_U))
    if with_gradients:
        if spec.elem_type == HEX8 and spec.jitter == 0.0:
            # regular lattice: every element is a translate of the first, so its
            # dN/dX and w are identical -- computed once, stored per element
            # (the kernel still streams the full per-element array)
            g1, w1 = shape_gradients(X, conn[:1], spec.elem_type)
            cfg["gradN"] = np.empty((conn.shape[0],) + g1.shape[1:])
            cfg["gradN"][:] = g1
            cfg["qp_w"] = np.empty((conn.shape[0], w1.shape[1]))
            cfg["qp_w"][:] = w1
        else:
            cfg["gradN"], cfg["qp_w"] = shape_gradients(X, conn, spec.elem_type)
    return cfg


def element_colours_hex(n: int) -> np.ndarray:
    """Not used by either side (each builds its own colouring); kept for tests
    that want an independent structured 8-colouring."""
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    return ((i % 2) + 2 * (j % 2) + 4 * (k % 2)).ravel()


# --------------------------------------------------------------------------
# z-slab partition (multi-GPU input preparation)
# --------------------------------------------------------------------------
def slab_layers(n: int, P: int, r: int):
    if P > n:
        raise ValueError(f"{P} slabs for {n} element layers")
    return r * n // P, (r + 1) * n // P


def rank_node_begin(elem_type: int, n: int, P: int) -> np.ndarray:
    """Ownership boundaries: rank r owns the node planes of its element layers
    (z-major numbering), the last rank also the top plane."""
    out = np.zeros(P + 1, np.int64)
    if elem_type == HEX8:
        m = n + 1
        for r in range(P):
            out[r] = slab_layers(n, P, r)[0] * m * m
        out[P] = m ** 3
    else:
        bounds = tet10_plane_bounds(n)
        for r in range(P):
            out[r] = bounds[2 * slab_layers(n, P, r)[0]]
        out[P] = bounds[-1]
    return out


def slab_partition(name: str, P: int, r: int, n: int | None = None, with_gradients: bool = True) -> dict:
    """Rank r's share of config `name` split into P z-slabs: its elements (with
    dN/dX, w), its owned node range, the ownership table and its ghost elements
    (the layer below, assembled by the rank beneath)."""
    spec = CONFIGS[name]
    n = spec.n if n is None else n
    k0, k1 = slab_layers(n, P, r)
    cfg = make_config(name, n=n, z_range=(k0, k1), with_gradients=with_gradients)
    rnb = rank_node_begin(spec.elem_type, n, P)
    cfg.update(n_ranks=P, rank=r, rank_node_begin=rnb, owned_node_begin=int(rnb[r]), owned_node_end=int(rnb[r + 1]))
    if r > 0:
        _, gconn = make_mesh(spec, n, (k0 - 1, k0))
        below = [q for q in range(P) if slab_layers(n, P, q)[0] <= k0 - 1 < slab_layers(n, P, q)[1]][0]
        cfg["ghost_conn"] = np.ascontiguousarray(gconn)
        cfg["ghost_rank"] = np.full(gconn.shape[0], below, np.int32)
    else:
        cfg["ghost_conn"] = np.zeros((0, cfg["conn"].shape[1]), np.int32)
        cfg["ghost_rank"] = np.zeros(0, np.int32)
    return cfg
