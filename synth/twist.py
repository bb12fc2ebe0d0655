"""Seeded inputs of the twist-cube benchmark (Fig. 7: "a unit
cube, fixed at one end, and subjected to a unit axial tensile displacement and a
half-rotation at the opposite end").  Problem data only -- mesh, NCM parameters,
constrained DOFs and their prescribed values -- no method arithmetic; shared by
the oracle tests and the GPU path.

Readings (R18-R21): the fixed end is z = 0 (all three components
zero), the moving end z = 1; both the axial displacement and the rotation angle
about the axis x = y = 1/2 are ramped linearly with the load factor t in (0, 1]
(SPEC's reading; the paper does not say); lateral faces are traction free.
The paper's trained NCM is unavailable: a stable stand-in is an input-convex
network (non-negative weights on I1 - 3, I2 - 3 and on every hidden and output
layer) so that W is polyconvex.
"""
from __future__ import annotations

import math

import numpy as np

from synth.gen import HEX8, SEED_W, hex_mesh, shape_gradients


def stable_ncm(width: int = 16, n_hidden: int = 2, std: float = 0.3, seed: int = SEED_W,
               kappa: float = 10.0) -> dict:
    """Convex, nondecreasing-in-(I1, I2) ICNN: |N(0, std^2)| on W1[:, :2], every
    hidden W_l and a; N(0, std^2) on W1[:, 2] and the biases (drawn in the
    order W1, b1, W2, b2, ..., a)."""
    rng = np.random.default_rng(seed)
    w, L = width, n_hidden
    W1 = rng.normal(0.0, std, size=(w, 3))
    W1[:, :2] = np.abs(W1[:, :2])
    b = np.empty((L, w))
    W = np.empty((max(L - 1, 0), w, w))
    b[0] = rng.normal(0.0, std, size=w)
    for l in range(1, L):
        W[l - 1] = np.abs(rng.normal(0.0, std, size=(w, w)))
        b[l] = rng.normal(0.0, std, size=w)
    a = np.abs(rng.normal(0.0, std, size=w))
    return dict(width=w, n_hidden=L, W1=W1, W=W, b=b, a=a, skip_out=None, skip_hidden=None,
                kappa=float(kappa), ref_shift=0.0)


def twist_mesh(n: int) -> dict:
    X, conn = hex_mesh(n, 0.0)
    gN, w = shape_gradients(X, conn, HEX8)
    return dict(elem_type=HEX8, n=n, X=X, conn=np.ascontiguousarray(conn), n_nodes=X.shape[0],
                gradN=gN, qp_w=w)


def twist_bc(X: np.ndarray):
    """Constrained global dofs: every component of the nodes on z = 0 and z = 1."""
    bottom = np.nonzero(np.abs(X[:, 2]) < 1e-12)[0]
    top = np.nonzero(np.abs(X[:, 2] - 1.0) < 1e-12)[0]
    nodes = np.concatenate([bottom, top])
    dofs = (3 * nodes[:, None] + np.arange(3)[None, :]).reshape(-1)
    return dofs.astype(np.int64), bottom, top


def twist_values(X: np.ndarray, dofs: np.ndarray, t: float, stretch: float = 1.0,
                 turns: float = 0.5) -> np.ndarray:
    """Prescribed displacement of the constrained dofs at load factor t:
    bottom 0; top x -> R(t * turns * 2 pi)(x - c) + c + t * stretch * e_z."""
    nodes = dofs // 3
    comp = dofs % 3
    Xn = X[nodes]
    th = t * turns * 2.0 * math.pi
    cx, cy = 0.5, 0.5
    dx, dy = Xn[:, 0] - cx, Xn[:, 1] - cy
    ux = cx + math.cos(th) * dx - math.sin(th) * dy - Xn[:, 0]
    uy = cy + math.sin(th) * dx + math.cos(th) * dy - Xn[:, 1]
    uz = np.full(Xn.shape[0], t * stretch)
    top = np.abs(Xn[:, 2] - 1.0) < 1e-12
    u = np.where(comp == 0, ux, np.where(comp == 1, uy, uz))
    return np.where(top, u, 0.0)


def uniaxial_problem(stretch: float):
    """One unit hex element with roller conditions: u_x = 0 on x = 0, u_y = 0 on
    y = 0, u_z = 0 on z = 0 and u_z = stretch - 1 on z = 1 (homogeneous uniaxial
    tension with free lateral faces)."""
    X, conn = hex_mesh(1, 0.0)
    gN, w = shape_gradients(X, conn, HEX8)
    dofs, vals = [], []
    for a in range(X.shape[0]):
        for i in range(3):
            if abs(X[a, i]) < 1e-12:
                dofs.append(3 * a + i)
                vals.append(0.0)
        if abs(X[a, 2] - 1.0) < 1e-12:
            dofs.append(3 * a + 2)
            vals.append(stretch - 1.0)
    return (dict(elem_type=HEX8, n=1, X=X, conn=np.ascontiguousarray(conn), n_nodes=X.shape[0], gradN=gN,
                 qp_w=w), np.array(dofs, np.int64), np.array(vals))
