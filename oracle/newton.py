"""Oracle of the Newton-Raphson step around the assembly.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy/scipy on top of
the plain-C oracle assembly; shares no code with the CUDA path.

  d <- d + Delta d,  K Delta d = -r                    (s2.1)

Dirichlet dofs are eliminated symmetrically (rows and columns zeroed, unit
diagonal, zero residual -- DESIGN.md reading R19); the linear system is solved
by a direct sparse factorisation (scipy spsolve: a library primitive), and,
separately, by the textbook Jacobi-preconditioned CG that
the GPU path implements, for its own pins.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle


def eliminate(row_ptr, col_idx, vals, r, mask):
    """Symmetric elimination of the constrained dofs (mask: bool per dof)."""
    vals = vals.copy()
    rows = np.repeat(np.arange(row_ptr.size - 1), np.diff(row_ptr))
    sel = mask[rows] | mask[col_idx]
    vals[sel] = np.where(rows[sel] == col_idx[sel], 1.0, 0.0)
    r = None if r is None else np.where(mask, 0.0, r)
    return vals, r


def block_diag_inverse(A, bs=3):
    """M^-1 for block Jacobi: the inverses of the bs x bs diagonal blocks of A (dense,
    numpy.linalg.inv per block) as a block-diagonal sparse matrix."""
    A = sp.csr_matrix(A)
    n = A.shape[0]
    blocks = [np.linalg.inv(A[i:i + bs, i:i + bs].toarray()) for i in range(0, n, bs)]
    return sp.block_diag(blocks, format="csr")


def cg_jacobi(A, b, rtol=1e-10, max_iter=100000, block=False):
    """Textbook preconditioned CG (Saad, Alg. 9.1), M = diag(A) -- the paper's choice
     -- or, block=True, the 3x3 nodal diagonal blocks of A.  -> (x, iters)."""
    A = sp.csr_matrix(A)
    if block:
        Minv = block_diag_inverse(A)
        prec = lambda v: Minv @ v  # noqa: E731
    else:
        dinv = 1.0 / A.diagonal()
        prec = lambda v: dinv * v  # noqa: E731
    x = np.zeros_like(b)
    r = b.copy()
    z = prec(r)
    p = z.copy()
    rz = r @ z
    bb = b @ b
    if bb == 0.0:
        return x, 0
    for it in range(1, max_iter + 1):
        q = A @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        if r @ r <= rtol * rtol * bb:
            return x, it
        z = prec(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    raise RuntimeError("cg_jacobi: no convergence in %d iterations" % max_iter)


def reference_shift(ncm: dict) -> float:
    """s0 with S(F = I) = 0 once W gets -s0 (J - 1) (R11).  At F = I the
    term adds -s0 J C^-1 = -s0 I to S, and S(I) = sigma I for an isotropic W, so
    s0 = S_11(I) of the unshifted model (= 2 g1 + 4 g2 + g3 for standard inputs)."""
    return float(oracle.material_point(dict(ncm, ref_shift=0.0), np.eye(3))["S"][0, 0])


def newton_step(ncm, mesh, row_ptr, col_idx, u, dofs, values, atol=1e-10, rtol=1e-10, max_iter=30):
    """One load step to u[dofs] = values by Newton iterations with a direct solve.
    The first iteration is the consistent predictor (R20): K and r at the
    previous u, the prescribed increment dc moved to the right-hand side,
      K_ff du_f = -(r + K dc)_f,
    so no assembly happens at the jumped boundary configuration; the others are
    plain Newton on the free dofs.  -> (u, residual norms, converged)."""
    u = u.copy()
    n = u.size
    mask = np.zeros(n, bool)
    mask[dofs] = True
    dc = np.zeros(n)
    dc[dofs] = values - u[dofs]
    norms = []
    for it in range(max_iter + 1):
        r, vals, bad = oracle.assemble(ncm, mesh["n_nodes"], mesh["conn"], mesh["gradN"], mesh["qp_w"], u,
                                       row_ptr, col_idx)
        if bad != -1:
            raise RuntimeError("det F <= 0 at flat qp %d" % bad)
        if it == 0:
            r = r + sp.csr_matrix((vals, col_idx, row_ptr), shape=(n, n)) @ dc
            u[dofs] = values
        vals, r = eliminate(row_ptr, col_idx, vals, r, mask)
        nrm = float(np.linalg.norm(r))
        norms.append(nrm)
        if nrm <= max(atol, rtol * norms[0]):
            return u, norms, True
        if it == max_iter:
            break
        K = sp.csr_matrix((vals, col_idx, row_ptr), shape=(n, n))
        u -= spla.spsolve(K.tocsc(), r)
    return u, norms, False


def max_trace_C(mesh, u) -> float:
    F = oracle.qp_F(mesh["conn"], mesh["gradN"], u)
    C = np.einsum("eqiI,eqiJ->eqIJ", F, F)
    return float(np.max(np.trace(C, axis1=2, axis2=3)))
