"""Hyper-dual numbers (a + b e1 + c e2 + d e1 e2, e1^2 = e2^2 = 0) for exact
first and second derivatives of W(F) straight from its definition -- an
independent derivation used to PIN the oracle's G-tensor algebra (no shared
code with oracle/ or the CUDA path).

Only what W(F) = N(k(F)) + kappa (J-1)^2 - s0 (J-1) needs: +, -, *, softplus,
powers, exp, log and the CANN activations (for the isochoric / CANN /
Gent-Thomas variants of SURVEY.md s8(f) rank 2).
Every component is a numpy array so all 81 direction pairs run at once.
"""
from __future__ import annotations

import numpy as np


class HD:
    __slots__ = ("a", "b", "c", "d")

    def __init__(self, a, b=0.0, c=0.0, d=0.0):
        self.a, self.b, self.c, self.d = a, b, c, d

    @staticmethod
    def lift(x):
        return x if isinstance(x, HD) else HD(x)

    def __add__(self, o):
        o = HD.lift(o)
        return HD(self.a + o.a, self.b + o.b, self.c + o.c, self.d + o.d)

    __radd__ = __add__

    def __neg__(self):
        return HD(-self.a, -self.b, -self.c, -self.d)

    def __sub__(self, o):
        return self + (-HD.lift(o))

    def __rsub__(self, o):
        return HD.lift(o) - self

    def __mul__(self, o):
        o = HD.lift(o)
        return HD(self.a * o.a, self.a * o.b + self.b * o.a, self.a * o.c + self.c * o.a,
                  self.a * o.d + self.b * o.c + self.c * o.b + self.d * o.a)

    __rmul__ = __mul__

    def apply(self, f0, f1, f2):
        """f(x) with f' = f1, f'' = f2 evaluated at the real part."""
        fa, d1, d2 = f0(self.a), f1(self.a), f2(self.a)
        return HD(fa, d1 * self.b, d1 * self.c, d1 * self.d + d2 * self.b * self.c)


def _sig(y):
    return np.where(y >= 0, 1.0 / (1.0 + np.exp(-np.abs(y))), np.exp(-np.abs(y)) / (1.0 + np.exp(-np.abs(y))))


def softplus(x: HD) -> HD:
    return x.apply(lambda y: np.maximum(y, 0) + np.log1p(np.exp(-np.abs(y))), _sig,
                   lambda y: _sig(y) * (1.0 - _sig(y)))


def hd_pow(x: HD, p: float) -> HD:
    return x.apply(lambda a: a ** p, lambda a: p * a ** (p - 1), lambda a: p * (p - 1) * a ** (p - 2))


def hd_exp(x: HD) -> HD:
    return x.apply(np.exp, np.exp, np.exp)


def hd_log(x: HD) -> HD:
    return x.apply(np.log, lambda a: 1.0 / a, lambda a: -1.0 / (a * a))


def _cann_hd(k, ncm):
    """N = sum_m sum_b w2 f2(f1(f0(K_m))) written from Eq. cann-def / cann-fs."""
    f, w1, w2 = ncm["cann_f"], ncm["cann_w1"], ncm["cann_w2"]
    N = HD(0.0)
    for m in range(len(k)):
        for b in range(f.shape[1]):
            t0, p, t2 = f[m, b]
            x = k[m]
            if t0 == 1:
                x = x.apply(lambda a: np.maximum(a, 0.0), lambda a: 0.5 * (1 + np.sign(a)), lambda a: 0.0 * a)
            elif t0 == 2:
                x = x.apply(np.abs, np.sign, lambda a: 0.0 * a)
            y = HD(1.0)
            for _ in range(p):
                y = y * x
            if t2 == 0:
                z = w1[m, b] * y
            elif t2 == 1:
                z = hd_exp(w1[m, b] * y) - 1.0
            else:
                z = -1.0 * hd_log(1.0 - w1[m, b] * y)
            N = N + w2[m, b] * z
    return N


def _bspline(c, k, t, span, x):
    """sum_i c_i B_{i,k}(x) by De Boor's recursion (B_{i,0} = 1 on the given knot span);
    x may be a float or an HD number."""
    nt = len(t)
    B = [HD(1.0) if i == span else HD(0.0) for i in range(nt)]
    for p in range(1, k + 1):
        Bn = []
        for i in range(nt - p - 1):
            v = HD(0.0)
            if t[i + p] > t[i]:
                v = v + (x - t[i]) * (1.0 / (t[i + p] - t[i])) * B[i]
            if t[i + p + 1] > t[i + 1]:
                v = v + (t[i + p + 1] - x) * (1.0 / (t[i + p + 1] - t[i + 1])) * B[i + 1]
            Bn.append(v)
        B = Bn
    return sum((c[i] * B[i] for i in range(len(c))), HD(0.0))


def _spline_hd(c, k, xmin, xmax, x: HD) -> HD:
    nb = len(c)
    h = (xmax - xmin) / (nb - k)
    t = [xmin + (i - k) * h for i in range(nb + k + 1)]
    xa = float(np.ravel(x.a)[0])
    xe = min(max(xa, xmin), xmax)
    span = k
    while span < nb - 1 and xe >= t[span + 1]:
        span += 1
    if xe == xa:
        return _bspline(c, k, t, span, x)
    # linear continuation with the end value and slope (one dual direction at the boundary)
    e = _bspline(c, k, t, span, HD(xe, 1.0, 0.0, 0.0))
    return e.a + e.b * (x - xe)


def _ickan_hd(k, ncm):
    widths, nb, kk = list(ncm["kan_width"]), int(ncm["kan_nb"]), int(ncm["kan_k"])
    z = list(k)
    e = 0
    for r in range(len(widths) - 1):
        xmin, xmax = ncm["kan_grid"][r]
        y = []
        for i in range(widths[r + 1]):
            s = HD(0.0)
            for j in range(widths[r]):
                s = s + ncm["kan_w"][e] * _spline_hd(ncm["kan_c"][e], kk, xmin, xmax, z[j])
                e += 1
            y.append(s)
        z = y
    return z[0]


def energy_hd(F: list, ncm: dict):
    """W(F) for a 3x3 list-of-lists of HD; written from the definitions:
    C = F^T F, I1 = tr C, I2 = (I1^2 - tr C^2)/2, J = det F (Sarrus),
    MLP/ICNN of Eq. icnn with softplus, penalty kappa (J-1)^2 - s0 (J-1)."""
    Cm = [[sum((F[i][I] * F[i][J] for i in range(3)), HD(0.0)) for J in range(3)] for I in range(3)]
    I1 = Cm[0][0] + Cm[1][1] + Cm[2][2]
    trC2 = sum((Cm[I][J] * Cm[J][I] for I in range(3) for J in range(3)), HD(0.0))
    I2 = 0.5 * (I1 * I1 - trC2)
    J = (F[0][0] * F[1][1] * F[2][2] + F[0][1] * F[1][2] * F[2][0] + F[0][2] * F[1][0] * F[2][1]
         - F[0][2] * F[1][1] * F[2][0] - F[0][0] * F[1][2] * F[2][1] - F[0][1] * F[1][0] * F[2][2])
    k = [I1 - 3.0, I2 - 3.0, J - 1.0]
    kin = ncm.get("kinematics", "standard")
    if kin in ("anisotropic", "isochoric_anisotropic"):
        # Eq. standard-inv-II: I4,ij = A_i . C A_j, I5,ij = A_i . C^2 A_j over the pairs i <= j
        # of the structural vectors; inputs I4,ij - A_i.A_j, I5,ij - A_i.A_j (zero at F = I).
        # Isochoric (App. A.2.2): Ibar_m = I3^e_m I_m, e = -1/3 (I1, I4,ij), -2/3 (I2, I5,ij); I3^-1/3 = J^-2/3
        s1 = hd_pow(J, -2.0 / 3.0) if kin == "isochoric_anisotropic" else HD(1.0)
        s2 = s1 * s1
        vecs = [np.asarray(ncm["a0"], float)] + ([np.asarray(ncm["a1"], float)] if ncm.get("a1") is not None else [])
        CAs = [[sum((Cm[I][Jx] * v[Jx] for Jx in range(3)), HD(0.0)) for I in range(3)] for v in vecs]
        k = [s1 * I1 - 3.0, s2 * I2 - 3.0, J - 1.0]
        for i in range(len(vecs)):
            for j in range(i, len(vecs)):
                aa = float(vecs[i] @ vecs[j])
                I4 = sum((vecs[i][I] * CAs[j][I] for I in range(3)), HD(0.0))
                I5 = sum((CAs[i][I] * CAs[j][I] for I in range(3)), HD(0.0))
                k += [s1 * I4 - aa, s2 * I5 - aa]
    if ncm.get("kinematics", "standard") == "isochoric":
        a23 = hd_pow(J, -2.0 / 3.0)
        k = [a23 * I1 - 3.0, a23 * a23 * I2 - 3.0, J - 1.0]
    kap, s0 = ncm.get("kappa", 0.0), ncm.get("ref_shift", 0.0)
    net = ncm.get("network", "icnn")
    if net == "cann":
        N = _cann_hd(k, ncm)
        if ncm.get("skip_out") is not None:
            for i in range(3):
                N = N + ncm["skip_out"][i] * k[i]
        return N + kap * (J - 1.0) * (J - 1.0) - s0 * (J - 1.0)
    if net == "ickan":
        N = _ickan_hd(k, ncm)
        return N + kap * (J - 1.0) * (J - 1.0) - s0 * (J - 1.0)
    if net == "gent_thomas":
        c = ncm["gt"]
        N = c[0] * k[0] + c[1] * hd_log((k[1] + 3.0) * (1.0 / 3.0)) + c[2] * k[2] * k[2]
        return N + kap * (J - 1.0) * (J - 1.0) - s0 * (J - 1.0)
    W1, b, a = ncm["W1"], ncm["b"], ncm["a"]
    L, w = ncm["n_hidden"], ncm["width"]
    Wh = ncm.get("W")
    Bh = ncm.get("skip_hidden")
    z = [sum((W1[j, i] * k[i] for i in range(len(k))), HD(0.0)) + b[0, j] for j in range(w)]
    z = [softplus(v) for v in z]
    for l in range(1, L):
        y = []
        for j in range(w):
            s = HD(b[l, j])
            for i in range(w):
                s = s + Wh[l - 1, j, i] * z[i]
            if Bh is not None:
                for i in range(3):
                    s = s + Bh[l - 1, j, i] * k[i]
            y.append(s)
        z = [softplus(v) for v in y]
    N = sum((a[j] * z[j] for j in range(w)), HD(0.0))
    if ncm.get("skip_out") is not None:
        for i in range(3):
            N = N + ncm["skip_out"][i] * k[i]
    kap, s0 = ncm.get("kappa", 0.0), ncm.get("ref_shift", 0.0)
    return N + kap * (J - 1.0) * (J - 1.0) - s0 * (J - 1.0)


def derivatives(F0: np.ndarray, ncm: dict):
    """-> (W, P = dW/dF (3x3), A = d2W/dFdF (3x3x3x3)) exactly (to rounding)."""
    idx = np.arange(81)
    p, q = idx // 9, idx % 9
    F = [[HD(np.full(81, F0[i, J]), (p == 3 * i + J).astype(float), (q == 3 * i + J).astype(float),
             np.zeros(81)) for J in range(3)] for i in range(3)]
    W = energy_hd(F, ncm)
    P = np.zeros(9)
    for pp in range(9):
        P[pp] = W.b[pp * 9]
    A = W.d.reshape(9, 9)
    return float(W.a[0]), P.reshape(3, 3), A.reshape(3, 3, 3, 3)
