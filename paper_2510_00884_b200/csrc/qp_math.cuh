// qp_math.cuh -- per-quadrature-point kinematics and stress/tangent algebra of
// the CUDA path.  Independent of
// oracle/ (different formulation: the tangent is assembled directly in
// F-space from structured rank-one terms instead of a 3^4 material tensor).
//
//  k = (I1-3, I2-3, J-1),  h1 = I, h2 = I1 I - C, h3 = J/2 C^-1
//  S = 2 (g1 h1 + g2 h2 + g3 h3)                    (Eq. stress-cgo)
//  A_iJkL = d_ik S_JL + F_iI CC_IJKL F_kK           (Eq. p-stiffness)
// with CC = 4 sum H_mn h_m (x) h_n + 4 sum g_m HH_m (Eq. stiffnes-cgo),
// pushed through F analytically (Phi_m = F h_m, F^-T = cof F / J):
//  A = d_ik T_JL + 4 sum_mn H'_mn Phi_m,iJ Phi_n,kL
//      - 2 g2 (b_ik d_JL + F_iL F_kJ) - g3 J F^-T_iL F^-T_kJ
//  Phi_1 = F, Phi_2 = I1 F - F C, Phi_3 = J/2 F^-T,
//  H' = H + diag(g2, 0, g3/J),  T = S - g3 J C^-1,  b = F F^T.
#pragma once
#include <cmath>
#include <cstdint>

namespace commet {

struct Kin {
  double F[9];     // row-major F[i*3+J]
  double C[9];
  double I1, I2, J;
  double FiT[9];   // F^-T
  double Ci[9];    // C^-1
};

__device__ __forceinline__ void kinematics(const double* __restrict__ F, Kin& k) {
#pragma unroll
  for (int i = 0; i < 9; i++) k.F[i] = F[i];
#pragma unroll
  for (int I = 0; I < 3; I++)
#pragma unroll
    for (int J = 0; J < 3; J++)
      k.C[I * 3 + J] = F[0 * 3 + I] * F[0 * 3 + J] + F[1 * 3 + I] * F[1 * 3 + J] + F[2 * 3 + I] * F[2 * 3 + J];
  // cofactor matrix of F: cof_iJ; det F = sum_J F_0J cof_0J
  double cof[9];
  cof[0] = F[4] * F[8] - F[5] * F[7];
  cof[1] = F[5] * F[6] - F[3] * F[8];
  cof[2] = F[3] * F[7] - F[4] * F[6];
  cof[3] = F[2] * F[7] - F[1] * F[8];
  cof[4] = F[0] * F[8] - F[2] * F[6];
  cof[5] = F[1] * F[6] - F[0] * F[7];
  cof[6] = F[1] * F[5] - F[2] * F[4];
  cof[7] = F[2] * F[3] - F[0] * F[5];
  cof[8] = F[0] * F[4] - F[1] * F[3];
  k.J = F[0] * cof[0] + F[1] * cof[1] + F[2] * cof[2];
  const double iJ = 1.0 / k.J;
#pragma unroll
  for (int i = 0; i < 9; i++) k.FiT[i] = cof[i] * iJ;
  // C^-1 = F^-1 F^-T ; (F^-1)_Ii = (F^-T)_iI
#pragma unroll
  for (int I = 0; I < 3; I++)
#pragma unroll
    for (int J = 0; J < 3; J++)
      k.Ci[I * 3 + J] = k.FiT[0 * 3 + I] * k.FiT[0 * 3 + J] + k.FiT[1 * 3 + I] * k.FiT[1 * 3 + J] +
                        k.FiT[2 * 3 + I] * k.FiT[2 * 3 + J];
  k.I1 = k.C[0] + k.C[4] + k.C[8];
  double trC2 = 0.0;
#pragma unroll
  for (int I = 0; I < 3; I++)
#pragma unroll
    for (int J = 0; J < 3; J++) trC2 += k.C[I * 3 + J] * k.C[I * 3 + J];
  k.I2 = 0.5 * (k.I1 * k.I1 - trC2);
}

// Per-qp part of the tangent: from g[3] = dW/dk and H[6] = d2W/dk2 (upper
// 00,01,02,11,12,22; penalty included) and the weight w, writes
//   post[0..8] F, [9..17] F^-T, [18..26] w T, [27..53] Phi_m, [54..80] Psi_m = 4w sum_n H'_mn Phi_n,
//   [81..89] b = F F^T, [90] c2 = -2 g2 w, [91] c3 = -g3 J w;   P[9] = w F S.
__device__ __forceinline__ void post_qp(const Kin& k, const double* __restrict__ g, const double* __restrict__ H6,
                                        double w, double* __restrict__ post, double* __restrict__ P) {
  const double* F = k.F;
  const double hJ = 0.5 * k.J;
  double S[9];
#pragma unroll
  for (int I = 0; I < 3; I++)
#pragma unroll
    for (int J = 0; J < 3; J++) {
      const double d = (I == J) ? 1.0 : 0.0;
      S[I * 3 + J] = 2.0 * (g[0] * d + g[1] * (k.I1 * d - k.C[I * 3 + J]) + g[2] * hJ * k.Ci[I * 3 + J]);
      post[18 + I * 3 + J] = w * (S[I * 3 + J] - g[2] * k.J * k.Ci[I * 3 + J]);
    }
  double Phi[3][9];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int J = 0; J < 3; J++) {
      const double FC = F[i * 3 + 0] * k.C[0 * 3 + J] + F[i * 3 + 1] * k.C[1 * 3 + J] + F[i * 3 + 2] * k.C[2 * 3 + J];
      Phi[0][i * 3 + J] = F[i * 3 + J];
      Phi[1][i * 3 + J] = k.I1 * F[i * 3 + J] - FC;
      Phi[2][i * 3 + J] = hJ * k.FiT[i * 3 + J];
    }
  double Hp[9];
  Hp[0] = H6[0] + g[1]; Hp[1] = H6[1]; Hp[2] = H6[2];
  Hp[3] = H6[1]; Hp[4] = H6[3]; Hp[5] = H6[4];
  Hp[6] = H6[2]; Hp[7] = H6[4]; Hp[8] = H6[5] + g[2] / k.J;
  const double w4 = 4.0 * w;
#pragma unroll
  for (int x = 0; x < 9; x++) {
    post[x] = F[x];
    post[9 + x] = k.FiT[x];
    post[27 + x] = Phi[0][x];
    post[36 + x] = Phi[1][x];
    post[45 + x] = Phi[2][x];
#pragma unroll
    for (int m = 0; m < 3; m++)
      post[54 + m * 9 + x] = w4 * (Hp[m * 3 + 0] * Phi[0][x] + Hp[m * 3 + 1] * Phi[1][x] + Hp[m * 3 + 2] * Phi[2][x]);
  }
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int kk = 0; kk < 3; kk++)
      post[81 + i * 3 + kk] = F[i * 3 + 0] * F[kk * 3 + 0] + F[i * 3 + 1] * F[kk * 3 + 1] + F[i * 3 + 2] * F[kk * 3 + 2];
  post[90] = -2.0 * g[1] * w;
  post[91] = -g[2] * k.J * w;
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int J = 0; J < 3; J++)
      P[i * 3 + J] = w * (F[i * 3 + 0] * S[0 * 3 + J] + F[i * 3 + 1] * S[1 * 3 + J] + F[i * 3 + 2] * S[2 * 3 + J]);
}

// post_qp split over four cooperating warps (part = warp index, one lane per qp): the same
// outputs, each part a quarter of the work after its own copy of the kinematics --
//   part 0: F, F^-T, b, c2, c3 and P = w F S;  part 1: T = w (S - g3 J C^-1), Phi_m, Psi_0;
//   part 2: Psi_1;  part 3: Psi_2
__device__ __forceinline__ void post_qp_part(const Kin& k, const double* __restrict__ g,
                                             const double* __restrict__ H6, double w, double* __restrict__ post,
                                             double* __restrict__ P, int part) {
  const double* F = k.F;
  const double hJ = 0.5 * k.J;
  if (part <= 1) {
    double S[9];
#pragma unroll
    for (int I = 0; I < 3; I++)
#pragma unroll
      for (int J = 0; J < 3; J++) {
        const double d = (I == J) ? 1.0 : 0.0;
        S[I * 3 + J] = 2.0 * (g[0] * d + g[1] * (k.I1 * d - k.C[I * 3 + J]) + g[2] * hJ * k.Ci[I * 3 + J]);
      }
    if (part == 0) {
#pragma unroll
      for (int x = 0; x < 9; x++) {
        post[x] = F[x];
        post[9 + x] = k.FiT[x];
      }
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int kk = 0; kk < 3; kk++)
          post[81 + i * 3 + kk] = F[i * 3 + 0] * F[kk * 3 + 0] + F[i * 3 + 1] * F[kk * 3 + 1] + F[i * 3 + 2] * F[kk * 3 + 2];
      post[90] = -2.0 * g[1] * w;
      post[91] = -g[2] * k.J * w;
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int J = 0; J < 3; J++)
          P[i * 3 + J] = w * (F[i * 3 + 0] * S[0 * 3 + J] + F[i * 3 + 1] * S[1 * 3 + J] + F[i * 3 + 2] * S[2 * 3 + J]);
      return;
    }
#pragma unroll
    for (int x = 0; x < 9; x++) post[18 + x] = w * (S[x] - g[2] * k.J * k.Ci[x]);
  }
  double Phi[3][9];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int J = 0; J < 3; J++) {
      const double FC = F[i * 3 + 0] * k.C[0 * 3 + J] + F[i * 3 + 1] * k.C[1 * 3 + J] + F[i * 3 + 2] * k.C[2 * 3 + J];
      Phi[0][i * 3 + J] = F[i * 3 + J];
      Phi[1][i * 3 + J] = k.I1 * F[i * 3 + J] - FC;
      Phi[2][i * 3 + J] = hJ * k.FiT[i * 3 + J];
    }
  // row m of H' = H + diag(g2, 0, g3/J)
  const int m = part == 1 ? 0 : part - 1;
  double hp[3];
  if (m == 0) { hp[0] = H6[0] + g[1]; hp[1] = H6[1]; hp[2] = H6[2]; }
  else if (m == 1) { hp[0] = H6[1]; hp[1] = H6[3]; hp[2] = H6[4]; }
  else { hp[0] = H6[2]; hp[1] = H6[4]; hp[2] = H6[5] + g[2] / k.J; }
  const double w4 = 4.0 * w;
#pragma unroll
  for (int x = 0; x < 9; x++) {
    if (part == 1) {
      post[27 + x] = Phi[0][x];
      post[36 + x] = Phi[1][x];
      post[45 + x] = Phi[2][x];
    }
    post[54 + m * 9 + x] = w4 * (hp[0] * Phi[0][x] + hp[1] * Phi[1][x] + hp[2] * Phi[2][x]);
  }
}

// Row iJ of w A:  A_iJkL = 4 sum_m Phi_m,iJ Psi_m,kL / (4w) ... (see header), kL = 0..8
__device__ __forceinline__ void tangent_row(const double* __restrict__ post, int iJ, double* __restrict__ out) {
  const int i = iJ / 3, J = iJ % 3;
  const double p0 = post[27 + iJ], p1 = post[36 + iJ], p2 = post[45 + iJ];
  const double c2 = post[90], c3 = post[91];
#pragma unroll
  for (int kk = 0; kk < 3; kk++) {
    const double FkJ = post[kk * 3 + J], GkJ = post[9 + kk * 3 + J];
#pragma unroll
    for (int L = 0; L < 3; L++) {
      const int kL = kk * 3 + L;
      double v = p0 * post[54 + kL] + p1 * post[63 + kL] + p2 * post[72 + kL];
      v += c2 * post[i * 3 + L] * FkJ + c3 * post[9 + i * 3 + L] * GkJ;
      if (J == L) v += c2 * post[81 + i * 3 + kk];
      if (i == kk) v += post[18 + J * 3 + L];
      out[kL] = v;
    }
  }
}

// Rows (i, J = 0..2) of w A (27 entries, out[J * 9 + kL]) -- tangent_row for three rows sharing
// their loads (Psi_m, F^-T, b, T of the qp are read once for the three rows)
__device__ __forceinline__ void tangent_rows_i(const double* __restrict__ post, int i, double* __restrict__ out) {
  const double c2 = post[90], c3 = post[91];
  double FiL[3], GiL[3], bik[3];
#pragma unroll
  for (int x = 0; x < 3; x++) {
    FiL[x] = post[i * 3 + x];
    GiL[x] = post[9 + i * 3 + x];
    bik[x] = post[81 + i * 3 + x];
  }
  double p[3][3];
#pragma unroll
  for (int J = 0; J < 3; J++) {
    p[J][0] = post[27 + i * 3 + J];
    p[J][1] = post[36 + i * 3 + J];
    p[J][2] = post[45 + i * 3 + J];
  }
#if COMMET_T7_ROLL
#pragma unroll 1
#else
#pragma unroll
#endif
  for (int kk = 0; kk < 3; kk++) {
    double FkJ[3], GkJ[3];
#pragma unroll
    for (int J = 0; J < 3; J++) {
      FkJ[J] = post[kk * 3 + J];
      GkJ[J] = post[9 + kk * 3 + J];
    }
#pragma unroll
    for (int L = 0; L < 3; L++) {
      const int kL = kk * 3 + L;
      const double s0 = post[54 + kL], s1 = post[63 + kL], s2 = post[72 + kL];
#pragma unroll
      for (int J = 0; J < 3; J++) {
        double v = p[J][0] * s0 + p[J][1] * s1 + p[J][2] * s2;
        v += c2 * FiL[L] * FkJ[J] + c3 * GiL[L] * GkJ[J];
        if (J == L) v += c2 * bik[kk];
        if (i == kk) v += post[18 + J * 3 + L];
        out[J * 9 + kL] = v;
      }
    }
  }
}

// Whole tangent of one qp (simple kernel): P[9] and A[81], both scaled by w.
__device__ __forceinline__ void stress_tangent(const Kin& k, const double* __restrict__ g,
                                               const double* __restrict__ H6, double w,
                                               double* __restrict__ P, double* __restrict__ A) {
  double post[92];
  post_qp(k, g, H6, w, post, P);
  for (int iJ = 0; iJ < 9; iJ++) tangent_row(post, iJ, A + iJ * 9);
}

// ---------------------------------------------------------------------------
// anisotropic inputs (App. A.2.1, Eq. standard-inv-II): NSV = 1 or 2
// structural vectors A_v (reference configuration), the pairs p = (i <= j) in the order (0,0),
// (0,1), (1,1), NK = 3 + 2 NP inputs
//   K = (I1-3, I2-3, J-1, then per pair I4,ij - A_i.A_j, I5,ij - A_i.A_j),
//   I4,ij = A_i.C A_j,  I5,ij = A_i.C^2 A_j = (C A_i).(C A_j)
// (one unit vector: I4 - 1, I5 - 1).  Tangent: the F-space factors of the header extended by
// (a_v = F A_v)
//   Phi_4p = 1/2 (a_i (x) A_j + a_j (x) A_i),
//   Phi_5p = 1/2 (F C A_j (x) A_i + a_i (x) C A_j + a_j (x) C A_i + F C A_i (x) A_j)
// (dK/dF = 2 Phi), and the second-derivative term of I5,ij (I4's is d_ik (dI4/dC)_JL, inside T):
//   g5p [F_kJ (a_i,i A_j,L + a_j,i A_i,L) + F_iL (A_i,J a_j,k + A_j,J a_i,k) + b_ik (A_i,J A_j,L +
//        A_j,J A_i,L) + d_JL (a_i,i a_j,k + a_j,i a_i,k)]
// (written from d2(u.v) with u = C A_i, v = C A_j; two i = j pairs reduce to the one-vector form).
// H below is the packed upper triangle of the NK x NK Hessian.
// ---------------------------------------------------------------------------
template <int NSV>
struct Aniso {
  static constexpr int NP = NSV * (NSV + 1) / 2, NK = 3 + 2 * NP, NH = NK * (NK + 1) / 2;
  // post layout (per qp): [0..8] F, [9..17] F^-T, [18..26] w T, [27 .. 27+9NK) Phi_m,
  // [PSI .. PSI+9NK) Psi_m = 4w sum_n H'_mn Phi_n, [B] b = F F^T, [C] c2 = -2 g2 w, c3 = -g3 J w,
  // [AV] a_v = F A_v, [A0] A_v, [C5] c5_p = g5p w;  P[9] = w F S.
  static constexpr int PSI = 27 + 9 * NK, B = PSI + 9 * NK, CC = B + 9, AV = CC + 2, A0 = AV + 3 * NSV,
                       C5 = A0 + 3 * NSV, SIZE = C5 + NP;
  __host__ __device__ static constexpr int pi(int p) { return NSV == 1 ? 0 : (p < 2 ? 0 : 1); }
  __host__ __device__ static constexpr int pj(int p) { return NSV == 1 ? 0 : (p == 0 ? 0 : 1); }
};
constexpr int kPostAniso = Aniso<1>::SIZE;   // 135
constexpr int kPostAniso2 = Aniso<2>::SIZE;  // 215

__host__ __device__ constexpr int packed_index(int n, int p, int q) { return p * n - p * (p - 1) / 2 + (q - p); }

// I4,ij = A_i.C A_j and I5,ij = A_i.C^2 A_j per pair p (Eq. standard-inv-II), and A_i.A_j
template <int NSV>
__device__ __forceinline__ void aniso_invariants(const Kin& k, const double* a0, const double* a1,
                                                 double (&I4)[Aniso<NSV>::NP], double (&I5)[Aniso<NSV>::NP],
                                                 double (&aa)[Aniso<NSV>::NP]) {
  using AN = Aniso<NSV>;
  const double* Av[2] = {a0, a1};
  double CA[NSV][3];
#pragma unroll
  for (int v = 0; v < NSV; v++)
#pragma unroll
    for (int I = 0; I < 3; I++) CA[v][I] = k.C[I * 3] * Av[v][0] + k.C[I * 3 + 1] * Av[v][1] + k.C[I * 3 + 2] * Av[v][2];
#pragma unroll
  for (int p = 0; p < AN::NP; p++) {
    const int i = AN::pi(p), j = AN::pj(p);
    aa[p] = Av[i][0] * Av[j][0] + Av[i][1] * Av[j][1] + Av[i][2] * Av[j][2];
    I4[p] = Av[i][0] * CA[j][0] + Av[i][1] * CA[j][1] + Av[i][2] * CA[j][2];
    I5[p] = CA[i][0] * CA[j][0] + CA[i][1] * CA[j][1] + CA[i][2] * CA[j][2];
  }
}

// network inputs; iso: the isochoric set of App. A.2.2 (reading R29):
// (Ibar1-3, Ibar2-3, J-1, Ibar4,ij - A_i.A_j, Ibar5,ij - A_i.A_j), Ibar_m = J^(2 e_m) I_m with
// e = -1/3 for I1, I4 and -2/3 for I2, I5
template <int NSV>
__device__ __forceinline__ void anisotropic_inputs(const Kin& k, const double* a0, const double* a1, double* kk,
                                                   bool iso = false) {
  using AN = Aniso<NSV>;
  double I4[AN::NP], I5[AN::NP], aa[AN::NP];
  aniso_invariants<NSV>(k, a0, a1, I4, I5, aa);
  const double s1 = iso ? 1.0 / (cbrt(k.J) * cbrt(k.J)) : 1.0, s2 = s1 * s1;
  kk[0] = s1 * k.I1 - 3.0;
  kk[1] = s2 * k.I2 - 3.0;
  kk[2] = k.J - 1.0;
#pragma unroll
  for (int p = 0; p < AN::NP; p++) {
    kk[3 + 2 * p] = s1 * I4[p] - aa[p];
    kk[4 + 2 * p] = s2 * I5[p] - aa[p];
  }
}

// in place: g[NK], H[NK(NK+1)/2] (packed upper) from the isochoric anisotropic inputs' derivatives to
// the standard anisotropic inputs' (I1, I2, J, I4,ij, I5,ij), by the chain rule through
// Ibar_m = J^(q_m) I_m (q = -2/3 for m = 1, 4; -4/3 for m = 2, 5):
//   g_m = a_m gb_m, g_J = gb_J + sum_m c_m gb_m, c_m = q_m Ibar_m / J, a_m = J^(q_m);
//   H_mn = a_m a_n Hb_mn, H_mJ = a_m t_m + q_m a_m gb_m / J, t_m = Hb_mJ + sum_n Hb_mn c_n;
//   H_JJ = t_J + sum_m c_m t_m + sum_m q_m (q_m - 1) Ibar_m gb_m / J^2
// (the three-input case is isochoric_to_standard below, term for term)
template <int NSV>
__device__ __forceinline__ void isochoric_aniso_to_standard(const Kin& k, const double* a0, const double* a1,
                                                            double* __restrict__ g, double* __restrict__ H) {
  using AN = Aniso<NSV>;
  constexpr int NK = AN::NK;
  double I4[AN::NP], I5[AN::NP], aa[AN::NP];
  aniso_invariants<NSV>(k, a0, a1, I4, I5, aa);
  const double s1 = 1.0 / (cbrt(k.J) * cbrt(k.J)), s2 = s1 * s1, iJ = 1.0 / k.J;
  double al[NK], qm[NK], c[NK];
#pragma unroll
  for (int m = 0; m < NK; m++) {
    const bool two = m == 1 || (m >= 3 && ((m - 3) & 1));  // I2, I5,ij: exponent -4/3
    const double Im = m == 0 ? k.I1 : m == 1 ? k.I2 : m == 2 ? 0.0 : ((m - 3) & 1) ? I5[(m - 3) >> 1] : I4[(m - 3) >> 1];
    al[m] = m == 2 ? 1.0 : (two ? s2 : s1);
    qm[m] = m == 2 ? 0.0 : (two ? -4.0 / 3.0 : -2.0 / 3.0);
    c[m] = m == 2 ? 1.0 : qm[m] * al[m] * Im * iJ;  // c_J = 1 folds Hb_mJ into t_m
  }
  double t[NK];
#pragma unroll
  for (int m = 0; m < NK; m++) {
    double s = 0.0;
#pragma unroll
    for (int n = 0; n < NK; n++) s += H[packed_index(NK, m < n ? m : n, m < n ? n : m)] * c[n];
    t[m] = s;
  }
  double hjj = t[2], gj = g[2];
#pragma unroll
  for (int m = 0; m < NK; m++) {
    if (m == 2) continue;
    hjj += c[m] * t[m] + qm[m] * (qm[m] - 1.0) * (c[m] / qm[m]) * iJ * g[m];  // c_m / q_m = Ibar_m / J
    gj += c[m] * g[m];
  }
#pragma unroll
  for (int m = 0; m < NK; m++)
#pragma unroll
    for (int n = m; n < NK; n++) {
      double& h = H[packed_index(NK, m, n)];
      if (m == 2 && n == 2)
        h = hjj;
      else if (n == 2)
        h = al[m] * t[m] + qm[m] * al[m] * iJ * g[m];
      else if (m == 2)
        h = al[n] * t[n] + qm[n] * al[n] * iJ * g[n];
      else
        h *= al[m] * al[n];
    }
#pragma unroll
  for (int m = 0; m < NK; m++)
    if (m != 2) g[m] *= al[m];
  g[2] = gj;
}


template <int NSV>
__device__ __forceinline__ void post_qp_aniso(const Kin& k, const double* a0, const double* a1,
                                              const double* __restrict__ g, const double* __restrict__ Hpk, double w,
                                              double* __restrict__ post, double* __restrict__ P) {
  using AN = Aniso<NSV>;
  constexpr int NK = AN::NK;
  const double* F = k.F;
  const double hJ = 0.5 * k.J;
  const double* Av[2] = {a0, a1};
  double CA[NSV][3], a[NSV][3], FCA[NSV][3];
#pragma unroll
  for (int v = 0; v < NSV; v++) {
#pragma unroll
    for (int I = 0; I < 3; I++) CA[v][I] = k.C[I * 3] * Av[v][0] + k.C[I * 3 + 1] * Av[v][1] + k.C[I * 3 + 2] * Av[v][2];
#pragma unroll
    for (int i = 0; i < 3; i++) {
      a[v][i] = F[i * 3] * Av[v][0] + F[i * 3 + 1] * Av[v][1] + F[i * 3 + 2] * Av[v][2];
      FCA[v][i] = F[i * 3] * CA[v][0] + F[i * 3 + 1] * CA[v][1] + F[i * 3 + 2] * CA[v][2];
    }
  }
  double S[9];
#pragma unroll
  for (int I = 0; I < 3; I++)
#pragma unroll
    for (int J = 0; J < 3; J++) {
      const double d = (I == J) ? 1.0 : 0.0;
      double s = 2.0 * (g[0] * d + g[1] * (k.I1 * d - k.C[I * 3 + J]) + g[2] * hJ * k.Ci[I * 3 + J]);
#pragma unroll
      for (int p = 0; p < AN::NP; p++) {
        const int vi = AN::pi(p), vj = AN::pj(p);
        s += g[3 + 2 * p] * (Av[vi][I] * Av[vj][J] + Av[vj][I] * Av[vi][J]) +
             g[4 + 2 * p] * (Av[vi][I] * CA[vj][J] + CA[vj][I] * Av[vi][J] + CA[vi][I] * Av[vj][J] + Av[vj][I] * CA[vi][J]);
      }
      S[I * 3 + J] = s;
      post[18 + I * 3 + J] = w * (s - g[2] * k.J * k.Ci[I * 3 + J]);
    }
  double Phi[NK][9];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int J = 0; J < 3; J++) {
      const double FC = F[i * 3 + 0] * k.C[0 * 3 + J] + F[i * 3 + 1] * k.C[1 * 3 + J] + F[i * 3 + 2] * k.C[2 * 3 + J];
      Phi[0][i * 3 + J] = F[i * 3 + J];
      Phi[1][i * 3 + J] = k.I1 * F[i * 3 + J] - FC;
      Phi[2][i * 3 + J] = hJ * k.FiT[i * 3 + J];
#pragma unroll
      for (int p = 0; p < AN::NP; p++) {
        const int vi = AN::pi(p), vj = AN::pj(p);
        Phi[3 + 2 * p][i * 3 + J] = 0.5 * (a[vi][i] * Av[vj][J] + a[vj][i] * Av[vi][J]);
        Phi[4 + 2 * p][i * 3 + J] = 0.5 * (FCA[vj][i] * Av[vi][J] + a[vi][i] * CA[vj][J] + a[vj][i] * CA[vi][J] +
                                           FCA[vi][i] * Av[vj][J]);
      }
    }
  const double w4 = 4.0 * w;
#pragma unroll
  for (int x = 0; x < 9; x++) {
    post[x] = F[x];
    post[9 + x] = k.FiT[x];
  }
#pragma unroll
  for (int m = 0; m < NK; m++) {
    double hr[NK];  // row m of H' = H + diag(g2, 0, g3/J, 0, ...)
#pragma unroll
    for (int n = 0; n < NK; n++) hr[n] = Hpk[m <= n ? packed_index(NK, m, n) : packed_index(NK, n, m)];
    if (m == 0) hr[0] += g[1];
    if (m == 2) hr[2] += g[2] / k.J;
#pragma unroll
    for (int x = 0; x < 9; x++) {
      post[27 + m * 9 + x] = Phi[m][x];
      double t = 0.0;
#pragma unroll
      for (int n = 0; n < NK; n++) t += hr[n] * Phi[n][x];
      post[AN::PSI + m * 9 + x] = w4 * t;
    }
  }
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int kk = 0; kk < 3; kk++)
      post[AN::B + i * 3 + kk] = F[i * 3 + 0] * F[kk * 3 + 0] + F[i * 3 + 1] * F[kk * 3 + 1] + F[i * 3 + 2] * F[kk * 3 + 2];
  post[AN::CC] = -2.0 * g[1] * w;
  post[AN::CC + 1] = -g[2] * k.J * w;
#pragma unroll
  for (int v = 0; v < NSV; v++)
#pragma unroll
    for (int i = 0; i < 3; i++) {
      post[AN::AV + 3 * v + i] = a[v][i];
      post[AN::A0 + 3 * v + i] = Av[v][i];
    }
#pragma unroll
  for (int p = 0; p < AN::NP; p++) post[AN::C5 + p] = g[4 + 2 * p] * w;
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int J = 0; J < 3; J++)
      P[i * 3 + J] = w * (F[i * 3 + 0] * S[0 * 3 + J] + F[i * 3 + 1] * S[1 * 3 + J] + F[i * 3 + 2] * S[2 * 3 + J]);
}

template <int NSV>
__device__ __forceinline__ void tangent_row_aniso(const double* __restrict__ post, int iJ, double* __restrict__ out) {
  using AN = Aniso<NSV>;
  constexpr int NK = AN::NK;
  const int i = iJ / 3, J = iJ % 3;
  double p[NK];
#pragma unroll
  for (int m = 0; m < NK; m++) p[m] = post[27 + m * 9 + iJ];
  const double c2 = post[AN::CC], c3 = post[AN::CC + 1];
#pragma unroll
  for (int kk = 0; kk < 3; kk++) {
    const double FkJ = post[kk * 3 + J], GkJ = post[9 + kk * 3 + J], bik = post[AN::B + i * 3 + kk];
#pragma unroll
    for (int L = 0; L < 3; L++) {
      const int kL = kk * 3 + L;
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < NK; m++) v += p[m] * post[AN::PSI + m * 9 + kL];
      v += c2 * post[i * 3 + L] * FkJ + c3 * post[9 + i * 3 + L] * GkJ;
      if (J == L) v += c2 * bik;
#pragma unroll
      for (int q = 0; q < AN::NP; q++) {
        const int vi = AN::pi(q), vj = AN::pj(q);
        const double* ai = post + AN::AV + 3 * vi;
        const double* aj = post + AN::AV + 3 * vj;
        const double* Ai = post + AN::A0 + 3 * vi;
        const double* Aj = post + AN::A0 + 3 * vj;
        double t = FkJ * (ai[i] * Aj[L] + aj[i] * Ai[L]) + post[i * 3 + L] * (Ai[J] * aj[kk] + Aj[J] * ai[kk]) +
                   bik * (Ai[J] * Aj[L] + Aj[J] * Ai[L]);
        if (J == L) t += ai[i] * aj[kk] + aj[i] * ai[kk];
        v += post[AN::C5 + q] * t;
      }
      if (i == kk) v += post[18 + J * 3 + L];
      out[kL] = v;
    }
  }
}

template <int NSV>
__device__ __forceinline__ void stress_tangent_aniso(const Kin& k, const double* a0, const double* a1,
                                                     const double* g, const double* H, double w, double* P, double* A) {
  double post[Aniso<NSV>::SIZE];
  post_qp_aniso<NSV>(k, a0, a1, g, H, w, post, P);
  for (int iJ = 0; iJ < 9; iJ++) tangent_row_aniso<NSV>(post, iJ, A + iJ * 9);
}

// ---------------------------------------------------------------------------
// kinematic variant: isochoric inputs (App. A.2.2)
//   kbar = (Ibar1 - 3, Ibar2 - 3, J - 1),  Ibar1 = J^-2/3 I1,  Ibar2 = J^-4/3 I2.
// The network's (gbar, Hbar) w.r.t. kbar are carried to (g, H) w.r.t. the standard
// k = (I1 - 3, I2 - 3, J - 1) by the chain rule, so S and the F-space tangent above
// apply unchanged (the oracle instead follows the paper's spatial G-tensor table):
//   g = D^T gbar,  H = D^T Hbar D + sum_m gbar_m d2y_m,  D = d(Ibar1, Ibar2, J)/d(I1, I2, J)
//   D = [[a, 0, c1], [0, b, c2], [0, 0, 1]],  a = J^-2/3, b = J^-4/3, c1 = -2/3 Ibar1/J, c2 = -4/3 Ibar2/J
//   d2Ibar1: (I1,J) = -2/3 a/J, (J,J) = 10/9 Ibar1/J^2;  d2Ibar2: (I2,J) = -4/3 b/J, (J,J) = 28/9 Ibar2/J^2
// ---------------------------------------------------------------------------
__device__ __forceinline__ void isochoric_inputs(const Kin& k, double kb[3]) {
  const double a = 1.0 / (cbrt(k.J) * cbrt(k.J));
  kb[0] = a * k.I1 - 3.0;
  kb[1] = a * a * k.I2 - 3.0;
  kb[2] = k.J - 1.0;
}

// in place: g[3], H6[6] (upper 00,01,02,11,12,22) from kbar- to k-derivatives
__device__ __forceinline__ void isochoric_to_standard(const Kin& k, double* __restrict__ g, double* __restrict__ H6) {
  const double a = 1.0 / (cbrt(k.J) * cbrt(k.J)), b = a * a, iJ = 1.0 / k.J;
  const double Ib1 = a * k.I1, Ib2 = b * k.I2;
  const double c1 = -2.0 / 3.0 * Ib1 * iJ, c2 = -4.0 / 3.0 * Ib2 * iJ;
  const double g0 = g[0], g1 = g[1], g2 = g[2];
  const double h00 = H6[0], h01 = H6[1], h02 = H6[2], h11 = H6[3], h12 = H6[4], h22 = H6[5];
  g[0] = a * g0;
  g[1] = b * g1;
  g[2] = c1 * g0 + c2 * g1 + g2;
  const double t0 = h00 * c1 + h01 * c2 + h02;  // (Hbar col3)_0
  const double t1 = h01 * c1 + h11 * c2 + h12;  // (Hbar col3)_1
  const double t2 = h02 * c1 + h12 * c2 + h22;  // (Hbar col3)_2
  H6[0] = a * a * h00;
  H6[1] = a * b * h01;
  H6[2] = a * t0 - 2.0 / 3.0 * a * iJ * g0;
  H6[3] = b * b * h11;
  H6[4] = b * t1 - 4.0 / 3.0 * b * iJ * g1;
  H6[5] = c1 * t0 + c2 * t1 + t2 + (10.0 / 9.0 * Ib1 * g0 + 28.0 / 9.0 * Ib2 * g1) * iJ * iJ;
}

// analytic inner networks: gradient and Hessian w.r.t. the inputs
//  CANN (Eq. cann-def / cann-chain-rule): diagonal Hessian
//  Gent-Thomas (App. C): N = gt0 k1 + gt1 ln(1 + k2/3) + gt2 k3^2
// nk network inputs (3, or 5 for anisotropic kinematics; Gent-Thomas: 3); H6 packed upper
// triangle of the nk x nk Hessian
__device__ __forceinline__ void analytic_net(int net, int n, const int32_t* __restrict__ f,
                                             const double* __restrict__ w1, const double* __restrict__ w2,
                                             const double* __restrict__ gt, const double* __restrict__ skip,
                                             const double* kin, double* __restrict__ g, double* __restrict__ H6,
                                             int nk = 3) {
  if (net == 2) {
    const double u = 1.0 / (kin[1] + 3.0);
    g[0] = gt[0];
    g[1] = gt[1] * u;
    g[2] = 2.0 * gt[2] * kin[2];
    H6[0] = H6[1] = H6[2] = H6[4] = 0.0;
    H6[3] = -gt[1] * u * u;
    H6[5] = 2.0 * gt[2];
    return;
  }
  for (int x = 0; x < nk * (nk + 1) / 2; x++) H6[x] = 0.0;
  for (int m = 0; m < nk; m++) {
    const double x = kin[m];
    double gm = m < 3 ? skip[m] : 0.0, hm = 0.0;
    for (int bb = 0; bb < n; bb++) {
      const int32_t* fb = f + (m * n + bb) * 3;
      const int t0 = __ldg(fb), p = __ldg(fb + 1), t2 = __ldg(fb + 2);
      const double a1 = __ldg(w1 + m * n + bb), a2 = __ldg(w2 + m * n + bb);
      // f0 and its slope (f0'' = 0)
      const double v0 = t0 == 0 ? x : (t0 == 1 ? fmax(x, 0.0) : fabs(x));
      const double d0 = t0 == 0 ? 1.0 : (t0 == 1 ? (x > 0.0 ? 1.0 : (x < 0.0 ? 0.0 : 0.5))
                                                  : (x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0)));
      // f1 = v0^p
      const double v1 = p == 1 ? v0 : (p == 2 ? v0 * v0 : v0 * v0 * v0);
      const double d1 = p == 1 ? 1.0 : (p == 2 ? 2.0 * v0 : 3.0 * v0 * v0);
      const double dd1 = p == 1 ? 0.0 : (p == 2 ? 2.0 : 6.0 * v0);
      // f2 (weight w1 inside)
      double d2, dd2;
      if (t2 == 0) {
        d2 = a1;
        dd2 = 0.0;
      } else if (t2 == 1) {
        const double e = exp(a1 * v1);
        d2 = a1 * e;
        dd2 = a1 * a1 * e;
      } else {
        const double r = 1.0 / (1.0 - a1 * v1);
        d2 = a1 * r;
        dd2 = a1 * a1 * r * r;
      }
      gm += a2 * d2 * d1 * d0;
      hm += a2 * (dd2 * d1 * d1 + d2 * dd1) * d0 * d0;
    }
    g[m] = gm;
    H6[m * nk - m * (m - 1) / 2] = hm;  // diagonal (m, m) of the packed triangle
  }
}

// value of the analytic networks (material-point outputs): same closed forms as above
__device__ __forceinline__ double analytic_value(int net, int n, const int32_t* __restrict__ f,
                                                 const double* __restrict__ w1, const double* __restrict__ w2,
                                                 const double* __restrict__ gt, const double* __restrict__ skip,
                                                 const double* kin, int nk = 3) {
  if (net == 2) return gt[0] * kin[0] + gt[1] * log1p(kin[1] / 3.0) + gt[2] * kin[2] * kin[2];
  double N = skip[0] * kin[0] + skip[1] * kin[1] + skip[2] * kin[2];
  for (int m = 0; m < nk; m++) {
    const double x = kin[m];
    for (int bb = 0; bb < n; bb++) {
      const int32_t* fb = f + (m * n + bb) * 3;
      const int t0 = __ldg(fb), p = __ldg(fb + 1), t2 = __ldg(fb + 2);
      const double a1 = __ldg(w1 + m * n + bb), a2 = __ldg(w2 + m * n + bb);
      const double v0 = t0 == 0 ? x : (t0 == 1 ? fmax(x, 0.0) : fabs(x));
      const double v1 = p == 1 ? v0 : (p == 2 ? v0 * v0 : v0 * v0 * v0);
      N += a2 * (t2 == 0 ? a1 * v1 : (t2 == 1 ? expm1(a1 * v1) : -log1p(-a1 * v1)));
    }
  }
  return N;
}

// ---------------------------------------------------------------------------
// softplus z = log(1 + e^y) and sigmoid s = softplus' (SURVEY s7 hard part 3),
// branch-free, fp64 FMA + integer ops only (no MUFU, no F2I, no libdevice slow
// paths), on tables of N = 2^TB entries:
//   e = exp(-|y|) = 2^(k/N) * p(r), r = -|y| - k ln2/N, |r| <= ln2/(2N), p the Taylor
//       polynomial of degree 5 (N = 64) / 4 (N = 256);
//   log1p(e) = log c_j + log1p(r2), c_j = 1 + j/N nearest to u = 1 + e, r2 = u/c_j - 1,
//       |r2| <= 1/(2N), log1p by its series to degree 7 / 6, the rounding of u corrected;
//   1/u = (1/c_j) / (1 + r2) by the series 1 - r2 + ... - r2^7 / - r2^5 (COMMET_SIG_RCP = 0), or
//       by rcp.approx + two Newton steps (COMMET_SIG_RCP = 1, the default: off the table, 4 fp64 ops).
// Truncation errors, relative: 6e-18 / 3.7e-17 (exp), 2.2e-16 / 1.2e-17 (log1p: r2^(d+1)/(d+1)
// relative to log1p(r2) ~ r2 when j = 0), 2e-17 / 5.7e-17 (1/u).  The fused kernels whose shared memory allows it use N = 256
// (4 fp64 ops per neuron fewer, measured on the round-2 A/B); the rest N = 64.
// tab layout: [0, N) 2^(j/N); [N, 2N+1) 1/c_j; [2N+1, 3N+2) log c_j.  Both tables sit back to
// back in one device array: N = 64 at offset 0, N = 256 at kActTab6 (kActTabSize doubles).
template <int TB>
struct ActTab {
  static constexpr int N = 1 << TB, SIZE = 3 * N + 2;
};
constexpr int kActTab6 = ActTab<6>::SIZE;                   // 194
constexpr int kActTabSize = ActTab<6>::SIZE + ActTab<8>::SIZE;  // both tables
template <int TB>
__host__ __device__ constexpr int act_tab_offset() { return TB == 6 ? 0 : kActTab6; }

template <int TB>
__device__ __forceinline__ double exp_neg_abs(double y, const double* __restrict__ tab, int& k_out) {
  constexpr int N = ActTab<TB>::N;
  const double MAGIC = 6755399441055744.0;  // 1.5 * 2^52: round-to-integer by addition
  const double x = fmax(-fabs(y), -708.0);
  double kd = fma(x, (double)N / 0.6931471805599453, MAGIC);
  const int k = __double2loint(kd);
  kd -= MAGIC;
  double r, p;
  if constexpr (TB == 6) {
    r = fma(kd, -0.010830424696249145, x);  // ln2/64 hi
    r = fma(kd, -3.623510646634843e-19, r); // ln2/64 lo
    p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
  } else {
    r = fma(kd, -0.0027076061740622863, x);  // ln2/256 hi
    r = fma(kd, -9.058776616587108e-20, r);  // ln2/256 lo
    p = fma(r, 1.0 / 24.0, 1.0 / 6.0);
  }
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double e = tab[k & (N - 1)] * p;
  k_out = k;
  return __hiloint2double(__double2hiint(e) + (k >> TB) * 1048576, __double2loint(e));  // * 2^(k >> TB)
}

#ifndef COMMET_SIG_RCP
#define COMMET_SIG_RCP 1  // sigmoid 1/(1 + e) by the MUFU reciprocal + two Newton steps instead of the table series (measured c3 -0.5 %, c4 -0.3 %, c5 -0.6 %; r02_ab_sig_rcp.txt)
#endif
// 1/u for u in [1, 2]: rcp.approx (MUFU, off the fp64 datapath) and two Newton steps (relative
// error eps0^4 + rounding: ~2 ulp), 4 fp64 ops instead of the 1/c_j table series (7-9)
__device__ __forceinline__ double rcp_u12(double u) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(u));
  r = fma(r, fma(-u, r, 1.0), r);
  return fma(r, fma(-u, r, 1.0), r);
}

template <int TB>
__device__ __forceinline__ void softplus_sig_t(double y, const double* __restrict__ tab, double& z, double& s) {
  constexpr int N = ActTab<TB>::N;
  const double MAGIC = 6755399441055744.0;
  int k;
  const double e = exp_neg_abs<TB>(y, tab, k);
  const double u = 1.0 + e;
  const int j = __double2loint(fma(e, (double)N, MAGIC));  // round(N e) in [0, N]
  const double invc = tab[N + j], logc = tab[2 * N + 1 + j];
  const double r2 = fma(u, invc, -1.0);
  const double r2s = r2 * r2;
  double q, v = 0.0;
  if constexpr (TB == 6) {
    q = fma(r2, 1.0 / 7.0, -1.0 / 6.0);
    q = fma(q, r2, 0.2);
    q = fma(q, r2, -0.25);
    q = fma(q, r2, 1.0 / 3.0);
    q = fma(q, r2, -0.5);
    if constexpr (!COMMET_SIG_RCP) {
      const double r4 = r2s * r2s;
      v = (1.0 - r2) * (1.0 + r2s) * (1.0 + r4);  // 1/(1 + r2), error r2^8
    }
  } else {  // degree 6: at j = 0 (e < 1/512) z = log1p(r2) ~ r2, so the RELATIVE error is r2^6/7
    q = fma(r2, -1.0 / 6.0, 0.2);
    q = fma(q, r2, -0.25);
    q = fma(q, r2, 1.0 / 3.0);
    q = fma(q, r2, -0.5);
    if constexpr (!COMMET_SIG_RCP) v = (1.0 - r2) * (fma(r2s, r2s, r2s) + 1.0);  // 1/(1 + r2), error r2^6
  }
  const double lp = fma(q, r2s, r2);                 // log1p(r2)
  const double d = e - (u - 1.0);                    // rounding error of u (exact)
  z = fmax(y, 0.0) + (logc + fma(d, invc, lp));      // max(y,0) + log1p(e)
  if constexpr (COMMET_SIG_RCP)
    s = (y >= 0.0 ? 1.0 : e) * rcp_u12(u);
  else
    s = (y >= 0.0 ? 1.0 : e) * (invc * v);
}

// sigmoid only (the last hidden layer needs s, not z): e = exp(-|y|) and 1/(1+e) as above
template <int TB>
__device__ __forceinline__ double sigmoid_t(double y, const double* __restrict__ tab) {
  constexpr int N = ActTab<TB>::N;
  const double MAGIC = 6755399441055744.0;
  int k;
  const double e = exp_neg_abs<TB>(y, tab, k);
  const double u = 1.0 + e;
  if constexpr (COMMET_SIG_RCP) return (y >= 0.0 ? 1.0 : e) * rcp_u12(u);  // as in softplus_sig_t
  const int j = __double2loint(fma(e, (double)N, MAGIC));
  const double invc = tab[N + j];
  const double r2 = fma(u, invc, -1.0);
  const double r2s = r2 * r2;
  double v;
  if constexpr (TB == 6)
    v = (1.0 - r2) * (1.0 + r2s) * (1.0 + r2s * r2s);
  else
    v = (1.0 - r2) * (fma(r2s, r2s, r2s) + 1.0);
  return (y >= 0.0 ? 1.0 : e) * (invc * v);
}

// the N = 64 forms (kernels that keep the small table: simple kernel, Alg. 4 helper, 3-pass)
__device__ __forceinline__ void softplus_sig(double y, const double* __restrict__ tab, double& z, double& s) {
  softplus_sig_t<6>(y, tab, z, s);
}
__device__ __forceinline__ double sigmoid_tab(double y, const double* __restrict__ tab) { return sigmoid_t<6>(y, tab); }

// host: fill both tables (long double for the reference values)
template <int TB>
inline void fill_act_table_t(double* tab) {
  constexpr int N = ActTab<TB>::N;
  for (int j = 0; j < N; j++) tab[j] = (double)exp2l((long double)j / N);
  for (int j = 0; j <= N; j++) {
    const double invc = (double)(1.0L / (1.0L + (long double)j / N));
    tab[N + j] = invc;
    tab[2 * N + 1 + j] = (double)(-logl((long double)invc));
  }
}
inline void fill_act_table(double* tab) {
  fill_act_table_t<6>(tab);
  fill_act_table_t<8>(tab + kActTab6);
}

}  // namespace commet
