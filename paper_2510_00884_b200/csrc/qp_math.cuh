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

// g[3] = dW/dk, H[6] = d2W/dk2 (upper: 00,01,02,11,12,22), penalty included.
// Outputs P[9] = F S and A[81] (A[(i*3+J)*9 + k*3+L]), both scaled by w.
__device__ __forceinline__ void stress_tangent(const Kin& k, const double* __restrict__ g,
                                               const double* __restrict__ H6, double w,
                                               double* __restrict__ P, double* __restrict__ A) {
  const double* F = k.F;
  double S[9], T[9], Phi[3][9], Psi[3][9];
  const double hJ = 0.5 * k.J;
#pragma unroll
  for (int I = 0; I < 3; I++)
#pragma unroll
    for (int J = 0; J < 3; J++) {
      const double d = (I == J) ? 1.0 : 0.0;
      S[I * 3 + J] = 2.0 * (g[0] * d + g[1] * (k.I1 * d - k.C[I * 3 + J]) + g[2] * hJ * k.Ci[I * 3 + J]);
      T[I * 3 + J] = S[I * 3 + J] - g[2] * k.J * k.Ci[I * 3 + J];
    }
  // Phi_1 = F, Phi_2 = I1 F - F C, Phi_3 = J/2 F^-T
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int J = 0; J < 3; J++) {
      double FC = F[i * 3 + 0] * k.C[0 * 3 + J] + F[i * 3 + 1] * k.C[1 * 3 + J] + F[i * 3 + 2] * k.C[2 * 3 + J];
      Phi[0][i * 3 + J] = F[i * 3 + J];
      Phi[1][i * 3 + J] = k.I1 * F[i * 3 + J] - FC;
      Phi[2][i * 3 + J] = hJ * k.FiT[i * 3 + J];
    }
  // H' (symmetric) with the folded g2 and g3/J terms; Psi_m = 4 w sum_n H'_mn Phi_n
  double Hp[9];
  Hp[0] = H6[0] + g[1]; Hp[1] = H6[1]; Hp[2] = H6[2];
  Hp[3] = H6[1]; Hp[4] = H6[3]; Hp[5] = H6[4];
  Hp[6] = H6[2]; Hp[7] = H6[4]; Hp[8] = H6[5] + g[2] / k.J;
  const double w4 = 4.0 * w;
#pragma unroll
  for (int m = 0; m < 3; m++)
#pragma unroll
    for (int x = 0; x < 9; x++)
      Psi[m][x] = w4 * (Hp[m * 3 + 0] * Phi[0][x] + Hp[m * 3 + 1] * Phi[1][x] + Hp[m * 3 + 2] * Phi[2][x]);
  double b[9];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int kk = 0; kk < 3; kk++)
      b[i * 3 + kk] = F[i * 3 + 0] * F[kk * 3 + 0] + F[i * 3 + 1] * F[kk * 3 + 1] + F[i * 3 + 2] * F[kk * 3 + 2];
  const double c2 = -2.0 * g[1] * w, c3 = -g[2] * k.J * w;
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int J = 0; J < 3; J++)
#pragma unroll
      for (int kk = 0; kk < 3; kk++)
#pragma unroll
        for (int L = 0; L < 3; L++) {
          double v = Phi[0][i * 3 + J] * Psi[0][kk * 3 + L] + Phi[1][i * 3 + J] * Psi[1][kk * 3 + L] +
                     Phi[2][i * 3 + J] * Psi[2][kk * 3 + L];
          v += c2 * F[i * 3 + L] * F[kk * 3 + J] + c3 * k.FiT[i * 3 + L] * k.FiT[kk * 3 + J];
          if (J == L) v += c2 * b[i * 3 + kk];
          if (i == kk) v += w * T[J * 3 + L];
          A[(i * 3 + J) * 9 + kk * 3 + L] = v;
        }
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int J = 0; J < 3; J++)
      P[i * 3 + J] = w * (F[i * 3 + 0] * S[0 * 3 + J] + F[i * 3 + 1] * S[1 * 3 + J] + F[i * 3 + 2] * S[2 * 3 + J]);
}

// softplus and its first two derivatives (stable forms, SURVEY s7 hard part 3)
__device__ __forceinline__ void softplus3(double y, double& z, double& s) {
  const double e = exp(-fabs(y));
  const double inv = 1.0 / (1.0 + e);
  z = fmax(y, 0.0) + log1p(e);
  s = (y >= 0.0) ? inv : e * inv;
}

}  // namespace commet
