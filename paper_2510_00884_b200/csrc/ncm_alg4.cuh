// ncm_alg4.cuh -- Alg. 4 of PAPER.md:987-1007 for one point: the inner network's
// gradient g = dN/dk and Hessian H (packed upper triangle) in one forward
// pass of 1 + NK + NH channels per neuron, in local memory.  Used by the one-thread-per-
// element cross-check kernel (kernel_simple.cu) and the material-point calls
// (material.cu); the fused kernel evaluates the same Hessian with DMMA passes.
#pragma once
#include "commet_internal.h"
#include "qp_math.cuh"
#include "ickan.cuh"

namespace commet {

// Alg. 4 with 1 + NK + NH channels per neuron (value, gradient, packed Hessian) in place;
// NK = 3 inputs, or 5 for anisotropic kinematics (W1 is [w][NK]; hidden skips act on the
// first three inputs).  Not inlined: the two instantiations keep separate local frames.
template <int NK>
__device__ __noinline__ void ncm_alg4(const NcmDev& m, const double* kin, double* g, double* H6) {
  constexpr int NH = NK * (NK + 1) / 2;
  double z[kMaxWidth], dz[kMaxWidth][NK], d2z[kMaxWidth][NH];
  double zn[kMaxWidth], dzn[kMaxWidth][NK], d2zn[kMaxWidth][NH];
  const int w = m.w;
  // layer 1: y = W1 k + b1, dy = W1, d2y = 0
  for (int j = 0; j < w; j++) {
    double y = m.b[j], dy[NK];
    for (int i = 0; i < NK; i++) {
      dy[i] = m.W1[j * NK + i];
      y += dy[i] * kin[i];
    }
    double zz, s;
    softplus_sig(y, m.act_tab, zz, s);
    const double s2 = s * (1.0 - s);
    z[j] = zz;
    for (int p = 0; p < NK; p++) dz[j][p] = s * dy[p];
    int c = 0;
    for (int p = 0; p < NK; p++)
      for (int q = p; q < NK; q++) d2z[j][c++] = s2 * dy[p] * dy[q];
  }
  for (int l = 1; l < m.L; l++) {
    const double* Wl = m.Wrow + (size_t)(l - 1) * w * w;
    const double* Bl = m.skip_h ? m.skip_h + (size_t)(l - 1) * w * 3 : nullptr;
    for (int j = 0; j < w; j++) {
      double y = m.b[l * w + j], dy[NK], d2y[NH];
      for (int p = 0; p < NK; p++) dy[p] = 0.0;
      for (int p = 0; p < NH; p++) d2y[p] = 0.0;
      for (int i = 0; i < w; i++) {
        const double a = Wl[j * w + i];
        y += a * z[i];
        for (int p = 0; p < NK; p++) dy[p] += a * dz[i][p];
        for (int p = 0; p < NH; p++) d2y[p] += a * d2z[i][p];
      }
      if (Bl)
        for (int p = 0; p < 3; p++) {
          y += Bl[j * 3 + p] * kin[p];
          dy[p] += Bl[j * 3 + p];
        }
      double zz, s;
      softplus_sig(y, m.act_tab, zz, s);
      const double s2 = s * (1.0 - s);
      zn[j] = zz;
      for (int p = 0; p < NK; p++) dzn[j][p] = s * dy[p];
      int c = 0;
      for (int p = 0; p < NK; p++)
        for (int q = p; q < NK; q++, c++) d2zn[j][c] = s * d2y[c] + s2 * dy[p] * dy[q];
    }
    for (int j = 0; j < w; j++) {
      z[j] = zn[j];
      for (int p = 0; p < NK; p++) dz[j][p] = dzn[j][p];
      for (int p = 0; p < NH; p++) d2z[j][p] = d2zn[j][p];
    }
  }
  for (int p = 0; p < NK; p++) g[p] = p < 3 ? m.skip_out[p] : 0.0;
  for (int p = 0; p < NH; p++) H6[p] = 0.0;
  for (int j = 0; j < w; j++) {
    for (int p = 0; p < NK; p++) g[p] += m.a[j] * dz[j][p];
    for (int p = 0; p < NH; p++) H6[p] += m.a[j] * d2z[j][p];
  }
}

// the ctx's inner network at its inputs k (3, or 5 for anisotropic kinematics): Alg. 4 for the
// ICNN, closed forms for CANN / Gent-Thomas / ICKAN; H6 = packed upper triangle of the Hessian
__device__ __forceinline__ void ncm_point(const NcmDev& m, const double* kin, double* g, double* H6) {
  if (m.net == 0 && m.kin == 2)
    ncm_alg4<5>(m, kin, g, H6);
  else if (m.net == 0)
    ncm_alg4<3>(m, kin, g, H6);
  else if (m.kin == 3)
    analytic_point<9>(m, kin, g, H6, nullptr);
  else if (m.kin == 2)
    analytic_point<5>(m, kin, g, H6, nullptr);
  else
    analytic_point<3>(m, kin, g, H6, nullptr);
}

}  // namespace commet
