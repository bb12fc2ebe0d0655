// ncm_alg4.cuh -- Alg. 4 of PAPER.md:987-1007 for one point: the inner network's
// gradient g = dN/dk and Hessian H (upper 00,01,02,11,12,22) in one forward
// pass of 10 channels per neuron, in local memory.  Used by the one-thread-per-
// element cross-check kernel (kernel_simple.cu) and the material-point calls
// (material.cu); the fused kernel evaluates the same Hessian with DMMA passes.
#pragma once
#include "commet_internal.h"
#include "qp_math.cuh"
#include "ickan.cuh"

namespace commet {

// Alg. 4 with 10 channels per neuron (value, 3 gradient, 6 Hessian) in place.
__device__ __forceinline__ void ncm_alg4(const NcmDev& m, const double* kin, double* g, double* H6) {
  double z[kMaxWidth], dz[kMaxWidth][3], d2z[kMaxWidth][6];
  double zn[kMaxWidth], dzn[kMaxWidth][3], d2zn[kMaxWidth][6];
  const int w = m.w;
  // layer 1: y = W1 k + b1, dy = W1, d2y = 0
  for (int j = 0; j < w; j++) {
    double y = m.b[j];
    for (int i = 0; i < 3; i++) y += m.W1[j * 3 + i] * kin[i];
    double zz, s;
    softplus_sig(y, m.act_tab, zz, s);
    const double s2 = s * (1.0 - s);
    z[j] = zz;
    double dy[3] = {m.W1[j * 3 + 0], m.W1[j * 3 + 1], m.W1[j * 3 + 2]};
    for (int p = 0; p < 3; p++) dz[j][p] = s * dy[p];
    int c = 0;
    for (int p = 0; p < 3; p++)
      for (int q = p; q < 3; q++) d2z[j][c++] = s2 * dy[p] * dy[q];
  }
  for (int l = 1; l < m.L; l++) {
    const double* Wl = m.Wrow + (size_t)(l - 1) * w * w;
    const double* Bl = m.skip_h ? m.skip_h + (size_t)(l - 1) * w * 3 : nullptr;
    for (int j = 0; j < w; j++) {
      double y = m.b[l * w + j], dy[3] = {0, 0, 0}, d2y[6] = {0, 0, 0, 0, 0, 0};
      for (int i = 0; i < w; i++) {
        const double a = Wl[j * w + i];
        y += a * z[i];
        for (int p = 0; p < 3; p++) dy[p] += a * dz[i][p];
        for (int p = 0; p < 6; p++) d2y[p] += a * d2z[i][p];
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
      for (int p = 0; p < 3; p++) dzn[j][p] = s * dy[p];
      int c = 0;
      for (int p = 0; p < 3; p++)
        for (int q = p; q < 3; q++, c++) d2zn[j][c] = s * d2y[c] + s2 * dy[p] * dy[q];
    }
    for (int j = 0; j < w; j++) {
      z[j] = zn[j];
      for (int p = 0; p < 3; p++) dz[j][p] = dzn[j][p];
      for (int p = 0; p < 6; p++) d2z[j][p] = d2zn[j][p];
    }
  }
  for (int p = 0; p < 3; p++) g[p] = m.skip_out[p];
  for (int p = 0; p < 6; p++) H6[p] = 0.0;
  for (int j = 0; j < w; j++) {
    for (int p = 0; p < 3; p++) g[p] += m.a[j] * dz[j][p];
    for (int p = 0; p < 6; p++) H6[p] += m.a[j] * d2z[j][p];
  }
}

// the ctx's inner network at its inputs k (3, or 5 for anisotropic kinematics): Alg. 4 for the
// ICNN, closed forms for CANN / Gent-Thomas / ICKAN; H6 = packed upper triangle of the Hessian
__device__ __forceinline__ void ncm_point(const NcmDev& m, const double* kin, double* g, double* H6) {
  if (m.net == 0)
    ncm_alg4(m, kin, g, H6);
  else if (m.kin == 2)
    analytic_point<5>(m, kin, g, H6, nullptr);
  else
    analytic_point<3>(m, kin, g, H6, nullptr);
}

}  // namespace commet
