// ickan.cuh -- the ICKAN inner network (App. B.3; SURVEY.md s8(f)
// rank 4) for one point: N, g = dN/dk, H = d2N/dk2 (upper 00,01,02,11,12,22) by
// forward mode through the layers.  Splines are uniform cubic B-splines evaluated
// with the closed-form local basis of a knot span (the oracle uses De Boor's
// recursion instead):  on span j, t in [0, 1),
//   psi = c_j (1-t)^3/6 + c_{j+1} (3t^3 - 6t^2 + 4)/6 + c_{j+2} (-3t^3 + 3t^2 + 3t + 1)/6 + c_{j+3} t^3/6,
// outside [xmin, xmax] continued linearly with the end slope (SPEC's reading).
#pragma once
#include "commet_internal.h"

namespace commet {

__device__ __forceinline__ void cubic_spline(const double* __restrict__ c, int nb, double xmin, double xmax,
                                             double x, double& v, double& d1, double& d2) {
  const int G = nb - 3;  // knot intervals inside [xmin, xmax]
  const double h = (xmax - xmin) / G, ih = 1.0 / h;
  const double xe = fmin(fmax(x, xmin), xmax);
  int j = (int)floor((xe - xmin) * ih);
  j = j < 0 ? 0 : (j > G - 1 ? G - 1 : j);
  const double t = (xe - xmin) * ih - j, t2 = t * t, t3 = t2 * t, s = 1.0 - t;
  const double c0 = __ldg(c + j), c1 = __ldg(c + j + 1), c2 = __ldg(c + j + 2), c3 = __ldg(c + j + 3);
  const double val = (c0 * s * s * s + c1 * (3.0 * t3 - 6.0 * t2 + 4.0) + c2 * (-3.0 * t3 + 3.0 * t2 + 3.0 * t + 1.0) +
                      c3 * t3) * (1.0 / 6.0);
  const double der = (-c0 * s * s + c1 * (3.0 * t2 - 4.0 * t) + c2 * (-3.0 * t2 + 2.0 * t + 1.0) + c3 * t2) * 0.5 * ih;
  const double sec = (c0 * s + c1 * (3.0 * t - 2.0) + c2 * (1.0 - 3.0 * t) + c3 * t) * ih * ih;
  if (x != xe) {
    v = val + der * (x - xe);
    d1 = der;
    d2 = 0.0;
  } else {
    v = val;
    d1 = der;
    d2 = sec;
  }
}

template <int NK, class M>
__device__ __forceinline__ double ickan_eval(const M& m, const double* kin, double* __restrict__ g,
                                             double* __restrict__ H6) {
  constexpr int MW = 16, NH = NK * (NK + 1) / 2;
  double z[MW], dz[MW][NK], hz[MW][NH], y[MW], dy[MW][NK], hy[MW][NH];
  int nin = NK;
  for (int j = 0; j < NK; j++) {
    z[j] = kin[j];
    for (int p = 0; p < NK; p++) dz[j][p] = (p == j) ? 1.0 : 0.0;
    for (int p = 0; p < NH; p++) hz[j][p] = 0.0;
  }
  int e = 0;
  for (int r = 0; r < m.kan_R; r++) {
    const int nout = m.kan_width[r + 1];
    const double xmin = __ldg(m.kan_grid + 2 * r), xmax = __ldg(m.kan_grid + 2 * r + 1);
    for (int i = 0; i < nout; i++) {
      double yy = 0.0, d[NK], hh[NH];
      for (int p = 0; p < NK; p++) d[p] = 0.0;
      for (int p = 0; p < NH; p++) hh[p] = 0.0;
      for (int j = 0; j < nin; j++, e++) {
        double v, d1, d2;
        cubic_spline(m.kan_c + (size_t)e * m.kan_nb, m.kan_nb, xmin, xmax, z[j], v, d1, d2);
        const double w = __ldg(m.kan_w + e), wd1 = w * d1, wd2 = w * d2;
        yy += w * v;
        for (int p = 0; p < NK; p++) d[p] += wd1 * dz[j][p];
        int x = 0;
        for (int p = 0; p < NK; p++)
          for (int q = p; q < NK; q++, x++) hh[x] += wd2 * dz[j][p] * dz[j][q] + wd1 * hz[j][x];
      }
      y[i] = yy;
      for (int p = 0; p < NK; p++) dy[i][p] = d[p];
      for (int p = 0; p < NH; p++) hy[i][p] = hh[p];
    }
    for (int i = 0; i < nout; i++) {
      z[i] = y[i];
      for (int p = 0; p < NK; p++) dz[i][p] = dy[i][p];
      for (int p = 0; p < NH; p++) hz[i][p] = hy[i][p];
    }
    nin = nout;
  }
  double N = z[0];
  for (int p = 0; p < NK; p++) g[p] = dz[0][p];
  for (int p = 0; p < 3; p++) {
    g[p] += m.skip_out[p];
    N += m.skip_out[p] * kin[p];
  }
  for (int p = 0; p < NH; p++) H6[p] = hz[0][p];
  return N;
}

// analytic networks (NET = 1 path) on NK inputs: gradient / packed Hessian (and value if N != nullptr)
template <int NK = 3, class M>
__device__ __forceinline__ void analytic_point(const M& m, const double* kin, double* g, double* H6, double* N) {
  if (m.net == 3) {
    const double v = ickan_eval<NK>(m, kin, g, H6);
    if (N) *N = v;
    return;
  }
  analytic_net(m.net, m.cann_n, m.cann_f, m.cann_w1, m.cann_w2, m.gt, m.skip_out, kin, g, H6, NK);
  if (N) *N = analytic_value(m.net, m.cann_n, m.cann_f, m.cann_w1, m.cann_w2, m.gt, m.skip_out, kin, NK);
}

}  // namespace commet
