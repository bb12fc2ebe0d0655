// kernel_simple.cu -- one thread per element, Alg. 4 per
// quadrature point in local memory, element matrix in local memory, coloured
// read-modify-write scatter.  A deliberately straightforward CUDA variant
// (COMMET_KERNEL_SIMPLE) kept as a second, algorithmically different GPU
// implementation to cross-check the fused kernel; not the product path.
#include <cuda_runtime.h>

#include "commet_internal.h"
#include "ncm_alg4.cuh"
#include "qp_math.cuh"

namespace commet {

constexpr int kMaxEn = 10;

__global__ void __launch_bounds__(64) simple_kernel(AsmArgs A) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= A.el_count) return;
  const int64_t e = A.el_begin + t;
  const int nen = A.n_en, nq = A.n_q, nd = 3 * nen;
  double ue[kMaxEn * 3];
  for (int a = 0; a < nen; a++) {
    const int64_t node = A.conn[e * nen + a];
    for (int i = 0; i < 3; i++) ue[a * 3 + i] = A.u[3 * node + i];
  }
  double Ke[kMaxEn * 3 * kMaxEn * 3];
  double re[kMaxEn * 3];
  for (int x = 0; x < nd * nd; x++) Ke[x] = 0.0;
  for (int x = 0; x < nd; x++) re[x] = 0.0;
  double trc = 0.0;
  for (int q = 0; q < nq; q++) {
    const double* gN = A.gradN + ((size_t)e * nq + q) * nen * 3;
    const double w = A.qp_w[e * nq + q];
    double F[9];
    for (int i = 0; i < 3; i++)
      for (int J = 0; J < 3; J++) {
        double s = (i == J) ? 1.0 : 0.0;
        for (int a = 0; a < nen; a++) s += ue[a * 3 + i] * gN[a * 3 + J];
        F[i * 3 + J] = s;
      }
    Kin kin;
    kinematics(F, kin);
    if (!(kin.J > 0.0)) atomicMin(A.bad, (unsigned long long)(A.orig[e] * nq + q));
    trc = fmax(trc, kin.I1);
    double kv[9] = {kin.I1 - 3.0, kin.I2 - 3.0, kin.J - 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (A.ncm.kin == 1) isochoric_inputs(kin, kv);
    if (A.ncm.kin == 2) anisotropic_inputs<1>(kin, A.ncm.a0, A.ncm.a1, kv, A.ncm.aniso_iso);
    if (A.ncm.kin == 3) anisotropic_inputs<2>(kin, A.ncm.a0, A.ncm.a1, kv, A.ncm.aniso_iso);
    double g[9], H6[45];
    ncm_point(A.ncm, kv, g, H6);
    if (A.ncm.kin == 1) isochoric_to_standard(kin, g, H6);
    if (A.ncm.kin == 2 && A.ncm.aniso_iso) isochoric_aniso_to_standard<1>(kin, A.ncm.a0, A.ncm.a1, g, H6);
    if (A.ncm.kin == 3 && A.ncm.aniso_iso) isochoric_aniso_to_standard<2>(kin, A.ncm.a0, A.ncm.a1, g, H6);
    const int nk = A.ncm.kin == 2 ? 5 : (A.ncm.kin == 3 ? 9 : 3);
    g[2] += 2.0 * A.ncm.kappa * (kin.J - 1.0) - A.ncm.ref_shift;
    H6[packed_index(nk, 2, 2)] += 2.0 * A.ncm.kappa;
    double P[9], Am[81];
    if (A.ncm.kin == 2)
      stress_tangent_aniso<1>(kin, A.ncm.a0, A.ncm.a1, g, H6, w, P, Am);
    else if (A.ncm.kin == 3)
      stress_tangent_aniso<2>(kin, A.ncm.a0, A.ncm.a1, g, H6, w, P, Am);
    else
      stress_tangent(kin, g, H6, w, P, Am);
    for (int a = 0; a < nen; a++) {
      const double* ga = gN + a * 3;
      for (int i = 0; i < 3; i++) re[a * 3 + i] += P[i * 3 + 0] * ga[0] + P[i * 3 + 1] * ga[1] + P[i * 3 + 2] * ga[2];
      for (int i = 0; i < 3; i++) {
        double X[9];  // X[k*3+L] = sum_J gN_aJ A_iJkL
        for (int kL = 0; kL < 9; kL++)
          X[kL] = ga[0] * Am[(i * 3 + 0) * 9 + kL] + ga[1] * Am[(i * 3 + 1) * 9 + kL] + ga[2] * Am[(i * 3 + 2) * 9 + kL];
        for (int b = 0; b < nen; b++) {
          const double* gb = gN + b * 3;
          for (int k = 0; k < 3; k++)
            Ke[(a * 3 + i) * nd + b * 3 + k] += X[k * 3 + 0] * gb[0] + X[k * 3 + 1] * gb[1] + X[k * 3 + 2] * gb[2];
        }
      }
    }
  }
  atomicMax(A.max_trc, (unsigned long long)__double_as_longlong(trc));
  const uint8_t* sl = A.slot + (size_t)e * nen * nen;
  for (int a = 0; a < nen; a++) {
    const int64_t ln = A.lrow[e * nen + a];
    const bool own = ln < A.n_owned;
    double* rb = own ? A.r_own : A.r_halo;
    double* vb = own ? A.v_own : A.v_halo;
    const int64_t rn = own ? ln : ln - A.n_owned;
    const int64_t rs = A.node_rs[ln];
    const int deg = A.node_deg[ln];
    for (int i = 0; i < 3; i++) {
      rb[3 * rn + i] += re[a * 3 + i];
      const int64_t row0 = rs + (int64_t)i * 3 * deg;
      for (int b = 0; b < nen; b++)
        for (int k = 0; k < 3; k++) vb[row0 + 3 * sl[a * nen + b] + k] += Ke[(a * 3 + i) * nd + b * 3 + k];
    }
  }
}

// the fused kernels' activation on its own: softplus and sigmoid (both forms: the sigmoid-only
// function of the last hidden layer must give the same s)
template <int TB>
__global__ void activation_kernel(const double* __restrict__ y, double* __restrict__ z, double* __restrict__ s,
                                  int64_t n, const double* __restrict__ tab) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    double zz, ss;
    softplus_sig_t<TB>(y[i], tab, zz, ss);
    const double s2 = sigmoid_t<TB>(y[i], tab);
    z[i] = zz;
    s[i] = ss == s2 ? ss : __longlong_as_double(0x7ff8000000000bad);  // NaN if the two forms differ
  }
}

int launch_activation(const double* y, double* z, double* s, int64_t n, const double* tab, int table_bits,
                      void* stream) {
  if (n <= 0) return 0;
  const unsigned g = (unsigned)((n + 255) / 256);
  if (table_bits == 8)
    activation_kernel<8><<<g, 256, 0, (cudaStream_t)stream>>>(y, z, s, n, tab + act_tab_offset<8>());
  else
    activation_kernel<6><<<g, 256, 0, (cudaStream_t)stream>>>(y, z, s, n, tab);
  return (int)cudaGetLastError();
}

int launch_simple(const AsmArgs& a, void* stream) {
  if (a.el_count <= 0) return 0;
  const int bs = 64;
  const int64_t grid = (a.el_count + bs - 1) / bs;
  simple_kernel<<<(unsigned)grid, bs, 0, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace commet
