// material.cu -- material-point calls on the ctx's NCM (SURVEY.md s8(f) rank 3
// groundwork): the inner network's gradient and Hessian on a batch of network
// inputs k (Alg. 4, or the CANN / Gent-Thomas closed forms),
// and the stress-free reference
// normalisation of DESIGN.md reading R11 (s0 = 2 g1 + 4 g2 + g3 at k = 0, so that
// S(F = I) = (2 g1 + 4 g2 + g3 - s0) I = 0).
#include <cuda_runtime.h>

#include "ctx.h"
#include "ncm_alg4.cuh"

namespace {

__global__ void ncm_eval_kernel(NcmDev m, const double* __restrict__ k, double* __restrict__ g,
                                double* __restrict__ H, int64_t n) {
  const int nk = m.kin == 2 ? 5 : (m.kin == 3 ? 9 : 3), nh = nk * (nk + 1) / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double gi[9], Hi[45];
    ncm_point(m, k + nk * i, gi, Hi);
    for (int p = 0; p < nk; p++) g[nk * i + p] = gi[p];
    for (int p = 0; p < nh; p++) H[nh * i + p] = Hi[p];
  }
}

__global__ void ref_shift_kernel(NcmDev m, double* out) {
  const double k0[3] = {0.0, 0.0, 0.0};
  double g[3], H[6];
  ncm_point(m, k0, g, H);
  if (m.kin == 1) {  // isochoric inputs: carry the gradient to (I1, I2, J) at F = I
    Kin ki{};
    ki.I1 = 3.0;
    ki.I2 = 3.0;
    ki.J = 1.0;
    isochoric_to_standard(ki, g, H);
  }
  out[0] = 2.0 * g[0] + 4.0 * g[1] + g[2];  // the penalty's 2 kappa (J - 1) vanishes at J = 1
}

}  // namespace

extern "C" commet_status commet_ncm_eval(commet_ctx c, const double* k, double* g, double* H, int64_t n,
                                         void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (n < 0 || (n > 0 && (!k || !g || !H))) return fail(c, COMMET_ERR_ARG, "k, g or H NULL, or n < 0");
  if (n == 0) return COMMET_OK;
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int64_t nb = std::min<int64_t>((n + 63) / 64, 148 * 16);
  ncm_eval_kernel<<<(unsigned)nb, 64, 0, (cudaStream_t)cuda_stream>>>(c->ncm, k, g, H, n);
  CUDA_TRY(c, cudaGetLastError());
  return COMMET_OK;
}

extern "C" commet_status commet_normalize_reference(commet_ctx c, double* s0) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (c->ncm.kin >= 2)
    return fail(c, COMMET_ERR_ARG, "anisotropic kinematics: S(I) has a structural part (2 g4 + 4 g5) A0 A0 that a "
                "volumetric -s0 (J - 1) term cannot cancel");
  CUDA_TRY(c, cudaSetDevice(c->device));
  DevBuf<double> d;
  CUDA_TRY(c, d.alloc(1));
  NcmDev m = c->ncm;
  ref_shift_kernel<<<1, 1>>>(m, d.p);
  CUDA_TRY(c, cudaGetLastError());
  double h = 0.0;
  CUDA_TRY(c, cudaMemcpy(&h, d.p, sizeof h, cudaMemcpyDeviceToHost));
  c->ncm.ref_shift = h;
  if (s0) *s0 = h;
  return COMMET_OK;
}

extern "C" commet_status commet_material_eval(commet_ctx c, const double* F, int64_t n, double* W, double* tau,
                                              double* cc, void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (n < 0 || (n > 0 && !F)) return fail(c, COMMET_ERR_ARG, "F is NULL or n = %lld < 0", (long long)n);
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  c->last_stream = st;
  CUDA_TRY(c, cudaMemsetAsync(c->bad.p, 0xff, sizeof(unsigned long long), st));
  CUDA_TRY(c, cudaMemsetAsync(c->max_trc.p, 0, sizeof(unsigned long long), st));
  if (n == 0) return COMMET_OK;
  AsmArgs a{};
  a.n_en = 1;
  a.n_q = 1;
  a.el_begin = 0;
  a.el_count = n;
  a.Fin = F;
  a.Wout = W;
  a.tau_out = tau;
  a.c_out = cc;
  a.bad = c->bad.p;
  a.max_trc = c->max_trc.p;
  a.ncm = c->ncm;
  const int rc = launch_material(a, st);
  if (rc) return fail(c, COMMET_ERR_CUDA, "material kernel launch: %s", cudaGetErrorString((cudaError_t)rc));
  return COMMET_OK;
}
