// exchange.cu -- unpack of received halo segments: owned CSR values and
// residual entries += received contributions (one launch per sender, in rank
// order, so the summation order is deterministic).
#include <cuda_runtime.h>

#include "commet_internal.h"

namespace commet {

__global__ void unpack_kernel(const double* __restrict__ vals, const int64_t* __restrict__ vmap, int64_t nv,
                              double* __restrict__ csr, const double* __restrict__ res,
                              const int64_t* __restrict__ rmap, int64_t nr, double* __restrict__ r) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) csr[vmap[i]] += vals[i];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += stride) r[rmap[i]] += res[i];
}

int launch_unpack(const double* vals, const int64_t* vmap, int64_t nv, double* csr, const double* res,
                  const int64_t* rmap, int64_t nr, double* r, void* stream) {
  const int64_t n = nv > nr ? nv : nr;
  if (n <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (n + 255) / 256;
  if (grid > 8 * sms) grid = 8 * sms;
  unpack_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(vals, vmap, nv, csr, res, rmap, nr, r);
  return (int)cudaGetLastError();
}

}  // namespace commet
