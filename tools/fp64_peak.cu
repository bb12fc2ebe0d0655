// fp64 roofline microbenchmark for the B200 (sm_100a): measures the DFMA and
// DMMA (mma.sync m8n8k4 f64) issue-limited peaks, their co-issue behaviour and
// the cost of the fp64 softplus/sigmoid pair the NCM needs per neuron.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
// Usage: fp64_peak [seconds_for_sustained]
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int NCH = 16;  // independent DFMA chains per thread

__global__ void dfma_kernel(double* out, double x, double y, int iters) {
  double acc[NCH];
#pragma unroll
  for (int i = 0; i < NCH; i++) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 8; r++)
#pragma unroll
      for (int i = 0; i < NCH; i++) acc[i] = fma(acc[i], x, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; i++) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

constexpr int NMMA = 8;  // independent DMMA accumulators per warp
__global__ void dmma_kernel(double* out, double x, int iters) {
  double a = x + threadIdx.x * 1e-6, b = x - threadIdx.x * 1e-6;
  double c[NMMA][2];
#pragma unroll
  for (int i = 0; i < NMMA; i++) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int i = 0; i < NMMA; i++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NMMA; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// warps alternate role: even warps DMMA, odd warps DFMA (same flop count per iter)
__global__ void mixed_kernel(double* out, double x, double y, int iters) {
  int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double acc[NCH];
#pragma unroll
    for (int i = 0; i < NCH; i++) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int i = 0; i < NCH; i++) acc[i] = fma(acc[i], x, y);
    }
#pragma unroll
    for (int i = 0; i < NCH; i++) s += acc[i];
  } else {
    double a = x + threadIdx.x * 1e-6, b = x - threadIdx.x * 1e-6;
    double c[NMMA][2];
#pragma unroll
    for (int i = 0; i < NMMA; i++) { c[i][0] = i; c[i][1] = -i; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int i = 0; i < NMMA; i++)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < NMMA; i++) s += c[i][0] + c[i][1];
  }
  if (s == 12345.678) out[0] = s;
}

// softplus + sigmoid per element, stable form (what the NCM epilogue needs)
__global__ void softplus_kernel(const double* in, double* out, long n, int reps) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double y = in[i], acc = 0;
  for (int r = 0; r < reps; r++) {
    double e = exp(-fabs(y));
    double sp = fmax(y, 0.0) + log1p(e);
    double inv = 1.0 / (1.0 + e);
    double sg = (y >= 0) ? inv : e * inv;
    acc += sp + sg;
    y = y * 0.999 + 1e-3 * sg;
  }
  out[i] = acc;
}

static float time_kernel(void (*launch)(void*), void* arg, int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  launch(arg); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; r++) launch(arg);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

struct Cfg { double* out; int grid, block, iters; };
static void l_dfma(void* p) { Cfg* c = (Cfg*)p; dfma_kernel<<<c->grid, c->block>>>(c->out, 1.0000001, 1e-9, c->iters); }
static void l_dmma(void* p) { Cfg* c = (Cfg*)p; dmma_kernel<<<c->grid, c->block>>>(c->out, 1.0000001, c->iters); }
static void l_mixed(void* p) { Cfg* c = (Cfg*)p; mixed_kernel<<<c->grid, c->block>>>(c->out, 1.0000001, 1e-9, c->iters); }

int main(int argc, char** argv) {
  double sustain_s = argc > 1 ? atof(argv[1]) : 4.0;
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"smem_optin_per_block\": %zu, \"regs_per_sm\": %d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  int sms = p.multiProcessorCount;
  for (int block : {128, 256, 512}) {
    for (int per_sm : {1, 2, 4}) {
      Cfg c{out, sms * per_sm, block, 2000};
      float ms = time_kernel(l_dfma, &c, 5);
      double fl = 2.0 * NCH * 8.0 * c.iters * (double)c.grid * c.block;
      printf("{\"kind\": \"dfma\", \"block\": %d, \"ctas_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", block, per_sm, ms, fl / ms / 1e9);
      Cfg d{out, sms * per_sm, block, 1000};
      ms = time_kernel(l_dmma, &d, 5);
      fl = 2.0 * 256 * NMMA * 4.0 * d.iters * (double)d.grid * (d.block / 32);
      printf("{\"kind\": \"dmma_m8n8k4\", \"block\": %d, \"ctas_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", block, per_sm, ms, fl / ms / 1e9);
    }
  }
  {
    // mixed: half the warps DFMA (flops per warp per iter: 32*NCH*8*2), half DMMA (NMMA*4*256*2)
    Cfg c{out, sms * 2, 256, 2000};
    float ms = time_kernel(l_mixed, &c, 5);
    double wps = c.grid * (c.block / 32) / 2.0;
    double fl = wps * c.iters * (32.0 * NCH * 8 * 2 + NMMA * 4.0 * 256 * 2);
    printf("{\"kind\": \"mixed_dfma_dmma\", \"ms\": %.4f, \"tflops\": %.3f}\n", ms, fl / ms / 1e9);
  }
  {
    long n = (long)sms * 2048 * 8; int reps = 64;
    double *in, *o; CK(cudaMalloc(&in, n * 8)); CK(cudaMalloc(&o, n * 8));
    CK(cudaMemset(in, 0, n * 8));
    softplus_kernel<<<(n + 255) / 256, 256>>>(in, o, n, reps); CK(cudaDeviceSynchronize());
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a));
    for (int r = 0; r < 5; r++) softplus_kernel<<<(n + 255) / 256, 256>>>(in, o, n, reps);
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= 5;
    printf("{\"kind\": \"softplus_sigmoid_f64\", \"evals_per_s\": %.4e}\n", n * (double)reps / (ms * 1e-3));
  }
  {
    // sustained DFMA and DMMA for ~sustain_s seconds each
    for (int which = 0; which < 2; which++) {
      Cfg c{out, sms * 2, 256, which == 0 ? 2000 : 1000};
      float ms1 = time_kernel(which == 0 ? l_dfma : l_dmma, &c, 3);
      int reps = (int)(sustain_s * 1000.0 / ms1) + 1;
      float ms = time_kernel(which == 0 ? l_dfma : l_dmma, &c, reps);
      double fl = which == 0 ? 2.0 * NCH * 8.0 * c.iters * (double)c.grid * c.block
                             : 2.0 * 256 * NMMA * 4.0 * c.iters * (double)c.grid * (c.block / 32);
      printf("{\"kind\": \"%s_sustained\", \"reps\": %d, \"seconds\": %.2f, \"tflops\": %.3f}\n",
             which == 0 ? "dfma" : "dmma_m8n8k4", reps, reps * ms / 1e3, fl / ms / 1e9);
    }
  }
  return 0;
}
