// DMMA (mma.sync m8n8k4 f64) throughput versus the number of independent
// accumulator chains per warp, one warp per SM sub-partition (128 threads, one
// CTA per SM): exposes the DMMA dependent-issue latency that bounds GEMM tiles
// with few accumulators.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_ilp dmma_ilp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NCH>
__global__ void chains(double* out, int iters) {
  double c[NCH][2];
  for (int i = 0; i < NCH; i++) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
  const double a = 1.0000001, b = 0.9999999;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NCH; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < NCH; i++) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

template <int NCH>
void run(double* d, int sms) {
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chains<NCH><<<sms, 128>>>(d, 100);
  cudaEventRecord(e0);
  chains<NCH><<<sms, 128>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double dmma_per_warp = (double)iters * NCH;
  const double cyc = ms * 1e-3 * clk * 1e3 / dmma_per_warp;  // cycles per DMMA per warp (at the rated clock)
  const double tf = 4.0 * sms * dmma_per_warp * 512.0 / (ms * 1e-3) / 1e12;
  printf("{\"chains\": %d, \"cycles_per_dmma_per_warp\": %.2f, \"tflops\": %.2f}\n", NCH, cyc, tf);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  run<1>(d, sms);
  run<2>(d, sms);
  run<3>(d, sms);
  run<4>(d, sms);
  run<6>(d, sms);
  run<8>(d, sms);
  run<12>(d, sms);
  return 0;
}
