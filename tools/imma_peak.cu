// Integer / half tensor-core throughput of the warp-level mma.sync path on the
// B200 (sm_100a), for the Ozaki-style fp64 emulation question of SURVEY.md
// s8(f) rank 4: an emulated w x w hidden-layer GEMM needs s(s+1)/2 int8 slice
// products, so the int8 rate available to a fused per-CTA kernel decides it.
// Measures mma.sync m16n8k32 s8.s8.s32 and m16n8k16 f16.f16.f32 (legacy warp
// MMA, what a fused kernel can issue without TMEM) at several CTAs/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imma_peak imma_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int NACC = 8;  // independent accumulators per warp

__global__ void imma_kernel(int* out, int x, int iters) {
  unsigned a0 = x + threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x5a5a, b1 = a0 ^ 0x3c3c;
  int c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; i++) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int i = 0; i < NACC; i++)
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 0x12345) out[0] = s;
}

__global__ void hmma_kernel(float* out, unsigned x, int iters) {
  unsigned a0 = x + threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x1111, b1 = a0 ^ 0x2222;
  float c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; i++) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int i = 0; i < NACC; i++)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int* di;
  float* df;
  CK(cudaMalloc(&di, 64));
  CK(cudaMalloc(&df, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 2000;
  printf("{\"what\": \"warp mma.sync tensor throughput (tools/imma_peak.cu)\", \"sms\": %d, \"results\": [\n", sms);
  bool first = true;
  for (int kind = 0; kind < 2; kind++)
    for (int block : {128, 256, 512})
      for (int per_sm : {1, 2, 4}) {
        const int grid = sms * per_sm;
        for (int w = 0; w < 2; w++) {  // warm-up, then timed
          CK(cudaEventRecord(e0));
          if (kind == 0) imma_kernel<<<grid, block>>>(di, 3, iters);
          else hmma_kernel<<<grid, block>>>(df, 3u, iters);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
        }
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        // ops per mma: 2 * M * N * K
        const double per = kind == 0 ? 2.0 * 16 * 8 * 32 : 2.0 * 16 * 8 * 16;
        const double ops = per * 4 * NACC * (double)iters * (block / 32) * grid;
        printf("%s  {\"kind\": \"%s\", \"block\": %d, \"ctas_per_sm\": %d, \"ms\": %.4f, \"tops\": %.1f}", first ? "" : ",\n",
               kind == 0 ? "imma_m16n8k32_s8" : "hmma_m16n8k16_f16_f32", block, per_sm, ms, ops / (ms * 1e-3) / 1e12);
        first = false;
      }
  printf("\n]}\n");
  return 0;
}
