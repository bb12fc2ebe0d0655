// kernel_fused.cu -- the product path: ONE kernel per element colour that runs
// every step of the hot path for a batch of
// elements held in shared memory; nothing but u, the element inputs and the
// scatter touch HBM.
//
// Per CTA iteration (E elements = Q quadrature points):
//   0  stage dN/dX, w, gather u_e                            (a1)
//   1  F, C, I1, I2, J -> k = (I1-3, I2-3, J-1), det F flag   (a2, a3)
//   2  layer 1 (3 -> w): y, softplus, sigmoid                 (a4)
//   3  value pass, hidden layers l = 2..L:  Y = W_l Z          (a4, DMMA GEMM)
//   4  adjoint pass l = L..2:  Lambda = W_l^T M               (a4, DMMA GEMM)
//   5  g = W1^T mu_1 (+skips), H_1 = W1^T diag(c_1) W1         (a4)
//   6  Jacobian pass l = 2..L: J_l = W_l (s_{l-1} (.) J_{l-1}) (a4, DMMA GEMM)
//      H += J_l^T diag(c_l) J_l on the fly, c_l = lambda_l s_l (1-s_l)
//   7  penalty, S, A = d2W/dFdF (scaled by w)                 (a5, a6)
//   8  element rows: K_e, r_e; coloured read-modify-write scatter (a7, a8)
// The inner-network derivatives are the exact Hessian of Alg. 4
// obtained with 5 w^2 FMA per hidden layer instead of
// Alg. 4's 10 w^2.  Hidden-layer contractions use the
// fp64 tensor path (mma.sync m8n8k4 f64 = SASS DMMA.8x8x4): on B200 it shares
// the fp64 datapath with DFMA (measured, profiles/r01_fp64_peak.json) but
// needs ~8x fewer issue slots and register-file reads per FMA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "commet_internal.h"
#include "qp_math.cuh"
#include "ickan.cuh"

// element stage on DMMA: 1 = hex8 only (measured: +6% c3, -4% c4 where 10 nodes pad to 16)
#ifndef COMMET_DMMA_ELEM
#define COMMET_DMMA_ELEM 1
#endif
#ifndef COMMET_PREFETCH
#define COMMET_PREFETCH 1
#endif
#ifndef COMMET_FRAG_PF
#define COMMET_FRAG_PF 2
#endif
#ifndef COMMET_PD_V
#define COMMET_PD_V 2
#endif
#ifndef COMMET_PD_J
#define COMMET_PD_J 2
#endif
// analytic-network (NET = 1) instantiations, measured on c3 (tools/ab_bench.py AB_NET=...):
// ICKAN and the 5-input networks run 32 qps per CTA iteration (one full warp in the per-qp
// stage 7a; 16: ICKAN -19 %, CANN-5 -21 %) at 2 CTAs/SM (no spills at 254 registers;
// 4 CTAs: ICKAN-5 -21 %, CANN-5 -20 %; ICKAN at 3: -2 %); Gent-Thomas / CANN keep
// 16 qps (32: -15 % / -6 %)
#ifndef COMMET_ICKAN_MINB
#define COMMET_ICKAN_MINB 2
#endif
#ifndef COMMET_ANALYTIC_Q
#define COMMET_ANALYTIC_Q 32  // qps per batch of the CANN / Gent-Thomas instantiation (round 2: 32 with the split stage 7a, GT -8 %, CANN -15 %)
#endif
#ifndef COMMET_ANALYTIC_MINB
#define COMMET_ANALYTIC_MINB 3  // CTAs per SM of the CANN / GT kernels (round 2 at 32 qps: 3 as fast as 4 for GT, CANN -2 %)
#endif
#ifndef COMMET_FWD
#define COMMET_FWD 1  // forward value+Jacobian sweep, Hessian terms in the backward pass (L <= 3, no skips)
#endif
#ifndef COMMET_FWD_MINW
#define COMMET_FWD_MINW 64  // narrowest width that takes the forward sweep (w = 64: measured -4.8 % c3 time, round 2)
#endif
#ifndef COMMET_ACT_TB
#define COMMET_ACT_TB 8  // forward-sweep activations on 256-entry tables (lower polynomial degrees)
#endif
#ifndef COMMET_POST_PAR
#define COMMET_POST_PAR 1  // ICNN with two network batches per element batch (32 qps): stage 7a split over the four warps (post_qp_part); at 16 qps measured no gain (c3 +0.3 %, c4 +3 %)
#endif
#ifndef COMMET_WS
#define COMMET_WS 0  // warp-specialised kernel (ws_kernel) for the hex8 forward-sweep ICNN: measured c3 -2.2 %, c5 +4 % -> off
#endif
#ifndef COMMET_WS_NWE
#define COMMET_WS_NWE 4  // element warps per CTA of the warp-specialised kernel (4: one warpgroup, setmaxnreg)
#endif
#ifndef COMMET_WS_NREG_NET
#define COMMET_WS_NREG_NET 168  // registers of the network warpgroup after setmaxnreg (element: 256 - this)
#endif
#ifndef COMMET_ROWS3
#define COMMET_ROWS3 1  // stage 7b: three A rows (i, J = 0..2) per item
#endif
#ifndef COMMET_ELEM_HALF
#define COMMET_ELEM_HALF 1  // hex8 ICNN stage 8 with 4 elements per element batch: one warp per (element, i-half) (at 2 elements: c3 9.75 -> 9.83 ms)
#endif
#ifndef COMMET_WS_PAR7
#define COMMET_WS_PAR7 0  // warp-specialised kernel: stage 7a split over the four element warps (measured: c3 9.52 -> 9.78 ms)
#endif
#ifndef COMMET_POST_PAR_NET1
#define COMMET_POST_PAR_NET1 1  // analytic networks: stage 7a split over the four warps (GT c3 -12 %, CANN -9 %)
#endif
#ifndef COMMET_ELEM_HALF_NET1
#define COMMET_ELEM_HALF_NET1 1  // analytic networks, hex8: stage 8 by (element, i-half) (GT / CANN c3 -1 %)
#endif
#ifndef COMMET_Q_KIN3
#define COMMET_Q_KIN3 16  // qps per batch of the two-vector (9-input) kernels
#endif
#ifndef COMMET_META_EARLY
#define COMMET_META_EARLY 0  // hex8 stage 8 by (element, i-half): scatter metadata, first hop (lrow, slots) issued at the end of stage 7a (1) or its start (2), the second (row starts, degrees) before the K_e DMMAs; 0: both after them (measured: 1 / 2 slower -- GT c3 1.57 -> 1.60 / 1.64 ms, ICNN c3 9.50 -> 9.74 / 9.78, c5 635 -> 646; r02_ab_meta_early.txt)
#endif
#ifndef COMMET_RS
#define COMMET_RS 1  // forward sweep: Hessian / gradient partials reduced over the tile rows by reduce-scatter shuffles
#endif
#ifndef COMMET_L2_EF
#define COMMET_L2_EF 0  // streamed element data and the scatter with an L2 evict-first policy (measured: c5 -0.1 %, c3 -0.3 %, c4 +0.3 %, Gent-Thomas c3 +4.7 % -> off; r02_ab_l2_hints.txt)
#endif
#ifndef COMMET_L2_EL
#define COMMET_L2_EL 0  // weight fragments with an L2 evict-last policy (with EF: c5 -0.2 %, c3 -0.5 % -> off)
#endif
#ifndef COMMET_KUNROLL
#define COMMET_KUNROLL 2  // k-loop unroll of the network GEMMs (0: full; 2 measured c5 603 -> 588 ms, c4 -0.9 %, c3 +0.4 %: the fully unrolled GEMMs overflow the instruction cache, r02_ab_kunroll.txt)
#endif
#define COMMET_PRAGMA(x) _Pragma(#x)
#define COMMET_UNROLL(n) COMMET_PRAGMA(unroll n)
#ifndef COMMET_FWD_LOOP
#define COMMET_FWD_LOOP 0  // forward sweep: layer loop kept rolled (1) or unrolled (0) (1 measured: spills 104 -> 240 B, c3 +4.9 %, c5 +3.3 %; r02_ab_fwd_loop.txt)
#endif
#ifndef COMMET_BPF
#define COMMET_BPF 1  // network GEMMs: B fragments loaded one half k-step ahead (measured c3 -0.8 %, c5 -0.35 %, c4 +0.1 %; r02_ab_bpf.txt)
#endif
#ifndef COMMET_E8_UNROLL
#define COMMET_E8_UNROLL 2  // ICNN hex8 stage 8 (element, i-half): unroll of the (q, J) k-loop (0: full; 2 measured c3 -1.9 %, c5 -2.8 %, spills 92 -> 0 B; the analytic networks keep the full unroll: Gent-Thomas +3.7 %, CANN +4.4 % with 2; r02_ab_e8.txt)
#endif
#ifndef COMMET_T7_ROLL
#define COMMET_T7_ROLL 0  // stage 7b three-rows item: the k loop rolled (smaller code; measured c3 +0.7 %, c5 +0.7 % -> off)
#endif
#ifndef COMMET_ACT_TB_EB
#define COMMET_ACT_TB_EB 6  // activation table bits of the two-batch kernels (8 fits only with COMMET_FUSE_GH; measured with it: c3 +0.6 %, c5 +0.2 % -> 6)
#endif
#ifndef COMMET_FUSE_GH
#define COMMET_FUSE_GH 0  // forward sweep + two-batch element stage: (g, H) written straight into qgH (one barrier and the qg / qH / gsk buffers fewer; measured c3 +0.1-0.3 %, c5 +0.15 % (8 B spill) -> off; r02_ab_fuse_gh.txt)
#endif
#ifndef COMMET_VSTORE
#define COMMET_VSTORE 1  // forward-sweep epilogue: the two qps of a lane stored with one 16-byte store per row (c3 -0.8 %, c4 -0.7 %, c5 564 -> 560 ms; r02_ab_vstore.txt)
#endif
#ifndef COMMET_VSTORE2
#define COMMET_VSTORE2 1  // forward-sweep backward epilogue (layer 3): 16-byte shared loads / stores of a lane's two qps  (c3 -0.1 %, c4 / c5 neutral; r02_ab_vstore2.txt)
#endif
#ifndef COMMET_EB
#define COMMET_EB 2  // network batches per element batch (ICNN assembly; c3 9.72 -> 9.43 ms with the two below)
#endif
#ifndef COMMET_PINGPONG
#define COMMET_PINGPONG 0  // measured neutral (c3 10.31 vs 10.26 ms): barriers kept
#endif

namespace commet {

#ifdef COMMET_STAGE_PROF
// tuning builds only: per-stage wall cycles seen by thread 0 of every CTA (summed over CTAs)
__device__ unsigned long long g_stage_cycles[16];
#define STAGE_MARK(i)                               \
  if (tid == 0) {                                   \
    const long long now_ = clock64();               \
    st_acc[i] += now_ - st_acc[15];                 \
    st_acc[15] = now_;                              \
  }
#else
#define STAGE_MARK(i)
#endif

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Sum of v[0..N) over the 8 lanes of a warp that share lane & 3 (the 8 rows g of a DMMA accumulator
// tile), scattered over those lanes (reduce-scatter, xor 16 / 8 / 4): ceil(N/2) + ceil(N/4) + ceil(N/8)
// shuffles instead of 3N for a full butterfly.  On return lane (g = lane >> 2) owns the sums of the
// entries rs_index<N>(g, i), i < RS3 (entries >= N are zero padding; rs_index < 0 marks them).
template <int N> struct RS {
  static constexpr int K1 = (N + 1) / 2, K2 = (K1 + 1) / 2, K3 = (K2 + 1) / 2;
};
template <int N>
__device__ __forceinline__ int rs_index(int g, int i) {
  constexpr int K1 = RS<N>::K1, K2 = RS<N>::K2, K3 = RS<N>::K3;
  const int b4 = (g >> 2) & 1, b3 = (g >> 1) & 1, b2 = g & 1;
  const int l3 = b2 * K3 + i, l2 = b3 * K2 + l3, idx = b4 * K1 + l2;
  return (l3 < K2 && l2 < K1 && idx < N) ? idx : -1;
}
template <int N>
__device__ __forceinline__ void reduce_scatter8(const double (&v)[N], double (&out)[RS<N>::K3]) {
  constexpr int K1 = RS<N>::K1, K2 = RS<N>::K2, K3 = RS<N>::K3;
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  double w1[K1], w2[K2];
#pragma unroll
  for (int i = 0; i < K1; i++) {
    const double lo = v[i], hi = i + K1 < N ? v[i + K1] : 0.0;
    w1[i] = (b4 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b4 ? lo : hi, 16);
  }
#pragma unroll
  for (int i = 0; i < K2; i++) {
    const double lo = w1[i], hi = i + K2 < K1 ? w1[i + K2] : 0.0;
    w2[i] = (b3 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b3 ? lo : hi, 8);
  }
#pragma unroll
  for (int i = 0; i < K3; i++) {
    const double lo = w2[i], hi = i + K3 < K2 ? w2[i + K3] : 0.0;
    out[i] = (b2 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b2 ? lo : hi, 4);
  }
}

// CTA-wide barrier of the network stages: __syncthreads, or in the warp-specialised kernel the
// named barrier 1 of the NTHR network threads (the element warps run their own schedule)
template <class C>
__device__ __forceinline__ void net_sync() {
  if constexpr (C::WS)
    asm volatile("bar.sync 1, %0;" ::"n"(C::NTHR) : "memory");
  else
    __syncthreads();
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// L1 prefetch of the first NK k-steps of a warp's A fragments for the NEXT GEMM, issued at the
// start of the current epilogue so the GEMM after the barrier does not start on an L2 round trip
// (measured: +1.6% at w = 128, -0.5% at w = 64 -> w >= 128 only)
template <int MT, int KT2, int NK>
__device__ __forceinline__ void frag_prefetch(const double* __restrict__ Af, int mt0) {
#if COMMET_FRAG_PF
  if (KT2 < 16) return;
  const int lane = threadIdx.x & 31;
  constexpr int NL = MT * NK * 4;  // 128-byte lines (a fragment is 512 bytes)
#pragma unroll
  for (int x = lane; x < NL; x += 32) {
    const int i = x / (NK * 4), r = x % (NK * 4);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(Af + ((size_t)(mt0 + i) * KT2 + r / 4) * 64 + (r % 4) * 16));
  }
#endif
}

// Output addresses of the scatter.  off: offset of the entry in this rank's owned CSR values,
// or in the halo buffer for halo rows (row-nodes la >= n_owned).  Peer mode (multi-GPU, NVLink
// P2P): halo rows go straight to the owning rank's buffers through the owner's receive maps,
// replacing the NCCL exchange + unpack.
__device__ __forceinline__ double* vout(const AsmArgs& A, int64_t la, int64_t off) {
#ifdef COMMET_DEBUG_CHECKS  // debug builds: every scatter address inside its buffer
  if (la < 0 || off < 0 || (la < A.n_owned ? off >= A.dbg_nnz : off >= A.dbg_nnz_halo)) {
    printf("commet debug: CSR scatter out of range (row node %lld, offset %lld)\n", (long long)la, (long long)off);
    __trap();
  }
#endif
  if (la < A.n_owned) return A.v_own + off;
  if (!A.peer) return A.v_halo + off;
  return A.peer_v[__ldg(A.halo_peer + (la - A.n_owned))] + __ldg(A.peer_vmap + off);
}
__device__ __forceinline__ double* rout(const AsmArgs& A, int64_t la, int i) {
#ifdef COMMET_DEBUG_CHECKS
  if (la < 0 || i < 0 || i > 2 || la >= A.n_owned + A.dbg_n_halo) {
    printf("commet debug: residual scatter out of range (row node %lld)\n", (long long)la);
    __trap();
  }
#endif
  if (la < A.n_owned) return A.r_own + 3 * la + i;
  const int64_t hr = 3 * (la - A.n_owned) + i;
  if (!A.peer) return A.r_halo + hr;
  return A.peer_r[__ldg(A.halo_peer + (la - A.n_owned))] + __ldg(A.peer_rmap + hr);
}

__device__ __forceinline__ double2 ldg2(const double* p) {
#if COMMET_L2_EL  // hidden-layer weight fragments: kept in L2 ahead of the streamed data
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  double2 v;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
#else
  return __ldg(reinterpret_cast<const double2*>(p));
#endif
}

// Streamed element data (dN/dX, w, conn, u, scatter metadata: each word read once per colour
// launch) and the CSR / residual scatter: L2 evict-first, so the lines that ARE reused -- the
// hidden-layer weight fragments, the activation tables and the kernel's own instructions -- are
// not evicted by the stream (at c5 the streamed data is ~60 GB per assembly against a 126 MB L2;
// ncu showed 12 % of the warp samples waiting on instruction fetch there against 5 % at c3)
#if COMMET_L2_EF
__device__ __forceinline__ uint64_t l2_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(l2_first()));
  return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_first()));
  return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2_first()));
  return v;
}
__device__ __forceinline__ int64_t ld_stream(const int64_t* p) {
  int64_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(l2_first()));
  return v;
}
__device__ __forceinline__ uint8_t ld_stream(const uint8_t* p) {
  uint16_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(l2_first()));
  return (uint8_t)v;
}
__device__ __forceinline__ void red_add(double* a, double v) {
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(l2_first()));
}
#else
template <class T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldg(p); }
__device__ __forceinline__ void red_add(double* a, double v) { atomicAdd(a, v); }
#endif

// ---------------------------------------------------------------------------
// compile-time tiling
// ---------------------------------------------------------------------------
// NET_: 0 = ICNN (DMMA network stages 2-6), 1 = analytic inner network (CANN or
// Gent-Thomas, evaluated per qp in stage 7a; W is then unused).  KIN_: 0 standard
// invariants, 1 isochoric, 2 / 3 anisotropic with one / two structural vectors, 4 / 5 the same on the
// isochoric inputs (all compile-time, so the standard path carries no extra code)
// MODE_: 0 = FE assembly; 1 = material points (F in; Psi, tau, c out; NEN = NQ = 1)
// WS_: warp-specialised kernel (ws_kernel): the NW_ network warps are joined by NWE element warps
// that run stages 7-8 of batch b (and load the inputs of batch b + 2) while the network warps
// compute batch b + 1; the network warps then synchronise among themselves with a named barrier
template <int W_, int Q_, int NEN_, int NQ_, int MINB_ = 3, int NET_ = 0, int KIN_ = 0, int MODE_ = 0, int NW_ = 4,
          int WS_ = 0>
struct Cfg {
  static constexpr int W = W_, Q = Q_, NEN = NEN_, NQ = NQ_, NET = NET_, KIN = KIN_, MODE = MODE_;
  static constexpr bool WS = WS_ != 0;
  static constexpr int NWE = WS ? COMMET_WS_NWE : 0, NTHR_ALL = 32 * (NW_ + NWE);
  // network inputs per qp: 3 (standard / isochoric invariants) or 5 (anisotropic: + I4, I5)
  // (KIN 2: one structural vector, 5 inputs; KIN 3: two vectors, 9 inputs -- App. A.2.1)
  // (KIN 4 / 5: the same on the isochoric inputs Ibar1, Ibar2, J, Ibar4,ij, Ibar5,ij -- App. A.2.2,
  //  compile-time so the plain anisotropic kernels carry none of the chain rule)
  static constexpr bool ISO_A = KIN >= 4;
  static constexpr int NSV = (KIN == 3 || KIN == 5) ? 2 : 1;
  static constexpr int NK = KIN >= 2 ? (NSV == 2 ? 9 : 5) : 3, NH = NK * (NK + 1) / 2;
  static constexpr int NP = NK + NH;  // adjoint-pass partials per qp: g (NK) and H_1 (NH)
  static constexpr int NWARP = NW_, NTHR = 32 * NW_;
  static constexpr int MINB = MINB_;               // CTAs per SM the register budget targets (3: <= 168 regs)
  static constexpr bool DMMA_ELEM = MODE == 0 && (COMMET_DMMA_ELEM == 2 || (COMMET_DMMA_ELEM == 1 && NEN == 8));
  static constexpr int E = Q / NQ;                 // elements per CTA iteration
  static constexpr int MTILES = W / 8, QB = Q / 8, KT2 = W / 8;
  // value / adjoint warp tiles: VMG x VNG warps, each MT_V x NT_V tiles
  static constexpr int TPW = MTILES * QB / NWARP;
  static constexpr int NT_V = (QB >= 2 && TPW % 2 == 0 && TPW >= 4) ? 2 : 1;
  static constexpr int MT_V = TPW / NT_V;
  static constexpr int VNG = QB / NT_V, VMG = MTILES / MT_V;
  // Jacobian warp tiles: JMG m-groups x QB qp blocks, each MT_J x 3 tiles
  static constexpr int JMG = NWARP / QB, MT_J = MTILES / JMG;
  // material mode: rows of per-qp partial sums of the network value a . z_L (value tiling: VMG
  // rows; forward sweep: JMG rows; L = 1: NTHR / Q rows)
  static constexpr int NPR0 = VMG > NTHR / Q ? VMG : NTHR / Q;
  static constexpr int NPR = MODE == 0 ? 0 : (JMG > NPR0 ? JMG : NPR0);
  // A-fragment register ring depth (k-steps) of the value/adjoint and Jacobian GEMMs
  static constexpr int PD_V = COMMET_PD_V, PD_J = COMMET_PD_J;
  // one forward sweep for the value and the Jacobian (3-input ICNN, L = 2 or 3): act
  // holds z | s (.) J (4 column groups per qp) and keeps s_2 (.) J_2 for the backward pass.
  // Measured (tools/ab_bench.py): round 1, w = 128 (c4) 41.10 -> 39.94 ms, w = 64 (c3) 10.29 ->
  // 10.64 ms; round 2 with the layer count a template parameter (unrolled, short live ranges)
  // and 1/s by rcp + Newton instead of an IEEE division: c3 10.34 -> 9.84 ms, c4 39.86 -> 37.85.
  static constexpr bool FWDC = COMMET_FWD && W >= COMMET_FWD_MINW && NET == 0 && NK == 3 && !COMMET_PINGPONG;
  // element batches: the element stages (0-1, 7-8) run on EB network batches at once -- QE qps,
  // EE elements -- while the network stages (2-6) run batch by batch (ICNN assembly, Q <= 16)
  // (tet10's scalar element stage keeps an X buffer of QE x NEN x 27 doubles in the dead network
  // buffers: two batches only where it still fits, Q = 8)
  static constexpr int EB = (NET == 0 && MODE == 0 && !WS && Q <= 16 && (NEN == 8 || Q <= 8)) ? COMMET_EB : 1;
  static constexpr int QE = EB * Q, EE = QE / NQ, NKH = NK + NH;
  static_assert(QE <= 32, "stage-1 threads (one per qp) must sit in warp 0");
  // activation table bits on the forward-sweep path (the 256-entry tables do not fit beside the
  // element buffers of two batches)
  static constexpr int TB_FWD = EB > 1 ? COMMET_ACT_TB_EB : COMMET_ACT_TB;
  static constexpr int LDA = (FWDC ? 4 : NK) * Q + 4;  // act row stride (= 4 mod 16: conflict-free B frags)
  static constexpr int LDS = Q + 2;                // s/c row stride (2-way conflicts at most)
  static_assert(W % 8 == 0 && Q % 8 == 0 && Q % NQ == 0, "tile");
  static_assert(Q <= 32, "stage-1 threads (one per qp) must sit in warp 0");
  static_assert(TPW >= 1 && VMG * VNG == NWARP && MT_V * NT_V == TPW, "value tiling");
  static_assert(JMG >= 1 && JMG * QB == NWARP && MT_J * JMG == MTILES, "jacobian tiling");
  // ping-pong of the value / adjoint passes between act column blocks [0, Q) and [Q, 2Q), the
  // adjoint-pass g/H_1 partials in rows 9 vm + x of the free block [2Q, 3Q) (needs VMG*9 <= W)
  static constexpr bool PP = COMMET_PINGPONG && NK == 3 && VMG * 9 <= W;
  static_assert(PP || VMG * Q * NP <= W * LDA, "adjoint partials must fit in act");
};

// shared-memory carve-up (doubles); L is a runtime value.  The post-NCM
// buffers (qP, post/X, qA) alias act/s/c, which are dead after stage 6.
template <class C>
struct Smem {
  // per-qp stride of the stage-7a outputs (odd: bank spread); anisotropic: 5 factor pairs
  static constexpr int PS = C::KIN >= 2 ? (C::NSV == 2 ? kPostAniso2 : kPostAniso) : 101;
  int act, sb, cb, qF, qk, qg, qH, hred, gsk, gN, ue, wq, qN, tab, qgH, qP, post, X, qA, total;
  // fwd: the forward-sweep path runs (C::FWDC, 2 <= L <= 3, no hidden skips): no c buffers
  __host__ __device__ static bool fwd_path(int L, bool skips) { return C::FWDC && L >= 2 && L <= 3 && !skips; }
  __host__ __device__ static bool fused_gh(int L, bool skips) { return COMMET_FUSE_GH && C::EB > 1 && fwd_path(L, skips); }
  __host__ __device__ Smem(int L, bool skips = false) {
    const bool fwd = fwd_path(L, skips);
    int o = 0;
    // the network buffers: ICNN only (the analytic networks run per qp in registers)
    const bool icnn = C::NET == 0;
    act = o; o += icnn ? C::W * C::LDA : 0;
    sb = o;  o += icnn ? (L > 1 ? L - 1 : 0) * C::W * C::LDS : 0;   // s_l, l = 1..L-1
    cb = o;  o += icnn && !fwd ? (L > 1 ? L - 1 : 1) * C::W * C::LDS : 0;   // c_l, l = 2..L (L == 1: c_1)
    const int dead = o;
    qF = o;  o += C::QE * 9;
    qk = o;  o += C::QE * C::NK;
    // (forward sweep with the two-batch element stage: (g, H) go straight to qgH and the hidden-skip
    // gradients are zero -- no qg / qH / gsk, which leaves room for the 256-entry activation tables)
    const bool fgh = fused_gh(L, skips);
    qg = o;  o += fgh ? 0 : C::Q * C::NK;
    qH = o;  o += fgh ? 0 : C::Q * C::NH;
    hred = o; o += (C::JMG + (C::FWDC ? C::VMG : 0)) * C::Q * C::NH;  // H partials per warp row group
    // (the adjoint-pass g/H_1 partials, VMG x Q x 9, live in act: dead at that point)
    gsk = o; o += fgh ? 0 : C::QE * C::NK;
    gN = o;  o += C::QE * C::NEN * 3;
    ue = o;  o += C::EE * C::NEN * 3;
    wq = o;  o += C::QE;
    qN = o;  o += C::NPR * C::Q;
    tab = o; o += fwd ? ActTab<C::TB_FWD>::SIZE : ActTab<6>::SIZE;
    qgH = o; o += C::EB > 1 ? C::QE * C::NKH : 0;  // (g, H) of each network batch for the element stage
    o = (o + 1) & ~1;
    const int xs = C::DMMA_ELEM ? 0 : C::QE * C::NEN * 27;  // X only for the scalar element path
    const int px = C::QE * PS > xs ? C::QE * PS : xs;
    const int need = C::QE * 9 + px + C::QE * 81;
    int base = 0;
    if (need > dead) { base = o; o += need; }
    qP = base;
    post = X = base + C::QE * 9;
    qA = post + px;
    total = o;
  }
};

// ---------------------------------------------------------------------------
// one warp tile of  C = A (M x K, fragments in global) * B (K x N, smem)
// ---------------------------------------------------------------------------
// A fragments stream from L2/L1 through a register ring of PD k-steps (PD - 1 in flight)
template <int MT, int NT, int KT2, int PD = 2>
__device__ __forceinline__ void warp_gemm(const double* __restrict__ Af, int mt0, const double* act,
                                          int lda, const int (&ncol)[NT], double (&acc)[MT][NT][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < MT; i++)
#pragma unroll
    for (int j = 0; j < NT; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  const double* ap = Af + (size_t)mt0 * KT2 * 64 + lane * 2;
  const double* bp = act + t * lda + g;
  double2 a[PD][MT];
#if COMMET_BPF
  double bn[NT];
#pragma unroll
  for (int j = 0; j < NT; j++) bn[j] = bp[ncol[j]];
#endif
#pragma unroll
  for (int p = 0; p < PD - 1 && p < KT2; p++)
#pragma unroll
    for (int i = 0; i < MT; i++) a[p][i] = ldg2(ap + ((size_t)i * KT2 + p) * 64);
#if COMMET_KUNROLL  // partial unroll (a multiple of PD: the ring indices stay static): smaller code
  COMMET_UNROLL(COMMET_KUNROLL)
#else
#pragma unroll
#endif
  for (int kt2 = 0; kt2 < KT2; kt2++) {
    const int cur = kt2 % PD;
    if (kt2 + PD - 1 < KT2) {
#pragma unroll
      for (int i = 0; i < MT; i++) a[(kt2 + PD - 1) % PD][i] = ldg2(ap + ((size_t)i * KT2 + kt2 + PD - 1) * 64);
    }
#if COMMET_BPF  // B fragments of the next half k-step loaded before this one's DMMAs
#pragma unroll
    for (int h = 0; h < 2; h++) {
      double b[NT];
#pragma unroll
      for (int j = 0; j < NT; j++) b[j] = bn[j];
      if (h == 0 || kt2 + 1 < KT2) {
        const double* bk = bp + (kt2 * 8 + h * 4 + 4) * lda;
#pragma unroll
        for (int j = 0; j < NT; j++) bn[j] = bk[ncol[j]];
      }
#pragma unroll
      for (int i = 0; i < MT; i++)
#pragma unroll
        for (int j = 0; j < NT; j++) dmma(acc[i][j], h ? a[cur][i].y : a[cur][i].x, b[j]);
    }
#else
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const double* bk = bp + (kt2 * 8 + h * 4) * lda;
      double b[NT];
#pragma unroll
      for (int j = 0; j < NT; j++) b[j] = bk[ncol[j]];
#pragma unroll
      for (int i = 0; i < MT; i++)
#pragma unroll
        for (int j = 0; j < NT; j++) dmma(acc[i][j], h ? a[cur][i].y : a[cur][i].x, b[j]);
    }
#endif
  }
}

// Material-point outputs of one batch (MODE 1): per point
// Psi = N + kappa (J-1)^2 - s0 (J-1), tau = F S F^T = P F^T and the spatial tangent
// c_ijkl = sum_JL A_iJkL F_jJ F_lL - d_ik tau_jl (App. A.1), Voigt
// order (00, 11, 22, 12, 02, 01); c as the 21 upper-triangle entries, row-major.
__constant__ int kVoigt[6][2] = {{0, 0}, {1, 1}, {2, 2}, {1, 2}, {0, 2}, {0, 1}};
__constant__ int kVoigtPair[21][2] = {{0, 0}, {0, 1}, {0, 2}, {0, 3}, {0, 4}, {0, 5}, {1, 1}, {1, 2}, {1, 3},
                                      {1, 4}, {1, 5}, {2, 2}, {2, 3}, {2, 4}, {2, 5}, {3, 3}, {3, 4}, {3, 5},
                                      {4, 4}, {4, 5}, {5, 5}};
// kVoigtPair -> (i, j, k, l), 2 bits each (i | j << 2 | k << 4 | l << 6), 8 entries per word
constexpr unsigned long long voigt_code_word(int w) {
  constexpr int V[6][2] = {{0, 0}, {1, 1}, {2, 2}, {1, 2}, {0, 2}, {0, 1}};
  unsigned long long c = 0;
  int vw = 0;
  for (int p = 0; p < 6; p++)
    for (int q = p; q < 6; q++, vw++)
      if (vw >> 3 == w)
        c |= (unsigned long long)(V[p][0] | V[p][1] << 2 | V[q][0] << 4 | V[q][1] << 6) << (8 * (vw & 7));
  return c;
}
constexpr unsigned long long kVoigtCode0 = voigt_code_word(0), kVoigtCode1 = voigt_code_word(1),
                             kVoigtCode2 = voigt_code_word(2);

template <class C>
__device__ __forceinline__ void material_outputs(const AsmArgs& A, const NcmDev& m, int L, int64_t e0, int ne,
                                                 const double* qF, const double* qk, const double* qg,
                                                 const double* qH, const double* hred, const double* qNp,
                                                 double* qP, double* post, double* qA) {
  constexpr int Q = C::Q, PS = Smem<C>::PS;
  const int tid = threadIdx.x;
  if (tid < Q) {
    const int q = tid;
    double gq[C::NK], H6[C::NH], N = 0.0;
    const double* kq = qk + q * C::NK;
    if constexpr (C::NET == 0) {
#pragma unroll
      for (int x = 0; x < C::NK; x++) gq[x] = qg[q * C::NK + x];
#pragma unroll
      for (int x = 0; x < C::NH; x++) {
        double s = qH[q * C::NH + x];
        if (L > 1)
#pragma unroll
          for (int r = 0; r < C::JMG; r++) s += hred[(r * Q + q) * C::NH + x];
        if constexpr (C::FWDC)
          if (Smem<C>::fwd_path(L, m.skip_h != nullptr) && L == 3)
#pragma unroll
            for (int r = 0; r < C::VMG; r++) s += hred[((C::JMG + r) * Q + q) * C::NH + x];
        H6[x] = s;
      }
      // partial sums of a . z_L: one row per value-tiling row group (forward sweep: per jm group)
      const int rows = L > 1 ? (C::FWDC && Smem<C>::fwd_path(L, m.skip_h != nullptr) ? C::JMG : C::VMG) : C::NTHR / Q;
      for (int r = 0; r < rows; r++) N += qNp[r * Q + q];
      N += __ldg(m.skip_out) * kq[0] + __ldg(m.skip_out + 1) * kq[1] + __ldg(m.skip_out + 2) * kq[2];
    } else {
      analytic_point<C::NK>(m, kq, gq, H6, &N);
    }
    Kin kin;
    kinematics(qF + q * 9, kin);
    if constexpr (C::KIN == 1) isochoric_to_standard(kin, gq, H6);
    if constexpr (C::KIN >= 2)
      if constexpr (C::ISO_A) isochoric_aniso_to_standard<C::NSV>(kin, m.a0, m.a1, gq, H6);
    const double jm1 = kin.J - 1.0;
    const double Wv = N + m.kappa * jm1 * jm1 - m.ref_shift * jm1;
    gq[2] += 2.0 * m.kappa * jm1 - m.ref_shift;
    H6[packed_index(C::NK, 2, 2)] += 2.0 * m.kappa;
    if constexpr (C::KIN >= 2)
      post_qp_aniso<C::NSV>(kin, m.a0, m.a1, gq, H6, 1.0, post + q * PS, qP + q * 9);
    else
      post_qp(kin, gq, H6, 1.0, post + q * PS, qP + q * 9);
    double tau[9];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int j = 0; j < 3; j++)
        tau[i * 3 + j] = qP[q * 9 + i * 3] * kin.F[j * 3] + qP[q * 9 + i * 3 + 1] * kin.F[j * 3 + 1] +
                         qP[q * 9 + i * 3 + 2] * kin.F[j * 3 + 2];
#pragma unroll
    for (int x = 0; x < 9; x++) qP[q * 9 + x] = tau[x];
    if (q < ne) {
      if (A.Wout) A.Wout[e0 + q] = Wv;
      if (A.tau_out)
#pragma unroll
        for (int v = 0; v < 6; v++) A.tau_out[(e0 + q) * 6 + v] = tau[kVoigt[v][0] * 3 + kVoigt[v][1]];
    }
  }
  __syncthreads();
  if (!A.c_out) return;
  for (int it = tid; it < Q * 9; it += C::NTHR) {
    const int q = it / 9, iJ = it % 9;
    if constexpr (C::KIN >= 2)
      tangent_row_aniso<C::NSV>(post + q * PS, iJ, qA + q * 81 + iJ * 9);
    else
      tangent_row(post + q * PS, iJ, qA + q * 81 + iJ * 9);
  }
  __syncthreads();
  for (int it = tid; it < Q * 21; it += C::NTHR) {
    const int q = it / 21, vw = it % 21;
    if (q >= ne) continue;
    // (i, j, k, l) of entry vw from a packed immediate (the per-thread index into the
    // __constant__ tables would serialise the constant cache)
    const unsigned long long cw = vw < 8 ? kVoigtCode0 : (vw < 16 ? kVoigtCode1 : kVoigtCode2);
    const unsigned code = (unsigned)(cw >> (8 * (vw & 7))) & 0xffu;
    const int i = code & 3, j = (code >> 2) & 3, k = (code >> 4) & 3, l = code >> 6;
    const double* F = qF + q * 9;
    const double* Aq = qA + q * 81;
    double c = (i == k) ? -qP[q * 9 + j * 3 + l] : 0.0;
#pragma unroll
    for (int J = 0; J < 3; J++)
#pragma unroll
      for (int Lx = 0; Lx < 3; Lx++) c += Aq[(i * 3 + J) * 9 + k * 3 + Lx] * F[j * 3 + J] * F[l * 3 + Lx];
    A.c_out[(e0 + q) * 21 + vw] = c;
  }
}


// ---------------------------------------------------------------------------
// Forward sweep (3-input ICNN, L = 2 or 3, no hidden skips): the value and the input Jacobian
// in one GEMM per layer -- y_l = W_l z_{l-1} and J_l = W_l (s_{l-1} (.) J_{l-1}) share their A
// operand -- so each hidden weight matrix is read once on the way forward.  The last layer's
// Hessian term is final at once (c_L = a s_L (1 - s_L)); the inner layer's (L = 3: layer 2)
// waits in act as s_2 (.) J_2 for lambda_2 from the backward pass:
//   c_2 J_2 J_2^T = lambda_2 (1 - s_2) / s_2 (s_2 J_2)(s_2 J_2)^T.
// The backward pass then gives g and H_1 as before (stage 4's l = 2 epilogue, stage 5).
// act: columns [0, Q) z_l / mu_l, [Q, 4Q) s_l (.) J_l; on entry z_1 | D_1 (stage 2).
// ---------------------------------------------------------------------------
// 1/x for x in [2^-500, 1]: MUFU seed (rcp.approx.ftz.f64, ~2^-23) + two Newton steps -- full
// precision, no IEEE-division slow path
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  return r * fma(-x, r, 2.0);
}

template <class C, int L>
__device__ __forceinline__ void fwd_sweep(const NcmDev& m, double* act, double* sb, double* hred, double* qg,
                                          double* qH, const double* gsk, const double* stab, double* qNp,
                                          double* qgH_h = nullptr) {
  constexpr int W = C::W, Q = C::Q, LDA = C::LDA, LDS = C::LDS, KT2 = C::KT2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const size_t frag_layer = (size_t)2 * W * W;
  // ---- forward: layers 2..L, warp tile = MT_J m-tiles x 4 column groups of one qp block ----
  {
    const int jm = warp / C::QB, qb = warp % C::QB;
    const int mt0 = jm * C::MT_J;
    int ncol[4];
#pragma unroll
    for (int c = 0; c < 4; c++) ncol[c] = c * Q + qb * 8;
    double hp[2][6], nacc[2] = {0.0, 0.0};  // nacc: material points, partial a . z_L
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
      for (int x = 0; x < 6; x++) hp[h][x] = 0.0;
#if COMMET_FWD_LOOP
#pragma unroll 1
#else
#pragma unroll
#endif
    for (int l = 2; l <= L; l++) {
      double acc[C::MT_J][4][2];
      warp_gemm<C::MT_J, 4, KT2, C::PD_J>(m.Wfrag + (l - 2) * frag_layer, mt0, act, LDA, ncol, acc);
      net_sync<C>();
#pragma unroll
      for (int i = 0; i < C::MT_J; i++) {
        const int j = (mt0 + i) * 8 + g;
        const double bj = __ldg(m.b + (l - 1) * W + j);
        const double aj = __ldg(m.a + j);
#if COMMET_VSTORE
        if (l < L) {  // both qps of the lane (q, q + 1: 16-byte aligned) with one vector store per row
          const int q = qb * 8 + 2 * t;
          double z[2], s[2];
#pragma unroll
          for (int h = 0; h < 2; h++) softplus_sig_t<C::TB_FWD>(acc[i][0][h] + bj, stab, z[h], s[h]);
          *reinterpret_cast<double2*>(sb + ((l - 1) * W + j) * LDS + q) = make_double2(s[0], s[1]);
          double* ar = act + j * LDA + q;
          *reinterpret_cast<double2*>(ar) = make_double2(z[0], z[1]);
#pragma unroll
          for (int c = 1; c < 4; c++)
            *reinterpret_cast<double2*>(ar + c * Q) = make_double2(s[0] * acc[i][c][0], s[1] * acc[i][c][1]);
          continue;
        }
#endif
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int q = qb * 8 + 2 * t + h;
          const double y = acc[i][0][h] + bj;
          const double J0 = acc[i][1][h], J1 = acc[i][2][h], J2 = acc[i][3][h];
          if (l < L) {
            double z, s;
            softplus_sig_t<C::TB_FWD>(y, stab, z, s);
            sb[((l - 1) * W + j) * LDS + q] = s;
            act[j * LDA + q] = z;
            act[j * LDA + Q + q] = s * J0;
            act[j * LDA + 2 * Q + q] = s * J1;
            act[j * LDA + 3 * Q + q] = s * J2;
          } else {  // last layer: mu_L = a s_L for the backward pass, c_L final
            double s;
            if constexpr (C::MODE == 1) {  // material points need the value: z_L too
              double z;
              softplus_sig_t<C::TB_FWD>(y, stab, z, s);
              nacc[h] += aj * z;
            } else {
              s = sigmoid_t<C::TB_FWD>(y, stab);
            }
            const double c = aj * s * (1.0 - s);
            const double c0 = c * J0, c1 = c * J1, c2 = c * J2;
            hp[h][0] += c0 * J0; hp[h][1] += c0 * J1; hp[h][2] += c0 * J2;
            hp[h][3] += c1 * J1; hp[h][4] += c1 * J2; hp[h][5] += c2 * J2;
            act[j * LDA + q] = aj * s;
          }
        }
      }
      net_sync<C>();
    }
    if constexpr (COMMET_RS) {
      double v[12], o[RS<12>::K3];
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int x = 0; x < 6; x++) v[h * 6 + x] = hp[h][x];
      reduce_scatter8<12>(v, o);
#pragma unroll
      for (int i = 0; i < RS<12>::K3; i++) {
        const int idx = rs_index<12>(g, i);
        if (idx >= 0) hred[(jm * Q + qb * 8 + 2 * t + idx / 6) * 6 + idx % 6] = o[i];
      }
    } else {
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
      for (int x = 0; x < 6; x++) {
        double v = hp[h][x];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        hp[h][x] = v;
      }
    if (g == 0) {
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int x = 0; x < 6; x++) hred[(jm * Q + qb * 8 + 2 * t + h) * 6 + x] = hp[h][x];
    }
    }
    if constexpr (C::MODE == 1) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        double v = nacc[h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (g == 0) qNp[jm * Q + qb * 8 + 2 * t + h] = v;
      }
    }
  }
  // ---- backward: mu_{l-1} = (W_l^T mu_l) (.) s_{l-1}; layer 1 -> g, H_1 partials -------------
  {
    const int vm = warp / C::VNG, vn = warp % C::VNG;
    const int mt0 = vm * C::MT_V;
    int ncol[C::NT_V];
#pragma unroll
    for (int j = 0; j < C::NT_V; j++) ncol[j] = (vn * C::NT_V + j) * 8;
#pragma unroll
    for (int l = L; l >= 2; l--) {
      double acc[C::MT_V][C::NT_V][2];
      warp_gemm<C::MT_V, C::NT_V, KT2, C::PD_V>(m.Wfrag + (l - 2) * frag_layer + (size_t)W * W, mt0, act, LDA, ncol,
                                               acc);
      net_sync<C>();
      if (l > 2) {  // l = 3: lambda_2 -> mu_2, and layer 2's Hessian term from s_2 (.) J_2
        double hb[C::NT_V][2][6];
#pragma unroll
        for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
          for (int h = 0; h < 2; h++)
#pragma unroll
            for (int x = 0; x < 6; x++) hb[jj][h][x] = 0.0;
#pragma unroll
        for (int i = 0; i < C::MT_V; i++) {
          const int j = (mt0 + i) * 8 + g;
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++) {
#if COMMET_VSTORE2  // the lane's two qps (q, q + 1) with 16-byte shared loads / stores
            const int q0 = ncol[jj] + 2 * t;
            const double2 s2 = *reinterpret_cast<const double2*>(sb + ((l - 2) * W + j) * LDS + q0);
            const double2 Pa = *reinterpret_cast<const double2*>(act + j * LDA + Q + q0);
            const double2 Pb = *reinterpret_cast<const double2*>(act + j * LDA + 2 * Q + q0);
            const double2 Pc = *reinterpret_cast<const double2*>(act + j * LDA + 3 * Q + q0);
            double mu[2];
#endif
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int q = ncol[jj] + 2 * t + h;
              const double lam = acc[i][jj][h];
#if COMMET_VSTORE2
              const double s = h ? s2.y : s2.x;
#else
              const double s = sb[((l - 2) * W + j) * LDS + q];
#endif
              // c_2 J_2 J_2^T = lam (1 - s)/s P P^T.  1/s of s clamped at 2^-500: finite for any lam
              // the weights can produce (a neuron with s < 2^-500 contributes < 1e-150 either way)
              const double k2 = lam * (1.0 - s) * rcp_nr(fmax(s, 0x1p-500));
#if COMMET_VSTORE2
              const double P0 = h ? Pa.y : Pa.x, P1 = h ? Pb.y : Pb.x, P2 = h ? Pc.y : Pc.x;
              (void)q;
#else
              const double P0 = act[j * LDA + Q + q], P1 = act[j * LDA + 2 * Q + q], P2 = act[j * LDA + 3 * Q + q];
#endif
              const double c0 = k2 * P0, c1 = k2 * P1, c2 = k2 * P2;
              double* hh = hb[jj][h];
              hh[0] += c0 * P0; hh[1] += c0 * P1; hh[2] += c0 * P2;
              hh[3] += c1 * P1; hh[4] += c1 * P2; hh[5] += c2 * P2;
#if COMMET_VSTORE2
              mu[h] = lam * s;
#else
              act[j * LDA + q] = lam * s;  // mu_2
#endif
            }
#if COMMET_VSTORE2
            *reinterpret_cast<double2*>(act + j * LDA + q0) = make_double2(mu[0], mu[1]);  // mu_2
#endif
          }
        }
        if constexpr (COMMET_RS) {
          constexpr int NV = C::NT_V * 12;
          double v[NV], o[RS<NV>::K3];
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++)
#pragma unroll
              for (int x = 0; x < 6; x++) v[(jj * 2 + h) * 6 + x] = hb[jj][h][x];
          reduce_scatter8<NV>(v, o);
#pragma unroll
          for (int i = 0; i < RS<NV>::K3; i++) {
            const int idx = rs_index<NV>(g, i);
            if (idx >= 0) {
              const int jh = idx / 6;
              hred[((C::JMG + vm) * Q + (vn * C::NT_V + jh / 2) * 8 + 2 * t + (jh & 1)) * 6 + idx % 6] = o[i];
            }
          }
        } else {
#pragma unroll
        for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
          for (int h = 0; h < 2; h++)
#pragma unroll
            for (int x = 0; x < 6; x++) {
              double v = hb[jj][h][x];
              v += __shfl_xor_sync(0xffffffffu, v, 4);
              v += __shfl_xor_sync(0xffffffffu, v, 8);
              v += __shfl_xor_sync(0xffffffffu, v, 16);
              hb[jj][h][x] = v;
            }
        if (g == 0) {
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++)
#pragma unroll
              for (int x = 0; x < 6; x++)
                hred[((C::JMG + vm) * Q + ncol[jj] + 2 * t + h) * 6 + x] = hb[jj][h][x];
        }
        }
      } else {  // l == 2: mu_1, c_1 -> partials of g = W1^T mu_1 and H_1 = W1^T diag(c_1) W1
        double pg[C::NT_V][2][9];
#pragma unroll
        for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
          for (int h = 0; h < 2; h++)
#pragma unroll
            for (int x = 0; x < 9; x++) pg[jj][h][x] = 0.0;
#pragma unroll
        for (int i = 0; i < C::MT_V; i++) {
          const int j = (mt0 + i) * 8 + g;
          const double w0 = __ldg(m.W1 + j * 3), w1 = __ldg(m.W1 + j * 3 + 1), w2 = __ldg(m.W1 + j * 3 + 2);
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int q = ncol[jj] + 2 * t + h;
              const double lam = acc[i][jj][h];
              const double s = sb[j * LDS + q];
              const double mu = lam * s, c = mu * (1.0 - s);
              double* P9 = pg[jj][h];
              P9[0] += w0 * mu; P9[1] += w1 * mu; P9[2] += w2 * mu;
              const double c0 = c * w0, c1 = c * w1;
              P9[3] += c0 * w0; P9[4] += c0 * w1; P9[5] += c0 * w2;
              P9[6] += c1 * w1; P9[7] += c1 * w2; P9[8] += c * w2 * w2;
            }
        }
        if constexpr (COMMET_RS) {  // act is dead now: partials at (vm, q)
          constexpr int NV = C::NT_V * 18;
          double v[NV], o[RS<NV>::K3];
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++)
#pragma unroll
              for (int x = 0; x < 9; x++) v[(jj * 2 + h) * 9 + x] = pg[jj][h][x];
          reduce_scatter8<NV>(v, o);
#pragma unroll
          for (int i = 0; i < RS<NV>::K3; i++) {
            const int idx = rs_index<NV>(g, i);
            if (idx >= 0) {
              const int jh = idx / 9;
              act[(vm * Q + (vn * C::NT_V + jh / 2) * 8 + 2 * t + (jh & 1)) * 9 + idx % 9] = o[i];
            }
          }
        } else {
#pragma unroll
        for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
          for (int h = 0; h < 2; h++)
#pragma unroll
            for (int x = 0; x < 9; x++) {
              double v = pg[jj][h][x];
              v += __shfl_xor_sync(0xffffffffu, v, 4);
              v += __shfl_xor_sync(0xffffffffu, v, 8);
              v += __shfl_xor_sync(0xffffffffu, v, 16);
              pg[jj][h][x] = v;
            }
        if (g == 0) {  // act is dead now: partials at (vm, q)
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++)
#pragma unroll
              for (int x = 0; x < 9; x++) act[(vm * Q + ncol[jj] + 2 * t + h) * 9 + x] = pg[jj][h][x];
        }
        }
      }
      net_sync<C>();
    }
  }
  // ---- g = W1^T mu_1 + skip_out, H_1 -----------------------------------------------------
  if (tid < Q) {
    const int q = tid;
    double v[9];
#pragma unroll
    for (int x = 0; x < 9; x++) v[x] = 0.0;
#pragma unroll
    for (int r = 0; r < C::VMG; r++)
#pragma unroll
      for (int x = 0; x < 9; x++) v[x] += act[(r * Q + q) * 9 + x];
    if (qgH_h) {  // two-batch element stage: (g, H) of this network batch straight into qgH, the
                  // row-group partials of hred added in the order of the separate copy (no hidden
                  // skips on this path: gsk = 0)
      double* o = qgH_h + q * C::NKH;
#pragma unroll
      for (int x = 0; x < 3; x++) o[x] = v[x] + 0.0 + __ldg(m.skip_out + x);
#pragma unroll
      for (int x = 0; x < 6; x++) {
        double hv = v[3 + x];
#pragma unroll
        for (int r = 0; r < C::JMG; r++) hv += hred[(r * Q + q) * 6 + x];
        if (L == 3)
#pragma unroll
          for (int r = 0; r < C::VMG; r++) hv += hred[((C::JMG + r) * Q + q) * 6 + x];
        o[3 + x] = hv;
      }
    } else {
#pragma unroll
      for (int x = 0; x < 3; x++) qg[q * 3 + x] = v[x] + gsk[q * 3 + x] + __ldg(m.skip_out + x);
#pragma unroll
      for (int x = 0; x < 6; x++) qH[q * 6 + x] = v[3 + x];
    }
  }
  if (!qgH_h) net_sync<C>();  // (fused: the caller's barrier after the batch orders qgH and act)
}

// ---- stage 2: layer 1 (3 -> W), elementwise.  Each thread: one qp, neurons j0, j0 + NTHR/Q, ...
// -- all loads issued up front and the NIT activations interleaved (independent chains).
// TB: activation table bits (8 on the forward-sweep path, 6 otherwise)
template <class C, int TB>
__device__ __forceinline__ void layer1(const NcmDev& m, int L, bool fwd, const double* qk, double* act, double* sb,
                                   double* cb, double* qNp, const double* stab) {
  constexpr int W = C::W, Q = C::Q, LDA = C::LDA, LDS = C::LDS;
  const int tid = threadIdx.x;
  constexpr int NIT = W * Q / C::NTHR, JS = C::NTHR / Q;
  static_assert(W * Q % C::NTHR == 0 && C::NTHR % Q == 0, "layer-1 split");
  const int q = tid % Q, j0 = tid / Q;
  double kq[C::NK];
#pragma unroll
  for (int x = 0; x < C::NK; x++) kq[x] = qk[q * C::NK + x];
  double yv[NIT];
#pragma unroll
  for (int i = 0; i < NIT; i++) {
    const int j = j0 + i * JS;
    double y = __ldg(m.b + j);
#pragma unroll
    for (int x = 0; x < C::NK; x++) y += __ldg(m.W1 + j * C::NK + x) * kq[x];
    yv[i] = y;
  }
  double nv = 0.0;  // material mode, L == 1: partial a . z_1 of this thread's neurons
#pragma unroll
  for (int i = 0; i < NIT; i++) {
    const int j = j0 + i * JS;
    double z, s;
    softplus_sig_t<TB>(yv[i], stab, z, s);
    if (L > 1) {
      sb[j * LDS + q] = s;
      act[j * LDA + q] = z;
      if constexpr (C::FWDC)
        if (fwd) {  // D_1 = s_1 (.) W1: the Jacobian columns of the forward sweep
#pragma unroll
          for (int c = 0; c < 3; c++) act[j * LDA + (c + 1) * Q + q] = s * __ldg(m.W1 + j * 3 + c);
        }
    } else {
      const double aj = __ldg(m.a + j);
      act[j * LDA + q] = aj * s;
      cb[j * LDS + q] = aj * s * (1.0 - s);
      nv += aj * z;
    }
  }
  if constexpr (C::MODE == 1)
    if (L == 1) qNp[j0 * Q + q] = nv;
}

template <class C>
__global__ void __launch_bounds__(C::NTHR, C::MINB) fused_kernel(AsmArgs A) {
  constexpr int W = C::W, Q = C::Q, NEN = C::NEN, NQ = C::NQ;
  // element-level sizes (stages 0-1, 7-8: EB network batches at once); the network stages use Q
  constexpr int QE = C::QE, EE = C::EE;
  constexpr int LDA = C::LDA, LDS = C::LDS, KT2 = C::KT2;
  extern __shared__ __align__(16) double smem[];
  const int L = A.ncm.L;
  const Smem<C> sm(L, A.ncm.skip_h != nullptr);
  double* act = smem + sm.act;
  double* sb = smem + sm.sb;
  double* cb = smem + sm.cb;
  double* qF = smem + sm.qF;
  double* qk = smem + sm.qk;
  double* qg = smem + sm.qg;
  double* qH = smem + sm.qH;
  double* hred = smem + sm.hred;
  double* gsk = smem + sm.gsk;
  double* sgN = smem + sm.gN;
  double* sue = smem + sm.ue;
  double* swq = smem + sm.wq;
  double* qNp = smem + sm.qN;
  double* stab = smem + sm.tab;
  double* qgH = smem + sm.qgH;
  double* qA = smem + sm.qA;
  double* qP = smem + sm.qP;
  double* post = smem + sm.post;
  double* Xb = smem + sm.X;
  constexpr int PS = Smem<C>::PS;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const NcmDev& m = A.ncm;
  const bool skips = m.skip_h != nullptr;
  const bool fwd = Smem<C>::fwd_path(L, skips);
  const bool fgh = Smem<C>::fused_gh(L, skips);  // forward sweep, two-batch element stage: (g, H) into qgH
  const int64_t n_batches = (A.el_count + EE - 1) / EE;
  const size_t frag_layer = (size_t)2 * W * W;  // W and W^T fragments per hidden layer
  {  // the activation table of this path (256 entries on the forward sweep, 64 otherwise)
    const int tb0 = fwd ? act_tab_offset<C::TB_FWD>() : 0, tbn = fwd ? ActTab<C::TB_FWD>::SIZE : ActTab<6>::SIZE;
    for (int x = threadIdx.x; x < tbn; x += C::NTHR) stab[x] = __ldg(A.ncm.act_tab + tb0 + x);
  }
  // (made visible by the first __syncthreads of the batch loop)
#ifdef COMMET_STAGE_PROF
  __shared__ long long st_acc[16];  // thread 0 only; [15] = previous mark
  if (tid == 0) {
    for (int i = 0; i < 15; i++) st_acc[i] = 0;
    st_acc[15] = clock64();
  }
#endif

  double trc_max = 0.0;  // running max of tr C = I1 over this thread's qps (stage 1 threads)
#if COMMET_PREFETCH
  // register prefetch of one batch's element inputs: (a) dN/dX, w, conn; (b) the u gather
  constexpr int NG2 = EE * NQ * NEN * 3 / 2, NU = EE * NEN * 3;
  constexpr int PG = (NG2 + C::NTHR - 1) / C::NTHR, PU = (NU + C::NTHR - 1) / C::NTHR;
  double2 pf_g[PG];
  double pf_u[PU], pf_w = 0.0;
  int pf_c[PU];

  auto pf_load_a = [&](int64_t b) {
    const int64_t f0 = A.el_begin + b * EE;
    const int64_t frem = A.el_begin + A.el_count - f0;
    const int fne = frem < EE ? (int)frem : EE;
    const double2* src = reinterpret_cast<const double2*>(A.gradN + (size_t)f0 * NQ * NEN * 3);
    const int n2 = fne * NQ * NEN * 3 / 2;
#pragma unroll
    for (int i = 0; i < PG; i++) {
      const int x = tid + i * C::NTHR;
      pf_g[i] = x < n2 ? ld_stream(src + x) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int i = 0; i < PU; i++) {
      const int x = tid + i * C::NTHR;
      const int e = x / (NEN * 3), ai = x % (NEN * 3);
      pf_c[i] = (x < NU && e < fne) ? ld_stream(A.conn + (f0 + e) * NEN + ai / 3) : -1;  // raw: no use here
    }
    if (tid < QE) pf_w = tid < fne * NQ ? ld_stream(A.qp_w + f0 * NQ + tid) : 0.0;
  };
  auto pf_load_b = [&]() {
#pragma unroll
    for (int i = 0; i < PU; i++)
      pf_u[i] = pf_c[i] >= 0 ? ld_stream(A.u + 3 * (int64_t)pf_c[i] + (tid + i * C::NTHR) % 3) : 0.0;
  };
  auto pf_store = [&]() {
    double2* dst = reinterpret_cast<double2*>(sgN);
#pragma unroll
    for (int i = 0; i < PG; i++) {
      const int x = tid + i * C::NTHR;
      if (x < NG2) dst[x] = pf_g[i];
    }
#pragma unroll
    for (int i = 0; i < PU; i++) {
      const int x = tid + i * C::NTHR;
      if (x < NU) sue[x] = pf_u[i];
    }
    if (tid < QE) swq[tid] = pf_w;
  };
#endif

  // adjoint-pass g/H_1 partial (row group r, qp q, entry x): with ping-pong in the block
  // [2Q, 3Q) of act, free during the value and adjoint passes; otherwise packed at the start
  auto part_at = [&](int r, int q, int x) {
    return C::PP ? (r * 9 + x) * LDA + 2 * Q + q : (r * Q + q) * C::NP + x;
  };

  for (int64_t batch = blockIdx.x; batch < n_batches; batch += gridDim.x) {
    const int64_t e0 = A.el_begin + batch * EE;
    const int64_t rem = A.el_begin + A.el_count - e0;
    const int ne = rem < EE ? (int)rem : EE;
    int cur = 0;  // act column block holding the current layer's input (value / adjoint passes)
#ifdef COMMET_DEBUG_CHECKS
    // race / stale-read check (debug builds, tools/race_check.py): every shared buffer except the
    // activation tables is poisoned with NaN before each batch, so a read that is not ordered after
    // this batch's write of the same word (a missing barrier, a wrong alias) returns NaN instead of
    // a plausible stale value and shows in the outputs
    {
      const int t0 = sm.tab, t1 = sm.tab + (fwd ? ActTab<C::TB_FWD>::SIZE : ActTab<6>::SIZE);
      __syncthreads();
      for (int x = tid; x < sm.total; x += C::NTHR)
        if (x < t0 || x >= t1) smem[x] = __longlong_as_double(0x7ff8deaddeadbeefLL);
      __syncthreads();
    }
#endif

    // ---- stage 0: stage element inputs --------------------------------------------
    if constexpr (C::MODE == 1) {  // material points: F rows (tail points get F = I)
      for (int x = tid; x < Q * 9; x += C::NTHR)
        qF[x] = x / 9 < ne ? __ldg(A.Fin + e0 * 9 + x) : ((x % 9) % 4 == 0 ? 1.0 : 0.0);
    } else {
#if COMMET_PREFETCH
    // the first batch loads here; later batches were loaded into registers during the
    // previous batch's element stage (pf_*), so only the shared-memory stores remain
    if (batch == blockIdx.x) {
      pf_load_a(batch);
      pf_load_b();
    }
    pf_store();
#else
    {
      const double2* src = reinterpret_cast<const double2*>(A.gradN + (size_t)e0 * NQ * NEN * 3);
      double2* dst = reinterpret_cast<double2*>(sgN);
      const int n2 = ne * NQ * NEN * 3 / 2;
      for (int x = tid; x < EE * NQ * NEN * 3 / 2; x += C::NTHR)
        dst[x] = x < n2 ? __ldg(src + x) : make_double2(0.0, 0.0);
      for (int x = tid; x < EE * NEN * 3; x += C::NTHR) {
        const int e = x / (NEN * 3), ai = x % (NEN * 3);
        sue[x] = e < ne ? ld_stream(A.u + 3 * (int64_t)ld_stream(A.conn + (e0 + e) * NEN + ai / 3) + ai % 3) : 0.0;
      }
      for (int x = tid; x < QE; x += C::NTHR) swq[x] = x < ne * NQ ? ld_stream(A.qp_w + e0 * NQ + x) : 0.0;
    }
#endif
    }  // MODE
    __syncthreads();
    STAGE_MARK(0)

    // ---- stage 1: kinematics ------------------------------------------------------
    if (tid < QE) {
      const int q = tid, e = q / NQ;
      const double* gq = sgN + q * NEN * 3;
      const double* ue = sue + e * NEN * 3;
      double F[9];
      if constexpr (C::MODE == 1) {
#pragma unroll
        for (int x = 0; x < 9; x++) F[x] = qF[q * 9 + x];
      } else {
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int J = 0; J < 3; J++) {
            double s = (i == J) ? 1.0 : 0.0;
#pragma unroll
            for (int a = 0; a < NEN; a++) s += ue[a * 3 + i] * gq[a * 3 + J];
            F[i * 3 + J] = s;
          }
      }
      Kin kin;
      kinematics(F, kin);
      if (e < ne) {
        if (!(kin.J > 0.0))
          atomicMin(A.bad, C::MODE == 1 ? (unsigned long long)(e0 + q)
                                        : (unsigned long long)(__ldg(A.orig + e0 + e) * NQ + q % NQ));
        trc_max = fmax(trc_max, kin.I1);  // one atomic per CTA at the end (a per-qp atomic on one
                                          // address serialises in L2: measured -6% on c3)
      }
#pragma unroll
      for (int x = 0; x < 9; x++) qF[q * 9 + x] = F[x];
      if constexpr (C::KIN >= 2) {  // anisotropic inputs (+ I4,ij, I5,ij per vector pair)
        double kb[C::NK];
        anisotropic_inputs<C::NSV>(kin, m.a0, m.a1, kb, C::ISO_A);
#pragma unroll
        for (int x = 0; x < C::NK; x++) qk[q * C::NK + x] = kb[x];
      } else if constexpr (C::KIN == 1) {  // isochoric inputs (App. A.2.2)
        double kb[3];
        isochoric_inputs(kin, kb);
        qk[q * 3 + 0] = kb[0];
        qk[q * 3 + 1] = kb[1];
        qk[q * 3 + 2] = kb[2];
      } else {
        qk[q * 3 + 0] = kin.I1 - 3.0;
        qk[q * 3 + 1] = kin.I2 - 3.0;
        qk[q * 3 + 2] = kin.J - 1.0;
      }
      if (!fgh)
#pragma unroll
        for (int x = 0; x < C::NK; x++) gsk[q * C::NK + x] = 0.0;
    }
#if !defined(COMMET_DEBUG_DROP) || COMMET_DEBUG_DROP != 2  // (planted race: tools/race_check.py)
    __syncthreads();
#endif
    STAGE_MARK(1)

    // ---- stages 2-6, once per network batch of Q qps (EB of them per element batch) ----------
    double* const qk_all = qk;
    double* const gsk_all = gsk;
    for (int h = 0; h < C::EB; h++) {
    double* qk = qk_all + h * Q * C::NK;    // this network batch's inputs and skip gradients
    double* gsk = gsk_all + h * Q * C::NK;
    (void)qk; (void)gsk;
#ifdef COMMET_EXP_SKIP_NCM
    if (false) {
#endif
    if constexpr (C::NET == 0) {
    // ---- stage 2: layer 1 (3 -> W), elementwise -------------------------------------
    if (L > 1) frag_prefetch<C::MT_V, KT2, COMMET_FRAG_PF + (COMMET_FRAG_PF == 0)>(m.Wfrag, (warp / C::VNG) * C::MT_V);
    if (C::FWDC && fwd) layer1<C, C::TB_FWD>(m, L, true, qk, act, sb, cb, qNp, stab);
    else layer1<C, 6>(m, L, false, qk, act, sb, cb, qNp, stab);
    __syncthreads();
    STAGE_MARK(2)

    if constexpr (C::FWDC) {
      if (fwd) {
        double* const gh = fgh ? qgH + h * Q * C::NKH : nullptr;
        if (L == 3) fwd_sweep<C, 3>(m, act, sb, hred, qg, qH, gsk, stab, qNp, gh);
        else fwd_sweep<C, 2>(m, act, sb, hred, qg, qH, gsk, stab, qNp, gh);
      }
    }
    if (!fwd) {
    // ---- stage 3: value pass, layers 2..L --------------------------------------------
    {
      const int vm = warp / C::VNG, vn = warp % C::VNG;
      const int mt0 = vm * C::MT_V;
      int ncol[C::NT_V];
#pragma unroll
      for (int j = 0; j < C::NT_V; j++) ncol[j] = (vn * C::NT_V + j) * 8;
      double nacc[C::NT_V][2];  // material mode: partial a . z_L per owned qp column
#pragma unroll
      for (int jj = 0; jj < C::NT_V; jj++) nacc[jj][0] = nacc[jj][1] = 0.0;
      for (int l = 2; l <= L; l++) {
        // ping-pong between act column blocks [0, Q) and [Q, 2Q): layer l reads block cur and
        // writes block cur ^ 1, so one barrier per layer suffices (the write of a fast warp
        // cannot hit the block a slow warp is still reading)
        double acc[C::MT_V][C::NT_V][2];
        int ncr[C::NT_V];
#pragma unroll
        for (int j = 0; j < C::NT_V; j++) ncr[j] = ncol[j] + cur * Q;
        warp_gemm<C::MT_V, C::NT_V, KT2, C::PD_V>(m.Wfrag + (l - 2) * frag_layer, mt0, act, LDA, ncr, acc);
        if constexpr (!C::PP) __syncthreads();
        const int wof = C::PP ? (cur ^ 1) * Q : 0;  // write block
        frag_prefetch<C::MT_V, KT2, COMMET_FRAG_PF + (COMMET_FRAG_PF == 0)>(
            m.Wfrag + (l < L ? (l - 1) * frag_layer : (L - 2) * frag_layer + (size_t)W * W), mt0);
#pragma unroll
        for (int i = 0; i < C::MT_V; i++) {
          const int j = (mt0 + i) * 8 + g;
          const double bj = __ldg(m.b + (l - 1) * W + j);
          double B3[3] = {0, 0, 0};
          if (skips) {
            const double* Bl = m.skip_h + ((size_t)(l - 2) * W + j) * 3;
            B3[0] = __ldg(Bl); B3[1] = __ldg(Bl + 1); B3[2] = __ldg(Bl + 2);
          }
          const double aj = (l == L) ? __ldg(m.a + j) : 0.0;
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int q = ncol[jj] + 2 * t + h;
              double y = acc[i][jj][h] + bj;
              if (skips) y += B3[0] * qk[q * C::NK] + B3[1] * qk[q * C::NK + 1] + B3[2] * qk[q * C::NK + 2];
              if constexpr (C::MODE == 1) {  // material points need the value: z_L too
                if (l == L) {
                  double z, s;
                  softplus_sig(y, stab, z, s);
                  act[j * LDA + wof + q] = aj * s;
                  cb[((l - 2) * W + j) * LDS + q] = aj * s * (1.0 - s);
                  nacc[jj][h] += aj * z;
                  continue;
                }
              }
              if (l < L) {
                double z, s;
                softplus_sig(y, stab, z, s);
                sb[((l - 1) * W + j) * LDS + q] = s;
                act[j * LDA + wof + q] = z;
              } else {  // z_L is not needed (only dN/dz_L = a): no log
                const double s = sigmoid_tab(y, stab);
                act[j * LDA + wof + q] = aj * s;                             // mu_L
                cb[((l - 2) * W + j) * LDS + q] = aj * s * (1.0 - s);        // c_L
              }
            }
        }
        __syncthreads();
        if constexpr (C::PP) cur ^= 1;
      }
      if constexpr (C::MODE == 1) {
        if (L > 1) {  // reduce the 8 row groups g of the warp, one partial per (vm, q)
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              double v = nacc[jj][h];
              v += __shfl_xor_sync(0xffffffffu, v, 4);
              v += __shfl_xor_sync(0xffffffffu, v, 8);
              v += __shfl_xor_sync(0xffffffffu, v, 16);
              if (g == 0) qNp[vm * Q + ncol[jj] + 2 * t + h] = v;
            }
        }
      }
    }

    STAGE_MARK(3)
    // ---- stage 4: adjoint pass, layers L..2 --------------------------------------------
    {
      const int vm = warp / C::VNG, vn = warp % C::VNG;
      const int mt0 = vm * C::MT_V;
      int ncol[C::NT_V];
#pragma unroll
      for (int j = 0; j < C::NT_V; j++) ncol[j] = (vn * C::NT_V + j) * 8;
      for (int l = L; l >= 2; l--) {
        if (skips && tid < Q) {  // g += B_l^T mu_l
          const double* Bl = m.skip_h + (size_t)(l - 2) * W * 3;
          double s0 = 0, s1 = 0, s2 = 0;
          for (int j = 0; j < W; j++) {
            const double mu = act[j * LDA + cur * Q + tid];
            s0 += __ldg(Bl + j * 3) * mu; s1 += __ldg(Bl + j * 3 + 1) * mu; s2 += __ldg(Bl + j * 3 + 2) * mu;
          }
          gsk[tid * C::NK] += s0; gsk[tid * C::NK + 1] += s1; gsk[tid * C::NK + 2] += s2;
        }
        double acc[C::MT_V][C::NT_V][2];
        int ncr[C::NT_V];
#pragma unroll
        for (int j = 0; j < C::NT_V; j++) ncr[j] = ncol[j] + cur * Q;
        warp_gemm<C::MT_V, C::NT_V, KT2, C::PD_V>(m.Wfrag + (l - 2) * frag_layer + (size_t)W * W, mt0, act, LDA,
                                                 ncr, acc);
        if constexpr (!C::PP) __syncthreads();
        const int wof = C::PP ? (cur ^ 1) * Q : 0;  // write block
        if (l > 2)
          frag_prefetch<C::MT_V, KT2, COMMET_FRAG_PF + (COMMET_FRAG_PF == 0)>(
              m.Wfrag + (l - 3) * frag_layer + (size_t)W * W, mt0);
        else
          frag_prefetch<C::MT_J, KT2, (COMMET_FRAG_PF + 1) / 2>(m.Wfrag, (warp / C::QB) * C::MT_J);
        if (l > 2) {
#pragma unroll
          for (int i = 0; i < C::MT_V; i++) {
            const int j = (mt0 + i) * 8 + g;
#pragma unroll
            for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
              for (int h = 0; h < 2; h++) {
                const int q = ncol[jj] + 2 * t + h;
                const double lam = acc[i][jj][h];
                const double s = sb[((l - 2) * W + j) * LDS + q];
                cb[((l - 3) * W + j) * LDS + q] = lam * s * (1.0 - s);  // c_{l-1}
                act[j * LDA + wof + q] = lam * s;                        // mu_{l-1}
              }
          }
        } else {
          // l == 2: lambda_1 -> mu_1, c_1 consumed here: g = W1^T mu_1, H_1 = W1^T diag(c_1) W1,
          // partial over this thread's rows, reduced over the warp's row groups g
          constexpr int NK = C::NK, NP = C::NP;
          double pg[C::NT_V][2][NP];
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++)
#pragma unroll
              for (int x = 0; x < NP; x++) pg[jj][h][x] = 0.0;
#pragma unroll
          for (int i = 0; i < C::MT_V; i++) {
            const int j = (mt0 + i) * 8 + g;
            double wv[NK];
#pragma unroll
            for (int x = 0; x < NK; x++) wv[x] = __ldg(m.W1 + j * NK + x);
#pragma unroll
            for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
              for (int h = 0; h < 2; h++) {
                const int q = ncol[jj] + 2 * t + h;
                const double lam = acc[i][jj][h];
                const double s = sb[j * LDS + q];
                const double mu = lam * s, c = mu * (1.0 - s);
                double* P9 = pg[jj][h];
                if constexpr (NK == 3) {  // (the generic form below costs ~1 % on c3: kept explicit)
                  const double w0 = wv[0], w1 = wv[1], w2 = wv[2];
                  P9[0] += w0 * mu; P9[1] += w1 * mu; P9[2] += w2 * mu;
                  const double c0 = c * w0, c1 = c * w1;
                  P9[3] += c0 * w0; P9[4] += c0 * w1; P9[5] += c0 * w2;
                  P9[6] += c1 * w1; P9[7] += c1 * w2; P9[8] += c * w2 * w2;
                } else {
#pragma unroll
                  for (int x = 0; x < NK; x++) P9[x] += wv[x] * mu;
                  int o = NK;
#pragma unroll
                  for (int a1 = 0; a1 < NK; a1++) {
                    const double ca = c * wv[a1];
#pragma unroll
                    for (int a2 = a1; a2 < NK; a2++) P9[o++] += ca * wv[a2];
                  }
                }
              }
          }
          if constexpr (COMMET_RS && NK == 3) {
            constexpr int NV = C::NT_V * 2 * NP;
            double v[NV], o[RS<NV>::K3];
#pragma unroll
            for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
              for (int h = 0; h < 2; h++)
#pragma unroll
                for (int x = 0; x < NP; x++) v[(jj * 2 + h) * NP + x] = pg[jj][h][x];
            reduce_scatter8<NV>(v, o);
#pragma unroll
            for (int i = 0; i < RS<NV>::K3; i++) {
              const int idx = rs_index<NV>(g, i);
              if (idx >= 0) {
                const int jh = idx / NP;
                act[part_at(vm, ncol[0] + (jh / 2) * 8 + 2 * t + (jh & 1), idx % NP)] = o[i];
              }
            }
          } else {
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++)
#pragma unroll
              for (int x = 0; x < NP; x++) {
                double v = pg[jj][h][x];
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                pg[jj][h][x] = v;
              }
          if (g == 0) {
#pragma unroll
            for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
              for (int h = 0; h < 2; h++)
#pragma unroll
                for (int x = 0; x < C::NP; x++) act[part_at(vm, ncol[jj] + 2 * t + h, x)] = pg[jj][h][x];
          }
          }
        }
        __syncthreads();
        if constexpr (C::PP) cur ^= 1;
      }
    }

    STAGE_MARK(4)
    // ---- stage 5: g = W1^T mu_1 + skips, H_1 = sum_j c1_j W1_j W1_j^T ------------------
    if (L > 1) {
      if (tid < Q) {
        const int q = tid;
        double v[C::NP];
#pragma unroll
        for (int x = 0; x < C::NP; x++) v[x] = 0.0;
#pragma unroll
        for (int r = 0; r < C::VMG; r++)
#pragma unroll
          for (int x = 0; x < C::NP; x++) v[x] += act[part_at(r, q, x)];
#pragma unroll
        for (int x = 0; x < C::NK; x++)
          qg[q * C::NK + x] = v[x] + gsk[q * C::NK + x] + (x < 3 ? __ldg(m.skip_out + x) : 0.0);
#pragma unroll
        for (int x = 0; x < C::NH; x++) qH[q * C::NH + x] = v[C::NK + x];
      }
    } else {
      constexpr int P = C::NTHR / Q;  // threads per qp (lanes q*P .. q*P+P-1 share a warp)
      const int q = tid / P, part = tid % P;
      double gs[C::NK], hs[C::NH];
#pragma unroll
      for (int x = 0; x < C::NK; x++) gs[x] = 0.0;
#pragma unroll
      for (int x = 0; x < C::NH; x++) hs[x] = 0.0;
      for (int j = part; j < W; j += P) {
        if constexpr (C::NK == 3) {
          const double w0 = __ldg(m.W1 + j * 3), w1 = __ldg(m.W1 + j * 3 + 1), w2 = __ldg(m.W1 + j * 3 + 2);
          const double mu = act[j * LDA + q], c = cb[j * LDS + q];
          gs[0] += w0 * mu; gs[1] += w1 * mu; gs[2] += w2 * mu;
          hs[0] += c * w0 * w0; hs[1] += c * w0 * w1; hs[2] += c * w0 * w2;
          hs[3] += c * w1 * w1; hs[4] += c * w1 * w2; hs[5] += c * w2 * w2;
        } else {
          double wv[C::NK];
#pragma unroll
          for (int x = 0; x < C::NK; x++) wv[x] = __ldg(m.W1 + j * C::NK + x);
          const double mu = act[j * LDA + q], c = cb[j * LDS + q];
#pragma unroll
          for (int x = 0; x < C::NK; x++) gs[x] += wv[x] * mu;
          int o = 0;
#pragma unroll
          for (int a1 = 0; a1 < C::NK; a1++)
#pragma unroll
            for (int a2 = a1; a2 < C::NK; a2++) hs[o++] += c * wv[a1] * wv[a2];
        }
      }
#pragma unroll
      for (int o = 1; o < P; o <<= 1) {
#pragma unroll
        for (int x = 0; x < C::NK; x++) gs[x] += __shfl_xor_sync(0xffffffffu, gs[x], o);
#pragma unroll
        for (int x = 0; x < C::NH; x++) hs[x] += __shfl_xor_sync(0xffffffffu, hs[x], o);
      }
      if (part == 0) {
#pragma unroll
        for (int x = 0; x < C::NK; x++)
          qg[q * C::NK + x] = gs[x] + gsk[q * C::NK + x] + (x < 3 ? __ldg(m.skip_out + x) : 0.0);
#pragma unroll
        for (int x = 0; x < C::NH; x++) qH[q * C::NH + x] = hs[x];
      }
    }
    __syncthreads();

    STAGE_MARK(5)
    // ---- stage 6: Jacobian pass, H += J_l^T diag(c_l) J_l -------------------------------
    if (L > 1) {
      {  // D_1 = s_1 (.) W1: one qp per thread, weights loaded up front
        constexpr int NIT = W * Q / C::NTHR, JS = C::NTHR / Q;
        const int q = tid % Q, j0 = tid / Q;
        double w1v[NIT][C::NK];
#pragma unroll
        for (int i = 0; i < NIT; i++)
#pragma unroll
          for (int c = 0; c < C::NK; c++) w1v[i][c] = __ldg(m.W1 + (j0 + i * JS) * C::NK + c);
#pragma unroll
        for (int i = 0; i < NIT; i++) {
          const int j = j0 + i * JS;
          const double s = sb[j * LDS + q];
#pragma unroll
          for (int c = 0; c < C::NK; c++) act[j * LDA + c * Q + q] = s * w1v[i][c];
        }
      }
      __syncthreads();
      const int jm = warp / C::QB, qb = warp % C::QB;
      const int mt0 = jm * C::MT_J;
      constexpr int NK = C::NK, NH = C::NH;
      int ncol[NK];
#pragma unroll
      for (int c = 0; c < NK; c++) ncol[c] = c * Q + qb * 8;
      double hp[2][NH];
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int x = 0; x < NH; x++) hp[h][x] = 0.0;
      for (int l = 2; l <= L; l++) {
        double acc[C::MT_J][NK][2];
        warp_gemm<C::MT_J, NK, KT2, C::PD_J>(m.Wfrag + (l - 2) * frag_layer, mt0, act, LDA, ncol, acc);
        __syncthreads();
        if (l < L) frag_prefetch<C::MT_J, KT2, (COMMET_FRAG_PF + 1) / 2>(m.Wfrag + (l - 1) * frag_layer, mt0);
#pragma unroll
        for (int i = 0; i < C::MT_J; i++) {
          const int j = (mt0 + i) * 8 + g;
          double B3[NK];
#pragma unroll
          for (int x = 0; x < NK; x++) B3[x] = 0.0;
          if (skips) {  // hidden skips act on the first three inputs only (API: NK == 3)
            const double* Bl = m.skip_h + ((size_t)(l - 2) * W + j) * 3;
            B3[0] = __ldg(Bl); B3[1] = __ldg(Bl + 1); B3[2] = __ldg(Bl + 2);
          }
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int q = qb * 8 + 2 * t + h;
            const double c = cb[((l - 2) * W + j) * LDS + q];
            if constexpr (NK == 3) {  // (explicit: the generic form costs ~1 % on c3)
              const double J0 = acc[i][0][h] + B3[0], J1 = acc[i][1][h] + B3[1], J2 = acc[i][2][h] + B3[2];
              const double c0 = c * J0, c1 = c * J1, c2 = c * J2;
              hp[h][0] += c0 * J0; hp[h][1] += c0 * J1; hp[h][2] += c0 * J2;
              hp[h][3] += c1 * J1; hp[h][4] += c1 * J2; hp[h][5] += c2 * J2;
              if (l < L) {
                const double s = sb[((l - 1) * W + j) * LDS + q];
                act[j * LDA + q] = s * J0;
                act[j * LDA + Q + q] = s * J1;
                act[j * LDA + 2 * Q + q] = s * J2;
              }
            } else {
              double Jv[NK];
#pragma unroll
              for (int x = 0; x < NK; x++) Jv[x] = acc[i][x][h] + B3[x];
              int o = 0;
#pragma unroll
              for (int a1 = 0; a1 < NK; a1++) {
                const double ca = c * Jv[a1];
#pragma unroll
                for (int a2 = a1; a2 < NK; a2++) hp[h][o++] += ca * Jv[a2];
              }
              if (l < L) {
                const double s = sb[((l - 1) * W + j) * LDS + q];
#pragma unroll
                for (int x = 0; x < NK; x++) act[j * LDA + x * Q + q] = s * Jv[x];
              }
            }
          }
        }
        __syncthreads();
      }
      // reduce over the 8 row-groups g of the warp (lane bits 2..4)
      if constexpr (COMMET_RS && NK == 3) {
        double v[2 * NH], o[RS<2 * NH>::K3];
#pragma unroll
        for (int h = 0; h < 2; h++)
#pragma unroll
          for (int x = 0; x < NH; x++) v[h * NH + x] = hp[h][x];
        reduce_scatter8<2 * NH>(v, o);
#pragma unroll
        for (int i = 0; i < RS<2 * NH>::K3; i++) {
          const int idx = rs_index<2 * NH>(g, i);
          if (idx >= 0) hred[(jm * Q + qb * 8 + 2 * t + idx / NH) * NH + idx % NH] = o[i];
        }
      } else {
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int x = 0; x < NH; x++) {
          double v = hp[h][x];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          hp[h][x] = v;
        }
      if (g == 0) {
#pragma unroll
        for (int h = 0; h < 2; h++)
#pragma unroll
          for (int x = 0; x < NH; x++) hred[(jm * Q + qb * 8 + 2 * t + h) * NH + x] = hp[h][x];
      }
      }
      __syncthreads();
    }

    }  // !fwd
    }  // NET == 0
    STAGE_MARK(6)
#ifdef COMMET_EXP_SKIP_NCM
    }
#endif
    if constexpr (C::EB > 1) {  // (g, H) of this network batch for the element stage
      if (!fgh && tid < Q) {
        const int q = tid;
        double* o = qgH + (h * Q + q) * C::NKH;
#pragma unroll
        for (int x = 0; x < C::NK; x++) o[x] = qg[q * C::NK + x];
#pragma unroll
        for (int x = 0; x < C::NH; x++) {
          double v = qH[q * C::NH + x];
          if (L > 1)
#pragma unroll
            for (int r = 0; r < C::JMG; r++) v += hred[(r * Q + q) * C::NH + x];
          if constexpr (C::FWDC)
            if (fwd && L == 3)
#pragma unroll
              for (int r = 0; r < C::VMG; r++) v += hred[((C::JMG + r) * Q + q) * C::NH + x];
          o[C::NK + x] = v;
        }
      }
      __syncthreads();
    }
    }  // network batches
#ifdef COMMET_EXP_SKIP_ELEM
    if (false) {
#endif
    if constexpr (C::MODE == 1) {
      material_outputs<C>(A, m, L, e0, ne, qF, qk, qg, qH, hred, qNp, qP, post, qA);
    } else {
    // ---- stage 7a: per qp -- penalty, S, T, Phi_m, Psi_m, b, P (all scaled by w) --------
#if COMMET_PREFETCH
    if (batch + gridDim.x < n_batches) pf_load_a(batch + gridDim.x);
#endif
    // stage 8's scatter metadata (hex8, one warp per (element, i-half) task): the first hop of the
    // lrow -> node_rs / node_deg chain and the slots, issued ahead so the L2 round trips overlap
    // stage 7 instead of stalling the scatter (ncu, Gent-Thomas c3: 21 % of the warp samples were
    // long-scoreboard waits on this chain)
    constexpr bool HALF8 = C::DMMA_ELEM && NEN == 8 &&
                           ((COMMET_ELEM_HALF && C::EB > 1) || (C::NET == 1 && COMMET_ELEM_HALF_NET1));
    constexpr bool MDE = HALF8 && COMMET_META_EARLY > 0;
    constexpr int TH8 = (2 * EE + C::NWARP - 1) / C::NWARP;  // stage-8 tasks per warp
    int md_la[TH8], md_lb[TH8][2], md_sab[TH8][2], md_sba[TH8][2];
    auto meta_hop1 = [&]() {
#pragma unroll
      for (int x = 0; x < TH8; x++) {
        const int task = warp + x * C::NWARP;
        const bool ok = task < ne * 2;
        const int64_t el = e0 + (ok ? task >> 1 : 0);
        md_la[x] = ok ? ld_stream(A.lrow + el * NEN + g) : 0;
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int b = 2 * t + h;
          md_lb[x][h] = ok ? ld_stream(A.lrow + el * NEN + b) : 0;
          md_sab[x][h] = ok ? 3 * (int)ld_stream(A.slot + ((size_t)el * NEN + g) * NEN + b) : 0;
          md_sba[x][h] = ok ? 3 * (int)ld_stream(A.slot + ((size_t)el * NEN + b) * NEN + g) : 0;
        }
      }
    };
    if constexpr (MDE && COMMET_META_EARLY == 2) meta_hop1();
    // ICNN, 3 inputs: four warps cooperate (warp = part of post_qp, lane = qp); otherwise one
    // thread per qp
    // (analytic networks: the CANN / Gent-Thomas instantiation (16 qps) only -- every warp repeats the
    // per-qp network, which for the ICKAN's forward mode (32 qps) costs more than it saves: 5.8 -> 9.3 ms)
    constexpr bool PAR7 = ((COMMET_POST_PAR && C::NET == 0 && C::EB > 1) ||
                           (COMMET_POST_PAR_NET1 && C::NET == 1 && C::MINB == COMMET_ANALYTIC_MINB)) &&
                          C::KIN < 2 && C::NWARP == 4;
#ifdef COMMET_EXP_SKIP_7A  // timing experiments only
    if (false) {
#else
    if (PAR7 ? lane < QE : tid < QE) {
#endif
      const int q = PAR7 ? lane : tid;
      double gq[C::NK], H6[C::NH];
      if constexpr (C::NET == 0 && C::EB > 1) {
#pragma unroll
        for (int x = 0; x < C::NK; x++) gq[x] = qgH[q * C::NKH + x];
#pragma unroll
        for (int x = 0; x < C::NH; x++) H6[x] = qgH[q * C::NKH + C::NK + x];
      } else if constexpr (C::NET == 0) {
#pragma unroll
        for (int x = 0; x < C::NK; x++) gq[x] = qg[q * C::NK + x];
#pragma unroll
        for (int x = 0; x < C::NH; x++) {
          double s = qH[q * C::NH + x];
          if (L > 1)
#pragma unroll
            for (int r = 0; r < C::JMG; r++) s += hred[(r * Q + q) * C::NH + x];
          if constexpr (C::FWDC)
            if (fwd && L == 3)  // the inner layer's Hessian term, from the backward pass
#pragma unroll
              for (int r = 0; r < C::VMG; r++) s += hred[((C::JMG + r) * Q + q) * C::NH + x];
          H6[x] = s;
        }
      } else {
        analytic_point<C::NK>(m, qk + q * C::NK, gq, H6, nullptr);
      }
      Kin kin;
      kinematics(qF + q * 9, kin);
      if constexpr (C::KIN == 1) isochoric_to_standard(kin, gq, H6);
      if constexpr (C::KIN >= 2)
        if constexpr (C::ISO_A) isochoric_aniso_to_standard<C::NSV>(kin, m.a0, m.a1, gq, H6);
      gq[2] += 2.0 * m.kappa * (kin.J - 1.0) - m.ref_shift;
      H6[packed_index(C::NK, 2, 2)] += 2.0 * m.kappa;
      if constexpr (C::KIN >= 2)
        post_qp_aniso<C::NSV>(kin, m.a0, m.a1, gq, H6, swq[q], post + q * PS, qP + q * 9);
      else if constexpr (PAR7)
        post_qp_part(kin, gq, H6, swq[q], post + q * PS, qP + q * 9, warp);
      else
        post_qp(kin, gq, H6, swq[q], post + q * PS, qP + q * 9);
    }
    if constexpr (MDE && COMMET_META_EARLY == 1) meta_hop1();
#if !defined(COMMET_DEBUG_DROP) || COMMET_DEBUG_DROP != 1  // (planted race: tools/race_check.py)
    __syncthreads();
#endif

    STAGE_MARK(7)
    // ---- stage 7b: A_q (81 entries, scaled by w), one (q, iJ) row per item ------------------
    // (three rows per item only with 16+ qps per batch: at Q = 8 the 24 items leave most threads
    // idle -- measured c4 38.0 -> 40.3 ms -- while at Q = 16 it is 0.2 % faster)
    if constexpr (C::KIN >= 2 || !COMMET_ROWS3 || QE < 16) {
#ifdef COMMET_EXP_SKIP_7B  // timing experiments only
    for (int it = tid; it < 0; it += C::NTHR) {
#else
    for (int it = tid; it < QE * 9; it += C::NTHR) {
#endif
      const int q = it / 9, iJ = it % 9;
      if constexpr (C::KIN >= 2)
        tangent_row_aniso<C::NSV>(post + q * PS, iJ, qA + q * 81 + iJ * 9);
      else
        tangent_row(post + q * PS, iJ, qA + q * 81 + iJ * 9);
    }
    } else {  // three rows (i, J = 0..2) per item: the qp's factors loaded once for the three
      for (int it = tid; it < QE * 3; it += C::NTHR)
        tangent_rows_i(post + (it / 3) * PS, it % 3, qA + (it / 3) * 81 + (it % 3) * 27);
    }
    __syncthreads();

    STAGE_MARK(8)
#if COMMET_PREFETCH
    if (batch + gridDim.x < n_batches) pf_load_b();
#endif
    if constexpr (C::DMMA_ELEM) {
    // ---- stage 8 (DMMA): K_ik[a][b] = sum_(q,J) dN_q[a][J] Y_q[J][b] for i <= k (K_ki = K_ik^T),
    //      Y_q[J][b] = sum_L A_q[(i,J),(k,L)] dN_q[b][L] formed in the B fragment (3 FMA per
    //      element); M = a, N = b, K = (q, J); r_e; RED scatter (+ mirror for i < k)
    {
      if constexpr (NEN == 8 && ((COMMET_ELEM_HALF && C::EB > 1) || (C::NET == 1 && COMMET_ELEM_HALF_NET1))) {
      // hex8: one warp per (element, i-half), the (i, k) blocks (0,0) (0,1) (0,2) or (1,1) (1,2)
      // (2,2) at once -- the dN/dX operands and the scatter metadata of the lane's node pair are
      // loaded once for the three
      constexpr int KS = NQ * 3 / 4;
      // second hop of the metadata for all of this warp's tasks, before the first task's DMMAs
      int64_t md_rsa[TH8], md_mb[TH8][2];
      int md_sa[TH8], md_sb3[TH8][2];
      if constexpr (MDE) {
#pragma unroll
        for (int x = 0; x < TH8; x++) {
          const bool ok = warp + x * C::NWARP < ne * 2;
          md_rsa[x] = ok ? ld_stream(A.node_rs + md_la[x]) : 0;
          md_sa[x] = ok ? 3 * ld_stream(A.node_deg + md_la[x]) : 0;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            md_sb3[x][h] = ok ? 3 * ld_stream(A.node_deg + md_lb[x][h]) : 0;
            md_mb[x][h] = ok ? ld_stream(A.node_rs + md_lb[x][h]) + md_sba[x][h] : 0;
          }
        }
      }
#if COMMET_META_EARLY
#pragma unroll
#else
#pragma unroll 1  // (a rolled task loop: the unrolled one costs Gent-Thomas ~1 % in instruction footprint)
#endif
      for (int x = 0; x < TH8; x++) {
        const int task = warp + x * C::NWARP;
        if (task >= ne * 2) break;
        const int e = task >> 1, i0 = task & 1;
        double c[3][2];
#pragma unroll
        for (int ik = 0; ik < 3; ik++) c[ik][0] = c[ik][1] = 0.0;
        constexpr int E8U = (C::NET == 0 && COMMET_E8_UNROLL) ? COMMET_E8_UNROLL : KS;
#pragma unroll E8U
        for (int kt = 0; kt < KS; kt++) {
          const int kk = 4 * kt + t, q = e * NQ + kk / 3, J = kk % 3;
          const double* Gg = sgN + (q * NEN + g) * 3;  // node a = b_row = g of the fragments
          const double g0 = Gg[0], g1 = Gg[1], g2 = Gg[2];
          const double av = J == 0 ? g0 : (J == 1 ? g1 : g2);
          const double* Aq = qA + q * 81 + J * 9;
#pragma unroll
          for (int ik = 0; ik < 3; ik++) {
            const int i = i0 ? (ik < 2 ? 1 : 2) : 0;
            const int k = i0 ? (ik < 2 ? ik + 1 : 2) : ik;
            const double* Ar = Aq + i * 27 + 3 * k;
            dmma(c[ik], av, Ar[0] * g0 + Ar[1] * g1 + Ar[2] * g2);
          }
        }
        const int64_t el = e0 + e;
        const int a = g;
        const int64_t la = MDE ? md_la[x] : ld_stream(A.lrow + el * NEN + a);
        const int64_t rsa = MDE ? md_rsa[x] : ld_stream(A.node_rs + la);
        const int sa = MDE ? md_sa[x] : 3 * ld_stream(A.node_deg + la);
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int b = 2 * t + h;
          const int sab = MDE ? md_sab[x][h] : 3 * (int)ld_stream(A.slot + ((size_t)el * NEN + a) * NEN + b);
          const int64_t lb = MDE ? md_lb[x][h] : ld_stream(A.lrow + el * NEN + b);
          const int sb3 = MDE ? md_sb3[x][h] : 3 * ld_stream(A.node_deg + lb);
          const int64_t mb =
              MDE ? md_mb[x][h] : ld_stream(A.node_rs + lb) + 3 * (int)ld_stream(A.slot + ((size_t)el * NEN + b) * NEN + a);
#pragma unroll
          for (int ik = 0; ik < 3; ik++) {
            const int i = i0 ? (ik < 2 ? 1 : 2) : 0;
            const int k = i0 ? (ik < 2 ? ik + 1 : 2) : ik;
            red_add(vout(A, la, rsa + i * sa + sab + k), c[ik][h]);
            if (i < k) red_add(vout(A, lb, mb + k * sb3 + i), c[ik][h]);
          }
        }
      }
      } else {
      constexpr int MTE = (NEN + 7) / 8, KS = NQ * 3 / 4;
      constexpr int NIK = 6;
      static_assert((NQ * 3) % 4 == 0, "k-steps");
      for (int task = warp; task < ne * NIK * MTE * MTE; task += C::NWARP) {
        const int nt = task % MTE, mt = (task / MTE) % MTE, ik = (task / (MTE * MTE)) % NIK,
                  e = task / (MTE * MTE * NIK);
        const int i = ik < 3 ? 0 : (ik < 5 ? 1 : 2);
        const int k = ik < 3 ? ik : (ik < 5 ? ik - 2 : 2);
        double c[2] = {0.0, 0.0};
        const int a = 8 * mt + g, bq = 8 * nt + g;
#ifdef COMMET_EXP_SKIP_KE  // timing experiments only
        c[0] = qA[tid]; c[1] = qA[tid + 1];
#pragma unroll
        for (int kt = 0; kt < 0; kt++) {
#else
#pragma unroll
        for (int kt = 0; kt < KS; kt++) {
#endif
          const int kk = 4 * kt + t, q = e * NQ + kk / 3, J = kk % 3;
          const double av = a < NEN ? sgN[(q * NEN + a) * 3 + J] : 0.0;
          double bv = 0.0;
          if (bq < NEN) {
            const double* Ar = qA + q * 81 + (3 * i + J) * 9 + 3 * k;
            const double* Gb = sgN + (q * NEN + bq) * 3;
            bv = Ar[0] * Gb[0] + Ar[1] * Gb[1] + Ar[2] * Gb[2];
          }
          dmma(c, av, bv);
        }
        const int64_t el = e0 + e;
#ifdef COMMET_EXP_SKIP_SCATTER  // timing experiments only: keep the values alive, no addresses
        if (c[0] == 1234.5678 && c[1] == 8765.4321) A.v_own[0] = c[0] + c[1];
        if (false) {
#else
        if (a < NEN) {
#endif
          const int64_t la = ld_stream(A.lrow + el * NEN + a);
          const int64_t rsa = ld_stream(A.node_rs + la);
          const int sa = 3 * ld_stream(A.node_deg + la);
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int b = 8 * nt + 2 * t + h;
            if (b < NEN) {
              red_add(vout(A, la, rsa + i * sa + 3 * (int)ld_stream(A.slot + ((size_t)el * NEN + a) * NEN + b) + k), c[h]);
              if (i < k) {
                const int64_t lb = ld_stream(A.lrow + el * NEN + b);
                const int sb3 = 3 * ld_stream(A.node_deg + lb);
                red_add(vout(A, lb, ld_stream(A.node_rs + lb) + k * sb3 +
                                          3 * (int)ld_stream(A.slot + ((size_t)el * NEN + b) * NEN + a) + i),
                          c[h]);
              }
            }
          }
        }
      }
      }
      // residual r_e[a][i] = sum_q P_q[i][:] . dN_q[a][:]
      for (int it = tid; it < ne * NEN * 3; it += C::NTHR) {
        const int i = it % 3, a = (it / 3) % NEN, e = it / (3 * NEN);
        double rr = 0.0;
#pragma unroll
        for (int qq = 0; qq < NQ; qq++) {
          const int q = e * NQ + qq;
          const double* ga = sgN + (q * NEN + a) * 3;
          rr += qP[q * 9 + i * 3] * ga[0] + qP[q * 9 + i * 3 + 1] * ga[1] + qP[q * 9 + i * 3 + 2] * ga[2];
        }
        red_add(rout(A, ld_stream(A.lrow + (e0 + e) * NEN + a), i), rr);
      }
    }
    } else {
    // ---- stage 8a: X[q][a][i][kL] = sum_J dN_aJ A_q[iJ][kL] -----------------------------------
    for (int it = tid; it < QE * 3 * NEN; it += C::NTHR) {
      const int a = it % NEN, qi = it / NEN, i = qi % 3, q = qi / 3;
      const double* ga = sgN + (q * NEN + a) * 3;
      const double g0 = ga[0], g1 = ga[1], g2 = ga[2];
      const double* Ai = qA + q * 81 + i * 27;
      double* Xo = Xb + ((q * NEN + a) * 3 + i) * 9;
#pragma unroll
      for (int kL = 0; kL < 9; kL++) Xo[kL] = g0 * Ai[kL] + g1 * Ai[9 + kL] + g2 * Ai[18 + kL];
    }
    __syncthreads();

    // ---- stage 8b: K_e[ai][bk] for node pairs b >= a only (K_e = K_e^T), r_e; RED scatter of
    //      (ai, bk) and its mirror (bk, ai)
    {
      constexpr int NP = NEN * (NEN + 1) / 2;
      for (int it = tid; it < ne * NP * 3; it += C::NTHR) {
        const int i = it % 3, ep = it / 3, e = ep / NP;
        int p = ep % NP, a = 0;
        while (p >= NEN - a) { p -= NEN - a; a++; }
        const int b = a + p;
        double K0 = 0.0, K1 = 0.0, K2 = 0.0, rr = 0.0;
#pragma unroll
        for (int qq = 0; qq < NQ; qq++) {
          const int q = e * NQ + qq;
          const double* gb = sgN + (q * NEN + b) * 3;
          const double h0 = gb[0], h1 = gb[1], h2 = gb[2];
          const double* Xr = Xb + ((q * NEN + a) * 3 + i) * 9;
          K0 += Xr[0] * h0 + Xr[1] * h1 + Xr[2] * h2;
          K1 += Xr[3] * h0 + Xr[4] * h1 + Xr[5] * h2;
          K2 += Xr[6] * h0 + Xr[7] * h1 + Xr[8] * h2;
          if (b == a) {
            const double* ga = sgN + (q * NEN + a) * 3;
            rr += qP[q * 9 + i * 3] * ga[0] + qP[q * 9 + i * 3 + 1] * ga[1] + qP[q * 9 + i * 3 + 2] * ga[2];
          }
        }
        const int64_t el = e0 + e;
        const int64_t la = ld_stream(A.lrow + el * NEN + a), lb = ld_stream(A.lrow + el * NEN + b);
        const int sa = 3 * ld_stream(A.node_deg + la);
        const int64_t dst = ld_stream(A.node_rs + la) + i * sa + 3 * (int)ld_stream(A.slot + ((size_t)el * NEN + a) * NEN + b);
        red_add(vout(A, la, dst), K0);
        red_add(vout(A, la, dst + 1), K1);
        red_add(vout(A, la, dst + 2), K2);
        if (b == a) {
          red_add(rout(A, la, i), rr);
        } else {
          const int sb3 = 3 * ld_stream(A.node_deg + lb);
          const int64_t mir = ld_stream(A.node_rs + lb) + 3 * (int)ld_stream(A.slot + ((size_t)el * NEN + b) * NEN + a) + i;
          red_add(vout(A, lb, mir), K0);
          red_add(vout(A, lb, mir + sb3), K1);
          red_add(vout(A, lb, mir + 2 * sb3), K2);
        }
      }
    }
    }  // DMMA_ELEM
    }  // MODE
#ifdef COMMET_EXP_SKIP_ELEM
    }
#endif
    __syncthreads();
    STAGE_MARK(10)
  }
  if (warp == 0) {  // stage-1 threads are tid < Q <= 32
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) trc_max = fmax(trc_max, __shfl_xor_sync(0xffffffffu, trc_max, o));
    if (lane == 0 && trc_max > 0.0) atomicMax(A.max_trc, (unsigned long long)__double_as_longlong(trc_max));
  }
#ifdef COMMET_STAGE_PROF
  if (tid == 0)
    for (int i = 0; i < 11; i++) atomicAdd(&g_stage_cycles[i], (unsigned long long)st_acc[i]);
#endif
}

// ---------------------------------------------------------------------------
// Warp-specialised kernel (the forward-sweep ICNN path, assembly): per CTA, NW = 4 network warps
// and NWE = 2 element warps in a three-slot pipeline.  Element warps: load the inputs of batch
// b + 2 (dN/dX, u_e, w) into slot (b + 2) % 3, and run stages 7-8 (penalty, S, A_q, K_e, r_e,
// scatter) of batch b from slot b % 3 -- while the network warps run stages 1-6 of batch b + 1.
// Named barriers: 1 network-internal (net_sync), FULL[3] (network -> element: F, g, H of the
// slot's batch are ready), EMPTY[3] (element -> network: the slot holds the next batch's inputs),
// 8 element-internal.  Measured motivation (profiles/r02_ab_elem_breakdown.txt, r02_ab_pad2.txt):
// in the one-role kernel the element stage adds 1.79 of 9.74 ms at c3 (it hardly overlaps the
// other CTAs' network phases) while the network alone loses only 5.5 % at 2 instead of 3 CTAs/SM.
// ---------------------------------------------------------------------------
constexpr int kBarFull0 = 2, kBarEmpty0 = 5, kBarElem = 8;

template <class C>
struct WsSmem {
  static constexpr int PS = 101;
  static constexpr int GN = C::Q * C::NEN * 3, UE = C::E * C::NEN * 3;
  // slot: dN/dX, u_e, w, F, (g, H)
  static constexpr int SLOT = ((GN + UE + C::Q + C::Q * 9 + C::Q * 9) + 1) & ~1;
  int act, sb, qk, qg, qH, hred, gsk, tab, slots, post, qA, qP, total;
  __host__ __device__ WsSmem() {
    int o = 0;
    act = o; o += C::W * C::LDA;
    sb = o; o += 2 * C::W * C::LDS;  // s_1, s_2 (L <= 3)
    qk = o; o += C::Q * 3;
    qg = o; o += C::Q * 3;
    qH = o; o += C::Q * 6;
    hred = o; o += (C::JMG + C::VMG) * C::Q * 6;
    gsk = o; o += C::Q * 3;
    tab = o; o += ActTab<C::TB_FWD>::SIZE;
    o = (o + 1) & ~1;
    slots = o; o += 3 * SLOT;
    post = o; o += C::Q * PS;
    qA = o; o += C::Q * 81;
    qP = o; o += C::Q * 9;
    total = o;
  }
  __device__ double* gN(double* sm, int s) const { return sm + slots + s * SLOT; }
  __device__ double* ue(double* sm, int s) const { return sm + slots + s * SLOT + GN; }
  __device__ double* wq(double* sm, int s) const { return sm + slots + s * SLOT + GN + UE; }
  __device__ double* qF(double* sm, int s) const { return sm + slots + s * SLOT + GN + UE + C::Q; }
  __device__ double* gH(double* sm, int s) const { return sm + slots + s * SLOT + GN + UE + C::Q + C::Q * 9; }
};

template <class C>
__device__ __forceinline__ void ws_network(const AsmArgs& A, double* smem, int L, int64_t n_it) {
  constexpr int Q = C::Q, NEN = C::NEN, NQ = C::NQ, E = C::E;
  const WsSmem<C> sm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const NcmDev& m = A.ncm;
  double* act = smem + sm.act;
  double* sb = smem + sm.sb;
  double* qk = smem + sm.qk;
  double* qg = smem + sm.qg;
  double* qH = smem + sm.qH;
  double* hred = smem + sm.hred;
  double* gsk = smem + sm.gsk;
  const double* stab = smem + sm.tab;
  double trc_max = 0.0;
  for (int64_t it = 0; it < n_it; it++) {
    const int s = (int)(it % 3);
    const int64_t e0 = A.el_begin + (blockIdx.x + it * gridDim.x) * E;
    const int64_t rem = A.el_begin + A.el_count - e0;
    const int ne = rem < E ? (int)rem : E;
    named_sync(kBarEmpty0 + s, C::NTHR_ALL);  // the element warps have put this batch's inputs in slot s
    // ---- stage 1: F, kinematics, k; det F flag ----------------------------------------------
    if (tid < Q) {
      const int q = tid, e = q / NQ;
      const double* gq = sm.gN(smem, s) + q * NEN * 3;
      const double* ue = sm.ue(smem, s) + e * NEN * 3;
      double F[9];
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int J = 0; J < 3; J++) {
          double v = (i == J) ? 1.0 : 0.0;
#pragma unroll
          for (int a = 0; a < NEN; a++) v += ue[a * 3 + i] * gq[a * 3 + J];
          F[i * 3 + J] = v;
        }
      Kin kin;
      kinematics(F, kin);
      if (e < ne) {
        if (!(kin.J > 0.0)) atomicMin(A.bad, (unsigned long long)(__ldg(A.orig + e0 + e) * NQ + q % NQ));
        trc_max = fmax(trc_max, kin.I1);
      }
      double* qF = sm.qF(smem, s);
#pragma unroll
      for (int x = 0; x < 9; x++) qF[q * 9 + x] = F[x];
      if constexpr (C::KIN == 1) {
        double kb[3];
        isochoric_inputs(kin, kb);
        qk[q * 3 + 0] = kb[0];
        qk[q * 3 + 1] = kb[1];
        qk[q * 3 + 2] = kb[2];
      } else {
        qk[q * 3 + 0] = kin.I1 - 3.0;
        qk[q * 3 + 1] = kin.I2 - 3.0;
        qk[q * 3 + 2] = kin.J - 1.0;
      }
      gsk[q * 3] = gsk[q * 3 + 1] = gsk[q * 3 + 2] = 0.0;
    }
    net_sync<C>();
    // ---- stages 2-6: layer 1, forward sweep, backward pass ----------------------------------
#ifndef COMMET_EXP_SKIP_NCM  // (timing experiments only)
    layer1<C, C::TB_FWD>(m, L, true, qk, act, sb, nullptr, nullptr, stab);
    net_sync<C>();
    if (L == 3)
      fwd_sweep<C, 3>(m, act, sb, hred, qg, qH, gsk, stab, nullptr);
    else
      fwd_sweep<C, 2>(m, act, sb, hred, qg, qH, gsk, stab, nullptr);
#endif
    // ---- g, H (summed over the warp row groups) into the slot; hand the batch over ----------
    if (tid < Q) {
      const int q = tid;
      double* gH = sm.gH(smem, s) + q * 9;
#pragma unroll
      for (int x = 0; x < 3; x++) gH[x] = qg[q * 3 + x];
#pragma unroll
      for (int x = 0; x < 6; x++) {
        double v = qH[q * 6 + x];
#pragma unroll
        for (int r = 0; r < C::JMG; r++) v += hred[(r * Q + q) * 6 + x];
        if (L == 3)
#pragma unroll
          for (int r = 0; r < C::VMG; r++) v += hred[((C::JMG + r) * Q + q) * 6 + x];
        gH[3 + x] = v;
      }
    }
    named_arrive(kBarFull0 + s, C::NTHR_ALL);
  }
  if (warp == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) trc_max = fmax(trc_max, __shfl_xor_sync(0xffffffffu, trc_max, o));
    if (lane == 0 && trc_max > 0.0) atomicMax(A.max_trc, (unsigned long long)__double_as_longlong(trc_max));
  }
}

template <class C>
__device__ __forceinline__ void ws_element(const AsmArgs& A, double* smem, int64_t n_it) {
  constexpr int Q = C::Q, NEN = C::NEN, NQ = C::NQ, E = C::E, NTE = 32 * C::NWE, PS = WsSmem<C>::PS;
  const WsSmem<C> sm;
  const int etid = threadIdx.x - C::NTHR, ewarp = etid >> 5, lane = etid & 31, g = lane >> 2, t = lane & 3;
  const NcmDev& m = A.ncm;
  double* post = smem + sm.post;
  double* qA = smem + sm.qA;
  double* qP = smem + sm.qP;
  // batch inputs: dN/dX (double2 chunks), the u gather through conn, w -- registers, then the slot
  constexpr int NG2 = Q * NEN * 3 / 2, NU = E * NEN * 3;
  constexpr int PG = (NG2 + NTE - 1) / NTE, PU = (NU + NTE - 1) / NTE, PW = (Q + NTE - 1) / NTE;
  double2 rg[PG];
  double ru[PU], rw[PW];
  auto load = [&](int64_t it) {
    const int64_t f0 = A.el_begin + (blockIdx.x + it * gridDim.x) * E;
    const int64_t frem = A.el_begin + A.el_count - f0;
    const int fne = frem < E ? (int)frem : E;
    const double2* src = reinterpret_cast<const double2*>(A.gradN + (size_t)f0 * NQ * NEN * 3);
    const int n2 = fne * NQ * NEN * 3 / 2;
#pragma unroll
    for (int i = 0; i < PG; i++) {
      const int x = etid + i * NTE;
      rg[i] = x < n2 ? __ldg(src + x) : make_double2(0.0, 0.0);
    }
    int cn[PU];
#pragma unroll
    for (int i = 0; i < PU; i++) {
      const int x = etid + i * NTE;
      const int e = x / (NEN * 3), ai = x % (NEN * 3);
      cn[i] = (x < NU && e < fne) ? ld_stream(A.conn + (f0 + e) * NEN + ai / 3) : -1;
    }
#pragma unroll
    for (int i = 0; i < PU; i++) ru[i] = cn[i] >= 0 ? ld_stream(A.u + 3 * (int64_t)cn[i] + (etid + i * NTE) % 3) : 0.0;
#pragma unroll
    for (int i = 0; i < PW; i++) {
      const int x = etid + i * NTE;
      rw[i] = x < fne * NQ ? ld_stream(A.qp_w + f0 * NQ + x) : 0.0;
    }
  };
  auto store = [&](int s) {
    double2* dg = reinterpret_cast<double2*>(sm.gN(smem, s));
#pragma unroll
    for (int i = 0; i < PG; i++) {
      const int x = etid + i * NTE;
      if (x < NG2) dg[x] = rg[i];
    }
    double* du = sm.ue(smem, s);
#pragma unroll
    for (int i = 0; i < PU; i++) {
      const int x = etid + i * NTE;
      if (x < NU) du[x] = ru[i];
    }
    double* dw = sm.wq(smem, s);
#pragma unroll
    for (int i = 0; i < PW; i++) {
      const int x = etid + i * NTE;
      if (x < Q) dw[x] = rw[i];
    }
  };
  for (int64_t it0 = 0; it0 < 2 && it0 < n_it; it0++) {
    load(it0);
    store((int)it0);
    named_arrive(kBarEmpty0 + (int)it0, C::NTHR_ALL);
  }
  for (int64_t it = 0; it < n_it; it++) {
    const int s = (int)(it % 3);
    const int64_t e0 = A.el_begin + (blockIdx.x + it * gridDim.x) * E;
    const int64_t rem = A.el_begin + A.el_count - e0;
    const int ne = rem < E ? (int)rem : E;
    const bool next = it + 2 < n_it;
    if (next) load(it + 2);  // in flight during this batch's element stage
    named_sync(kBarFull0 + s, C::NTHR_ALL);
    const double* sgN = sm.gN(smem, s);
#ifdef COMMET_EXP_SKIP_ELEM  // (timing experiments only)
    if (false) {
#endif
    // ---- stage 7a: penalty, S, T, Phi_m, Psi_m, b, P (scaled by w), one thread per qp --------
    //      with four element warps: warp = part of post_qp (post_qp_part), lane = qp
    constexpr bool PAR = C::NWE == 4 && COMMET_WS_PAR7;
#ifdef COMMET_EXP_SKIP_7A
    if (false) {
#else
    if (PAR ? lane < Q : etid < Q) {
#endif
      const int q = PAR ? lane : etid;
      const double* gH = sm.gH(smem, s) + q * 9;
      double gq[3], H6[6];
#pragma unroll
      for (int x = 0; x < 3; x++) gq[x] = gH[x];
#pragma unroll
      for (int x = 0; x < 6; x++) H6[x] = gH[3 + x];
      Kin kin;
      kinematics(sm.qF(smem, s) + q * 9, kin);
      if constexpr (C::KIN == 1) isochoric_to_standard(kin, gq, H6);
      if constexpr (C::KIN >= 2)
        if constexpr (C::ISO_A) isochoric_aniso_to_standard<C::NSV>(kin, m.a0, m.a1, gq, H6);
      gq[2] += 2.0 * m.kappa * (kin.J - 1.0) - m.ref_shift;
      H6[5] += 2.0 * m.kappa;
      if constexpr (PAR)
        post_qp_part(kin, gq, H6, sm.wq(smem, s)[q], post + q * PS, qP + q * 9, ewarp);
      else
        post_qp(kin, gq, H6, sm.wq(smem, s)[q], post + q * PS, qP + q * 9);
    }
    named_sync(kBarElem, NTE);
    // ---- stage 7b: A_q, three rows (i, J = 0..2) per item ------------------------------------
#ifndef COMMET_EXP_SKIP_7B
    for (int x = etid; x < Q * 3; x += NTE) tangent_rows_i(post + (x / 3) * PS, x % 3, qA + (x / 3) * 81 + (x % 3) * 27);
#endif
    named_sync(kBarElem, NTE);
    // ---- stage 8: K_ik[a][b] = sum_(q,J) dN_q[a][J] Y_q[J][b] (i <= k, DMMA), RED scatter ------
    //      hex8: one warp per (element, i-half): the (i, k) blocks (0,0) (0,1) (0,2) or (1,1) (1,2)
    //      (2,2) at once -- the dN/dX operands and the scatter metadata of the lane's node pair are
    //      loaded once for the three
    {
      constexpr int KS = NQ * 3 / 4;
      static_assert((NQ * 3) % 4 == 0 && NEN == 8, "k-steps / one 8x8 tile per (i, k) block");
      for (int task = ewarp; task < ne * 2; task += C::NWE) {
        const int e = task >> 1, i0 = task & 1;  // blocks (0,0..2) or (1,1..2),(2,2)
        double c[3][2];
#pragma unroll
        for (int ik = 0; ik < 3; ik++) c[ik][0] = c[ik][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < KS; kt++) {
          const int kk = 4 * kt + t, q = e * NQ + kk / 3, J = kk % 3;
          const double* Gg = sgN + (q * NEN + g) * 3;  // node a = b_row = g of the fragments
          const double g0 = Gg[0], g1 = Gg[1], g2 = Gg[2];
          const double av = J == 0 ? g0 : (J == 1 ? g1 : g2);
          const double* Aq = qA + q * 81 + J * 9;
#pragma unroll
          for (int ik = 0; ik < 3; ik++) {
            const int i = i0 ? (ik < 2 ? 1 : 2) : 0;
            const int k = i0 ? (ik < 2 ? ik + 1 : 2) : ik;
            const double* Ar = Aq + i * 27 + 3 * k;
#ifdef COMMET_EXP_SKIP_KE
            c[ik][0] += Ar[0] * g0; c[ik][1] += av;
#else
            dmma(c[ik], av, Ar[0] * g0 + Ar[1] * g1 + Ar[2] * g2);
#endif
          }
        }
        const int64_t el = e0 + e;
        const int a = g;
#ifdef COMMET_EXP_SKIP_SCATTER
        if (c[0][0] == 1234.5678 && c[2][1] == 8765.4321) A.v_own[0] = c[1][0];
        if (false) {
#else
        {
#endif
        const int64_t la = ld_stream(A.lrow + el * NEN + a);
        const int64_t rsa = ld_stream(A.node_rs + la);
        const int sa = 3 * ld_stream(A.node_deg + la);
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int b = 2 * t + h;
          const int sab = 3 * (int)ld_stream(A.slot + ((size_t)el * NEN + a) * NEN + b);
          const int64_t lb = ld_stream(A.lrow + el * NEN + b);
          const int sb3 = 3 * ld_stream(A.node_deg + lb);
          const int64_t mb = ld_stream(A.node_rs + lb) + 3 * (int)ld_stream(A.slot + ((size_t)el * NEN + b) * NEN + a);
#pragma unroll
          for (int ik = 0; ik < 3; ik++) {
            const int i = i0 ? (ik < 2 ? 1 : 2) : 0;
            const int k = i0 ? (ik < 2 ? ik + 1 : 2) : ik;
            red_add(vout(A, la, rsa + i * sa + sab + k), c[ik][h]);
            if (i < k) red_add(vout(A, lb, mb + k * sb3 + i), c[ik][h]);
          }
        }
        }
      }
      // residual r_e[a][i] = sum_q P_q[i][:] . dN_q[a][:]
      for (int x = etid; x < ne * NEN * 3; x += NTE) {
        const int i = x % 3, a = (x / 3) % NEN, e = x / (3 * NEN);
        double rr = 0.0;
#pragma unroll
        for (int qq = 0; qq < NQ; qq++) {
          const int q = e * NQ + qq;
          const double* ga = sgN + (q * NEN + a) * 3;
          rr += qP[q * 9 + i * 3] * ga[0] + qP[q * 9 + i * 3 + 1] * ga[1] + qP[q * 9 + i * 3 + 2] * ga[2];
        }
        red_add(rout(A, ld_stream(A.lrow + (e0 + e) * NEN + a), i), rr);
      }
    }
#ifdef COMMET_EXP_SKIP_ELEM
    }
#endif
    // slot s is free for batch it + 3 once both element warps are past stage 8 (the next batch's
    // 7a barrier orders that); the inputs of batch it + 2 go to slot (it + 2) % 3 now
    if (next) {
      store((int)((it + 2) % 3));
      named_arrive(kBarEmpty0 + (int)((it + 2) % 3), C::NTHR_ALL);
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::NTHR_ALL, C::MINB) ws_kernel(AsmArgs A) {
  static_assert(C::WS && C::FWDC && C::NET == 0 && C::MODE == 0 && C::NK == 3 && C::NWARP == 4, "ws config");
  extern __shared__ __align__(16) double smem[];
  const WsSmem<C> sm;
  const int L = A.ncm.L;
  for (int x = threadIdx.x; x < ActTab<C::TB_FWD>::SIZE; x += C::NTHR_ALL)
    smem[sm.tab + x] = __ldg(A.ncm.act_tab + act_tab_offset<C::TB_FWD>() + x);
  __syncthreads();
  const int64_t nb = (A.el_count + C::E - 1) / C::E;
  const int64_t n_it = nb > blockIdx.x ? (nb - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if constexpr (C::NWE == 4) {  // two warpgroups: move registers from the element to the network one
    if (threadIdx.x < C::NTHR) {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(COMMET_WS_NREG_NET));
      ws_network<C>(A, smem, L, n_it);
    } else {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(256 - COMMET_WS_NREG_NET));
      ws_element<C>(A, smem, n_it);
    }
  } else {
    if (threadIdx.x < C::NTHR)
      ws_network<C>(A, smem, L, n_it);
    else
      ws_element<C>(A, smem, n_it);
  }
}

// ---------------------------------------------------------------------------
// host side: dispatch and weight fragments
// ---------------------------------------------------------------------------

#ifdef COMMET_STAGE_PROF
}  // namespace commet
extern "C" int commet_debug_stage_cycles(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, commet::g_stage_cycles, 11 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(commet::g_stage_cycles, z, sizeof(z));
  }
  return 0;
}
namespace commet {
#endif

int fused_supported(int n_en, int n_q, int w, int L) {
  if (!((n_en == 8 && n_q == 8) || (n_en == 10 && n_q == 4))) return 0;
  if (!(w == 8 || w == 16 || w == 32 || w == 64 || w == 128)) return 0;
  if (L < 1 || L > kMaxLayers) return 0;
  return 1;
}

int64_t fused_weight_frag_size(int w, int L) { return (int64_t)(L > 1 ? L - 1 : 1) * 2 * w * w; }

// fragment (mt, kt2), lane (g,t), half h  <-  M[8 mt + g][8 kt2 + 4 h + t]
void fused_weight_frag_fill(int w, int L, const double* Wrow, double* out) {
  const int KT2 = w / 8;
  for (int l = 0; l < L - 1; l++) {
    const double* Wl = Wrow + (size_t)l * w * w;
    double* fw = out + (size_t)l * 2 * w * w;
    double* ft = fw + (size_t)w * w;
    for (int mt = 0; mt < w / 8; mt++)
      for (int kt2 = 0; kt2 < KT2; kt2++)
        for (int lane = 0; lane < 32; lane++)
          for (int h = 0; h < 2; h++) {
            const int g = lane >> 2, t = lane & 3;
            const int r = 8 * mt + g, c = 8 * kt2 + 4 * h + t;
            const size_t o = ((size_t)(mt * KT2 + kt2) * 32 + lane) * 2 + h;
            fw[o] = Wl[(size_t)r * w + c];   // W_l
            ft[o] = Wl[(size_t)c * w + r];   // W_l^T
          }
  }
}

// One launch of kernel `fn` (nthr threads, `bytes` of dynamic shared memory, E elements per
// batch): a persistent grid of min(batches, SMs x resident CTAs).  The shared-memory attribute,
// SM count and occupancy are queried once per (kernel, device, smem size) -- the host-side launch
// cost matters for small batches -- under a lock (several contexts on one device may launch from
// different host threads) and used as one consistent snapshot.
template <class Tag>
static int launch_persistent(void (*fn)(AsmArgs), int nthr, size_t bytes, int E, const AsmArgs& a, cudaStream_t st,
                             int* launches, int kind = 0, int q_net = 0, int q_elem = 0) {
  constexpr int kDev = 16;
  static std::mutex mu;
  static size_t attr_bytes[kDev] = {0};
  static int sms_c[kDev] = {0}, per_sm_c[kDev] = {0};
  static size_t occ_bytes[kDev] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kDev) return (int)cudaErrorInvalidDevice;
  int sms = 0, per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (attr_bytes[dev] < bytes) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (e != cudaSuccess) return (int)e;
      attr_bytes[dev] = bytes;
    }
    if (occ_bytes[dev] != bytes) {
      int sc = 0, ps = 0;
      cudaError_t e = cudaDeviceGetAttribute(&sc, cudaDevAttrMultiProcessorCount, dev);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, fn, nthr, bytes);
      if (e != cudaSuccess) return (int)e;
      sms_c[dev] = sc;
      per_sm_c[dev] = ps < 1 ? 1 : ps;
      occ_bytes[dev] = bytes;
    }
    sms = sms_c[dev];
    per_sm = per_sm_c[dev];
  }
  if (a.query) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, fn);
    a.query[0] = (int)bytes;
    a.query[1] = per_sm;
    a.query[2] = fa.numRegs;
    a.query[3] = nthr;
    a.query[4] = kind;  // 0 one-role fused kernel, 1 warp-specialised
    a.query[5] = q_net;   // qps per network batch
    a.query[6] = q_elem;  // qps per element batch
    return 0;
  }
  const int64_t nb = (a.el_count + E - 1) / E;
  const int64_t grid = std::min<int64_t>(nb, (int64_t)sms * per_sm);
  if (nb <= 0) return 0;
  if (grid <= 0) return (int)cudaErrorInvalidConfiguration;  // never a silent no-op with work to do
  fn<<<(unsigned)grid, nthr, bytes, st>>>(a);
  if (launches) (*launches)++;
  return (int)cudaGetLastError();
}

template <class C>
static int launch_cfg(const AsmArgs& a, cudaStream_t st, int* launches) {
  const Smem<C> sm(a.ncm.L, a.ncm.skip_h != nullptr);
  size_t bytes = (size_t)sm.total * sizeof(double);
#ifdef COMMET_EXP_SMEM_PAD
  bytes += COMMET_EXP_SMEM_PAD;  // experiments only: limit resident CTAs per SM
#endif
  return launch_persistent<C>(fused_kernel<C>, C::NTHR, bytes, C::EE, a, st, launches, 0, C::Q, C::QE);
}

// the warp-specialised kernel (forward-sweep ICNN path of the assembly)
template <class C>
struct WsTag {};
template <class C>
static int launch_ws(const AsmArgs& a, cudaStream_t st, int* launches) {
  const size_t bytes = (size_t)WsSmem<C>().total * sizeof(double);
  return launch_persistent<WsTag<C>>(ws_kernel<C>, C::NTHR_ALL, bytes, C::E, a, st, launches, 1, C::Q, C::Q);
}

template <int NEN, int NQ, int K>
static int launch_k(const AsmArgs& a, cudaStream_t st, int* launches) {
#ifdef COMMET_AB_MIN
  if constexpr (K == 0) {
    if constexpr (NEN == 8 && COMMET_WS)
      if (a.ncm.net == 0 && a.ncm.L >= 2 && a.ncm.L <= 3 && a.ncm.skip_h == nullptr) {
        if (a.ncm.w == 64) return launch_ws<Cfg<64, 16, NEN, NQ, 2, 0, 0, 0, 4, 1>>(a, st, launches);
        if (a.ncm.w == 128) return launch_ws<Cfg<128, 8, NEN, NQ, 2, 0, 0, 0, 4, 1>>(a, st, launches);
      }
    if (a.ncm.net == 0 && a.ncm.w == 64) return launch_cfg<Cfg<64, 16, NEN, NQ, 3, 0, 0>>(a, st, launches);
    if (a.ncm.net == 0 && a.ncm.w == 128) return launch_cfg<Cfg<128, 8, NEN, NQ, 3, 0, 0>>(a, st, launches);
    if (a.ncm.net == 1 || a.ncm.net == 2)  // CANN / Gent-Thomas (element-stage tuning)
      return launch_cfg<Cfg<16, COMMET_ANALYTIC_Q, NEN, NQ, COMMET_ANALYTIC_MINB, 1, 0>>(a, st, launches);
  }
  return (int)cudaErrorInvalidValue;
#else
  if constexpr (K == 3 || K == 5) {  // two structural vectors, 9 inputs: the per-qp (analytic) networks only
    if (a.ncm.net != 0) return launch_cfg<Cfg<16, COMMET_Q_KIN3, NEN, NQ, 2, 1, K>>(a, st, launches);
    return (int)cudaErrorInvalidValue;  // (an ICNN on 9 inputs is refused at setup)
  } else {
  if constexpr (K == 2 || K == 4) {  // 5 inputs: packed 5x5 Hessians and the extended F-space factors
    if (a.ncm.net != 0) return launch_cfg<Cfg<16, 32, NEN, NQ, 2, 1, K>>(a, st, launches);
  } else {
    if (a.ncm.net == 3)  // ICKAN: its per-qp forward mode needs the registers (4 CTAs/SM: spills, -14 %)
      return launch_cfg<Cfg<16, 32, NEN, NQ, COMMET_ICKAN_MINB, 1, K>>(a, st, launches);
    // (tet10 keeps 16 qps: its scalar element stage's X buffer grows with the batch)
    if (a.ncm.net != 0)
      return launch_cfg<Cfg<16, NEN == 8 ? COMMET_ANALYTIC_Q : 16, NEN, NQ, COMMET_ANALYTIC_MINB, 1, K>>(a, st, launches);
  }
  // the forward-sweep ICNN (w = 64 / 128, L = 2 or 3, no hidden skips) on hex8: warp-specialised
  // kernel (tet10 keeps the one-role kernel: its scalar element stage needs the aliased X buffer)
  if constexpr (K < 2 && NEN == 8 && COMMET_WS) {
    if (a.ncm.L >= 2 && a.ncm.L <= 3 && a.ncm.skip_h == nullptr) {
      if (a.ncm.w == 64) return launch_ws<Cfg<64, 16, NEN, NQ, 2, 0, K, 0, 4, 1>>(a, st, launches);
      if (a.ncm.w == 128) return launch_ws<Cfg<128, 8, NEN, NQ, 2, 0, K, 0, 4, 1>>(a, st, launches);
    }
  }
  // 5-input ICNN: the Jacobian pass carries 5 columns and 15 Hessian partials -> 2 CTAs/SM
  constexpr int MB = K >= 2 ? 2 : 3;
  switch (a.ncm.w) {
    case 8: return launch_cfg<Cfg<8, 32, NEN, NQ, MB, 0, K>>(a, st, launches);
    case 16: return launch_cfg<Cfg<16, 16, NEN, NQ, MB, 0, K>>(a, st, launches);
    case 32: return launch_cfg<Cfg<32, 16, NEN, NQ, MB, 0, K>>(a, st, launches);
    case 64: return launch_cfg<Cfg<64, 16, NEN, NQ, MB, 0, K>>(a, st, launches);
    case 128: return launch_cfg<Cfg<128, 8, NEN, NQ, MB, 0, K>>(a, st, launches);
  }
  return (int)cudaErrorInvalidValue;
  }
#endif
}

// material points: NEN = NQ = 1, one "element" per point
template <int K>
static int launch_mat_k(const AsmArgs& a, cudaStream_t st) {
#ifdef COMMET_AB_MIN
  return (int)cudaErrorInvalidValue;
#else
  if constexpr (K == 3 || K == 5) {  // two structural vectors: analytic networks only
    if (a.ncm.net != 0) return launch_cfg<Cfg<16, 16, 1, 1, 2, 1, K, 1>>(a, st, nullptr);
    return (int)cudaErrorInvalidValue;
  } else {
  if (a.ncm.net != 0) return launch_cfg<Cfg<16, 16, 1, 1, 3, 1, K, 1>>(a, st, nullptr);
  constexpr int MB = K >= 2 ? 2 : 3;
  switch (a.ncm.w) {
    case 8: return launch_cfg<Cfg<8, 32, 1, 1, MB, 0, K, 1>>(a, st, nullptr);
    case 16: return launch_cfg<Cfg<16, 16, 1, 1, MB, 0, K, 1>>(a, st, nullptr);
    case 32: return launch_cfg<Cfg<32, 16, 1, 1, MB, 0, K, 1>>(a, st, nullptr);
    case 64: return launch_cfg<Cfg<64, 16, 1, 1, MB, 0, K, 1>>(a, st, nullptr);
    case 128: return launch_cfg<Cfg<128, 8, 1, 1, MB, 0, K, 1>>(a, st, nullptr);
  }
  return (int)cudaErrorInvalidValue;
  }
#endif
}

int launch_material(const AsmArgs& a, void* stream) {
  if (a.el_count <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (a.ncm.kin >= 2 && a.ncm.aniso_iso)  // isochoric anisotropic: the KIN 4 / 5 instantiations
    return a.ncm.kin == 3 ? launch_mat_k<5>(a, st) : launch_mat_k<4>(a, st);
  if (a.ncm.kin == 3) return launch_mat_k<3>(a, st);
  return a.ncm.kin == 2 ? launch_mat_k<2>(a, st) : a.ncm.kin == 1 ? launch_mat_k<1>(a, st) : launch_mat_k<0>(a, st);
}

template <int NEN, int NQ>
static int launch_et(const AsmArgs& a, cudaStream_t st, int* launches) {
#ifdef COMMET_AB_MIN
  return launch_k<NEN, NQ, 0>(a, st, launches);
#else
  if (a.ncm.kin >= 2 && a.ncm.aniso_iso)  // isochoric anisotropic: the KIN 4 / 5 instantiations
    return a.ncm.kin == 3 ? launch_k<NEN, NQ, 5>(a, st, launches) : launch_k<NEN, NQ, 4>(a, st, launches);
  if (a.ncm.kin == 3) return launch_k<NEN, NQ, 3>(a, st, launches);
  if (a.ncm.kin == 2) return launch_k<NEN, NQ, 2>(a, st, launches);
  return a.ncm.kin == 1 ? launch_k<NEN, NQ, 1>(a, st, launches) : launch_k<NEN, NQ, 0>(a, st, launches);
#endif
}

int launch_fused(const AsmArgs& a, void* stream, int* launches) {
  if (a.el_count <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (a.n_en == 8) return launch_et<8, 8>(a, st, launches);
  return launch_et<10, 4>(a, st, launches);
}

}  // namespace commet
