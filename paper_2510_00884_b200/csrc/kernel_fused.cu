// kernel_fused.cu -- the product path: ONE kernel per element colour that runs
// every step of the hot path for a batch of
// elements held in shared memory; nothing but u, the element inputs and the
// scatter touch HBM.
//
// Per CTA iteration (E elements = Q quadrature points):
//   0  wait for this batch's inputs (cp.async, issued one batch ahead), issue
//      the next batch's                                         (a1)
//   2  per qp: F, C, I1, I2, J -> k, det F flag; layer 1 (3 -> w) (a2, a3, a4)
//   3  value pass, hidden layers l = 2..L:  Y = W_l Z           (a4, DMMA GEMM)
//   4  adjoint pass l = L..2:  Lambda = W_l^T M                 (a4, DMMA GEMM)
//   5  [g; H_1] = [W1^T 0; 0 V] [mu_1; c_1]                     (a4, DMMA GEMM)
//   6  Jacobian pass l = 2..L: J_l = W_l (s_{l-1} (.) J_{l-1})   (a4, DMMA GEMM)
//      H += J_l^T diag(c_l) J_l on the fly, c_l = lambda_l s_l (1-s_l)
//   7  penalty, S and the F-space tangent factors per qp        (a5, a6)
//   8a X[q][a][i][kL] = sum_J dN_aJ A_q[iJ][kL] from the factors (a6, a7)
//   8b K_e, r_e; coloured RED scatter                           (a7, a8)
// The inner-network derivatives are the exact Hessian of Alg. 4
// obtained with 5 w^2 FMA per hidden layer instead of
// Alg. 4's 10 w^2.  Hidden-layer contractions use the fp64
// tensor path (mma.sync m8n8k4 f64 = SASS DMMA.8x8x4): on B200 it shares the
// fp64 datapath with DFMA (measured, profiles/r01_fp64_peak.json) but needs
// ~8x fewer issue slots and register-file reads per FMA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "commet_internal.h"
#include "qp_math.cuh"

namespace commet {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// global -> shared asynchronous copies (LDGSTS), 16 / 8 / 4 bytes
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------------------
// compile-time tiling
// ---------------------------------------------------------------------------
template <int W_, int Q_, int NEN_, int NQ_, int MINB_ = 3>
struct Cfg {
  static constexpr int W = W_, Q = Q_, NEN = NEN_, NQ = NQ_;
  static constexpr int NWARP = 4, NTHR = 128;
  static constexpr int MINB = MINB_;               // CTAs per SM the register budget targets
  static constexpr int E = Q / NQ;                 // elements per CTA iteration
  static constexpr int MTILES = W / 8, QB = Q / 8, KT2 = W / 8;
  // value / adjoint warp tiles: VMG x VNG warps, each MT_V x NT_V tiles
  static constexpr int TPW = MTILES * QB / NWARP;
  static constexpr int NT_V = (QB >= 2 && TPW % 2 == 0 && TPW >= 4) ? 2 : 1;
  static constexpr int MT_V = TPW / NT_V;
  static constexpr int VNG = QB / NT_V, VMG = MTILES / MT_V;
  // Jacobian warp tiles: JMG m-groups x QB qp blocks, each MT_J x 3 tiles
  static constexpr int JMG = NWARP / QB, MT_J = MTILES / JMG;
  // stage 5: 2 m-tiles x QB n-tiles, K split over the remaining warps
  static constexpr int G5T = 2 * QB;
  static constexpr int G5S = NWARP > G5T ? NWARP / G5T : 1;
  static constexpr int LDA = 3 * Q + 4;            // act row stride (2 LDA = 8 or 24 mod 32: conflict-free B frags)
  static constexpr int LDS = Q + 1;                // s/c row stride (odd: <= 2-way conflicts)
  static constexpr int UPT = (E * NEN * 3 + NTHR - 1) / NTHR;  // prefetched u values per thread
  static_assert(W % 8 == 0 && Q % 8 == 0 && Q % NQ == 0 && NTHR % Q == 0, "tile");
  static_assert(TPW >= 1 && VMG * VNG == NWARP && MT_V * NT_V == TPW, "value tiling");
  static_assert(JMG >= 1 && JMG * QB == NWARP && MT_J * JMG == MTILES, "jacobian tiling");
  static_assert((KT2 % G5S) == 0 && (G5S == 1 || W >= 16 * G5S), "stage-5 split");
  static_assert(E * NEN <= NTHR, "one scatter base per thread");
  static_assert((W * Q) % NTHR == 0, "layer-1 items per thread");
};

// shared-memory carve-up (doubles); L is a runtime value.  act/s/c are dead
// after stage 6 and host the post-NCM buffers (qP, post/X, qA) and the
// Jacobian-pass partials.  Per-batch inputs are double-buffered.
template <class C>
struct Smem {
  static constexpr int PS = 101;  // per-qp stride of the stage-7 outputs (odd: bank spread)
  // per-batch input block (doubles): gN, w, u_e, CSR value / residual bases, row strides,
  // conn, lrow, slots
  static constexpr int IN_GN = 0;
  static constexpr int IN_W = IN_GN + C::Q * C::NEN * 3;
  static constexpr int IN_U = IN_W + C::Q;
  static constexpr int IN_VB = IN_U + C::E * C::NEN * 3;
  static constexpr int IN_RB = IN_VB + C::E * C::NEN;
  static constexpr int IN_RS = IN_RB + C::E * C::NEN;                 // int
  static constexpr int IN_CONN = IN_RS + (C::E * C::NEN + 1) / 2;     // int
  static constexpr int IN_LROW = IN_CONN + (C::E * C::NEN + 1) / 2;   // int
  static constexpr int IN_SLOT = IN_LROW + (C::E * C::NEN + 1) / 2;   // uint8
  static constexpr int IN_SIZE = ((IN_SLOT + (C::E * C::NEN * C::NEN + 7) / 8) + 1) & ~1;
  int act, sb, cb, qF, qk, qg, qH, hred, gsk, tab, in0, qP, post, X, total;
  __host__ __device__ Smem(int L) {
    int o = 0;
    act = o; o += C::W * C::LDA;
    sb = o;  o += (L > 1 ? L - 1 : 0) * C::W * C::LDS;   // s_l, l = 1..L-1
    cb = o;  o += (L > 1 ? L - 1 : 0) * C::W * C::LDS;   // c_l, l = 2..L
    const int dead = o;
    qF = o;  o += C::Q * 9;
    qk = o;  o += C::Q * 3;
    qg = o;  o += C::Q * 3;
    qH = o;  o += C::Q * 6;
    gsk = o; o += C::Q * 3;
    tab = o; o += kActTabSize;
    o = (o + 1) & ~1;
    in0 = o; o += 2 * IN_SIZE;
    const int need = C::Q * 9 + C::Q * PS + C::Q * C::NEN * 27 + C::JMG * C::Q * 6;
    int base = 0;
    if (need > dead) { base = o; o += need; }
    qP = base;
    post = qP + C::Q * 9;
    X = post + C::Q * PS;
    hred = X + C::Q * C::NEN * 27;
    total = o;
  }
};

// ---------------------------------------------------------------------------
// one warp tile of  C (+)= A (M x K, fragments in global) * B (K x N, smem)
// KS k-pair steps starting at fragment column k0 of a matrix with KT2 pairs
// ---------------------------------------------------------------------------
template <int MT, int NT, int KS, int KT2, bool ACC = false>
__device__ __forceinline__ void warp_gemm(const double* __restrict__ Af, int mt0, const double* act,
                                          int lda, const int (&ncol)[NT], double (&acc)[MT][NT][2],
                                          int k0 = 0) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (!ACC) {
#pragma unroll
    for (int i = 0; i < MT; i++)
#pragma unroll
      for (int j = 0; j < NT; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  }
  const double* ap = Af + ((size_t)mt0 * KT2 + k0) * 64 + lane * 2;
  const double* bp = act + (k0 * 8 + t) * lda + g;
  // A fragments stream from L2 (L1 is mostly shared memory): 3-deep register pipeline
  double2 a[3][MT];
#pragma unroll
  for (int i = 0; i < MT; i++) a[0][i] = ldg2(ap + (size_t)i * KT2 * 64);
  if (KS > 1) {
#pragma unroll
    for (int i = 0; i < MT; i++) a[1][i] = ldg2(ap + ((size_t)i * KT2 + 1) * 64);
  }
#pragma unroll
  for (int kt2 = 0; kt2 < KS; kt2++) {
    const int cur = kt2 % 3;
    if (kt2 + 2 < KS) {
#pragma unroll
      for (int i = 0; i < MT; i++) a[(kt2 + 2) % 3][i] = ldg2(ap + ((size_t)i * KT2 + kt2 + 2) * 64);
    }
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
  }
}

// issue the asynchronous copies of batch `batch`'s contiguous inputs into block `in`
template <class C>
__device__ __forceinline__ void stage_inputs(const AsmArgs& A, int64_t batch, double* in) {
  using S = Smem<C>;
  constexpr int NEN = C::NEN, NQ = C::NQ, E = C::E, Q = C::Q;
  const int64_t e0 = A.el_begin + batch * E;
  const int64_t rem = A.el_begin + A.el_count - e0;
  const int ne = rem < E ? (int)rem : E;
  const int tid = threadIdx.x;
  {
    const double* src = A.gradN + (size_t)e0 * NQ * NEN * 3;
    double* dst = in + S::IN_GN;
    const int n2 = ne * NQ * NEN * 3 / 2;
    for (int x = tid; x < E * NQ * NEN * 3 / 2; x += C::NTHR) {
      if (x < n2) cp_async16(dst + 2 * x, src + 2 * x);
      else dst[2 * x] = dst[2 * x + 1] = 0.0;
    }
  }
  for (int x = tid; x < Q; x += C::NTHR) {
    if (x < ne * NQ) cp_async8(in + S::IN_W + x, A.qp_w + e0 * NQ + x);
    else in[S::IN_W + x] = 0.0;
  }
  int* conn = reinterpret_cast<int*>(in + S::IN_CONN);
  int* lrow = reinterpret_cast<int*>(in + S::IN_LROW);
  for (int x = tid; x < ne * NEN; x += C::NTHR) {
    cp_async4(conn + x, A.conn + e0 * NEN + x);
    cp_async4(lrow + x, A.lrow + e0 * NEN + x);
  }
  {
    const uint32_t* src32 = reinterpret_cast<const uint32_t*>(A.slot + (size_t)e0 * NEN * NEN);
    uint32_t* dst32 = reinterpret_cast<uint32_t*>(in + S::IN_SLOT);
    for (int x = tid; x < ne * NEN * NEN / 4; x += C::NTHR) cp_async4(dst32 + x, src32 + x);
  }
  cp_async_commit();
}

// dependent gathers of a batch whose conn/lrow are in `in`: u_e (returned in registers,
// stored by commit_gathers) and the CSR scatter bases (stored directly)
template <class C>
struct Gathered {
  double u[C::UPT];
  double* vb;
  double* rb;
  int rs;
};

template <class C>
__device__ __forceinline__ void issue_gathers(const AsmArgs& A, int ne, const double* in, Gathered<C>& G) {
  using S = Smem<C>;
  constexpr int NEN = C::NEN;
  const int tid = threadIdx.x;
  const int* conn = reinterpret_cast<const int*>(in + S::IN_CONN);
  const int* lrow = reinterpret_cast<const int*>(in + S::IN_LROW);
#pragma unroll
  for (int k = 0; k < C::UPT; k++) {
    const int x = tid + k * C::NTHR;
    const int e = x / (NEN * 3), ai = x % (NEN * 3);
    G.u[k] = (x < C::E * NEN * 3 && e < ne) ? __ldg(A.u + 3 * (int64_t)conn[e * NEN + ai / 3] + ai % 3) : 0.0;
  }
  G.vb = nullptr;
  G.rb = nullptr;
  G.rs = 0;
  if (tid < ne * NEN) {
    const int64_t ln = lrow[tid];
    const bool own = ln < A.n_owned;
    G.vb = (own ? A.v_own : A.v_halo) + __ldg(A.node_rs + ln);
    G.rb = (own ? A.r_own : A.r_halo) + 3 * (own ? ln : ln - A.n_owned);
    G.rs = 3 * __ldg(A.node_deg + ln);
  }
}

template <class C>
__device__ __forceinline__ void commit_gathers(int ne, double* in, const Gathered<C>& G) {
  using S = Smem<C>;
  const int tid = threadIdx.x;
#pragma unroll
  for (int k = 0; k < C::UPT; k++) {
    const int x = tid + k * C::NTHR;
    if (x < C::E * C::NEN * 3) in[S::IN_U + x] = G.u[k];
  }
  if (tid < ne * C::NEN) {
    reinterpret_cast<double**>(in + S::IN_VB)[tid] = G.vb;
    reinterpret_cast<double**>(in + S::IN_RB)[tid] = G.rb;
    reinterpret_cast<int*>(in + S::IN_RS)[tid] = G.rs;
  }
}

template <class C>
__global__ void __launch_bounds__(C::NTHR, C::MINB) fused_kernel(AsmArgs A) {
  using S = Smem<C>;
  constexpr int W = C::W, Q = C::Q, NEN = C::NEN, NQ = C::NQ, E = C::E;
  constexpr int LDA = C::LDA, LDS = C::LDS, KT2 = C::KT2;
  constexpr int PS = S::PS;
  extern __shared__ __align__(16) double smem[];
  const int L = A.ncm.L;
  const S sm(L);
  double* act = smem + sm.act;
  double* sb = smem + sm.sb;
  double* cb = smem + sm.cb;
  double* qF = smem + sm.qF;
  double* qk = smem + sm.qk;
  double* qg = smem + sm.qg;
  double* qH = smem + sm.qH;
  double* hred = smem + sm.hred;
  double* gsk = smem + sm.gsk;
  double* qP = smem + sm.qP;
  double* post = smem + sm.post;
  double* Xb = smem + sm.X;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const NcmDev& m = A.ncm;
  double* tab = smem + sm.tab;  // softplus tables (L1 is mostly carved out as shared memory)
  for (int x = tid; x < kActTabSize; x += C::NTHR) tab[x] = __ldg(m.act_tab + x);
  const bool skips = m.skip_h != nullptr;
  const int64_t n_batches = (A.el_count + E - 1) / E;
  const size_t frag_layer = (size_t)2 * W * W;  // W and W^T fragments per hidden layer
  if ((int64_t)blockIdx.x >= n_batches) return;

  // prologue: inputs of the first batch, synchronously
  {
    double* in = smem + sm.in0;
    stage_inputs<C>(A, blockIdx.x, in);
    cp_async_wait_all();
    __syncthreads();
    const int64_t rem = A.el_count - (int64_t)blockIdx.x * E;
    Gathered<C> G;
    issue_gathers<C>(A, rem < E ? (int)rem : E, in, G);
    commit_gathers<C>(rem < E ? (int)rem : E, in, G);
  }

  int buf = 0;
  for (int64_t batch = blockIdx.x; batch < n_batches; batch += gridDim.x, buf ^= 1) {
    const int64_t e0 = A.el_begin + batch * E;
    const int64_t rem = A.el_begin + A.el_count - e0;
    const int ne = rem < E ? (int)rem : E;
    double* in = smem + sm.in0 + buf * S::IN_SIZE;
    double* nin = smem + sm.in0 + (buf ^ 1) * S::IN_SIZE;
    const double* sgN = in + S::IN_GN;
    const double* swq = in + S::IN_W;
    const double* sue = in + S::IN_U;
    double* const* svb = reinterpret_cast<double* const*>(in + S::IN_VB);
    double* const* srb = reinterpret_cast<double* const*>(in + S::IN_RB);
    const int* srs = reinterpret_cast<const int*>(in + S::IN_RS);
    const uint8_t* sslot = reinterpret_cast<const uint8_t*>(in + S::IN_SLOT);
    const int64_t nbatch = batch + gridDim.x;
    const bool has_next = nbatch < n_batches;
    int nne = 0;
    if (has_next) {
      const int64_t nrem = A.el_begin + A.el_count - (A.el_begin + nbatch * E);
      nne = nrem < E ? (int)nrem : E;
    }

    // ---- stage 0: this batch's inputs are resident; prefetch the next batch's ---------
    __syncthreads();
    if (has_next) stage_inputs<C>(A, nbatch, nin);

    // ---- stage 2: per-qp kinematics + layer 1 --------------------------------------------
    // TPQ consecutive lanes per qp: F's 9 entries are split over them and shared by
    // shuffles; each lane then forms k and evaluates W/TPQ neurons of layer 1
    {
      constexpr int TPQ = C::NTHR / Q;
      const int q = tid / TPQ, r = tid % TPQ, e = q / NQ;
      const int gbase = lane & ~(TPQ - 1);
      const double* gq = sgN + q * NEN * 3;
      const double* ue = sue + e * NEN * 3;
      constexpr int NV = (9 + TPQ - 1) / TPQ;
      double fv[NV];
#pragma unroll
      for (int h = 0; h < NV; h++) {
        fv[h] = 0.0;
        const int x = r + h * TPQ;
        if (x < 9) {
          const int i = x / 3, J = x % 3;
          double s = (i == J) ? 1.0 : 0.0;
#pragma unroll
          for (int a = 0; a < NEN; a++) s += ue[a * 3 + i] * gq[a * 3 + J];
          fv[h] = s;
        }
      }
      double F[9];
#pragma unroll
      for (int x = 0; x < 9; x++)
        F[x] = __shfl_sync(0xffffffffu, fv[x / TPQ], gbase + x % TPQ);
      // k = (I1-3, I2-3, J-1), J by cofactor expansion
      double C6[6];
      C6[0] = F[0] * F[0] + F[3] * F[3] + F[6] * F[6];
      C6[1] = F[1] * F[1] + F[4] * F[4] + F[7] * F[7];
      C6[2] = F[2] * F[2] + F[5] * F[5] + F[8] * F[8];
      C6[3] = F[0] * F[1] + F[3] * F[4] + F[6] * F[7];
      C6[4] = F[1] * F[2] + F[4] * F[5] + F[7] * F[8];
      C6[5] = F[0] * F[2] + F[3] * F[5] + F[6] * F[8];
      const double I1 = C6[0] + C6[1] + C6[2];
      const double trC2 = C6[0] * C6[0] + C6[1] * C6[1] + C6[2] * C6[2] + 2.0 * (C6[3] * C6[3] + C6[4] * C6[4] + C6[5] * C6[5]);
      const double Jd = F[0] * (F[4] * F[8] - F[5] * F[7]) + F[1] * (F[5] * F[6] - F[3] * F[8]) +
                        F[2] * (F[3] * F[7] - F[4] * F[6]);
      const double k0 = I1 - 3.0, k1 = 0.5 * (I1 * I1 - trC2) - 3.0, k2 = Jd - 1.0;
      if (r == 0) {
        if (e < ne && !(Jd > 0.0)) atomicMin(A.bad, (unsigned long long)(__ldg(A.orig + e0 + e) * NQ + q % NQ));
#pragma unroll
        for (int x = 0; x < 9; x++) qF[q * 9 + x] = F[x];
        qk[q * 3 + 0] = k0;
        qk[q * 3 + 1] = k1;
        qk[q * 3 + 2] = k2;
        gsk[q * 3 + 0] = gsk[q * 3 + 1] = gsk[q * 3 + 2] = 0.0;
      }
#pragma unroll
      for (int it = 0; it < W / TPQ; it++) {
        const int j = r + it * TPQ;
        const double y = __ldg(m.b + j) + __ldg(m.W1 + j * 3 + 0) * k0 + __ldg(m.W1 + j * 3 + 1) * k1 +
                         __ldg(m.W1 + j * 3 + 2) * k2;
        if (L > 1) {
          double z, s;
          softplus_sig(y, tab, z, s);
          sb[j * LDS + q] = s;
          act[j * LDA + q] = z;
        } else {
          const double s = sigmoid_tab(y, tab), aj = __ldg(m.a + j);
          act[j * LDA + q] = aj * s;                  // mu_1
          act[j * LDA + Q + q] = aj * s * (1.0 - s);  // c_1
        }
      }
    }
    __syncthreads();

    // ---- stage 3: value pass, layers 2..L --------------------------------------------
    {
      const int vm = warp / C::VNG, vn = warp % C::VNG;
      const int mt0 = vm * C::MT_V;
      int ncol[C::NT_V];
#pragma unroll
      for (int j = 0; j < C::NT_V; j++) ncol[j] = (vn * C::NT_V + j) * 8;
      for (int l = 2; l <= L; l++) {
        double bias[C::MT_V], aw[C::MT_V];  // issued before the GEMM: L2 latency hidden behind it
#pragma unroll
        for (int i = 0; i < C::MT_V; i++) {
          bias[i] = __ldg(m.b + (l - 1) * W + (mt0 + i) * 8 + g);
          aw[i] = (l == L) ? __ldg(m.a + (mt0 + i) * 8 + g) : 0.0;
        }
        double acc[C::MT_V][C::NT_V][2];
        warp_gemm<C::MT_V, C::NT_V, KT2, KT2>(m.Wfrag + (l - 2) * frag_layer, mt0, act, LDA, ncol, acc);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < C::MT_V; i++) {
          const int j = (mt0 + i) * 8 + g;
          const double bj = bias[i];
          double B3[3] = {0, 0, 0};
          if (skips) {
            const double* Bl = m.skip_h + ((size_t)(l - 2) * W + j) * 3;
            B3[0] = __ldg(Bl); B3[1] = __ldg(Bl + 1); B3[2] = __ldg(Bl + 2);
          }
          const double aj = aw[i];
#pragma unroll
          for (int jj = 0; jj < C::NT_V; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int q = ncol[jj] + 2 * t + h;
              double y = acc[i][jj][h] + bj;
              if (skips) y += B3[0] * qk[q * 3] + B3[1] * qk[q * 3 + 1] + B3[2] * qk[q * 3 + 2];
              if (l < L) {
                double z, s;
                softplus_sig(y, tab, z, s);
                sb[((l - 1) * W + j) * LDS + q] = s;
                act[j * LDA + q] = z;
              } else {  // z_L is not needed (only dN/dz_L = a), so no log
                const double s = sigmoid_tab(y, tab);
                act[j * LDA + q] = aj * s;                                  // mu_L
                cb[((l - 2) * W + j) * LDS + q] = aj * s * (1.0 - s);       // c_L
              }
            }
        }
        __syncthreads();
      }
    }

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
            const double mu = act[j * LDA + tid];
            s0 += __ldg(Bl + j * 3) * mu; s1 += __ldg(Bl + j * 3 + 1) * mu; s2 += __ldg(Bl + j * 3 + 2) * mu;
          }
          gsk[tid * 3] += s0; gsk[tid * 3 + 1] += s1; gsk[tid * 3 + 2] += s2;
        }
        double acc[C::MT_V][C::NT_V][2];
        warp_gemm<C::MT_V, C::NT_V, KT2, KT2>(m.Wfrag + (l - 2) * frag_layer + (size_t)W * W, mt0, act, LDA,
                                              ncol, acc);
        __syncthreads();
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
              const double mu = lam * s, c = mu * (1.0 - s);
              if (l > 2) {
                cb[((l - 3) * W + j) * LDS + q] = c;  // c_{l-1}
                act[j * LDA + q] = mu;                 // mu_{l-1}
              } else {                                 // mu_1, c_1 for stage 5
                act[j * LDA + q] = mu;
                act[j * LDA + Q + q] = c;
              }
            }
        }
        __syncthreads();
      }
    }

    // ---- stage 5: g = W1^T mu_1 (+skips), H_1 = W1^T diag(c_1) W1 --------------------------
    // P consecutive lanes per qp split the sum over j, then reduce with shuffles
    {
      constexpr int P = C::NTHR / Q;
      const int q = tid / P, part = tid % P;
      double gs[3] = {0, 0, 0}, hs[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll 4
      for (int j = part; j < W; j += P) {
        const double w0 = __ldg(m.W1 + j * 3), w1 = __ldg(m.W1 + j * 3 + 1), w2 = __ldg(m.W1 + j * 3 + 2);
        const double mu = act[j * LDA + q], c = act[j * LDA + Q + q];
        gs[0] += w0 * mu; gs[1] += w1 * mu; gs[2] += w2 * mu;
        const double c0 = c * w0, c1 = c * w1;
        hs[0] += c0 * w0; hs[1] += c0 * w1; hs[2] += c0 * w2;
        hs[3] += c1 * w1; hs[4] += c1 * w2; hs[5] += c * w2 * w2;
      }
#pragma unroll
      for (int o = 1; o < P; o <<= 1) {
#pragma unroll
        for (int x = 0; x < 3; x++) gs[x] += __shfl_xor_sync(0xffffffffu, gs[x], o);
#pragma unroll
        for (int x = 0; x < 6; x++) hs[x] += __shfl_xor_sync(0xffffffffu, hs[x], o);
      }
      if (part == 0) {
#pragma unroll
        for (int x = 0; x < 3; x++) qg[q * 3 + x] = gs[x] + gsk[q * 3 + x] + __ldg(m.skip_out + x);
#pragma unroll
        for (int x = 0; x < 6; x++) qH[q * 6 + x] = hs[x];
      }
    }
    __syncthreads();

    // ---- mid-batch: the next batch's conn/lrow have landed -> issue its dependent gathers --
    // (u_e and CSR bases; the loads complete under stages 6-8, stored at the end of the batch)
    Gathered<C> G;
    if (has_next) {
      cp_async_wait_all();
      __syncthreads();
      issue_gathers<C>(A, nne, nin, G);
    }

    // ---- stage 6: Jacobian pass, H += J_l^T diag(c_l) J_l -------------------------------
    if (L > 1) {
      for (int x = tid; x < W * Q; x += C::NTHR) {  // D_1 = s_1 (.) W1
        const int j = x / Q, q = x % Q;
        const double s = sb[j * LDS + q];
#pragma unroll
        for (int c = 0; c < 3; c++) act[j * LDA + c * Q + q] = s * __ldg(m.W1 + j * 3 + c);
      }
      __syncthreads();
      const int jm = warp / C::QB, qb = warp % C::QB;
      const int mt0 = jm * C::MT_J;
      int ncol[3];
#pragma unroll
      for (int c = 0; c < 3; c++) ncol[c] = c * Q + qb * 8;
      double hp[2][6];
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int x = 0; x < 6; x++) hp[h][x] = 0.0;
      for (int l = 2; l <= L; l++) {
        double acc[C::MT_J][3][2];
        warp_gemm<C::MT_J, 3, KT2, KT2>(m.Wfrag + (l - 2) * frag_layer, mt0, act, LDA, ncol, acc);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < C::MT_J; i++) {
          const int j = (mt0 + i) * 8 + g;
          double B3[3] = {0, 0, 0};
          if (skips) {
            const double* Bl = m.skip_h + ((size_t)(l - 2) * W + j) * 3;
            B3[0] = __ldg(Bl); B3[1] = __ldg(Bl + 1); B3[2] = __ldg(Bl + 2);
          }
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int q = qb * 8 + 2 * t + h;
            const double J0 = acc[i][0][h] + B3[0], J1 = acc[i][1][h] + B3[1], J2 = acc[i][2][h] + B3[2];
            const double c = cb[((l - 2) * W + j) * LDS + q];
            const double c0 = c * J0, c1 = c * J1, c2 = c * J2;
            hp[h][0] += c0 * J0; hp[h][1] += c0 * J1; hp[h][2] += c0 * J2;
            hp[h][3] += c1 * J1; hp[h][4] += c1 * J2; hp[h][5] += c2 * J2;
            if (l < L) {
              const double s = sb[((l - 1) * W + j) * LDS + q];
              act[j * LDA + q] = s * J0;
              act[j * LDA + Q + q] = s * J1;
              act[j * LDA + 2 * Q + q] = s * J2;
            }
          }
        }
        __syncthreads();
      }
      // reduce over the 8 row groups g of the warp (lane bits 2..4); act/s/c are dead now
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
      __syncthreads();
    }

    // ---- stage 7: per qp -- penalty, S, T, Phi_m, Psi_m, b, P (all scaled by w) ------------
    if (tid < Q) {
      const int q = tid;
      double gq[3], H6[6];
#pragma unroll
      for (int x = 0; x < 3; x++) gq[x] = qg[q * 3 + x];
#pragma unroll
      for (int x = 0; x < 6; x++) {
        double s = qH[q * 6 + x];
        if (L > 1)
#pragma unroll
          for (int r = 0; r < C::JMG; r++) s += hred[(r * Q + q) * 6 + x];
        H6[x] = s;
      }
      Kin kin;
      kinematics(qF + q * 9, kin);
      gq[2] += 2.0 * m.kappa * (kin.J - 1.0) - m.ref_shift;
      H6[5] += 2.0 * m.kappa;
      post_qp(kin, gq, H6, swq[q], post + q * PS, qP + q * 9);
    }
    __syncthreads();

    // ---- stage 8a: X[q][a][i][kL] = sum_J dN_aJ A_q[iJ][kL] straight from the factors -------
    //   = d_ik t_L + sum_m phi_m,i Psi_m,kL + c2 F_iL p_k + c3 F^-T_iL r_k + c2 dN_aL b_ik
    //   phi_m = Phi_m dN_a, p = F dN_a, r = F^-T dN_a, t = (wT) dN_a
    for (int it = tid; it < Q * NEN; it += C::NTHR) {
      const int q = it / NEN, a = it % NEN;
      const double* P = post + q * PS;
      const double* ga = sgN + (q * NEN + a) * 3;
      const double n0 = ga[0], n1 = ga[1], n2 = ga[2];
      double phi[3][3], pv[3], rv[3], tv[3];
#pragma unroll
      for (int i = 0; i < 3; i++) {
#pragma unroll
        for (int mm = 0; mm < 3; mm++)
          phi[mm][i] = P[27 + mm * 9 + i * 3] * n0 + P[27 + mm * 9 + i * 3 + 1] * n1 + P[27 + mm * 9 + i * 3 + 2] * n2;
        pv[i] = phi[0][i];  // Phi_1 = F
        rv[i] = P[9 + i * 3] * n0 + P[9 + i * 3 + 1] * n1 + P[9 + i * 3 + 2] * n2;
        tv[i] = P[18 + i] * n0 + P[18 + 3 + i] * n1 + P[18 + 6 + i] * n2;
      }
      const double c2 = P[90], c3 = P[91];
      const double nv[3] = {n0, n1, n2};
      double* Xo = Xb + (q * NEN + a) * 27;
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int kk = 0; kk < 3; kk++)
#pragma unroll
          for (int Lx = 0; Lx < 3; Lx++) {
            const int kL = kk * 3 + Lx;
            double v = phi[0][i] * P[54 + kL] + phi[1][i] * P[63 + kL] + phi[2][i] * P[72 + kL];
            v += c2 * P[i * 3 + Lx] * pv[kk] + c3 * P[9 + i * 3 + Lx] * rv[kk] + c2 * nv[Lx] * P[81 + i * 3 + kk];
            if (i == kk) v += tv[Lx];
            Xo[i * 9 + kL] = v;
          }
    }
    __syncthreads();

    // ---- stage 8b: K_e[ai][bk] = sum_q sum_L X dN_bL for node pairs b >= a (K_e = K_e^T), r_e;
    //      coloured RED scatter of both (ai, bk) and its mirror (bk, ai)
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
        // fire-and-forget RED.ADD.F64: the colouring makes the updates conflict-free (and the
        // per-entry summation order deterministic: one update per colour launch)
        const int ea = e * NEN + a, eb = e * NEN + b;
        double* dst = svb[ea] + i * srs[ea] + 3 * (int)sslot[ea * NEN + b];
        atomicAdd(dst, K0);
        atomicAdd(dst + 1, K1);
        atomicAdd(dst + 2, K2);
        if (b == a) {
          atomicAdd(srb[ea] + i, rr);
        } else {
          double* mir = svb[eb] + 3 * (int)sslot[eb * NEN + a] + i;
          const int st = srs[eb];
          atomicAdd(mir, K0);
          atomicAdd(mir + st, K1);
          atomicAdd(mir + 2 * st, K2);
        }
      }
    }
    // the next batch's gathered inputs go to its buffer (made visible by the next stage-0 sync)
    if (has_next) commit_gathers<C>(nne, nin, G);
  }
}

// ---------------------------------------------------------------------------
// host side: dispatch and weight fragments
// ---------------------------------------------------------------------------

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

void fused_gfrag_fill(int w, const double* W1, double* out) {
  const int KT2 = w / 8;
  for (int which = 0; which < 2; which++) {
    double* f = out + (size_t)which * 16 * w;
    for (int mt = 0; mt < 2; mt++)
      for (int kt2 = 0; kt2 < KT2; kt2++)
        for (int lane = 0; lane < 32; lane++)
          for (int h = 0; h < 2; h++) {
            const int g = lane >> 2, t = lane & 3;
            const int r = 8 * mt + g, j = 8 * kt2 + 4 * h + t;
            double v = 0.0;
            if (which == 0 && r < 3) v = W1[j * 3 + r];
            if (which == 1 && r >= 3 && r < 9) {
              static const int pm[6] = {0, 0, 0, 1, 1, 2}, pn[6] = {0, 1, 2, 1, 2, 2};
              v = W1[j * 3 + pm[r - 3]] * W1[j * 3 + pn[r - 3]];
            }
            f[((size_t)(mt * KT2 + kt2) * 32 + lane) * 2 + h] = v;
          }
  }
}

template <class C>
static int launch_cfg(const AsmArgs& a, cudaStream_t st, int* launches) {
  const Smem<C> sm(a.ncm.L);
  const size_t bytes = (size_t)sm.total * sizeof(double);
  static bool attr_set = false;
  static size_t attr_bytes = 0;
  if (!attr_set || attr_bytes < bytes) {
    cudaError_t e = cudaFuncSetAttribute(fused_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
    attr_bytes = bytes;
  }
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<C>, C::NTHR, bytes);
  if (per_sm < 1) per_sm = 1;
  const int64_t nb = (a.el_count + C::E - 1) / C::E;
  const int64_t grid = std::min<int64_t>(nb, (int64_t)sms * per_sm);
  if (grid <= 0) return 0;
  fused_kernel<C><<<(unsigned)grid, C::NTHR, bytes, st>>>(a);
  if (launches) (*launches)++;
  return (int)cudaGetLastError();
}

// COMMET_FUSED_VARIANT=1 (environment, read once): alternative tiling for tuning
// experiments (w = 64: one element per batch, 4 CTAs/SM at <= 128 registers).
static int fused_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("COMMET_FUSED_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <class C>
static void occ_cfg(int L, int* smem_bytes, int* ctas_per_sm, int* regs) {
  const Smem<C> sm(L);
  const size_t bytes = (size_t)sm.total * sizeof(double);
  cudaFuncSetAttribute(fused_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<C>, C::NTHR, bytes);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, fused_kernel<C>);
  *smem_bytes = (int)bytes;
  *ctas_per_sm = per_sm;
  *regs = fa.numRegs;
}

template <int NEN, int NQ>
static void occ_et(int w, int L, int* a, int* b, int* c) {
  switch (w) {
    case 8: occ_cfg<Cfg<8, 32, NEN, NQ>>(L, a, b, c); break;
    case 16: occ_cfg<Cfg<16, 16, NEN, NQ>>(L, a, b, c); break;
    case 32: occ_cfg<Cfg<32, 16, NEN, NQ>>(L, a, b, c); break;
    case 64:
      if (fused_variant() == 1) occ_cfg<Cfg<64, 8, NEN, NQ, 4>>(L, a, b, c);
      else occ_cfg<Cfg<64, 16, NEN, NQ>>(L, a, b, c);
      break;
    case 128: occ_cfg<Cfg<128, 8, NEN, NQ>>(L, a, b, c); break;
  }
}

void fused_occupancy(int n_en, int w, int L, int* smem_bytes, int* ctas_per_sm, int* regs) {
  if (n_en == 8) occ_et<8, 8>(w, L, smem_bytes, ctas_per_sm, regs);
  else occ_et<10, 4>(w, L, smem_bytes, ctas_per_sm, regs);
}

template <int NEN, int NQ>
static int launch_et(const AsmArgs& a, cudaStream_t st, int* launches) {
  switch (a.ncm.w) {
    case 8: return launch_cfg<Cfg<8, 32, NEN, NQ>>(a, st, launches);
    case 16: return launch_cfg<Cfg<16, 16, NEN, NQ>>(a, st, launches);
    case 32: return launch_cfg<Cfg<32, 16, NEN, NQ>>(a, st, launches);
    case 64:
      if (fused_variant() == 1) return launch_cfg<Cfg<64, 8, NEN, NQ, 4>>(a, st, launches);
      return launch_cfg<Cfg<64, 16, NEN, NQ>>(a, st, launches);
    case 128: return launch_cfg<Cfg<128, 8, NEN, NQ>>(a, st, launches);
  }
  return (int)cudaErrorInvalidValue;
}

int launch_fused(const AsmArgs& a, void* stream, int* launches) {
  if (a.el_count <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (a.n_en == 8) return launch_et<8, 8>(a, st, launches);
  return launch_et<10, 4>(a, st, launches);
}

}  // namespace commet
