// solver.cu -- Newton-Raphson around the fused assembly:
//   d <- d + Delta d,  K Delta d = -r                      (s2.1)
// with the linear system solved by conjugate gradients with Jacobi
// preconditioning (s4.2), Dirichlet DOFs eliminated
// symmetrically (rows and columns zeroed, unit diagonal, zero residual), all on
// the GPU.  Single GPU (n_ranks <= 1).
//
// CG kernels (HBM-bound), three launches per iteration k:
//  * update_p (k): from the partials of the previous update, rz_k = r.z and r.r
//    (every block reduces the same partials in the same order: deterministic),
//    the convergence test, beta = rz_k / rz_{k-1}, p = z + beta p.
//  * spmv_dot (k): q = K p and the partials of p.q.  One warp per node-row
//    triple: rows 3a, 3a+1, 3a+2 share their column list (every node pair is a
//    full 3x3 block), so col_idx and the gathered p are read once for three
//    rows: 8 + 4/3 bytes of matrix per nonzero.  (Forming p = z + beta p at the
//    gathered columns instead, to drop update_p, measured slower: two gathered
//    vectors per nonzero through L2.)
//  * update_xr (k): alpha = rz_k / p.q, x += alpha p, r -= alpha q, z = D^-1 r,
//    partials of r.z and r.r.
//  Block 0 of update_p raises the converged flag; every kernel returns at once
//  when it is set, so the host only synchronises every kCheck iterations.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "ctx.h"

namespace {

constexpr int kThreads = 256;
constexpr int kCheck = 32;  // host convergence check interval (iterations)

struct CgScal {
  double rz[2];   // r.z of the current iterate (ping-pong by iteration parity)
  double bb;      // b.b
  double tol2;    // (rtol ||b||)^2
  double rr;      // last r.r
  int done;       // iteration count at convergence (0 = running)
  int it;         // iterations performed
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block reduction of NV values per thread into part[blockIdx.x * NV + k]
template <int NV>
__device__ __forceinline__ void block_partials(double (&v)[NV], double* part) {
  __shared__ double red[kThreads / 32][NV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; k++) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; k++) red[wid][k] = v[k];
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; w++) s += red[w][threadIdx.x];
    part[blockIdx.x * NV + threadIdx.x] = s;
  }
}

// sum of the nb partials part[i*NV + k], same order in every block
template <int NV>
__device__ __forceinline__ void sum_partials(const double* part, int nb, double (&out)[NV]) {
  __shared__ double red[kThreads / 32][NV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; k++) v[k] = 0.0;
  for (int i = threadIdx.x; i < nb; i += kThreads)
#pragma unroll
    for (int k = 0; k < NV; k++) v[k] += part[i * NV + k];
#pragma unroll
  for (int k = 0; k < NV; k++) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; k++) red[wid][k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; k++) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; w++) s += red[w][k];
    out[k] = s;
  }
  __syncthreads();
}

// ---- Dirichlet ---------------------------------------------------------------------------
__global__ void bc_eliminate_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                    double* __restrict__ vals, double* __restrict__ r,
                                    const uint8_t* __restrict__ mask, int64_t n_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n_rows; row += nw) {
    const bool rm = mask[row];
    for (int64_t j = row_ptr[row] + lane; j < row_ptr[row + 1]; j += 32) {
      const int32_t c = col_idx[j];
      if (rm || mask[c]) vals[j] = (c == row) ? 1.0 : 0.0;
    }
    if (lane == 0 && rm && r) r[row] = 0.0;
  }
}

__global__ void scatter_values_kernel(double* __restrict__ u, const int64_t* __restrict__ dofs,
                                      const double* __restrict__ v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    u[dofs[i]] = v[i];
}

__global__ void set_mask_kernel(uint8_t* __restrict__ mask, const int64_t* __restrict__ dofs, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mask[dofs[i]] = 1;
}

// D^-1 (Jacobi); a non-positive diagonal records the lowest such row in *bad (atomicMin)
__global__ void jacobi_diag_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                   const double* __restrict__ vals, double* __restrict__ dinv, int64_t n_rows,
                                   unsigned long long* bad) {
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n_rows;
       row += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = row_ptr[row], hi = row_ptr[row + 1];
    double d = 0.0;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const int32_t c = col_idx[mid];
      if (c == row) { d = vals[mid]; break; }
      if (c < row) lo = mid + 1; else hi = mid;
    }
    if (!(d > 0.0)) atomicMin(bad, (unsigned long long)row);
    dinv[row] = 1.0 / d;
  }
}

// Block Jacobi: the inverse of the 3x3 diagonal block of every node (its own slot in the node
// adjacency), by cofactors; a block that is not SPD (a leading minor <= 0) records the node's
// first row in *bad (atomicMin)
__global__ void block_jacobi_kernel(const int64_t* __restrict__ node_rs, const int32_t* __restrict__ node_deg,
                                    const int32_t* __restrict__ adj, const double* __restrict__ vals,
                                    double* __restrict__ binv, int64_t n_nodes, unsigned long long* bad) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n_nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rs = node_rs[a];
    const int deg = node_deg[a], st = 3 * deg;
    const int32_t* nb = adj + rs / 9;
    int sl = -1;
    for (int t = 0; t < deg; t++)
      if (nb[t] == (int32_t)a) { sl = t; break; }
    double B[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (sl >= 0)
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int k = 0; k < 3; k++) B[i * 3 + k] = vals[rs + i * st + 3 * sl + k];
    double cof[9];
    cof[0] = B[4] * B[8] - B[5] * B[7];
    cof[1] = B[5] * B[6] - B[3] * B[8];
    cof[2] = B[3] * B[7] - B[4] * B[6];
    cof[3] = B[2] * B[7] - B[1] * B[8];
    cof[4] = B[0] * B[8] - B[2] * B[6];
    cof[5] = B[1] * B[6] - B[0] * B[7];
    cof[6] = B[1] * B[5] - B[2] * B[4];
    cof[7] = B[2] * B[3] - B[0] * B[5];
    cof[8] = B[0] * B[4] - B[1] * B[3];
    const double det = B[0] * cof[0] + B[1] * cof[1] + B[2] * cof[2];
    if (!(B[0] > 0.0 && cof[8] > 0.0 && det > 0.0)) atomicMin(bad, (unsigned long long)(3 * a));
    const double id = 1.0 / det;
    // (B^-1)_ik = cof_ki / det
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int k = 0; k < 3; k++) binv[9 * a + i * 3 + k] = cof[k * 3 + i] * id;
  }
}

__device__ __forceinline__ void bj_apply(const double* __restrict__ binv, int64_t a, const double (&r)[3],
                                         double (&z)[3]) {
  const double* Bi = binv + 9 * a;
#pragma unroll
  for (int i = 0; i < 3; i++) z[i] = Bi[3 * i] * r[0] + Bi[3 * i + 1] * r[1] + Bi[3 * i + 2] * r[2];
}

// ---- CG ------------------------------------------------------------------------------------
// init: x = 0, r = b, z = D^-1 b, p = z; partials (r.z, b.b)
__global__ void cg_init_kernel(const double* __restrict__ b, const double* __restrict__ dinv, double* __restrict__ x,
                               double* __restrict__ r, double* __restrict__ z, double* __restrict__ p, int64_t n,
                               double* part) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i], zi = dinv[i] * bi;
    x[i] = 0.0;
    r[i] = bi;
    z[i] = zi;
    p[i] = zi;
    v[0] += bi * zi;
    v[1] += bi * bi;
  }
  block_partials<2>(v, part);
}

// block-Jacobi init: per node, z = B^-1 b
__global__ void cg_init_bj_kernel(const double* __restrict__ b, const double* __restrict__ binv, double* __restrict__ x,
                                  double* __restrict__ r, double* __restrict__ z, double* __restrict__ p,
                                  int64_t n_nodes, double* part) {
  double v[2] = {0.0, 0.0};
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n_nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    double bv[3], zv[3];
#pragma unroll
    for (int i = 0; i < 3; i++) bv[i] = b[3 * a + i];
    bj_apply(binv, a, bv, zv);
#pragma unroll
    for (int i = 0; i < 3; i++) {
      x[3 * a + i] = 0.0;
      r[3 * a + i] = bv[i];
      z[3 * a + i] = zv[i];
      p[3 * a + i] = zv[i];
      v[0] += bv[i] * zv[i];
      v[1] += bv[i] * bv[i];
    }
  }
  block_partials<2>(v, part);
}

__global__ void cg_init_scal_kernel(const double* part, int nb, double rtol, CgScal* s) {
  double t[2];
  sum_partials<2>(part, nb, t);
  if (threadIdx.x == 0) {
    s->rz[0] = t[0];
    s->rz[1] = 0.0;
    s->bb = t[1];
    s->tol2 = rtol * rtol * t[1];
    s->rr = t[1];
    s->it = 0;
    s->done = (t[1] == 0.0) ? -1 : 0;  // b = 0: x = 0 is exact
  }
}

// iteration k, first: rz_k = r.z and r.r from the previous update's partials, the convergence test,
// beta = rz_k / rz_{k-1}, p_k = z + beta p_{k-1} in place (k = 0: p = z)
__global__ void cg_update_p_kernel(double* __restrict__ p, const double* __restrict__ z, int64_t n,
                                   const double* part2, int nb, CgScal* s, int k, int max_iter) {
  if (s->done) return;
  double t[2];
  sum_partials<2>(part2, nb, t);  // (r.z, r.r) of the current residual (k = 0: (r.z, b.b) from init)
  if (t[1] <= s->tol2 || k >= max_iter) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      s->rr = t[1];
      s->it = k;
      s->done = k > 0 ? k : -1;
    }
    return;
  }
  const double beta = k == 0 ? 0.0 : t[0] / s->rz[(k - 1) & 1];
  if (blockIdx.x == 0 && threadIdx.x == 0) s->rz[k & 1] = t[0];  // the other slot from the one read above
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

// q = K p by node blocks: the row triple of node a is deg(a) 3x3 blocks, block s at
// node_rs[a] + 3 s (+ 3 deg(a) per row), its column node from the node adjacency (one int32 per
// block instead of nine col_idx entries: 8 + 4/9 bytes per nonzero); a lane per neighbour node
// reads 3 consecutive values of each row and 3 consecutive entries of p.  Single GPU: node_rs[a]
// = 9 x (the adjacency offset of a).
__global__ void cg_spmv_dot_nb_kernel(const int64_t* __restrict__ node_rs, const int32_t* __restrict__ node_deg,
                                      const int32_t* __restrict__ adj, const double* __restrict__ vals,
                                      const double* __restrict__ p, double* __restrict__ q, int64_t n_nodes,
                                      double* part, const CgScal* s) {
  if (s->done) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const int64_t chunk = (n_nodes + gridDim.x - 1) / gridDim.x;
  const int64_t a_end = min(n_nodes, (int64_t)(blockIdx.x + 1) * chunk);
  double v[1] = {0.0};
  for (int64_t a = (int64_t)blockIdx.x * chunk + wid; a < a_end; a += nwb) {
    const int64_t rs = __ldg(node_rs + a);
    const int deg = __ldg(node_deg + a), st = 3 * deg;
    const int32_t* nb = adj + rs / 9;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int sl = lane; sl < deg; sl += 32) {
      const int64_t b = __ldcs(nb + sl);
      const double p0 = __ldg(p + 3 * b), p1 = __ldg(p + 3 * b + 1), p2 = __ldg(p + 3 * b + 2);
      const double* v0 = vals + rs + 3 * sl;
      s0 = fma(__ldcs(v0), p0, fma(__ldcs(v0 + 1), p1, fma(__ldcs(v0 + 2), p2, s0)));
      s1 = fma(__ldcs(v0 + st), p0, fma(__ldcs(v0 + st + 1), p1, fma(__ldcs(v0 + st + 2), p2, s1)));
      s2 = fma(__ldcs(v0 + 2 * st), p0, fma(__ldcs(v0 + 2 * st + 1), p1, fma(__ldcs(v0 + 2 * st + 2), p2, s2)));
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      q[3 * a] = s0;
      q[3 * a + 1] = s1;
      q[3 * a + 2] = s2;
      v[0] += p[3 * a] * s0 + p[3 * a + 1] * s1 + p[3 * a + 2] * s2;
    }
  }
  block_partials<1>(v, part);
}

// q = K p, partials of p.q (scalar CSR: the column list, kept for reference).  A contiguous node range per block (neighbouring nodes share most of
// their stencil columns: the p gathers hit L1); the matrix streams with evict-first loads, all
// lane loads of a row triple issued before the FMAs
__global__ void cg_spmv_dot_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                   const double* __restrict__ vals, const double* __restrict__ p,
                                   double* __restrict__ q, int64_t n_nodes, double* part, const CgScal* s) {
  if (s->done) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const int64_t chunk = (n_nodes + gridDim.x - 1) / gridDim.x;
  const int64_t a_end = min(n_nodes, (int64_t)(blockIdx.x + 1) * chunk);
  double v[1] = {0.0};
  for (int64_t a = (int64_t)blockIdx.x * chunk + wid; a < a_end; a += nwb) {
    const int64_t r0 = row_ptr[3 * a], r1 = row_ptr[3 * a + 1], r2 = row_ptr[3 * a + 2];
    const int64_t len = r1 - r0;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int64_t j0 = 0; j0 < len; j0 += 96) {  // up to three lane passes with their loads in flight
      int32_t c[3];
      double v0[3], v1[3], v2[3];
#pragma unroll
      for (int u = 0; u < 3; u++) {
        const int64_t j = j0 + u * 32 + lane;
        const bool in = j < len;
        c[u] = in ? __ldcs(col_idx + r0 + j) : 0;
        v0[u] = in ? __ldcs(vals + r0 + j) : 0.0;
        v1[u] = in ? __ldcs(vals + r1 + j) : 0.0;
        v2[u] = in ? __ldcs(vals + r2 + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 3; u++) {
        const double pv = __ldg(p + c[u]);
        s0 = fma(v0[u], pv, s0);
        s1 = fma(v1[u], pv, s1);
        s2 = fma(v2[u], pv, s2);
      }
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      q[3 * a] = s0;
      q[3 * a + 1] = s1;
      q[3 * a + 2] = s2;
      v[0] += p[3 * a] * s0 + p[3 * a + 1] * s1 + p[3 * a + 2] * s2;
    }
  }
  block_partials<1>(v, part);
}

__global__ void cg_update_xr_kernel(double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                                    const double* __restrict__ p, const double* __restrict__ q,
                                    const double* __restrict__ dinv, int64_t n, const double* part_pq, int nb,
                                    double* part, const CgScal* s, int it) {
  if (s->done) return;
  double pq[1];
  sum_partials<1>(part_pq, nb, pq);
  const double alpha = s->rz[it & 1] / pq[0];
  double v[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    const double zi = dinv[i] * ri;
    z[i] = zi;
    v[0] += ri * zi;
    v[1] += ri * ri;
  }
  block_partials<2>(v, part);
}

// block-Jacobi update: per node, x += alpha p, r -= alpha q, z = B^-1 r; partials (r.z, r.r)
__global__ void cg_update_xr_bj_kernel(double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                                       const double* __restrict__ p, const double* __restrict__ q,
                                       const double* __restrict__ binv, int64_t n_nodes, const double* part_pq,
                                       int nb, double* part, const CgScal* s, int it) {
  if (s->done) return;
  double pq[1];
  sum_partials<1>(part_pq, nb, pq);
  const double alpha = s->rz[it & 1] / pq[0];
  double v[2] = {0.0, 0.0};
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n_nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    double rv[3], zv[3];
#pragma unroll
    for (int i = 0; i < 3; i++) {
      const int64_t j = 3 * a + i;
      x[j] = fma(alpha, p[j], x[j]);
      rv[i] = fma(-alpha, q[j], r[j]);
      r[j] = rv[i];
    }
    bj_apply(binv, a, rv, zv);
#pragma unroll
    for (int i = 0; i < 3; i++) {
      z[3 * a + i] = zv[i];
      v[0] += rv[i] * zv[i];
      v[1] += rv[i] * rv[i];
    }
  }
  block_partials<2>(v, part);
}

// increment of the constrained dofs: d = 0, d[dofs] = v - u[dofs]
__global__ void bc_increment_kernel(double* __restrict__ d, const double* __restrict__ u,
                                    const int64_t* __restrict__ dofs, const double* __restrict__ v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[dofs[i]] = v[i] - u[dofs[i]];
}

// y += K x (node-row triples, as cg_spmv_dot_kernel)
__global__ void spmv_add_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                const double* __restrict__ vals, const double* __restrict__ x,
                                double* __restrict__ y, int64_t n_nodes) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < n_nodes; a += nw) {
    const int64_t r0 = row_ptr[3 * a], r1 = row_ptr[3 * a + 1], r2 = row_ptr[3 * a + 2];
    const int64_t len = r1 - r0;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int64_t j = lane; j < len; j += 32) {
      const double xv = __ldg(x + __ldg(col_idx + r0 + j));
      s0 = fma(__ldg(vals + r0 + j), xv, s0);
      s1 = fma(__ldg(vals + r1 + j), xv, s1);
      s2 = fma(__ldg(vals + r2 + j), xv, s2);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      y[3 * a] += s0;
      y[3 * a + 1] += s1;
      y[3 * a + 2] += s2;
    }
  }
}

__global__ void axpy_kernel(double* __restrict__ y, double a, const double* __restrict__ x, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* part) {
  double v[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[0] += a[i] * b[i];
  block_partials<1>(v, part);
}

__global__ void sum_kernel(const double* part, int nb, double* out) {
  double t[1];
  sum_partials<1>(part, nb, t);
  if (threadIdx.x == 0) *out = t[0];
}

}  // namespace

struct SolverWork {
  int64_t n_bc = 0;
  std::vector<int64_t> bc_host;
  DevBuf<int64_t> bc_dofs;
  DevBuf<uint8_t> mask;
  DevBuf<double> bc_vals;
  DevBuf<double> r, vals, dinv, x, cr, z, p, q, part, part2, dotv;
  DevBuf<double> binv;  // block Jacobi: [n_nodes][3][3]
  DevBuf<int32_t> adj;  // node adjacency (column node of every 3x3 block), node order
  DevBuf<CgScal> scal;
  DevBuf<unsigned long long> bad;
  int nb = 0;
  cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
  ~SolverWork() {
    for (auto ev : e)
      if (ev) cudaEventDestroy(ev);
  }
};

void solver_work_free(SolverWork* w) { delete w; }

static commet_status work(commet_ctx c, SolverWork** out) {
  if (!c->solver) {
    c->solver = new (std::nothrow) SolverWork();
    if (!c->solver) return fail(c, COMMET_ERR_OOM, "host allocation failed");
  }
  SolverWork* w = c->solver;
  const Plan& p = c->plan;
  if (!w->dinv.p) {
    const int64_t n = 3 * p.n_owned;
    int dev = 0, sms = 148;
    CUDA_TRY(c, cudaGetDevice(&dev));
    CUDA_TRY(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    w->nb = sms * 8;  // 8 blocks of 256 per SM (the spmv is a grid-stride warp-per-node loop)
    CUDA_TRY(c, w->dinv.alloc(n));
    CUDA_TRY(c, w->cr.alloc(n));
    CUDA_TRY(c, w->z.alloc(n));
    CUDA_TRY(c, w->p.alloc(n));
    {
      std::vector<int32_t> adj(p.adj.nbr.size());
      for (size_t x = 0; x < adj.size(); x++) adj[x] = (int32_t)p.adj.nbr[x];
      CUDA_TRY(c, w->adj.alloc(std::max<size_t>(adj.size(), 1)));
      if (!adj.empty()) CUDA_TRY(c, cudaMemcpy(w->adj.p, adj.data(), adj.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    CUDA_TRY(c, w->q.alloc(n));
    CUDA_TRY(c, w->part.alloc(2 * (size_t)w->nb));
    CUDA_TRY(c, w->part2.alloc(2 * (size_t)w->nb));
    CUDA_TRY(c, w->dotv.alloc(1));
    CUDA_TRY(c, w->scal.alloc(1));
    CUDA_TRY(c, w->bad.alloc(1));
    for (auto& ev : w->e) CUDA_TRY(c, cudaEventCreate(&ev));
  }
  *out = w;
  return COMMET_OK;
}

static bool single_gpu(commet_ctx c) { return c->plan.n_ranks <= 1; }

extern "C" commet_status commet_set_dirichlet(commet_ctx c, const int64_t* dofs, int64_t n) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (!single_gpu(c)) return fail(c, COMMET_ERR_ARG, "Newton/CG calls support a single GPU (n_ranks <= 1)");
  if (n < 0 || (n > 0 && !dofs)) return fail(c, COMMET_ERR_ARG, "dofs NULL or n = %lld < 0", (long long)n);
  const int64_t nd = 3 * c->plan.n_nodes;
  for (int64_t i = 0; i < n; i++)
    if (dofs[i] < 0 || dofs[i] >= nd)
      return fail(c, COMMET_ERR_ARG, "dirichlet dof %lld at position %lld outside [0, %lld)", (long long)dofs[i],
                  (long long)i, (long long)nd);
  SolverWork* w;
  commet_status s = work(c, &w);
  if (s != COMMET_OK) return s;
  CUDA_TRY(c, cudaSetDevice(c->device));
  w->n_bc = n;
  w->bc_host.assign(dofs, dofs + n);
  CUDA_TRY(c, w->mask.alloc(nd));
  CUDA_TRY(c, cudaMemset(w->mask.p, 0, nd));
  CUDA_TRY(c, w->bc_dofs.alloc(std::max<int64_t>(n, 1)));
  CUDA_TRY(c, w->bc_vals.alloc(std::max<int64_t>(n, 1)));
  if (n) {
    CUDA_TRY(c, cudaMemcpy(w->bc_dofs.p, dofs, n * sizeof(int64_t), cudaMemcpyHostToDevice));
    set_mask_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256>>>(w->mask.p, w->bc_dofs.p, n);
    CUDA_TRY(c, cudaGetLastError());
  }
  CUDA_TRY(c, cudaDeviceSynchronize());
  return COMMET_OK;
}

static commet_status eliminate(commet_ctx c, SolverWork* w, double* r, double* vals, cudaStream_t st) {
  const Plan& p = c->plan;
  const int64_t n_rows = 3 * p.n_owned;
  if (!w->mask.p) return fail(c, COMMET_ERR_ARG, "commet_set_dirichlet has not been called");
  bc_eliminate_kernel<<<w->nb, kThreads, 0, st>>>(c->row_ptr.p, c->col_idx.p, vals, r, w->mask.p, n_rows);
  CUDA_TRY(c, cudaGetLastError());
  return COMMET_OK;
}

extern "C" commet_status commet_apply_dirichlet(commet_ctx c, double* residual, double* csr_values,
                                                void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (!single_gpu(c)) return fail(c, COMMET_ERR_ARG, "Newton/CG calls support a single GPU (n_ranks <= 1)");
  if (!csr_values) return fail(c, COMMET_ERR_ARG, "csr_values is NULL");
  SolverWork* w;
  commet_status s = work(c, &w);
  if (s != COMMET_OK) return s;
  CUDA_TRY(c, cudaSetDevice(c->device));
  return eliminate(c, w, residual, csr_values, (cudaStream_t)cuda_stream);
}

// CG-Jacobi on the ctx pattern: K x = b from x = 0; synchronous.
static commet_status cg(commet_ctx c, SolverWork* w, const double* vals, const double* b, double* x, double rtol,
                        int max_iter, int* iters, double* rel_res, cudaStream_t st) {
  const Plan& p = c->plan;
  const int64_t n = 3 * p.n_owned, n_nodes = p.n_owned;
  const int nb = w->nb;
  const bool bj = c->precond == COMMET_PC_BLOCK_JACOBI;
  if (bj && !w->binv.p) CUDA_TRY(c, w->binv.alloc(9 * (size_t)std::max<int64_t>(n_nodes, 1)));
  CUDA_TRY(c, cudaMemsetAsync(w->bad.p, 0xff, sizeof(unsigned long long), st));
  if (bj) {
    block_jacobi_kernel<<<nb, kThreads, 0, st>>>(c->node_rs.p, c->node_deg.p, w->adj.p, vals, w->binv.p, n_nodes,
                                                 w->bad.p);
    cg_init_bj_kernel<<<nb, kThreads, 0, st>>>(b, w->binv.p, x, w->cr.p, w->z.p, w->p.p, n_nodes, w->part2.p);
  } else {
    jacobi_diag_kernel<<<nb, kThreads, 0, st>>>(c->row_ptr.p, c->col_idx.p, vals, w->dinv.p, n, w->bad.p);
    cg_init_kernel<<<nb, kThreads, 0, st>>>(b, w->dinv.p, x, w->cr.p, w->z.p, w->p.p, n, w->part2.p);
  }
  cg_init_scal_kernel<<<1, kThreads, 0, st>>>(w->part2.p, nb, rtol, w->scal.p);
  CUDA_TRY(c, cudaGetLastError());
  unsigned long long bad = ~0ULL;
  CUDA_TRY(c, cudaMemcpyAsync(&bad, w->bad.p, sizeof bad, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  if (bad != ~0ULL)
    return fail(c, COMMET_ERR_DOMAIN, bj ? "CG-Jacobi: the 3x3 diagonal block at row %llu is not positive definite"
                                         : "CG-Jacobi: diagonal entry of row %llu is not positive", bad);
  CgScal hs{};
  for (int it0 = 0; it0 <= max_iter; it0 += kCheck) {
    const int nk = std::min(kCheck, max_iter + 1 - it0);
    for (int kk = 0; kk < nk; kk++) {
      const int k = it0 + kk;
      cg_update_p_kernel<<<nb, kThreads, 0, st>>>(w->p.p, w->z.p, n, w->part2.p, nb, w->scal.p, k, max_iter);
      cg_spmv_dot_nb_kernel<<<nb, kThreads, 0, st>>>(c->node_rs.p, c->node_deg.p, w->adj.p, vals, w->p.p, w->q.p,
                                                     n_nodes, w->part.p, w->scal.p);
      if (bj)
        cg_update_xr_bj_kernel<<<nb, kThreads, 0, st>>>(x, w->cr.p, w->z.p, w->p.p, w->q.p, w->binv.p, n_nodes,
                                                        w->part.p, nb, w->part2.p, w->scal.p, k);
      else
        cg_update_xr_kernel<<<nb, kThreads, 0, st>>>(x, w->cr.p, w->z.p, w->p.p, w->q.p, w->dinv.p, n, w->part.p, nb,
                                                     w->part2.p, w->scal.p, k);
    }
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemcpyAsync(&hs, w->scal.p, sizeof hs, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    if (hs.done) break;
  }
  if (iters) *iters = hs.it;
  const double rr = hs.rr;
  if (rel_res) *rel_res = hs.bb > 0.0 ? std::sqrt(rr / hs.bb) : 0.0;
  if (!(rr <= hs.tol2))
    return fail(c, COMMET_ERR_DOMAIN, "CG-Jacobi did not reach rtol %.3g in %d iterations (rel. residual %.3g)", rtol,
                max_iter, hs.bb > 0 ? std::sqrt(rr / hs.bb) : 0.0);
  return COMMET_OK;
}

extern "C" commet_status commet_set_preconditioner(commet_ctx c, int32_t kind) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (kind != COMMET_PC_JACOBI && kind != COMMET_PC_BLOCK_JACOBI)
    return fail(c, COMMET_ERR_ARG, "preconditioner %d unknown", kind);
  c->precond = kind;
  return COMMET_OK;
}

extern "C" commet_status commet_cg_jacobi(commet_ctx c, const double* csr_values, const double* b, double* x,
                                          double rtol, int32_t max_iter, int32_t* iters, double* rel_res,
                                          void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (!single_gpu(c)) return fail(c, COMMET_ERR_ARG, "Newton/CG calls support a single GPU (n_ranks <= 1)");
  if (!csr_values || !b || !x) return fail(c, COMMET_ERR_ARG, "csr_values, b or x is NULL");
  if (!(rtol > 0.0 && rtol < 1.0) || max_iter < 1)
    return fail(c, COMMET_ERR_ARG, "rtol %.3g not in (0,1) or max_iter %d < 1", rtol, max_iter);
  SolverWork* w;
  commet_status s = work(c, &w);
  if (s != COMMET_OK) return s;
  CUDA_TRY(c, cudaSetDevice(c->device));
  int it = 0;
  s = cg(c, w, csr_values, b, x, rtol, max_iter, &it, rel_res, (cudaStream_t)cuda_stream);
  if (iters) *iters = it;
  return s;
}

static commet_status norm2(commet_ctx c, SolverWork* w, const double* v, int64_t n, double* out, cudaStream_t st) {
  dot_kernel<<<w->nb, kThreads, 0, st>>>(v, v, n, w->part.p);
  sum_kernel<<<1, kThreads, 0, st>>>(w->part.p, w->nb, w->dotv.p);
  CUDA_TRY(c, cudaGetLastError());
  double h = 0.0;
  CUDA_TRY(c, cudaMemcpyAsync(&h, w->dotv.p, sizeof h, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  *out = std::sqrt(h);
  return COMMET_OK;
}

extern "C" commet_status commet_newton_step(commet_ctx c, const double* bc_values, const commet_newton_cfg* cfg,
                                            double* u, commet_newton_report* rep, void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (!single_gpu(c)) return fail(c, COMMET_ERR_ARG, "Newton/CG calls support a single GPU (n_ranks <= 1)");
  if (!cfg || !u || !rep) return fail(c, COMMET_ERR_ARG, "cfg, u or report is NULL");
  if (cfg->max_iter < 1 || cfg->max_iter > COMMET_NEWTON_MAX_LOG - 1 || !(cfg->atol >= 0.0) || !(cfg->rtol >= 0.0))
    return fail(c, COMMET_ERR_ARG, "newton cfg: max_iter %d not in 1..%d or negative tolerance", cfg->max_iter,
                COMMET_NEWTON_MAX_LOG - 1);
  SolverWork* w;
  commet_status s = work(c, &w);
  if (s != COMMET_OK) return s;
  if (!w->mask.p) return fail(c, COMMET_ERR_ARG, "commet_set_dirichlet has not been called");
  if (w->n_bc && !bc_values) return fail(c, COMMET_ERR_ARG, "bc_values is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const Plan& p = c->plan;
  const int64_t n = 3 * p.n_owned;
  if (!w->r.p) {
    CUDA_TRY(c, w->r.alloc(n));
    CUDA_TRY(c, w->vals.alloc(p.nnz));
    CUDA_TRY(c, w->x.alloc(n));
  }
  std::memset(rep, 0, sizeof *rep);
  const unsigned nbc_blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((w->n_bc + 255) / 256, 4096));
  if (w->n_bc) {
    // prescribed increment dc (x doubles as its buffer until the first solve)
    CUDA_TRY(c, cudaMemcpyAsync(w->bc_vals.p, bc_values, w->n_bc * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemsetAsync(w->x.p, 0, n * sizeof(double), st));
    bc_increment_kernel<<<nbc_blocks, 256, 0, st>>>(w->x.p, u, w->bc_dofs.p, w->bc_vals.p, w->n_bc);
    CUDA_TRY(c, cudaGetLastError());
  }
  double nrm0 = 0.0;
  float ms = 0.0f;
  for (int it = 0;; it++) {
    CUDA_TRY(c, cudaEventRecord(w->e[0], st));
    s = commet_assemble(c, u, w->r.p, w->vals.p, st);
    if (s != COMMET_OK) return s;
    if (it == 0 && w->n_bc) {
      // consistent predictor (R20): K and r at the previous u, the prescribed
      // increment on the right-hand side, K_ff du_f = (r + K dc)_f; then u[dofs] = values
      spmv_add_kernel<<<w->nb, kThreads, 0, st>>>(c->row_ptr.p, c->col_idx.p, w->vals.p, w->x.p, w->r.p, p.n_owned);
      scatter_values_kernel<<<nbc_blocks, 256, 0, st>>>(u, w->bc_dofs.p, w->bc_vals.p, w->n_bc);
      CUDA_TRY(c, cudaGetLastError());
    }
    s = eliminate(c, w, w->r.p, w->vals.p, st);
    if (s != COMMET_OK) return s;
    CUDA_TRY(c, cudaEventRecord(w->e[1], st));
    int64_t badqp = -1;
    s = commet_check(c, &badqp);
    if (s != COMMET_OK) return s;
    CUDA_TRY(c, cudaEventElapsedTime(&ms, w->e[0], w->e[1]));
    rep->ms_assemble += ms;
    rep->n_assemble++;
    double nrm = 0.0;
    s = norm2(c, w, w->r.p, n, &nrm, st);
    if (s != COMMET_OK) return s;
    rep->res_norm[it] = nrm;
    rep->iters = it;
    if (it == 0) nrm0 = nrm;
    if (nrm <= std::max(cfg->atol, cfg->rtol * nrm0)) {
      rep->converged = 1;
      break;
    }
    if (it >= cfg->max_iter) break;
    // K du = r  ->  u -= du   (du = 0 on constrained dofs: unit rows, zero residual)
    CUDA_TRY(c, cudaEventRecord(w->e[2], st));
    int cit = 0;
    double rel = 0.0;
    s = cg(c, w, w->vals.p, w->r.p, w->x.p, cfg->cg_rtol, cfg->cg_max_iter, &cit, &rel, st);
    rep->cg_iters[it] = cit;
    rep->cg_iters_total += cit;
    if (s != COMMET_OK) return s;
    axpy_kernel<<<w->nb, kThreads, 0, st>>>(u, -1.0, w->x.p, n);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaEventRecord(w->e[3], st));
    CUDA_TRY(c, cudaEventSynchronize(w->e[3]));
    CUDA_TRY(c, cudaEventElapsedTime(&ms, w->e[2], w->e[3]));
    rep->ms_solve += ms;
  }
  s = commet_max_trace_C(c, &rep->max_trC);
  return s;
}
