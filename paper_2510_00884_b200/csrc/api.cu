// api.cu -- the C ABI of libcommet (include/commet.h): setup (validation,
// CSR pattern, element colouring, scatter slots, device uploads) and the
// assemble orchestration (zeroing, one fused launch per colour, interface
// exchange over NCCL for multi-GPU slabs).
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "commet.h"
#include "commet_internal.h"

using namespace commet;

namespace {

thread_local std::string g_last_error;

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t count) {
    n = count;
    return count ? cudaMalloc(&p, count * sizeof(T)) : cudaSuccess;
  }
};

}  // namespace

struct commet_ctx_s {
  int device = 0;
  int elem_type = 0, n_en = 0, n_q = 0;
  int64_t n_nodes = 0, n_el = 0, node_begin = 0, node_end = 0, n_owned = 0, n_halo = 0;
  int64_t n_rows = 0, nnz = 0, nnz_halo = 0;
  int n_colours = 0;
  std::vector<int64_t> colour_start;
  int kernel = COMMET_KERNEL_FUSED;
  std::string err;
  cudaStream_t last_stream = nullptr;
  // device data
  DevBuf<int32_t> conn, lrow, col_idx;
  DevBuf<double> gradN, qp_w;
  DevBuf<uint8_t> slot;
  DevBuf<int64_t> orig, node_rs, row_ptr;
  DevBuf<int32_t> node_deg;
  DevBuf<double> W1, b, a, skip_out, skip_h, Wrow, Wfrag;
  DevBuf<double> r_halo, v_halo;
  DevBuf<unsigned long long> bad;
  NcmDev ncm{};
  // timing ring
  std::vector<cudaEvent_t> ev0, ev1;
  int64_t n_assembled = 0;
  ~commet_ctx_s() {
    for (auto e : ev0) cudaEventDestroy(e);
    for (auto e : ev1) cudaEventDestroy(e);
  }
};

static commet_status fail(commet_ctx c, commet_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  g_last_error = buf;
  return s;
}

#define CUDA_TRY(ctx, x)                                                                     \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? COMMET_ERR_OOM : COMMET_ERR_CUDA,    \
                  "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), __FILE__, __LINE__, #x); \
  } while (0)

template <class T>
static commet_status upload(commet_ctx c, DevBuf<T>& d, const T* h, size_t n, cudaStream_t st) {
  CUDA_TRY(c, d.alloc(n));
  if (n) CUDA_TRY(c, cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
  return COMMET_OK;
}

// ---------------------------------------------------------------------------
// pattern: per local row-node, sorted unique neighbour nodes
// ---------------------------------------------------------------------------
struct Adjacency {
  std::vector<int64_t> ptr;   // [n_rownodes+1]
  std::vector<int64_t> nbr;   // global node ids
};

// rows: local row-node of (e, a) ; neighbours: all nodes of e.
static void build_adjacency(int64_t n_rownodes, int64_t n_el, int n_en, const int32_t* conn,
                            const std::vector<int32_t>& lrow, Adjacency& adj) {
  // incidence lists rownode -> elements (counting sort)
  std::vector<int64_t> cnt(n_rownodes + 1, 0);
  for (int64_t x = 0; x < n_el * n_en; x++) cnt[lrow[x] + 1]++;
  for (int64_t v = 0; v < n_rownodes; v++) cnt[v + 1] += cnt[v];
  std::vector<int64_t> inc(cnt[n_rownodes]);
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t x = 0; x < n_el * n_en; x++) inc[pos[lrow[x]]++] = x / n_en;
  }
  adj.ptr.assign(n_rownodes + 1, 0);
  // two passes (count, fill) with a per-thread scratch vector
#pragma omp parallel
  {
    std::vector<int64_t> tmp;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n_rownodes; v++) {
      tmp.clear();
      for (int64_t p = cnt[v]; p < cnt[v + 1]; p++)
        for (int b = 0; b < n_en; b++) tmp.push_back(conn[inc[p] * n_en + b]);
      std::sort(tmp.begin(), tmp.end());
      adj.ptr[v + 1] = std::unique(tmp.begin(), tmp.end()) - tmp.begin();
    }
  }
  for (int64_t v = 0; v < n_rownodes; v++) adj.ptr[v + 1] += adj.ptr[v];
  adj.nbr.resize(adj.ptr[n_rownodes]);
#pragma omp parallel
  {
    std::vector<int64_t> tmp;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n_rownodes; v++) {
      tmp.clear();
      for (int64_t p = cnt[v]; p < cnt[v + 1]; p++)
        for (int b = 0; b < n_en; b++) tmp.push_back(conn[inc[p] * n_en + b]);
      std::sort(tmp.begin(), tmp.end());
      auto end = std::unique(tmp.begin(), tmp.end());
      std::copy(tmp.begin(), end, adj.nbr.begin() + adj.ptr[v]);
    }
  }
}

// ---------------------------------------------------------------------------
extern "C" commet_status commet_setup(const commet_mesh_desc* mesh, const commet_ncm_desc* ncm,
                                      int device, void* cuda_stream, void* nccl_comm,
                                      commet_ctx* out) {
  if (!out) return fail(nullptr, COMMET_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (!mesh || !ncm) return fail(nullptr, COMMET_ERR_ARG, "mesh or ncm descriptor is NULL");
  std::unique_ptr<commet_ctx_s> c(new (std::nothrow) commet_ctx_s());
  if (!c) return fail(nullptr, COMMET_ERR_OOM, "host allocation failed");
  commet_ctx C = c.get();
  if (mesh->elem_type == COMMET_HEX8) { c->n_en = 8; c->n_q = 8; }
  else if (mesh->elem_type == COMMET_TET10) { c->n_en = 10; c->n_q = 4; }
  else return fail(C, COMMET_ERR_ARG, "elem_type %d unknown", mesh->elem_type);
  c->elem_type = mesh->elem_type;
  const int n_en = c->n_en, n_q = c->n_q;
  if (mesh->n_nodes <= 0 || mesh->n_nodes > ((int64_t)1 << 31) / 3)
    return fail(C, COMMET_ERR_ARG, "n_nodes %lld out of range (1 .. 2^31/3)", (long long)mesh->n_nodes);
  if (mesh->n_elems < 0) return fail(C, COMMET_ERR_ARG, "n_elems %lld < 0", (long long)mesh->n_elems);
  if (mesh->n_elems > 0 && (!mesh->conn || !mesh->grad_N || !mesh->qp_w))
    return fail(C, COMMET_ERR_ARG, "conn, grad_N or qp_w is NULL");
  if (mesh->owned_node_begin < 0 || mesh->owned_node_end > mesh->n_nodes ||
      mesh->owned_node_begin > mesh->owned_node_end)
    return fail(C, COMMET_ERR_ARG, "owned node range [%lld, %lld) invalid for n_nodes %lld",
                (long long)mesh->owned_node_begin, (long long)mesh->owned_node_end, (long long)mesh->n_nodes);
  const int L = ncm->n_hidden, w = ncm->width;
  if (L < 1 || L > kMaxLayers) return fail(C, COMMET_ERR_ARG, "n_hidden %d not in 1..%d", L, kMaxLayers);
  if (!fused_supported(n_en, n_q, w, L))
    return fail(C, COMMET_ERR_ARG, "width %d unsupported (8, 16, 32, 64 or 128)", w);
  if (!ncm->W1 || !ncm->b || !ncm->a || (L > 1 && !ncm->W))
    return fail(C, COMMET_ERR_ARG, "NCM weight pointer NULL (W1, b, a or W)");
  c->n_nodes = mesh->n_nodes;
  c->n_el = mesh->n_elems;
  c->node_begin = mesh->owned_node_begin;
  c->node_end = mesh->owned_node_end;
  c->n_owned = c->node_end - c->node_begin;
  c->device = device;
  const int64_t n_el = c->n_el;
  const int32_t* conn = mesh->conn;
  // ---- validation (host only, before any CUDA call) ----------------------------------
  for (int64_t x = 0; x < n_el * n_en; x++)
    if (conn[x] < 0 || conn[x] >= c->n_nodes)
      return fail(C, COMMET_ERR_ARG, "conn[%lld][%d] = %d out of range [0, %lld)", (long long)(x / n_en),
                  (int)(x % n_en), conn[x], (long long)c->n_nodes);
  for (int64_t x = 0; x < n_el * n_q; x++)
    if (!(mesh->qp_w[x] > 0.0))
      return fail(C, COMMET_ERR_ARG, "qp_w[%lld][%d] = %g is not > 0", (long long)(x / n_q), (int)(x % n_q),
                  mesh->qp_w[x]);

  // ---- local row-nodes: owned [begin,end) then halo (sorted global ids) -----------------
  std::vector<int64_t> halo;
  for (int64_t x = 0; x < n_el * n_en; x++)
    if (conn[x] < c->node_begin || conn[x] >= c->node_end) halo.push_back(conn[x]);
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  c->n_halo = (int64_t)halo.size();
  if (c->n_halo)
    return fail(C, COMMET_ERR_ARG, "%lld nodes referenced by conn are outside the owned range "
                "(first: node %lld); multi-rank partitions need the NCCL path", (long long)c->n_halo, (long long)halo[0]);
  (void)nccl_comm;
  CUDA_TRY(C, cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int64_t n_rn = c->n_owned + c->n_halo;
  std::vector<int32_t> lrow(n_el * n_en);
#pragma omp parallel for
  for (int64_t x = 0; x < n_el * n_en; x++) {
    int64_t v = conn[x];
    lrow[x] = (v >= c->node_begin && v < c->node_end)
                  ? (int32_t)(v - c->node_begin)
                  : (int32_t)(c->n_owned + (std::lower_bound(halo.begin(), halo.end(), v) - halo.begin()));
  }

  // ---- adjacency of local rows; multi-GPU: merge neighbours' halo rows into owned rows --
  Adjacency adj;
  build_adjacency(n_rn, n_el, n_en, conn, lrow, adj);
  for (int64_t v = 0; v < n_rn; v++)
    if (adj.ptr[v + 1] - adj.ptr[v] > 255)
      return fail(C, COMMET_ERR_ARG, "node row %lld has %lld neighbours (> 255)", (long long)v,
                  (long long)(adj.ptr[v + 1] - adj.ptr[v]));

  // ---- CSR of owned rows + halo rows ----------------------------------------------------
  std::vector<int64_t> node_rs(n_rn);
  std::vector<int32_t> node_deg(n_rn);
  int64_t off = 0;
  for (int64_t v = 0; v < n_rn; v++) {
    if (v == c->n_owned) { c->nnz = off; off = 0; }
    node_rs[v] = off;
    node_deg[v] = (int32_t)(adj.ptr[v + 1] - adj.ptr[v]);
    off += 9 * (int64_t)node_deg[v];
  }
  if (c->n_halo == 0) c->nnz = off; else c->nnz_halo = off;
  if (n_rn == c->n_owned) c->nnz = off;
  c->n_rows = 3 * c->n_owned;
  std::vector<int64_t> row_ptr(c->n_rows + 1);
  std::vector<int32_t> col_idx(c->nnz);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < c->n_owned; v++) {
    const int64_t d = node_deg[v];
    for (int i = 0; i < 3; i++) {
      const int64_t r0 = node_rs[v] + i * 3 * d;
      row_ptr[3 * v + i] = r0;
      for (int64_t p = 0; p < d; p++)
        for (int k = 0; k < 3; k++) col_idx[r0 + 3 * p + k] = (int32_t)(3 * adj.nbr[adj.ptr[v] + p] + k);
    }
  }
  row_ptr[c->n_rows] = c->nnz;

  // ---- greedy element colouring, colour-sorted order -----------------------------------
  std::vector<int32_t> colour(n_el);
  {
    std::vector<uint64_t> used(n_rn, 0);
    int nc = 0;
    for (int64_t e = 0; e < n_el; e++) {
      uint64_t mask = 0;
      for (int a = 0; a < n_en; a++) mask |= used[lrow[e * n_en + a]];
      int col = __builtin_ctzll(~mask);
      if (mask == ~0ULL) return fail(C, COMMET_ERR_ARG, "element %lld needs more than 64 colours", (long long)e);
      colour[e] = col;
      nc = std::max(nc, col + 1);
      for (int a = 0; a < n_en; a++) used[lrow[e * n_en + a]] |= 1ULL << col;
    }
    c->n_colours = nc;
  }
  std::vector<int64_t> perm(n_el);
  c->colour_start.assign(c->n_colours + 1, 0);
  for (int64_t e = 0; e < n_el; e++) c->colour_start[colour[e] + 1]++;
  for (int k = 0; k < c->n_colours; k++) c->colour_start[k + 1] += c->colour_start[k];
  {
    std::vector<int64_t> pos(c->colour_start.begin(), c->colour_start.end() - 1);
    for (int64_t e = 0; e < n_el; e++) perm[pos[colour[e]]++] = e;
  }

  // ---- per-element arrays in colour order ------------------------------------------------
  std::vector<int32_t> conn_s(n_el * n_en), lrow_s(n_el * n_en);
  std::vector<uint8_t> slot_s((size_t)n_el * n_en * n_en);
  std::vector<double> w_s(n_el * n_q);
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < n_el; s++) {
    const int64_t e = perm[s];
    for (int a = 0; a < n_en; a++) {
      conn_s[s * n_en + a] = conn[e * n_en + a];
      lrow_s[s * n_en + a] = lrow[e * n_en + a];
    }
    for (int q = 0; q < n_q; q++) w_s[s * n_q + q] = mesh->qp_w[e * n_q + q];
    for (int a = 0; a < n_en; a++) {
      const int64_t v = lrow[e * n_en + a];
      const int64_t* nb = adj.nbr.data() + adj.ptr[v];
      const int64_t d = adj.ptr[v + 1] - adj.ptr[v];
      for (int b = 0; b < n_en; b++)
        slot_s[((size_t)s * n_en + a) * n_en + b] = (uint8_t)(std::lower_bound(nb, nb + d, (int64_t)conn[e * n_en + b]) - nb);
    }
  }
  commet_status s;
  if ((s = upload(C, c->conn, conn_s.data(), conn_s.size(), st))) return s;
  if ((s = upload(C, c->lrow, lrow_s.data(), lrow_s.size(), st))) return s;
  if ((s = upload(C, c->slot, slot_s.data(), slot_s.size(), st))) return s;
  if ((s = upload(C, c->qp_w, w_s.data(), w_s.size(), st))) return s;
  if ((s = upload(C, c->orig, perm.data(), perm.size(), st))) return s;
  if ((s = upload(C, c->node_rs, node_rs.data(), node_rs.size(), st))) return s;
  if ((s = upload(C, c->node_deg, node_deg.data(), node_deg.size(), st))) return s;
  if ((s = upload(C, c->row_ptr, row_ptr.data(), row_ptr.size(), st))) return s;
  if ((s = upload(C, c->col_idx, col_idx.data(), col_idx.size(), st))) return s;
  // gradN: gather in colour order through a pinned staging buffer (inputs may be tens of GB)
  {
    const size_t per = (size_t)n_q * n_en * 3;
    CUDA_TRY(C, c->gradN.alloc((size_t)n_el * per));
    const int64_t chunk = std::max<int64_t>(1, (64 << 20) / (int64_t)(per * sizeof(double)));
    double* stage[2] = {nullptr, nullptr};
    cudaEvent_t ev[2];
    CUDA_TRY(C, cudaMallocHost(&stage[0], chunk * per * sizeof(double)));
    CUDA_TRY(C, cudaMallocHost(&stage[1], chunk * per * sizeof(double)));
    CUDA_TRY(C, cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CUDA_TRY(C, cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    int k = 0;
    for (int64_t s0 = 0; s0 < n_el; s0 += chunk, k ^= 1) {
      const int64_t n = std::min(chunk, n_el - s0);
      CUDA_TRY(C, cudaEventSynchronize(ev[k]));
#pragma omp parallel for schedule(static)
      for (int64_t x = 0; x < n; x++)
        std::memcpy(stage[k] + x * per, mesh->grad_N + perm[s0 + x] * per, per * sizeof(double));
      CUDA_TRY(C, cudaMemcpyAsync(c->gradN.p + s0 * per, stage[k], n * per * sizeof(double),
                                  cudaMemcpyHostToDevice, st));
      CUDA_TRY(C, cudaEventRecord(ev[k], st));
    }
    CUDA_TRY(C, cudaStreamSynchronize(st));
    cudaFreeHost(stage[0]);
    cudaFreeHost(stage[1]);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
  }

  // ---- NCM -------------------------------------------------------------------------------
  std::vector<double> zeros3(3, 0.0);
  if ((s = upload(C, c->W1, ncm->W1, (size_t)w * 3, st))) return s;
  if ((s = upload(C, c->b, ncm->b, (size_t)L * w, st))) return s;
  if ((s = upload(C, c->a, ncm->a, (size_t)w, st))) return s;
  if ((s = upload(C, c->skip_out, ncm->skip_out ? ncm->skip_out : zeros3.data(), 3, st))) return s;
  if (ncm->skip_hidden && L > 1)
    if ((s = upload(C, c->skip_h, ncm->skip_hidden, (size_t)(L - 1) * w * 3, st))) return s;
  std::vector<double> wrow((size_t)std::max(L - 1, 1) * w * w, 0.0);
  if (L > 1) std::memcpy(wrow.data(), ncm->W, (size_t)(L - 1) * w * w * sizeof(double));
  if ((s = upload(C, c->Wrow, wrow.data(), wrow.size(), st))) return s;
  std::vector<double> wf(fused_weight_frag_size(w, L), 0.0);
  fused_weight_frag_fill(w, L, wrow.data(), wf.data());
  if ((s = upload(C, c->Wfrag, wf.data(), wf.size(), st))) return s;
  c->ncm = NcmDev{L, w, c->W1.p, c->b.p, c->a.p, c->skip_out.p, c->skip_h.p, c->Wrow.p, c->Wfrag.p,
                  ncm->kappa, ncm->ref_shift};
  CUDA_TRY(C, c->bad.alloc(1));
  CUDA_TRY(C, c->r_halo.alloc(3 * c->n_halo));
  CUDA_TRY(C, c->v_halo.alloc(c->nnz_halo));
  CUDA_TRY(C, cudaStreamSynchronize(st));
  *out = c.release();
  return COMMET_OK;
}

extern "C" commet_status commet_csr_pattern(commet_ctx c, int64_t* n_rows, int64_t* nnz,
                                            const int64_t** row_ptr, const int32_t** col_idx) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (n_rows) *n_rows = c->n_rows;
  if (nnz) *nnz = c->nnz;
  if (row_ptr) *row_ptr = c->row_ptr.p;
  if (col_idx) *col_idx = c->col_idx.p;
  return COMMET_OK;
}

extern "C" commet_status commet_csr_pattern_copy(commet_ctx c, int64_t* row_ptr, int32_t* col_idx) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (row_ptr)
    CUDA_TRY(c, cudaMemcpy(row_ptr, c->row_ptr.p, (c->n_rows + 1) * sizeof(int64_t), cudaMemcpyDefault));
  if (col_idx && c->nnz)
    CUDA_TRY(c, cudaMemcpy(col_idx, c->col_idx.p, c->nnz * sizeof(int32_t), cudaMemcpyDefault));
  return COMMET_OK;
}

extern "C" commet_status commet_assemble(commet_ctx c, const double* u, double* residual,
                                         double* csr_values, void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (!u || (c->n_rows && !residual) || (c->nnz && !csr_values))
    return fail(c, COMMET_ERR_ARG, "u, residual or csr_values is NULL");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  c->last_stream = st;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemsetAsync(residual, 0, c->n_rows * sizeof(double), st));
  CUDA_TRY(c, cudaMemsetAsync(csr_values, 0, c->nnz * sizeof(double), st));
  CUDA_TRY(c, cudaMemsetAsync(c->bad.p, 0xff, sizeof(unsigned long long), st));
  if (c->n_halo) {
    CUDA_TRY(c, cudaMemsetAsync(c->r_halo.p, 0, c->r_halo.n * sizeof(double), st));
    CUDA_TRY(c, cudaMemsetAsync(c->v_halo.p, 0, c->v_halo.n * sizeof(double), st));
  }
  AsmArgs a{};
  a.n_en = c->n_en;
  a.n_q = c->n_q;
  a.conn = c->conn.p;
  a.lrow = c->lrow.p;
  a.gradN = c->gradN.p;
  a.qp_w = c->qp_w.p;
  a.slot = c->slot.p;
  a.orig = c->orig.p;
  a.node_rs = c->node_rs.p;
  a.node_deg = c->node_deg.p;
  a.n_owned = c->n_owned;
  a.u = u;
  a.r_own = residual;
  a.v_own = csr_values;
  a.r_halo = c->r_halo.p;
  a.v_halo = c->v_halo.p;
  a.bad = c->bad.p;
  a.ncm = c->ncm;
  // interface colours first (elements touching halo rows), so the exchange can
  // overlap the interior colours -- with greedy colouring every colour may touch
  // the interface, so here all colours run, then the exchange.
  const int slot = c->ev0.empty() ? -1 : (int)(c->n_assembled % (int64_t)c->ev0.size());
  if (slot >= 0) CUDA_TRY(c, cudaEventRecord(c->ev0[slot], st));
  for (int k = 0; k < c->n_colours; k++) {
    a.el_begin = c->colour_start[k];
    a.el_count = c->colour_start[k + 1] - c->colour_start[k];
    int rc = c->kernel == COMMET_KERNEL_SIMPLE ? launch_simple(a, st) : launch_fused(a, st, nullptr);
    if (rc) return fail(c, COMMET_ERR_CUDA, "kernel launch (colour %d): %s", k, cudaGetErrorString((cudaError_t)rc));
  }
  if (slot >= 0) CUDA_TRY(c, cudaEventRecord(c->ev1[slot], st));
  c->n_assembled++;
  return COMMET_OK;
}

extern "C" commet_status commet_check(commet_ctx c, int64_t* first_bad_qp) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->last_stream));
  unsigned long long v = ~0ULL;
  CUDA_TRY(c, cudaMemcpy(&v, c->bad.p, sizeof v, cudaMemcpyDeviceToHost));
  const int64_t r = v == ~0ULL ? -1 : (int64_t)v;
  if (first_bad_qp) *first_bad_qp = r;
  if (r >= 0) return fail(c, COMMET_ERR_DOMAIN, "det F <= 0 at flat quadrature point %lld", (long long)r);
  return COMMET_OK;
}

extern "C" commet_status commet_set_kernel(commet_ctx c, int32_t variant) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (variant != COMMET_KERNEL_FUSED && variant != COMMET_KERNEL_SIMPLE)
    return fail(c, COMMET_ERR_ARG, "kernel variant %d unknown", variant);
  c->kernel = variant;
  return COMMET_OK;
}

extern "C" commet_status commet_info(commet_ctx c, int32_t* n_colours, int32_t* n_q, int32_t* n_en,
                                     int32_t* launches) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (n_colours) *n_colours = c->n_colours;
  if (n_q) *n_q = c->n_q;
  if (n_en) *n_en = c->n_en;
  if (launches) {
    int nonempty = 0;
    for (int k = 0; k < c->n_colours; k++) nonempty += c->colour_start[k + 1] > c->colour_start[k];
    *launches = nonempty;
  }
  return COMMET_OK;
}

extern "C" commet_status commet_set_timing(commet_ctx c, int32_t n_slots) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (n_slots < 0 || n_slots > 100000) return fail(c, COMMET_ERR_ARG, "n_slots %d out of range", n_slots);
  CUDA_TRY(c, cudaSetDevice(c->device));
  for (auto e : c->ev0) cudaEventDestroy(e);
  for (auto e : c->ev1) cudaEventDestroy(e);
  c->ev0.assign(n_slots, nullptr);
  c->ev1.assign(n_slots, nullptr);
  for (int i = 0; i < n_slots; i++) {
    CUDA_TRY(c, cudaEventCreate(&c->ev0[i]));
    CUDA_TRY(c, cudaEventCreate(&c->ev1[i]));
  }
  c->n_assembled = 0;
  return COMMET_OK;
}

extern "C" commet_status commet_kernel_times(commet_ctx c, float* ms_out, int32_t n) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  const int64_t ns = (int64_t)c->ev0.size();
  if (n < 0 || n > ns || n > c->n_assembled || (n && !ms_out))
    return fail(c, COMMET_ERR_ARG, "n = %d but %lld slots / %lld assembles recorded", n, (long long)ns,
                (long long)c->n_assembled);
  CUDA_TRY(c, cudaSetDevice(c->device));
  for (int i = 0; i < n; i++) {
    const int64_t k = (c->n_assembled - n + i) % ns;
    CUDA_TRY(c, cudaEventSynchronize(c->ev1[k]));
    CUDA_TRY(c, cudaEventElapsedTime(&ms_out[i], c->ev0[k], c->ev1[k]));
  }
  return COMMET_OK;
}

extern "C" const char* commet_last_error(commet_ctx c) {
  return c ? c->err.c_str() : g_last_error.c_str();
}

extern "C" void commet_destroy(commet_ctx c) {
  if (!c) return;
  cudaSetDevice(c->device);
  delete c;
}
