// api.cu -- the C ABI of libcommet (include/commet.h): setup (host plan from
// plan.cpp, device uploads), the assemble orchestration (zeroing, one fused
// launch per colour, halo exchange over NCCL for multi-GPU partitions) and
// the host-only plan inspection calls.
#include <cuda_runtime.h>
#include <nccl.h>
#include <omp.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "commet.h"
#include "commet_internal.h"
#include "ctx.h"
#include "plan.h"
#include "qp_math.cuh"

using namespace commet;

thread_local std::string commet_detail::g_last_error;

// ---------------------------------------------------------------------------
extern "C" commet_status commet_setup(const commet_mesh_desc* mesh, const commet_ncm_desc* ncm,
                                      int device, void* cuda_stream, void* nccl_comm,
                                      commet_ctx* out) {
  if (!out) return fail(nullptr, COMMET_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (!ncm) return fail(nullptr, COMMET_ERR_ARG, "ncm descriptor is NULL");
  std::unique_ptr<commet_ctx_s> c(new (std::nothrow) commet_ctx_s());
  if (!c) return fail(nullptr, COMMET_ERR_OOM, "host allocation failed");
  commet_ctx C = c.get();
  // NCM arguments (host checks, before any CUDA call)
  const int net = ncm->network, kin = ncm->kinematics;
  if (kin != COMMET_KIN_STANDARD && kin != COMMET_KIN_ISOCHORIC && kin != COMMET_KIN_ANISOTROPIC &&
      kin != COMMET_KIN_ISOCHORIC_ANISOTROPIC)
    return fail(C, COMMET_ERR_ARG, "kinematics %d unknown", kin);
  // anisotropic: one structural vector (a0; n_sv 0 or 1) -> 5 inputs, two (a0, a1) -> 9 inputs
  const bool aniso = kin == COMMET_KIN_ANISOTROPIC || kin == COMMET_KIN_ISOCHORIC_ANISOTROPIC;
  const int n_sv = aniso ? (ncm->n_sv > 1 ? ncm->n_sv : 1) : 0;
  if (aniso && (ncm->n_sv < 0 || ncm->n_sv > 2))
    return fail(C, COMMET_ERR_ARG, "n_sv %d not in 0..2 (structural vectors)", ncm->n_sv);
  const int nk = n_sv == 2 ? 9 : (n_sv == 1 ? 5 : 3);  // network inputs
  if (nk > 3 && net == COMMET_NET_GENT_THOMAS)
    return fail(C, COMMET_ERR_ARG, "anisotropic kinematics need an ICNN, CANN or ICKAN inner network (%d inputs)", nk);
  if (nk == 9 && net == COMMET_NET_ICNN)
    return fail(C, COMMET_ERR_ARG, "two structural vectors (9 inputs): CANN or ICKAN inner network (the ICNN kernels "
                "take up to 5 inputs)");
  if (net != COMMET_NET_ICNN && net != COMMET_NET_CANN && net != COMMET_NET_GENT_THOMAS && net != COMMET_NET_ICKAN)
    return fail(C, COMMET_ERR_ARG, "network %d unknown", net);
  // analytic networks use no hidden layers (the ICNN fields are ignored)
  const int L = net == COMMET_NET_ICNN ? ncm->n_hidden : 1, w = net == COMMET_NET_ICNN ? ncm->width : 16;
  const bool tet = mesh && mesh->elem_type == COMMET_TET10;
  if (net == COMMET_NET_ICNN) {
    if (L < 1 || L > kMaxLayers) return fail(C, COMMET_ERR_ARG, "n_hidden %d not in 1..%d", L, kMaxLayers);
    if (!fused_supported(tet ? 10 : 8, tet ? 4 : 8, w, L))
      return fail(C, COMMET_ERR_ARG, "width %d unsupported (8, 16, 32, 64 or 128)", w);
    if (!ncm->W1 || !ncm->b || !ncm->a || (L > 1 && !ncm->W))
      return fail(C, COMMET_ERR_ARG, "NCM weight pointer NULL (W1, b, a or W)");
    if (nk != 3 && ncm->skip_hidden)
      return fail(C, COMMET_ERR_ARG, "hidden skips B^(k) act on (K1, K2, K3) only: skip_hidden must be NULL for 5 inputs");
  }
  int64_t kan_edges = 0;
  if (net == COMMET_NET_ICKAN) {
    const int R = ncm->kan_layers;
    if (R < 1 || R > 4) return fail(C, COMMET_ERR_ARG, "kan_layers %d not in 1..4", R);
    if (!ncm->kan_width || !ncm->kan_grid || !ncm->kan_w || !ncm->kan_c)
      return fail(C, COMMET_ERR_ARG, "ICKAN pointer NULL (kan_width, kan_grid, kan_w or kan_c)");
    if (ncm->kan_width[0] != nk || ncm->kan_width[R] != 1)
      return fail(C, COMMET_ERR_ARG, "kan_width must start at %d inputs and end at 1 output", nk);
    for (int r = 0; r <= R; r++)
      if (ncm->kan_width[r] < 1 || ncm->kan_width[r] > 16)
        return fail(C, COMMET_ERR_ARG, "kan_width[%d] = %d not in 1..16", r, ncm->kan_width[r]);
    if (ncm->kan_k != 3) return fail(C, COMMET_ERR_ARG, "kan_k %d: the CUDA path evaluates cubic splines (3)", ncm->kan_k);
    if (ncm->kan_nb < 4 || ncm->kan_nb > 32) return fail(C, COMMET_ERR_ARG, "kan_nb %d not in 4..32", ncm->kan_nb);
    for (int r = 0; r < R; r++) {
      if (!(ncm->kan_grid[2 * r + 1] > ncm->kan_grid[2 * r]))
        return fail(C, COMMET_ERR_ARG, "kan_grid layer %d: xmax <= xmin", r);
      kan_edges += (int64_t)ncm->kan_width[r] * ncm->kan_width[r + 1];
    }
  }
  if (net == COMMET_NET_CANN) {
    if (ncm->cann_n < 1 || ncm->cann_n > 16) return fail(C, COMMET_ERR_ARG, "cann_n %d not in 1..16", ncm->cann_n);
    if (!ncm->cann_f || !ncm->cann_w1 || !ncm->cann_w2)
      return fail(C, COMMET_ERR_ARG, "CANN pointer NULL (cann_f, cann_w1 or cann_w2)");
    for (int x = 0; x < nk * ncm->cann_n; x++) {
      const int32_t* f = ncm->cann_f + 3 * x;
      if (f[0] < 0 || f[0] > 2 || f[1] < 1 || f[1] > 3 || f[2] < 0 || f[2] > 2)
        return fail(C, COMMET_ERR_ARG, "cann_f entry %d = (%d, %d, %d) outside the menus (f0 0..2, f1 1..3, f2 0..2)",
                    x, f[0], f[1], f[2]);
    }
  }
  Plan& p = c->plan;
  c->material_only = (mesh == nullptr);
  if (mesh) {
    std::string err;
    commet_status s = plan_build(mesh, p, err);
    if (s != COMMET_OK) return fail(C, s, "%s", err.c_str());
  }
  const int n_en = p.n_en, n_q = p.n_q;
  const int64_t n_el = p.n_el;
  c->device = device;
  c->comm = (ncclComm_t)nccl_comm;
  CUDA_TRY(C, cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)cuda_stream;

  // ---- per-element arrays in colour order -------------------------------------------------
  if (mesh) {
    std::vector<int32_t> conn_s(n_el * n_en), lrow_s(n_el * n_en);
    std::vector<double> w_s(n_el * n_q);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < n_el; s++) {
      const int64_t e = p.perm[s];
      for (int a = 0; a < n_en; a++) {
        conn_s[s * n_en + a] = mesh->conn[e * n_en + a];
        lrow_s[s * n_en + a] = p.lrow[e * n_en + a];
      }
      for (int q = 0; q < n_q; q++) w_s[s * n_q + q] = mesh->qp_w[e * n_q + q];
    }
    commet_status s;
    if ((s = upload(C, c->conn, conn_s.data(), conn_s.size(), st))) return s;
    if ((s = upload(C, c->lrow, lrow_s.data(), lrow_s.size(), st))) return s;
    if ((s = upload(C, c->slot, p.slot.data(), p.slot.size(), st))) return s;
    if ((s = upload(C, c->qp_w, w_s.data(), w_s.size(), st))) return s;
    if ((s = upload(C, c->orig, p.perm.data(), p.perm.size(), st))) return s;
    if ((s = upload(C, c->node_rs, p.node_rs.data(), p.node_rs.size(), st))) return s;
    if ((s = upload(C, c->node_deg, p.node_deg.data(), p.node_deg.size(), st))) return s;
    if ((s = upload(C, c->row_ptr, p.row_ptr.data(), p.row_ptr.size(), st))) return s;
    if ((s = upload(C, c->col_idx, p.col_idx.data(), p.col_idx.size(), st))) return s;
    if ((s = upload(C, c->recv_val_map, p.recv_val_map.data(), p.recv_val_map.size(), st))) return s;
    if ((s = upload(C, c->recv_row_map, p.recv_row_map.data(), p.recv_row_map.size(), st))) return s;
    CUDA_TRY(C, cudaStreamSynchronize(st));
  }
  // gradN: gather in colour order through pinned staging buffers (inputs may be tens of GB)
  if (mesh) {
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
        std::memcpy(stage[k] + x * per, mesh->grad_N + p.perm[s0 + x] * per, per * sizeof(double));
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

  // ---- NCM ---------------------------------------------------------------------------------
  commet_status s;
  std::vector<double> zeros3(3, 0.0), zw((size_t)L * w * 5 + 5, 0.0);
  const bool icnn = net == COMMET_NET_ICNN;
  if ((s = upload(C, c->W1, icnn ? ncm->W1 : zw.data(), (size_t)w * nk, st))) return s;
  if ((s = upload(C, c->b, icnn ? ncm->b : zw.data(), (size_t)L * w, st))) return s;
  if ((s = upload(C, c->a, icnn ? ncm->a : zw.data(), (size_t)w, st))) return s;
  if (net == COMMET_NET_ICKAN) {
    if ((s = upload(C, c->kan_grid, ncm->kan_grid, (size_t)2 * ncm->kan_layers, st))) return s;
    if ((s = upload(C, c->kan_w, ncm->kan_w, (size_t)kan_edges, st))) return s;
    if ((s = upload(C, c->kan_c, ncm->kan_c, (size_t)kan_edges * ncm->kan_nb, st))) return s;
  }
  if (net == COMMET_NET_CANN) {
    const size_t nb = (size_t)nk * ncm->cann_n;
    if ((s = upload(C, c->cann_f, ncm->cann_f, 3 * nb, st))) return s;
    if ((s = upload(C, c->cann_w1, ncm->cann_w1, nb, st))) return s;
    if ((s = upload(C, c->cann_w2, ncm->cann_w2, nb, st))) return s;
  }
  if ((s = upload(C, c->skip_out, ncm->skip_out ? ncm->skip_out : zeros3.data(), 3, st))) return s;
  if (icnn && ncm->skip_hidden && L > 1)
    if ((s = upload(C, c->skip_h, ncm->skip_hidden, (size_t)(L - 1) * w * 3, st))) return s;
  std::vector<double> wrow((size_t)std::max(L - 1, 1) * w * w, 0.0);
  if (icnn && L > 1) std::memcpy(wrow.data(), ncm->W, (size_t)(L - 1) * w * w * sizeof(double));
  if ((s = upload(C, c->Wrow, wrow.data(), wrow.size(), st))) return s;
  std::vector<double> wf(fused_weight_frag_size(w, L), 0.0);
  fused_weight_frag_fill(w, L, wrow.data(), wf.data());
  if ((s = upload(C, c->Wfrag, wf.data(), wf.size(), st))) return s;
  std::vector<double> tab(kActTabSize);
  fill_act_table(tab.data());
  if ((s = upload(C, c->act_tab, tab.data(), tab.size(), st))) return s;
  c->ncm = NcmDev{L, w, c->W1.p, c->b.p, c->a.p, c->skip_out.p, c->skip_h.p, c->Wrow.p, c->Wfrag.p,
                  c->act_tab.p, ncm->kappa, ncm->ref_shift, aniso ? (int)COMMET_KIN_ANISOTROPIC : kin, net,
                  net == COMMET_NET_CANN ? ncm->cann_n : 0, c->cann_f.p, c->cann_w1.p, c->cann_w2.p,
                  {ncm->gt[0], ncm->gt[1], ncm->gt[2]},
                  net == COMMET_NET_ICKAN ? ncm->kan_layers : 0, net == COMMET_NET_ICKAN ? ncm->kan_nb : 0,
                  {0, 0, 0, 0, 0}, c->kan_grid.p, c->kan_w.p, c->kan_c.p, {ncm->a0[0], ncm->a0[1], ncm->a0[2]},
                  {n_sv == 2 ? ncm->a1[0] : 0.0, n_sv == 2 ? ncm->a1[1] : 0.0, n_sv == 2 ? ncm->a1[2] : 0.0}};
  if (n_sv == 2) c->ncm.kin = 3;  // internal: anisotropic with two structural vectors
  c->ncm.aniso_iso = kin == COMMET_KIN_ISOCHORIC_ANISOTROPIC;  // internal: kin 2 / 3 on the isochoric inputs
  if (net == COMMET_NET_ICKAN)
    for (int r = 0; r <= ncm->kan_layers; r++) c->ncm.kan_width[r] = ncm->kan_width[r];
  CUDA_TRY(C, c->bad.alloc(1));
  CUDA_TRY(C, c->max_trc.alloc(1));
  CUDA_TRY(C, c->r_halo.alloc(3 * p.n_halo));
  CUDA_TRY(C, c->v_halo.alloc(p.nnz_halo));
  CUDA_TRY(C, c->r_recv.alloc(p.recv_row_map.size()));
  CUDA_TRY(C, c->v_recv.alloc(p.recv_val_map.size()));
  CUDA_TRY(C, cudaStreamSynchronize(st));

  // ---- NCCL: check that every sender's halo layout matches what this rank derived --------
  if (c->comm && p.n_ranks > 1) {
    int nr = 0, rk = 0;
    NCCL_TRY(C, ncclCommCount(c->comm, &nr));
    NCCL_TRY(C, ncclCommUserRank(c->comm, &rk));
    if (nr != p.n_ranks || rk != p.rank)
      return fail(C, COMMET_ERR_ARG, "NCCL comm is rank %d of %d, mesh says rank %d of %d", rk, nr, p.rank,
                  p.n_ranks);
    const size_t ns = p.send_rank.size(), nrv = p.recv_rank.size();
    DevBuf<int64_t> sizes;
    CUDA_TRY(C, sizes.alloc(2 * (ns + nrv) + 2));
    std::vector<int64_t> h(2 * (ns + nrv) + 2, -1);
    for (size_t k2 = 0; k2 < ns; k2++) {
      h[2 * k2] = p.send_val_off[k2 + 1] - p.send_val_off[k2];
      h[2 * k2 + 1] = p.send_row_off[k2 + 1] - p.send_row_off[k2];
    }
    CUDA_TRY(C, cudaMemcpy(sizes.p, h.data(), h.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    NCCL_TRY(C, ncclGroupStart());
    for (size_t k2 = 0; k2 < ns; k2++)
      NCCL_TRY(C, ncclSend(sizes.p + 2 * k2, 2, ncclInt64, p.send_rank[k2], c->comm, st));
    for (size_t k2 = 0; k2 < nrv; k2++)
      NCCL_TRY(C, ncclRecv(sizes.p + 2 * (ns + k2), 2, ncclInt64, p.recv_rank[k2], c->comm, st));
    NCCL_TRY(C, ncclGroupEnd());
    CUDA_TRY(C, cudaMemcpyAsync(h.data(), sizes.p, h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(C, cudaStreamSynchronize(st));
    for (size_t k2 = 0; k2 < nrv; k2++) {
      const int64_t nv = p.recv_val_off[k2 + 1] - p.recv_val_off[k2];
      const int64_t nrr = p.recv_row_off[k2 + 1] - p.recv_row_off[k2];
      if (h[2 * (ns + k2)] != nv || h[2 * (ns + k2) + 1] != nrr)
        return fail(C, COMMET_ERR_ARG,
                    "halo from rank %d has %lld values / %lld rows, this rank's ghost elements imply %lld / %lld "
                    "(ghost_conn inconsistent with that rank's elements)",
                    p.recv_rank[k2], (long long)h[2 * (ns + k2)], (long long)h[2 * (ns + k2) + 1], (long long)nv,
                    (long long)nrr);
    }
  }
  if (c->comm && p.n_ranks > 1) {
    CUDA_TRY(C, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    CUDA_TRY(C, cudaEventCreateWithFlags(&c->ev_iface, cudaEventDisableTiming));
    CUDA_TRY(C, cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));
    CUDA_TRY(C, c->check_buf.alloc(1));
  }
  // element-order arrays live on the device now
  std::vector<int32_t>().swap(p.lrow);
  std::vector<uint8_t>().swap(p.slot);
  *out = c.release();
  return COMMET_OK;
}

extern "C" commet_status commet_csr_pattern(commet_ctx c, int64_t* n_rows, int64_t* nnz,
                                            const int64_t** row_ptr, const int32_t** col_idx) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (n_rows) *n_rows = 3 * c->plan.n_owned;
  if (nnz) *nnz = c->plan.nnz;
  if (row_ptr) *row_ptr = c->row_ptr.p;
  if (col_idx) *col_idx = c->col_idx.p;
  return COMMET_OK;
}

extern "C" commet_status commet_csr_pattern_copy(commet_ctx c, int64_t* row_ptr, int32_t* col_idx) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (row_ptr)
    CUDA_TRY(c, cudaMemcpy(row_ptr, c->row_ptr.p, (3 * c->plan.n_owned + 1) * sizeof(int64_t), cudaMemcpyDefault));
  if (col_idx && c->plan.nnz)
    CUDA_TRY(c, cudaMemcpy(col_idx, c->col_idx.p, c->plan.nnz * sizeof(int32_t), cudaMemcpyDefault));
  return COMMET_OK;
}

static commet_status unpack(commet_ctx c, int k, const double* vals, const double* res, double* residual,
                            double* csr_values, cudaStream_t st) {
  const Plan& p = c->plan;
  const int64_t v0 = p.recv_val_off[k], v1 = p.recv_val_off[k + 1];
  const int64_t r0 = p.recv_row_off[k], r1 = p.recv_row_off[k + 1];
  int rc = launch_unpack(vals, c->recv_val_map.p + v0, v1 - v0, csr_values, res, c->recv_row_map.p + r0, r1 - r0,
                         residual, st);
  if (rc) return fail(c, COMMET_ERR_CUDA, "unpack kernel: %s", cudaGetErrorString((cudaError_t)rc));
  return COMMET_OK;
}

extern "C" commet_status commet_assemble(commet_ctx c, const double* u, double* residual,
                                         double* csr_values, void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  const Plan& p = c->plan;
  if (c->material_only) return fail(c, COMMET_ERR_ARG, "ctx was set up without a mesh (material points only)");
  if (!u || (p.n_owned && !residual) || (p.nnz && !csr_values))
    return fail(c, COMMET_ERR_ARG, "u, residual or csr_values is NULL");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  c->last_stream = st;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->peer && c->kernel != COMMET_KERNEL_FUSED)
    return fail(c, COMMET_ERR_ARG, "peer mode needs the fused kernel (its halo-row writes are atomic)");
  // peer mode: other ranks add into these buffers -- every rank must have zeroed its outputs
  // before any rank's kernels run (NCCL barrier with a comm; the caller's job without one, see
  // commet_zero_outputs), and the step ends only when every rank's kernels are done
  const bool zero_here = !(c->peer && !c->comm);
  if (zero_here) {
    CUDA_TRY(c, cudaMemsetAsync(residual, 0, 3 * p.n_owned * sizeof(double), st));
    CUDA_TRY(c, cudaMemsetAsync(csr_values, 0, p.nnz * sizeof(double), st));
  }
  if (c->peer && c->comm)
    NCCL_TRY(c, ncclAllReduce(c->barrier_buf.p, c->barrier_buf.p, 1, ncclFloat, ncclSum, c->comm, st));
  CUDA_TRY(c, cudaMemsetAsync(c->bad.p, 0xff, sizeof(unsigned long long), st));
  CUDA_TRY(c, cudaMemsetAsync(c->max_trc.p, 0, sizeof(unsigned long long), st));
  if (p.n_halo && !c->peer) {
    CUDA_TRY(c, cudaMemsetAsync(c->r_halo.p, 0, c->r_halo.n * sizeof(double), st));
    CUDA_TRY(c, cudaMemsetAsync(c->v_halo.p, 0, c->v_halo.n * sizeof(double), st));
  }
  AsmArgs a{};
  a.n_en = p.n_en;
  a.n_q = p.n_q;
  a.conn = c->conn.p;
  a.lrow = c->lrow.p;
  a.gradN = c->gradN.p;
  a.qp_w = c->qp_w.p;
  a.slot = c->slot.p;
  a.orig = c->orig.p;
  a.node_rs = c->node_rs.p;
  a.node_deg = c->node_deg.p;
  a.n_owned = p.n_owned;
  a.u = u;
  a.r_own = residual;
  a.v_own = csr_values;
  a.r_halo = c->r_halo.p;
  a.v_halo = c->v_halo.p;
  a.bad = c->bad.p;
  a.max_trc = c->max_trc.p;
  a.dbg_nnz = p.nnz;
  a.dbg_nnz_halo = p.nnz_halo;
  a.dbg_n_halo = p.n_halo;
  if (c->peer) {
    a.peer = 1;
    a.halo_peer = c->halo_peer.p;
    a.peer_vmap = c->peer_vmap.p;
    a.peer_rmap = c->peer_rmap.p;
    for (size_t k = 0; k < c->peer_v.size(); k++) {
      a.peer_v[k] = c->peer_v[k];
      a.peer_r[k] = c->peer_r[k];
    }
  }
  a.ncm = c->ncm;
  const int slot = c->ev0.empty() ? -1 : (int)(c->n_assembled % (int64_t)c->ev0.size());
  if (slot >= 0) CUDA_TRY(c, cudaEventRecord(c->ev0[slot], st));
  // NCCL exchange with a partition: phase 0 launches every colour's interface elements (the only
  // writers of halo rows), then the exchange starts on the comm stream while phase 1 launches the
  // interiors; the unpack follows both.  Otherwise one phase of whole colours.
  const bool exch = !c->peer && c->comm && p.n_ranks > 1 && (!p.send_rank.empty() || !p.recv_rank.empty());
  for (int phase = 0; phase < (exch ? 2 : 1); phase++) {
    for (int k = 0; k < p.n_colours; k++) {
      const int64_t b0 = p.colour_start[k], b1 = p.colour_start[k + 1], bi = b0 + p.colour_iface[k];
      a.el_begin = !exch ? b0 : (phase == 0 ? b0 : bi);
      a.el_count = !exch ? b1 - b0 : (phase == 0 ? bi - b0 : b1 - bi);
      if (a.el_count == 0) continue;
      int rc = c->kernel == COMMET_KERNEL_SIMPLE ? launch_simple(a, st) : launch_fused(a, st, nullptr);
      if (rc) return fail(c, COMMET_ERR_CUDA, "kernel launch (colour %d): %s", k, cudaGetErrorString((cudaError_t)rc));
    }
    if (exch && phase == 0) {
      // ---- halo exchange over NCCL on the comm stream: one group of point-to-point transfers --
      CUDA_TRY(c, cudaEventRecord(c->ev_iface, st));
      CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_iface, 0));
      cudaStream_t cs = c->comm_stream;
      NCCL_TRY(c, ncclGroupStart());
      for (size_t k = 0; k < p.send_rank.size(); k++) {
        const int64_t v0 = p.send_val_off[k], v1 = p.send_val_off[k + 1];
        const int64_t r0 = p.send_row_off[k], r1 = p.send_row_off[k + 1];
        NCCL_TRY(c, ncclSend(c->v_halo.p + v0, v1 - v0, ncclDouble, p.send_rank[k], c->comm, cs));
        NCCL_TRY(c, ncclSend(c->r_halo.p + r0, r1 - r0, ncclDouble, p.send_rank[k], c->comm, cs));
      }
      for (size_t k = 0; k < p.recv_rank.size(); k++) {
        const int64_t v0 = p.recv_val_off[k], v1 = p.recv_val_off[k + 1];
        const int64_t r0 = p.recv_row_off[k], r1 = p.recv_row_off[k + 1];
        NCCL_TRY(c, ncclRecv(c->v_recv.p + v0, v1 - v0, ncclDouble, p.recv_rank[k], c->comm, cs));
        NCCL_TRY(c, ncclRecv(c->r_recv.p + r0, r1 - r0, ncclDouble, p.recv_rank[k], c->comm, cs));
      }
      NCCL_TRY(c, ncclGroupEnd());
      NCCL_ASYNC_CHECK(c, c->comm);
      CUDA_TRY(c, cudaEventRecord(c->ev_comm, cs));
    }
  }
  if (slot >= 0) CUDA_TRY(c, cudaEventRecord(c->ev1[slot], st));
  c->n_assembled++;
  if (c->peer) {  // halo rows went straight to their owners: only the closing barrier
    if (c->comm) {
      NCCL_TRY(c, ncclAllReduce(c->barrier_buf.p, c->barrier_buf.p, 1, ncclFloat, ncclSum, c->comm, st));
      NCCL_ASYNC_CHECK(c, c->comm);
    }
    return COMMET_OK;
  }
  if (exch) {  // unpack in sender order (deterministic) once the exchange and the interior are done
    CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_comm, 0));
    for (size_t k = 0; k < p.recv_rank.size(); k++) {
      commet_status s = unpack(c, (int)k, c->v_recv.p + p.recv_val_off[k], c->r_recv.p + p.recv_row_off[k],
                               residual, csr_values, st);
      if (s != COMMET_OK) return s;
    }
  }
  return COMMET_OK;
}

// ---- end-to-end call on host buffers (DESIGN.md s9 "e2e") ------------------------------------
// Step s uses staging set k = s % 2: the upload of u waits for the assembly of step s-2 (the last
// reader of u[k]), the assembly waits for the upload and for the read-back of step s-2 (the last
// reader of r[k], v[k]); the read-back of step s runs on the copy streams behind its assembly.
// So step s's read-back and step s+1's upload overlap step s+1's assembly.
static commet_status host_pipe_init(commet_ctx c) {
  const Plan& p = c->plan;
  HostPipe* h = new HostPipe();
  c->host = h;
  if (const char* e = getenv("COMMET_HOST_COPY_STREAMS")) h->n_streams = std::max(1, std::min(HostPipe::kCopyStreams, atoi(e)));
  if (const char* e = getenv("COMMET_HOST_CHUNKS")) h->n_chunks = std::max(1, std::min(1024, atoi(e)));
  for (int k = 0; k < 2; k++) {
    CUDA_TRY(c, h->u[k].alloc(3 * p.n_nodes));
    CUDA_TRY(c, h->r[k].alloc(3 * p.n_owned));
    CUDA_TRY(c, h->v[k].alloc(p.nnz));
    CUDA_TRY(c, cudaEventCreateWithFlags(&h->done_h[k], cudaEventDisableTiming));
    CUDA_TRY(c, cudaEventCreateWithFlags(&h->done_c[k], cudaEventDisableTiming));
    for (int i = 0; i < HostPipe::kCopyStreams; i++)
      CUDA_TRY(c, cudaEventCreateWithFlags(&h->done_d[k][i], cudaEventDisableTiming));
  }
  CUDA_TRY(c, cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
  for (int i = 0; i < HostPipe::kCopyStreams; i++) CUDA_TRY(c, cudaStreamCreateWithFlags(&h->d2h[i], cudaStreamNonBlocking));
  return COMMET_OK;
}

extern "C" commet_status commet_assemble_host(commet_ctx c, const double* u_host, double* residual_host,
                                              double* csr_values_host, void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  const Plan& p = c->plan;
  if (c->material_only) return fail(c, COMMET_ERR_ARG, "ctx was set up without a mesh (material points only)");
  if (c->peer) return fail(c, COMMET_ERR_ARG, "commet_assemble_host: peer mode writes into registered device outputs");
  if (!u_host || (p.n_owned && !residual_host) || (p.nnz && !csr_values_host))
    return fail(c, COMMET_ERR_ARG, "u_host, residual_host or csr_values_host is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (!c->host) {
    commet_status s = host_pipe_init(c);
    if (s != COMMET_OK) {
      delete c->host;
      c->host = nullptr;
      return s;
    }
  }
  HostPipe* h = c->host;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int k = (int)(h->n_calls % 2);
  const bool reuse = h->n_calls >= 2;
  if (reuse) CUDA_TRY(c, cudaStreamWaitEvent(h->h2d, h->done_c[k], 0));
  CUDA_TRY(c, cudaMemcpyAsync(h->u[k].p, u_host, 3 * p.n_nodes * sizeof(double), cudaMemcpyHostToDevice, h->h2d));
  CUDA_TRY(c, cudaEventRecord(h->done_h[k], h->h2d));
  CUDA_TRY(c, cudaStreamWaitEvent(st, h->done_h[k], 0));
  if (reuse)
    for (int i = 0; i < h->n_streams; i++) CUDA_TRY(c, cudaStreamWaitEvent(st, h->done_d[k][i], 0));
  commet_status s = commet_assemble(c, h->u[k].p, h->r[k].p, h->v[k].p, cuda_stream);
  if (s != COMMET_OK) return s;
  CUDA_TRY(c, cudaEventRecord(h->done_c[k], st));
  for (int i = 0; i < h->n_streams; i++) CUDA_TRY(c, cudaStreamWaitEvent(h->d2h[i], h->done_c[k], 0));
  if (p.n_owned)
    CUDA_TRY(c, cudaMemcpyAsync(residual_host, h->r[k].p, 3 * p.n_owned * sizeof(double), cudaMemcpyDeviceToHost,
                                h->d2h[0]));
  for (int j = 0; j < h->n_chunks; j++) {  // one copy engine per stream: chunks round-robin
    const int64_t a0 = p.nnz * j / h->n_chunks, a1 = p.nnz * (j + 1) / h->n_chunks;
    if (a1 > a0)
      CUDA_TRY(c, cudaMemcpyAsync(csr_values_host + a0, h->v[k].p + a0, (a1 - a0) * sizeof(double),
                                  cudaMemcpyDeviceToHost, h->d2h[j % h->n_streams]));
  }
  for (int i = 0; i < h->n_streams; i++) CUDA_TRY(c, cudaEventRecord(h->done_d[k][i], h->d2h[i]));
  h->n_calls++;
  return COMMET_OK;
}

extern "C" commet_status commet_host_wait(commet_ctx c, void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (!c->host) return COMMET_OK;
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  for (int k = 0; k < 2 && k < c->host->n_calls; k++)
    for (int i = 0; i < c->host->n_streams; i++) {
      if (st) CUDA_TRY(c, cudaStreamWaitEvent(st, c->host->done_d[k][i], 0));
      else CUDA_TRY(c, cudaEventSynchronize(c->host->done_d[k][i]));
    }
  return COMMET_OK;
}

// cross-rank key of a rank's first bad qp: (rank, flat index) in one word, ordered by rank first
static constexpr int kBadIdxBits = 44;

// det F <= 0 status of the last assemble.  local: this rank's lowest bad flat index (-1: none);
// with an NCCL partition, (rank, qp) = the lowest rank that has one and its index (collective)
static commet_status check_impl(commet_ctx c, int64_t* local, int32_t* bad_rank, int64_t* first_bad_qp) {
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->last_stream));
  unsigned long long v = ~0ULL;
  CUDA_TRY(c, cudaMemcpy(&v, c->bad.p, sizeof v, cudaMemcpyDeviceToHost));
  *local = v == ~0ULL ? -1 : (int64_t)v;
  int32_t rk = v == ~0ULL ? -1 : c->plan.rank;
  int64_t q = *local;
  if (c->comm && c->plan.n_ranks > 1) {  // collective: MIN over the ranks of (rank, first bad qp)
    unsigned long long key = ~0ULL;
    if (q >= 0) key = ((unsigned long long)c->plan.rank << kBadIdxBits) | ((unsigned long long)q & ((1ULL << kBadIdxBits) - 1));
    cudaStream_t st = c->comm_stream;
    CUDA_TRY(c, cudaMemcpyAsync(c->check_buf.p, &key, sizeof key, cudaMemcpyHostToDevice, st));
    NCCL_TRY(c, ncclAllReduce(c->check_buf.p, c->check_buf.p, 1, ncclUint64, ncclMin, c->comm, st));
    CUDA_TRY(c, cudaMemcpyAsync(&key, c->check_buf.p, sizeof key, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    NCCL_ASYNC_CHECK(c, c->comm);
    rk = key == ~0ULL ? -1 : (int32_t)(key >> kBadIdxBits);
    q = key == ~0ULL ? -1 : (int64_t)(key & ((1ULL << kBadIdxBits) - 1));
  }
  if (bad_rank) *bad_rank = rk;
  if (first_bad_qp) *first_bad_qp = q;
  if (q >= 0)
    return fail(c, COMMET_ERR_DOMAIN, "det F <= 0 at flat quadrature point %lld of rank %d", (long long)q, rk);
  return COMMET_OK;
}

extern "C" commet_status commet_check_ranks(commet_ctx c, int32_t* bad_rank, int64_t* first_bad_qp) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  int64_t local = -1;
  return check_impl(c, &local, bad_rank, first_bad_qp);
}

extern "C" commet_status commet_check(commet_ctx c, int64_t* first_bad_qp) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  int64_t local = -1;
  const commet_status s = check_impl(c, &local, nullptr, nullptr);
  if (first_bad_qp) *first_bad_qp = local;
  return s;
}

extern "C" commet_status commet_max_trace_C(commet_ctx c, double* max_trC) {
  if (!c || !max_trC) return fail(c, COMMET_ERR_ARG, "ctx or max_trC is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->last_stream));
  unsigned long long v = 0;
  CUDA_TRY(c, cudaMemcpy(&v, c->max_trc.p, sizeof v, cudaMemcpyDeviceToHost));
  double d;
  std::memcpy(&d, &v, sizeof d);
  *max_trC = d;
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
  const Plan& p = c->plan;
  if (n_colours) *n_colours = p.n_colours;
  if (n_q) *n_q = p.n_q;
  if (n_en) *n_en = p.n_en;
  if (launches) {
    const bool exch = !c->peer && c->comm && p.n_ranks > 1 && (!p.send_rank.empty() || !p.recv_rank.empty());
    int nonempty = 0;
    for (int k = 0; k < p.n_colours; k++) {
      const int64_t n = p.colour_start[k + 1] - p.colour_start[k], ni = p.colour_iface[k];
      nonempty += exch ? (ni > 0) + (n - ni > 0) : n > 0;
    }
    const int unpacks = exch ? (int)p.recv_rank.size() : 0;
    *launches = nonempty + unpacks;
  }
  return COMMET_OK;
}

static commet_status kernel_query(commet_ctx c, int (&q)[7]) {
  CUDA_TRY(c, cudaSetDevice(c->device));
  // the instantiation the assembly (or material-point) dispatch launches for this ctx
  AsmArgs a{};
  a.n_en = c->material_only ? 1 : c->plan.n_en;
  a.n_q = c->material_only ? 1 : c->plan.n_q;
  a.el_count = 1;
  a.ncm = c->ncm;
  a.query = q;
  const int e = c->material_only ? launch_material(a, nullptr) : launch_fused(a, nullptr, nullptr);
  if (e) return fail(c, COMMET_ERR_CUDA, "kernel query: %s", cudaGetErrorString((cudaError_t)e));
  return COMMET_OK;
}

extern "C" commet_status commet_kernel_info(commet_ctx c, int32_t* smem_bytes, int32_t* ctas_per_sm,
                                            int32_t* regs_per_thread) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  int q[7] = {0, 0, 0, 128, 0, 0, 0};
  const commet_status s = kernel_query(c, q);
  if (s != COMMET_OK) return s;
  if (smem_bytes) *smem_bytes = q[0];
  if (ctas_per_sm) *ctas_per_sm = q[1];
  if (regs_per_thread) *regs_per_thread = q[2];
  return COMMET_OK;
}

extern "C" commet_status commet_kernel_config(commet_ctx c, int32_t* threads_per_cta, int32_t* warp_specialised) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  int q[7] = {0, 0, 0, 128, 0, 0, 0};
  const commet_status s = kernel_query(c, q);
  if (s != COMMET_OK) return s;
  if (threads_per_cta) *threads_per_cta = q[3];
  if (warp_specialised) *warp_specialised = q[4];
  return COMMET_OK;
}

extern "C" commet_status commet_kernel_batch(commet_ctx c, int32_t* qps_network_batch, int32_t* qps_element_batch) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  int q[7] = {0, 0, 0, 128, 0, 0, 0};
  const commet_status s = kernel_query(c, q);
  if (s != COMMET_OK) return s;
  if (qps_network_batch) *qps_network_batch = q[5];
  if (qps_element_batch) *qps_element_batch = q[6];
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

// ---- NCCL helpers and caller-driven halo exchange -----------------------------------------
extern "C" commet_status commet_nccl_unique_id(void* id128) {
  if (!id128) return fail(nullptr, COMMET_ERR_ARG, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  NCCL_TRY(nullptr, ncclGetUniqueId(reinterpret_cast<ncclUniqueId*>(id128)));
  return COMMET_OK;
}

extern "C" commet_status commet_nccl_comm_init(const void* id128, int32_t n_ranks, int32_t rank, int device,
                                               void** comm) {
  if (!id128 || !comm || n_ranks < 1 || rank < 0 || rank >= n_ranks)
    return fail(nullptr, COMMET_ERR_ARG, "bad arguments (rank %d of %d)", rank, n_ranks);
  CUDA_TRY(nullptr, cudaSetDevice(device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t cm = nullptr;
  NCCL_TRY(nullptr, ncclCommInitRank(&cm, n_ranks, id, rank));
  *comm = cm;
  return COMMET_OK;
}

extern "C" commet_status commet_nccl_comm_destroy(void* comm) {
  if (comm) NCCL_TRY(nullptr, ncclCommDestroy((ncclComm_t)comm));
  return COMMET_OK;
}

extern "C" commet_status commet_halo_info(commet_ctx c, int32_t* n_send, int32_t* n_recv) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (n_send) *n_send = (int32_t)c->plan.send_rank.size();
  if (n_recv) *n_recv = (int32_t)c->plan.recv_rank.size();
  return COMMET_OK;
}

extern "C" commet_status commet_halo_send(commet_ctx c, int32_t k, int32_t* peer, const double** vals,
                                          int64_t* n_vals, const double** res, int64_t* n_res) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  const Plan& p = c->plan;
  if (k < 0 || k >= (int32_t)p.send_rank.size()) return fail(c, COMMET_ERR_ARG, "send segment %d does not exist", k);
  if (peer) *peer = p.send_rank[k];
  if (vals) *vals = c->v_halo.p + p.send_val_off[k];
  if (n_vals) *n_vals = p.send_val_off[k + 1] - p.send_val_off[k];
  if (res) *res = c->r_halo.p + p.send_row_off[k];
  if (n_res) *n_res = p.send_row_off[k + 1] - p.send_row_off[k];
  return COMMET_OK;
}

extern "C" commet_status commet_halo_recv(commet_ctx c, int32_t k, int32_t* peer, int64_t* n_vals, int64_t* n_res) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  const Plan& p = c->plan;
  if (k < 0 || k >= (int32_t)p.recv_rank.size()) return fail(c, COMMET_ERR_ARG, "recv segment %d does not exist", k);
  if (peer) *peer = p.recv_rank[k];
  if (n_vals) *n_vals = p.recv_val_off[k + 1] - p.recv_val_off[k];
  if (n_res) *n_res = p.recv_row_off[k + 1] - p.recv_row_off[k];
  return COMMET_OK;
}

extern "C" commet_status commet_halo_recv_maps(commet_ctx c, int32_t k, const int64_t** val_map,
                                               const int64_t** row_map) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  const Plan& p = c->plan;
  if (k < 0 || k >= (int)p.recv_rank.size()) return fail(c, COMMET_ERR_ARG, "recv segment %d out of range", k);
  if (val_map) *val_map = p.recv_val_map.data() + p.recv_val_off[k];
  if (row_map) *row_map = p.recv_row_map.data() + p.recv_row_off[k];
  return COMMET_OK;
}

extern "C" commet_status commet_set_peer(commet_ctx c, int32_t k, double* peer_residual, double* peer_csr_values,
                                         const int64_t* val_map, int64_t n_vals, const int64_t* row_map,
                                         int64_t n_res) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  const Plan& p = c->plan;
  const int ns = (int)p.send_rank.size();
  if (k < 0 || k >= ns) return fail(c, COMMET_ERR_ARG, "send segment %d out of range (%d)", k, ns);
  if (ns > kMaxPeers) return fail(c, COMMET_ERR_ARG, "%d send segments > %d", ns, kMaxPeers);
  const int64_t v0 = p.send_val_off[k], v1 = p.send_val_off[k + 1], r0 = p.send_row_off[k], r1 = p.send_row_off[k + 1];
  if (n_vals != v1 - v0 || n_res != r1 - r0)
    return fail(c, COMMET_ERR_ARG, "segment %d: maps of %lld values / %lld rows, the segment has %lld / %lld", k,
                (long long)n_vals, (long long)n_res, (long long)(v1 - v0), (long long)(r1 - r0));
  if (!peer_residual || !peer_csr_values || (n_vals && !val_map) || (n_res && !row_map))
    return fail(c, COMMET_ERR_ARG, "peer pointer or map is NULL");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->peer_v.empty()) {
    c->peer_v.assign(ns, nullptr);
    c->peer_r.assign(ns, nullptr);
    c->peer_set.assign(ns, 0);
    CUDA_TRY(c, c->peer_vmap.alloc(std::max<int64_t>(1, p.nnz_halo)));
    CUDA_TRY(c, c->peer_rmap.alloc(std::max<int64_t>(1, 3 * p.n_halo)));
    std::vector<int8_t> hp(std::max<int64_t>(1, p.n_halo), 0);
    for (int kk = 0; kk < ns; kk++)
      for (int64_t r = p.send_row_off[kk]; r < p.send_row_off[kk + 1]; r += 3) hp[r / 3] = (int8_t)kk;
    CUDA_TRY(c, c->halo_peer.alloc(hp.size()));
    CUDA_TRY(c, cudaMemcpy(c->halo_peer.p, hp.data(), hp.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(c, c->barrier_buf.alloc(1));
    CUDA_TRY(c, cudaMemset(c->barrier_buf.p, 0, sizeof(float)));
  }
  if (n_vals) CUDA_TRY(c, cudaMemcpy(c->peer_vmap.p + v0, val_map, n_vals * sizeof(int64_t), cudaMemcpyHostToDevice));
  if (n_res) CUDA_TRY(c, cudaMemcpy(c->peer_rmap.p + r0, row_map, n_res * sizeof(int64_t), cudaMemcpyHostToDevice));
  c->peer_v[k] = peer_csr_values;
  c->peer_r[k] = peer_residual;
  c->peer_set[k] = 1;
  return COMMET_OK;
}

extern "C" commet_status commet_set_peer_mode(commet_ctx c, int32_t on) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (!on) {
    c->peer = false;
    return COMMET_OK;
  }
  const Plan& p = c->plan;
  if (p.n_ranks <= 1) return fail(c, COMMET_ERR_ARG, "peer mode needs a multi-rank partition");
  for (size_t k = 0; k < p.send_rank.size(); k++)
    if (k >= c->peer_set.size() || !c->peer_set[k])
      return fail(c, COMMET_ERR_ARG, "send segment %zu (to rank %d) has no peer (commet_set_peer)", k, p.send_rank[k]);
  if (c->peer_v.empty()) {  // no send segments (the top slab): only the barrier buffer is needed
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, c->barrier_buf.alloc(1));
    CUDA_TRY(c, cudaMemset(c->barrier_buf.p, 0, sizeof(float)));
  }
  c->peer = true;
  return COMMET_OK;
}

extern "C" commet_status commet_zero_outputs(commet_ctx c, double* residual, double* csr_values, void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  const Plan& p = c->plan;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (residual) CUDA_TRY(c, cudaMemsetAsync(residual, 0, 3 * p.n_owned * sizeof(double), st));
  if (csr_values) CUDA_TRY(c, cudaMemsetAsync(csr_values, 0, p.nnz * sizeof(double), st));
  return COMMET_OK;
}

extern "C" commet_status commet_halo_unpack(commet_ctx c, int32_t k, const double* vals, const double* res,
                                            double* residual, double* csr_values, void* cuda_stream) {
  if (!c) return fail(nullptr, COMMET_ERR_ARG, "ctx is NULL");
  if (k < 0 || k >= (int32_t)c->plan.recv_rank.size())
    return fail(c, COMMET_ERR_ARG, "recv segment %d does not exist", k);
  CUDA_TRY(c, cudaSetDevice(c->device));
  return unpack(c, k, vals, res, residual, csr_values, (cudaStream_t)cuda_stream);
}

// ---- host-only plan -------------------------------------------------------------------------
extern "C" commet_status commet_plan_create(const commet_mesh_desc* mesh, commet_plan* out) {
  if (!out) return fail(nullptr, COMMET_ERR_ARG, "out is NULL");
  *out = nullptr;
  std::unique_ptr<commet_plan_s> p(new (std::nothrow) commet_plan_s());
  if (!p) return fail(nullptr, COMMET_ERR_OOM, "host allocation failed");
  std::string err;
  commet_status s = plan_build(mesh, p->p, err);
  if (s != COMMET_OK) return fail(nullptr, s, "%s", err.c_str());
  *out = p.release();
  return COMMET_OK;
}

extern "C" commet_status commet_plan_info(commet_plan pl, int64_t* n_rows, int64_t* nnz, int64_t* n_halo,
                                          int64_t* nnz_halo, int32_t* n_colours, int32_t* n_send,
                                          int32_t* n_recv) {
  if (!pl) return fail(nullptr, COMMET_ERR_ARG, "plan is NULL");
  const Plan& p = pl->p;
  if (n_rows) *n_rows = 3 * p.n_owned;
  if (nnz) *nnz = p.nnz;
  if (n_halo) *n_halo = p.n_halo;
  if (nnz_halo) *nnz_halo = p.nnz_halo;
  if (n_colours) *n_colours = p.n_colours;
  if (n_send) *n_send = (int32_t)p.send_rank.size();
  if (n_recv) *n_recv = (int32_t)p.recv_rank.size();
  return COMMET_OK;
}

extern "C" commet_status commet_plan_csr(commet_plan pl, const int64_t** row_ptr, const int32_t** col_idx) {
  if (!pl) return fail(nullptr, COMMET_ERR_ARG, "plan is NULL");
  if (row_ptr) *row_ptr = pl->p.row_ptr.data();
  if (col_idx) *col_idx = pl->p.col_idx.data();
  return COMMET_OK;
}

extern "C" commet_status commet_plan_halo(commet_plan pl, const int64_t** halo_nodes, const int64_t** halo_row_ptr,
                                          const int32_t** halo_col_idx) {
  if (!pl) return fail(nullptr, COMMET_ERR_ARG, "plan is NULL");
  if (halo_nodes) *halo_nodes = pl->p.halo.data();
  if (halo_row_ptr) *halo_row_ptr = pl->p.halo_row_ptr.data();
  if (halo_col_idx) *halo_col_idx = pl->p.halo_col_idx.data();
  return COMMET_OK;
}

extern "C" commet_status commet_plan_send(commet_plan pl, int32_t k, int32_t* peer, int64_t* val_begin,
                                          int64_t* val_end, int64_t* res_begin, int64_t* res_end) {
  if (!pl) return fail(nullptr, COMMET_ERR_ARG, "plan is NULL");
  const Plan& p = pl->p;
  if (k < 0 || k >= (int32_t)p.send_rank.size())
    return fail(nullptr, COMMET_ERR_ARG, "send segment %d does not exist", k);
  if (peer) *peer = p.send_rank[k];
  if (val_begin) *val_begin = p.send_val_off[k];
  if (val_end) *val_end = p.send_val_off[k + 1];
  if (res_begin) *res_begin = p.send_row_off[k];
  if (res_end) *res_end = p.send_row_off[k + 1];
  return COMMET_OK;
}

extern "C" commet_status commet_plan_recv(commet_plan pl, int32_t k, int32_t* peer, int64_t* n_vals,
                                          const int64_t** val_map, int64_t* n_res, const int64_t** res_map) {
  if (!pl) return fail(nullptr, COMMET_ERR_ARG, "plan is NULL");
  const Plan& p = pl->p;
  if (k < 0 || k >= (int32_t)p.recv_rank.size())
    return fail(nullptr, COMMET_ERR_ARG, "recv segment %d does not exist", k);
  if (peer) *peer = p.recv_rank[k];
  if (n_vals) *n_vals = p.recv_val_off[k + 1] - p.recv_val_off[k];
  if (val_map) *val_map = p.recv_val_map.data() + p.recv_val_off[k];
  if (n_res) *n_res = p.recv_row_off[k + 1] - p.recv_row_off[k];
  if (res_map) *res_map = p.recv_row_map.data() + p.recv_row_off[k];
  return COMMET_OK;
}

extern "C" commet_status commet_plan_colours(commet_plan pl, const int64_t** colour_start, const int64_t** perm) {
  if (!pl) return fail(nullptr, COMMET_ERR_ARG, "plan is NULL");
  if (colour_start) *colour_start = pl->p.colour_start.data();
  if (perm) *perm = pl->p.perm.data();
  return COMMET_OK;
}

extern "C" commet_status commet_plan_colour_iface(commet_plan pl, const int64_t** colour_iface) {
  if (!pl) return fail(nullptr, COMMET_ERR_ARG, "plan is NULL");
  if (colour_iface) *colour_iface = pl->p.colour_iface.data();
  return COMMET_OK;
}

extern "C" void commet_plan_destroy(commet_plan pl) { delete pl; }

extern "C" commet_status commet_selftest_activation_tab(const double* y, double* z, double* s, int64_t n,
                                                        int32_t table_bits, void* cuda_stream) {
  if (n < 0 || (n && (!y || !z || !s)))
    return fail(nullptr, COMMET_ERR_ARG, "bad arguments (n = %lld)", (long long)n);
  if (table_bits != 6 && table_bits != 8) return fail(nullptr, COMMET_ERR_ARG, "table_bits %d not 6 or 8", table_bits);
  static std::mutex mu;
  static double* d_tab = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!d_tab) {
      std::vector<double> tab(kActTabSize);
      fill_act_table(tab.data());
      CUDA_TRY(nullptr, cudaMalloc(&d_tab, tab.size() * sizeof(double)));
      CUDA_TRY(nullptr, cudaMemcpy(d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
  }
  int rc = launch_activation(y, z, s, n, d_tab, table_bits, cuda_stream);
  if (rc) return fail(nullptr, COMMET_ERR_CUDA, "activation kernel: %s", cudaGetErrorString((cudaError_t)rc));
  return COMMET_OK;
}

extern "C" commet_status commet_selftest_activation(const double* y, double* z, double* s, int64_t n,
                                                    void* cuda_stream) {
  return commet_selftest_activation_tab(y, z, s, n, 6, cuda_stream);
}

extern "C" const char* commet_last_error(commet_ctx c) {
  return c ? c->err.c_str() : commet_detail::g_last_error.c_str();
}

extern "C" void commet_destroy(commet_ctx c) {
  if (!c) return;
  cudaSetDevice(c->device);
  delete c;
}
