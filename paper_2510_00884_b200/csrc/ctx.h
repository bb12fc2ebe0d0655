// ctx.h -- the library context (struct commet_ctx_s) and the error helpers
// shared by the C ABI implementation files (api.cu, solver.cu).  Internal.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "commet.h"
#include "commet_internal.h"
#include "plan.h"

using namespace commet;

namespace commet_detail {
extern thread_local std::string g_last_error;

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    return count ? cudaMalloc(&p, count * sizeof(T)) : cudaSuccess;
  }
};

}  // namespace commet_detail
using commet_detail::DevBuf;

// commet_assemble_host: two device staging sets (u, residual, CSR values) and the copy streams
// that overlap step s's read-back and step s+1's upload with step s+1's assembly
struct HostPipe {
  // read-back streams (one copy engine each) and CSR-value chunks, round-robin over the streams;
  // COMMET_HOST_COPY_STREAMS / COMMET_HOST_CHUNKS override the defaults (A/B)
  static constexpr int kCopyStreams = 4;
  int n_streams = 2, n_chunks = 8;
  DevBuf<double> u[2], r[2], v[2];
  cudaStream_t h2d = nullptr, d2h[kCopyStreams] = {};
  cudaEvent_t done_h[2] = {}, done_c[2] = {}, done_d[2][kCopyStreams] = {};
  int64_t n_calls = 0;
  ~HostPipe() {  // the copies still in flight finish before their buffers go
    if (h2d) cudaStreamSynchronize(h2d);
    for (auto s : d2h) if (s) cudaStreamSynchronize(s);
    if (h2d) cudaStreamDestroy(h2d);
    for (auto s : d2h) if (s) cudaStreamDestroy(s);
    for (int k = 0; k < 2; k++) {
      if (done_h[k]) cudaEventDestroy(done_h[k]);
      if (done_c[k]) cudaEventDestroy(done_c[k]);
      for (auto e : done_d[k]) if (e) cudaEventDestroy(e);
    }
  }
};

struct SolverWork;  // solver.cu: Dirichlet set, CG / Newton workspace
void solver_work_free(SolverWork* w);

struct commet_ctx_s {
  int device = 0;
  Plan plan;  // host copy (pattern, maps); element-order arrays are dropped after upload
  int kernel = COMMET_KERNEL_FUSED;
  int precond = 0;              // COMMET_PC_JACOBI (the paper's) or COMMET_PC_BLOCK_JACOBI
  bool material_only = false;  // commet_setup(mesh = NULL): material-point calls only
  std::string err;
  cudaStream_t last_stream = nullptr;
  ncclComm_t comm = nullptr;
  // NCCL mode with a partition: the halo exchange runs on its own stream, after the interface
  // elements' launches (ev_iface) and beside the interior's; the unpack waits for ev_comm
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_iface = nullptr, ev_comm = nullptr;
  DevBuf<unsigned long long> check_buf;  // cross-rank MIN of (rank, first bad qp)
  // device data
  DevBuf<int32_t> conn, lrow, col_idx;
  DevBuf<double> gradN, qp_w;
  DevBuf<uint8_t> slot;
  DevBuf<int64_t> orig, node_rs, row_ptr;
  DevBuf<int32_t> node_deg;
  DevBuf<double> W1, b, a, skip_out, skip_h, Wrow, Wfrag, act_tab;
  DevBuf<int32_t> cann_f;
  DevBuf<double> cann_w1, cann_w2, kan_grid, kan_w, kan_c;
  DevBuf<double> r_halo, v_halo, r_recv, v_recv;
  DevBuf<int64_t> recv_val_map, recv_row_map;
  DevBuf<unsigned long long> bad, max_trc;
  // peer mode (fused interface reduction over NVLink P2P)
  bool peer = false;
  std::vector<double*> peer_v, peer_r;  // per send segment: the owner's output buffers
  std::vector<char> peer_set;
  DevBuf<int8_t> halo_peer;
  DevBuf<int64_t> peer_vmap, peer_rmap;
  DevBuf<float> barrier_buf;
  SolverWork* solver = nullptr;
  HostPipe* host = nullptr;  // commet_assemble_host staging, allocated on first use
  NcmDev ncm{};
  // timing ring
  std::vector<cudaEvent_t> ev0, ev1;
  int64_t n_assembled = 0;
  ~commet_ctx_s() {
    solver_work_free(solver);
    delete host;
    if (ev_iface) cudaEventDestroy(ev_iface);
    if (ev_comm) cudaEventDestroy(ev_comm);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    for (auto e : ev0) cudaEventDestroy(e);
    for (auto e : ev1) cudaEventDestroy(e);
  }
};

struct commet_plan_s {
  Plan p;
};

inline commet_status fail(commet_ctx c, commet_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  commet_detail::g_last_error = buf;
  return s;
}

#define CUDA_TRY(ctx, x)                                                                     \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? COMMET_ERR_OOM : COMMET_ERR_CUDA,    \
                  "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), __FILE__, __LINE__, #x); \
  } while (0)

#define NCCL_TRY(ctx, x)                                                                           \
  do {                                                                                             \
    ncclResult_t r_ = (x);                                                                         \
    if (r_ != ncclSuccess)                                                                         \
      return fail(ctx, COMMET_ERR_NCCL, "NCCL error %s at %s:%d (%s)", ncclGetErrorString(r_), __FILE__, \
                  __LINE__, #x);                                                                   \
  } while (0)

// NCCL reports errors of operations already enqueued (a peer died, a network error) only
// through the communicator's asynchronous error state
#define NCCL_ASYNC_CHECK(ctx, comm)                                                                \
  do {                                                                                             \
    ncclResult_t a_ = ncclSuccess;                                                                 \
    ncclResult_t q_ = ncclCommGetAsyncError((comm), &a_);                                           \
    if (q_ != ncclSuccess) a_ = q_;                                                                \
    if (a_ != ncclSuccess && a_ != ncclInProgress)                                                 \
      return fail(ctx, COMMET_ERR_NCCL, "NCCL asynchronous error %s at %s:%d", ncclGetErrorString(a_), \
                  __FILE__, __LINE__);                                                             \
  } while (0)

template <class T>
inline commet_status upload(commet_ctx c, DevBuf<T>& d, const T* h, size_t n, cudaStream_t st) {
  CUDA_TRY(c, d.alloc(n));
  if (n) CUDA_TRY(c, cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
  return COMMET_OK;
}

