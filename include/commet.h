/*
 * commet.h -- C ABI of libcommet.so, the B200 (sm_100a) fused neural-
 * constitutive-model (NCM) update + finite-element assembly library.
 *
 * The operation (arXiv 2510.00884, "COMMET"):
 *   For every element e and quadrature point q (Alg. 1):
 *     F   = I + sum_a u_a (x) GradN_a^{e,q}              (Alg. 1 l.3)
 *     k   = (I1-3, I2-3, J-1),  C = F^T F
 *     W   = N(k) + kappa (J-1)^2 - s0 (J-1),  N an (M)ICNN (Eq. icnn)
 *     g = dW/dk, H = d2W/dk2 analytically, one forward value pass, one adjoint
 *     pass and one Jacobian pass -- no autodiff ("CGO"; the
 *     exact Hessian equals Alg. 4)
 *     S = 2 dW/dC, CC = 4 d2W/dCdC (Eq. stress-cgo / stiffnes-cgo, PAPER.md:796-801,
 *     material form, App. A.1)
 *     r^a_i      += w P_iJ GradN_aJ                        (Eq. r-quad)
 *     K^{ab}_{ik} += w GradN_aJ (d_ik S_JL + F_iI CC_IJKL F_kK) GradN_bL
 *                                                         (Eq. k-quad)
 *   with w = w^{e,q} the quadrature "volume" weight.  r is the
 *   internal force only (no traction, no Dirichlet elimination).
 *
 * Conventions
 *  - DOF numbering: dof = 3*node + component.  Rows of the CSR are the owned
 *    DOFs [3*owned_node_begin, 3*owned_node_end), in order; column indices are
 *    GLOBAL dofs, ascending within a row.  Every node pair sharing >= 1
 *    element contributes a full 3x3 block (even if numerically zero).
 *  - Ownership: commet_setup copies every host input; the caller may free its
 *    arrays on return.  The library owns its device copies and the pattern
 *    arrays (valid until commet_destroy).  Output buffers are caller-owned
 *    device memory and are OVERWRITTEN (not accumulated) by commet_assemble.
 *  - Asynchrony: commet_assemble is asynchronous on the given CUDA stream; it
 *    returns COMMET_OK unless an argument is invalid.  Domain errors
 *    (det F <= 0 at some quadrature point) are recorded on the device as the
 *    lowest flat index e*n_q+q and reported by commet_check; the outputs are
 *    still fully computed (reading R10).
 *  - Errors never throw across the ABI.  commet_last_error(ctx) returns a
 *    message naming the offending index/argument (NULL ctx: last global error).
 *  - Threading: one ctx per device per host thread; no global state except the
 *    CUDA context and the last-error buffer for NULL contexts.
 *  - Multi-GPU (z-slabs): each rank passes the elements
 *    it assembles and its owned node range; the library builds the owned-row
 *    CSR plus the interface maps and exchanges non-owned contributions with
 *    the owning rank over NCCL during commet_assemble.
 */
#ifndef COMMET_H_
#define COMMET_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct commet_ctx_s* commet_ctx;

typedef enum {
  COMMET_OK = 0,
  COMMET_ERR_ARG = 1,    /* invalid argument; message names it */
  COMMET_ERR_CUDA = 2,   /* CUDA runtime error */
  COMMET_ERR_NCCL = 3,   /* NCCL error */
  COMMET_ERR_OOM = 4,    /* device or host allocation failed */
  COMMET_ERR_DOMAIN = 5  /* det F <= 0 at some quadrature point (outputs still written) */
} commet_status;

enum {
  COMMET_HEX8 = 0,  /* 8-node trilinear hexahedron, n_q = 8 (2x2x2 Gauss) */
  COMMET_TET10 = 1  /* 10-node quadratic tetrahedron, n_q = 4 */
};

typedef struct {
  int32_t elem_type;          /* COMMET_HEX8 | COMMET_TET10 */
  int64_t n_nodes;            /* global node count */
  int64_t n_elems;            /* elements assembled by THIS rank (>= 0) */
  const int32_t* conn;        /* host [n_elems][n_en]: global node ids, 0-based */
  const double* grad_N;       /* host [n_elems][n_q][n_en][3]: dN_a/dX (reference config) */
  const double* qp_w;         /* host [n_elems][n_q]: Gauss weight * det(dX/dxi), > 0 */
  int64_t owned_node_begin;   /* rows owned by this rank: nodes [begin, end) */
  int64_t owned_node_end;     /* single GPU: [0, n_nodes) */
  /* Partition (multi-GPU).  Single GPU: n_ranks = 0 or 1, the rest 0 / NULL. */
  int32_t n_ranks;
  int32_t rank;
  const int64_t* rank_node_begin; /* host [n_ranks+1]: rank r owns nodes [rnb[r], rnb[r+1]) (ascending) */
  int64_t n_ghost;            /* elements assembled by OTHER ranks that contain owned nodes */
  const int32_t* ghost_conn;  /* host [n_ghost][n_en]: their connectivity (global node ids) */
  const int32_t* ghost_rank;  /* host [n_ghost]: the rank that assembles each ghost element */
  /* Scatter order.  COMMET_ORDER_COLOURED: one launch per element colour, each CSR
   * entry gets at most one update per launch -> bitwise reproducible results.
   * COMMET_ORDER_ELEMENT: one launch in element order, concurrent updates resolved by
   * the fp64 L2 reductions (RED.ADD.F64): neighbouring elements run together, so
   * the CSR rows stay in L2, but the summation order (last bits) varies run to run. */
  int32_t scatter_order;
} commet_mesh_desc;

enum { COMMET_ORDER_COLOURED = 0, COMMET_ORDER_ELEMENT = 1 };

/* (M)ICNN inner network of Eq. icnn with softplus
 * activation, on the kinematic inputs k = (I1-3, I2-3, J-1) (nk = 3; anisotropic: nk = 5, see a0):
 *   y1 = W1 k + b1;  y_l = W_l z_{l-1} + B_l k + b_l (l = 2..L);  z_l = softplus(y_l)
 *   N  = a . z_L + skip_out . k                                                 */
typedef struct {
  int32_t n_hidden;            /* L >= 1 */
  int32_t width;               /* w; multiple of 8, 8 <= w <= 128 */
  const double* W1;            /* host [w][nk] */
  const double* W;             /* host [L-1][w][w] row-major (out, in); may be NULL if L == 1 */
  const double* b;             /* host [L][w] */
  const double* a;             /* host [w] output weights (no output bias: no effect on S, CC) */
  const double* skip_out;      /* host [3] or NULL (= 0): output skip B^(n) on k1..k3 */
  const double* skip_hidden;   /* host [L-1][w][3] or NULL (= 0): hidden skips B^(l), l >= 2, on k1..k3;
                                  must be NULL for nk = 5 (COMMET_ERR_ARG) */
  double kappa;                /* volumetric penalty kappa (J-1)^2 */
  double ref_shift;            /* s0: adds -s0 (J-1) to W; 0 = off (reading R11) */
  /* ---- variants; a zero-initialised tail = the ICNN on k above ---- */
  int32_t kinematics;          /* COMMET_KIN_STANDARD: k = (I1-3, I2-3, J-1); COMMET_KIN_ANISOTROPIC: see a0;
                                  COMMET_KIN_ISOCHORIC: k = (Ibar1-3, Ibar2-3, J-1), Ibar1 = J^-2/3 I1,
                                  Ibar2 = J^-4/3 I2 (App. A.2.2);
                                  COMMET_KIN_ISOCHORIC_ANISOTROPIC: the anisotropic inputs below on the
                                  isochoric set Ibar = {1, 2, (4,ij), (5,ij)} of App. A.2.2:
                                  (Ibar1-3, Ibar2-3, J-1, Ibar4,ij - A_i.A_j, Ibar5,ij - A_i.A_j),
                                  Ibar4,ij = J^-2/3 I4,ij, Ibar5,ij = J^-4/3 I5,ij (reading R29) */
  int32_t network;             /* COMMET_NET_ICNN (the fields above), COMMET_NET_CANN, COMMET_NET_GENT_THOMAS */
  int32_t cann_n;              /* CANN: branches per kinematic input, 1..16 */
  const int32_t* cann_f;       /* CANN host [n_in][cann_n][3] (n_in = 3, or 5 anisotropic): f0 (0 x, 1 <x>, 2 |x|), f1 power (1..3),
                                  f2 (0 w1 x, 1 exp(w1 x) - 1, 2 -ln(1 - w1 x))  (Eq. cann-fs) */
  const double* cann_w1;       /* CANN host [3][cann_n] */
  const double* cann_w2;       /* CANN host [3][cann_n]: N = sum_m sum_b w2 f2(f1(f0(k_m)); w1)  (Eq. cann-def) */
  double gt[3];                /* Gent-Thomas (App. C): N = gt0 k1 + gt1 ln(1 + k2/3) + gt2 k3^2
                                  (the paper's model: gt = (0.5, 1, 1), isochoric kinematics, kappa = 0) */
  /* ICKAN (App. B.3): R layers of widths n_0 = 3, n_1, ..., n_R = 1; edge (r, i, j)
   * (output i of layer r+1, input j of layer r) carries s(x) = w psi(x), psi a B-spline of order kan_k
   * with kan_nb control points on the uniform knots of layer r's interval [xmin, xmax] (kan_k extra
   * knots on each side); outside the interval psi continues linearly with its end slope (SPEC's reading);
   * z^(r+1)_i = sum_j s_rij(z^(r)_j), N = z^(R)_0.  The CUDA path supports kan_k = 3 (cubic). */
  int32_t kan_layers;          /* R, 1..4 */
  const int32_t* kan_width;    /* host [R+1]: n_0 = 3, ..., n_R = 1, each <= 16 */
  int32_t kan_nb;              /* control points per edge, kan_k+1 .. 32 */
  int32_t kan_k;               /* spline order (3) */
  const double* kan_grid;      /* host [R][2]: xmin, xmax of layer r's inputs */
  const double* kan_w;         /* host [edges]: spline weights, edges in (r, i, j) order */
  const double* kan_c;         /* host [edges][kan_nb]: control points */
  /* COMMET_KIN_ANISOTROPIC (and _ISOCHORIC_ANISOTROPIC): n_sv structural vectors A_v (reference configuration): a0, and a1
   * when n_sv = 2 (n_sv 0 or 1: a0 only).  The network inputs are k = (I1-3, I2-3, J-1, then for
   * each pair i <= j in the order (0,0), (0,1), (1,1): I4,ij - A_i.A_j, I5,ij - A_i.A_j) with
   * I4,ij = A_i.C A_j, I5,ij = A_i.C^2 A_j (Eq. standard-inv-II; App. A.2.1 table,
   * PAPER.md:810-826; readings R27, R28) -- 5 inputs for one vector (I4-1, I5-1 for a
   * unit A0): ICNN (W1 [w][5]), CANN (cann_* arrays over 5 inputs) or ICKAN (kan_width[0] = 5);
   * 9 inputs for two: CANN or ICKAN (an ICNN on 9 inputs: COMMET_ERR_ARG); never Gent-Thomas. */
  double a0[3];
  int32_t n_sv;
  double a1[3];
} commet_ncm_desc;

enum { COMMET_KIN_STANDARD = 0, COMMET_KIN_ISOCHORIC = 1, COMMET_KIN_ANISOTROPIC = 2, COMMET_KIN_ISOCHORIC_ANISOTROPIC = 3 };
enum { COMMET_NET_ICNN = 0, COMMET_NET_CANN = 1, COMMET_NET_GENT_THOMAS = 2, COMMET_NET_ICKAN = 3 };

/* Kernel variants (commet_set_kernel).  FUSED is the product path; SIMPLE is
 * a one-thread-per-element CUDA kernel kept as an independent GPU cross-check. */
enum { COMMET_KERNEL_FUSED = 0, COMMET_KERNEL_SIMPLE = 1 };

/* Build the CSR pattern, element colouring and scatter maps, upload inputs
 * (mesh may be NULL: a ctx for the material-point calls only).
 *   device     CUDA device ordinal
 *   cuda_stream  cudaStream_t for the uploads (NULL = legacy default stream)
 *   nccl_comm  ncclComm_t of the partition (see commet_nccl_comm_init), or NULL
 *              (single GPU, or caller-driven halo exchange)
 *   out        receives the context on success.
 * Errors: COMMET_ERR_ARG (bad sizes, node id out of range at element e,
 * w <= 0 at (e,q), unsupported width), COMMET_ERR_OOM, COMMET_ERR_CUDA. */
commet_status commet_setup(const commet_mesh_desc* mesh, const commet_ncm_desc* ncm, int device,
                           void* cuda_stream, void* nccl_comm, commet_ctx* out);

/* Device pointers to the pattern of the owned rows (valid until destroy):
 * row_ptr int64 [n_rows+1], col_idx int32 [nnz] (global dof columns). */
commet_status commet_csr_pattern(commet_ctx ctx, int64_t* n_rows, int64_t* nnz,
                                 const int64_t** row_ptr, const int32_t** col_idx);

/* Copy the pattern into caller buffers (host or device memory; cudaMemcpyDefault):
 * row_ptr int64 [n_rows+1], col_idx int32 [nnz].  Synchronous. */
commet_status commet_csr_pattern_copy(commet_ctx ctx, int64_t* row_ptr, int32_t* col_idx);

/* Assemble: u device fp64 [3*n_nodes] (global, every rank passes the full
 * vector); residual device fp64 [n_rows]; csr_values device fp64 [nnz].
 * Asynchronous on cuda_stream.  With an NCCL communicator and a partition
 * (n_ranks > 1, NCCL mode): every colour's interface elements (those touching a
 * halo row) are launched first, the halo send/recv group then runs on an
 * internal stream while the interior elements are launched, and the unpack of
 * the received rows follows both on cuda_stream.  NCCL
 * asynchronous errors are checked after the group (COMMET_ERR_NCCL). */
commet_status commet_assemble(commet_ctx ctx, const double* u, double* residual,
                              double* csr_values, void* cuda_stream);

/* Assemble on HOST buffers (the end-to-end call; the same r / K as commet_assemble,
 * Eq. r-quad / k-quad): u_host fp64 [3*n_nodes] is read, residual_host
 * fp64 [n_rows] and csr_values_host fp64 [nnz] are written.  The caller owns the host
 * buffers; pinned memory (cudaHostAlloc / cudaHostRegister) makes the copies
 * asynchronous, pageable memory works but serialises them.  Asynchronous: the call
 * enqueues the upload of u (internal copy stream), the assembly (cuda_stream) and the
 * read-back (two internal copy streams, the CSR values in 8 chunks) and returns; the
 * host outputs are valid after commet_host_wait.  The ctx owns two device staging sets
 * (allocated on the first call: 2 x (u + residual + CSR values) doubles; freed by
 * commet_destroy), used alternately, so call s's read-back and call s+1's upload overlap
 * call s+1's assembly.  The caller must not modify u_host, nor read the outputs, before
 * commet_host_wait; successive calls writing the same host outputs complete in call
 * order.  COMMET_ERR_ARG for NULL buffers, a material-only ctx or peer mode;
 * COMMET_ERR_OOM if the staging sets do not fit.  det F <= 0: commet_check. */
commet_status commet_assemble_host(commet_ctx ctx, const double* u_host, double* residual_host,
                                   double* csr_values_host, void* cuda_stream);

/* Completion of every commet_assemble_host call issued so far: with cuda_stream != NULL
 * that stream waits (device side) for the read-backs; with NULL the host blocks until
 * they are done.  COMMET_OK if no host call was made. */
commet_status commet_host_wait(commet_ctx ctx, void* cuda_stream);

/* Synchronises the ctx's last assemble stream; *first_bad_qp = this rank's
 * lowest e*n_q+q (local element index) with det F <= 0, else -1.  Returns
 * COMMET_ERR_DOMAIN if some det F <= 0 (R10), else COMMET_OK.
 * With an NCCL communicator and n_ranks > 1 the call is COLLECTIVE (every rank
 * must call it): one MIN all-reduce of (rank, first bad qp) over the
 * communicator, so every rank returns COMMET_ERR_DOMAIN when any rank saw a
 * bad point (the message names the lowest such rank and its index); an NCCL
 * asynchronous error (ncclCommGetAsyncError) returns COMMET_ERR_NCCL. */
commet_status commet_check(commet_ctx ctx, int64_t* first_bad_qp);

/* As commet_check, but reports the cross-rank result: *bad_rank = the lowest
 * rank with a det F <= 0 point and *first_bad_qp = its lowest local flat index
 * (-1, -1 if none).  Collective under the same conditions. */
commet_status commet_check_ranks(commet_ctx ctx, int32_t* bad_rank, int64_t* first_bad_qp);

/* Select the kernel variant used by subsequent commet_assemble calls. */
commet_status commet_set_kernel(commet_ctx ctx, int32_t variant);

/* Info: n_colours, n_q, n_en and the number of kernel launches one
 * commet_assemble issues (for the bench's gpu_launches). */
commet_status commet_info(commet_ctx ctx, int32_t* n_colours, int32_t* n_q, int32_t* n_en,
                          int32_t* launches_per_assemble);

/* Launch shape of the fused kernel for this ctx: dynamic shared memory per CTA,
 * resident CTAs per SM and registers per thread at launch (diagnostics; the
 * warp-specialised kernel then moves registers between its warpgroups with
 * setmaxnreg: 168 network / 88 element). */
commet_status commet_kernel_info(commet_ctx ctx, int32_t* smem_bytes, int32_t* ctas_per_sm,
                                 int32_t* regs_per_thread);
/* Which kernel the assembly launches for this ctx: threads per CTA, and 1 for the
 * warp-specialised kernel (hex8, forward-sweep ICNN: 4 network + 4 element warps,
 * DESIGN.md s7), 0 for the one-role fused kernel (diagnostics). */
commet_status commet_kernel_config(commet_ctx ctx, int32_t* threads_per_cta, int32_t* warp_specialised);
/* Batch sizes of that kernel: quadrature points per network batch (stages 2-6) and per element
 * batch (stages 0-1, 7-8; two network batches for the ICNN assembly). */
commet_status commet_kernel_batch(commet_ctx ctx, int32_t* qps_network_batch, int32_t* qps_element_batch);

/* Kernel-time instrumentation for benchmarks: with n_slots > 0, every
 * commet_assemble records a CUDA event pair on its stream around its kernel
 * launches (first colour launch .. last launch, zeroing excluded) into a ring
 * of n_slots pairs; n_slots = 0 turns it off. */
commet_status commet_set_timing(commet_ctx ctx, int32_t n_slots);
/* Elapsed kernel milliseconds of the last n assembles (oldest first); n <=
 * min(n_slots, assembles so far).  Synchronises on the recorded events. */
commet_status commet_kernel_times(commet_ctx ctx, float* ms_out, int32_t n);

/* ---- multi-GPU ---------------------------------------------------------------
 * A rank's elements may contain nodes owned by other ranks ("halo" rows).  Their
 * contributions are accumulated in internal halo buffers laid out exactly like
 * the owner expects (the owner derives the layout from its ghost elements), then
 *  - with an NCCL comm (commet_setup's nccl_comm): commet_assemble sends each
 *    halo segment to its owner (ncclSend/ncclRecv in one group, on the assemble
 *    stream) and the owner adds what it receives into its rows (deterministic,
 *    one unpack launch per sender in rank order);
 *  - without a comm (n_ranks > 1, nccl_comm NULL): the caller moves the segments
 *    (commet_halo_send / commet_halo_recv / commet_halo_unpack), e.g. to emulate
 *    several ranks on one device.                                                */
commet_status commet_nccl_unique_id(void* id128);
commet_status commet_nccl_comm_init(const void* id128, int32_t n_ranks, int32_t rank, int device,
                                    void** comm);
commet_status commet_nccl_comm_destroy(void* comm);

/* number of peers this rank sends halo segments to / receives from */
commet_status commet_halo_info(commet_ctx ctx, int32_t* n_send, int32_t* n_recv);
/* k-th send segment (device pointers into the ctx's halo buffers, valid after
 * commet_assemble on its stream completes) */
commet_status commet_halo_send(commet_ctx ctx, int32_t k, int32_t* peer, const double** vals,
                               int64_t* n_vals, const double** residual, int64_t* n_res);
/* size of the k-th receive segment */
commet_status commet_halo_recv(commet_ctx ctx, int32_t k, int32_t* peer, int64_t* n_vals,
                               int64_t* n_res);
/* add a received segment (device arrays of the sizes above) into this rank's
 * residual / csr_values; asynchronous on cuda_stream */
commet_status commet_halo_unpack(commet_ctx ctx, int32_t k, const double* vals, const double* res,
                                 double* residual, double* csr_values, void* cuda_stream);

/* ---- fused interface reduction over peer memory (NVLink P2P) ----------
 * Instead of halo buffers + NCCL send/recv + unpack, the colour kernels add every halo-row
 * contribution straight into the owning rank's residual / CSR values (RED.ADD.F64 through
 * peer pointers), so the transfer overlaps the element math.  Per send segment k
 * (0 <= k < n_send of commet_halo_info):
 *   commet_set_peer(ctx, k, owner_residual, owner_csr_values, val_map, n_vals, row_map, n_res)
 * with the owner's output buffers mapped into this process (e.g. CUDA IPC through torch) and
 * the owner's receive maps for this rank (commet_halo_recv_maps on the owner: its segment for
 * this sender).  commet_set_peer_mode(ctx, 1) then switches commet_assemble to peer mode; its
 * output buffers must stay the ones the peers were given.  With an NCCL comm, commet_assemble
 * zeroes its outputs and brackets the kernels with two NCCL barriers (all ranks zeroed before
 * any rank adds; all added before the step ends).  Without a comm it does NOT zero: the caller
 * runs commet_zero_outputs on every rank, synchronises the ranks, assembles, synchronises.
 * The fused kernel only (its halo writes are atomic); at most 8 send segments. */
commet_status commet_halo_recv_maps(commet_ctx ctx, int32_t k, const int64_t** val_map, const int64_t** row_map);
commet_status commet_set_peer(commet_ctx ctx, int32_t k, double* peer_residual, double* peer_csr_values,
                              const int64_t* val_map, int64_t n_vals, const int64_t* row_map, int64_t n_res);
commet_status commet_set_peer_mode(commet_ctx ctx, int32_t on);
commet_status commet_zero_outputs(commet_ctx ctx, double* residual, double* csr_values, void* cuda_stream);

/* ---- host-only plan (no GPU needed): what commet_setup builds, for inspection --- */
typedef struct commet_plan_s* commet_plan;
commet_status commet_plan_create(const commet_mesh_desc* mesh, commet_plan* out);
commet_status commet_plan_info(commet_plan p, int64_t* n_rows, int64_t* nnz, int64_t* n_halo_nodes,
                               int64_t* nnz_halo, int32_t* n_colours, int32_t* n_send, int32_t* n_recv);
/* host pointers owned by the plan */
commet_status commet_plan_csr(commet_plan p, const int64_t** row_ptr, const int32_t** col_idx);
commet_status commet_plan_halo(commet_plan p, const int64_t** halo_nodes, const int64_t** halo_row_ptr,
                               const int32_t** halo_col_idx);
commet_status commet_plan_send(commet_plan p, int32_t k, int32_t* peer, int64_t* val_begin,
                               int64_t* val_end, int64_t* res_begin, int64_t* res_end);
commet_status commet_plan_recv(commet_plan p, int32_t k, int32_t* peer, int64_t* n_vals,
                               const int64_t** val_map, int64_t* n_res, const int64_t** res_map);
commet_status commet_plan_colours(commet_plan p, const int64_t** colour_start, const int64_t** perm);
/* [n_colours]: colour k's first colour_iface[k] elements (perm[colour_start[k] ..]) are its
 * interface elements -- those with a node outside the owned range; 0 without a partition.
 * commet_assemble launches them before the interiors so the NCCL exchange overlaps the latter. */
commet_status commet_plan_colour_iface(commet_plan p, const int64_t** colour_iface);
void commet_plan_destroy(commet_plan p);

/* Max over all quadrature points of tr C = I1 at the last commet_assemble
 * (synchronises its stream).  The paper's twist-cube robustness check reports
 * tr C > 16 (Fig. 7 caption). */
commet_status commet_max_trace_C(commet_ctx ctx, double* max_trC);

/* ---- material-point calls on the ctx's NCM ------------------------------------
 * The inner network's gradient g = dN/dk [n][nk] and Hessian H [n][nk(nk+1)/2] (packed
 * upper triangle, row by row: 00,01,02,11,12,22 for nk = 3) at n network inputs k [n][nk]
 * (device arrays; nk = 3, or 5 for anisotropic kinematics), by Alg. 4
 * or the analytic networks' closed forms; output skip included, penalty and ref_shift
 * excluded.  Asynchronous on cuda_stream. */
commet_status commet_ncm_eval(commet_ctx ctx, const double* k, double* g, double* H, int64_t n,
                              void* cuda_stream);
/* Material-point batch (the paper's material point
 * benchmarks): for n deformation gradients F (device [n][9],
 * row-major F_iJ) the strain energy density Psi (device [n]), the Kirchhoff stress
 * tau = F S F^T (device [n][6], Voigt order 00, 11, 22, 12, 02, 01) and the spatial
 * tangent c_ijkl = F_iI F_jJ F_kK F_lL CC_IJKL (device [n][21]: the upper triangle
 * of its 6x6 Voigt matrix, row-major) -- the (Psi, tau, c) tables of Alg. 2/3
 * (PAPER.md:254-327).  Any output may be NULL.  Runs the fused kernel's network
 * stages on batches of points; works on a ctx set up with mesh = NULL.
 * Asynchronous; det F <= 0 is reported by commet_check as the point index. */
commet_status commet_material_eval(commet_ctx ctx, const double* F, int64_t n, double* W, double* tau,
                                   double* c, void* cuda_stream);

/* Stress-free reference (reading R11): sets the ctx's ref_shift to
 * s0 = 2 g1 + 4 g2 + g3 at k = 0, so that S(F = I) = 0 for subsequent assembles,
 * and returns it in *s0 (may be NULL).  Synchronous.  COMMET_ERR_ARG for anisotropic
 * kinematics (S(I) then has a structural part no volumetric term cancels). */
commet_status commet_normalize_reference(commet_ctx ctx, double* s0);

/* ---- Newton-Raphson around the assembly --------------
 * d <- d + Delta d with K Delta d = -r, the linear system solved
 * by conjugate gradients with Jacobi preconditioning, all on the
 * GPU.  Single GPU only (n_ranks <= 1; otherwise COMMET_ERR_ARG).
 *
 * Dirichlet conditions are a fixed set of constrained GLOBAL dofs.  Elimination is
 * the symmetric one for Newton increments: once u carries the prescribed values the
 * increment vanishes on constrained dofs, so their rows AND columns of K are zeroed,
 * the diagonal set to 1 and the residual entries set to 0 (K stays SPD when the
 * free block is). */
commet_status commet_set_dirichlet(commet_ctx ctx, const int64_t* dofs /* host [n] */, int64_t n);
/* Eliminate in place: csr_values device [nnz] (this ctx's pattern), residual device
 * [n_rows] or NULL.  Asynchronous on cuda_stream. */
commet_status commet_apply_dirichlet(commet_ctx ctx, double* residual, double* csr_values, void* cuda_stream);
/* Preconditioner of the CG solves of this ctx (commet_cg_jacobi, commet_newton_step):
 * COMMET_PC_JACOBI (default; the paper's "conjugate gradient ... with Jacobi relaxation
 * as the preconditioner") or COMMET_PC_BLOCK_JACOBI (the inverses of the
 * 3x3 nodal diagonal blocks of K).  COMMET_ERR_ARG for another kind. */
enum { COMMET_PC_JACOBI = 0, COMMET_PC_BLOCK_JACOBI = 1 };
commet_status commet_set_preconditioner(commet_ctx ctx, int32_t kind);
/* Solve K x = b (K: csr_values on this ctx's pattern, device; b, x device [n_rows])
 * from x = 0 with (block-)Jacobi-preconditioned CG until ||b - K x||_2 <= rtol ||b||_2.
 * Synchronous.  *iters, *rel_res (may be NULL) report the outcome.  Errors:
 * COMMET_ERR_DOMAIN if a diagonal entry is <= 0 / a 3x3 diagonal block is not positive
 * definite (message names the row) or the tolerance is not met in max_iter iterations
 * (x holds the last iterate). */
commet_status commet_cg_jacobi(commet_ctx ctx, const double* csr_values, const double* b, double* x,
                               double rtol, int32_t max_iter, int32_t* iters, double* rel_res,
                               void* cuda_stream);

#define COMMET_NEWTON_MAX_LOG 64
typedef struct {
  double atol, rtol;      /* converged when ||r_free||_2 <= max(atol, rtol ||r_free^(0)||_2) */
  int32_t max_iter;       /* linear solves per call, 1 .. COMMET_NEWTON_MAX_LOG-1 */
  double cg_rtol;         /* CG relative tolerance per linear solve */
  int32_t cg_max_iter;
} commet_newton_cfg;

typedef struct {
  int32_t iters;          /* linear solves performed */
  int32_t converged;      /* 1 if the residual criterion was met */
  int32_t n_assemble;     /* assemblies (= iters + 1) */
  int64_t cg_iters_total;
  double res_norm[COMMET_NEWTON_MAX_LOG];  /* ||r_free|| after each assembly, [0..iters] */
  int32_t cg_iters[COMMET_NEWTON_MAX_LOG]; /* CG iterations of each linear solve */
  double max_trC;         /* max tr C over qps at the final iterate */
  double ms_assemble;     /* device time: assembly + elimination, summed */
  double ms_solve;        /* device time: CG + update, summed */
} commet_newton_report;

/* One load step of Newton-Raphson to u[dirichlet dofs] = bc_values (host [n]):
 * iteration 0 is the consistent predictor -- r, K = assemble(u) at the previous u,
 * r += K dc with dc the prescribed increment (zero on free dofs), u[dofs] = bc_values
 * (reading R20) -- then every iteration: eliminate; stop if converged;
 * CG: K du = r; u -= du; r, K = assemble(u).
 * u: device [3 n_nodes], in/out.  Synchronous.  Errors: COMMET_ERR_DOMAIN (det F <= 0
 * at some qp, or CG failure; the message says which), COMMET_ERR_ARG. */
commet_status commet_newton_step(commet_ctx ctx, const double* bc_values, const commet_newton_cfg* cfg,
                                 double* u, commet_newton_report* report, void* cuda_stream);

/* Diagnostic: evaluates the kernels' activation on n device values y:
 * z = softplus(y) = log(1+e^y), s = sigmoid(y) (device fp64 arrays).
 * Asynchronous on cuda_stream.  Used by the tests to pin the table-driven
 * softplus/sigmoid of the fused kernel on its own.  commet_selftest_activation
 * uses the 64-entry tables (3-pass kernels); the _tab form takes table_bits 6
 * or 8 (the 256-entry tables of the forward-sweep kernels).  s is NaN where the
 * sigmoid-only form (last hidden layer) differs from the softplus+sigmoid one. */
commet_status commet_selftest_activation_tab(const double* y, double* z, double* s, int64_t n,
                                             int32_t table_bits, void* cuda_stream);
commet_status commet_selftest_activation(const double* y, double* z, double* s, int64_t n,
                                         void* cuda_stream);

const char* commet_last_error(commet_ctx ctx);
void commet_destroy(commet_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* COMMET_H_ */
