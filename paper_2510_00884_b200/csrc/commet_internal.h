// commet_internal.h -- device-side data layout of libcommet (not part of the ABI).
//
// HBM layout (per rank, all device memory owned by the ctx):
//  * element data in COLOUR-SORTED order (colour c = [colour_start[c], colour_start[c+1])):
//      conn   int32 [n_el][n_en]        global node ids (u gather)
//      lrow   int32 [n_el][n_en]        local row-node id (owned: node-begin; halo: n_owned + h)
//      gradN  fp64  [n_el][n_q][n_en][3]  contiguous per element (1536 B hex8, 960 B tet10)
//      qp_w   fp64  [n_el][n_q]
//      slot   uint8 [n_el][n_en][n_en]  position of node b in the adjacency of node a's row
//      orig   int64 [n_el]               original element index (det F <= 0 report)
//  * per local row-node: node_rs int64 (first CSR entry of its row 3a+0), node_deg int32;
//    row 3a+i starts at node_rs[a] + i*3*deg[a]; entry (3a+i, 3b+k) at + 3*slot + k.
//  * NCM weights in DMMA m8n8k4 A-fragment order (see kernel_fused.cu).
#pragma once
#include <cstdint>

namespace commet {

constexpr int kMaxLayers = 4;
constexpr int kMaxWidth = 128;
constexpr int kMaxPeers = 8;  // send segments (peer ranks) of the peer-mode scatter

struct NcmDev {
  int L, w;
  const double* W1;       // [w][3]
  const double* b;        // [L][w]
  const double* a;        // [w]
  const double* skip_out; // [3] (zeros if absent)
  const double* skip_h;   // [L-1][w][3] or nullptr
  const double* Wrow;     // [L-1][w][w] row-major (simple kernel)
  const double* Wfrag;    // [L-1][2][frag] fragment-ordered W and W^T (fused kernel)
  const double* act_tab;  // [kActTabSize] softplus tables (qp_math.cuh)
  double kappa, ref_shift;
  int kin, net, cann_n;   // variants (commet.h COMMET_KIN_* / COMMET_NET_*)
  const int32_t* cann_f;  // [3][n][3]
  const double* cann_w1;  // [3][n]
  const double* cann_w2;  // [3][n]
  double gt[3];
  int kan_R, kan_nb;      // ICKAN (net 3)
  int kan_width[5];
  const double* kan_grid;  // [R][2]
  const double* kan_w;     // [edges]
  const double* kan_c;     // [edges][nb]
  double a0[3];            // anisotropic kinematics: structural vector (reference configuration)
  double a1[3];            // anisotropic kinematics, two vectors (kin 3): the second structural vector
  int aniso_iso;           // anisotropic kinematics (kin 2, 3) on the isochoric inputs (App. A.2.2, R29): the fused
                           // kernel dispatches the compile-time KIN 4 / 5 instantiations, the simple kernel branches
};

struct AsmArgs {
  int n_en, n_q;
  int64_t el_begin, el_count;  // colour range in sorted order
  const int32_t* conn;
  const int32_t* lrow;
  const double* gradN;
  const double* qp_w;
  const uint8_t* slot;
  const int64_t* orig;
  const int64_t* node_rs;
  const int32_t* node_deg;
  int64_t n_owned;  // local row-nodes < n_owned -> user buffers
  const double* u;
  double* r_own;
  double* v_own;
  double* r_halo;
  double* v_halo;
  unsigned long long* bad;
  unsigned long long* max_trc;  // max over qps of tr C = I1 (> 0: the bit pattern orders like the value)
  // peer mode (multi-GPU over NVLink P2P): halo rows added straight into the owners' buffers
  int peer;
  const int8_t* halo_peer;      // [n_halo] send segment (= peer slot) of each halo row-node
  const int64_t* peer_vmap;     // [nnz_halo] halo value -> position in the owner's CSR values
  const int64_t* peer_rmap;     // [3 n_halo] halo row -> position in the owner's residual
  double* peer_v[kMaxPeers];
  double* peer_r[kMaxPeers];
  // material-point mode (launch_material): F [n][9] in; Psi [n], tau [n][6], c [n][21] out (each may be NULL)
  const double* Fin;
  double* Wout;
  double* tau_out;
  double* c_out;
  NcmDev ncm;
  // launch query: when set, the dispatcher writes the chosen instantiation's {smem bytes,
  // CTAs per SM, registers per thread} here and launches nothing (commet_kernel_info)
  int* query;
  // debug builds (COMMET_DEBUG_CHECKS): buffer sizes for the scatter bounds checks
  int64_t dbg_nnz, dbg_nnz_halo, dbg_n_halo;
};

// launchers (kernel_simple.cu / kernel_fused.cu); return cudaError_t as int
int launch_simple(const AsmArgs& a, void* stream);
int launch_unpack(const double* vals, const int64_t* vmap, int64_t nv, double* csr, const double* res,
                  const int64_t* rmap, int64_t nr, double* r, void* stream);
int launch_activation(const double* y, double* z, double* s, int64_t n, const double* tab, int table_bits,
                      void* stream);
int launch_fused(const AsmArgs& a, void* stream, int* launches);
int launch_material(const AsmArgs& a, void* stream);
int fused_supported(int n_en, int n_q, int w, int L);
// prepares the fragment-ordered weight array on the host (size in doubles)
int64_t fused_weight_frag_size(int w, int L);
void fused_weight_frag_fill(int w, int L, const double* Wrow, double* out);
// stage-5 fragments: 2 matrices of 16 x w (rows 0-2 W1^T; rows 3-8 W1_jm W1_jn)

}  // namespace commet
