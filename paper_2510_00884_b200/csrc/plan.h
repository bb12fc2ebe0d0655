// plan.h -- host-only rank-local plan (no CUDA): validation, local row-nodes,
// CSR pattern of owned rows (own + ghost elements), halo rows, element
// colouring, scatter slots and the per-peer interface maps.  commet_setup
// uploads it; commet_plan_* expose it for inspection and CPU tests.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "commet.h"

namespace commet {

struct Adjacency {
  std::vector<int64_t> ptr;  // [n_rownodes+1]
  std::vector<int64_t> nbr;  // global node ids, ascending per row
};

struct Plan {
  int elem_type = 0, n_en = 0, n_q = 0;
  int32_t n_ranks = 1, rank = 0;
  int64_t n_nodes = 0, n_el = 0, node_begin = 0, node_end = 0, n_owned = 0, n_halo = 0;
  std::vector<int64_t> halo;       // halo node global ids, ascending
  std::vector<int32_t> lrow;       // [n_el*n_en] local row-node (original element order)
  Adjacency adj;                   // per local row-node
  std::vector<int64_t> node_rs;    // per local row-node: first entry of row 3a (owned: in vals; halo: in halo vals)
  std::vector<int32_t> node_deg;
  int64_t nnz = 0, nnz_halo = 0;
  std::vector<int64_t> row_ptr;    // owned rows [3 n_owned + 1]
  std::vector<int32_t> col_idx;
  std::vector<int64_t> halo_row_ptr;  // halo rows [3 n_halo + 1] (relative to the halo buffer)
  std::vector<int32_t> halo_col_idx;
  // colouring
  int n_colours = 0;
  std::vector<int64_t> colour_start;  // [n_colours+1] into perm
  // multi-rank: interface elements (touching a halo row) first within each colour, so the
  // assembly can launch them first and overlap the halo exchange with the interior
  std::vector<int64_t> colour_iface;  // [n_colours] interface elements at the start of colour k
  std::vector<int64_t> perm;          // sorted position -> original element
  std::vector<uint8_t> slot;          // [n_el][n_en][n_en] in SORTED order
  // interface: this rank sends halo rows to their owners, receives from ranks whose
  // elements touch its owned rows (ghost elements)
  std::vector<int32_t> send_rank;
  std::vector<int64_t> send_val_off, send_row_off;  // [n_send+1] offsets in halo vals / halo r
  std::vector<int32_t> recv_rank;
  std::vector<int64_t> recv_val_off, recv_row_off;  // [n_recv+1] offsets in the recv buffers
  std::vector<int64_t> recv_val_map, recv_row_map;  // recv entry -> owned vals / owned r position
};

// Builds the plan; on failure returns the status and sets err (message names the index).
commet_status plan_build(const commet_mesh_desc* mesh, Plan& p, std::string& err);

}  // namespace commet
