// plan.cpp -- see plan.h.  Pure host C++17 + OpenMP.
#include "plan.h"

#include <omp.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>

namespace commet {

static commet_status perr(std::string& err, commet_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  err = buf;
  return s;
}

// adj row v = sorted unique nodes of the elements el[ptr[v]..ptr[v+1]) (>= 0: local
// element, < 0: ghost element -1-g).
static void adjacency_from(const std::vector<int64_t>& ptr, const std::vector<int64_t>& el, int n_en,
                           const int32_t* conn, const int32_t* gconn, Adjacency& adj) {
  const int64_t n = (int64_t)ptr.size() - 1;
  adj.ptr.assign(n + 1, 0);
  auto gather = [&](int64_t v, std::vector<int64_t>& tmp) {
    tmp.clear();
    for (int64_t p = ptr[v]; p < ptr[v + 1]; p++) {
      const int64_t e = el[p];
      const int32_t* c = e >= 0 ? conn + e * n_en : gconn + (-1 - e) * n_en;
      for (int b = 0; b < n_en; b++) tmp.push_back(c[b]);
    }
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
  };
#pragma omp parallel
  {
    std::vector<int64_t> tmp;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; v++) {
      gather(v, tmp);
      adj.ptr[v + 1] = (int64_t)tmp.size();
    }
  }
  for (int64_t v = 0; v < n; v++) adj.ptr[v + 1] += adj.ptr[v];
  adj.nbr.resize(adj.ptr[n]);
#pragma omp parallel
  {
    std::vector<int64_t> tmp;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; v++) {
      gather(v, tmp);
      std::copy(tmp.begin(), tmp.end(), adj.nbr.begin() + adj.ptr[v]);
    }
  }
}

commet_status plan_build(const commet_mesh_desc* mesh, Plan& p, std::string& err) {
  if (!mesh) return perr(err, COMMET_ERR_ARG, "mesh descriptor is NULL");
  if (mesh->elem_type == COMMET_HEX8) { p.n_en = 8; p.n_q = 8; }
  else if (mesh->elem_type == COMMET_TET10) { p.n_en = 10; p.n_q = 4; }
  else return perr(err, COMMET_ERR_ARG, "elem_type %d unknown", mesh->elem_type);
  p.elem_type = mesh->elem_type;
  const int n_en = p.n_en, n_q = p.n_q;
  if (mesh->n_nodes <= 0 || mesh->n_nodes > ((int64_t)1 << 31) / 3)
    return perr(err, COMMET_ERR_ARG, "n_nodes %lld out of range (1 .. 2^31/3)", (long long)mesh->n_nodes);
  if (mesh->n_elems < 0) return perr(err, COMMET_ERR_ARG, "n_elems %lld < 0", (long long)mesh->n_elems);
  if (mesh->n_elems > 0 && (!mesh->conn || !mesh->grad_N || !mesh->qp_w))
    return perr(err, COMMET_ERR_ARG, "conn, grad_N or qp_w is NULL");
  if (mesh->owned_node_begin < 0 || mesh->owned_node_end > mesh->n_nodes ||
      mesh->owned_node_begin > mesh->owned_node_end)
    return perr(err, COMMET_ERR_ARG, "owned node range [%lld, %lld) invalid for n_nodes %lld",
                (long long)mesh->owned_node_begin, (long long)mesh->owned_node_end, (long long)mesh->n_nodes);
  p.n_ranks = mesh->n_ranks > 1 ? mesh->n_ranks : 1;
  p.rank = p.n_ranks > 1 ? mesh->rank : 0;
  p.n_nodes = mesh->n_nodes;
  p.n_el = mesh->n_elems;
  p.node_begin = mesh->owned_node_begin;
  p.node_end = mesh->owned_node_end;
  p.n_owned = p.node_end - p.node_begin;
  const int64_t n_el = p.n_el;
  const int32_t* conn = mesh->conn;
  std::vector<int64_t> rnb;
  if (p.n_ranks > 1) {
    if (p.rank < 0 || p.rank >= p.n_ranks) return perr(err, COMMET_ERR_ARG, "rank %d not in [0, %d)", p.rank, p.n_ranks);
    if (!mesh->rank_node_begin) return perr(err, COMMET_ERR_ARG, "rank_node_begin is NULL with n_ranks %d", p.n_ranks);
    rnb.assign(mesh->rank_node_begin, mesh->rank_node_begin + p.n_ranks + 1);
    if (rnb[0] != 0 || rnb[p.n_ranks] != p.n_nodes)
      return perr(err, COMMET_ERR_ARG, "rank_node_begin must start at 0 and end at n_nodes");
    for (int r = 0; r < p.n_ranks; r++)
      if (rnb[r] > rnb[r + 1]) return perr(err, COMMET_ERR_ARG, "rank_node_begin not ascending at rank %d", r);
    if (rnb[p.rank] != p.node_begin || rnb[p.rank + 1] != p.node_end)
      return perr(err, COMMET_ERR_ARG, "owned range [%lld, %lld) differs from rank_node_begin of rank %d",
                  (long long)p.node_begin, (long long)p.node_end, p.rank);
  }
  const int64_t n_ghost = p.n_ranks > 1 ? mesh->n_ghost : 0;
  if (n_ghost < 0) return perr(err, COMMET_ERR_ARG, "n_ghost %lld < 0", (long long)n_ghost);
  if (n_ghost > 0 && (!mesh->ghost_conn || !mesh->ghost_rank))
    return perr(err, COMMET_ERR_ARG, "ghost_conn or ghost_rank is NULL with n_ghost %lld", (long long)n_ghost);
  const int32_t* gconn = mesh->ghost_conn;
  // ---- validation -------------------------------------------------------------------
  for (int64_t x = 0; x < n_el * n_en; x++)
    if (conn[x] < 0 || conn[x] >= p.n_nodes)
      return perr(err, COMMET_ERR_ARG, "conn[%lld][%d] = %d out of range [0, %lld)", (long long)(x / n_en),
                  (int)(x % n_en), conn[x], (long long)p.n_nodes);
  for (int64_t x = 0; x < n_el * n_q; x++)
    if (!(mesh->qp_w[x] > 0.0))
      return perr(err, COMMET_ERR_ARG, "qp_w[%lld][%d] = %g is not > 0", (long long)(x / n_q), (int)(x % n_q),
                  mesh->qp_w[x]);
  for (int64_t x = 0; x < n_ghost * n_en; x++)
    if (gconn[x] < 0 || gconn[x] >= p.n_nodes)
      return perr(err, COMMET_ERR_ARG, "ghost_conn[%lld][%d] = %d out of range", (long long)(x / n_en),
                  (int)(x % n_en), gconn[x]);
  for (int64_t g = 0; g < n_ghost; g++)
    if (mesh->ghost_rank[g] < 0 || mesh->ghost_rank[g] >= p.n_ranks || mesh->ghost_rank[g] == p.rank)
      return perr(err, COMMET_ERR_ARG, "ghost_rank[%lld] = %d invalid", (long long)g, mesh->ghost_rank[g]);

  // ---- local row-nodes: owned then halo --------------------------------------------------
  auto owned = [&](int64_t v) { return v >= p.node_begin && v < p.node_end; };
  for (int64_t x = 0; x < n_el * n_en; x++)
    if (!owned(conn[x])) p.halo.push_back(conn[x]);
  std::sort(p.halo.begin(), p.halo.end());
  p.halo.erase(std::unique(p.halo.begin(), p.halo.end()), p.halo.end());
  p.n_halo = (int64_t)p.halo.size();
  if (p.n_halo && p.n_ranks <= 1)
    return perr(err, COMMET_ERR_ARG, "%lld nodes referenced by conn are outside the owned range "
                "(first: node %lld) and no partition (n_ranks > 1) was given", (long long)p.n_halo,
                (long long)p.halo[0]);
  const int64_t n_rn = p.n_owned + p.n_halo;
  p.lrow.resize(n_el * n_en);
#pragma omp parallel for
  for (int64_t x = 0; x < n_el * n_en; x++) {
    const int64_t v = conn[x];
    p.lrow[x] = owned(v) ? (int32_t)(v - p.node_begin)
                         : (int32_t)(p.n_owned + (std::lower_bound(p.halo.begin(), p.halo.end(), v) - p.halo.begin()));
  }

  // ---- incidence: row-node -> local elements, plus ghost elements for owned rows ---------
  {
    std::vector<int64_t> ptr(n_rn + 1, 0);
    for (int64_t x = 0; x < n_el * n_en; x++) ptr[p.lrow[x] + 1]++;
    for (int64_t x = 0; x < n_ghost * n_en; x++)
      if (owned(gconn[x])) ptr[gconn[x] - p.node_begin + 1]++;
    for (int64_t v = 0; v < n_rn; v++) ptr[v + 1] += ptr[v];
    std::vector<int64_t> el(ptr[n_rn]);
    std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
    for (int64_t x = 0; x < n_el * n_en; x++) el[pos[p.lrow[x]]++] = x / n_en;
    for (int64_t x = 0; x < n_ghost * n_en; x++)
      if (owned(gconn[x])) el[pos[gconn[x] - p.node_begin]++] = -1 - x / n_en;
    adjacency_from(ptr, el, n_en, conn, gconn, p.adj);
  }
  for (int64_t v = 0; v < n_rn; v++)
    if (p.adj.ptr[v + 1] - p.adj.ptr[v] > 255)
      return perr(err, COMMET_ERR_ARG, "node row %lld has %lld neighbours (> 255)", (long long)v,
                  (long long)(p.adj.ptr[v + 1] - p.adj.ptr[v]));

  // ---- CSR: owned rows (user buffer) and halo rows (internal buffer) ---------------------
  p.node_rs.resize(n_rn);
  p.node_deg.resize(n_rn);
  int64_t off = 0;
  for (int64_t v = 0; v < n_rn; v++) {
    if (v == p.n_owned) { p.nnz = off; off = 0; }
    p.node_rs[v] = off;
    p.node_deg[v] = (int32_t)(p.adj.ptr[v + 1] - p.adj.ptr[v]);
    off += 9 * (int64_t)p.node_deg[v];
  }
  if (p.n_halo == 0) p.nnz = off; else p.nnz_halo = off;
  auto fill_csr = [&](int64_t v0, int64_t v1, std::vector<int64_t>& rp, std::vector<int32_t>& ci, int64_t nz) {
    rp.assign(3 * (v1 - v0) + 1, 0);
    ci.assign(nz, 0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = v0; v < v1; v++) {
      const int64_t d = p.node_deg[v];
      for (int i = 0; i < 3; i++) {
        const int64_t r0 = p.node_rs[v] + i * 3 * d;
        rp[3 * (v - v0) + i] = r0;
        for (int64_t q = 0; q < d; q++)
          for (int k = 0; k < 3; k++) ci[r0 + 3 * q + k] = (int32_t)(3 * p.adj.nbr[p.adj.ptr[v] + q] + k);
      }
    }
    rp[3 * (v1 - v0)] = nz;
  };
  fill_csr(0, p.n_owned, p.row_ptr, p.col_idx, p.nnz);
  fill_csr(p.n_owned, n_rn, p.halo_row_ptr, p.halo_col_idx, p.nnz_halo);

  // ---- greedy element colouring (local row-nodes shared => conflict), colour-sorted order -
  //      (element order: a single "colour" holding every element in input order)
  std::vector<int32_t> colour(n_el, 0);
  if (mesh->scatter_order == COMMET_ORDER_ELEMENT) {
    p.n_colours = n_el > 0 ? 1 : 0;
  } else if (mesh->scatter_order != COMMET_ORDER_COLOURED) {
    return perr(err, COMMET_ERR_ARG, "scatter_order %d unknown", mesh->scatter_order);
  } else {
    std::vector<uint64_t> used(n_rn, 0);
    int nc = 0;
    for (int64_t e = 0; e < n_el; e++) {
      uint64_t mask = 0;
      for (int a = 0; a < n_en; a++) mask |= used[p.lrow[e * n_en + a]];
      if (mask == ~0ULL) return perr(err, COMMET_ERR_ARG, "element %lld needs more than 64 colours", (long long)e);
      const int col = __builtin_ctzll(~mask);
      colour[e] = col;
      nc = std::max(nc, col + 1);
      for (int a = 0; a < n_en; a++) used[p.lrow[e * n_en + a]] |= 1ULL << col;
    }
    p.n_colours = nc;
  }
  p.colour_start.assign(p.n_colours + 1, 0);
  for (int64_t e = 0; e < n_el; e++) p.colour_start[colour[e] + 1]++;
  for (int k = 0; k < p.n_colours; k++) p.colour_start[k + 1] += p.colour_start[k];
  p.perm.resize(n_el);
  p.colour_iface.assign(p.n_colours, 0);
  {
    // within a colour: interface elements (a node in the halo) first, then the interior, each in
    // input order -- the colour's update set, hence the summation order, is unchanged
    std::vector<char> iface(n_el, 0);
    if (p.n_halo)
      for (int64_t e = 0; e < n_el; e++)
        for (int a = 0; a < n_en; a++) iface[e] |= p.lrow[e * n_en + a] >= p.n_owned;
    std::vector<int64_t> pos(p.colour_start.begin(), p.colour_start.end() - 1);
    for (int pass = 1; pass >= 0; pass--)
      for (int64_t e = 0; e < n_el; e++)
        if (iface[e] == pass) {
          p.perm[pos[colour[e]]++] = e;
          if (pass) p.colour_iface[colour[e]]++;
        }
  }
  p.slot.resize((size_t)n_el * n_en * n_en);
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < n_el; s++) {
    const int64_t e = p.perm[s];
    for (int a = 0; a < n_en; a++) {
      const int64_t v = p.lrow[e * n_en + a];
      const int64_t* nb = p.adj.nbr.data() + p.adj.ptr[v];
      const int64_t d = p.adj.ptr[v + 1] - p.adj.ptr[v];
      for (int b = 0; b < n_en; b++)
        p.slot[((size_t)s * n_en + a) * n_en + b] =
            (uint8_t)(std::lower_bound(nb, nb + d, (int64_t)conn[e * n_en + b]) - nb);
    }
  }

  // ---- interface maps ------------------------------------------------------------------
  if (p.n_ranks > 1) {
    // send: halo rows grouped by owner (ascending node ids => contiguous per owner)
    int64_t h = 0;
    p.send_val_off.push_back(0);
    p.send_row_off.push_back(0);
    while (h < p.n_halo) {
      const int owner = (int)(std::upper_bound(rnb.begin(), rnb.end(), p.halo[h]) - rnb.begin()) - 1;
      int64_t h1 = h;
      while (h1 < p.n_halo && p.halo[h1] < rnb[owner + 1]) h1++;
      p.send_rank.push_back(owner);
      p.send_val_off.push_back(p.node_rs[p.n_owned + h1 - 1] + 9 * (int64_t)p.node_deg[p.n_owned + h1 - 1]);
      p.send_row_off.push_back(3 * h1);
      h = h1;
    }
    // recv: for each sender s (ascending), its halo rows = owned nodes touched by its ghost
    // elements, each with the adjacency of those ghost elements -- the layout the sender
    // builds from the same elements.
    std::vector<int32_t> senders;
    for (int64_t g = 0; g < n_ghost; g++) senders.push_back(mesh->ghost_rank[g]);
    std::sort(senders.begin(), senders.end());
    senders.erase(std::unique(senders.begin(), senders.end()), senders.end());
    p.recv_val_off.push_back(0);
    p.recv_row_off.push_back(0);
    for (int32_t s : senders) {
      std::vector<int64_t> ptr(p.n_owned + 1, 0);
      for (int64_t x = 0; x < n_ghost * n_en; x++)
        if (mesh->ghost_rank[x / n_en] == s && owned(gconn[x])) ptr[gconn[x] - p.node_begin + 1]++;
      for (int64_t v = 0; v < p.n_owned; v++) ptr[v + 1] += ptr[v];
      std::vector<int64_t> el(ptr[p.n_owned]);
      std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
      for (int64_t x = 0; x < n_ghost * n_en; x++)
        if (mesh->ghost_rank[x / n_en] == s && owned(gconn[x])) el[pos[gconn[x] - p.node_begin]++] = -1 - x / n_en;
      Adjacency sa;
      adjacency_from(ptr, el, n_en, conn, gconn, sa);
      for (int64_t v = 0; v < p.n_owned; v++) {
        const int64_t d = sa.ptr[v + 1] - sa.ptr[v];
        if (!d) continue;
        const int64_t* mine = p.adj.nbr.data() + p.adj.ptr[v];
        const int64_t md = p.node_deg[v];
        for (int i = 0; i < 3; i++) {
          p.recv_row_map.push_back(3 * v + i);
          for (int64_t q = 0; q < d; q++) {
            const int64_t nb = sa.nbr[sa.ptr[v] + q];
            const int64_t sl = std::lower_bound(mine, mine + md, nb) - mine;
            for (int k = 0; k < 3; k++) p.recv_val_map.push_back(p.node_rs[v] + i * 3 * md + 3 * sl + k);
          }
        }
      }
      p.recv_rank.push_back(s);
      p.recv_val_off.push_back((int64_t)p.recv_val_map.size());
      p.recv_row_off.push_back((int64_t)p.recv_row_map.size());
    }
  }
  return COMMET_OK;
}

}  // namespace commet
