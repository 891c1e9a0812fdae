// Host-side pattern builder: reduced-system DOF maps, node-level sparsity, element->slot maps,
// element colouring, Dirichlet-lift structure and the bit-exact vector-CSR export.
//
// Restates the *symbolic* part of assemble_mode_system (reference
// pkg/src/spectralstokes/assembly.py:403-479): the reduced matrix a_full[free][:, free] whose
// pattern is the element-pair pattern of [[kron(S, I), D], [D^T, 0]] with explicit zeros kept
// (COO->CSR, kron, bmat and fancy indexing all keep them).  Values are not
// computed here: the device element kernel (assemble.cu) fills them through the element maps.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "spectralstokes_b200.h"

#include "ss_common.h"
#include "ss_pattern.h"
#include "ss_spmv.cuh"

// Last error message per calling thread (like errno): the pointer ss_last_error returns stays
// valid until the same thread's next failing call, whatever other threads do.
static thread_local std::string g_err;
static int64_t g_launches = 0;

void ss_set_error(const std::string& msg) { g_err = msg; }
void ss_count_launch(int64_t n) { __atomic_fetch_add(&g_launches, n, __ATOMIC_RELAXED); }
int64_t ss_launch_counter() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

extern "C" const char* ss_last_error(void) { return g_err.c_str(); }
extern "C" int64_t ss_launch_count(void) { return ss_launch_counter(); }
extern "C" int ss_version(void) { return SS_ABI_VERSION; }

// Device arrays carry 64 zero bytes of tail padding: the staged SpMV rounds its bulk copies to
// 16-byte boundaries (ss_spmv.cuh stream_layout) and may read up to 15 bytes past the last entry.
constexpr size_t SS_TAIL_PAD = 64;

template <class T>
static int upload(ss_pattern* P, const std::vector<T>& h, T** d) {
  size_t bytes = std::max<size_t>(1, h.size()) * sizeof(T) + SS_TAIL_PAD;
  SS_CUDA(cudaMalloc((void**)d, bytes));
  P->allocs.push_back((void*)*d);
  SS_CUDA(cudaMemset(*d, 0, bytes));
  if (!h.empty()) SS_CUDA(cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return SS_OK;
}

template <class T>
static int alloc_zero(ss_pattern* P, size_t count, T** d) {
  size_t bytes = std::max<size_t>(1, count) * sizeof(T) + SS_TAIL_PAD;
  SS_CUDA(cudaMalloc((void**)d, bytes));
  P->allocs.push_back((void*)*d);
  SS_CUDA(cudaMemset(*d, 0, bytes));
  return SS_OK;
}

// Sorted unique neighbour lists per row, built from a row -> element incidence.
static void collect_rows(const std::vector<int>& row_node, const std::vector<int64_t>& inc_ptr,
                         const std::vector<int>& inc, const int64_t* conn, int nloc, int take,
                         std::vector<std::vector<int>>& out) {
  const int64_t nrows = (int64_t)row_node.size();
  out.assign(nrows, {});
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t r = 0; r < nrows; ++r) {
    int A = row_node[r];
    std::vector<int>& v = out[r];
    v.reserve((inc_ptr[A + 1] - inc_ptr[A]) * take);
    for (int64_t q = inc_ptr[A]; q < inc_ptr[A + 1]; ++q) {
      const int64_t* c = conn + (int64_t)inc[q] * nloc;
      for (int a = 0; a < take; ++a) v.push_back((int)c[a]);
    }
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
}

static int lb(const int* row, int len, int key) {
  return (int)(std::lower_bound(row, row + len, key) - row);
}

extern "C" int ss_pattern_create(int dim, int64_t n_vel_nodes, int64_t n_vertices, int64_t n_elements,
                                 const int64_t* vel_conn, const uint8_t* fixed_mask,
                                 int pinned_pressure, int device, ss_pattern** out) {
  if (dim != 2 && dim != 3) { ss_set_error("unsupported dimension"); return SS_ERR_ARG; }
  if (n_vel_nodes <= 0 || n_vertices <= 0 || n_elements <= 0 || !vel_conn || !fixed_mask || !out) {
    ss_set_error("ss_pattern_create: empty mesh or null argument");
    return SS_ERR_ARG;
  }
  if (n_vel_nodes >= (int64_t)1 << 31) { ss_set_error("mesh too large for int32 node ids"); return SS_ERR_ARG; }
  SS_CUDA(cudaSetDevice(device));
  ss_pattern* P = new ss_pattern();
  P->device = device;
  P->dim = dim;
  P->nloc = dim == 2 ? 6 : 10;
  P->nvloc = dim + 1;
  P->nvn = n_vel_nodes;
  P->nvert = n_vertices;
  P->ne = n_elements;
  P->pinned = pinned_pressure ? 1 : 0;
  const int nloc = P->nloc, nvloc = P->nvloc;
  for (int64_t i = 0; i < n_elements * nloc; ++i) {
    if (vel_conn[i] < 0 || vel_conn[i] >= n_vel_nodes) {
      delete P;
      ss_set_error("vel_conn references a node outside the node table");
      return SS_ERR_MESH;
    }
  }
  for (int64_t e = 0; e < n_elements; ++e)
    for (int a = 0; a < nvloc; ++a)
      if (vel_conn[e * nloc + a] >= n_vertices) {
        delete P;
        ss_set_error("element vertex id >= n_vertices");
        return SS_ERR_MESH;
      }

  // DOF maps (assembly.py:455-475).
  P->rank.assign(n_vel_nodes, -1);
  for (int64_t A = 0; A < n_vel_nodes; ++A)
    if (!fixed_mask[A]) { P->rank[A] = (int)P->free_nodes.size(); P->free_nodes.push_back((int)A); }
  const int first_p = P->pinned ? 1 : 0;
  P->vert_pdof.assign(n_vertices, -1);
  for (int64_t v = first_p; v < n_vertices; ++v) {
    P->vert_pdof[v] = (int)P->pres_of_row.size();
    P->pres_of_row.push_back((int)v);
  }
  const int nfree = (int)P->free_nodes.size();
  const int npf = (int)P->pres_of_row.size();
  P->nfree = nfree;
  P->npf = npf;

  // node -> element incidence (elements ascending).
  std::vector<int64_t> inc_ptr(n_vel_nodes + 1, 0);
  for (int64_t i = 0; i < n_elements * nloc; ++i) inc_ptr[vel_conn[i] + 1]++;
  for (int64_t A = 0; A < n_vel_nodes; ++A) inc_ptr[A + 1] += inc_ptr[A];
  std::vector<int> inc(n_elements * nloc);
  {
    std::vector<int64_t> fill(inc_ptr.begin(), inc_ptr.end() - 1);
    for (int64_t e = 0; e < n_elements; ++e)
      for (int a = 0; a < nloc; ++a) inc[fill[vel_conn[e * nloc + a]]++] = (int)e;
  }

  // Free velocity rows: node neighbours (free -> ncol ranks, fixed -> lift) and pressure cols.
  std::vector<std::vector<int>> nodes_rows, vert_rows, prow_nodes;
  collect_rows(P->free_nodes, inc_ptr, inc, vel_conn, nloc, nloc, nodes_rows);
  collect_rows(P->free_nodes, inc_ptr, inc, vel_conn, nloc, nvloc, vert_rows);
  collect_rows(P->pres_of_row, inc_ptr, inc, vel_conn, nloc, nloc, prow_nodes);

  P->nptr.assign(nfree + 1, 0);
  P->lptr.assign(nfree + 1, 0);
  P->pptr.assign(nfree + 1, 0);
  for (int r = 0; r < nfree; ++r) {
    int nf = 0, nx = 0, np = 0;
    for (int B : nodes_rows[r]) (P->rank[B] >= 0 ? nf : nx)++;
    for (int v : vert_rows[r]) if (P->vert_pdof[v] >= 0) np++;
    P->nptr[r + 1] = P->nptr[r] + nf;
    P->lptr[r + 1] = P->lptr[r] + nx;
    P->pptr[r + 1] = P->pptr[r] + np;
  }
  P->ncol.resize(P->nptr[nfree]);
  P->lcol.resize(P->lptr[nfree]);
  P->pcol.resize(P->pptr[nfree]);
  P->diag_slot.assign(nfree, -1);
#pragma omp parallel for schedule(dynamic, 256)
  for (int r = 0; r < nfree; ++r) {
    int f = P->nptr[r], x = P->lptr[r], p = P->pptr[r];
    for (int B : nodes_rows[r]) {
      if (P->rank[B] >= 0) {
        if (P->rank[B] == r) P->diag_slot[r] = f;
        P->ncol[f++] = P->rank[B];
      } else {
        P->lcol[x++] = B;
      }
    }
    for (int v : vert_rows[r]) if (P->vert_pdof[v] >= 0) P->pcol[p++] = P->vert_pdof[v];
  }
  P->tptr.assign(npf + 1, 0);
  P->ltptr.assign(npf + 1, 0);
  for (int j = 0; j < npf; ++j) {
    int nf = 0, nx = 0;
    for (int B : prow_nodes[j]) (P->rank[B] >= 0 ? nf : nx)++;
    P->tptr[j + 1] = P->tptr[j] + nf;
    P->ltptr[j + 1] = P->ltptr[j] + nx;
  }
  P->tcol.resize(P->tptr[npf]);
  P->ltcol.resize(P->ltptr[npf]);
#pragma omp parallel for schedule(dynamic, 256)
  for (int j = 0; j < npf; ++j) {
    int f = P->tptr[j], x = P->ltptr[j];
    for (int B : prow_nodes[j]) {
      if (P->rank[B] >= 0) P->tcol[f++] = P->rank[B];
      else P->ltcol[x++] = B;
    }
  }
  nodes_rows.clear(); vert_rows.clear(); prow_nodes.clear();

  // SpMV row schedule (block -> rows).  Default: natural order (the GMRES tick measured fastest,
  // pass C having just written P in that order).  SS_SPMV_SCHED=1: anchor schedule --
  // anchor(node) = smallest vertex of any element containing it (the generators number vertices
  // coherently in space, so rows with close anchors share columns); rows sorted by anchor are cut
  // into the saddle block count with balanced gather work, velocity rows first inside a block
  // (3% faster standalone SpMV, 2% slower inside the tick).  Results never depend on it: every
  // (row, mode) sum is still formed by one thread in CSR order.
  {
    std::vector<int> anchor(n_vel_nodes, INT32_MAX);
    for (int64_t e = 0; e < n_elements; ++e) {
      int mv = INT32_MAX;
      for (int a = 0; a < nvloc; ++a) mv = std::min(mv, (int)vel_conn[e * nloc + a]);
      for (int a = 0; a < nloc; ++a) {
        int& an = anchor[vel_conn[e * nloc + a]];
        an = std::min(an, mv);
      }
    }
    const int nitems = nfree + npf;
    std::vector<int64_t> key(nitems);
    for (int r = 0; r < nfree; ++r) key[r] = ((int64_t)anchor[P->free_nodes[r]] << 32) | (int64_t)r;
    for (int j = 0; j < npf; ++j) key[nfree + j] = ((int64_t)anchor[P->pres_of_row[j]] << 32) | (int64_t)(nfree + j);
    std::sort(key.begin(), key.end());
    std::vector<int> items(nitems);
    std::vector<double> wsum(nitems + 1, 0.0);
    for (int i = 0; i < nitems; ++i) {
      const int it = (int)(key[i] & 0xffffffff);
      items[i] = it;
      const double w = it < nfree ? (double)dim * (P->nptr[it + 1] - P->nptr[it]) + (P->pptr[it + 1] - P->pptr[it])
                                  : (double)dim * (P->tptr[it - nfree + 1] - P->tptr[it - nfree]);
      wsum[i + 1] = wsum[i] + w + 4.0;   // + per-row overhead
    }
    const int nsb = saddle_nsb_host(nfree, npf);
    P->sbptr.assign(nsb + 1, nitems);
    P->sbptr[0] = 0;
    int i = 0;
    for (int b = 1; b < nsb; ++b) {
      const double target = wsum[nitems] * b / nsb;
      while (i < nitems && wsum[i] < target) ++i;
      P->sbptr[b] = i;
    }
    for (int b = 0; b < nsb; ++b) std::sort(items.begin() + P->sbptr[b], items.begin() + P->sbptr[b + 1]);
    const char* sched = getenv("SS_SPMV_SCHED");
    if (!sched || atoi(sched) == 0) {   // default, natural order: 128 node rows / 32 pressure rows per block
      for (int q = 0; q < nitems; ++q) items[q] = q;
      const int nvb = (nfree + SPMV_VROWS - 1) / SPMV_VROWS;
      for (int b = 0; b < nsb; ++b)
        P->sbptr[b] = b < nvb ? b * SPMV_VROWS : std::min(nfree + (b - nvb) * SPMV_PROWS, nitems);
      P->sbptr[nsb] = nitems;
    }
    P->sitems = items;
  }

  // Chunks of the TMA-staged row-layout SpMV: consecutive rows while the chunk's staged matrix
  // ranges fit one shared-memory stage (ss_spmv.cuh stream_layout), at most STREAM_VROWS node rows
  // / STREAM_PROWS pressure rows.  A row too large for a stage disables the staged path.
  {
    P->crow.clear();
    P->cent.clear();
    bool fits = true;
    auto vel_ent = [&](int r0, int r1) {
      return make_int4(P->nptr[r0], P->nptr[r1], P->pptr[r0], P->pptr[r1]);
    };
    auto pres_ent = [&](int j0, int j1) { return make_int4(P->tptr[j0], P->tptr[j1], 0, 0); };
    for (int r = 0; r < nfree && fits;) {
      int r1 = r + 1;
      if (stream_layout(vel_ent(r, r1), true, dim).bytes > STREAM_STAGE_BYTES) { fits = false; break; }
      while (r1 < nfree && r1 - r < STREAM_VROWS &&
             stream_layout(vel_ent(r, r1 + 1), true, dim).bytes <= STREAM_STAGE_BYTES) ++r1;
      P->crow.push_back(make_int2(r, r1));
      P->cent.push_back(vel_ent(r, r1));
      r = r1;
    }
    const int nvchunk = (int)P->crow.size();
    for (int j = 0; j < npf && fits;) {
      int j1 = j + 1;
      if (stream_layout(pres_ent(j, j1), false, dim).bytes > STREAM_STAGE_BYTES) { fits = false; break; }
      while (j1 < npf && j1 - j < STREAM_PROWS &&
             stream_layout(pres_ent(j, j1 + 1), false, dim).bytes <= STREAM_STAGE_BYTES) ++j1;
      P->crow.push_back(make_int2(j, j1));
      P->cent.push_back(pres_ent(j, j1));
      j = j1;
    }
    if (!fits || (int64_t)P->pcol.size() * dim >= INT32_MAX || (int64_t)P->tcol.size() * dim >= INT32_MAX) {
      P->crow.clear();
      P->cent.clear();
      P->nvchunk = 0;
    } else {
      P->nvchunk = nvchunk;
    }
  }

  // Constrained rows a_full[fixed_idx] (assembly.py:471-476,491): rows of fixed velocity nodes
  // (all node / vertex neighbours, global ids) and, if the pressure is pinned, the row of vertex 0.
  {
    std::vector<int> fixed;
    for (int64_t A = 0; A < n_vel_nodes; ++A) if (P->rank[A] < 0) fixed.push_back((int)A);
    P->fixed_nodes = fixed;
    P->frank.assign(n_vel_nodes, -1);
    for (size_t i = 0; i < fixed.size(); ++i) P->frank[fixed[i]] = (int)i;
    std::vector<std::vector<int>> xn, xv, pin;
    collect_rows(fixed, inc_ptr, inc, vel_conn, nloc, nloc, xn);
    collect_rows(fixed, inc_ptr, inc, vel_conn, nloc, nvloc, xv);
    P->xptr.assign(fixed.size() + 1, 0);
    P->xpptr.assign(fixed.size() + 1, 0);
    for (size_t i = 0; i < fixed.size(); ++i) {
      P->xptr[i + 1] = P->xptr[i] + (int)xn[i].size();
      P->xpptr[i + 1] = P->xpptr[i] + (int)xv[i].size();
    }
    for (size_t i = 0; i < fixed.size(); ++i) {
      P->xcol.insert(P->xcol.end(), xn[i].begin(), xn[i].end());
      P->xpcol.insert(P->xpcol.end(), xv[i].begin(), xv[i].end());
    }
    if (P->pinned) {
      std::vector<int> v0 = {0};
      collect_rows(v0, inc_ptr, inc, vel_conn, nloc, nloc, pin);
      P->pincol = pin[0];
    }
  }

  // Element -> slot maps: [vv nloc*nloc][vp nloc*nvloc][pv nvloc*nloc] per element.
  // Codes: >= 0 free-row slot, <= -2 Dirichlet-lift slot, >= SS_FIXED_BASE constrained-row slot
  // (fixed velocity rows for vv/vp, the pinned pressure row for pv), -1 unused.
  const int per = nloc * nloc + 2 * nloc * nvloc;
  P->emap_stride = per;
  P->emap.assign((size_t)n_elements * per, -1);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < n_elements; ++e) {
    const int64_t* c = vel_conn + e * nloc;
    int* m = P->emap.data() + (size_t)e * per;
    for (int a = 0; a < nloc; ++a) {
      const int A = (int)c[a], rA = P->rank[A];
      for (int b = 0; b < nloc; ++b) {
        const int B = (int)c[b], rB = P->rank[B];
        int s = -1;
        if (rA >= 0) {
          if (rB >= 0) {
            s = P->nptr[rA] + lb(P->ncol.data() + P->nptr[rA], P->nptr[rA + 1] - P->nptr[rA], rB);
          } else {
            s = -(2 + P->lptr[rA] + lb(P->lcol.data() + P->lptr[rA], P->lptr[rA + 1] - P->lptr[rA], B));
          }
        } else {
          const int f = P->frank[A];
          s = SS_FIXED_BASE + P->xptr[f] + lb(P->xcol.data() + P->xptr[f], P->xptr[f + 1] - P->xptr[f], B);
        }
        m[a * nloc + b] = s;
      }
      for (int q = 0; q < nvloc; ++q) {
        const int pd = P->vert_pdof[c[q]];
        int s = -1;
        if (rA >= 0 && pd >= 0) {
          s = P->pptr[rA] + lb(P->pcol.data() + P->pptr[rA], P->pptr[rA + 1] - P->pptr[rA], pd);
        } else if (rA < 0) {
          const int f = P->frank[A];
          s = SS_FIXED_BASE + P->xpptr[f] + lb(P->xpcol.data() + P->xpptr[f], P->xpptr[f + 1] - P->xpptr[f], (int)c[q]);
        }
        m[nloc * nloc + a * nvloc + q] = s;
      }
    }
    for (int q = 0; q < nvloc; ++q) {
      const int pd = P->vert_pdof[c[q]];
      for (int a = 0; a < nloc; ++a) {
        const int A = (int)c[a], rA = P->rank[A];
        int s = -1;
        if (pd >= 0) {
          if (rA >= 0)
            s = P->tptr[pd] + lb(P->tcol.data() + P->tptr[pd], P->tptr[pd + 1] - P->tptr[pd], rA);
          else
            s = -(2 + P->ltptr[pd] + lb(P->ltcol.data() + P->ltptr[pd], P->ltptr[pd + 1] - P->ltptr[pd], A));
        } else if (P->pinned && c[q] == 0) {
          s = SS_FIXED_BASE + lb(P->pincol.data(), (int)P->pincol.size(), A);
        }
        m[nloc * nloc + nloc * nvloc + q * nloc + a] = s;
      }
    }
  }

  // Greedy vertex-conflict colouring: elements of one colour share no vertex, hence no slot.
  {
    const int W = 8;  // up to 512 colours
    std::vector<uint64_t> used((size_t)n_vertices * W, 0);
    std::vector<int> color(n_elements);
    int ncolors = 0;
    for (int64_t e = 0; e < n_elements; ++e) {
      uint64_t m[W] = {0};
      for (int a = 0; a < nvloc; ++a) {
        const uint64_t* u = used.data() + (size_t)vel_conn[e * nloc + a] * W;
        for (int w = 0; w < W; ++w) m[w] |= u[w];
      }
      int col = -1;
      for (int w = 0; w < W && col < 0; ++w)
        if (~m[w]) col = w * 64 + __builtin_ctzll(~m[w]);
      if (col < 0) { delete P; ss_set_error("element colouring exceeded 512 colours"); return SS_ERR_MESH; }
      color[e] = col;
      ncolors = std::max(ncolors, col + 1);
      for (int a = 0; a < nvloc; ++a) used[(size_t)vel_conn[e * nloc + a] * W + col / 64] |= 1ull << (col % 64);
    }
    P->color_ptr.assign(ncolors + 1, 0);
    for (int64_t e = 0; e < n_elements; ++e) P->color_ptr[color[e] + 1]++;
    for (int k = 0; k < ncolors; ++k) P->color_ptr[k + 1] += P->color_ptr[k];
    P->color_elems.resize(n_elements);
    std::vector<int> fill(P->color_ptr.begin(), P->color_ptr.end() - 1);
    for (int64_t e = 0; e < n_elements; ++e) P->color_elems[fill[color[e]]++] = (int)e;
    P->ncolors = ncolors;
  }

  // Device copies.
  std::vector<int> conn32((size_t)n_elements * nloc);
  for (size_t i = 0; i < conn32.size(); ++i) conn32[i] = (int)vel_conn[i];
  int rc = SS_OK;
  SsOperatorDev& op = P->op;
  op.dim = dim; op.nfree = nfree; op.npf = npf; op.nfv = nfree * dim; op.n = nfree * dim + npf;
  op.nnz_n = P->ncol.size(); op.nnz_p = P->pcol.size(); op.nnz_t = P->tcol.size();
  int *d;
#define UP(vec, field) do { rc = upload(P, vec, &d); if (rc) { delete P; return rc; } op.field = d; } while (0)
  UP(P->nptr, nptr); UP(P->ncol, ncol); UP(P->diag_slot, diag_slot);
  UP(P->pptr, pptr); UP(P->pcol, pcol); UP(P->tptr, tptr); UP(P->tcol, tcol);
  UP(P->lptr, lptr); UP(P->lcol, lcol); UP(P->ltptr, ltptr); UP(P->ltcol, ltcol);
  UP(P->free_nodes, free_nodes); UP(P->rank, node_rank); UP(P->pres_of_row, pres_of_row);
  UP(P->vert_pdof, vert_pdof);
  UP(P->sitems, sitems); UP(P->sbptr, sbptr);
#undef UP
  {
    int2* dcrow = nullptr;
    int4* dcent = nullptr;
    if ((rc = upload(P, P->crow, &dcrow)) || (rc = upload(P, P->cent, &dcent))) { delete P; return rc; }
    op.crow = dcrow;
    op.cent = dcent;
    op.nvchunk = P->nvchunk;
    op.nchunk = (int)P->crow.size();
  }
  if ((rc = upload(P, conn32, &P->d_conn))) { delete P; return rc; }
  if ((rc = upload(P, P->emap, &P->d_emap))) { delete P; return rc; }
  if ((rc = upload(P, P->color_elems, &P->d_color_elems))) { delete P; return rc; }
  if ((rc = alloc_zero(P, op.nnz_n, &op.sm))) { delete P; return rc; }
  if ((rc = alloc_zero(P, (size_t)nfree, &op.dsm))) { delete P; return rc; }
  if ((rc = alloc_zero(P, op.nnz_p * dim, &op.dp))) { delete P; return rc; }
  if ((rc = alloc_zero(P, op.nnz_t * dim, &op.dt))) { delete P; return rc; }
  if ((rc = alloc_zero(P, P->lcol.size(), &op.lsm))) { delete P; return rc; }
  if ((rc = alloc_zero(P, P->ltcol.size() * dim, &op.ldt))) { delete P; return rc; }
  if ((rc = alloc_zero(P, (size_t)n_vertices * dim, &P->d_vnodes))) { delete P; return rc; }
  if ((rc = alloc_zero(P, P->xcol.size(), &P->d_xsm))) { delete P; return rc; }
  if ((rc = alloc_zero(P, P->xpcol.size() * dim, &P->d_xdp))) { delete P; return rc; }
  if ((rc = alloc_zero(P, P->pincol.size() * dim, &P->d_pinv))) { delete P; return rc; }
  if ((rc = alloc_zero(P, 4, &P->d_flag))) { delete P; return rc; }
  *out = P;
  return SS_OK;
}

extern "C" void ss_pattern_destroy(ss_pattern* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  for (void* p : P->allocs) cudaFree(p);
  delete P;
}

// info: [n, nnz_vec, nfree, npf, nnz_n, nnz_p, nnz_t, ncolors, nnz_lift, nnz_lift_t, dim, pinned,
//        emap_bytes, nvn, nvert, ne]
extern "C" int ss_pattern_info(const ss_pattern* P, int64_t* info) {
  if (!P || !info) { ss_set_error("null argument"); return SS_ERR_ARG; }
  const int64_t dim = P->dim;
  info[0] = P->op.n;
  info[1] = dim * (P->op.nnz_n + P->op.nnz_p) + dim * P->op.nnz_t;
  info[2] = P->nfree; info[3] = P->npf;
  info[4] = P->op.nnz_n; info[5] = P->op.nnz_p; info[6] = P->op.nnz_t;
  info[7] = P->ncolors; info[8] = (int64_t)P->lcol.size(); info[9] = (int64_t)P->ltcol.size();
  info[10] = dim; info[11] = P->pinned; info[12] = (int64_t)P->emap.size() * 4;
  info[13] = P->nvn; info[14] = P->nvert; info[15] = P->ne;
  return SS_OK;
}

// Vector CSR of the reduced matrix, bit-identical to the reference's matrix.indptr/indices.
extern "C" int ss_pattern_export(const ss_pattern* P, int32_t* indptr, int32_t* indices) {
  if (!P || !indptr) { ss_set_error("null argument"); return SS_ERR_ARG; }
  const int dim = P->dim, nfv = P->nfree * dim;
  int64_t pos = 0;
  int64_t row = 0;
  indptr[0] = 0;
  for (int r = 0; r < P->nfree; ++r) {
    for (int d = 0; d < dim; ++d) {
      if (indices) {
        for (int e = P->nptr[r]; e < P->nptr[r + 1]; ++e) indices[pos++] = P->ncol[e] * dim + d;
        for (int e = P->pptr[r]; e < P->pptr[r + 1]; ++e) indices[pos++] = nfv + P->pcol[e];
      } else {
        pos += (P->nptr[r + 1] - P->nptr[r]) + (P->pptr[r + 1] - P->pptr[r]);
      }
      indptr[++row] = (int32_t)pos;
    }
  }
  for (int j = 0; j < P->npf; ++j) {
    for (int e = P->tptr[j]; e < P->tptr[j + 1]; ++e)
      for (int d = 0; d < dim; ++d) {
        if (indices) indices[pos] = P->tcol[e] * dim + d;
        pos++;
      }
    indptr[++row] = (int32_t)pos;
  }
  return SS_OK;
}

// vel_dof (nvn x dim) and pres_dof (nvert) as in ComplexSaddleSystem (assembly.py:319-320).
extern "C" int ss_pattern_dof_maps(const ss_pattern* P, int64_t* vel_dof, int64_t* pres_dof) {
  if (!P || !vel_dof || !pres_dof) { ss_set_error("null argument"); return SS_ERR_ARG; }
  for (int64_t A = 0; A < P->nvn; ++A)
    for (int d = 0; d < P->dim; ++d)
      vel_dof[A * P->dim + d] = P->rank[A] >= 0 ? (int64_t)P->rank[A] * P->dim + d : -1;
  const int64_t nfv = (int64_t)P->nfree * P->dim;
  for (int64_t v = 0; v < P->nvert; ++v) pres_dof[v] = P->vert_pdof[v] >= 0 ? nfv + P->vert_pdof[v] : -1;
  return SS_OK;
}

// ------------------------------------------------------------------------------------------------
// Consistent traction load on a Neumann patch (restates assembly.py:265-305; host, boundary only).
// h_kind: 0 = uniform (dim complex), 1 = per face (nfaces x dim), 2 = nodal (nvn x dim).
// Accumulates into load (nvn x dim complex) face by face, node by node, like np.add.at.
// ------------------------------------------------------------------------------------------------
extern "C" int ss_surface_load(int dim, int64_t nvn, const double* nodes, int64_t nfaces,
                               const int64_t* face_conn, int h_kind, const double* h, double* load) {
  if ((dim != 2 && dim != 3) || (nfaces > 0 && (!nodes || !face_conn || !h || !load))) {
    ss_set_error("ss_surface_load: bad arguments");
    return SS_ERR_ARG;
  }
  const int nfl = dim == 2 ? 3 : 6;
  double w[6], vals[6][6];
  int nq;
  if (dim == 2) {
    const double g = std::sqrt(3.0 / 5.0);
    const double t[3] = {0.5 * (1 - g), 0.5 * 1.0, 0.5 * (1 + g)};
    nq = 3;
    for (int q = 0; q < 3; ++q) {
      w[q] = (q == 1 ? 8.0 : 5.0) / 18.0;
      vals[q][0] = (1 - t[q]) * (1 - 2 * t[q]);
      vals[q][1] = t[q] * (2 * t[q] - 1);
      vals[q][2] = 4 * t[q] * (1 - t[q]);
    }
  } else {
    const double A[2] = {0.445948490915965, 0.091576213509771};
    const double Wt[2] = {0.223381589678011, 0.109951743655322};
    nq = 6;
    for (int q = 0; q < 6; ++q) {
      const double a = A[q / 3];
      double l[3] = {a, a, a};
      l[q % 3] = 1 - 2 * a;
      w[q] = 0.5 * Wt[q / 3];
      // points are (l1, l2) with l0 = 1 - l1 - l2; the P2 triangle basis in VTK order
      const double x = l[1], y = l[2];
      const double L[3] = {1.0 - (x + y), x, y};
      for (int v = 0; v < 3; ++v) vals[q][v] = L[v] * (2.0 * L[v] - 1.0);
      const int E[3][2] = {{0, 1}, {1, 2}, {2, 0}};
      for (int k = 0; k < 3; ++k) vals[q][3 + k] = 4.0 * L[E[k][0]] * L[E[k][1]];
    }
  }
  double ref_int[6] = {0};
  for (int a = 0; a < nfl; ++a)
    for (int q = 0; q < nq; ++q) ref_int[a] += w[q] * vals[q][a];
  for (int64_t f = 0; f < nfaces; ++f) {
    const int64_t* c = face_conn + f * nfl;
    for (int a = 0; a < nfl; ++a)
      if (c[a] < 0 || c[a] >= nvn) { ss_set_error("face_conn out of range"); return SS_ERR_MESH; }
    double jac;
    const double* p0 = nodes + c[0] * dim;
    const double* p1 = nodes + c[1] * dim;
    if (dim == 2) {
      jac = std::hypot(p1[0] - p0[0], p1[1] - p0[1]);
    } else {
      const double* p2 = nodes + c[2] * dim;
      const double e1[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
      const double e2[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
      const double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                            e1[0] * e2[1] - e1[1] * e2[0]};
      jac = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
    }
    for (int a = 0; a < nfl; ++a) {
      for (int d = 0; d < dim; ++d) {
        double re, im;
        if (h_kind == 0 || h_kind == 1) {
          const double* hv = h + 2 * ((h_kind == 1 ? f * dim : 0) + d);
          const double s = jac * ref_int[a];
          re = s * hv[0];
          im = s * hv[1];
        } else {
          double acc_re = 0, acc_im = 0;
          for (int q = 0; q < nq; ++q) {
            double hq_re = 0, hq_im = 0;
            for (int b = 0; b < nfl; ++b) {
              hq_re += vals[q][b] * h[2 * (c[b] * dim + d)];
              hq_im += vals[q][b] * h[2 * (c[b] * dim + d) + 1];
            }
            acc_re += w[q] * vals[q][a] * hq_re;
            acc_im += w[q] * vals[q][a] * hq_im;
          }
          re = jac * acc_re;
          im = jac * acc_im;
        }
        load[2 * (c[a] * dim + d)] += re;
        load[2 * (c[a] * dim + d) + 1] += im;
      }
    }
  }
  return SS_OK;
}

// Column indices of selected rows of the reduced vector CSR (same order as ss_pattern_export), for
// sampled parity checks on meshes too large to export whole.  counts[i] = nnz of rows[i];
// indices receives the concatenated columns (capacity cap); returns SS_ERR_ARG if cap is short.
extern "C" int ss_pattern_export_rows(const ss_pattern* P, int64_t nrows, const int64_t* rows, int64_t* counts,
                                      int32_t* indices, int64_t cap) {
  if (!P || (nrows > 0 && (!rows || !counts))) { ss_set_error("null argument"); return SS_ERR_ARG; }
  const int dim = P->dim, nfv = P->nfree * dim;
  int64_t pos = 0;
  for (int64_t i = 0; i < nrows; ++i) {
    const int64_t row = rows[i];
    if (row < 0 || row >= (int64_t)nfv + P->npf) { ss_set_error("row out of range"); return SS_ERR_ARG; }
    int64_t c = 0;
    if (row < nfv) {
      const int r = (int)(row / dim), d = (int)(row % dim);
      c = (P->nptr[r + 1] - P->nptr[r]) + (P->pptr[r + 1] - P->pptr[r]);
      if (indices) {
        if (pos + c > cap) { ss_set_error("index buffer too small"); return SS_ERR_ARG; }
        for (int e = P->nptr[r]; e < P->nptr[r + 1]; ++e) indices[pos++] = P->ncol[e] * dim + d;
        for (int e = P->pptr[r]; e < P->pptr[r + 1]; ++e) indices[pos++] = nfv + P->pcol[e];
      }
    } else {
      const int j = (int)(row - nfv);
      c = (int64_t)dim * (P->tptr[j + 1] - P->tptr[j]);
      if (indices) {
        if (pos + c > cap) { ss_set_error("index buffer too small"); return SS_ERR_ARG; }
        for (int e = P->tptr[j]; e < P->tptr[j + 1]; ++e)
          for (int dd = 0; dd < dim; ++dd) indices[pos++] = P->tcol[e] * dim + dd;
      }
    }
    counts[i] = c;
  }
  return SS_OK;
}


// Constrained rows a_full[fixed_idx] in the unreduced numbering (assembly.py:471-476,491): one row
// per (fixed node, component) in ascending order, then the pinned pressure row if any.  Columns are
// sorted full indices (velocity B*dim+d, pressure n_vel_nodes*dim + P); explicit zeros kept.
// indptr (nrows+1) / indices / data (complex) may be NULL to query sizes via info_out[2] = {nrows, nnz}.
extern "C" int ss_constrained_rows(const ss_pattern* P, double omega, int64_t* info_out, int64_t* indptr,
                                   int32_t* indices, double* data) {
  if (!P || !info_out) { ss_set_error("null argument"); return SS_ERR_ARG; }
  if (!P->assembled) { ss_set_error("pattern not assembled"); return SS_ERR_STATE; }
  const int dim = P->dim;
  const int64_t nf = (int64_t)P->fixed_nodes.size();
  const int64_t nrows = nf * dim + (P->pinned ? 1 : 0);
  const int64_t nnz = (int64_t)dim * ((int64_t)P->xcol.size() + (int64_t)P->xpcol.size()) +
                      (int64_t)dim * (int64_t)P->pincol.size();
  info_out[0] = nrows;
  info_out[1] = nnz;
  if (!indptr || !indices || !data) return SS_OK;
  std::vector<double2> xsm(P->xcol.size());
  std::vector<double> xdp(P->xpcol.size() * dim), pinv(P->pincol.size() * dim);
  if (!xsm.empty()) SS_CUDA(cudaMemcpy(xsm.data(), P->d_xsm, sizeof(double2) * xsm.size(), cudaMemcpyDeviceToHost));
  if (!xdp.empty()) SS_CUDA(cudaMemcpy(xdp.data(), P->d_xdp, sizeof(double) * xdp.size(), cudaMemcpyDeviceToHost));
  if (!pinv.empty()) SS_CUDA(cudaMemcpy(pinv.data(), P->d_pinv, sizeof(double) * pinv.size(), cudaMemcpyDeviceToHost));
  const int64_t pbase = P->nvn * dim;
  int64_t pos = 0, row = 0;
  indptr[0] = 0;
  for (int64_t i = 0; i < nf; ++i) {
    for (int d = 0; d < dim; ++d) {
      for (int e = P->xptr[i]; e < P->xptr[i + 1]; ++e) {
        indices[pos] = (int32_t)((int64_t)P->xcol[e] * dim + d);
        data[2 * pos] = xsm[e].x;
        data[2 * pos + 1] = omega == 0.0 ? 0.0 : omega * xsm[e].y;
        ++pos;
      }
      for (int e = P->xpptr[i]; e < P->xpptr[i + 1]; ++e) {
        indices[pos] = (int32_t)(pbase + P->xpcol[e]);
        data[2 * pos] = xdp[(size_t)e * dim + d];
        data[2 * pos + 1] = 0.0;
        ++pos;
      }
      indptr[++row] = pos;
    }
  }
  if (P->pinned) {
    for (size_t e = 0; e < P->pincol.size(); ++e)
      for (int d = 0; d < dim; ++d) {
        indices[pos] = (int32_t)((int64_t)P->pincol[e] * dim + d);
        data[2 * pos] = pinv[e * dim + d];
        data[2 * pos + 1] = 0.0;
        ++pos;
      }
    indptr[++row] = pos;
  }
  return SS_OK;
}
