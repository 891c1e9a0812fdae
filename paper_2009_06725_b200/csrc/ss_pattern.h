// Opaque pattern handle (host + device halves).  Internal to the library.
#pragma once
#include <vector>

#include "ss_common.h"

constexpr int SS_FIXED_BASE = 1 << 30;   // element-map code offset of constrained-row slots

struct ss_pattern {
  int device = 0;
  int dim = 0, nloc = 0, nvloc = 0;
  int64_t nvn = 0, nvert = 0, ne = 0;
  int pinned = 0;
  int nfree = 0, npf = 0, ncolors = 0;
  int emap_stride = 0;
  std::vector<int> rank, free_nodes, vert_pdof, pres_of_row;
  std::vector<int> nptr, ncol, pptr, pcol, tptr, tcol, lptr, lcol, ltptr, ltcol, diag_slot;
  std::vector<int> emap, color_ptr, color_elems;
  // constrained rows (fixed velocity nodes; pinned pressure row)
  std::vector<int> fixed_nodes, frank, xptr, xcol, xpptr, xpcol, pincol;
  std::vector<int> sitems, sbptr;   // SpMV locality schedule (ss_common.h SsOperatorDev)
  std::vector<int2> crow;           // staged-SpMV chunks (ss_spmv.cuh saddle_stream)
  std::vector<int4> cent;
  int nvchunk = 0;
  double2* d_xsm = nullptr;
  double* d_xdp = nullptr;
  double* d_pinv = nullptr;
  // device
  SsOperatorDev op{};
  int* d_conn = nullptr;         // int32 vel_conn
  int* d_emap = nullptr;
  int* d_color_elems = nullptr;
  double* d_vnodes = nullptr;    // vertex coordinates (nvert x dim)
  int* d_flag = nullptr;         // [0] = degenerate-element flag
  double density = 0, viscosity = 0;
  bool assembled = false;
  std::vector<void*> allocs;
};
