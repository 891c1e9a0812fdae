// Shared definitions for the spectral-Stokes B200 library (libss_b200.so).
//
// Layout conventions:
//  * complex128 values are double2 {re, im};
//  * per-mode vectors are mode-major: vec[b * ld + i], ld = round_up(n, 32) (padding rows are 0);
//  * reduced DOF numbering is the reference's (assembly.py:455-475): free velocity nodes in
//    ascending node order with interleaved components (rank*dim + d), then free pressures.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#define SS_OK 0
#define SS_ERR_ARG 1        // ValueError
#define SS_ERR_MESH 2       // MeshError
#define SS_ERR_CUDA 3       // DeviceError
#define SS_ERR_STATE 4      // RuntimeError (misuse)

void ss_set_error(const std::string& msg);
void ss_count_launch(int64_t n = 1);
int64_t ss_launch_counter();

#define SS_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess) {                                                                \
      ss_set_error(std::string("CUDA error ") + cudaGetErrorString(_e) + " at " + __FILE__ + \
                   ":" + std::to_string(__LINE__));                                         \
      return SS_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

#define SS_LAUNCH_CHECK()                                                                   \
  do {                                                                                      \
    ss_count_launch();                                                                      \
    cudaError_t _e = cudaGetLastError();                                                    \
    if (_e != cudaSuccess) {                                                                \
      ss_set_error(std::string("kernel launch failed: ") + cudaGetErrorString(_e) + " at " + \
                   __FILE__ + ":" + std::to_string(__LINE__));                              \
      return SS_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

// Device-resident structured saddle operator (one per mesh + fluid).  All arrays device.
struct SsOperatorDev {
  int dim;
  int nfree;        // free velocity nodes
  int npf;          // free pressure dofs
  int nfv;          // nfree * dim
  int n;            // nfv + npf
  int64_t nnz_n;    // free x free node pairs
  int64_t nnz_p;    // free node x free pressure pairs
  int64_t nnz_t;    // free pressure x free node pairs (transpose of nnz_p)
  // free x free node graph with (S', M') per pair; dsm = diagonal (S'_AA, M'_AA)
  const int* nptr; const int* ncol; double2* sm; double2* dsm; const int* diag_slot;
  // velocity rows -> pressure columns, D[(A,d),P] as dim doubles per pair
  const int* pptr; const int* pcol; double* dp;
  // pressure rows -> velocity node columns, D[(B,d),P] as dim doubles per pair
  const int* tptr; const int* tcol; double* dt;
  // Dirichlet lift: free node rows x fixed node columns (global node id), and pressure rows x
  // fixed node columns.
  const int* lptr; const int* lcol; double2* lsm;
  const int* ltptr; const int* ltcol; double* ldt;
  const int* free_nodes;   // rank -> node
  const int* node_rank;    // node -> rank or -1
  const int* pres_of_row;  // pressure dof j -> vertex
  const int* vert_pdof;    // vertex -> pressure dof (0..npf-1) or -1
  // Locality schedule of the mode-interleaved SpMV: block b processes rows sitems[sbptr[b] ..
  // sbptr[b+1]) (velocity node rank r, or nfree + pressure dof), rows grouped by anchor vertex so
  // that concurrently running blocks gather from one compact window of x.
  const int* sitems; const int* sbptr;
  // Chunks of the TMA-staged row-layout SpMV (ss_spmv.cuh saddle_stream): velocity chunks first
  // (crow = node-rank range, cent = {nptr range, pptr range}), then pressure chunks (crow = pressure
  // dof range, cent = {tptr range, -, -}); nchunk = 0 disables the staged path.
  const int2* crow; const int4* cent; int nvchunk, nchunk;
};

// Generic complex CSR operator (drop-in gmres(matrix, rhs) on arbitrary matrices).
struct SsCsrDev {
  int n;
  int64_t nnz;
  int nvals;                // number of value sets (1 = shared by all modes, else one per mode)
  const int* indptr; const int* indices; const double2* vals;  // vals[set * nnz + e]
  const double2* scale;     // optional per-set Jacobi scale [set * n + i] (nullptr = identity)
};

static inline int64_t ss_round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
