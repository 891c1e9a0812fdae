// Mode-field collective over NCCL (NVLink/NVSwitch on one node), behind the C ABI.
//
// The reference solves modes on a host thread pool and keeps every ModeSolution in one process
// (spectral.py:296-305).  Sharded over GPUs (one process per GPU) the only data
// movement is gathering the solved complex modal fields to the rank that reconstructs: one grouped
// ncclSend/ncclRecv round per gather, each field landing directly in its global mode slot on the
// root (no staging buffer, no reorder pass).
//
// NCCL is opened with dlopen at first use (SS_NCCL_LIB or "libnccl.so.2"), so the library has no
// link-time NCCL dependency and shares the process's already-loaded NCCL (e.g. PyTorch's).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "spectralstokes_b200.h"
#include "ss_common.h"

namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  ncclResult_t (*getVersion)(int*) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;
std::string g_nccl_path;

int nccl_load() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.handle) return SS_OK;
  const char* env = getenv("SS_NCCL_LIB");
  const char* path = env && *env ? env : "libnccl.so.2";
  void* h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    ss_set_error(std::string("cannot load NCCL (") + path + "): " + dlerror());
    return SS_ERR_CUDA;
  }
  NcclApi api;
  api.handle = h;
  bool ok = true;
  auto sym = [&](const char* name) {
    void* p = dlsym(h, name);
    if (!p) ok = false;
    return p;
  };
  api.getUniqueId = (decltype(api.getUniqueId))sym("ncclGetUniqueId");
  api.commInitRank = (decltype(api.commInitRank))sym("ncclCommInitRank");
  api.commDestroy = (decltype(api.commDestroy))sym("ncclCommDestroy");
  api.groupStart = (decltype(api.groupStart))sym("ncclGroupStart");
  api.groupEnd = (decltype(api.groupEnd))sym("ncclGroupEnd");
  api.send = (decltype(api.send))sym("ncclSend");
  api.recv = (decltype(api.recv))sym("ncclRecv");
  api.allReduce = (decltype(api.allReduce))sym("ncclAllReduce");
  api.reduce = (decltype(api.reduce))sym("ncclReduce");
  api.errorString = (decltype(api.errorString))sym("ncclGetErrorString");
  api.getVersion = (decltype(api.getVersion))sym("ncclGetVersion");
  if (!ok) {
    ss_set_error(std::string("NCCL library ") + path + " lacks a required symbol");
    dlclose(h);
    return SS_ERR_CUDA;
  }
  g_nccl = api;
  g_nccl_path = path;
  return SS_OK;
}

#define SS_NCCL(call)                                                                        \
  do {                                                                                       \
    ncclResult_t _r = (call);                                                                \
    if (_r != ncclSuccess) {                                                                 \
      ss_set_error(std::string("NCCL error: ") + g_nccl.errorString(_r) + " at " + __FILE__ + \
                   ":" + std::to_string(__LINE__));                                          \
      return SS_ERR_CUDA;                                                                    \
    }                                                                                        \
  } while (0)

}  // namespace

struct ss_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0, device = 0;
};

extern "C" int ss_comm_nccl_version(void) {
  if (nccl_load()) return -1;
  int v = 0;
  if (g_nccl.getVersion(&v) != ncclSuccess) return -1;
  return v;
}

extern "C" int ss_comm_unique_id(uint8_t* id_out) {
  if (!id_out) { ss_set_error("null argument"); return SS_ERR_ARG; }
  int rc = nccl_load();
  if (rc) return rc;
  ncclUniqueId id;
  SS_NCCL(g_nccl.getUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == SS_COMM_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof(id));
  return SS_OK;
}

extern "C" int ss_comm_create(int nranks, int rank, const uint8_t* id, int device, ss_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  int rc = nccl_load();
  if (rc) return rc;
  SS_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ss_comm* c = new ss_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclResult_t r = g_nccl.commInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    ss_set_error(std::string("ncclCommInitRank: ") + g_nccl.errorString(r));
    delete c;
    return SS_ERR_CUDA;
  }
  *out = c;
  return SS_OK;
}

extern "C" void ss_comm_destroy(ss_comm* c) {
  if (!c) return;
  if (c->comm && g_nccl.commDestroy) {
    cudaSetDevice(c->device);
    g_nccl.commDestroy(c->comm);
  }
  delete c;
}

// Every rank sends its n_local fields (count complex values each, stride ld complex, from send);
// the root receives field j of rank r into recv + dest[off_r + j] * ld (complex), off_r =
// counts[0] + ... + counts[r-1].  One NCCL group: all transfers overlap on NVLink.
extern "C" int ss_comm_gather_modes(ss_comm* c, const double* send, int64_t n_local, int64_t count, int64_t ld,
                                    double* recv, const int64_t* counts, const int64_t* dest, int root,
                                    void* stream_) {
  if (!c || !counts || !dest || count < 0 || ld < count || root < 0 || root >= c->nranks) {
    ss_set_error("bad arguments");
    return SS_ERR_ARG;
  }
  if (n_local != counts[c->rank]) { ss_set_error("n_local does not match counts[rank]"); return SS_ERR_ARG; }
  if (n_local > 0 && !send) { ss_set_error("null send buffer"); return SS_ERR_ARG; }
  if (c->rank == root && !recv) { ss_set_error("null receive buffer on the root"); return SS_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream_;
  SS_CUDA(cudaSetDevice(c->device));
  const size_t words = (size_t)count * 2;   // complex128 as pairs of float64
  SS_NCCL(g_nccl.groupStart());
  int rc = SS_OK;
  if (c->rank == root) {
    int64_t off = 0;
    for (int r = 0; r < c->nranks && !rc; ++r) {
      for (int64_t j = 0; j < counts[r]; ++j) {
        double* dst = recv + (size_t)dest[off + j] * ld * 2;
        if (r == root) {
          if (cudaMemcpyAsync(dst, send + (size_t)j * ld * 2, words * sizeof(double), cudaMemcpyDeviceToDevice, st)
              != cudaSuccess) { rc = SS_ERR_CUDA; break; }
        } else if (g_nccl.recv(dst, words, ncclFloat64, r, c->comm, st) != ncclSuccess) {
          rc = SS_ERR_CUDA;
          break;
        }
      }
      off += counts[r];
    }
  } else {
    for (int64_t j = 0; j < n_local; ++j)
      if (g_nccl.send(send + (size_t)j * ld * 2, words, ncclFloat64, root, c->comm, st) != ncclSuccess) {
        rc = SS_ERR_CUDA;
        break;
      }
  }
  ncclResult_t ge = g_nccl.groupEnd();
  if (rc) { ss_set_error("NCCL send/recv or copy failed while posting the gather"); return rc; }
  if (ge != ncclSuccess) { ss_set_error(std::string("ncclGroupEnd: ") + g_nccl.errorString(ge)); return SS_ERR_CUDA; }
  return SS_OK;
}

// Elementwise max over ranks of n doubles (device buffer, in place): the bench's max-over-ranks timing.
extern "C" int ss_comm_allreduce_max(ss_comm* c, double* buf, int64_t n, void* stream_) {
  if (!c || (n > 0 && !buf)) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  SS_CUDA(cudaSetDevice(c->device));
  SS_NCCL(g_nccl.allReduce(buf, buf, (size_t)n, ncclFloat64, ncclMax, c->comm, (cudaStream_t)stream_));
  return SS_OK;
}

// Sum of n doubles over ranks into the root's buffer (in place on every rank's send buffer; the
// root's holds the result): per-GPU partial reconstructions -> the full u(x, t) on one rank.
extern "C" int ss_comm_reduce_sum(ss_comm* c, double* buf, int64_t n, int root, void* stream_) {
  if (!c || (n > 0 && !buf) || root < 0 || root >= c->nranks) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  SS_CUDA(cudaSetDevice(c->device));
  SS_NCCL(g_nccl.reduce(buf, buf, (size_t)n, ncclFloat64, ncclSum, root, c->comm, (cudaStream_t)stream_));
  return SS_OK;
}
