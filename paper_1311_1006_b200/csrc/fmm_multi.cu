// fmm-b200 — multi-GPU plumbing of the near field.
//
// The near field shards by target leaf with no data-path reduction: a leaf's
// potentials depend only on its evals and its strong list (reference
// backend.cpp:41-69).  A rank stages its shard halo-only (fmmcu_p2p_stage
// with leaf_begin/leaf_end: only the sources its strong lists read cross
// PCIe), runs the mutual kernel over its range, and its potentials reach the
// root by one of two routes:
//
//  * fused peer stores (default): the root exports its device output buffer
//    (cudaIpcGetMemHandle, fmmcu_p2p_out_ipc_handle); every other rank maps
//    it (fmmcu_p2p_bind_peer_out) and its finalize / TMA bulk stores write
//    the shard's slice straight into the root's HBM over NVLink, overlapped
//    with the compute -- the gather costs no extra pass and no collective;
//  * NCCL (fmmcu_nccl_*): a library-owned communicator over the job's ranks
//    (libnccl.so.2, loaded at run time -- the torch-bundled copy when it is
//    already mapped) and one grouped ncclSend / ncclRecv of every slice into
//    the root's buffer at its own offset (no padding, no extra copies),
//    enqueued on the context stream right behind the kernels.
//
// Both are plain device memory operations; neither falls back to the host.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "fmm_cuda.h"
#include "fmmcu_internal.cuh"

using fmmcu::detail::set_err;

namespace {

struct NcclApi {
  bool loaded = false;
  std::string err;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer a copy already mapped into the process (torch's), else load one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.loaded = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.send &&
                 api.recv && api.group_start && api.group_end && api.error_string;
    if (!api.loaded) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

#define NCCL_TRY(ctx, expr)                                                             \
  do {                                                                                 \
    ncclResult_t _r = (expr);                                                          \
    if (_r != ncclSuccess)                                                             \
      return set_err(ctx, FMMCU_ENCCL, std::string(#expr) + ": " + nccl().error_string(_r)); \
  } while (0)

}  // namespace

namespace fmmcu::detail {

// close the peer mapping and the communicator (fmmcu_destroy)
void multi_release(fmmcu_ctx* c) {
  if (c->peer_out) {
    if (c->ext_out == static_cast<double2*>(c->peer_out)) c->ext_out = nullptr;
    cudaIpcCloseMemHandle(c->peer_out);
    c->peer_out = nullptr;
  }
  if (c->nccl_comm) {
    nccl().comm_destroy(static_cast<ncclComm_t>(c->nccl_comm));
    c->nccl_comm = nullptr;
  }
}

}  // namespace fmmcu::detail

extern "C" {

int fmmcu_p2p_out_ipc_handle(fmmcu_ctx* c, void* handle) {
  if (!c || !handle) return FMMCU_EINVAL;
  if (!c->staged) return set_err(c, FMMCU_ESTATE, "no staged job");
  if (c->ext_out) return set_err(c, FMMCU_ESTATE, "output bound to external memory");
  CU_TRY(c, cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  CU_TRY(c, cudaIpcGetMemHandle(&h, c->d_out.p));
  static_assert(sizeof(h) == FMMCU_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof h);
  return FMMCU_OK;
}

int fmmcu_p2p_bind_peer_out(fmmcu_ctx* c, const void* handle) {
  if (!c) return FMMCU_EINVAL;
  CU_TRY(c, cudaSetDevice(c->device));
  if (c->peer_out) {
    if (c->ext_out == static_cast<double2*>(c->peer_out)) c->ext_out = nullptr;
    CU_TRY(c, cudaStreamSynchronize(c->stream));
    CU_TRY(c, cudaIpcCloseMemHandle(c->peer_out));
    c->peer_out = nullptr;
  }
  if (!handle) return FMMCU_OK;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void* p = nullptr;
  CU_TRY(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  c->peer_out = p;
  c->ext_out = static_cast<double2*>(p);
  return FMMCU_OK;
}

int fmmcu_nccl_unique_id(void* id) {
  if (!id) return FMMCU_EINVAL;
  NcclApi& api = nccl();
  if (!api.loaded) return FMMCU_ENCCL;
  ncclUniqueId u;
  if (api.get_unique_id(&u) != ncclSuccess) return FMMCU_ENCCL;
  static_assert(sizeof(u) == FMMCU_NCCL_ID_BYTES, "NCCL unique id size");
  std::memcpy(id, &u, sizeof u);
  return FMMCU_OK;
}

int fmmcu_nccl_init(fmmcu_ctx* c, const void* id, int rank, int world) {
  if (!c || !id || world < 1 || rank < 0 || rank >= world) return FMMCU_EINVAL;
  NcclApi& api = nccl();
  if (!api.loaded) return set_err(c, FMMCU_ENCCL, api.err);
  CU_TRY(c, cudaSetDevice(c->device));
  if (c->nccl_comm) {
    api.comm_destroy(static_cast<ncclComm_t>(c->nccl_comm));
    c->nccl_comm = nullptr;
  }
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclComm_t comm = nullptr;
  NCCL_TRY(c, api.comm_init_rank(&comm, world, u, rank));
  c->nccl_comm = comm;
  c->nccl_rank = rank;
  c->nccl_world = world;
  return FMMCU_OK;
}

int fmmcu_nccl_gather_out(fmmcu_ctx* c, int root, const uint32_t* eval_cuts) {
  if (!c || !eval_cuts) return FMMCU_EINVAL;
  if (!c->nccl_comm) return set_err(c, FMMCU_ESTATE, "no NCCL communicator (fmmcu_nccl_init)");
  if (!c->staged) return set_err(c, FMMCU_ESTATE, "no staged job");
  const int R = c->nccl_world, me = c->nccl_rank;
  if (root < 0 || root >= R) return set_err(c, FMMCU_EINVAL, "bad root");
  for (int r = 0; r < R; ++r)
    if (eval_cuts[r] > eval_cuts[r + 1] || eval_cuts[r + 1] > c->n_eval)
      return set_err(c, FMMCU_EINVAL, "bad eval cuts");
  NcclApi& api = nccl();
  CU_TRY(c, cudaSetDevice(c->device));
  auto comm = static_cast<ncclComm_t>(c->nccl_comm);
  double* out = reinterpret_cast<double*>(c->out_ptr());
  NCCL_TRY(c, api.group_start());
  if (me == root) {
    for (int r = 0; r < R; ++r) {
      if (r == root || eval_cuts[r + 1] == eval_cuts[r]) continue;
      NCCL_TRY(c, api.recv(out + 2 * size_t(eval_cuts[r]), 2 * size_t(eval_cuts[r + 1] - eval_cuts[r]),
                           ncclFloat64, r, comm, c->stream));
    }
  } else if (eval_cuts[me + 1] > eval_cuts[me]) {
    NCCL_TRY(c, api.send(out + 2 * size_t(eval_cuts[me]), 2 * size_t(eval_cuts[me + 1] - eval_cuts[me]),
                         ncclFloat64, root, comm, c->stream));
  }
  NCCL_TRY(c, api.group_end());
  return FMMCU_OK;
}

}  // extern "C"
