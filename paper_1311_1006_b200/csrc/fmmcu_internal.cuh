// fmm-b200 — internals shared by the translation units of libfmmcuda.so
// (fmmcu.cu: near field + M2L; fmm_device.cu: the device FMM pipeline).
// Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <functional>
#include <vector>

#include "fmm_cuda.h"
#include "p2p_kernels.cuh"
#include "p2p_warp.cuh"
#include "m2l_args.cuh"
#include "p2p_worklist_types.cuh"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace fmmcu {

// FMMCU_TRACE_SLOW: report buffer (re)allocations slower than 5 ms
inline void slow_alloc_note(const char* what, size_t bytes,
                            std::chrono::steady_clock::time_point t0,
                            std::chrono::steady_clock::time_point t1 =
                                std::chrono::steady_clock::time_point::max()) {
  static const bool on = std::getenv("FMMCU_TRACE_SLOW") != nullptr;
  if (!on) return;
  if (t1 == std::chrono::steady_clock::time_point::max()) t1 = std::chrono::steady_clock::now();
  const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  if (ms > 5.0) std::fprintf(stderr, "[fmmcu] slow %s allocation: %.1f MB in %.1f ms\n", what,
                             double(bytes) / 1e6, ms);
}

// The current device's default memory pool keeps what is freed into it
// (called before every DevBuf allocation; cheap after the first per device).
inline void keep_pool_memory() {
  static thread_local int done_mask = 0;  // devices 0..30
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev > 30) return;
  if (done_mask & (1 << dev)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~uint64_t(0);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    // Reserve the pool up front (FMMCU_POOL_RESERVE_GB, default 16; 0: off):
    // growing it maps new pages, 10-15 ms per GB and up to ~0.4 s for one
    // allocation under autotuned time stepping, where a level probe can need
    // a few GB of symmetric contributions at once.  One allocation + free
    // maps the memory once; later buffers are carved from it.  Failure is
    // ignored (the pool then grows on demand as before).
    const char* env = std::getenv("FMMCU_POOL_RESERVE_GB");
    const double gb = env ? std::atof(env) : 16.0;
    uint64_t have = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &have);
    const uint64_t want = uint64_t(gb * double(1ull << 30));
    if (want > have) {
      size_t free_b = 0, total_b = 0;
      if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && want - have < free_b / 2) {
        void* r = nullptr;
        if (cudaMallocAsync(&r, size_t(want - have), 0) == cudaSuccess) {
          cudaFreeAsync(r, 0);
          cudaStreamSynchronize(0);
        }
      }
    }
  }
  cudaGetLastError();
  done_mask |= 1 << dev;
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool plain = false;  // cudaMalloc (a buffer exported over CUDA IPC), not the pool
  // Grows only.  A buffer that has to grow again grows by at least half its
  // size: autotuned time stepping changes the level count and theta every few
  // steps, and each regrowth is a cudaFree (device-wide sync) + cudaMalloc.
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    const size_t grown = cap ? cap + cap / 2 : 0;
    const auto t0 = std::chrono::steady_clock::now();
    // Stream-ordered allocations from the device's default pool, which keeps
    // freed memory (release threshold raised once per device): regrowing a
    // buffer reuses pooled memory instead of mapping new pages, which took
    // up to hundreds of ms per cudaMalloc in autotuned time stepping.  The
    // old buffer may still be read by queued work on any stream, so the
    // device is synchronized before it goes back to the pool (as cudaFree
    // would); the new one is complete once the legacy stream is.
    if (p && plain) {
      cudaFree(p);
    } else if (p) {
      cudaDeviceSynchronize();
      cudaFreeAsync(p, 0);
    }
    const auto t1 = std::chrono::steady_clock::now();
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(std::max(bytes, grown), 256);
    cudaError_t e;
    if (plain) {
      e = cudaMalloc(&p, want);
    } else {
      keep_pool_memory();
      e = cudaMallocAsync(&p, want, 0);
      if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    }
    if (e == cudaSuccess) cap = want;
    slow_alloc_note("device free", want, t0, t1);
    slow_alloc_note("device malloc", want, t1);
    if (e == cudaSuccess && std::getenv("FMMCU_DEBUG_POISON")) e = cudaMemset(p, 0xFF, want);
    return e;
  }
  void release() {
    if (p && plain) {
      cudaFree(p);
    } else if (p) {
      cudaDeviceSynchronize();
      cudaFreeAsync(p, 0);
      cudaStreamSynchronize(0);
    }
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {  // grows only, by at least half (see DevBuf)
    if (bytes <= cap) return cudaSuccess;
    const size_t grown = cap ? cap + cap / 2 : 0;
    const auto t0 = std::chrono::steady_clock::now();
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(std::max(bytes, grown), 256);
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocPortable | cudaHostAllocMapped);
    if (e == cudaSuccess) cap = want;
    slow_alloc_note("pinned host", want, t0);
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// std::allocator replacement backed by pinned host memory: a vector built
// with it can be DMA'd without a staging copy.
template <class T>
struct PinnedAllocator {
  using value_type = T;
  PinnedAllocator() = default;
  template <class U>
  PinnedAllocator(const PinnedAllocator<U>&) {}
  T* allocate(std::size_t n) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocPortable) != cudaSuccess) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, std::size_t) { cudaFreeHost(p); }
  template <class U>
  bool operator==(const PinnedAllocator<U>&) const { return true; }
  template <class U>
  bool operator!=(const PinnedAllocator<U>&) const { return false; }
};
template <class T>
using pinned_vector = std::vector<T, PinnedAllocator<T>>;

using Clock = std::chrono::steady_clock;

// Host memcpy split across the OpenMP threads (pinned staging copies).
inline void par_memcpy(void* dst, const void* src, size_t bytes) {
  if (bytes < (size_t(1) << 22)) {
    if (bytes) std::memcpy(dst, src, bytes);
    return;
  }
  const int64_t blocks = int64_t((bytes + (size_t(1) << 20) - 1) >> 20);
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < blocks; ++b) {
    const size_t o = size_t(b) << 20;
    std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                std::min<size_t>(size_t(1) << 20, bytes - o));
  }
}

// True when [p, p + bytes) is page-locked host memory the DMA engines can read
// or write in place (cudaHostRegister'ed or cudaHostAlloc'ed at both ends).
inline bool host_locked(const void* p, size_t bytes) {
  if (!p || !bytes) return false;
  auto one = [](const void* q) {
    cudaPointerAttributes at{};
    const bool ok = cudaPointerGetAttributes(&at, q) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
  };
  return one(p) && one(static_cast<const char*>(p) + bytes - 1);
}

// Wait for a recorded event from a finish() call.  The host has nothing
// else to do there (the engine calls finish after its CPU far field), so it
// polls instead of sleeping: a blocking-sync wait wakes up ~0.3-0.5 ms after
// the event completes, which is ~5% of a 10M end-to-end near-field step.
// FMMCU_BLOCKING_SYNC=1 restores the sleeping wait.
inline cudaError_t wait_event(cudaEvent_t ev) {
  static const bool blocking = std::getenv("FMMCU_BLOCKING_SYNC") != nullptr;
  if (blocking) return cudaEventSynchronize(ev);
  for (;;) {
    const cudaError_t e = cudaEventQuery(ev);
    if (e != cudaErrorNotReady) return e;
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
}

struct DevicePipeline;  // fmm_device.cu
void destroy_pipeline(DevicePipeline* p);

}  // namespace fmmcu

using fmmcu::Clock;
using fmmcu::DevBuf;
using fmmcu::HostBuf;
using fmmcu::par_memcpy;
using fmmcu::P2PFinal;
using fmmcu::P2PItem;

struct fmmcu_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // current (own or external)
  cudaStream_t m2l_stream = nullptr;
  cudaStream_t d2h_stream = nullptr;  // potentials D2H, overlapping the next slice's kernels
  cudaStream_t wl_stream = nullptr;   // highest priority: the device pipeline's work-list build
  static constexpr int kMaxSlices = 8;
  cudaEvent_t ev_kslice[kMaxSlices] = {}, ev_cslice[kMaxSlices] = {};
  int n_slices = 0;
  uint32_t slice_eb[kMaxSlices + 1] = {};
  bool direct_out = false;  // job->out is page-locked: written in place
  // overlapped launch: upload chunks (leaf-aligned) and need-ordered groups
  cudaStream_t h2d_stream = nullptr;
  static constexpr int kMaxChunks = 32;
  cudaEvent_t ev_chunk[kMaxChunks] = {}, ev_group[kMaxChunks] = {};
  cudaEvent_t ev_prep[kMaxChunks] = {};  // chunk k prepared on the stream (two-stream groups)
  cudaEvent_t ev_fin[kMaxChunks] = {}, ev_copy[kMaxChunks] = {};  // grouped mutual: finalize k, D2H k
  cudaStream_t grp_stream[2] = {};       // group kernels alternate between these
  int n_groups = 0;
  cudaEvent_t ev_evals = nullptr;  // evals uploaded (overlapped launch, non-self layouts)
  cudaEvent_t ev_staged = nullptr;  // CSR + work list uploaded (overlapped launch)
  int group_k = 0;                      // > 0: build_worklist groups leaves by need chunk
  std::vector<uint32_t> chunk_leaf;     // [group_k + 1] leaf boundaries of the upload chunks
  std::vector<uint32_t> grp_pos;        // [group_k + 1] first position of each group
  bool grouped = false;                 // items / fins are in grouped order
  double2* out_dev = nullptr;           // device view of the launch's output (host memory)
  bool overlapped = false;              // the in-flight launch took launch_overlapped
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_m2l0 = nullptr, ev_m2l1 = nullptr;
  std::string err;
  uint64_t launches = 0;

  // staged job (device)
  DevBuf d_zin, d_min;  // caller z / m DMA'd as-is (page-locked inputs)
  DevBuf d_src, d_evy, d_eself, d_pt, d_ev, d_soff, d_sidx, d_items, d_fin, d_out, d_partial,
      d_hits, d_seg, d_counter, d_evr;
  // pinned staging
  HostBuf h_src, h_evy, h_eself, h_out, h_hits, h_csr;
  std::vector<uint32_t> invperm;
  // host mirror of the staged job
  uint32_t n_leaves = 0, n_src = 0, n_eval = 0;
  uint32_t n_strong = 0;  // strong entries of the finest CSR (device work list)
  int kernel = 0, smoother = 0, mode = 0;
  double delta = 0.0;
  std::vector<uint32_t> ev_off;        // host copy
  std::vector<uint64_t> leaf_work;     // prefix of nt * S
  fmmcu::pinned_vector<P2PItem> items;   // pinned: uploaded without a staging copy
  std::vector<uint32_t> item_first;    // [n_leaves + 1]
  fmmcu::pinned_vector<P2PFinal> fins;
  std::vector<uint32_t> fin_first;     // [n_leaves + 1]
  // work-list scratch kept across launches (no reallocation / page faults)
  std::vector<uint64_t> wl_S, wl_pev;
  std::vector<uint32_t> wl_kc, wl_order, wl_need;
  // mutual (symmetric) P2P for self-evaluation (p2p_sym.cuh)
  bool sym_request = false;             // caller: evals are the sources, harmonic, fast
  bool sym_items = false;               // the staged work list is symmetric
  uint32_t sym_lb = 0, sym_le = 0;      // leaf range the symmetric list covers
  std::vector<uint4> sym_seg;           // per-leaf entries: (slot, n, kind, 0)
  std::vector<uint32_t> sym_first;      // [range + 1] first entry of each leaf
  std::vector<uint4> sym_info;          // per leaf: first entry / item / slot, sym sources
  std::vector<uint32_t> sw_ent, sw_nblk;
  std::vector<uint64_t> sw_ssym, sw_sord, sw_slots;
  uint64_t sym_slots = 0;               // contrib slots
  bool no_sym_once = false;             // next overlapped launch: ordered list (self check failed)
  bool sym_grouped = false;             // symmetric list grouped by upload chunk
  const uint32_t* sym_order = nullptr;  // grouped: leaf position -> leaf (device)
  bool sym_rounds = false;              // some symmetric item has more than 32 entries
  uint32_t sym_n_items = 0;             // items of the symmetric list (host or device built)
  DevBuf d_wls;                         // device symmetric-list scratch
  DevBuf d_symseg, d_syminfo, d_symcnt, d_tgt, d_contrib, d_cloff, d_clcnt, d_clbase, d_cubtmp;
  HostBuf h_sym;
  // device-built work list (worklist_dev.cu): items / fins for [dev_wl_lb,
  // dev_wl_le) only, group ranges in dev_grp_item / dev_grp_fin
  bool dev_wl = false;          // the ordered list is device-built
  uint32_t dev_wl_lb = 0, dev_wl_le = 0;
  bool dev_list = false;        // the staged list (ordered or symmetric) is device-built
  uint64_t dev_list_total = 0;  // its range's sum of n_evals * |strong sources|
  std::vector<uint32_t> dev_grp_item, dev_grp_fin;
  DevBuf d_wl_head, d_wl_key, d_wl_val, d_wl_S, d_wl_work, d_wl_cnt, d_wl_off;
  HostBuf h_wl_head;
  bool staged = false;
  uint64_t staged_src = 0;     // source slots uploaded by the last stage (halo-only for a shard)
  bool self_layout = false;    // eval e is source slot e (EvalSet::self_of, perm == eval_perm)
  bool warp_items = false;     // work list built for p2p_warp_kernel
  int warp_e = 4;              // evals per lane of the warp kernel (choose_warp_e)
  uint64_t partial_evals = 0;  // partial-sum slots of split items
  bool trace = std::getenv("FMMCU_TRACE") != nullptr;
  double2* ext_out = nullptr;  // caller-bound output (torch tensor), or null
  double2* out_ptr() const { return ext_out ? ext_out : d_out.as<double2>(); }

  // in-flight reference-facing launch
  bool inflight = false;
  fmmcu_p2p_job job{};
  uint32_t run_lb = 0, run_le = 0;
  uint32_t run_eb = 0, run_ee = 0;  // eval slots of the in-flight overlapped launch
  double prep_seconds = 0.0;
  Clock::time_point t_evstart{};
  uint64_t run_total_pairs = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;

  // m2l
  DevBuf m_centers, m_coeffs, m_tbox, m_woff, m_widx, m_table, m_out, m_flag;
  DevBuf m_items, m_iscan, m_nitems, m_partial, m_cubtmp;  // m2l_run work items
  HostBuf mh_out, mh_flag;
  HostBuf mb_centers, mb_coeffs, mb_out, mb_tbox, mb_woff, mb_widx;  // fmmcu_m2l_host_buffers
  bool m2l_direct_out = false;  // the launched job's out is page-locked: D2H in place
  int table_p = -1, table_kernel = -1;
  bool m2l_inflight = false;
  fmmcu_m2l_job m2l_job{};
  bool m2l_keep = false;            // M2L sums left on the device (fmmcu_m2l_downward)
  DevBuf m_loc, m_tof, m_binom;     // downward pass: locals, target slots, binomials
  std::vector<double> m_binom_host;
  std::vector<int32_t> m_tof_host;
  uint64_t m2l_ops = 0;
  double m2l_prep = 0.0;

  // multi-GPU (fmm_multi.cu): the root's output mapped over IPC, NCCL comm
  void* peer_out = nullptr;
  void* nccl_comm = nullptr;
  int nccl_rank = 0, nccl_world = 1;

  // device FMM pipeline state (fmm_device.cu), created on first use
  fmmcu::DevicePipeline* pipe = nullptr;
};

#define CU_TRY(ctx, expr)                                                          \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      (ctx)->err = std::string(#expr) + ": " + cudaGetErrorString(_e);            \
      return _e == cudaErrorMemoryAllocation ? FMMCU_ENOMEM : FMMCU_ECUDA;        \
    }                                                                             \
  } while (0)

namespace fmmcu::detail {

int set_err(fmmcu_ctx* c, int code, const std::string& msg);
P2PArgs make_args(fmmcu_ctx* c);
// Work list of a job from its host CSR (pt_off, ev_off, strong_off, strong_idx).
int build_worklist(fmmcu_ctx* c, const fmmcu_p2p_job* j);
// Work list built on the device from the CSR already in d_pt / d_ev / d_soff /
// d_sidx (c->n_leaves leaves, c->n_strong entries), over leaves [lb, le),
// grouped by upload chunk when g.K > 1 (worklist_dev.cu); also fills the run
// table d_seg.  Same items as build_worklist; synchronizes `s` once.
// The job's CSR H2D on `stream` (in place when page-locked); returns the
// bytes moved, ~0 on error.
uint64_t upload_csr(fmmcu_ctx* c, const fmmcu_p2p_job* j, cudaStream_t stream);
int build_worklist_dev(fmmcu_ctx* c, uint32_t lb, uint32_t le, const WlGroups& g, cudaStream_t s,
                       const std::function<void()>& while_waiting = {});
// Symmetric (mutual-kernel) list + contribution lists on the device over
// [lb, le) of the staged CSR (worklist_dev.cu); -1 = the job does not qualify.
int build_sym_worklist_dev(fmmcu_ctx* c, uint32_t lb, uint32_t le, cudaStream_t s,
                           const WlGroups* g = nullptr);
// Device-resident CSR -> context staging, run table and device work list on
// stream `w` (records `done` there); want_sym: the mutual kernel's list when
// the job qualifies.  Eval records are left to the caller.
int stage_csr_dev(fmmcu_ctx* c, const uint32_t* pt, const uint32_t* ev, const uint32_t* so,
                  const uint32_t* si, uint32_t nl, uint32_t nnz, uint32_t ne, cudaStream_t w,
                  cudaEvent_t done, bool want_sym);
// Device buffers for the CSR + work list, their H2D, the run table and the
// eval records (needs d_src, d_evy, d_eself filled unless c->self_layout).
int stage_csr(fmmcu_ctx* c, const fmmcu_p2p_job* j, bool evals);
// P2P kernels over leaves [lb, le) of the staged job on c->stream.
int run_kernels(fmmcu_ctx* c, uint32_t lb, uint32_t le, int mode, int* nlaunch,
                bool reset_hits = true);
// Batched M2L on `stream` from device-resident arrays (see m2l_kernels.cuh).
int m2l_table(fmmcu_ctx* c, int p, int kernel, cudaStream_t stream);
int m2l_run(fmmcu_ctx* c, fmmcu::M2LArgs a, uint64_t nnz, cudaStream_t s);
// close the peer output mapping and the NCCL communicator (fmm_multi.cu)
void multi_release(fmmcu_ctx* c);

}  // namespace fmmcu::detail
