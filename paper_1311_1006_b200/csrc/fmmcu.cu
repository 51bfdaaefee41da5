// fmm-b200 — libfmmcuda.so: the C ABI of include/fmm_cuda.h.
//
// Host side of the device near field: validates the flattened NearFieldJob
// (reference backend.hpp:27-37), packs sources into 32-byte device records
// in pinned staging memory, builds the P2P work list (one item per target
// leaf; heavy leaves split into strong-list chunks reduced in a fixed
// order), enqueues H2D -> kernels -> D2H on the context stream and reports
// NearFieldStats (exact pair count, busy seconds) at finish.  Also hosts the
// batched M2L launch and an FP64 peak micro-benchmark.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <new>
#include <string>
#include <vector>

#include "fmm_cuda.h"
#include "fmmcu_internal.cuh"
#include "m2l_kernels.cuh"
#include "p2p_kernels.cuh"
#include "p2p_warp.cuh"
#include "p2p_sym.cuh"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace fmmcu;

namespace {

// Warp-kernel shape variant (see launch_warp_e); FMMCU_P2P_VARIANT overrides
// the measured default for experiments.
int variant_index() {
  static int v = [] {
    const char* s = std::getenv("FMMCU_P2P_VARIANT");
    int i = s ? std::atoi(s) : 0;
    return (i >= 0 && i < 6) ? i : 0;
  }();
  return v;
}

constexpr size_t warp_smem(int warps, int chunk, int e) {
  return size_t(warps) * warp_region_bytes(chunk, e);
}


}  // namespace

namespace fmmcu::detail {

// packed source records of slots [i0, i1) from interleaved z and m (DMA'd
// straight from page-locked caller arrays)
__global__ void pack_zm_kernel(const double2* __restrict__ z, const double2* __restrict__ m,
                               uint32_t i0, uint32_t i1, double4* __restrict__ src) {
  const uint32_t i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < i1) {
    const double2 a = z[i], b = m[i];
    src[i] = make_double4(a.x, a.y, b.x, b.y);
  }
}

int set_err(fmmcu_ctx* c, int code, const std::string& msg) {
  c->err = msg;
  return code;
}

// FMMCU_TRACE=1: host phase times of a launch on stderr.
struct Trace {
  fmmcu_ctx* c;
  Clock::time_point t = Clock::now();
  explicit Trace(fmmcu_ctx* cc) : c(cc) {}
  void mark(const char* what) {
    if (!c->trace) return;
    const auto now = Clock::now();
    std::fprintf(stderr, "[fmmcu] %-22s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

P2PArgs make_args(fmmcu_ctx* c) {
  P2PArgs a{};
  a.src = c->d_src.as<double4>();
  a.evy = c->d_evy.as<double2>();
  a.eself = c->d_eself.as<uint32_t>();
  a.pt_off = c->d_pt.as<uint32_t>();
  a.ev_off = c->d_ev.as<uint32_t>();
  a.s_off = c->d_soff.as<uint32_t>();
  a.s_idx = c->d_sidx.as<uint32_t>();
  a.items = c->d_items.as<P2PItem>();
  a.seg = c->d_seg.as<uint2>();
  a.evr = c->d_evr.as<double4>();
  a.next_item = c->d_counter.as<unsigned int>();
  a.out = c->out_ptr();
  a.partial = c->d_partial.as<double2>();
  a.hits = c->d_hits.as<unsigned long long>();
  a.delta = c->delta;
  a.delta2 = c->delta * c->delta;
  a.inv_delta2 = c->delta != 0.0 ? 1.0 / (c->delta * c->delta) : 0.0;
  return a;
}

template <int KN, int SM>
void launch_exact(const P2PArgs& a, uint32_t lb, uint32_t le, uint32_t eb, uint32_t ee,
                  cudaStream_t s) {
  const uint32_t n = ee - eb;
  p2p_exact_kernel<KN, SM><<<(n + 127) / 128, 128, 0, s>>>(a, lb, le, eb, ee);
}

template <int KN, int SM, int W, int E, int C, int U, int MINB>
void launch_warp_v(const P2PArgs& a, uint32_t n_items, cudaStream_t s) {
  auto kfn = p2p_warp_kernel<KN, SM, E, W, C, U, MINB>;
  constexpr size_t smem = warp_smem(W, C, E);
  static int grid_cap = [&] {
    cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, W * 32, smem);
    // FMMCU_GRID_PCT (experiments): persistent grid as a percentage of full residency
    const char* pct = std::getenv("FMMCU_GRID_PCT");
    const int g = sms * std::max(1, per_sm);
    return std::max(1, pct ? g * std::atoi(pct) / 100 : g);
  }();
  const uint32_t need = (n_items + W - 1) / W;
  const uint32_t grid = std::max(1u, std::min<uint32_t>(need, uint32_t(grid_cap)));
  kfn<<<grid, W * 32, smem, s>>>(a);
}

// warp-kernel variants (warps/CTA, chunk, unroll, min CTAs/SM) for the hot
// instantiation (harmonic, no smoother); E (evals per lane) is chosen per
// staged job by choose_warp_e():
//   0 = 4w c128 u2 m4   1 = 4w c128 u2 m3   2 = 4w c128 u1 m5
//   3 = 8w c128 u1 m2              4 = 4w c256 u1 m4   5 = 4w c128 u2 m4
template <int KN, int SM, int E>
void launch_warp_e(const P2PArgs& a, uint32_t n_items, cudaStream_t s) {
  constexpr int U0 = 2;  // E5 U2 measured best (profiles/r01: 1.027 vs 1.018 Tpairs/s for U1)
  if (KN == 0 && SM == 0) {
    switch (variant_index()) {
      case 1: launch_warp_v<KN, SM, 4, E, 128, 2, 3>(a, n_items, s); return;
      case 2: launch_warp_v<KN, SM, 4, E, 128, 1, 5>(a, n_items, s); return;
      case 3: launch_warp_v<KN, SM, 8, E, 128, 1, 2>(a, n_items, s); return;
      case 4: launch_warp_v<KN, SM, 4, E, 256, 1, 4>(a, n_items, s); return;
      case 5: launch_warp_v<KN, SM, 4, E, 128, 2, 4>(a, n_items, s); return;
      default: break;
    }
  }
  launch_warp_v<KN, SM, 4, E, 128, U0, 4>(a, n_items, s);
}

template <int KN, int SM>
void launch_warp(const P2PArgs& a, uint32_t n_items, cudaStream_t s, int E) {
  if (E == 5) launch_warp_e<KN, SM, 5>(a, n_items, s);
  else launch_warp_e<KN, SM, 4>(a, n_items, s);
}

void dispatch_tile(int kn, int sm, const P2PArgs& a, uint32_t n, cudaStream_t s, int E) {
  if (kn == 0) {
    if (sm == 0) launch_warp<0, 0>(a, n, s, E);
    else if (sm == 1) launch_warp<0, 1>(a, n, s, E);
    else launch_warp<0, 2>(a, n, s, E);
  } else {
    if (sm == 0) launch_warp<1, 0>(a, n, s, E);
    else if (sm == 1) launch_warp<1, 1>(a, n, s, E);
    else launch_warp<1, 2>(a, n, s, E);
  }
}

void dispatch_exact(int kn, int sm, const P2PArgs& a, uint32_t lb, uint32_t le, uint32_t eb,
                    uint32_t ee, cudaStream_t s) {
  if (kn == 0) {
    if (sm == 0) launch_exact<0, 0>(a, lb, le, eb, ee, s);
    else if (sm == 1) launch_exact<0, 1>(a, lb, le, eb, ee, s);
    else launch_exact<0, 2>(a, lb, le, eb, ee, s);
  } else {
    if (sm == 0) launch_exact<1, 0>(a, lb, le, eb, ee, s);
    else if (sm == 1) launch_exact<1, 1>(a, lb, le, eb, ee, s);
    else launch_exact<1, 2>(a, lb, le, eb, ee, s);
  }
}

template <int SM, int E, int W = 4, int C = 128, int U = 1, int MINB = 3, int SS = 1,
          bool ROUNDS = false>
void launch_sym_v(const P2PArgs& a, const P2PSymArgs& sa, uint32_t n_items, cudaStream_t s) {
  auto kfn = p2p_sym_kernel<SM, E, W, C, U, MINB, SS, ROUNDS>;
  constexpr size_t smem = size_t(W) * sym_region_bytes(C, E);
  static int grid_cap = [&] {
    cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, W * 32, smem);
    return std::max(1, sms * std::max(1, per_sm));
  }();
  const uint32_t need = (n_items + W - 1) / W;
  const uint32_t grid = std::max(1u, std::min<uint32_t>(need, uint32_t(grid_cap)));
  kfn<<<grid, W * 32, smem, s>>>(a, sa);
}

// mutual-kernel shapes (FMMCU_SYM_VARIANT, harmonic / no smoother):
//   E = 5: 0 = 4w c128 u1 m3, one symmetric source per step   1 = c256   2 = 2w m6
//          3 = u2   4 = m4 (128 registers)   5 = two sources per step   6 = three
// (r2, 10M / L10: 0 4.06 ms, 4 4.25, 5 4.27-4.45, 6 4.67; E = 4 5.89 ms)
int sym_variant() {
  static int v = [] {
    const char* e = std::getenv("FMMCU_SYM_VARIANT");
    const int i = e ? std::atoi(e) : 0;
    return (i >= 0 && i < 7) ? i : 0;
  }();
  return v;
}

void dispatch_sym(int sm, const P2PArgs& a, const P2PSymArgs& sa, uint32_t n, cudaStream_t s,
                  int E, bool rounds) {
  if (rounds) {  // items with more than 32 entries: the entry-round instantiation
    if (E == 5) {
      if (sm == 0) launch_sym_v<0, 5, 4, 128, 1, 3, 1, true>(a, sa, n, s);
      else if (sm == 1) launch_sym_v<1, 5, 4, 128, 1, 3, 1, true>(a, sa, n, s);
      else launch_sym_v<2, 5, 4, 128, 1, 3, 1, true>(a, sa, n, s);
    } else {
      if (sm == 0) launch_sym_v<0, 4, 4, 128, 1, 3, 1, true>(a, sa, n, s);
      else if (sm == 1) launch_sym_v<1, 4, 4, 128, 1, 3, 1, true>(a, sa, n, s);
      else launch_sym_v<2, 4, 4, 128, 1, 3, 1, true>(a, sa, n, s);
    }
    return;
  }
  if (E == 5 && sm == 0) {
    switch (sym_variant()) {
      case 1: launch_sym_v<0, 5, 4, 256, 1, 3>(a, sa, n, s); return;
      case 2: launch_sym_v<0, 5, 2, 128, 1, 6>(a, sa, n, s); return;
      case 3: launch_sym_v<0, 5, 4, 128, 2, 3>(a, sa, n, s); return;
      case 4: launch_sym_v<0, 5, 4, 128, 1, 4, 1>(a, sa, n, s); return;
      case 5: launch_sym_v<0, 5, 4, 128, 1, 3, 2>(a, sa, n, s); return;
      case 6: launch_sym_v<0, 5, 4, 128, 1, 3, 3>(a, sa, n, s); return;
      default: break;
    }
  }
  if (E == 5) {
    if (sm == 0) launch_sym_v<0, 5>(a, sa, n, s);
    else if (sm == 1) launch_sym_v<1, 5>(a, sa, n, s);
    else launch_sym_v<2, 5>(a, sa, n, s);
  } else {
    if (sm == 0) launch_sym_v<0, 4>(a, sa, n, s);
    else if (sm == 1) launch_sym_v<1, 4>(a, sa, n, s);
    else launch_sym_v<2, 4>(a, sa, n, s);
  }
}

int validate(fmmcu_ctx* c, const fmmcu_p2p_job* j) {
  if (!j) return set_err(c, FMMCU_EINVAL, "null job");
  if (j->kernel < 0 || j->kernel > 1) return set_err(c, FMMCU_EINVAL, "unknown kernel");
  if (j->smoother < 0 || j->smoother > 2) return set_err(c, FMMCU_EINVAL, "unknown smoother");
  if (j->mode < 0 || j->mode > 1) return set_err(c, FMMCU_EINVAL, "unknown mode");
  if (j->smoother != 0 && !(j->delta > 0.0))
    return set_err(c, FMMCU_EINVAL, "smoother delta must be > 0");
  if (!j->pt_off || !j->ev_off || !j->strong_off)
    return set_err(c, FMMCU_EINVAL, "null leaf offsets");
  if (j->n_src > 0 && (!j->src_z || !j->src_m || !j->perm))
    return set_err(c, FMMCU_EINVAL, "null source arrays");
  if (j->n_eval > 0 && !j->eval_y) return set_err(c, FMMCU_EINVAL, "null eval array");
  const uint32_t nl = j->n_leaves;
  if (j->pt_off[0] != 0 || j->pt_off[nl] != j->n_src)
    return set_err(c, FMMCU_EINVAL, "pt_off does not span the sources");
  if (j->ev_off[0] != 0 || j->ev_off[nl] != j->n_eval)
    return set_err(c, FMMCU_EINVAL, "ev_off does not span the evals");
  if (j->leaf_begin > j->leaf_end || j->leaf_end > nl)
    return set_err(c, FMMCU_EINVAL, "bad leaf shard");
  if (j->strong_off[nl] > 0 && !j->strong_idx) return set_err(c, FMMCU_EINVAL, "null strong list");
  return FMMCU_OK;
}

// The O(leaves + strong entries) part of validate: offsets monotone, strong
// indices in range.  launch_overlapped runs it while the first copies move.
int validate_csr(fmmcu_ctx* c, const fmmcu_p2p_job* j) {
  const uint32_t nl = j->n_leaves;
  const uint32_t nnz = j->strong_off[nl];
  const uint32_t* pt = j->pt_off;
  const uint32_t* ev = j->ev_off;
  const uint32_t* so = j->strong_off;
  const uint32_t* si = j->strong_idx;
  // one parallel region, branch-free (vectorised) reductions: a descent in
  // any offset array, and the largest strong index
  uint32_t desc = 0, top = 0;
#pragma omp parallel reduction(| : desc) reduction(max : top)
  {
#pragma omp for schedule(static) nowait
    for (int64_t i = 0; i < int64_t(nl); ++i)
      desc |= uint32_t(pt[i] > pt[i + 1]) | uint32_t(ev[i] > ev[i + 1]) |
              uint32_t(so[i] > so[i + 1]);
#pragma omp for schedule(static) nowait
    for (int64_t q = 0; q < int64_t(nnz); ++q) top = std::max(top, si[q]);
  }
  if (desc) return set_err(c, FMMCU_EINVAL, "leaf offsets not monotone");
  if (nnz && top >= nl) return set_err(c, FMMCU_EINVAL, "strong index out of range");
  return FMMCU_OK;
}

// Evals per lane of the warp kernel.  An eval block of nt <= 8E evals runs
// as G = ceil(nt/E) eval slots x K = floor(32/G) source lanes; a lane sweeps
// S/K sources for E evals, so the block costs ~ E * S / K lane-pair slots
// for nt * S / 32 useful ones.  Pick the E with the least modelled cost over
// the job's leaves (38-39 evals/leaf -> E = 5: 8 x 4 lanes, 95% useful,
// against 89% for E = 4).  FMMCU_P2P_E overrides.
double lane_cost(uint32_t ntl, uint64_t S, int E) {
  if (!ntl || !S) return 0.0;
  const uint32_t max_ev = uint32_t(kWarpSlots * E);
  const uint32_t nblk = (ntl + max_ev - 1) / max_ev;
  const uint32_t nt = (ntl + nblk - 1) / nblk;
  const uint32_t G = (nt + E - 1) / E;
  const uint32_t K = 32 / G;
  return double(nblk) * double(E) * double((S + K - 1) / K);
}

int choose_warp_e(double cost4, double cost5) {
  if (const char* env = std::getenv("FMMCU_P2P_E")) {
    const int e = std::atoi(env);
    if (e == 4 || e == 5) return e;
  }
  return cost5 < cost4 ? 5 : 4;
}

template <class T>
void par_prefix(T* v, int64_t n);

// Symmetric (mutual) work list over the job's leaf range [lb, le) (see
// p2p_sym.cuh).  Returns 1 when the job does not qualify (a leaf with more
// than 32 entries, or a source count that needs budget splitting): the caller
// then builds the ordinary list.
int build_sym_worklist(fmmcu_ctx* c, const fmmcu_p2p_job* j, uint32_t max_ev) {
  Trace tr(c);
  const uint32_t lb = j->leaf_begin, le = j->leaf_end, np = le - lb;
  const uint32_t* po = j->pt_off;
  auto npts = [&](uint32_t b) { return po[b + 1] - po[b]; };
  // scratch kept in the context (no reallocation / first-touch faults per call)
  std::vector<uint32_t>& ent = c->sw_ent;
  std::vector<uint32_t>& nblk = c->sw_nblk;
  std::vector<uint64_t>& ssym = c->sw_ssym;
  std::vector<uint64_t>& sord = c->sw_sord;
  std::vector<uint64_t>& slots = c->sw_slots;
  ent.resize(np + 1);
  nblk.resize(np + 1);
  ssym.resize(np);
  sord.resize(np);
  slots.resize(np + 1);
  ent[0] = 0;
  nblk[0] = 0;
  slots[0] = 0;
  bool ok = true;
  uint32_t max_n = 0;
#pragma omp parallel for schedule(static) reduction(&& : ok) reduction(max : max_n)
  for (int64_t i = 0; i < int64_t(np); ++i) {
    const uint32_t t = lb + uint32_t(i);
    uint32_t n = 0;
    uint64_t so = 0, ss = 0;
    for (uint32_t q = j->strong_off[t]; q < j->strong_off[t + 1]; ++q) {
      const uint32_t B = j->strong_idx[q];
      if (B >= lb && B < le && B < t) continue;  // the lower partner's item covers it
      ++n;
      if (B > t && B < le && B >= lb) ss += npts(B);
      else so += npts(B);
    }
    const uint32_t ntl = j->ev_off[t + 1] - j->ev_off[t];
    const uint32_t nb = ntl ? (ntl + max_ev - 1) / max_ev : 0;
    ok = ok && n <= uint32_t(kSymMaxEntries) && so + ss < (1ull << 31);
    max_n = std::max(max_n, n);
    ent[i + 1] = n;
    nblk[i + 1] = nb;
    ssym[i] = ss;
    sord[i] = so;
    slots[i + 1] = uint64_t(nb) * ss;
  }
  if (!ok) return 1;
  tr.mark("sym: count");
  par_prefix(ent.data(), int64_t(np));
  par_prefix(nblk.data(), int64_t(np));
  par_prefix(slots.data(), int64_t(np));
  if (slots[np] > 0xFFFFFFF0ull) return 1;
  c->sym_seg.resize(ent[np]);
  c->items.resize(nblk[np]);
  c->item_first.assign(nblk.begin(), nblk.end());
  c->fin_first.assign(np + 1, 0);
  c->fins.clear();
  c->partial_evals = 0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < int64_t(np); ++i) {
    const uint32_t t = lb + uint32_t(i);
    uint4* sg = c->sym_seg.data() + ent[i];
    uint32_t o = 0;
    for (int pass = 0; pass < 2; ++pass)  // ordered runs first, then symmetric
      for (uint32_t q = j->strong_off[t]; q < j->strong_off[t + 1]; ++q) {
        const uint32_t B = j->strong_idx[q];
        const bool inr = B >= lb && B < le;
        if (inr && B < t) continue;
        const bool sym = inr && B > t;
        if (sym != (pass == 1)) continue;
        const uint32_t kind = sym ? kRunSym : (B == t ? kRunSelf : kRunOrdered);
        sg[o++] = make_uint4(po[B], npts(B), kind, 0u);
      }
    const uint32_t ntl = j->ev_off[t + 1] - j->ev_off[t];
    const uint32_t nb = nblk[i + 1] - nblk[i];
    for (uint32_t b = 0, e0 = 0; b < nb; ++b) {
      const uint32_t nt = (ntl - e0) / (nb - b) + ((ntl - e0) % (nb - b) ? 1u : 0u);
      P2PItem it{t, j->ev_off[t] + e0, nt, ent[i], ent[i + 1], uint32_t(sord[i] + ssym[i]),
                 uint32_t(slots[i] + uint64_t(b) * ssym[i]), uint32_t(sord[i])};
      c->items[nblk[i] + b] = it;
      e0 += nt;
    }
  }
  tr.mark("sym: entries + items");
  // per leaf of the range: (first entry, first item, first contrib slot,
  // symmetric sources per item); the finalize kernel finds each lower
  // partner's contributions from these and the strong lists
  c->sym_info.resize(size_t(np) + 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i <= int64_t(np); ++i)
    c->sym_info[i] = make_uint4(ent[i], nblk[i], uint32_t(slots[i]),
                                i < int64_t(np) ? uint32_t(ssym[i]) : 0u);
  tr.mark("sym: contributions");
  c->sym_slots = slots[np];
  c->sym_n_items = uint32_t(c->items.size());
  c->sym_rounds = max_n > uint32_t(kWarpMaxEntries);
  c->sym_grouped = false;
  c->sym_lb = lb;
  c->sym_le = le;
  c->sym_items = true;
  c->grouped = false;
  return FMMCU_OK;
}

// Work list of a job (host, OpenMP): per-leaf pair work and its prefix,
// evals-per-lane choice, and the item / finalize lists.  Touches only the
// job's CSR and host-side context fields, so it runs on a helper thread
// while the main thread packs and uploads the sources.
// In-place inclusive prefix sum of v[1..n] (v[0] = 0 stays), blocked over the
// OpenMP threads: per-block sums, a serial scan of the block sums, then each
// block adds its offset.
template <class T>
void par_prefix(T* v, int64_t n) {
  if (n <= 0) return;
  if (n < (int64_t(1) << 15)) {
    for (int64_t i = 1; i <= n; ++i) v[i] += v[i - 1];
    return;
  }
  int nb = 1;
#ifdef _OPENMP
  nb = omp_get_max_threads();
#endif
  std::vector<T> part(nb + 1, T(0));
  const int64_t per = (n + nb - 1) / nb;
#pragma omp parallel for schedule(static, 1) num_threads(nb)
  for (int b = 0; b < nb; ++b) {
    const int64_t i0 = 1 + b * per, i1 = std::min<int64_t>(n, i0 + per - 1);
    T acc = 0;
    for (int64_t i = i0; i <= i1; ++i) acc += v[i];
    part[b + 1] = acc;
  }
  for (int b = 0; b < nb; ++b) part[b + 1] += part[b];
#pragma omp parallel for schedule(static, 1) num_threads(nb)
  for (int b = 0; b < nb; ++b) {
    const int64_t i0 = 1 + b * per, i1 = std::min<int64_t>(n, i0 + per - 1);
    T acc = part[b];
    for (int64_t i = i0; i <= i1; ++i) {
      acc += v[i];
      v[i] = acc;
    }
  }
}

int build_worklist(fmmcu_ctx* c, const fmmcu_p2p_job* j) {
  Trace tr(c);
  c->dev_wl = false;
  c->dev_list = false;
  const uint32_t nl = j->n_leaves;
  c->ev_off.resize(nl + 1);
  c->leaf_work.resize(nl + 1);
  c->wl_S.resize(nl);
  std::vector<uint64_t>& S = c->wl_S;
  uint32_t* evo = c->ev_off.data();
  uint64_t* work = c->leaf_work.data();
  work[0] = 0;
  c->wl_need.resize(nl);
  uint32_t* needv = c->wl_need.data();
  // one pass: sources of the strong list S, last source slot it reads (need),
  // pair work, and the modelled lane cost of E = 4 and E = 5 (choose_warp_e)
  double cost4 = 0.0, cost5 = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : cost4, cost5)
  for (int64_t t = 0; t < int64_t(nl); ++t) {
    uint64_t s = 0;
    uint32_t need = j->pt_off[t + 1];
    for (uint32_t q = j->strong_off[t]; q < j->strong_off[t + 1]; ++q) {
      const uint32_t sb = j->strong_idx[q];
      const uint32_t e1 = j->pt_off[sb + 1];
      s += e1 - j->pt_off[sb];
      need = std::max(need, e1);
    }
    S[t] = s;
    needv[t] = need;
    evo[t] = j->ev_off[t];
    const uint32_t ntl = j->ev_off[t + 1] - j->ev_off[t];
    work[t + 1] = uint64_t(ntl) * s;
    cost4 += lane_cost(ntl, s, 4);
    cost5 += lane_cost(ntl, s, 5);
  }
  evo[nl] = j->ev_off[nl];
  par_prefix(work, int64_t(nl));
  const uint64_t total = work[nl];
  tr.mark("wl: S + work prefix");
  const uint64_t budget = std::max<uint64_t>(1ull << 16, total / (148ull * 16ull));
  const bool warp_kernel = true;
  c->warp_e = warp_kernel ? choose_warp_e(cost4, cost5) : 4;
  const uint32_t max_ev = uint32_t(kWarpSlots * c->warp_e);
  const uint32_t max_ent = warp_kernel ? uint32_t(kWarpMaxEntries) : 0xFFFFFFFFu;
  c->warp_items = warp_kernel;
  c->sym_items = false;
  if (c->sym_request && warp_kernel && c->group_k == 0 && j->kernel == 0) {
    if (build_sym_worklist(c, j, max_ev) == FMMCU_OK) {
      tr.mark("wl: symmetric");
      return FMMCU_OK;
    }
  }
  tr.mark("wl: choose E");
  // Items: eval blocks of <= max_ev evals (balanced: ceil(ntl / max_ev)
  // blocks of near-equal size); a block whose pair work exceeds the budget is
  // split into strong-list chunks whose partials are summed in chunk order by
  // p2p_finalize_kernel.  Two parallel passes over the leaves (count, then
  // fill at prefix offsets) give the same list as a serial build.
  struct LeafCount {
    uint32_t items, fins, pevals;
  };
  auto leaf_items = [&](uint32_t t, P2PItem* it, P2PFinal* fin, uint32_t pbase) {
    LeafCount n{0, 0, 0};
    const uint32_t ntl = j->ev_off[t + 1] - j->ev_off[t];
    const uint32_t sb0 = j->strong_off[t], sb1 = j->strong_off[t + 1];
    const uint32_t nblk = (ntl + max_ev - 1) / max_ev;
    for (uint32_t b = 0, e0 = 0; b < nblk; ++b) {
      const uint32_t nt = (ntl - e0) / (nblk - b) + ((ntl - e0) % (nblk - b) ? 1u : 0u);
      const uint32_t evb = j->ev_off[t] + e0;
      e0 += nt;
      const uint64_t pairs = uint64_t(nt) * S[t];
      if ((pairs <= budget || sb1 - sb0 <= 1) && sb1 - sb0 <= max_ent && S[t] <= 0xFFFFFFFFull) {
        if (it) it[n.items] = P2PItem{t, evb, nt, sb0, sb1, uint32_t(S[t]), kNoSelf, 0};
        ++n.items;
        continue;
      }
      const uint64_t src_per_chunk = std::max<uint64_t>(1, budget / nt);
      const uint32_t base = pbase + n.pevals;
      uint32_t n_chunks = 0;
      uint32_t q = sb0;
      while (q < sb1) {
        uint32_t q1 = q;
        uint64_t acc = 0;
        while (q1 < sb1 && q1 - q < max_ent &&
               (acc == 0 || acc + (j->pt_off[j->strong_idx[q1] + 1] -
                                   j->pt_off[j->strong_idx[q1]]) <= src_per_chunk)) {
          acc += j->pt_off[j->strong_idx[q1] + 1] - j->pt_off[j->strong_idx[q1]];
          ++q1;
        }
        if (it) it[n.items] = P2PItem{t, evb, nt, q, q1, uint32_t(acc), pbase + n.pevals, 0};
        ++n.items;
        n.pevals += nt;
        ++n_chunks;
        q = q1;
      }
      if (fin) fin[n.fins] = P2PFinal{evb, nt, base, n_chunks};
      ++n.fins;
    }
    return n;
  };
  // Leaf processing order.  Default: every leaf, ascending (item_first is
  // indexed by leaf).  Grouped (overlapped launch, c->group_k > 0): the
  // shard's leaves ordered by the upload chunk holding the last source slot
  // their strong list reads, so group g can run as soon as chunks 0..g are on
  // the device; item_first / fin_first are then indexed by position and
  // grp_item / grp_fin delimit the groups.
  std::vector<uint32_t>& order = c->wl_order;
  const bool grouped = c->group_k > 0;
  const uint32_t np = grouped ? j->leaf_end - j->leaf_begin : nl;
  if (grouped) {
    const int K = c->group_k;
    std::vector<uint32_t>& kc = c->wl_kc;
    kc.resize(np);
    // chunk k holds leaves [chunk_leaf[k], chunk_leaf[k+1]), i.e. slots below slot_end[k]
    uint32_t slot_end[fmmcu_ctx::kMaxChunks];
    for (int k = 0; k < K; ++k) slot_end[k] = j->pt_off[c->chunk_leaf[k + 1]];
    // stable parallel counting sort of the shard's leaves by chunk
    int nb = 1;
#ifdef _OPENMP
    nb = omp_get_max_threads();
#endif
    const int64_t per = (int64_t(np) + nb - 1) / nb;
    std::vector<uint32_t> hist(size_t(nb) * (K + 1), 0);
#pragma omp parallel for schedule(static, 1) num_threads(nb)
    for (int b = 0; b < nb; ++b) {
      uint32_t* hb = hist.data() + size_t(b) * (K + 1);
      const int64_t i1 = std::min<int64_t>(np, (b + 1) * per);
      for (int64_t i = b * per; i < i1; ++i) {
        const uint32_t need = needv[j->leaf_begin + i];
        int k = 0;
        while (k < K - 1 && slot_end[k] < need) ++k;
        kc[i] = uint32_t(k);
        ++hb[k];
      }
    }
    // offsets: group k first, then block b within it
    std::vector<uint32_t> cnt(K + 1, 0);
    uint32_t run = 0;
    for (int k = 0; k < K; ++k) {
      cnt[k] = run;
      for (int b = 0; b < nb; ++b) {
        uint32_t& hb = hist[size_t(b) * (K + 1) + k];
        const uint32_t n = hb;
        hb = run;
        run += n;
      }
    }
    cnt[K] = run;
    c->grp_pos.assign(cnt.begin(), cnt.end());
    order.resize(np);
#pragma omp parallel for schedule(static, 1) num_threads(nb)
    for (int b = 0; b < nb; ++b) {
      uint32_t* hb = hist.data() + size_t(b) * (K + 1);
      const int64_t i1 = std::min<int64_t>(np, (b + 1) * per);
      for (int64_t i = b * per; i < i1; ++i) order[hb[kc[i]]++] = j->leaf_begin + uint32_t(i);
    }
  }
  tr.mark("wl: grouping");
  auto leaf_at = [&](int64_t pos) { return grouped ? order[pos] : uint32_t(pos); };
  std::vector<uint64_t>& pev_first = c->wl_pev;
  pev_first.resize(np + 1);
  c->item_first.resize(np + 1);
  c->fin_first.resize(np + 1);
  pev_first[0] = 0;
  c->item_first[0] = 0;
  c->fin_first[0] = 0;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < int64_t(np); ++t) {
    const LeafCount n = leaf_items(leaf_at(t), nullptr, nullptr, 0);
    c->item_first[t + 1] = n.items;
    c->fin_first[t + 1] = n.fins;
    pev_first[t + 1] = n.pevals;
  }
  par_prefix(c->item_first.data(), int64_t(np));
  par_prefix(c->fin_first.data(), int64_t(np));
  par_prefix(pev_first.data(), int64_t(np));
  const uint64_t partial_evals = pev_first[np];
  tr.mark("wl: count + prefix");
  if (partial_evals > 0xFFFFFFF0ull) return set_err(c, FMMCU_EINVAL, "partial buffer too large");
  c->partial_evals = partial_evals;
  c->items.resize(c->item_first[np]);
  c->fins.resize(c->fin_first[np]);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < int64_t(np); ++t)
    leaf_items(leaf_at(t), c->items.data() + c->item_first[t], c->fins.data() + c->fin_first[t],
               uint32_t(pev_first[t]));
  c->grouped = grouped;
  tr.mark("wl: fill");

  return FMMCU_OK;
}

// Host packing + work list + H2D.  `sync` = wait for the uploads.
int stage_job(fmmcu_ctx* c, const fmmcu_p2p_job* j) {
  if (int rc = validate(c, j)) return rc;
  if (int rc = validate_csr(c, j)) return rc;
  CU_TRY(c, cudaSetDevice(c->device));
  c->group_k = 0;
  const uint32_t nl = j->n_leaves, ns = j->n_src, ne = j->n_eval;
  c->n_leaves = nl;
  c->n_src = ns;
  c->n_eval = ne;
  c->kernel = j->kernel;
  c->smoother = j->smoother;
  c->mode = j->mode;
  c->delta = j->delta;

  Trace tr(c);
  // Plausibly self-evaluation (cheap test): the work list waits for the
  // per-element check of the packing loop, and is built symmetric if it holds.
  const bool maybe_sym = j->eval_sid && ne == ns && ns > 0 && j->kernel == 0 &&
                         j->mode == FMMCU_MODE_FAST && !std::getenv("FMMCU_NO_SYM") &&
                         std::memcmp(j->ev_off, j->pt_off, size_t(nl + 1) * 4) == 0;
  c->sym_request = false;
  std::future<int> worklist;
  if (!maybe_sym)
    worklist = std::async(std::launch::async, [c, j] { return build_worklist(c, j); });
  cudaStream_t s = c->stream;
  CU_TRY(c, c->d_src.ensure(size_t(ns) * 32));
  CU_TRY(c, c->d_evy.ensure(size_t(ne) * 16));
  CU_TRY(c, c->d_eself.ensure(size_t(ne) * 4));
  CU_TRY(c, cudaEventRecord(c->ev_start, s));
  c->t_evstart = Clock::now();

  // ---- sources: pack 32-byte records into pinned chunks, each chunk's H2D
  // issued as soon as it is packed (host packing overlaps the PCIe copy) ----
  CU_TRY(c, c->h_src.ensure(size_t(ns) * 32));
  CU_TRY(c, c->h_evy.ensure(size_t(ne) * 16));
  CU_TRY(c, c->h_eself.ensure(size_t(ne) * 4));
  double* hs = c->h_src.as<double>();
  const double* z = j->src_z;
  const double* m = j->src_m;
  // Self layout (EvalSet::self_of with perm == eval_perm): eval e is source
  // slot e.  Detected while packing; the eval arrays are then derived on the
  // device instead of uploaded (saves 20 B/eval of PCIe traffic).
  const bool maybe_self = j->eval_sid && ne == ns && ns > 0;
  bool self_layout = maybe_self;
  // Halo-only staging for a leaf shard [leaf_begin, leaf_end) (multi-GPU
  // ranks): the shard's kernels read exactly the sources of its strong lists
  // (backend.cpp:55-57) -- its own leaves plus a halo -- so only those source
  // runs are packed and uploaded; the other slots of the device array are
  // never read.  A full range uploads everything in one run.
  const uint32_t lb = j->leaf_begin, le = j->leaf_end;
  const bool partial = lb > 0 || le < nl;
  std::vector<std::pair<int64_t, int64_t>> runs;  // source slot runs [a, b)
  if (partial) {
    std::vector<uint8_t> need(nl, 0);
#pragma omp parallel for schedule(static)
    for (int64_t t = lb; t < int64_t(le); ++t)
      for (uint32_t q = j->strong_off[t]; q < j->strong_off[t + 1]; ++q) need[j->strong_idx[q]] = 1;
    for (uint32_t t = 0; t < nl;) {
      if (!need[t]) {
        ++t;
        continue;
      }
      uint32_t t1 = t + 1;
      while (t1 < nl && need[t1]) ++t1;
      if (j->pt_off[t1] > j->pt_off[t]) runs.emplace_back(j->pt_off[t], j->pt_off[t1]);
      t = t1;
    }
  } else if (ns) {
    runs.emplace_back(0, int64_t(ns));
  }
  uint64_t uploaded = 0;
  constexpr int64_t kChunk = 1 << 20;  // sources per pipelined chunk (32 MB)
  for (const auto& run : runs)
    for (int64_t c0 = run.first; c0 < run.second; c0 += kChunk) {
      const int64_t c1 = std::min<int64_t>(run.second, c0 + kChunk);
      bool same = true;
#pragma omp parallel for schedule(static) reduction(&& : same)
      for (int64_t i = c0; i < c1; ++i) {
        hs[4 * i + 0] = z[2 * i];
        hs[4 * i + 1] = z[2 * i + 1];
        hs[4 * i + 2] = m[2 * i];
        hs[4 * i + 3] = m[2 * i + 1];
        if (maybe_self)
          same = same && j->eval_sid[i] == int64_t(j->perm[i]) &&
                 j->eval_y[2 * i] == z[2 * i] && j->eval_y[2 * i + 1] == z[2 * i + 1];
      }
      self_layout = self_layout && same;
      CU_TRY(c, cudaMemcpyAsync(c->d_src.as<double>() + 4 * c0, hs + 4 * c0, size_t(c1 - c0) * 32,
                                cudaMemcpyHostToDevice, s));
      uploaded += uint64_t(c1 - c0);
    }
  // a shard's own evals are its own leaves' slots: under the self layout
  // they are checked above; other slots are never read
  tr.mark("pack+h2d sources");
  c->self_layout = self_layout;
  uint32_t* eself = c->h_eself.as<uint32_t>();
  if (self_layout) {
    // built on the device after the uploads (p2p_self_evals_kernel)
  } else if (j->eval_sid && ns > 0) {
    par_memcpy(c->h_evy.p, j->eval_y, size_t(ne) * 16);
    c->invperm.resize(ns);
    uint32_t* inv = c->invperm.data();
    const uint32_t* perm = j->perm;
    bool ok = true;
#pragma omp parallel for schedule(static) reduction(&& : ok)
    for (int64_t i = 0; i < int64_t(ns); ++i) {
      if (perm[i] >= ns) ok = false;
      else inv[perm[i]] = uint32_t(i);
    }
    if (!ok) return set_err(c, FMMCU_EINVAL, "perm is not a permutation of the sources");
    const int64_t* sid = j->eval_sid;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < int64_t(ne); ++e) {
      const int64_t sv = sid[e];
      eself[e] = (sv >= 0 && sv < int64_t(ns)) ? inv[sv] : kNoSelf;
    }
  } else {
    par_memcpy(c->h_evy.p, j->eval_y, size_t(ne) * 16);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < int64_t(ne); ++e) eself[e] = kNoSelf;
  }
  if (!self_layout && ne) {
    CU_TRY(c, cudaMemcpyAsync(c->d_evy.p, c->h_evy.p, size_t(ne) * 16, cudaMemcpyHostToDevice, s));
    CU_TRY(c, cudaMemcpyAsync(c->d_eself.p, c->h_eself.p, size_t(ne) * 4, cudaMemcpyHostToDevice, s));
  }
  tr.mark("evals");

  // ---- work list (built concurrently with the source packing above) -------
  if (maybe_sym) {
    c->sym_request = self_layout;
    if (int rc = build_worklist(c, j)) return rc;
  } else if (int rc = worklist.get()) {
    return rc;
  }
  tr.mark("worklist");
  if (int rc = stage_csr(c, j, true)) return rc;
  c->h2d_bytes -= (uint64_t(ns) - uploaded) * 32;
  c->staged_src = uploaded;
  tr.mark("csr+worklist h2d");
  return FMMCU_OK;
}

// The job's finest CSR (pt_off, ev_off, strong_off, strong_idx) H2D on
// `stream` into d_pt / d_ev / d_soff / d_sidx: DMA'd in place from page-locked
// caller arrays, else through one pinned block.  Returns the bytes moved, or
// ~0 on a CUDA error (c->err set).
uint64_t upload_csr(fmmcu_ctx* c, const fmmcu_p2p_job* j, cudaStream_t stream) {
  const uint32_t nl = j->n_leaves;
  const uint32_t nnz = j->strong_off[nl];
  auto fail = [&](cudaError_t e, const char* what) {
    c->err = std::string(what) + ": " + cudaGetErrorString(e);
    return ~0ull;
  };
  cudaError_t e;
  if ((e = c->d_pt.ensure(size_t(nl + 1) * 4)) != cudaSuccess ||
      (e = c->d_ev.ensure(size_t(nl + 1) * 4)) != cudaSuccess ||
      (e = c->d_soff.ensure(size_t(nl + 1) * 4)) != cudaSuccess ||
      (e = c->d_sidx.ensure(size_t(std::max(nnz, 1u)) * 4)) != cudaSuccess)
    return fail(e, "csr buffers");
  auto locked = [](const void* p) {
    cudaPointerAttributes at{};
    const bool ok = p && cudaPointerGetAttributes(&at, p) == cudaSuccess &&
                    at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
  };
  const size_t csr_bytes = size_t(nl + 1) * 12 + size_t(nnz) * 4;
  if ((e = c->h_csr.ensure(csr_bytes)) != cudaSuccess) return fail(e, "csr staging");
  unsigned char* hc = c->h_csr.as<unsigned char>();
  size_t o = 0;
  auto put = [&](const void* src, size_t bytes) -> const void* {
    if (!bytes) return src;
    if (locked(src)) return src;
    par_memcpy(hc + o, src, bytes);
    const void* at = hc + o;
    o += bytes;
    return at;
  };
  const void* s_pt = put(j->pt_off, size_t(nl + 1) * 4);
  const void* s_ev = put(j->ev_off, size_t(nl + 1) * 4);
  const void* s_so = put(j->strong_off, size_t(nl + 1) * 4);
  const void* s_si = put(j->strong_idx, size_t(nnz) * 4);
  if ((e = cudaMemcpyAsync(c->d_pt.p, s_pt, size_t(nl + 1) * 4, cudaMemcpyHostToDevice,
                           stream)) != cudaSuccess ||
      (e = cudaMemcpyAsync(c->d_ev.p, s_ev, size_t(nl + 1) * 4, cudaMemcpyHostToDevice,
                           stream)) != cudaSuccess ||
      (e = cudaMemcpyAsync(c->d_soff.p, s_so, size_t(nl + 1) * 4, cudaMemcpyHostToDevice,
                           stream)) != cudaSuccess ||
      (nnz && (e = cudaMemcpyAsync(c->d_sidx.p, s_si, size_t(nnz) * 4, cudaMemcpyHostToDevice,
                                   stream)) != cudaSuccess))
    return fail(e, "csr h2d");
  return csr_bytes;
}

int stage_csr(fmmcu_ctx* c, const fmmcu_p2p_job* j, bool evals) {
  const uint32_t nl = j->n_leaves, ne = j->n_eval;
  const uint32_t nnz = j->strong_off[nl];
  const bool self_layout = c->self_layout;
  cudaStream_t s = c->stream;
  // ---- device buffers -------------------------------------------------------
  CU_TRY(c, c->d_pt.ensure(size_t(nl + 1) * 4));
  CU_TRY(c, c->d_ev.ensure(size_t(nl + 1) * 4));
  CU_TRY(c, c->d_soff.ensure(size_t(nl + 1) * 4));
  CU_TRY(c, c->d_sidx.ensure(size_t(nnz) * 4));
  CU_TRY(c, c->d_items.ensure(c->items.size() * sizeof(P2PItem)));
  CU_TRY(c, c->d_fin.ensure(c->fins.size() * sizeof(P2PFinal)));
  CU_TRY(c, c->d_out.ensure(size_t(ne) * 16));
  CU_TRY(c, c->d_partial.ensure(size_t(c->partial_evals) * 16));
  CU_TRY(c, c->d_hits.ensure(8));
  CU_TRY(c, c->d_counter.ensure(8));
  CU_TRY(c, c->d_seg.ensure(size_t(nnz) * 8));
  CU_TRY(c, c->d_evr.ensure(size_t(ne) * 32));
  CU_TRY(c, c->h_hits.ensure(8));
  // CSR through one pinned block, unless the caller's arrays are page-locked
  // (then DMA'd in place); the work list is already in pinned vectors
  const size_t ib = c->items.size() * sizeof(P2PItem), fb = c->fins.size() * sizeof(P2PFinal);
  const uint64_t csr_bytes = upload_csr(c, j, s);
  if (csr_bytes == ~0ull) return FMMCU_ECUDA;
  c->h2d_bytes = uint64_t(c->n_src) * 32 + (self_layout ? 0 : uint64_t(ne) * 20) + csr_bytes +
                 ib + fb;
  if (ib) CU_TRY(c, cudaMemcpyAsync(c->d_items.p, c->items.data(), ib, cudaMemcpyHostToDevice, s));
  if (fb) CU_TRY(c, cudaMemcpyAsync(c->d_fin.p, c->fins.data(), fb, cudaMemcpyHostToDevice, s));
  if (nnz) {
    p2p_segments_kernel<<<(nnz + 255) / 256, 256, 0, s>>>(c->d_sidx.as<uint32_t>(),
                                                          c->d_pt.as<uint32_t>(), nnz,
                                                          c->d_seg.as<uint2>());
    c->launches += 1;
  }
  if (ne && evals) {
    if (self_layout) {
      p2p_self_evals_kernel<<<(ne + 255) / 256, 256, 0, s>>>(c->d_src.as<double4>(), 0, ne,
                                                             c->d_evy.as<double2>(),
                                                             c->d_eself.as<uint32_t>());
      c->launches += 1;
    }
    // eval records {x, y, self slot, strong entry of the self slot}; needs seg
    p2p_evrec_kernel<<<(nl + 7) / 8, 256, 0, s>>>(make_args(c), 0, nl, c->d_evr.as<double4>());
    c->launches += 1;
  }
  if (c->sym_items) {
    const size_t nseg = c->sym_seg.size(), ninfo = c->sym_info.size();
    CU_TRY(c, c->d_symseg.ensure(std::max<size_t>(nseg, 1) * 16));
    CU_TRY(c, c->d_syminfo.ensure(std::max<size_t>(ninfo, 1) * 16));
    CU_TRY(c, c->d_tgt.ensure(size_t(std::max(ne, 1u)) * 16));
    CU_TRY(c, c->d_contrib.ensure(std::max<uint64_t>(c->sym_slots, 1) * 16));
    const size_t sym_bytes = (nseg + ninfo) * 16;
    CU_TRY(c, c->h_sym.ensure(sym_bytes));
    unsigned char* hb = c->h_sym.as<unsigned char>();
    par_memcpy(hb, c->sym_seg.data(), nseg * 16);
    par_memcpy(hb + nseg * 16, c->sym_info.data(), ninfo * 16);
    if (nseg) CU_TRY(c, cudaMemcpyAsync(c->d_symseg.p, hb, nseg * 16, cudaMemcpyHostToDevice, s));
    CU_TRY(c, cudaMemcpyAsync(c->d_syminfo.p, hb + nseg * 16, ninfo * 16, cudaMemcpyHostToDevice,
                              s));
    c->h2d_bytes += sym_bytes;
    // per-leaf contribution lists (count, scan, fill) on the device
    const uint32_t nr = c->sym_le - c->sym_lb;
    CU_TRY(c, c->d_cloff.ensure((size_t(nr) + 1) * 4));
    CU_TRY(c, c->d_clcnt.ensure((size_t(nr) + 1) * 4));
    CU_TRY(c, cudaMemsetAsync(c->d_clcnt.p, 0, (size_t(nr) + 1) * 4, s));
    const uint32_t gb = (nr + 7) / 8;
    p2p_sym_lists_kernel<false><<<gb, 256, 0, s>>>(
        c->sym_lb, nr, c->d_pt.as<uint32_t>(), c->d_soff.as<uint32_t>(), c->d_sidx.as<uint32_t>(),
        c->d_syminfo.as<uint4>(), c->d_symseg.as<uint4>(), c->d_clcnt.as<uint32_t>(), nullptr,
        nullptr);
    size_t tb = 0;
    CU_TRY(c, cub::DeviceScan::ExclusiveSum(nullptr, tb, c->d_clcnt.as<uint32_t>(),
                                            c->d_cloff.as<uint32_t>(), int64_t(nr) + 1, s));
    CU_TRY(c, c->d_cubtmp.ensure(tb));
    CU_TRY(c, cub::DeviceScan::ExclusiveSum(c->d_cubtmp.p, tb, c->d_clcnt.as<uint32_t>(),
                                            c->d_cloff.as<uint32_t>(), int64_t(nr) + 1, s));
    CU_TRY(c, cudaMemcpyAsync(c->h_hits.p, c->d_cloff.as<uint32_t>() + nr, 4,
                              cudaMemcpyDeviceToHost, s));
    CU_TRY(c, cudaStreamSynchronize(s));
    const uint32_t ncl = *c->h_hits.as<uint32_t>();
    CU_TRY(c, c->d_clbase.ensure(size_t(std::max(ncl, 1u)) * 4));
    p2p_sym_lists_kernel<true><<<gb, 256, 0, s>>>(
        c->sym_lb, nr, c->d_pt.as<uint32_t>(), c->d_soff.as<uint32_t>(), c->d_sidx.as<uint32_t>(),
        c->d_syminfo.as<uint4>(), c->d_symseg.as<uint4>(), nullptr, c->d_cloff.as<uint32_t>(),
        c->d_clbase.as<uint32_t>());
    c->launches += 3;
  }
  CU_TRY(c, cudaGetLastError());
  c->staged = true;
  return FMMCU_OK;
}

// ---------------------------------------------------------------------------
// Reference-facing launch, fast mode: the upload overlaps the kernels.
//  * sources go H2D in K leaf-aligned chunks on the copy stream;
//  * the work list (helper thread) orders the shard's leaves by the chunk
//    holding the last source slot their strong list reads, so group g runs
//    as soon as chunks 0..g have landed;
//  * eval records of a chunk's leaves are derived on the device from its
//    sources when every eval there is its own source (self layout), else the
//    chunk's eval arrays ride the copy stream with it;
//  * potentials are written by the kernels' TMA bulk stores straight into
//    the page-locked output (the caller's, or pinned staging): no D2H pass.
int launch_overlapped(fmmcu_ctx* c, const fmmcu_p2p_job* j) {
  Trace tr(c);
  if (int rc = validate(c, j)) return rc;
  // Whole-job launches with the device work list check the CSR while the
  // CSR and the source chunks are already moving (0.27 ms of host time at
  // 10M off the critical path); the copies only read [pt_off[cut k],
  // pt_off[cut k+1]) ranges, checked below.  Leaf ranges walk the strong
  // lists on the host first, so they check up front.
  const bool defer_csr = !std::getenv("FMMCU_HOST_WL") && !std::getenv("FMMCU_NO_DEFER") &&
                         j->leaf_begin == 0 && j->leaf_end == j->n_leaves;
  if (!defer_csr)
    if (int rc = validate_csr(c, j)) return rc;
  tr.mark("validate");
  CU_TRY(c, cudaSetDevice(c->device));
  const uint32_t nl = j->n_leaves, ns = j->n_src, ne = j->n_eval;
  const uint32_t lb = j->leaf_begin, le = j->leaf_end;
  c->n_leaves = nl;
  c->n_src = ns;
  c->n_eval = ne;
  c->kernel = j->kernel;
  c->smoother = j->smoother;
  c->mode = j->mode;
  c->delta = j->delta;
  // Leaf-aligned upload chunks of ~kChunkSrc sources.  Group k's kernels
  // start when chunk k lands, so the step ends one group's compute after the
  // last chunk: with a tail (FMMCU_TAIL=n) the last n chunks halve in
  // size, 1/2, 1/4, ... of kChunkSrc, to shorten that final group.
  static const uint32_t kChunkSrc =
      std::getenv("FMMCU_CHUNK") ? uint32_t(std::atol(std::getenv("FMMCU_CHUNK"))) : (1u << 20);
  static const int kTail = std::getenv("FMMCU_TAIL") ? std::atoi(std::getenv("FMMCU_TAIL")) : 0;
  std::vector<uint64_t> cut_src{0};
  {
    uint64_t rest = ns;
    const uint64_t cs = std::max<uint32_t>(kChunkSrc, 1u << 14);
    // full chunks while more than the tail (cs * (1 - 2^-kTail)) plus one chunk remain
    const uint64_t tail_total = kTail > 0 ? cs - (cs >> kTail) : 0;
    while (rest > cs + tail_total && cut_src.size() < size_t(fmmcu_ctx::kMaxChunks - kTail)) {
      cut_src.push_back(cut_src.back() + cs);
      rest -= cs;
    }
    // the remainder: halving pieces, the last two equal
    for (int t = 0; t < kTail && rest > (cs >> (kTail + 1)); ++t) {
      const uint64_t piece = rest / 2;
      cut_src.push_back(cut_src.back() + (rest - piece));
      rest = piece;
    }
    if (rest > 0 || cut_src.size() == 1) cut_src.push_back(ns);
    cut_src.back() = ns;
  }
  const int K = int(cut_src.size()) - 1;
  c->chunk_leaf.assign(K + 1, nl);
  c->chunk_leaf[0] = 0;
  for (int k = 1; k < K; ++k) {
    const uint32_t t = uint32_t(std::lower_bound(j->pt_off, j->pt_off + nl + 1,
                                                 uint32_t(cut_src[k])) - j->pt_off);
    c->chunk_leaf[k] = std::max(c->chunk_leaf[k - 1], std::min(t, nl));
  }
  for (int k = 0; k < K; ++k)  // the copies' source ranges (pt_off[nl] == ns checked)
    if (j->pt_off[c->chunk_leaf[k]] > j->pt_off[c->chunk_leaf[k + 1]])
      return set_err(c, FMMCU_EINVAL, "leaf offsets not monotone");
  c->group_k = K;
  c->sym_request = false;

  cudaStream_t s = c->stream, h = c->h2d_stream;
  CU_TRY(c, c->d_src.ensure(size_t(ns) * 32));
  CU_TRY(c, c->d_evy.ensure(size_t(ne) * 16));
  CU_TRY(c, c->d_eself.ensure(size_t(ne) * 4));
  CU_TRY(c, c->h_src.ensure(size_t(ns) * 32));
  CU_TRY(c, c->h_evy.ensure(size_t(ne) * 16));
  CU_TRY(c, c->h_eself.ensure(size_t(ne) * 4));
  CU_TRY(c, c->d_evr.ensure(size_t(ne) * 32));
  CU_TRY(c, c->d_hits.ensure(8));
  CU_TRY(c, c->d_counter.ensure(8));
  CU_TRY(c, c->h_hits.ensure(8));
  // output: the caller's page-locked buffer, else pinned (mapped) staging
  const uint32_t eb = j->ev_off[lb], ee = j->ev_off[le];
  cudaPointerAttributes pa{};
  void* dev_out = nullptr;
  c->direct_out = ne && cudaPointerGetAttributes(&pa, j->out) == cudaSuccess &&
                  pa.type == cudaMemoryTypeHost &&
                  cudaHostGetDevicePointer(&dev_out, j->out, 0) == cudaSuccess;
  cudaGetLastError();
  if (!c->direct_out) {
    CU_TRY(c, c->h_out.ensure(size_t(ne) * 16 + 16));
    CU_TRY(c, cudaHostGetDevicePointer(&dev_out, c->h_out.p, 0));
  }
  c->out_dev = static_cast<double2*>(dev_out);
  // host address of the same output (copy-engine D2H of the grouped mutual list)
  double2* host_out = c->direct_out ? reinterpret_cast<double2*>(j->out) : c->h_out.as<double2>();
  CU_TRY(c, c->d_out.ensure(size_t(std::max(ne, 1u)) * 16));
  tr.mark("chunks + buffers");
  CU_TRY(c, cudaEventRecord(c->ev_start, s));
  c->t_evstart = Clock::now();
  CU_TRY(c, cudaStreamWaitEvent(h, c->ev_start, 0));
  CU_TRY(c, cudaMemsetAsync(c->d_hits.p, 0, 8, s));

  const double* z = j->src_z;
  const double* m = j->src_m;
  double* hs = c->h_src.as<double>();
  uint64_t h2d = uint64_t(ns) * 32;
  // page-locked caller inputs: DMA z and m as they are and pack on the device
  // (no host staging copy); the host only runs the self-layout check
  auto pinned = [](const void* p) {
    cudaPointerAttributes at{};
    const bool ok = p && cudaPointerGetAttributes(&at, p) == cudaSuccess &&
                    at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
  };
  const bool direct_in = ns > 0 && pinned(z) && pinned(m);
  if (direct_in) {
    CU_TRY(c, c->d_zin.ensure(size_t(ns) * 16));
    CU_TRY(c, c->d_min.ensure(size_t(ns) * 16));
  }
  // Halo-only upload for a leaf range: only the sources of the range's
  // strong lists (its own leaves + a halo) are read by its kernels; the rest
  // of the device array is left untouched.
  const bool partial = lb > 0 || le < nl;
  std::vector<uint8_t> needed;
  if (partial) {
    needed.assign(nl, 0);
#pragma omp parallel for schedule(static)
    for (int64_t t = lb; t < int64_t(le); ++t)
      for (uint32_t q = j->strong_off[t]; q < j->strong_off[t + 1]; ++q)
        needed[j->strong_idx[q]] = 1;
    h2d -= uint64_t(ns) * 32;
  }
  // visit the source runs of chunk k that the range reads
  auto for_runs = [&](int k, auto&& fn) -> int {
    const uint32_t l0 = c->chunk_leaf[k], l1 = c->chunk_leaf[k + 1];
    if (!partial) return fn(int64_t(j->pt_off[l0]), int64_t(j->pt_off[l1]));
    for (uint32_t t = l0; t < l1;) {
      if (!needed[t]) {
        ++t;
        continue;
      }
      uint32_t t1 = t + 1;
      while (t1 < l1 && needed[t1]) ++t1;
      if (int rc = fn(int64_t(j->pt_off[t]), int64_t(j->pt_off[t1]))) return rc;
      t = t1;
    }
    return FMMCU_OK;
  };
  // Page-locked inputs: the first kPre chunks start moving before the work
  // list is built (~1.5 ms at 10M, two to three chunks of DMA), so the copy
  // engine never idles; the CSR and work list then queue behind only those.
  // Measured alternatives: the work list on a helper thread starves behind
  // the OpenMP team; all chunks first makes the work list upload wait for
  // the whole 320 MB (13.2 vs 10.4 ms per 10M step).
  static const int kPre = std::getenv("FMMCU_KPRE") ? std::atoi(std::getenv("FMMCU_KPRE")) : 2;
  auto dma = [&](int64_t c0, int64_t c1) -> int {
    if (c1 <= c0) return FMMCU_OK;
    CU_TRY(c, cudaMemcpyAsync(c->d_zin.as<double>() + 2 * c0, z + 2 * c0, size_t(c1 - c0) * 16,
                              cudaMemcpyHostToDevice, h));
    CU_TRY(c, cudaMemcpyAsync(c->d_min.as<double>() + 2 * c0, m + 2 * c0, size_t(c1 - c0) * 16,
                              cudaMemcpyHostToDevice, h));
    if (partial) h2d += uint64_t(c1 - c0) * 32;
    return FMMCU_OK;
  };
  // Work list.  Default: built on the device (p2p_worklist.cuh) from the CSR,
  // which leads the copy queue (~15 MB at 10M); page-locked source chunks
  // queue right behind it, so the copy engine streams from t = 0 and the
  // host only waits for one small header.  FMMCU_HOST_WL=1: the host builder
  // (~1.5 ms at 10M) with the first kPre chunks moving meanwhile, the CSR and
  // work list queued behind those only.
  const bool dev_list = !std::getenv("FMMCU_HOST_WL");
  // self layout per chunk requires eval slot e == source slot e
  const bool maybe_self = j->eval_sid && ne == ns && ns > 0 &&
                          std::memcmp(j->ev_off, j->pt_off, size_t(nl + 1) * 4) == 0;
  // the per-chunk self check reads 44 B per point, which paces the chunks at
  // host memory speed; a caller passing one array for both positions saves
  // the 32 B position comparison
  const bool y_is_z = j->eval_y == j->src_z;
  // slots [c0, c1) are self layout (ids and positions), branch-free
  // (vectorised) reductions: a short-circuit && does not vectorise
  auto self_check = [&](int64_t c0, int64_t c1) -> bool {
    const int64_t* sid = j->eval_sid;
    const uint32_t* pm = j->perm;
    const double* ey = j->eval_y;
    const double* zz = j->src_z;
    uint32_t diff = 0;
    if (y_is_z) {  // the positions are the same array: ids only
#pragma omp parallel for schedule(static) reduction(| : diff)
      for (int64_t i = c0; i < c1; ++i) diff |= uint32_t(sid[i] != int64_t(pm[i]));
    } else {
#pragma omp parallel for schedule(static) reduction(| : diff)
      for (int64_t i = c0; i < c1; ++i)
        diff |= uint32_t(sid[i] != int64_t(pm[i])) | uint32_t(ey[2 * i] != zz[2 * i]) |
                uint32_t(ey[2 * i + 1] != zz[2 * i + 1]);
    }
    return diff == 0;
  };
  // chunk 0's check runs while the work-list header is in flight (whole
  // jobs with page-locked inputs: one run per chunk)
  int self0 = -1;  // -1: not checked yet
  // FMMCU_E2E_SYM=1: the grouped mutual list for self-evaluation.  Off by
  // default: the launch is PCIe bound (H2D + D2H share the link, ~75 GB/s
  // together), the ordered kernels store each result over PCIe while they
  // compute, and the mutual list needs a finalize + copy-engine D2H per group
  // after its kernel -- 10M / L10: 8.0-8.3 ms against 7.5-7.6 ms ordered
  // (e2e).
  const bool e2e_sym = std::getenv("FMMCU_E2E_SYM") != nullptr;
  bool sym_candidate = false;
  if (dev_list && e2e_sym && j->kernel == 0 && !c->no_sym_once && !std::getenv("FMMCU_NO_SYM") &&
      j->eval_sid && ne == ns && ns > 0 &&
      std::memcmp(j->ev_off, j->pt_off, size_t(nl + 1) * 4) == 0) {
    sym_candidate = true;
    const uint32_t nchk = std::min<uint32_t>(ns, 4096);
    for (uint32_t i = 0; i < nchk && sym_candidate; ++i)
      sym_candidate = j->eval_sid[i] == int64_t(j->perm[i]) &&
                      (j->eval_y == j->src_z ||
                       (j->eval_y[2 * i] == j->src_z[2 * i] &&
                        j->eval_y[2 * i + 1] == j->src_z[2 * i + 1]));
  }
  c->no_sym_once = false;
  int pre = 0;
  if (dev_list) {
    const uint64_t csr_bytes = upload_csr(c, j, h);
    if (csr_bytes == ~0ull) return FMMCU_ECUDA;
    h2d += csr_bytes;
    CU_TRY(c, cudaEventRecord(c->ev_staged, h));
    if (direct_in) {
      pre = K;
      for (int k = 0; k < K; ++k) {
        if (int rc = for_runs(k, dma)) return rc;
        CU_TRY(c, cudaEventRecord(c->ev_chunk[k], h));
      }
    }
    if (defer_csr) {
      const int rc = validate_csr(c, j);
      tr.mark("validate (overlapped)");
      if (rc) {  // the queued copies read the caller's arrays: drain them first
        cudaStreamSynchronize(h);
        return rc;
      }
    }
    CU_TRY(c, cudaStreamWaitEvent(s, c->ev_staged, 0));
    WlGroups g{};
    g.K = uint32_t(K);
    for (int k = 0; k < K; ++k) g.slot_end[k] = j->pt_off[c->chunk_leaf[k + 1]];
    c->n_strong = j->strong_off[nl];
    // Self-evaluation with the harmonic kernel: the mutual kernel, its list
    // grouped by upload chunk (pairs inside a group once, across groups
    // ordered).  The per-chunk self-layout check below confirms it chunk by
    // chunk; a sample of the first ids decides here.
    int rc_sym = -1;
    if (sym_candidate) {
      rc_sym = build_sym_worklist_dev(c, lb, le, s, &g);
      if (rc_sym != FMMCU_OK && rc_sym != -1) return rc_sym;
    }
    if (rc_sym != FMMCU_OK) {
      const bool pre0 = maybe_self && direct_in && lb == 0 && le == nl && K > 0;
      auto check0 = [&] {
        self0 = self_check(int64_t(j->pt_off[c->chunk_leaf[0]]),
                           int64_t(j->pt_off[c->chunk_leaf[1]])) ? 1 : 0;
      };
      if (int rc = build_worklist_dev(c, lb, le, g, s,
                                      pre0 ? std::function<void()>(check0) : std::function<void()>()))
        return rc;  // + the run table
    }
    tr.mark("csr + device worklist");
  } else {
    pre = direct_in ? std::min(K, std::max(0, kPre)) : 0;
    for (int k = 0; k < pre; ++k) {
      if (int rc = for_runs(k, dma)) return rc;
      CU_TRY(c, cudaEventRecord(c->ev_chunk[k], h));
    }
    if (int rc = build_worklist(c, j)) return rc;
    tr.mark("worklist");
    if (int rc = stage_csr(c, j, false)) return rc;
    // the remaining chunks queue behind the CSR and work list: on their own
    // stream the copy engine would serve them first and starve the kernels
    CU_TRY(c, cudaEventRecord(c->ev_staged, s));
    CU_TRY(c, cudaStreamWaitEvent(h, c->ev_staged, 0));
    h2d += c->h2d_bytes - uint64_t(ns) * 32 - (c->self_layout ? 0 : uint64_t(ne) * 20);
  }
  c->run_eb = eb;
  c->run_ee = ee;
  const P2PItem* items_dev = c->d_items.as<P2PItem>();
  const P2PFinal* fins_dev = c->d_fin.as<P2PFinal>();
  tr.mark("csr");
  double2* hy = c->h_evy.as<double2>();
  uint32_t* hself = c->h_eself.as<uint32_t>();
  bool all_self = maybe_self;
  // eval arrays of slots [e0, e1) on the host (non-self chunks / layouts)
  bool inv_ready = false;
  auto host_evals = [&](int64_t e0, int64_t e1) -> int {
    if (j->eval_sid && !inv_ready) {
      c->invperm.resize(ns);
      uint32_t* inv = c->invperm.data();
      bool ok = true;
#pragma omp parallel for schedule(static) reduction(&& : ok)
      for (int64_t i = 0; i < int64_t(ns); ++i) {
        if (j->perm[i] >= ns) ok = false;
        else inv[j->perm[i]] = uint32_t(i);
      }
      if (!ok) return set_err(c, FMMCU_EINVAL, "perm is not a permutation of the sources");
      inv_ready = true;
    }
    const uint32_t* inv = c->invperm.data();
#pragma omp parallel for schedule(static)
    for (int64_t e = e0; e < e1; ++e) {
      hy[e] = make_double2(j->eval_y[2 * e], j->eval_y[2 * e + 1]);
      const int64_t sv = j->eval_sid ? j->eval_sid[e] : -1;
      hself[e] = (sv >= 0 && sv < int64_t(ns)) ? inv[sv] : kNoSelf;
    }
    return FMMCU_OK;
  };
  bool evals_event = false;
  if (!maybe_self && ne) {
    if (int rc = host_evals(0, ne)) return rc;
    CU_TRY(c, cudaMemcpyAsync(c->d_evy.p, hy, size_t(ne) * 16, cudaMemcpyHostToDevice, h));
    CU_TRY(c, cudaMemcpyAsync(c->d_eself.p, hself, size_t(ne) * 4, cudaMemcpyHostToDevice, h));
    CU_TRY(c, cudaEventRecord(c->ev_evals, h));
    evals_event = true;
    h2d += uint64_t(ne) * 20;
  }

  std::vector<char> chunk_self(K, 0);
  int launched = 0;
  int nk = 0;
  static const bool two_streams = !(std::getenv("FMMCU_GRP_STREAMS") &&
                                    std::atoi(std::getenv("FMMCU_GRP_STREAMS")) == 1);
  auto run_group = [&](int k) -> int {
    CU_TRY(c, cudaStreamWaitEvent(s, c->ev_chunk[k], 0));
    if (evals_event) CU_TRY(c, cudaStreamWaitEvent(s, c->ev_evals, 0));
    const uint32_t l0 = c->chunk_leaf[k], l1 = c->chunk_leaf[k + 1];
    const uint32_t a0 = j->ev_off[l0], a1 = j->ev_off[l1];
    if (maybe_self && !chunk_self[k] && a1 > a0) {  // this chunk's evals are not its sources
      CU_TRY(c, cudaMemcpyAsync(c->d_evy.as<double2>() + a0, hy + a0, size_t(a1 - a0) * 16,
                                cudaMemcpyHostToDevice, s));
      CU_TRY(c, cudaMemcpyAsync(c->d_eself.as<uint32_t>() + a0, hself + a0,
                                size_t(a1 - a0) * 4, cudaMemcpyHostToDevice, s));
    }
    if (direct_in) {
      const uint32_t s0 = j->pt_off[l0], s1 = j->pt_off[l1];
      if (s1 > s0) {
        pack_zm_kernel<<<(s1 - s0 + 255) / 256, 256, 0, s>>>(c->d_zin.as<double2>(),
                                                            c->d_min.as<double2>(), s0, s1,
                                                            c->d_src.as<double4>());
        ++nk;
      }
    }
    P2PArgs a = make_args(c);
    a.out = c->out_dev;
    if (a1 > a0) {
      if (chunk_self[k]) {
        p2p_self_evals_kernel<<<(a1 - a0 + 255) / 256, 256, 0, s>>>(
            c->d_src.as<double4>(), a0, a1, c->d_evy.as<double2>(), c->d_eself.as<uint32_t>());
        ++nk;
      }
      p2p_evrec_kernel<<<(l1 - l0 + 7) / 8, 256, 0, s>>>(a, l0, l1, c->d_evr.as<double4>());
      ++nk;
    }
    uint32_t i0, i1, f0, f1;
    if (c->dev_wl || c->sym_items) {  // device-built lists (ordered or mutual)
      i0 = c->dev_grp_item[k];
      i1 = c->dev_grp_item[k + 1];
      f0 = c->dev_grp_fin[k];
      f1 = c->dev_grp_fin[k + 1];
    } else {
      const uint32_t p0 = c->grp_pos[k], p1 = c->grp_pos[k + 1];
      i0 = c->item_first[p0];
      i1 = c->item_first[p1];
      f0 = c->fin_first[p0];
      f1 = c->fin_first[p1];
    }
    // The group's P2P kernels alternate between two streams behind the chunk
    // preparation on s, so group k+1 fills the SMs while group k's last items
    // drain; each stream has its own scheduler counter.  Group k reads only
    // sources and eval records of chunks <= k, all prepared on s before
    // ev_prep[k]; partial slots are per item.  FMMCU_GRP_STREAMS=1: one stream.
    cudaStream_t gs = s;
    unsigned int* counter = c->d_counter.as<unsigned int>();
    if (two_streams) {
      CU_TRY(c, cudaEventRecord(c->ev_prep[k], s));
      gs = c->grp_stream[k & 1];
      CU_TRY(c, cudaStreamWaitEvent(gs, c->ev_prep[k], 0));
      counter += (k & 1);
    }
    if (c->sym_items) {  // grouped mutual list: f0 / f1 are leaf positions
      if (i1 > i0) {
        CU_TRY(c, cudaMemsetAsync(counter, 0, 4, gs));
        P2PArgs aa = a;
        aa.items = items_dev + i0;
        aa.n_items = i1 - i0;
        aa.next_item = counter;
        P2PSymArgs sa{c->d_symseg.as<uint4>(), c->d_tgt.as<double2>(),
                      c->d_contrib.as<double2>()};
        dispatch_sym(c->smoother, aa, sa, i1 - i0, gs, c->warp_e, c->sym_rounds);
        ++nk;
      }
      // Results.  Leaves of chunk k go to device memory and chunk k's eval
      // range goes down by one copy-engine D2H (d2h stream, in chunk order)
      // after this finalize; the few leaves of earlier chunks that land in
      // group k (a partner in chunk k) are written straight into the host
      // output by TMA bulk stores -- after the D2H of chunk k - 1, hence of
      // their own chunk, whose stale copy of them they replace.  (All 160 MB
      // as SM stores to mapped memory held each group's finalize for the
      // whole transfer and slowed the H2D chunks by 14%.)
      const uint32_t c0 = std::max(lb, l0), c1 = std::min(le, l1);
      auto fin = [&](int host_part) {
        p2p_sym_finalize_bulk_kernel<<<(f1 - f0 + kFinWarps - 1) / kFinWarps, kFinWarps * 32, 0,
                                       gs>>>(
            lb, f1 - f0, c->d_pt.as<uint32_t>(), c->d_cloff.as<uint32_t>(),
            c->d_clbase.as<uint32_t>(), c->d_tgt.as<double2>(), c->d_contrib.as<double2>(),
            c->out_dev, c->sym_order, f0, c0, c1, c->d_out.as<double2>(), host_part);
        ++nk;
      };
      if (f1 > f0) fin(0);
      CU_TRY(c, cudaEventRecord(c->ev_fin[k], gs));
      CU_TRY(c, cudaStreamWaitEvent(c->d2h_stream, c->ev_fin[k], 0));
      if (c1 > c0) {
        const uint32_t e0 = j->ev_off[c0], e1 = j->ev_off[c1];
        if (e1 > e0)
          CU_TRY(c, cudaMemcpyAsync(host_out + e0, c->d_out.as<double2>() + e0,
                                    size_t(e1 - e0) * 16, cudaMemcpyDeviceToHost, c->d2h_stream));
      }
      CU_TRY(c, cudaEventRecord(c->ev_copy[k], c->d2h_stream));
      if (k > 0 && f1 > f0) {  // leaves of earlier chunks: after those chunks' copies
        CU_TRY(c, cudaStreamWaitEvent(gs, c->ev_copy[k - 1], 0));
        fin(1);
      }
      CU_TRY(c, cudaEventRecord(c->ev_group[k], gs));
      CU_TRY(c, cudaGetLastError());
      return FMMCU_OK;
    }
    if (i1 > i0) {
      CU_TRY(c, cudaMemsetAsync(counter, 0, 4, gs));
      P2PArgs aa = a;
      aa.items = items_dev + i0;
      aa.n_items = i1 - i0;
      aa.next_item = counter;
      dispatch_tile(c->kernel, c->smoother, aa, i1 - i0, gs, c->warp_e);
      ++nk;
    }
    if (f1 > f0) {
      p2p_finalize_kernel<<<f1 - f0, 128, 0, gs>>>(fins_dev + f0, f1 - f0,
                                                    c->d_partial.as<double2>(), c->out_dev);
      ++nk;
    }
    CU_TRY(c, cudaEventRecord(c->ev_group[k], gs));
    CU_TRY(c, cudaGetLastError());
    return FMMCU_OK;
  };

  // pack / DMA source slots [c0, c1) and self-check them; returns the check
  auto upload = [&](int64_t c0, int64_t c1, int k) -> int {
    bool same = maybe_self;
    if (direct_in) {
      if (k >= pre)
        if (int rc = dma(c0, c1)) return rc;
      if (maybe_self) same = (k == 0 && self0 >= 0) ? self0 == 1 : self_check(c0, c1);
    } else {
#pragma omp parallel for schedule(static) reduction(&& : same)
      for (int64_t i = c0; i < c1; ++i) {
        hs[4 * i + 0] = z[2 * i];
        hs[4 * i + 1] = z[2 * i + 1];
        hs[4 * i + 2] = m[2 * i];
        hs[4 * i + 3] = m[2 * i + 1];
        if (maybe_self)
          same = same && j->eval_sid[i] == int64_t(j->perm[i]) &&
                 j->eval_y[2 * i] == z[2 * i] && j->eval_y[2 * i + 1] == z[2 * i + 1];
      }
      if (c1 > c0)
        CU_TRY(c, cudaMemcpyAsync(c->d_src.as<double>() + 4 * c0, hs + 4 * c0,
                                  size_t(c1 - c0) * 32, cudaMemcpyHostToDevice, h));
    }
    if (partial && !direct_in) h2d += uint64_t(c1 - c0) * 32;
    if (maybe_self && !same && c1 > c0) {
      if (int rc = host_evals(c0, c1)) return rc;
      h2d += uint64_t(c1 - c0) * 20;
    }
    if (!same) chunk_self[k] = 0;
    return FMMCU_OK;
  };

  for (int k = 0; k < K; ++k) {
    chunk_self[k] = maybe_self ? 1 : 0;
    if (int rc = for_runs(k, [&](int64_t c0, int64_t c1) { return upload(c0, c1, k); })) return rc;
    if (k >= pre) CU_TRY(c, cudaEventRecord(c->ev_chunk[k], h));
    if (c->sym_items && !chunk_self[k]) {
      // the mutual list assumed the self layout and chunk k breaks it: drain
      // what was queued and redo the job with the ordered list (correct
      // either way; only jobs whose first ids match their sources get here)
      for (cudaStream_t q : {s, h, c->grp_stream[0], c->grp_stream[1]})
        if (q) CU_TRY(c, cudaStreamSynchronize(q));
      c->no_sym_once = true;
      return launch_overlapped(c, j);
    }
    const bool same = chunk_self[k] != 0;
    all_self = all_self && same;
    if (c->trace)
      std::fprintf(stderr, "[fmmcu] chunk %2d enqueued at %8.3f ms\n", k,
                   std::chrono::duration<double, std::milli>(Clock::now() - c->t_evstart).count());
    if (int rc = run_group(launched++)) return rc;
  }
  tr.mark("pack+h2d (overlapped)");
  c->self_layout = all_self;
  if (two_streams)  // the last group of each group stream
    for (int g = std::max(0, K - 2); g < K; ++g) CU_TRY(c, cudaStreamWaitEvent(s, c->ev_group[g], 0));
  if (c->sym_items && K > 0)  // the last chunk's D2H (grouped mutual list)
    CU_TRY(c, cudaStreamWaitEvent(s, c->ev_copy[K - 1], 0));
  CU_TRY(c, cudaMemcpyAsync(c->h_hits.p, c->d_hits.p, 8, cudaMemcpyDeviceToHost, s));
  CU_TRY(c, cudaEventRecord(c->ev_end, s));
  tr.mark("enqueue done");
  c->launches += uint64_t(nk);
  c->h2d_bytes = h2d;
  c->d2h_bytes = uint64_t(ee - eb) * 16 + 8;
  c->n_slices = 0;
  c->n_groups = K;
  return FMMCU_OK;
}

// Kernels over [lb, le) of the staged job.
int run_kernels(fmmcu_ctx* c, uint32_t lb, uint32_t le, int mode, int* nlaunch,
                bool reset_hits) {
  cudaStream_t s = c->stream;
  int n = 0;
  if (reset_hits) CU_TRY(c, cudaMemsetAsync(c->d_hits.p, 0, 8, s));
  CU_TRY(c, cudaMemsetAsync(c->d_counter.p, 0, 8, s));
  const P2PArgs a = make_args(c);
  if (le > lb) {
    if (mode == FMMCU_MODE_EXACT) {
      const uint32_t eb = c->ev_off[lb], ee = c->ev_off[le];
      if (ee > eb) {
        dispatch_exact(c->kernel, c->smoother, a, lb, le, eb, ee, s);
        ++n;
      }
    } else if (c->sym_items) {
      if (lb != c->sym_lb || le != c->sym_le)
        return set_err(c, FMMCU_ESTATE, "symmetric work list staged for another leaf range");
      const uint32_t ni = c->sym_n_items;
      P2PSymArgs sa{c->d_symseg.as<uint4>(), c->d_tgt.as<double2>(), c->d_contrib.as<double2>()};
      if (ni) {
        P2PArgs aa = a;
        aa.n_items = ni;
        dispatch_sym(c->smoother, aa, sa, ni, s, c->warp_e, c->sym_rounds);
        ++n;
      }
      const uint32_t nlr = le - lb;
      p2p_sym_finalize_kernel<<<(nlr + 7) / 8, 256, 0, s>>>(
          lb, nlr, c->d_pt.as<uint32_t>(), c->d_cloff.as<uint32_t>(), c->d_clbase.as<uint32_t>(),
          c->d_tgt.as<double2>(), c->d_contrib.as<double2>(), c->out_ptr());
      ++n;
    } else {
      uint32_t i0, i1, f0, f1;
      if (c->dev_wl) {  // device-built list: its whole (ungrouped) range only
        if (lb != c->dev_wl_lb || le != c->dev_wl_le || c->grouped)
          return set_err(c, FMMCU_ESTATE, "device work list staged for another leaf range");
        i0 = c->dev_grp_item.front();
        i1 = c->dev_grp_item.back();
        f0 = c->dev_grp_fin.front();
        f1 = c->dev_grp_fin.back();
      } else {
        i0 = c->item_first[lb];
        i1 = c->item_first[le];
        f0 = c->fin_first[lb];
        f1 = c->fin_first[le];
      }
      if (i1 > i0) {
        P2PArgs aa = a;
        aa.items = c->d_items.as<P2PItem>() + i0;
        aa.n_items = i1 - i0;
        dispatch_tile(c->kernel, c->smoother, aa, i1 - i0, s, c->warp_e);
        ++n;
      }
      if (f1 > f0) {
        p2p_finalize_kernel<<<f1 - f0, 128, 0, s>>>(c->d_fin.as<P2PFinal>() + f0, f1 - f0,
                                                     c->d_partial.as<double2>(),
                                                     c->out_ptr());
        ++n;
      }
    }
  }
  CU_TRY(c, cudaGetLastError());
  c->launches += uint64_t(n);
  if (nlaunch) *nlaunch = n;
  return FMMCU_OK;
}

// FP64 peak: independent DFMA chains, 8 per thread.
__global__ void dfma_peak_kernel(double* sink, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4,
         a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, b = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, b); a1 = fma(a1, m, b); a2 = fma(a2, m, b); a3 = fma(a3, m, b);
      a4 = fma(a4, m, b); a5 = fma(a5, m, b); a6 = fma(a6, m, b); a7 = fma(a7, m, b);
    }
  }
  const double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (r == 12345.678) sink[0] = r;
}

// binomial table T[k][l] of the M2L kernel (Pascal recurrence in doubles,
// as the reference's table, expansion.cpp:12-26)
int m2l_table(fmmcu_ctx* c, int p, int kernel, cudaStream_t stream) {
  if (c->table_p == p && c->table_kernel == kernel) return FMMCU_OK;
  const int P1 = p + 1;
  const int rows = 2 * P1 + 2;
  std::vector<double> pas(size_t(rows) * rows, 0.0);
  for (int i = 0; i < rows; ++i) {
    pas[size_t(i) * rows] = 1.0;
    for (int k = 1; k <= i; ++k)
      pas[size_t(i) * rows + k] = pas[size_t(i - 1) * rows + k - 1] + pas[size_t(i - 1) * rows + k];
  }
  std::vector<double> T(size_t(P1) * P1, 0.0);
  for (int k = 0; k < P1; ++k)
    for (int l = 0; l < P1; ++l) {
      if (kernel == 0) T[size_t(k) * P1 + l] = pas[size_t(l + k) * rows + k];
      else if (k >= 1) T[size_t(k) * P1 + l] = pas[size_t(l + k - 1) * rows + (k - 1)];
    }
  CU_TRY(c, c->m_table.ensure(T.size() * 8));
  // Stream-ordered upload on the consuming stream. A legacy-stream cudaMemcpy
  // from pageable memory may return before the DMA lands, and the consumers
  // (cudaMemcpyToSymbolAsync into c_m2l_table, the M2L kernels) run on
  // non-blocking streams that do not order behind the legacy stream. The
  // pageable source is staged before cudaMemcpyAsync returns, so T may die.
  CU_TRY(c, cudaMemcpyAsync(c->m_table.p, T.data(), T.size() * 8, cudaMemcpyHostToDevice, stream));
  c->table_p = p;
  c->table_kernel = kernel;
  return FMMCU_OK;
}

// All M2L sums of a job on `s` (C-ABI M2L and device pipeline): the binomial
// table, then the register kernel over work items (weak lists longer than
// kM2LChunk split into chunks, reduced in chunk order) for the orders it is
// instantiated for, else the r1 per-target kernels.  a.p, a.kernel, centres,
// coefficients, targets, lists, out and singular must be set; nnz is the
// weak-list length (a bound for the item and partial buffers).
int m2l_run(fmmcu_ctx* c, M2LArgs a, uint64_t nnz, cudaStream_t s) {
  if (a.n_targets == 0) return FMMCU_OK;
  if (int rc = m2l_table(c, a.p, a.kernel, s)) return rc;
  const int P1 = a.p + 1;
  a.table = c->m_table.as<double>();
  // (p+2) log10|w| >= 250  <=>  |w|^2 >= 10^(500/(p+2))
  a.big_w2 = std::pow(10.0, 500.0 / double(a.p + 2));
  // FMMCU_M2L=old (or FMMCU_M2L_OLD=1): the r1 per-target kernels, for A/B
  // runs.  (A warp-per-item variant -- lane = partner, rows staged with
  // cp.async, shuffle-tree reduction -- measured 2.9 ms against 1.27 ms at
  // 10M / L10 and was dropped.)
  static const bool old = [] {
    const char* e = std::getenv("FMMCU_M2L");
    return m2l_old_kernel() || (e && std::strcmp(e, "old") == 0);
  }();
  int tb = 64;
  M2LKernelFn reg = nullptr;
  if (!old) reg = a.kernel == 0 ? m2l_reg_for<true>(P1, &tb) : m2l_reg_for<false>(P1, &tb);
  const uint32_t chunk = kM2LChunk;
  if (!reg) {
    CU_TRY(c, m2l_set_const_table(c->m_table.as<double>(), P1, s));
    launch_m2l_targets(a, s);
    CU_TRY(c, cudaGetLastError());
    c->launches += 1;
    return FMMCU_OK;
  }
  const uint32_t nt = a.n_targets;
  const uint64_t max_items = uint64_t(nt) + nnz / chunk + 1;
  const uint64_t max_slots = 2 * (nnz / chunk) + 2;
  if (max_items > 0xFFFFFFF0ull || max_slots > 0xFFFFFFF0ull)
    return set_err(c, FMMCU_EINVAL, "m2l: too many work items");
  CU_TRY(c, c->m_items.ensure(max_items * 16));
  CU_TRY(c, c->m_iscan.ensure((uint64_t(nt) + 1) * 8 * 2));
  CU_TRY(c, c->m_nitems.ensure(8));
  CU_TRY(c, c->m_partial.ensure(max_slots * uint64_t(P1) * 16));
  auto* cnt = c->m_iscan.as<unsigned long long>();
  auto* off = cnt + (nt + 1);
  m2l_item_count_kernel<<<(nt + 256) / 256, 256, 0, s>>>(a.weak_off, nt, chunk, cnt);
  size_t tmp = 0;
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, off, int64_t(nt) + 1, s));
  CU_TRY(c, c->m_cubtmp.ensure(tmp));
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(c->m_cubtmp.p, tmp, cnt, off, int64_t(nt) + 1, s));
  m2l_item_fill_kernel<<<(nt + 255) / 256, 256, 0, s>>>(a.weak_off, nt, off,
                                                        c->m_items.as<uint4>(),
                                                        c->m_nitems.as<uint32_t>());
  a.items = c->m_items.as<uint4>();
  a.n_items = c->m_nitems.as<uint32_t>();
  a.partial = c->m_partial.as<double2>();
  // one item per thread over a grid covering the item bound: the block
  // scheduler balances the tail (a persistent grid measured 1.45 against
  // 1.27 ms at 10M)
  const uint32_t grid = uint32_t(std::max<uint64_t>(1, (max_items + tb - 1) / tb));
  reg<<<grid, tb, 0, s>>>(a);
  const uint64_t nred = uint64_t(nt) * P1;
  m2l_reduce_kernel<<<uint32_t((nred + 255) / 256), 256, 0, s>>>(off, nt, P1, a.partial, a.out);
  CU_TRY(c, cudaGetLastError());
  c->launches += 4;
  return FMMCU_OK;
}

}  // namespace fmmcu::detail

using namespace fmmcu::detail;

// =============================================================== C ABI ====
extern "C" {

int fmmcu_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (count) *count = (e == cudaSuccess) ? n : 0;
  return e == cudaSuccess ? FMMCU_OK : FMMCU_ECUDA;
}

int fmmcu_create(fmmcu_ctx** out, int device) {
  if (!out) return FMMCU_EINVAL;
  *out = nullptr;
  auto* c = new (std::nothrow) fmmcu_ctx();
  if (!c) return FMMCU_ENOMEM;
  c->device = device;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || device < 0 || device >= n) {
    // keep the context so the caller can read the message, then fail
    static thread_local std::string last;
    last = std::string("no CUDA device ") + std::to_string(device) + " (" +
           (e == cudaSuccess ? std::to_string(n) + " visible" : cudaGetErrorString(e)) + ")";
    c->err = last;
    *out = c;
    return FMMCU_ECUDA;
  }
  auto fail = [&](cudaError_t er) {
    c->err = cudaGetErrorString(er);
    *out = c;
    return FMMCU_ECUDA;
  };
  if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(e);
  c->d_out.plain = true;  // exported over CUDA IPC (fmmcu_p2p_out_ipc_handle)
  if ((e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(e);
  if ((e = cudaStreamCreateWithFlags(&c->m2l_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(e);
  if ((e = cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(e);
  if ((e = cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(e);
  {
    // the device work list is a short chain of small latency-bound kernels on
    // the pipeline's critical path, run beside the far-field kernels: give
    // it the highest stream priority
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if ((e = cudaStreamCreateWithPriority(&c->wl_stream, cudaStreamNonBlocking, hi)) != cudaSuccess)
      return fail(e);
  }
  if ((e = cudaEventCreateWithFlags(&c->ev_evals, cudaEventDisableTiming)) != cudaSuccess)
    return fail(e);
  if ((e = cudaEventCreateWithFlags(&c->ev_staged, cudaEventDisableTiming)) != cudaSuccess)
    return fail(e);
  for (cudaStream_t& gs : c->grp_stream)
    if ((e = cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  for (cudaEvent_t& ep : c->ev_prep)
    if ((e = cudaEventCreateWithFlags(&ep, cudaEventDisableTiming)) != cudaSuccess) return fail(e);
  for (int i = 0; i < fmmcu_ctx::kMaxChunks; ++i)
    if ((e = cudaEventCreateWithFlags(&c->ev_fin[i], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_copy[i], cudaEventDisableTiming)) != cudaSuccess)
      return fail(e);
  for (int i = 0; i < fmmcu_ctx::kMaxChunks; ++i)
    if ((e = cudaEventCreateWithFlags(&c->ev_chunk[i], cudaEventDefault)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_group[i], cudaEventDefault)) != cudaSuccess)
      return fail(e);
  c->stream = c->own_stream;
  const unsigned flags = cudaEventBlockingSync;
  for (int i = 0; i < fmmcu_ctx::kMaxSlices; ++i) {
    if ((e = cudaEventCreateWithFlags(&c->ev_kslice[i], cudaEventDefault)) != cudaSuccess)
      return fail(e);
    if ((e = cudaEventCreateWithFlags(&c->ev_cslice[i], cudaEventDisableTiming | flags)) !=
        cudaSuccess)
      return fail(e);
  }
  if ((e = cudaEventCreateWithFlags(&c->ev_start, flags)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreateWithFlags(&c->ev_end, flags)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreateWithFlags(&c->ev_m2l0, flags)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreateWithFlags(&c->ev_m2l1, flags)) != cudaSuccess) return fail(e);
  *out = c;
  return FMMCU_OK;
}

void fmmcu_destroy(fmmcu_ctx* c) {
  if (!c) return;
  int n = 0;
  if (cudaGetDeviceCount(&n) == cudaSuccess && c->device < n && c->own_stream) {
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->own_stream);
    if (c->stream != c->own_stream) cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->m2l_stream);
    cudaStreamSynchronize(c->d2h_stream);
    cudaStreamSynchronize(c->h2d_stream);
    if (c->wl_stream) cudaStreamSynchronize(c->wl_stream);
    fmmcu::destroy_pipeline(c->pipe);
    c->pipe = nullptr;
    multi_release(c);
    for (DevBuf* b : {&c->d_symseg, &c->d_syminfo, &c->d_symcnt, &c->d_tgt, &c->d_contrib, &c->d_cloff,
                      &c->d_clcnt, &c->d_clbase, &c->d_cubtmp})
      b->release();
    c->h_sym.release();
    for (DevBuf* b : {&c->d_zin, &c->d_min, &c->d_src, &c->d_evy, &c->d_eself, &c->d_pt, &c->d_ev, &c->d_soff,
                      &c->d_sidx, &c->d_items, &c->d_fin, &c->d_out, &c->d_partial, &c->d_hits, &c->d_seg, &c->d_counter, &c->d_evr,
                      &c->m_centers, &c->m_coeffs, &c->m_tbox, &c->m_woff, &c->m_widx,
                      &c->m_table, &c->m_out, &c->m_flag, &c->m_items, &c->m_iscan, &c->m_nitems,
                      &c->m_partial, &c->m_cubtmp, &c->d_wl_head, &c->d_wl_key, &c->d_wl_val,
                      &c->d_wl_S, &c->d_wl_work, &c->d_wl_cnt, &c->d_wl_off, &c->d_wls,
                      &c->m_loc, &c->m_tof, &c->m_binom})
      b->release();
    for (HostBuf* b : {&c->h_src, &c->h_evy, &c->h_eself, &c->h_out, &c->h_hits, &c->h_csr,
                       &c->mh_out, &c->mh_flag, &c->h_wl_head, &c->mb_centers, &c->mb_coeffs,
                       &c->mb_out, &c->mb_tbox, &c->mb_woff, &c->mb_widx})
      b->release();
    for (cudaEvent_t ev : {c->ev_start, c->ev_end, c->ev_m2l0, c->ev_m2l1})
      if (ev) cudaEventDestroy(ev);
    for (int i = 0; i < fmmcu_ctx::kMaxSlices; ++i) {
      if (c->ev_kslice[i]) cudaEventDestroy(c->ev_kslice[i]);
      if (c->ev_cslice[i]) cudaEventDestroy(c->ev_cslice[i]);
    }
    cudaStreamDestroy(c->own_stream);
    cudaStreamDestroy(c->m2l_stream);
    cudaStreamDestroy(c->d2h_stream);
    cudaStreamDestroy(c->h2d_stream);
    if (c->wl_stream) cudaStreamDestroy(c->wl_stream);
    if (c->ev_evals) cudaEventDestroy(c->ev_evals);
    if (c->ev_staged) cudaEventDestroy(c->ev_staged);
    for (cudaStream_t gs : c->grp_stream)
      if (gs) cudaStreamSynchronize(gs), cudaStreamDestroy(gs);
    for (cudaEvent_t ep : c->ev_prep)
      if (ep) cudaEventDestroy(ep);
    for (int i = 0; i < fmmcu_ctx::kMaxChunks; ++i) {
      if (c->ev_fin[i]) cudaEventDestroy(c->ev_fin[i]);
      if (c->ev_copy[i]) cudaEventDestroy(c->ev_copy[i]);
    }
    for (int i = 0; i < fmmcu_ctx::kMaxChunks; ++i)
      if (c->ev_chunk[i]) cudaEventDestroy(c->ev_chunk[i]);
    for (int i = 0; i < fmmcu_ctx::kMaxChunks; ++i)
      if (c->ev_group[i]) cudaEventDestroy(c->ev_group[i]);
  }
  delete c;
}

const char* fmmcu_last_error(const fmmcu_ctx* c) { return c ? c->err.c_str() : "null context"; }

uint64_t fmmcu_kernel_launches(const fmmcu_ctx* c) { return c ? c->launches : 0; }

int fmmcu_last_transfer_bytes(const fmmcu_ctx* c, uint64_t* h2d, uint64_t* d2h) {
  if (!c) return FMMCU_EINVAL;
  if (h2d) *h2d = c->h2d_bytes;
  if (d2h) *d2h = c->d2h_bytes;
  return FMMCU_OK;
}

int fmmcu_set_stream(fmmcu_ctx* c, void* stream) {
  if (!c) return FMMCU_EINVAL;
  c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
  return FMMCU_OK;
}

int fmmcu_synchronize(fmmcu_ctx* c) {
  if (!c) return FMMCU_EINVAL;
  CU_TRY(c, cudaSetDevice(c->device));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return FMMCU_OK;
}

int fmmcu_p2p_launch(fmmcu_ctx* c, const fmmcu_p2p_job* j) {
  if (!c) return FMMCU_EINVAL;
  if (c->inflight) return set_err(c, FMMCU_ESTATE, "launch while a job is in flight");
  const auto t0 = Clock::now();
  if (j && j->n_eval > 0 && !j->out) return set_err(c, FMMCU_EINVAL, "null output");
  if (j && j->mode == FMMCU_MODE_FAST && !std::getenv("FMMCU_NO_OVERLAP")) {
    if (int rc = launch_overlapped(c, j)) return rc;
    c->overlapped = true;
    c->job = *j;
    c->run_lb = j->leaf_begin;
    c->run_le = j->leaf_end;
    c->run_total_pairs = c->dev_list ? c->dev_list_total
                                     : c->leaf_work[j->leaf_end] - c->leaf_work[j->leaf_begin];
    c->prep_seconds = std::chrono::duration<double>(c->t_evstart - t0).count();
    c->inflight = true;
    return FMMCU_OK;
  }
  c->overlapped = false;
  if (int rc = stage_job(c, j)) return rc;
  const uint32_t lb = j->leaf_begin, le = j->leaf_end;
  const uint32_t eb = c->ev_off[lb], ee = c->ev_off[le];
  // A page-locked output (cudaHostRegister / fmmcu_host_register) receives
  // the D2H directly; otherwise it goes through pinned staging.
  cudaPointerAttributes pa{};
  c->direct_out = j->out && cudaPointerGetAttributes(&pa, j->out) == cudaSuccess &&
                  pa.type == cudaMemoryTypeHost;
  cudaGetLastError();  // clear a "not a device pointer" status on old drivers
  double2* dst = reinterpret_cast<double2*>(j->out);
  if (!c->direct_out) {
    CU_TRY(c, c->h_out.ensure(size_t(c->n_eval) * 16 + 16));
    dst = c->h_out.as<double2>();
  }
  // Kernels in pair-work-balanced leaf slices; slice i's potentials go D2H
  // on the copy stream while slice i+1 computes.
  const uint64_t w0 = c->leaf_work[lb], w1 = c->leaf_work[le];
  int ns = (ee - eb > (1u << 20) && j->mode == FMMCU_MODE_FAST) ? fmmcu_ctx::kMaxSlices : 1;
  uint32_t cut[fmmcu_ctx::kMaxSlices + 1];
  cut[0] = lb;
  for (int i = 1; i < ns; ++i) {
    const uint64_t target = w0 + (w1 - w0) * uint64_t(i) / uint64_t(ns);
    const uint64_t* b = c->leaf_work.data();
    uint32_t t = uint32_t(std::lower_bound(b + cut[i - 1], b + le, target) - b);
    cut[i] = std::max(cut[i - 1], std::min(t, le));
  }
  cut[ns] = le;
  c->n_slices = ns;
  for (int i = 0; i < ns; ++i) {
    int nl = 0;
    if (int rc = run_kernels(c, cut[i], cut[i + 1], j->mode, &nl, i == 0)) return rc;
    const uint32_t sb = c->ev_off[cut[i]], se = c->ev_off[cut[i + 1]];
    c->slice_eb[i] = sb;
    c->slice_eb[i + 1] = se;
    CU_TRY(c, cudaEventRecord(c->ev_kslice[i], c->stream));
    CU_TRY(c, cudaStreamWaitEvent(c->d2h_stream, c->ev_kslice[i], 0));
    if (se > sb)
      CU_TRY(c, cudaMemcpyAsync(dst + sb, c->out_ptr() + sb, size_t(se - sb) * 16,
                                cudaMemcpyDeviceToHost, c->d2h_stream));
    if (i == ns - 1)
      CU_TRY(c, cudaMemcpyAsync(c->h_hits.p, c->d_hits.p, 8, cudaMemcpyDeviceToHost,
                                c->d2h_stream));
    CU_TRY(c, cudaEventRecord(c->ev_cslice[i], c->d2h_stream));
  }
  CU_TRY(c, cudaEventRecord(c->ev_end, c->d2h_stream));
  if (c->trace)
    std::fprintf(stderr, "[fmmcu] launch total (host)     %8.3f ms  (%d slices)\n",
                 std::chrono::duration<double, std::milli>(Clock::now() - t0).count(), ns);
  // the compute stream must not run ahead of the copies that read d_out
  CU_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_end, 0));
  c->job = *j;
  c->d2h_bytes = uint64_t(ee - eb) * 16 + 8;
  c->run_lb = lb;
  c->run_le = le;
  c->run_total_pairs = w1 - w0;
  // busy time = host work before the first device operation + device span
  // (ev_start .. ev_end covers packing-overlapped uploads, kernels, D2H)
  c->prep_seconds = std::chrono::duration<double>(c->t_evstart - t0).count();
  c->inflight = true;
  return FMMCU_OK;
}

int fmmcu_p2p_finish(fmmcu_ctx* c, uint64_t* pair_evals, double* seconds) {
  if (!c) return FMMCU_EINVAL;
  if (!c->inflight) return set_err(c, FMMCU_ESTATE, "finish without launch");
  c->inflight = false;
  CU_TRY(c, cudaSetDevice(c->device));
  // staged output: copy each slice out as soon as its D2H has landed
  for (int i = 0; i < c->n_slices; ++i) {
    CU_TRY(c, wait_event(c->ev_cslice[i]));
    const uint32_t sb = c->slice_eb[i], se = c->slice_eb[i + 1];
    if (!c->direct_out && se > sb)
      par_memcpy(c->job.out + 2 * size_t(sb), c->h_out.as<double2>() + sb, size_t(se - sb) * 16);
  }
  CU_TRY(c, wait_event(c->ev_end));
  CU_TRY(c, cudaGetLastError());
  if (c->overlapped && c->trace) {
    for (int k = 0; k < c->n_groups; ++k) {
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, c->ev_start, c->ev_chunk[k]);
      cudaEventElapsedTime(&b, c->ev_start, c->ev_group[k]);
      std::fprintf(stderr,
                   "[fmmcu] group %2d: chunk landed %8.3f ms, kernels done %8.3f ms, items %u\n",
                   k, a, b,
                   (c->dev_wl || c->sym_items) ? c->dev_grp_item[k + 1] - c->dev_grp_item[k]
                             : c->item_first[c->grp_pos[k + 1]] - c->item_first[c->grp_pos[k]]);
    }
  }
  if (c->overlapped && !c->direct_out) {
    const uint32_t eb = c->run_eb, ee = c->run_ee;
    if (ee > eb)
      par_memcpy(c->job.out + 2 * size_t(eb), c->h_out.as<double2>() + eb, size_t(ee - eb) * 16);
  }
  float ms = 0.f;
  CU_TRY(c, cudaEventElapsedTime(&ms, c->ev_start, c->ev_end));
  if (c->trace && c->overlapped)
    std::fprintf(stderr, "[fmmcu] device span %8.3f ms, host prep %8.3f ms, finish returns at %8.3f ms\n",
                 ms, 1e3 * c->prep_seconds,
                 std::chrono::duration<double, std::milli>(Clock::now() - c->t_evstart).count());
  if (c->trace && !c->overlapped) {
    float kms = 0.f;
    cudaEventElapsedTime(&kms, c->ev_start, c->ev_kslice[c->n_slices - 1]);
    std::fprintf(stderr, "[fmmcu] device span %8.3f ms (start->last kernel %8.3f ms), prep %8.3f ms\n",
                 ms, kms, 1e3 * c->prep_seconds);
  }
  const uint64_t hits = *c->h_hits.as<unsigned long long>();
  if (pair_evals) *pair_evals = c->run_total_pairs - hits;
  if (seconds) *seconds = c->prep_seconds + 1e-3 * double(ms);
  return FMMCU_OK;
}

/* Page-lock caller memory so fmmcu_p2p_launch can DMA straight into it. */
int fmmcu_host_register(fmmcu_ctx* c, void* ptr, uint64_t bytes) {
  if (!c || !ptr || !bytes) return FMMCU_EINVAL;
  CU_TRY(c, cudaSetDevice(c->device));
  CU_TRY(c, cudaHostRegister(ptr, size_t(bytes), cudaHostRegisterPortable | cudaHostRegisterMapped));
  return FMMCU_OK;
}

int fmmcu_pin_host(void* ptr, uint64_t bytes) {
  if (!ptr || !bytes) return FMMCU_EINVAL;
  const cudaError_t e =
      cudaHostRegister(ptr, size_t(bytes), cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? FMMCU_ENOMEM : FMMCU_ECUDA;
  }
  return FMMCU_OK;
}

int fmmcu_unpin_host(void* ptr) {
  if (!ptr) return FMMCU_EINVAL;
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return FMMCU_ECUDA;
  }
  return FMMCU_OK;
}

int fmmcu_host_unregister(fmmcu_ctx* c, void* ptr) {
  if (!c || !ptr) return FMMCU_EINVAL;
  CU_TRY(c, cudaSetDevice(c->device));
  CU_TRY(c, cudaHostUnregister(ptr));
  return FMMCU_OK;
}

int fmmcu_p2p_stage(fmmcu_ctx* c, const fmmcu_p2p_job* j) {
  if (!c) return FMMCU_EINVAL;
  if (c->inflight) return set_err(c, FMMCU_ESTATE, "stage while a job is in flight");
  if (int rc = stage_job(c, j)) return rc;
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return FMMCU_OK;
}

int fmmcu_p2p_run_staged(fmmcu_ctx* c, uint32_t lb, uint32_t le, int mode, int* launches) {
  if (!c) return FMMCU_EINVAL;
  if (!c->staged || c->grouped) return set_err(c, FMMCU_ESTATE, "no staged job (fmmcu_p2p_stage)");
  if (lb > le || le > c->n_leaves) return set_err(c, FMMCU_EINVAL, "bad leaf shard");
  if (mode < 0 || mode > 1) return set_err(c, FMMCU_EINVAL, "unknown mode");
  CU_TRY(c, cudaSetDevice(c->device));
  c->run_lb = lb;
  c->run_le = le;
  c->run_total_pairs = c->leaf_work[le] - c->leaf_work[lb];
  return run_kernels(c, lb, le, mode, launches);
}

int fmmcu_p2p_device_out(fmmcu_ctx* c, double** dptr) {
  if (!c || !dptr) return FMMCU_EINVAL;
  if (!c->staged) return set_err(c, FMMCU_ESTATE, "no staged job");
  *dptr = reinterpret_cast<double*>(c->out_ptr());
  return FMMCU_OK;
}

int fmmcu_p2p_bind_device_out(fmmcu_ctx* c, double* dptr) {
  if (!c) return FMMCU_EINVAL;
  c->ext_out = reinterpret_cast<double2*>(dptr);
  return FMMCU_OK;
}

int fmmcu_p2p_copy_out(fmmcu_ctx* c, double* host, uint32_t eb, uint32_t ee) {
  if (!c || (!host && ee > eb)) return FMMCU_EINVAL;
  if (!c->staged) return set_err(c, FMMCU_ESTATE, "no staged job");
  if (eb > ee || ee > c->n_eval) return set_err(c, FMMCU_EINVAL, "bad eval range");
  CU_TRY(c, cudaSetDevice(c->device));
  if (ee > eb)
    CU_TRY(c, cudaMemcpyAsync(host + 2 * size_t(eb), c->out_ptr() + eb, size_t(ee - eb) * 16,
                              cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  return FMMCU_OK;
}

int fmmcu_p2p_pairs(fmmcu_ctx* c, uint64_t* pairs) {
  if (!c || !pairs) return FMMCU_EINVAL;
  if (!c->staged) return set_err(c, FMMCU_ESTATE, "no staged job");
  CU_TRY(c, cudaSetDevice(c->device));
  unsigned long long h = 0;
  CU_TRY(c, cudaMemcpyAsync(&h, c->d_hits.p, 8, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(c, cudaStreamSynchronize(c->stream));
  *pairs = c->run_total_pairs - h;
  return FMMCU_OK;
}

int fmmcu_p2p_work_prefix(fmmcu_ctx* c, uint64_t* prefix) {
  if (!c || !prefix) return FMMCU_EINVAL;
  if (!c->staged) return set_err(c, FMMCU_ESTATE, "no staged job");
  std::memcpy(prefix, c->leaf_work.data(), sizeof(uint64_t) * c->leaf_work.size());
  return FMMCU_OK;
}

int fmmcu_p2p_kernel_info(const fmmcu_ctx* c, int* symmetric, int* evals_per_lane) {
  if (!c) return FMMCU_EINVAL;
  if (symmetric) *symmetric = c->sym_items ? 1 : 0;
  if (evals_per_lane) *evals_per_lane = c->warp_e;
  return FMMCU_OK;
}

int fmmcu_fp64_peak(fmmcu_ctx* c, double* tflops) {
  if (!c || !tflops) return FMMCU_EINVAL;
  CU_TRY(c, cudaSetDevice(c->device));
  int sms = 0;
  CU_TRY(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  DevBuf sink;
  CU_TRY(c, sink.ensure(64));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  CU_TRY(c, cudaEventCreate(&e0));
  CU_TRY(c, cudaEventCreate(&e1));
  dfma_peak_kernel<<<blocks, threads, 0, c->stream>>>(sink.as<double>(), 64, 1.0);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    CU_TRY(c, cudaEventRecord(e0, c->stream));
    dfma_peak_kernel<<<blocks, threads, 0, c->stream>>>(sink.as<double>(), iters, 1.0);
    CU_TRY(c, cudaEventRecord(e1, c->stream));
    CU_TRY(c, cudaEventSynchronize(e1));
    float ms = 0;
    CU_TRY(c, cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  CU_TRY(c, cudaGetLastError());
  c->launches += 4;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  sink.release();
  const double flops = double(blocks) * threads * iters * 16.0 * 8.0 * 2.0;
  *tflops = flops / (best * 1e-3) / 1e12;
  return FMMCU_OK;
}

// ------------------------------------------------------------------- M2L --
int fmmcu_m2l_launch(fmmcu_ctx* c, const fmmcu_m2l_job* j) {
  if (!c) return FMMCU_EINVAL;
  if (c->m2l_inflight) return set_err(c, FMMCU_ESTATE, "m2l launch while in flight");
  if (!j) return set_err(c, FMMCU_EINVAL, "null m2l job");
  if (j->p < 1 || j->p > kM2LMaxP) return set_err(c, FMMCU_EINVAL, "m2l order out of range");
  if (j->kernel < 0 || j->kernel > 1) return set_err(c, FMMCU_EINVAL, "unknown kernel");
  const auto t0 = Clock::now();
  CU_TRY(c, cudaSetDevice(c->device));
  const int P1 = j->p + 1;
  const uint32_t nb = j->n_boxes, nt = j->n_targets;
  const uint32_t nnz = nt ? j->weak_off[nt] : 0;
  // branch-free (vectorised) checks
  uint32_t bad_t = 0, top_w = 0;
#pragma omp parallel for schedule(static) reduction(| : bad_t)
  for (int64_t t = 0; t < int64_t(nt); ++t)
    bad_t |= uint32_t(j->target_box[t] >= nb) | uint32_t(j->weak_off[t] > j->weak_off[t + 1]);
  if (bad_t) return set_err(c, FMMCU_EINVAL, "bad m2l target list");
#pragma omp parallel for schedule(static) reduction(max : top_w)
  for (int64_t q = 0; q < int64_t(nnz); ++q) top_w = std::max(top_w, j->weak_idx[q]);
  if (nnz && top_w >= nb) return set_err(c, FMMCU_EINVAL, "bad m2l weak index");
  CU_TRY(c, c->m_centers.ensure(size_t(nb) * 16));
  CU_TRY(c, c->m_coeffs.ensure(size_t(nb) * P1 * 16));
  CU_TRY(c, c->m_tbox.ensure(size_t(nt) * 4));
  CU_TRY(c, c->m_woff.ensure(size_t(nt + 1) * 4));
  CU_TRY(c, c->m_widx.ensure(size_t(nnz) * 4));
  CU_TRY(c, c->m_out.ensure(size_t(nt) * P1 * 16));
  CU_TRY(c, c->m_flag.ensure(8));
  CU_TRY(c, c->mh_flag.ensure(8));
  // out == NULL: the sums stay on the device for fmmcu_m2l_downward
  c->m2l_keep = j->out == nullptr;
  c->m2l_direct_out = nt && !c->m2l_keep && host_locked(j->out, size_t(nt) * P1 * 16);
  if (!c->m2l_direct_out && !c->m2l_keep) CU_TRY(c, c->mh_out.ensure(size_t(nt) * P1 * 16));
  cudaStream_t s = c->m2l_stream;
  CU_TRY(c, cudaEventRecord(c->ev_m2l0, s));
  CU_TRY(c, cudaMemcpyAsync(c->m_centers.p, j->centers, size_t(nb) * 16, cudaMemcpyHostToDevice, s));
  CU_TRY(c, cudaMemcpyAsync(c->m_coeffs.p, j->coeffs, size_t(nb) * P1 * 16, cudaMemcpyHostToDevice, s));
  if (nt) {
    CU_TRY(c, cudaMemcpyAsync(c->m_tbox.p, j->target_box, size_t(nt) * 4, cudaMemcpyHostToDevice, s));
    CU_TRY(c, cudaMemcpyAsync(c->m_woff.p, j->weak_off, size_t(nt + 1) * 4, cudaMemcpyHostToDevice, s));
  }
  if (nnz) CU_TRY(c, cudaMemcpyAsync(c->m_widx.p, j->weak_idx, size_t(nnz) * 4, cudaMemcpyHostToDevice, s));
  CU_TRY(c, cudaMemsetAsync(c->m_flag.p, 0, 8, s));
  if (nt) {
    M2LArgs a{};
    a.p = j->p;
    a.kernel = j->kernel;
    a.centers = c->m_centers.as<double2>();
    a.coeffs = c->m_coeffs.as<double2>();
    a.target_box = c->m_tbox.as<uint32_t>();
    a.weak_off = c->m_woff.as<uint32_t>();
    a.weak_idx = c->m_widx.as<uint32_t>();
    a.n_targets = nt;
    a.out = c->m_out.as<double2>();
    a.singular = c->m_flag.as<int>();
    if (int rc = m2l_run(c, a, nnz, s)) return rc;
    if (!c->m2l_keep)
      CU_TRY(c, cudaMemcpyAsync(c->m2l_direct_out ? static_cast<void*>(j->out) : c->mh_out.p,
                                c->m_out.p, size_t(nt) * P1 * 16, cudaMemcpyDeviceToHost, s));
  }
  CU_TRY(c, cudaMemcpyAsync(c->mh_flag.p, c->m_flag.p, 4, cudaMemcpyDeviceToHost, s));
  CU_TRY(c, cudaEventRecord(c->ev_m2l1, s));
  c->m2l_job = *j;
  c->m2l_ops = nnz;
  c->m2l_prep = std::chrono::duration<double>(Clock::now() - t0).count();
  c->m2l_inflight = true;
  return FMMCU_OK;
}

int fmmcu_m2l_host_buffers(fmmcu_ctx* c, uint32_t n_boxes, int p, uint32_t n_targets,
                           uint64_t nnz, fmmcu_m2l_buffers* b) {
  if (!c || !b) return FMMCU_EINVAL;
  if (p < 1 || p > kM2LMaxP) return set_err(c, FMMCU_EINVAL, "m2l order out of range");
  if (c->m2l_inflight) return set_err(c, FMMCU_ESTATE, "m2l buffers while a launch is in flight");
  CU_TRY(c, cudaSetDevice(c->device));
  const size_t P1 = size_t(p) + 1;
  CU_TRY(c, c->mb_centers.ensure(size_t(n_boxes) * 16));
  CU_TRY(c, c->mb_coeffs.ensure(size_t(n_boxes) * P1 * 16));
  CU_TRY(c, c->mb_out.ensure(size_t(n_targets) * P1 * 16));
  CU_TRY(c, c->mb_tbox.ensure(size_t(n_targets) * 4));
  CU_TRY(c, c->mb_woff.ensure((size_t(n_targets) + 1) * 4));
  CU_TRY(c, c->mb_widx.ensure(size_t(nnz) * 4));
  b->centers = c->mb_centers.as<double>();
  b->coeffs = c->mb_coeffs.as<double>();
  b->out = c->mb_out.as<double>();
  b->target_box = c->mb_tbox.as<uint32_t>();
  b->weak_off = c->mb_woff.as<uint32_t>();
  b->weak_idx = c->mb_widx.as<uint32_t>();
  return FMMCU_OK;
}

int fmmcu_m2l_finish(fmmcu_ctx* c, uint64_t* ops, double* seconds) {
  if (!c) return FMMCU_EINVAL;
  if (!c->m2l_inflight) return set_err(c, FMMCU_ESTATE, "m2l finish without launch");
  c->m2l_inflight = false;
  CU_TRY(c, cudaSetDevice(c->device));
  CU_TRY(c, wait_event(c->ev_m2l1));
  CU_TRY(c, cudaGetLastError());
  float ms = 0.f;
  CU_TRY(c, cudaEventElapsedTime(&ms, c->ev_m2l0, c->ev_m2l1));
  const int P1 = c->m2l_job.p + 1;
  if (c->m2l_job.n_targets && !c->m2l_direct_out && !c->m2l_keep)
    par_memcpy(c->m2l_job.out, c->mh_out.p, size_t(c->m2l_job.n_targets) * P1 * 16);
  if (ops) *ops = c->m2l_ops;
  if (seconds) *seconds = c->m2l_prep + 1e-3 * double(ms);
  if (*c->mh_flag.as<int>())
    return set_err(c, FMMCU_ESINGULAR, "m2l: target center coincides with source center");
  return FMMCU_OK;
}

}  // extern "C"
