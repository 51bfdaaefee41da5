// fmm-b200 — P2P near-field kernels for sm_100a.
//
// Device restatement of the reference near-field loop near_box()
// (proj/src/backend.cpp:41-69) with the per-pair arithmetic of
// kernel_term()/smoother_factor() (proj/src/expansion.cpp:78-92).
//
// Fast path (p2p_tile_kernel), FP64 CUDA-core pipe, no tensor cores:
//   * persistent CTAs pull work items (a target leaf, or an eval block /
//     strong-list chunk of a heavy leaf) from a global counter;
//   * an item's source leaves are contiguous runs of packed 32-byte records
//     {x, y, m_re, m_im}; warp 0 builds the run list of the next tile with
//     one coalesced load + shuffle scan over the precomputed (begin, length)
//     of each strong entry and issues one TMA bulk copy
//     (cp.async.bulk + mbarrier complete_tx) per run into the other of two
//     shared tiles -- the next tile streams in while this one is computed;
//   * thread (g, k) owns E evals of eval-slot g and walks sources
//     k, k+K, k+2K, ... of the tile (broadcast LDS.128); the K partials of
//     an eval are reduced in fixed k order through shared memory, so results
//     are deterministic;
//   * per pair: 2 DADD, r^2 (DMUL+DFMA), 1/r^2 = MUFU.RCP64H seed + one
//     cubic Newton step (3 DFMA), m*conj(d) (2 DMUL + 2 DFMA), 2 DFMA
//     accumulate -- 13 FP64 instructions for 23 algorithmic flops.
// Exact path (p2p_exact_kernel): one thread per eval, reference order,
// libgcc __divdc3 restated with non-contracted __d*_rn intrinsics -- bitwise
// equal to the reference for the harmonic kernel without smoother.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fmmcu {

constexpr uint32_t kNoSelf = 0xFFFFFFFFu;

// Work item: evals [ev_begin, ev_begin + nt) of target leaf `leaf` against
// strong entries [s_begin, s_end) of its list.
struct P2PItem {
  uint32_t leaf;
  uint32_t ev_begin;
  uint32_t nt;
  uint32_t s_begin;
  uint32_t s_end;
  uint32_t n_src;        // sources covered by this item
  uint32_t partial_off;  // kNoSelf: write out[] directly; else base (in evals) into partial[]
  uint32_t pad;
};

struct P2PArgs {
  const double4* __restrict__ src;     // packed sources, permuted order
  const double2* __restrict__ evy;     // eval positions, permuted order
  const double4* __restrict__ evr;     // eval records {x, y, self bits, 0} (fast path)
  const uint32_t* __restrict__ eself;  // permuted slot of the eval's own source, or kNoSelf
  const uint32_t* __restrict__ pt_off;
  const uint32_t* __restrict__ ev_off;
  const uint32_t* __restrict__ s_off;
  const uint32_t* __restrict__ s_idx;
  const uint2* __restrict__ seg;       // per strong entry: (pt_off[s], n_points(s))
  const P2PItem* __restrict__ items;
  uint32_t n_items;
  unsigned int* __restrict__ next_item;  // dynamic scheduler counter (zeroed per launch)
  double2* __restrict__ out;
  double2* __restrict__ partial;
  unsigned long long* __restrict__ hits;  // self pairs skipped (pair count correction)
  double delta;       // smoother radius
  double delta2;      // delta^2
  double inv_delta2;  // 1/delta^2
};

// ---------------------------------------------------------------- helpers --
__device__ __forceinline__ double rcp_fast(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // cubic Newton-Raphson: y(1 + e + e^2), e = 1 - x*y  (error ~ e^3)
  const double e = fma(-x, y, 1.0);
  const double q = fma(e, e, e);
  return fma(y, q, y);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA 1-D bulk copy global -> shared, completion signalled on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA 1-D bulk copy shared -> global (bulk async-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile(
      "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
      "cp.async.bulk.commit_group;\n" ::"l"(dst),
      "r"(smem_u32(src)), "r"(bytes)
      : "memory");
}

// wait until every committed bulk store has finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// wait until every committed bulk store has completed
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Per-pair contribution accumulated with the sign folded out:
//   harmonic: acc += m * conj(d) / |d|^2     (term = -acc)
//   log     : acc += m * log(d)              (term = +acc)
// The smoother multiplies the term; g == 0 contributes nothing (backend.cpp:61-63).
template <int KERNEL, int SMOOTH>
__device__ __forceinline__ void pair_accum(double yx, double yy, const double4 s, double inv_d2,
                                           double d2, bool live, double& ar, double& ai) {
  const double dx = yx - s.x;
  const double dy = yy - s.y;
  const double r2 = fma(dx, dx, dy * dy);
  if (KERNEL == 0) {
    double inv = rcp_fast(r2);
    if (SMOOTH == 1) {
      const double g = 1.0 - exp(-r2 * inv_d2);
      inv = (g == 0.0) ? 0.0 : inv * g;
    } else if (SMOOTH == 2) {
      const double g = sqrt(r2 / (d2 + r2));
      inv = (g == 0.0) ? 0.0 : inv * g;
    }
    inv = live ? inv : 0.0;
    const double tr = fma(s.z, dx, s.w * dy);   // Re(m conj d)
    const double ti = fma(s.w, dx, -s.z * dy);  // Im(m conj d)
    ar = fma(tr, inv, ar);
    ai = fma(ti, inv, ai);
  } else {
    // log(d) = 0.5 log r^2 + i atan2(dy, dx)
    double L = 0.5 * log(r2);
    double T = atan2(dy, dx);
    double g = 1.0;
    if (SMOOTH == 1) g = 1.0 - exp(-r2 * inv_d2);
    if (SMOOTH == 2) g = sqrt(r2 / (d2 + r2));
    const bool use = live && (g != 0.0);
    L = use ? L * g : 0.0;
    T = use ? T * g : 0.0;
    ar = fma(s.z, L, fma(-s.w, T, ar));
    ai = fma(s.z, T, fma(s.w, L, ai));
  }
}

// Sources p, p+K, p+2K, ... < end without the self test: blocks of U
// independent sources with no branch inside a block (so the compiler
// interleaves the U*E pair chains), then a tail.  Per eval the accumulation
// order is still ascending in the source position.
template <int KERNEL, int SMOOTH, int E, int U>
__device__ __forceinline__ const double4* run_unchecked(const double4* p, const double4* end,
                                                        uint32_t K, const double* yx,
                                                        const double* yy, double inv_d2, double d2,
                                                        double* ar, double* ai) {
  const ptrdiff_t step = ptrdiff_t(K);
  while (p + (U - 1) * step < end) {
    double4 s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = p[u * step];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < E; ++e)
        pair_accum<KERNEL, SMOOTH>(yx[e], yy[e], s[u], inv_d2, d2, true, ar[e], ai[e]);
    p += U * step;
  }
  for (; p < end; p += step) {
    const double4 s = *p;
#pragma unroll
    for (int e = 0; e < E; ++e)
      pair_accum<KERNEL, SMOOTH>(yx[e], yy[e], s, inv_d2, d2, true, ar[e], ai[e]);
  }
  return p;
}

// seg[q] = (first permuted source slot, source count) of strong entry q.
static __global__ void p2p_segments_kernel(const uint32_t* __restrict__ s_idx,
                                    const uint32_t* __restrict__ pt_off, uint32_t nnz,
                                    uint2* __restrict__ seg) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nnz) {
    const uint32_t b = s_idx[q];
    const uint32_t p0 = pt_off[b];
    seg[q] = make_uint2(p0, pt_off[b + 1] - p0);
  }
}

constexpr int kMaxSeg = 128;  // source runs per tile

// ------------------------------------------------------------ fast kernel --
// Eval record as staged on the device: {x, y, self slot (bits), q_self (bits)}
// where q_self is the global strong-entry index (position in strong_idx) of
// the eval's own leaf's entry whose source run holds the self slot, or
// kNoSelf -- this makes the per-tile self lookup O(1).
__device__ __forceinline__ uint32_t find_self_entry(const P2PArgs& a, uint32_t leaf,
                                                    uint32_t self) {
  if (self == kNoSelf) return kNoSelf;
  for (uint32_t q = a.s_off[leaf]; q < a.s_off[leaf + 1]; ++q) {
    const uint2 sg = a.seg[q];
    if (self - sg.x < sg.y) return q;
  }
  return kNoSelf;
}

// One warp per leaf of [leaf_begin, leaf_end), lanes over its evals.
static __global__ void p2p_evrec_kernel(const P2PArgs a, uint32_t leaf_begin, uint32_t leaf_end,
                                        double4* __restrict__ evr) {
  const uint32_t leaf = leaf_begin + blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (leaf >= leaf_end) return;
  for (uint32_t e = a.ev_off[leaf] + (threadIdx.x & 31); e < a.ev_off[leaf + 1]; e += 32) {
    const double2 y = a.evy[e];
    const uint32_t self = a.eself[e];
    const uint32_t q = find_self_entry(a, leaf, self);
    evr[e] = make_double4(y.x, y.y, __longlong_as_double((long long)self),
                          __longlong_as_double((long long)q));
  }
}

// Self layout (eval e == source slot e): derive the eval arrays from the
// already uploaded sources instead of uploading them.
static __global__ void p2p_self_evals_kernel(const double4* __restrict__ src, uint32_t i0,
                                             uint32_t i1, double2* __restrict__ evy,
                                             uint32_t* __restrict__ eself) {
  const uint32_t i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < i1) {
    const double4 s = src[i];
    evy[i] = make_double2(s.x, s.y);
    eself[i] = i;
  }
}

// Dynamic smem: [2 mbarriers | pad to 128][src tile 0][src tile 1]
//               [eval tile 0][eval tile 1][reduction 0][reduction 1]
template <int KERNEL, int SMOOTH, int E, int THREADS, int TILE, int MAXEV, int U, bool PRODUCER,
          int MINB>
__global__ void __launch_bounds__(THREADS, MINB) p2p_tile_kernel(const P2PArgs a) {
  // PRODUCER: warp 0 only stages tiles; otherwise warp 0 stages and computes.
  constexpr int TC = PRODUCER ? THREADS - 32 : THREADS;  // consumer threads
  static_assert(TILE % 32 == 0 && MAXEV <= TC * E, "shape");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double4* tiles = reinterpret_cast<double4*>(smem_raw + 128);
  double4* evt = tiles + 2 * TILE;
  double2* red = reinterpret_cast<double2*>(evt + 2 * MAXEV);
  // run r of a tile = strong entry q0 + r (runs are 1:1 with entries,
  // empty leaves give empty runs)
  __shared__ uint32_t seg_gbeg[2][kMaxSeg];
  __shared__ uint32_t seg_tpos[2][kMaxSeg + 1];
  __shared__ uint32_t meta_item[2], meta_nseg[2], meta_flags[2], meta_ev[2], meta_nt[2],
      meta_poff[2], meta_q0[2];
  __shared__ unsigned int s_hits;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  constexpr unsigned FULL = 0xffffffffu;

  // ---- producer state (warp 0, warp-uniform registers) ----------------------
  uint32_t st_item = kNoSelf, st_ent = 0, st_off = 0, st_end = 0, st_left = 0;
  uint32_t st_ev = 0, st_nt = 0, st_poff = kNoSelf;
  // lane 0 of warp 0 claims the next item id one item ahead, so the atomic's
  // latency is hidden behind a whole item of compute
  uint32_t claim = 0;
  if (tid == 0) claim = atomicAdd(a.next_item, 1u);

  auto stage = [&](int b) {
    uint32_t flags = 0;
    if (st_left == 0) {  // current item exhausted: take the claimed one, claim another
      const uint32_t nxt = __shfl_sync(FULL, claim, 0);
      if (nxt >= a.n_items) {
        if (lane == 0) meta_item[b] = kNoSelf;
        return;
      }
      if (lane == 0) claim = atomicAdd(a.next_item, 1u);
      const P2PItem it = a.items[nxt];
      st_item = nxt;
      st_ent = it.s_begin;
      st_end = it.s_end;
      st_off = 0;
      st_left = it.n_src;
      st_ev = it.ev_begin;
      st_nt = it.nt;
      st_poff = it.partial_off;
      flags |= 1u;
    }
    const uint32_t q0 = st_ent;
    uint32_t filled = 0, nseg = 0;
    while (filled < TILE && st_ent < st_end && nseg + 32 <= kMaxSeg) {
      const uint32_t q = st_ent + lane;
      const bool valid = q < st_end;
      const uint2 sg = valid ? a.seg[q] : make_uint2(0u, 0u);
      uint32_t b0 = sg.x, n = sg.y;
      if (lane == 0) {
        b0 += st_off;
        n -= st_off;
      }
      uint32_t incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t excl = incl - n;
      const uint32_t room = TILE - filled;
      const bool in = valid && excl < room;  // a prefix of the lanes
      const uint32_t take = in ? min(n, room - excl) : 0u;
      if (in) {
        seg_gbeg[b][nseg + lane] = b0;
        seg_tpos[b][nseg + lane] = filled + excl;
      }
      const unsigned part = __ballot_sync(FULL, valid && take < n);
      const uint32_t n_in = __popc(__ballot_sync(FULL, in));
      const uint32_t total = __shfl_sync(FULL, incl, 31);
      const uint32_t got = min(total, room);
      if (part == 0) {
        st_ent += min(32u, st_end - st_ent);
        st_off = 0;
      } else {
        const int L = __ffs(part) - 1;
        const uint32_t tL = __shfl_sync(FULL, take, L);
        st_off = (L == 0 ? st_off : 0u) + tL;
        st_ent += uint32_t(L);
      }
      filled += got;
      nseg += n_in;
      st_left -= got;
    }
    if (st_left == 0) flags |= 2u;
    const uint32_t ev_bytes = (flags & 1u) ? st_nt * 32u : 0u;
    if (lane == 0) {
      seg_tpos[b][nseg] = filled;
      meta_item[b] = st_item;
      meta_nseg[b] = nseg;
      meta_flags[b] = flags;
      meta_ev[b] = st_ev;
      meta_nt[b] = st_nt;
      meta_poff[b] = st_poff;
      meta_q0[b] = q0;
      fence_proxy_async();
      mbar_expect_tx(&bar[b], filled * 32u + ev_bytes);
      if (ev_bytes) bulk_g2s(evt + b * MAXEV, a.evr + st_ev, ev_bytes, &bar[b]);
    }
    __syncwarp();
    for (uint32_t s = lane; s < nseg; s += 32) {
      const uint32_t t0 = seg_tpos[b][s];
      const uint32_t t1 = seg_tpos[b][s + 1];
      if (t1 > t0)
        bulk_g2s(tiles + b * TILE + t0, a.src + seg_gbeg[b][s], (t1 - t0) * 32u, &bar[b]);
    }
  };

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    s_hits = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) stage(0);
  __syncthreads();

  // ---- consumer state ---------------------------------------------------------
  uint32_t parity[2] = {0u, 0u};
  uint32_t nt = 0, G = 1, K = 1, g = 0, k = 0, ev0 = 0, poff = kNoSelf;
  bool active = false;
  double yx[E], yy[E], ar[E], ai[E];
  uint32_t sg[E], sq[E];
  unsigned int hits = 0;
  // pending reduction of the previous item (deferred by one tile: no extra
  // barrier), done by the highest warps (warp 0 also stages)
  uint32_t r_nt = 0, r_G = 1, r_K = 1, r_ev0 = 0, r_poff = kNoSelf, r_buf = 0, items_done = 0;
  bool r_pending = false;

  const int ctid = PRODUCER ? tid - 32 : tid;  // consumer index (< 0: producer warp)
  auto reduce_pending = [&]() {
    const double2* rb = red + r_buf * (TC * E);
    const int rt = THREADS - 1 - tid;  // highest threads first
    for (uint32_t le = uint32_t(rt); le < r_nt; le += THREADS) {
      const uint32_t gg = le / E, ee = le % E;
      const double2* p = rb + ee * r_K * r_G + gg;
      double sr = 0.0, si = 0.0;
      for (uint32_t kk = 0; kk < r_K; ++kk, p += r_G) {
        const double2 v = *p;
        sr += v.x;
        si += v.y;
      }
      const double2 res = (KERNEL == 0) ? make_double2(-sr, -si) : make_double2(sr, si);
      if (r_poff == kNoSelf)
        a.out[r_ev0 + le] = res;
      else
        a.partial[r_poff + le] = res;
    }
    r_pending = false;
  };

  for (uint32_t n = 0;; ++n) {
    const int b = int(n & 1u);
    const uint32_t item = meta_item[b];
    if (item == kNoSelf) break;
    const uint32_t flags = meta_flags[b];
    const uint32_t nseg = meta_nseg[b];
    const uint32_t q0 = meta_q0[b];
    if (flags & 1u) {  // first tile of an item: thread roles (no integer division)
      nt = meta_nt[b];
      ev0 = meta_ev[b];
      poff = meta_poff[b];
      G = (nt + E - 1) / E;  // E is a power of two; host guarantees nt <= MAXEV <= E * TC
      const float rG = 1.0f / float(G);
      K = uint32_t(float(TC) * rG + 1e-4f);
      k = uint32_t((float(ctid) + 0.5f) * rG);
      g = uint32_t(ctid) - k * G;
      active = ctid >= 0 && k < K;
    }
    if (warp == 0) stage(b ^ 1);  // next tile streams in while this one is computed
    if (r_pending) reduce_pending();

    mbar_wait(&bar[b], parity[b]);
    parity[b] ^= 1u;
    if (flags & 1u) {  // eval registers from the staged eval records
      const double4* ev = evt + b * MAXEV;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t le = g * E + e;
        const bool ok = active && le < nt;
        const double4 r = ok ? ev[le] : make_double4(0.0, 0.0, 0.0, 0.0);
        yx[e] = r.x;
        yy[e] = r.y;
        sg[e] = ok ? uint32_t(__double_as_longlong(r.z)) : kNoSelf;
        sq[e] = ok ? uint32_t(__double_as_longlong(r.w)) : kNoSelf;
        ar[e] = 0.0;
        ai[e] = 0.0;
      }
    }

    // O(1) tile position of each eval's own source: its entry's run r = q - q0
    const uint32_t ntile = seg_tpos[b][nseg];
    uint32_t ps[E];
    uint32_t plo = kNoSelf, phi = 0u;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      ps[e] = kNoSelf;
      const uint32_t r = sq[e] - q0;
      if (sq[e] != kNoSelf && r < nseg) {
        const uint32_t d = sg[e] - seg_gbeg[b][r];
        const uint32_t t0 = seg_tpos[b][r];
        if (d < seg_tpos[b][r + 1] - t0) {
          ps[e] = t0 + d;
          plo = min(plo, ps[e]);
          phi = max(phi, ps[e]);
        }
      }
    }
    // Self pairs of this warp sit at tile positions [plo, phi] (the target
    // leaf's own run for self-evaluation): only that stretch pays for the
    // per-pair exclusion test.
    plo = __reduce_min_sync(FULL, plo);
    phi = __reduce_max_sync(FULL, phi);

    if (active) {
      const double4* tile = tiles + b * TILE;
      const double4* p = tile + k;
      const double4* const end1 = tile + min(plo, ntile);
      const double4* const end = tile + ntile;
      p = run_unchecked<KERNEL, SMOOTH, E, U>(p, end1, K, yx, yy, a.inv_delta2, a.delta2, ar, ai);
      if (plo != kNoSelf) {
        const double4* const end2 = tile + min(phi + 1u, ntile);
        for (; p < end2; p += K) {
          const double4 s = *p;
          const uint32_t j = uint32_t(p - tile);
#pragma unroll
          for (int e = 0; e < E; ++e)
            pair_accum<KERNEL, SMOOTH>(yx[e], yy[e], s, a.inv_delta2, a.delta2, j != ps[e], ar[e],
                                       ai[e]);
        }
        run_unchecked<KERNEL, SMOOTH, E, U>(p, end, K, yx, yy, a.inv_delta2, a.delta2, ar, ai);
        // each skipped self pair is seen by exactly one source lane
#pragma unroll
        for (int e = 0; e < E; ++e) hits += (ps[e] != kNoSelf && ps[e] % K == k) ? 1u : 0u;
      }
    }

    if (flags & 2u) {  // last tile of the item: park the K partials, reduce next tile
      const uint32_t rb = items_done & 1u;
      if (active) {
#pragma unroll
        for (int e = 0; e < E; ++e)
          red[rb * (TC * E) + (e * K + k) * G + g] = make_double2(ar[e], ai[e]);
      }
      r_pending = true;
      r_nt = nt;
      r_G = G;
      r_K = K;
      r_ev0 = ev0;
      r_poff = poff;
      r_buf = rb;
      ++items_done;
    }
    __syncthreads();  // tile b free, partials visible, meta[b^1] visible
  }
  if (r_pending) reduce_pending();
  for (int o = 16; o > 0; o >>= 1) hits += __shfl_down_sync(FULL, hits, o);
  if (lane == 0 && hits) atomicAdd(&s_hits, hits);
  __syncthreads();
  if (tid == 0 && s_hits) atomicAdd(a.hits, (unsigned long long)s_hits);
}

// Sum the chunk partials of split eval blocks in chunk order (deterministic).
struct P2PFinal {
  uint32_t ev_begin;
  uint32_t nt;
  uint32_t base;
  uint32_t n_chunks;
};

static __global__ void p2p_finalize_kernel(const P2PFinal* __restrict__ fin, uint32_t n_fin,
                                    const double2* __restrict__ partial,
                                    double2* __restrict__ out) {
  const uint32_t f = blockIdx.x;
  if (f >= n_fin) return;
  const P2PFinal F = fin[f];
  for (uint32_t e = threadIdx.x; e < F.nt; e += blockDim.x) {
    double sr = 0.0, si = 0.0;
    for (uint32_t c = 0; c < F.n_chunks; ++c) {
      const double2 v = partial[F.base + c * F.nt + e];
      sr += v.x;
      si += v.y;
    }
    out[F.ev_begin + e] = make_double2(sr, si);
  }
}

// ----------------------------------------------------------- exact kernel --
// libgcc __divdc3 (GCC >= 12) with every operation rounded separately.
__device__ __forceinline__ void divdc3_rn(double a, double b, double c, double d, double& xo,
                                          double& yo) {
  const double RBIG = 8.98846567431157953865e+307;  // DBL_MAX / 2
  const double RMIN = 2.2250738585072014e-308;      // DBL_MIN
  const double RMIN2 = 2.220446049250313080847e-16; // DBL_EPSILON
  const double RMINSCAL = 4503599627370496.0;       // 1 / DBL_EPSILON
  const double RMAX2 = 1.99584030953471981166e+292; // RBIG * RMIN2
  double denom, ratio, x, y;
  if (fabs(c) < fabs(d)) {
    if (fabs(d) >= RBIG) {
      a = __dmul_rn(a, 0.5); b = __dmul_rn(b, 0.5); c = __dmul_rn(c, 0.5); d = __dmul_rn(d, 0.5);
    }
    if (fabs(d) < RMIN2) {
      a = __dmul_rn(a, RMINSCAL); b = __dmul_rn(b, RMINSCAL);
      c = __dmul_rn(c, RMINSCAL); d = __dmul_rn(d, RMINSCAL);
    } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(d) < RMAX2)) ||
               ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(d) < RMAX2))) {
      a = __dmul_rn(a, RMINSCAL); b = __dmul_rn(b, RMINSCAL);
      c = __dmul_rn(c, RMINSCAL); d = __dmul_rn(d, RMINSCAL);
    }
    ratio = __ddiv_rn(c, d);
    denom = __dadd_rn(__dmul_rn(c, ratio), d);
    if (fabs(ratio) > RMIN) {
      x = __ddiv_rn(__dadd_rn(__dmul_rn(a, ratio), b), denom);
      y = __ddiv_rn(__dsub_rn(__dmul_rn(b, ratio), a), denom);
    } else {
      x = __ddiv_rn(__dadd_rn(__dmul_rn(c, __ddiv_rn(a, d)), b), denom);
      y = __ddiv_rn(__dsub_rn(__dmul_rn(c, __ddiv_rn(b, d)), a), denom);
    }
  } else {
    if (fabs(c) >= RBIG) {
      a = __dmul_rn(a, 0.5); b = __dmul_rn(b, 0.5); c = __dmul_rn(c, 0.5); d = __dmul_rn(d, 0.5);
    }
    if (fabs(c) < RMIN2) {
      a = __dmul_rn(a, RMINSCAL); b = __dmul_rn(b, RMINSCAL);
      c = __dmul_rn(c, RMINSCAL); d = __dmul_rn(d, RMINSCAL);
    } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(c) < RMAX2)) ||
               ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(c) < RMAX2))) {
      a = __dmul_rn(a, RMINSCAL); b = __dmul_rn(b, RMINSCAL);
      c = __dmul_rn(c, RMINSCAL); d = __dmul_rn(d, RMINSCAL);
    }
    ratio = __ddiv_rn(d, c);
    denom = __dadd_rn(__dmul_rn(d, ratio), c);
    if (fabs(ratio) > RMIN) {
      x = __ddiv_rn(__dadd_rn(__dmul_rn(b, ratio), a), denom);
      y = __ddiv_rn(__dsub_rn(b, __dmul_rn(a, ratio)), denom);
    } else {
      x = __ddiv_rn(__dadd_rn(a, __dmul_rn(d, __ddiv_rn(b, c))), denom);
      y = __ddiv_rn(__dsub_rn(b, __dmul_rn(d, __ddiv_rn(a, c))), denom);
    }
  }
  if (isnan(x) && isnan(y)) {
    if (c == 0.0 && d == 0.0 && (!isnan(a) || !isnan(b))) {
      x = __dmul_rn(copysign(__longlong_as_double(0x7ff0000000000000LL), c), a);
      y = __dmul_rn(copysign(__longlong_as_double(0x7ff0000000000000LL), c), b);
    } else if ((isinf(a) || isinf(b)) && isfinite(c) && isfinite(d)) {
      a = copysign(isinf(a) ? 1.0 : 0.0, a);
      b = copysign(isinf(b) ? 1.0 : 0.0, b);
      const double inf = __longlong_as_double(0x7ff0000000000000LL);
      x = __dmul_rn(inf, __dadd_rn(__dmul_rn(a, c), __dmul_rn(b, d)));
      y = __dmul_rn(inf, __dsub_rn(__dmul_rn(b, c), __dmul_rn(a, d)));
    } else if ((isinf(c) || isinf(d)) && isfinite(a) && isfinite(b)) {
      c = copysign(isinf(c) ? 1.0 : 0.0, c);
      d = copysign(isinf(d) ? 1.0 : 0.0, d);
      x = __dmul_rn(0.0, __dadd_rn(__dmul_rn(a, c), __dmul_rn(b, d)));
      y = __dmul_rn(0.0, __dsub_rn(__dmul_rn(b, c), __dmul_rn(a, d)));
    }
  }
  xo = x;
  yo = y;
}

// One thread per eval of the leaf range; sources in reference order.
template <int KERNEL, int SMOOTH>
__global__ void __launch_bounds__(128)
    p2p_exact_kernel(const P2PArgs a, uint32_t leaf_begin, uint32_t leaf_end,
                     uint32_t ev_begin, uint32_t ev_end) {
  const uint32_t e = ev_begin + blockIdx.x * blockDim.x + threadIdx.x;
  unsigned int hit = 0;
  if (e < ev_end) {
    // leaf of eval e: binary search in ev_off[leaf_begin..leaf_end]
    uint32_t lo = leaf_begin, hi = leaf_end;  // invariant: ev_off[lo] <= e < ev_off[hi]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (a.ev_off[mid] <= e) lo = mid; else hi = mid;
    }
    const uint32_t leaf = lo;
    const double2 y = a.evy[e];
    const uint32_t self = a.eself[e];
    double ar = 0.0, ai = 0.0;
    for (uint32_t s = a.s_off[leaf]; s < a.s_off[leaf + 1]; ++s) {
      const uint32_t sb = a.s_idx[s];
      for (uint32_t j = a.pt_off[sb]; j < a.pt_off[sb + 1]; ++j) {
        if (j == self) {
          ++hit;
          continue;
        }
        const double4 src = a.src[j];
        const double dx = __dsub_rn(y.x, src.x), dy = __dsub_rn(y.y, src.y);
        double g = 1.0;
        if (SMOOTH != 0) {
          const double r = hypot(dx, dy);
          if (SMOOTH == 1)
            g = __dsub_rn(1.0, exp(-__ddiv_rn(__dmul_rn(r, r), __dmul_rn(a.delta, a.delta))));
          else
            g = __ddiv_rn(r, sqrt(__dadd_rn(a.delta2, __dmul_rn(r, r))));
          if (g == 0.0) continue;
        }
        double tr, ti;
        if (KERNEL == 0) {
          divdc3_rn(-src.z, -src.w, dx, dy, tr, ti);
        } else {
          const double L = log(hypot(dx, dy));
          const double T = atan2(dy, dx);
          tr = __dsub_rn(__dmul_rn(src.z, L), __dmul_rn(src.w, T));
          ti = __dadd_rn(__dmul_rn(src.z, T), __dmul_rn(src.w, L));
        }
        ar = __dadd_rn(ar, __dmul_rn(tr, g));
        ai = __dadd_rn(ai, __dmul_rn(ti, g));
      }
    }
    a.out[e] = make_double2(ar, ai);
  }
  // warp-aggregate the self-hit count
  for (int o = 16; o > 0; o >>= 1) hit += __shfl_down_sync(0xffffffffu, hit, o);
  if ((threadIdx.x & 31) == 0 && hit) atomicAdd(a.hits, (unsigned long long)hit);
}

}  // namespace fmmcu
