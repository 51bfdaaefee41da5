// fmm-b200 — warp-pipelined P2P kernel (fast FP64 path) for sm_100a.
//
// FP64 restatement of near_box() (proj/src/backend.cpp:41-69) with the
// per-pair arithmetic of p2p_kernels.cuh.  Every warp is an independent
// pipeline with no CTA-level synchronisation at all.
//   * a warp claims work items (<= 8E evals of one target leaf x <= 32
//     strong-list entries) from a global counter;
//   * lane q holds the source run (first slot, length) of strong entry q and
//     its offset in the item's virtual source stream (warp prefix scan);
//   * the stream is consumed in chunks of C records double-buffered in
//     warp-private shared memory: while chunk c is computed, the lanes issue
//     the TMA bulk copies (cp.async.bulk + per-warp mbarrier) of the runs
//     overlapping chunk c+1;
//   * lane (g, k) owns E evals of eval-slot g and strides the chunk by K
//     (broadcast LDS.128); the K partials of each eval are summed over the
//     lanes g, g+G, g+2G, ... with shuffles in fixed order (deterministic);
//   * the item's results are staged in shared memory and written with one
//     TMA bulk store (cp.async.bulk.global.shared::cta), so the output may
//     live in page-locked host memory (zero-copy over PCIe) as well as HBM.
#pragma once

#include "p2p_kernels.cuh"

namespace fmmcu {

constexpr int kWarpSlots = 8;        // eval slots per warp item: <= 8E evals, K >= 4 source lanes
constexpr int kWarpMaxEntries = 32;  // strong entries per warp item (one per lane)
// strong entries per mutual-kernel item: rounds of 32 (p2p_sym.cuh ROUNDS)
constexpr int kSymMaxEntries = 256;

constexpr size_t warp_region_bytes(int C, int E) {
  return 128 + size_t(2 * C) * 32 + size_t(kWarpSlots * E) * 16;
}

template <int KERNEL, int SMOOTH, int E, int WARPS, int C, int U, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) p2p_warp_kernel(const P2PArgs a) {
  static_assert(E >= 1 && kWarpSlots <= 32 && C % 32 == 0, "shape");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr unsigned FULL = 0xffffffffu;
  // per-warp region: [2 mbarriers | pad 128][chunk 0][chunk 1][item results]
  constexpr size_t kWarpBytes = warp_region_bytes(C, E);
  unsigned char* base = smem_raw + size_t(warp) * kWarpBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base);
  double4* buf = reinterpret_cast<double4*>(base + 128);
  double2* stage = reinterpret_cast<double2*>(base + 128 + size_t(2 * C) * 32);

  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t parity0 = 0, parity1 = 0;
  unsigned int hits = 0;

  // claim-ahead: lane 0 holds the id of the next item to run
  uint32_t claim = 0;
  if (lane == 0) claim = atomicAdd(a.next_item, 1u);

  for (;;) {
    const uint32_t id = __shfl_sync(FULL, claim, 0);
    if (id >= a.n_items) break;
    if (lane == 0) claim = atomicAdd(a.next_item, 1u);
    const P2PItem it = a.items[id];
    const uint32_t nt = it.nt, ev0 = it.ev_begin;
    const uint32_t nent = it.s_end - it.s_begin;  // <= 32 (host)
    const uint32_t nsrc = it.n_src;

    // lane q: run of strong entry q and its offset in the virtual stream
    uint32_t rb = 0, rn = 0;
    if (uint32_t(lane) < nent) {
      const uint2 sg = a.seg[it.s_begin + lane];
      rb = sg.x;
      rn = sg.y;
    }
    uint32_t incl = rn;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t roff = incl - rn;

    auto issue_chunk = [&](uint32_t c, int b) {
      const uint32_t v0 = c * C;
      const uint32_t v1 = min(nsrc, v0 + C);
      if (lane == 0) {
        fence_proxy_async();
        mbar_expect_tx(&bar[b], (v1 - v0) * 32u);
      }
      __syncwarp();
      const uint32_t lo = max(roff, v0), hi = min(roff + rn, v1);
      if (hi > lo) bulk_g2s(buf + b * C + (lo - v0), a.src + rb + (lo - roff), (hi - lo) * 32u, &bar[b]);
    };
    const uint32_t nchunk = (nsrc + C - 1) / C;
    if (nchunk > 0) issue_chunk(0, 0);

    // roles: G eval slots of E evals, K source lanes per slot
    const uint32_t G = (nt + E - 1) / E;
    const float rG = 1.0f / float(G);
    const uint32_t K = uint32_t(32.0f * rG + 1e-4f);
    const uint32_t k = uint32_t((float(lane) + 0.5f) * rG);
    const uint32_t g = uint32_t(lane) - k * G;
    const bool active = k < K;

    double yx[E], yy[E], ar[E], ai[E];
    uint32_t vself[E];  // position of the eval's own source in the virtual stream
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t le = g * E + e;
      const bool ok = active && le < nt;
      const double4 r = ok ? a.evr[ev0 + le] : make_double4(0.0, 0.0, 0.0, 0.0);
      yx[e] = r.x;
      yy[e] = r.y;
      ar[e] = 0.0;
      ai[e] = 0.0;
      const uint32_t self = ok ? uint32_t(__double_as_longlong(r.z)) : kNoSelf;
      const uint32_t q = ok ? uint32_t(__double_as_longlong(r.w)) : kNoSelf;
      const uint32_t qq = q - it.s_begin;  // entry of the self run within this item
      const uint32_t src_lane = qq < nent ? qq : 0u;
      const uint32_t qb = __shfl_sync(FULL, rb, src_lane);
      const uint32_t qo = __shfl_sync(FULL, roff, src_lane);
      vself[e] = (q != kNoSelf && qq < nent) ? qo + (self - qb) : kNoSelf;
      if (vself[e] != kNoSelf && k == 0) ++hits;  // skipped exactly once
    }

    for (uint32_t c = 0; c < nchunk; ++c) {
      const int b = int(c & 1u);
      if (c + 1 < nchunk) issue_chunk(c + 1, b ^ 1);
      const uint32_t v0 = c * C;
      const uint32_t len = min(nsrc - v0, uint32_t(C));
      // self positions inside this chunk and the warp's window [plo, phi]
      uint32_t ps[E];
      uint32_t plo = kNoSelf, phi = 0u;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t d = vself[e] - v0;
        ps[e] = (vself[e] != kNoSelf && d < len) ? d : kNoSelf;
        if (ps[e] != kNoSelf) {
          plo = min(plo, ps[e]);
          phi = max(phi, ps[e]);
        }
      }
      plo = __reduce_min_sync(FULL, plo);
      phi = __reduce_max_sync(FULL, phi);
      if (b == 0) {
        mbar_wait(&bar[0], parity0);
        parity0 ^= 1u;
      } else {
        mbar_wait(&bar[1], parity1);
        parity1 ^= 1u;
      }
      if (active) {
        const double4* chunk = buf + b * C;
        const double4* p = chunk + k;
        const double4* const end = chunk + len;
        p = run_unchecked<KERNEL, SMOOTH, E, U>(p, chunk + min(plo, len), K, yx, yy, a.inv_delta2,
                                                a.delta2, ar, ai);
        if (plo != kNoSelf) {
          const double4* const end2 = chunk + min(phi + 1u, len);
          for (; p < end2; p += K) {
            const double4 s = *p;
            const uint32_t j = uint32_t(p - chunk);
#pragma unroll
            for (int e = 0; e < E; ++e)
              pair_accum<KERNEL, SMOOTH>(yx[e], yy[e], s, a.inv_delta2, a.delta2, j != ps[e],
                                         ar[e], ai[e]);
          }
          run_unchecked<KERNEL, SMOOTH, E, U>(p, end, K, yx, yy, a.inv_delta2, a.delta2, ar, ai);
        }
      }
      __syncwarp();  // chunk b fully read before it is refilled
    }

    // the previous item's result store must have read the staging area
    if (lane == 0) bulk_wait_read();
    __syncwarp();
    // sum the K partials of every eval over lanes g, g+G, ... (fixed order)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      double sr = ar[e], si = ai[e];
      for (uint32_t kk = 1; kk < K; ++kk) {
        const int src = int(g + kk * G) & 31;
        const double vr = __shfl_sync(FULL, ar[e], src);
        const double vi = __shfl_sync(FULL, ai[e], src);
        sr += vr;
        si += vi;
      }
      const uint32_t le = g * E + e;
      if (k == 0 && active && le < nt)
        stage[le] = (KERNEL == 0) ? make_double2(-sr, -si) : make_double2(sr, si);
    }
    // one TMA bulk store of the item's nt contiguous results (device memory,
    // or page-locked host memory written straight over PCIe)
    fence_proxy_async();
    __syncwarp();
    if (lane == 0 && nt) {
      double2* dst = (it.partial_off == kNoSelf) ? a.out + ev0 : a.partial + it.partial_off;
      bulk_s2g(dst, stage, nt * 16u);
    }
  }
  if (lane == 0) bulk_wait_all();
  for (int o = 16; o > 0; o >>= 1) hits += __shfl_down_sync(FULL, hits, o);
  if (lane == 0 && hits) atomicAdd(a.hits, (unsigned long long)hits);
}

}  // namespace fmmcu
