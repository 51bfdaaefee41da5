// fmm-b200 — P2P near-field kernels for sm_100a.
//
// Device restatement of the reference near-field loop near_box()
// (proj/src/backend.cpp:41-69) with the per-pair arithmetic of
// kernel_term()/smoother_factor() (proj/src/expansion.cpp:78-92).
//
// Fast path (p2p_tile_kernel):
//   * one work item (= one target leaf, or one chunk of a heavy leaf's
//     strong list) per CTA;
//   * the item's source leaves are contiguous runs of packed 32-byte records
//     {x, y, m_re, m_im}; an elected thread issues one TMA bulk copy
//     (cp.async.bulk + mbarrier complete_tx) per run into a shared tile;
//   * thread (g, k) owns E evals of eval-slot g and walks sources
//     k, k+K, k+2K, ... of the tile (broadcast LDS.128); partials are reduced
//     over k in a fixed order through shared memory (deterministic);
//   * per pair: 2 DADD, r^2 (DMUL+DFMA), 1/r^2 = MUFU.RCP64H seed + one
//     cubic Newton step (3 DFMA), m*conj(d) (2 DMUL + 2 DFMA), 2 DFMA
//     accumulate -- 13 FP64 instructions, 23 algorithmic flops.
// Exact path (p2p_exact_kernel): one thread per eval, reference order,
// libgcc __divdc3 restated with non-contracted __d*_rn intrinsics -- bitwise
// equal to the reference for the harmonic kernel without smoother.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fmmcu {

constexpr uint32_t kNoSelf = 0xFFFFFFFFu;

// Work item: target leaf `leaf`, strong entries [s_begin, s_end) of its list.
struct P2PItem {
  uint32_t leaf;
  uint32_t s_begin;
  uint32_t s_end;
  uint32_t n_src;        // sources covered by this item
  uint32_t partial_off;  // kNoSelf: write out[] directly; else base (in evals) into partial[]
  uint32_t pad;
};

struct P2PArgs {
  const double4* __restrict__ src;   // packed sources, permuted order
  const double2* __restrict__ evy;   // eval positions, permuted order
  const uint32_t* __restrict__ eself;  // permuted slot of the eval's own source, or kNoSelf
  const uint32_t* __restrict__ pt_off;
  const uint32_t* __restrict__ ev_off;
  const uint32_t* __restrict__ s_off;
  const uint32_t* __restrict__ s_idx;
  const P2PItem* __restrict__ items;
  uint32_t n_items;
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

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

// ------------------------------------------------------------ fast kernel --
// Dynamic smem layout: [mbarrier 16 B][tile: TILE double4][reduction scratch]
template <int KERNEL, int SMOOTH, int E, int THREADS, int TILE>
__global__ void __launch_bounds__(THREADS)
    p2p_tile_kernel(const P2PArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double4* tile = reinterpret_cast<double4*>(smem_raw + 128);
  __shared__ uint32_t seg_gbeg[64];  // segments (source leaf runs) of the current tile
  __shared__ uint32_t seg_tpos[65];
  __shared__ uint32_t s_nseg;
  __shared__ uint32_t s_cursor_entry, s_cursor_off;
  __shared__ unsigned int s_hits;

  const P2PItem it = a.items[blockIdx.x];
  const uint32_t ev0 = a.ev_off[it.leaf];
  const uint32_t nt = a.ev_off[it.leaf + 1] - ev0;
  const int tid = threadIdx.x;
  if (nt == 0 || it.n_src == 0) {  // host never emits these; keep the kernel total
    if (it.partial_off != kNoSelf)
      for (uint32_t e = tid; e < nt; e += THREADS) a.partial[it.partial_off + e] = make_double2(0.0, 0.0);
    else
      for (uint32_t e = tid; e < nt; e += THREADS) a.out[ev0 + e] = make_double2(0.0, 0.0);
    return;
  }

  // eval-slot g owns evals [g*E, g*E+E); K source lanes share the slot.
  const uint32_t G = (nt + E - 1) / E;
  const uint32_t Gc = G < THREADS ? G : THREADS;  // slots per pass
  const uint32_t K = THREADS / Gc;

  if (tid == 0) {
    mbar_init(bar, 1);
    s_hits = 0;
    s_cursor_entry = it.s_begin;
    s_cursor_off = 0;
  }
  __syncthreads();
  uint32_t phase = 0;

  for (uint32_t g0 = 0; g0 < G; g0 += Gc) {  // eval passes (only > 1 for huge leaves)
    const uint32_t g = g0 + (uint32_t)tid % Gc;
    const uint32_t k = (uint32_t)tid / Gc;
    const bool active = (k < K) && (g < G);
    double yx[E], yy[E], ar[E], ai[E];
    uint32_t sg[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t le = g * E + e;
      const bool ok = active && le < nt;
      const double2 y = ok ? a.evy[ev0 + le] : make_double2(1e300, 1e300);
      yx[e] = y.x;
      yy[e] = y.y;
      sg[e] = ok ? a.eself[ev0 + le] : kNoSelf;
      ar[e] = 0.0;
      ai[e] = 0.0;
    }

    if (tid == 0) {
      s_cursor_entry = it.s_begin;
      s_cursor_off = 0;
    }
    __syncthreads();

    uint32_t remaining = it.n_src;
    while (remaining > 0) {
      // ---- stage one tile: elected thread issues bulk copies -------------
      if (tid == 0) {
        uint32_t filled = 0, nseg = 0;
        uint32_t ent = s_cursor_entry, off = s_cursor_off;
        // count bytes first (expect_tx must precede completion accounting)
        uint32_t ent2 = ent, off2 = off, bytes = 0, f2 = 0;
        while (f2 < TILE && ent2 < it.s_end && nseg < 64) {
          const uint32_t sb = a.s_idx[ent2];
          const uint32_t b = a.pt_off[sb], n = a.pt_off[sb + 1] - b;
          const uint32_t take = min(n - off2, (uint32_t)TILE - f2);
          if (take > 0) {
            seg_gbeg[nseg] = b + off2;
            seg_tpos[nseg] = f2;
            ++nseg;
          }
          f2 += take;
          bytes += take * 32u;
          off2 += take;
          if (off2 == n) {
            ++ent2;
            off2 = 0;
          }
        }
        seg_tpos[nseg] = f2;
        s_nseg = nseg;
        fence_proxy_async();
        mbar_expect_tx(bar, bytes);
        for (uint32_t sIdx = 0; sIdx < nseg; ++sIdx) {
          const uint32_t n = seg_tpos[sIdx + 1] - seg_tpos[sIdx];
          bulk_g2s(tile + seg_tpos[sIdx], a.src + seg_gbeg[sIdx], n * 32u, bar);
        }
        filled = f2;
        (void)filled;
        s_cursor_entry = ent2;
        s_cursor_off = off2;
      }
      __syncthreads();
      const uint32_t nseg = s_nseg;
      const uint32_t ntile = seg_tpos[nseg];
      // tile position of each eval's own source (segments ascend in gbeg)
      uint32_t ps[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        ps[e] = kNoSelf;
        const uint32_t s = sg[e];
        if (s != kNoSelf && nseg > 0 && s >= seg_gbeg[0]) {
          uint32_t lo = 0, hi = nseg;  // seg_gbeg[lo] <= s < seg_gbeg[hi]
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (seg_gbeg[mid] <= s) lo = mid; else hi = mid;
          }
          const uint32_t n = seg_tpos[lo + 1] - seg_tpos[lo];
          if (s - seg_gbeg[lo] < n) ps[e] = seg_tpos[lo] + (s - seg_gbeg[lo]);
        }
      }
      if (ntile == 0) break;  // defensive: never spin on an empty tile
      mbar_wait(bar, phase);
      phase ^= 1u;

      bool my_self = false;
#pragma unroll
      for (int e = 0; e < E; ++e) my_self |= (ps[e] != kNoSelf);
      const bool warp_self = __any_sync(0xffffffffu, my_self);  // warp-uniform path choice
      if (active) {
        if (!warp_self) {
#pragma unroll 2
          for (uint32_t j = k; j < ntile; j += K) {
            const double4 s = tile[j];
#pragma unroll
            for (int e = 0; e < E; ++e)
              pair_accum<KERNEL, SMOOTH>(yx[e], yy[e], s, a.inv_delta2, a.delta2, true, ar[e],
                                         ai[e]);
          }
        } else {
#pragma unroll 2
          for (uint32_t j = k; j < ntile; j += K) {
            const double4 s = tile[j];
#pragma unroll
            for (int e = 0; e < E; ++e)
              pair_accum<KERNEL, SMOOTH>(yx[e], yy[e], s, a.inv_delta2, a.delta2, j != ps[e],
                                         ar[e], ai[e]);
          }
          // a self pair is skipped by exactly one source lane
          unsigned int h = 0;
#pragma unroll
          for (int e = 0; e < E; ++e)
            h += (ps[e] != kNoSelf && (ps[e] % K) == k && g * E + e < nt) ? 1u : 0u;
          if (h) atomicAdd(&s_hits, h);
        }
      }
      remaining -= ntile;
      __syncthreads();  // tile consumed before it is overwritten
    }

    // ---- reduce the K partials of each eval in fixed k order -------------
    double2* red = reinterpret_cast<double2*>(tile);  // reuse the tile
    if (active) {
#pragma unroll
      for (int e = 0; e < E; ++e) red[k * (Gc * E) + (g - g0) * E + e] = make_double2(ar[e], ai[e]);
    }
    __syncthreads();
    const uint32_t nslot = min(Gc * E, nt - g0 * E);
    for (uint32_t le = tid; le < nslot; le += THREADS) {
      double sr = 0.0, si = 0.0;
      for (uint32_t kk = 0; kk < K; ++kk) {
        const double2 v = red[kk * (Gc * E) + le];
        sr += v.x;
        si += v.y;
      }
      const double2 res = (KERNEL == 0) ? make_double2(-sr, -si) : make_double2(sr, si);
      const uint32_t gl = g0 * E + le;
      if (it.partial_off == kNoSelf)
        a.out[ev0 + gl] = res;
      else
        a.partial[it.partial_off + gl] = res;
    }
    __syncthreads();
  }
  if (tid == 0 && s_hits) atomicAdd(a.hits, (unsigned long long)s_hits);
}

// Sum the partials of split leaves in chunk order.  One thread per eval.
// fin: per split leaf {leaf, first partial base, n_chunks}; chunks of one
// leaf are consecutive, each nt evals long.
struct P2PFinal {
  uint32_t leaf;
  uint32_t base;
  uint32_t n_chunks;
  uint32_t pad;
};

__global__ void p2p_finalize_kernel(const P2PFinal* __restrict__ fin, uint32_t n_fin,
                                    const uint32_t* __restrict__ ev_off,
                                    const double2* __restrict__ partial,
                                    double2* __restrict__ out) {
  const uint32_t f = blockIdx.x;
  if (f >= n_fin) return;
  const P2PFinal F = fin[f];
  const uint32_t ev0 = ev_off[F.leaf];
  const uint32_t nt = ev_off[F.leaf + 1] - ev0;
  for (uint32_t e = threadIdx.x; e < nt; e += blockDim.x) {
    double sr = 0.0, si = 0.0;
    for (uint32_t c = 0; c < F.n_chunks; ++c) {
      const double2 v = partial[F.base + c * nt + e];
      sr += v.x;
      si += v.y;
    }
    out[ev0 + e] = make_double2(sr, si);
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
