// fmm-b200 — P2P near-field kernels for sm_100a.
//
// Device restatement of the reference near-field loop near_box()
// (proj/src/backend.cpp:41-69) with the per-pair arithmetic of
// kernel_term()/smoother_factor() (proj/src/expansion.cpp:78-92).
//
// Shared pieces of the fast paths (p2p_warp.cuh, p2p_sym.cuh): work items,
// TMA bulk-copy / mbarrier helpers, the per-pair arithmetic (FP64 CUDA-core
// pipe, no tensor cores: 2 DADD, r^2 (DMUL+DFMA), 1/r^2 = MUFU.RCP64H seed +
// one cubic Newton step (3 DFMA), m*conj(d) (2 DMUL + 2 DFMA), 2 DFMA
// accumulate -- 13 FP64 instructions for 23 algorithmic flops), eval records
// and the fixed-order reduction of split heavy leaves.
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
// Gaussian smoother factor 1 - exp(-x), x = r^2 / delta^2 (expansion.cpp:83).
// For x >= 38, exp(-x) < 2^-54, so the difference rounds to exactly 1.0:
// when every active lane of the warp is that far (source runs of distant
// strong partners), the whole warp skips the exp -- same bits.
__device__ __forceinline__ double gauss_g(double x) {
  if (__all_sync(__activemask(), x >= 38.0)) return 1.0;
  return 1.0 - exp(-x);
}

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
      const double g = gauss_g(r2 * inv_d2);
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
    if (SMOOTH == 1) g = gauss_g(r2 * inv_d2);
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

// ------------------------------------------------------------ fast kernel --
// Eval record as staged on the device: {x, y, self slot (bits), q_self (bits)}
// where q_self is the global strong-entry index (position in strong_idx) of
// the eval's own leaf's entry whose source run holds the self slot, or
// kNoSelf -- this makes the per-tile self lookup O(1).  The runs of a strong
// list are disjoint and ascending in slot order (the list is sorted by leaf
// and pt_off is monotone), so the entry holding the slot is the last one
// starting at or before it: a binary search (clustered leaves have lists of
// thousands of entries; the former linear scan cost 0.67 ms at 1M gauss8).
__device__ __forceinline__ uint32_t find_self_entry(const P2PArgs& a, uint32_t leaf,
                                                    uint32_t self) {
  if (self == kNoSelf) return kNoSelf;
  uint32_t lo = a.s_off[leaf], hi = a.s_off[leaf + 1];  // answer in [lo, hi)
  if (lo == hi || a.seg[lo].x > self) return kNoSelf;
  while (hi - lo > 1) {  // invariant: seg[lo].x <= self, entries >= hi start after self
    const uint32_t mid = (lo + hi) >> 1;
    if (a.seg[mid].x <= self) lo = mid;
    else hi = mid;
  }
  const uint2 sg = a.seg[lo];
  return self - sg.x < sg.y ? lo : kNoSelf;
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
