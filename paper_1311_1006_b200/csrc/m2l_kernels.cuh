// fmm-b200 — batched M2L (multipole-to-local) translations for sm_100a.
//
// Device restatement of m2l_add() (proj/src/expansion.cpp:188-269) as called
// by the downward pass for every weak partner of every box with evaluation
// points (proj/src/engine.cpp:96-114).  Because every outgoing expansion is
// known after the upward pass, the M2L sums of *all* levels are independent
// and run in one launch:
//     out[t][l] = sum_{w in weak(t), ascending} M2L(outgoing[w] -> centre[t])[l]
// The host then forms local = L2L(parent) + out[t] level by level.
//
// Mapping: one warp per target box, lanes over the local index l (chunks of
// 32 for p >= 32).  Per partner: w = 1/z0; powers w^j by a warp shuffle scan;
// v_k = b_k (-1)^{k+1} w^{k+1} (harmonic) or u_k = b_k (-1)^k w^k (log)
// staged in shared memory; acc_l = sum_k T[k][l] v_k with the binomial table
// T read coalesced through L1; c_l += w^l acc_l.
// Reference semantics kept: z0 == 0 raises SingularConfiguration (flag);
// when (p+2) log10|w| >= 250 (the reference's long double branch,
// expansion.cpp:196-199) the power chains are formed progressively,
// b_k w^(k+1) = (((b_k w) w) ...), so no intermediate exceeds the final value.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>

#include "m2l_args.cuh"

namespace fmmcu {



__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

__device__ __forceinline__ double2 shfl_up2(double2 v, int d) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// acc += t * v for a compile-time t: t == 0 drops out, t == 1 is an add
__device__ __forceinline__ void constexpr_fma_pair(const double t, const double2 v, double& ar,
                                                   double& ai) {
  if (t == 0.0) return;
  if (t == 1.0) {
    ar += v.x;
    ai += v.y;
    return;
  }
  ar = fma(t, v.x, ar);
  ai = fma(t, v.y, ai);
}

constexpr int kM2LWarps = 4;

static __global__ void __launch_bounds__(kM2LWarps * 32) m2l_batched_kernel(const M2LArgs a) {
  __shared__ double2 s_v[kM2LWarps][kM2LMaxP + 1];
  __shared__ double2 s_pw[kM2LWarps][kM2LMaxP + 2];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const uint32_t t = blockIdx.x * kM2LWarps + wid;
  if (t >= a.n_targets) return;
  const int P1 = a.p + 1;
  const int nchunk = (P1 + 31) >> 5;
  double2* v = s_v[wid];
  double2* pw = s_pw[wid];
  const double2 ct = a.centers[a.target_box[t]];

  double2 c[4];  // local coefficients l = lane + 32*q
#pragma unroll
  for (int q = 0; q < 4; ++q) c[q] = make_double2(0.0, 0.0);

  for (uint32_t wi = a.weak_off[t]; wi < a.weak_off[t + 1]; ++wi) {
    const uint32_t sb = a.weak_idx[wi];
    const double2 cs = a.centers[sb];
    const double2 z0 = make_double2(cs.x - ct.x, cs.y - ct.y);
    if (z0.x == 0.0 && z0.y == 0.0) {
      if (lane == 0) atomicOr(a.singular, 1);
      continue;
    }
    const double zz = fma(z0.x, z0.x, z0.y * z0.y);
    const double2 w = make_double2(z0.x / zz, -z0.y / zz);
    const double w2 = fma(w.x, w.x, w.y * w.y);
    const double2* b = a.coeffs + (size_t)sb * P1;

    if (w2 < a.big_w2) {
      // powers w^j, j = 1..p+1, by a shuffle scan (lane L -> w^(L+1))
      double2 x = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double2 y = shfl_up2(x, o);
        if (lane >= o) x = cmul(x, y);
      }
      const double2 w32 = shfl2(x, 31);
      if (lane == 0) pw[0] = make_double2(1.0, 0.0);
      double2 xc = x;
      for (int q = 0; q < nchunk; ++q) {
        const int j = lane + 32 * q + 1;
        if (j <= P1) pw[j] = xc;
        xc = cmul(xc, w32);
      }
      __syncwarp();
      // source vector
      for (int k = lane; k < P1; k += 32) {
        const double2 bk = b[k];
        double2 val;
        if (a.kernel == 0) {
          const double sgn = (k & 1) ? 1.0 : -1.0;  // (-1)^(k+1)
          val = cmul(make_double2(sgn * bk.x, sgn * bk.y), pw[k + 1]);
        } else {
          const double sgn = (k & 1) ? -1.0 : 1.0;  // (-1)^k
          val = cmul(make_double2(sgn * bk.x, sgn * bk.y), pw[k]);
        }
        v[k] = val;
      }
    } else {
      // overflow-safe progressive chains (rare: nearly coincident centres)
      if (lane == 0) pw[0] = make_double2(1.0, 0.0);
      for (int k = lane; k < P1; k += 32) {
        const double2 bk = b[k];
        const int n = (a.kernel == 0) ? k + 1 : k;
        const double sgn = (a.kernel == 0) ? ((k & 1) ? 1.0 : -1.0) : ((k & 1) ? -1.0 : 1.0);
        double2 val = make_double2(sgn * bk.x, sgn * bk.y);
        for (int r = 0; r < n; ++r) val = cmul(val, w);
        v[k] = val;
      }
    }
    __syncwarp();

    // acc_l = sum_k T[k][l] v_k
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q >= nchunk) break;
      const int l = lane + 32 * q;
      if (l >= P1) break;
      double2 acc = make_double2(0.0, 0.0);
      const int kbeg = (a.kernel == 0) ? 0 : 1;
      for (int k = kbeg; k < P1; ++k) {
        const double tk = __ldg(a.table + (size_t)k * P1 + l);
        const double2 vk = v[k];
        acc.x = fma(tk, vk.x, acc.x);
        acc.y = fma(tk, vk.y, acc.y);
      }
      if (a.kernel != 0) {
        const double2 a0 = b[0];
        if (l == 0) {
          // a0 * log(-z0)
          const double lr = 0.5 * log(zz);
          const double th = atan2(-z0.y, -z0.x);
          acc.x += a0.x * lr - a0.y * th;
          acc.y += a0.x * th + a0.y * lr;
        } else {
          acc.x -= a0.x / (double)l;
          acc.y -= a0.y / (double)l;
        }
      }
      double2 add;
      if (w2 < a.big_w2) {
        add = cmul(pw[l], acc);
      } else {
        add = acc;
        for (int r = 0; r < l; ++r) add = cmul(add, w);
      }
      if (a.kernel != 0 && l == 0) add = acc;
      c[q].x += add.x;
      c[q].y += add.y;
    }
    __syncwarp();
  }
  double2* o = a.out + (size_t)t * P1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int l = lane + 32 * q;
    if (l < P1) o[l] = c[q];
  }
}

// ---------------------------------------------------------------------------
// Thread-per-target M2L (the default for p + 1 <= kM2LConstP1).  One thread
// owns a target box and its p+1 local coefficients in registers; for each
// weak partner it forms v_k in registers and applies the binomial matrix
// T[k][l] read from constant memory (every thread of a warp reads the same
// entry at the same time: a broadcast), then c_l += w^l acc_l.  All lanes do
// useful work (the warp kernel above keeps only p+1 of 32 lanes busy) and
// there is no shared memory or shuffle traffic.  Same arithmetic and the
// same overflow-safe branch as m2l_batched_kernel.
constexpr int kM2LConstP1 = 40;
static __constant__ double c_m2l_table[kM2LConstP1 * kM2LConstP1];

template <int P1, int TBK = (P1 > 20 ? 64 : 128)>
static __global__ void __launch_bounds__(TBK, 384 / TBK) m2l_thread_kernel(const M2LArgs a) {
  // local coefficients in shared memory, [l][thread] (conflict-free), so the
  // registers hold only the partner's v_k: 12 warps/SM instead of 8
  __shared__ double2 s_c[P1][TBK];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const int tid = threadIdx.x;
#pragma unroll
  for (int l = 0; l < P1; ++l) s_c[l][tid] = make_double2(0.0, 0.0);
  if (t >= a.n_targets) return;
  const double2 ct = a.centers[a.target_box[t]];
  const bool harm = a.kernel == 0;
  const uint32_t w0 = a.weak_off[t], w1 = a.weak_off[t + 1];
  for (uint32_t wi = w0; wi < w1; ++wi) {
    const uint32_t sb = a.weak_idx[wi];
    const double2 cs = a.centers[sb];
    const double2 z0 = make_double2(cs.x - ct.x, cs.y - ct.y);
    if (z0.x == 0.0 && z0.y == 0.0) {
      atomicOr(a.singular, 1);
      continue;
    }
    const double zz = fma(z0.x, z0.x, z0.y * z0.y);
    const double2 w = make_double2(z0.x / zz, -z0.y / zz);
    const double w2 = fma(w.x, w.x, w.y * w.y);
    const bool safe = w2 >= a.big_w2;  // rare: nearly coincident centres
    const double2* b = a.coeffs + (size_t)sb * P1;
    double vr[P1], vi[P1];
    double2 wp = harm ? w : make_double2(1.0, 0.0);  // w^(k+1) | w^k
#pragma unroll
    for (int k = 0; k < P1; ++k) {
      const double2 bk = b[k];
      const double sgn = harm ? ((k & 1) ? 1.0 : -1.0) : ((k & 1) ? -1.0 : 1.0);
      double2 val = make_double2(sgn * bk.x, sgn * bk.y);
      if (!safe) {
        val = cmul(val, wp);
        wp = cmul(wp, w);
      } else {
        const int n = harm ? k + 1 : k;
        for (int r = 0; r < n; ++r) val = cmul(val, w);
      }
      vr[k] = val.x;
      vi[k] = val.y;
    }
    double2 wl = make_double2(1.0, 0.0);
    const double2 a0 = b[0];
#pragma unroll
    for (int l = 0; l < P1; ++l) {
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int k = 0; k < P1; ++k) {
        const double tk = c_m2l_table[k * P1 + l];  // zero row k = 0 for the log kernel
        sr = fma(tk, vr[k], sr);
        si = fma(tk, vi[k], si);
      }
      double2 acc = make_double2(sr, si);
      if (!harm) {
        if (l == 0) {
          const double lr = 0.5 * log(zz);
          const double th = atan2(-z0.y, -z0.x);
          acc.x += a0.x * lr - a0.y * th;
          acc.y += a0.x * th + a0.y * lr;
        } else {
          acc.x -= a0.x / (double)l;
          acc.y -= a0.y / (double)l;
        }
      }
      double2 add;
      if (!harm && l == 0) {
        add = acc;
      } else if (!safe) {
        add = cmul(wl, acc);
      } else {
        add = acc;
        for (int r = 0; r < l; ++r) add = cmul(add, w);
      }
      double2 cur = s_c[l][tid];
      cur.x += add.x;
      cur.y += add.y;
      s_c[l][tid] = cur;
      wl = cmul(wl, w);
    }
  }
  double2* o = a.out + (size_t)t * P1;
#pragma unroll
  for (int l = 0; l < P1; ++l) o[l] = s_c[l][tid];
}

// ---------------------------------------------------------------------------
// Register-accumulator M2L (the default for the orders m2l_run instantiates).
//
// Work items, not targets: m2l_run cuts every weak list longer than
// kM2LChunk partners into balanced chunks (clustered trees have lists of
// thousands: one thread per target left a single thread walking them, 48 ms
// for 3.1M ops at 1M gauss8 against 0.4 ms for 3.5M uniform ops).  A chunk of
// a split list writes its partial local to `partial`, and m2l_reduce_kernel
// sums a target's chunks in chunk order (deterministic); an unsplit target
// writes `out` directly.  One thread per item (m2l_run sizes the grid to the
// item bound; threads past the device count exit).
//
// Per item, one thread; per partner:
//   pass 1: v_k = (-1)^(k+1) b_k w^(k+1) (harmonic) | (-1)^k b_k w^k (log)
//           into the thread's shared column s_v[k][tid];
//   pass 2: acc_l = sum_k T[k][l] v_k, k-outer / l-inner, so a thread carries
//           2 LB independent FMA chains (the r1 l-outer order was two serial
//           chains per l: FP64 pipe waiting on its own latency); l runs in
//           blocks of LB so the accumulators stay in registers at any order;
//   then local_l += w^l acc_l in shared memory [l][tid] (conflict-free).
// T is compile-time: T[k][l] = C(l+k, k) (harmonic) or C(l+k-1, k-1) (log,
// row 0 zero), unrolled structurally (integer_sequence folds), so each entry
// is an immediate / constant-bank operand and the ones and zeros of row 0 /
// column 0 cost nothing.  Same per-partner arithmetic as the reference
// m2l_add (expansion.cpp:188-269) up to the order of the power chains; the
// overflow-safe branch (the reference's long double path,
// expansion.cpp:196-199) runs progressive chains.
constexpr uint32_t kM2LChunk = 48;  // partners per work item

__host__ __device__ constexpr double binom_c(int n, int k) {
  if (k < 0 || k > n) return 0.0;
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * double(n - k + i) / double(i);
  return r;
}

template <bool HARM>
__host__ __device__ constexpr double m2l_t(int k, int l) {
  return HARM ? binom_c(l + k, k) : (k == 0 ? 0.0 : binom_c(l + k - 1, k - 1));
}

template <bool HARM, int K, int L>
struct M2LT {
  static constexpr double value = m2l_t<HARM>(K, L);
};

// acc[j] += T[K][L0 + j] v for the LB columns of one l-block
template <bool HARM, int K, int L0, int... Js>
__device__ __forceinline__ void m2l_row(const double2 v, double* ar, double* ai,
                                        std::integer_sequence<int, Js...>) {
  (constexpr_fma_pair(M2LT<HARM, K, L0 + Js>::value, v, ar[Js], ai[Js]), ...);
}

template <bool HARM, int TB, int L0, int LB, int... Ks>
__device__ __forceinline__ void m2l_rows(const double2 (*s_v)[TB], int tid, double* ar, double* ai,
                                         std::integer_sequence<int, Ks...>) {
  ((HARM || Ks > 0
        ? m2l_row<HARM, Ks, L0>(s_v[Ks][tid], ar, ai, std::make_integer_sequence<int, LB>{})
        : void()),
   ...);
}

// one l-block [L0, L0 + LB): product, log-kernel terms, w^l scaling, add
template <bool HARM, int P1, int TB, int L0, int LB>
__device__ __forceinline__ void m2l_block(const double2 (*s_v)[TB], double2 (*s_c)[TB], int tid,
                                          const double2 w, const double2 z0, const double zz,
                                          const double2 a0, double2& wl) {
  double ar[LB], ai[LB];
#pragma unroll
  for (int j = 0; j < LB; ++j) ar[j] = ai[j] = 0.0;
  m2l_rows<HARM, TB, L0, LB>(s_v, tid, ar, ai, std::make_integer_sequence<int, P1>{});
#pragma unroll
  for (int j = 0; j < LB; ++j) {
    const int l = L0 + j;
    double2 acc = make_double2(ar[j], ai[j]);
    double2 add;
    if (!HARM && l == 0) {
      const double lr = 0.5 * log(zz);
      const double th = atan2(-z0.y, -z0.x);
      add = make_double2(acc.x + (a0.x * lr - a0.y * th), acc.y + (a0.x * th + a0.y * lr));
    } else {
      if (!HARM) {
        acc.x -= a0.x / (double)l;
        acc.y -= a0.y / (double)l;
      }
      add = (l == 0) ? acc : cmul(wl, acc);
    }
    double2 cur = s_c[l][tid];
    cur.x += add.x;
    cur.y += add.y;
    s_c[l][tid] = cur;
    if (l + 1 < P1) wl = (l == 0) ? w : cmul(wl, w);
  }
}

template <bool HARM, int P1, int TB, int LB, int... Bs>
__device__ __forceinline__ void m2l_blocks(const double2 (*s_v)[TB], double2 (*s_c)[TB], int tid,
                                           const double2 w, const double2 z0, const double zz,
                                           const double2 a0, std::integer_sequence<int, Bs...>) {
  double2 wl = make_double2(1.0, 0.0);
  (m2l_block<HARM, P1, TB, Bs * LB, (P1 - Bs * LB < LB ? P1 - Bs * LB : LB)>(s_v, s_c, tid, w, z0,
                                                                              zz, a0, wl),
   ...);
}

template <int P1>
struct M2LRegShape {
  static constexpr int TB = P1 <= 22 ? 64 : 32;  // 2*P1*TB*16 B of shared memory per CTA
  static constexpr int LB = P1 <= 18 ? P1 : (P1 + 1) / 2;  // accumulators per l-block
  static constexpr int NB = (P1 + LB - 1) / LB;
  static constexpr int MINB = P1 <= 18 ? 6 : P1 <= 22 ? 4 : 8;
};

template <int P1, bool HARM>
static __global__ void __launch_bounds__(M2LRegShape<P1>::TB, M2LRegShape<P1>::MINB)
m2l_reg_kernel(const M2LArgs a) {
  using Sh = M2LRegShape<P1>;
  constexpr int TB = Sh::TB;
  __shared__ double2 s_c[P1][TB];
  __shared__ double2 s_v[P1][TB];
  const int tid = threadIdx.x;
  const uint32_t n_items = *a.n_items;
  for (uint32_t it = blockIdx.x * TB + tid; it < n_items; it += gridDim.x * TB) {  // one pass when the grid covers the items
    const uint4 item = a.items[it];
#pragma unroll
    for (int l = 0; l < P1; ++l) s_c[l][tid] = make_double2(0.0, 0.0);
    const double2 ct = a.centers[a.target_box[item.x]];
    const uint32_t w0 = item.y, w1 = item.z;
    uint32_t sb_next = (w0 < w1) ? __ldg(a.weak_idx + w0) : 0u;
    for (uint32_t wi = w0; wi < w1; ++wi) {
      const uint32_t sb = sb_next;
      if (wi + 1 < w1) sb_next = __ldg(a.weak_idx + wi + 1);
      const double2 cs = __ldg(a.centers + sb);
      const double2 z0 = make_double2(cs.x - ct.x, cs.y - ct.y);
      if (z0.x == 0.0 && z0.y == 0.0) {
        atomicOr(a.singular, 1);
        continue;
      }
      const double zz = fma(z0.x, z0.x, z0.y * z0.y);
      const double2 w = make_double2(z0.x / zz, -z0.y / zz);
      const double w2 = fma(w.x, w.x, w.y * w.y);
      const double2* b = a.coeffs + (size_t)sb * P1;
      if (w2 >= a.big_w2) {
        // rare (nearly coincident centres): progressive chains, no table
        for (int l = 0; l < P1; ++l) {
          double2 acc = make_double2(0.0, 0.0);
          for (int k = HARM ? 0 : 1; k < P1; ++k) {
            const double2 bk = b[k];
            const double sgn = HARM ? ((k & 1) ? 1.0 : -1.0) : ((k & 1) ? -1.0 : 1.0);
            double2 val = make_double2(sgn * bk.x, sgn * bk.y);
            for (int r = 0; r < (HARM ? k + 1 : k); ++r) val = cmul(val, w);
            const double tk = m2l_t<HARM>(k, l);
            acc.x = fma(tk, val.x, acc.x);
            acc.y = fma(tk, val.y, acc.y);
          }
          if (!HARM) {
            const double2 a0 = b[0];
            if (l == 0) {
              const double lr = 0.5 * log(zz);
              const double th = atan2(-z0.y, -z0.x);
              acc.x += a0.x * lr - a0.y * th;
              acc.y += a0.x * th + a0.y * lr;
            } else {
              acc.x -= a0.x / (double)l;
              acc.y -= a0.y / (double)l;
            }
          }
          if (HARM || l > 0)
            for (int r = 0; r < l; ++r) acc = cmul(acc, w);
          double2 cur = s_c[l][tid];
          cur.x += acc.x;
          cur.y += acc.y;
          s_c[l][tid] = cur;
        }
        continue;
      }
      {
        double2 wp = HARM ? w : make_double2(1.0, 0.0);  // w^(k+1) | w^k
#pragma unroll
        for (int k = 0; k < P1; ++k) {
          const double2 bk = __ldg(b + k);
          const double sgn = HARM ? ((k & 1) ? 1.0 : -1.0) : ((k & 1) ? -1.0 : 1.0);
          s_v[k][tid] = cmul(make_double2(sgn * bk.x, sgn * bk.y), wp);
          if (k + 1 < P1) wp = cmul(wp, w);
        }
      }
      const double2 a0 = HARM ? make_double2(0.0, 0.0) : __ldg(b);
      m2l_blocks<HARM, P1, TB, Sh::LB>(s_v, s_c, tid, w, z0, zz, a0,
                                       std::make_integer_sequence<int, Sh::NB>{});
    }
    double2* o = (item.w == 0xFFFFFFFFu) ? a.out + (size_t)item.x * P1
                                         : a.partial + (size_t)item.w * P1;
#pragma unroll
    for (int l = 0; l < P1; ++l) o[l] = s_c[l][tid];
  }
}

// Items of m2l_reg_kernel.  scan[t] (t < n_targets) = items of target t in
// the low 32 bits | partial slots in the high 32 bits (0 when unsplit);
// exclusive-scanned by CUB between count and fill.
static __global__ void m2l_item_count_kernel(const uint32_t* __restrict__ weak_off, uint32_t nt,
                                             uint32_t chunk, unsigned long long* __restrict__ scan) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > nt) return;
  if (t == nt) {
    scan[t] = 0;
    return;
  }
  const uint32_t len = weak_off[t + 1] - weak_off[t];
  const uint32_t nch = len > chunk ? (len + chunk - 1) / chunk : 1u;
  scan[t] = (unsigned long long)nch | ((unsigned long long)(nch > 1 ? nch : 0) << 32);
}

static __global__ void m2l_item_fill_kernel(const uint32_t* __restrict__ weak_off, uint32_t nt,
                                            const unsigned long long* __restrict__ off,
                                            uint4* __restrict__ items,
                                            uint32_t* __restrict__ n_items) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const uint32_t w0 = weak_off[t], len = weak_off[t + 1] - w0;
  const uint32_t i0 = uint32_t(off[t]), nch = uint32_t(off[t + 1]) - i0;
  const uint32_t p0 = uint32_t(off[t] >> 32);
  for (uint32_t c = 0; c < nch; ++c) {
    const uint32_t a = w0 + uint32_t(uint64_t(len) * c / nch);
    const uint32_t b = w0 + uint32_t(uint64_t(len) * (c + 1) / nch);
    items[i0 + c] = make_uint4(t, a, b, nch > 1 ? p0 + c : 0xFFFFFFFFu);
  }
  if (t == nt - 1) *n_items = i0 + nch;
}

// out[t][l] = sum of the target's chunk partials, in chunk order
static __global__ void m2l_reduce_kernel(const unsigned long long* __restrict__ off, uint32_t nt,
                                         int P1, const double2* __restrict__ partial,
                                         double2* __restrict__ out) {
  const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= uint64_t(nt) * P1) return;
  const uint32_t t = uint32_t(g / P1);
  const int l = int(g - uint64_t(t) * P1);
  const uint32_t p0 = uint32_t(off[t] >> 32), p1 = uint32_t(off[t + 1] >> 32);
  if (p1 == p0) return;  // unsplit: written by its item
  double2 acc = make_double2(0.0, 0.0);
  for (uint32_t q = p0; q < p1; ++q) {
    const double2 v = partial[size_t(q) * P1 + l];
    acc.x += v.x;
    acc.y += v.y;
  }
  out[size_t(t) * P1 + l] = acc;
}

// Upload the binomial table of the thread kernel (this translation unit's
// constant bank) -- T is [(p+1)][(p+1)], row k, column l.
static inline cudaError_t m2l_set_const_table(const double* T, int P1, cudaStream_t s) {
  if (P1 > kM2LConstP1) return cudaSuccess;
  return cudaMemcpyToSymbolAsync(c_m2l_table, T, size_t(P1) * P1 * sizeof(double), 0,
                                 cudaMemcpyDeviceToDevice, s);
}

// Launch the M2L sums: thread-per-target for the common orders, warp kernel
// otherwise.  The constant table must have been set for a.p (thread path).
static inline bool m2l_old_kernel() {
  static const bool old = [] {
    const char* e = std::getenv("FMMCU_M2L_OLD");
    return e && e[0] == '1';
  }();
  return old;
}

// The register kernel for an order (and its CTA size), or null (the r1
// kernels then run).
using M2LKernelFn = void (*)(const M2LArgs);
template <int P1, bool HARM>
static inline M2LKernelFn m2l_reg_pick(int* tb) {
  *tb = M2LRegShape<P1>::TB;
  return m2l_reg_kernel<P1, HARM>;
}
template <bool HARM>
static inline M2LKernelFn m2l_reg_for(int P1, int* tb) {
  switch (P1) {
    case 12: return m2l_reg_pick<12, HARM>(tb);
    case 14: return m2l_reg_pick<14, HARM>(tb);
    case 16: return m2l_reg_pick<16, HARM>(tb);
    case 18: return m2l_reg_pick<18, HARM>(tb);
    case 20: return m2l_reg_pick<20, HARM>(tb);
    case 22: return m2l_reg_pick<22, HARM>(tb);
    case 25: return m2l_reg_pick<25, HARM>(tb);
    case 29: return m2l_reg_pick<29, HARM>(tb);
    default: return nullptr;
  }
}

// r1 kernels, one thread (or warp) per target: orders without a register
// kernel, and FMMCU_M2L_OLD=1 for A/B runs.  The constant table must have
// been set for a.p (thread path).
static inline void launch_m2l_targets(const M2LArgs& a, cudaStream_t s) {
  if (a.n_targets == 0) return;
  auto go = [&](auto kern, uint32_t tb) {
    kern<<<(a.n_targets + tb - 1) / tb, tb, 0, s>>>(a);
  };
  switch (a.p + 1) {
    case 12: go(m2l_thread_kernel<12>, 128); return;
    case 14: go(m2l_thread_kernel<14>, 128); return;
    case 15: go(m2l_thread_kernel<15>, 128); return;
    case 17: go(m2l_thread_kernel<17>, 128); return;
    case 18: go(m2l_thread_kernel<18>, 128); return;
    case 19: go(m2l_thread_kernel<19>, 128); return;
    case 20: go(m2l_thread_kernel<20>, 128); return;
    case 22: go(m2l_thread_kernel<22>, 64); return;
    case 25: go(m2l_thread_kernel<25>, 64); return;
    default:
      m2l_batched_kernel<<<(a.n_targets + kM2LWarps - 1) / kM2LWarps, kM2LWarps * 32, 0, s>>>(a);
  }
}

}  // namespace fmmcu
