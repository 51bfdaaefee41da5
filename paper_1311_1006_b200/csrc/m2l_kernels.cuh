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
#include <cuda_runtime.h>

namespace fmmcu {

struct M2LArgs {
  int p;
  int kernel;
  const double2* __restrict__ centers;
  const double2* __restrict__ coeffs;  // [n_boxes][p+1]
  const uint32_t* __restrict__ target_box;
  const uint32_t* __restrict__ weak_off;
  const uint32_t* __restrict__ weak_idx;
  const double* __restrict__ table;  // [(p+1)][(p+1)]: T[k][l]
  uint32_t n_targets;
  double big_w2;                     // |w|^2 threshold of the overflow-safe branch
  double2* __restrict__ out;         // [n_targets][p+1]
  int* __restrict__ singular;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

__device__ __forceinline__ double2 shfl_up2(double2 v, int d) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

constexpr int kM2LWarps = 4;
constexpr int kM2LMaxP = 96;

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

// Upload the binomial table of the thread kernel (this translation unit's
// constant bank) -- T is [(p+1)][(p+1)], row k, column l.
static inline cudaError_t m2l_set_const_table(const double* T, int P1, cudaStream_t s) {
  if (P1 > kM2LConstP1) return cudaSuccess;
  return cudaMemcpyToSymbolAsync(c_m2l_table, T, size_t(P1) * P1 * sizeof(double), 0,
                                 cudaMemcpyDeviceToDevice, s);
}

// Launch the M2L sums: thread-per-target for the common orders, warp kernel
// otherwise.  The constant table must have been set for a.p (thread path).
static inline void launch_m2l(const M2LArgs& a, cudaStream_t s) {
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
