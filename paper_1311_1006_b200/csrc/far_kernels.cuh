// fmm-b200 — device far field: P2M, M2M, L2L and L2P + assembly
// (proj/src/expansion.cpp:124-186, 271-317; engine.cpp:244-286, 316-339).
//
// These translations are cheap next to P2P and M2L (O(N p) and O(boxes p^2)),
// so they are written for exactness, not speed: every complex product and sum
// follows the reference's operation order with non-contracted __d*_rn
// intrinsics (GCC's inline complex multiply re = ac - bd, im = ad + bc; the
// reference is compiled without FMA), one warp per box, lane = coefficient
// index, partners / sources / children in the reference's ascending order.
// Power chains (t^k, s^k) are formed incrementally exactly as the reference
// does (tp *= t).  Coefficients of box g (global id = level_base + index) live
// at coef[g * (p+1) + k] as double2.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fmmcu {

__device__ __forceinline__ double2 cx_mul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cx_add(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 cx_sub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 cx_scale(double s, double2 a) {
  return make_double2(__dmul_rn(s, a.x), __dmul_rn(s, a.y));
}
__device__ __forceinline__ double2 cx_div_real(double2 a, double d) {
  return make_double2(__ddiv_rn(a.x, d), __ddiv_rn(a.y, d));
}

constexpr int kFarWarps = 4;
constexpr int kFarMaxP1 = 97;

struct FarArgs {
  int p;
  int kernel;                         // 0 harmonic, 1 log
  const double* __restrict__ binom;   // Pascal rows: binom[n * brow + k]
  int brow;
  const double2* __restrict__ center; // all levels, global box ids
  const uint32_t* __restrict__ soff_l;  // this level's point offsets [nbox + 1]
  const uint32_t* __restrict__ eoff_l;  // this level's eval offsets [nbox + 1]
  const uint32_t* __restrict__ soff_c;  // child level point offsets (M2M)
  uint32_t base;                       // global id of box 0 of this level
  uint32_t cbase;                      // ... of the child level (M2M) / parent level (L2L)
  uint32_t nbox;
  double2* __restrict__ out;           // outgoing coefficients (all levels)
  double2* __restrict__ loc;           // local coefficients (all levels)
  const double2* __restrict__ m2l;     // M2L sums per target row
  const int32_t* __restrict__ m2l_row; // global box id -> row (or -1)
};

// P2M of every finest box with sources (expansion.cpp:124-149).  Sources go
// in batches of 32: lane j forms the power chain of source j into shared
// memory (tp *= t, exactly the reference's sequence), then lane k sums
// coefficient k over the batch in ascending source order.
__global__ void __launch_bounds__(kFarWarps * 32) p2m_kernel(const FarArgs a,
                                                             const double4* __restrict__ src) {
  extern __shared__ double2 s_p2m[];  // [warps][32 sources][P1 powers] + [warps][32] strengths
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const uint32_t box = blockIdx.x * (blockDim.x >> 5) + w;
  if (box >= a.nbox) return;
  const uint32_t b = a.soff_l[box], e = a.soff_l[box + 1];
  if (b == e) return;
  const int P1 = a.p + 1;
  double2* pw = s_p2m + size_t(w) * 32 * P1;
  double2* ms = s_p2m + size_t(blockDim.x >> 5) * 32 * P1 + w * 32;
  const double2 c = a.center[a.base + box];
  double2 acc[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) acc[r] = make_double2(0.0, 0.0);
  for (uint32_t j0 = b; j0 < e; j0 += 32) {
    const uint32_t nb = min(32u, e - j0);
    __syncwarp();
    if (uint32_t(lane) < nb) {
      const double4 s4 = src[j0 + lane];
      const double2 t = cx_sub(make_double2(s4.x, s4.y), c);
      ms[lane] = make_double2(s4.z, s4.w);
      double2* my = pw + size_t(lane) * P1;
      if (a.kernel == 0) {
        double2 tp = make_double2(1.0, 0.0);
        for (int k = 0; k < P1; ++k) {
          my[k] = tp;
          tp = cx_mul(tp, t);
        }
      } else {
        double2 tp = t;
        for (int k = 1; k < P1; ++k) {
          my[k] = tp;
          tp = cx_mul(tp, t);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = r * 32 + lane;
      if (k >= P1) break;
      for (uint32_t j = 0; j < nb; ++j) {
        const double2 m = ms[j];
        if (a.kernel == 0) {
          acc[r] = cx_sub(acc[r], cx_mul(m, pw[size_t(j) * P1 + k]));
        } else if (k == 0) {
          acc[r] = cx_add(acc[r], m);
        } else {
          acc[r] = cx_sub(acc[r], cx_div_real(cx_mul(m, pw[size_t(j) * P1 + k]), double(k)));
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int k = r * 32 + lane;
    if (k < P1) a.out[size_t(a.base + box) * P1 + k] = acc[r];
  }
}

// M2M of one level (expansion.cpp:151-186, engine.cpp:266-283): parent
// coefficient l = sum over non-empty children (ascending) of
// sum_k C(l,k) s^(l-k) b_k, s = child centre - parent centre.
__global__ void __launch_bounds__(kFarWarps * 32) m2m_kernel(const FarArgs a) {
  __shared__ double2 s_pow[kFarWarps][kFarMaxP1];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const uint32_t box = blockIdx.x * kFarWarps + w;
  if (box >= a.nbox) return;
  if (a.soff_l[box] == a.soff_l[box + 1]) return;
  const int P1 = a.p + 1;
  const double2 pc = a.center[a.base + box];
  double2 acc[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) acc[r] = make_double2(0.0, 0.0);
  for (uint32_t ch = 4 * box; ch < 4 * box + 4; ++ch) {
    if (a.soff_c[ch] == a.soff_c[ch + 1]) continue;
    const uint32_t g = a.cbase + ch;
    const double2 s = cx_sub(a.center[g], pc);
    __syncwarp();
    if (lane == 0) {
      double2 v = make_double2(1.0, 0.0);
      s_pow[w][0] = v;
      for (int k = 1; k < P1; ++k) {
        v = cx_mul(v, s);
        s_pow[w][k] = v;
      }
    }
    __syncwarp();
    const double2* cc = a.out + size_t(g) * P1;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int l = r * 32 + lane;
      if (l >= P1) break;
      const double* bl = a.binom + size_t(l) * a.brow;
      double2 sh;
      if (a.kernel == 0) {
        sh = make_double2(0.0, 0.0);
        for (int k = 0; k <= l; ++k)
          sh = cx_add(sh, cx_mul(cx_scale(bl[k], s_pow[w][l - k]), cc[k]));
      } else if (l == 0) {
        sh = cc[0];
      } else {
        const double2 c0 = cc[0];
        sh = cx_div_real(cx_mul(make_double2(-c0.x, -c0.y), s_pow[w][l]), double(l));
        for (int k = 1; k <= l; ++k) {
          const double f = __dmul_rn(__ddiv_rn(double(k), double(l)), bl[k]);
          sh = cx_add(sh, cx_mul(cx_scale(f, s_pow[w][l - k]), cc[k]));
        }
      }
      acc[r] = cx_add(acc[r], sh);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int l = r * 32 + lane;
    if (l < P1) a.out[size_t(a.base + box) * P1 + l] = acc[r];
  }
}

// Local expansions of one level l >= 1 (engine.cpp:96-114): boxes with evals
// get L2L(parent local) for l >= 2 (expansion.cpp:285-296), plus the sum of
// their M2L contributions (computed by m2l_batched_kernel).
__global__ void __launch_bounds__(kFarWarps * 32) local_kernel(const FarArgs a, int level) {
  __shared__ double2 s_pow[kFarWarps][kFarMaxP1];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const uint32_t box = blockIdx.x * kFarWarps + w;
  if (box >= a.nbox) return;
  if (a.eoff_l[box] == a.eoff_l[box + 1]) return;
  const int P1 = a.p + 1;
  const uint32_t g = a.base + box;
  double2 acc[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) acc[r] = make_double2(0.0, 0.0);
  if (level >= 2) {
    const uint32_t pg = a.cbase + (box >> 2);
    const double2 s = cx_sub(a.center[g], a.center[pg]);
    if (lane == 0) {
      double2 v = make_double2(1.0, 0.0);
      s_pow[w][0] = v;
      for (int k = 1; k < P1; ++k) {
        v = cx_mul(v, s);
        s_pow[w][k] = v;
      }
    }
    __syncwarp();
    const double2* pc = a.loc + size_t(pg) * P1;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int l = r * 32 + lane;
      if (l >= P1) break;
      double2 t = make_double2(0.0, 0.0);
      for (int k = l; k < P1; ++k)
        t = cx_add(t, cx_mul(cx_scale(a.binom[size_t(k) * a.brow + l], s_pow[w][k - l]), pc[k]));
      acc[r] = cx_add(acc[r], t);
    }
  }
  const int32_t row = a.m2l_row[g];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int l = r * 32 + lane;
    if (l >= P1) break;
    if (row >= 0) acc[r] = cx_add(acc[r], a.m2l[size_t(row) * P1 + l]);
    a.loc[size_t(g) * P1 + l] = acc[r];
  }
}

// Assembly (engine.cpp:316-339): potential of permuted eval e in finest box
// t = near[e] + eval_local(local_t, y_e) (Horner, expansion.cpp:298-303),
// written to its original slot eval_perm[e].  One warp per finest box, lanes
// over its evals (the box's coefficients are read by the whole warp at once;
// a thread per eval binary-searched its box over all leaves, 18 dependent
// loads at 10M / L10).
__global__ void assemble_kernel(const FarArgs a, const double2* __restrict__ near,
                                const double2* __restrict__ evy, const uint32_t* __restrict__ eperm,
                                uint32_t n_eval, int has_local, double2* __restrict__ out) {
  (void)n_eval;
  const uint32_t box = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (box >= a.nbox) return;
  const uint32_t e0 = a.eoff_l[box], e1 = a.eoff_l[box + 1];
  const uint32_t g = a.base + box;
  const int P1 = a.p + 1;
  const double2 c = a.center[g];
  const double2* cf = a.loc + size_t(g) * P1;
  for (uint32_t e = e0 + lane; e < e1; e += 32) {
    double2 v = near[e];
    if (has_local) {
      const double2 w = cx_sub(evy[e], c);
      double2 acc = make_double2(0.0, 0.0);
      for (int k = P1 - 1; k >= 0; --k) acc = cx_add(cx_mul(acc, w), cf[k]);
      v = cx_add(v, acc);
    }
    out[eperm[e]] = v;
  }
}

// ---- permutation / packing ------------------------------------------------
// packed source records {x, y, m_re, m_im} in permuted order
__global__ void pack_sources_kernel(const double2* __restrict__ z, const double2* __restrict__ m,
                                    const uint32_t* __restrict__ perm, uint32_t n,
                                    double4* __restrict__ src) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t o = perm[i];
  const double2 zz = z[o], mm = m[o];
  src[i] = make_double4(zz.x, zz.y, mm.x, mm.y);
}

// Self layout (evals are the sources, eval order == source order): the
// packed sources and the eval arrays in one pass over the permutation (no
// inverse permutation, no second gather): evy[i] = z[perm[i]], eself[i] = i.
__global__ void pack_self_kernel(const double2* __restrict__ z, const double2* __restrict__ m,
                                 const uint32_t* __restrict__ perm, uint32_t n,
                                 double4* __restrict__ src, double2* __restrict__ evy,
                                 uint32_t* __restrict__ eself) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t o = perm[i];
  const double2 zz = z[o], mm = m[o];
  src[i] = make_double4(zz.x, zz.y, mm.x, mm.y);
  evy[i] = zz;
  eself[i] = i;
}

__global__ void inverse_perm_kernel(const uint32_t* __restrict__ perm, uint32_t n,
                                    uint32_t* __restrict__ inv) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) inv[perm[i]] = i;
}

// permuted eval positions and the permuted slot of each eval's own source
// (kNoSelf without an id); self_eval: eval i is source i.
__global__ void permute_evals_kernel(const double2* __restrict__ y, const int64_t* __restrict__ sid,
                                     int self_eval, const uint32_t* __restrict__ eperm,
                                     const uint32_t* __restrict__ inv, uint32_t n_eval,
                                     uint32_t n_src, double2* __restrict__ evy,
                                     uint32_t* __restrict__ eself) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_eval) return;
  const uint32_t o = eperm[e];
  evy[e] = y[o];
  int64_t s = -1;
  if (self_eval) s = int64_t(o);
  else if (sid) s = sid[o];
  eself[e] = (s >= 0 && s < int64_t(n_src)) ? inv[s] : 0xFFFFFFFFu;
}

}  // namespace fmmcu
