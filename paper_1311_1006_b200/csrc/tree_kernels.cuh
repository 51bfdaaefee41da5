// fmm-b200 — device pyramid build and theta connectivity, bit-exact with the
// reference build_pyramid / build_connectivity (proj/src/geometry.cpp:13-216).
//
// Pyramid (median splits, geometry.cpp:106-164).  The reference splits each
// box at the point-count median with nth_element on the key (coord, index):
// the lower half is the SET of the ceil(n/2) smallest keys, whatever order
// nth_element leaves it in.  The device keeps, per level, the sources of every
// box in two lists sorted by (x, index) and by (y, index) -- one global radix
// sort each at the start.  An x split then takes the first k entries of the
// box's x-list segment (the same set), and the y-list is stably partitioned
// by the resulting low/high flag, so both lists stay sorted inside every
// child.  Evals follow the split values ("<= split goes low") with the same
// two-list scheme; their final order inside a leaf is the original index
// order (stable_partition from the identity), as the reference's.  Box
// extents are the first/last entries of the four sorted segments, so
// make_box (geometry.cpp:69-104) needs no reduction.  Leaf-internal source
// order is the index order (geometry.cpp:156-161): one stable radix sort of
// the identity by leaf id.
//
// Connectivity (classify_level, geometry.cpp:166-207): for box a of level l
// the candidates are the children of its parent's strong partners; iterating
// the parent list ascending yields each row already sorted.  theta_criterion
// (geometry.cpp:13-19) uses std::abs(complex) (glibc cabs -> __hypot) and
// the radius is std::hypot: both run through fmm_hypot, a restatement of the
// glibc 2.39 __hypot pinned bitwise against libm (tests/test_oracle.py).
// All arithmetic uses non-contracted __d*_rn intrinsics (the reference is
// compiled for generic x86-64, no FMA).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fmmcu {

// ------------------------------------------------------------- hypot -----
__device__ __forceinline__ double fmm_hypot_kernel(double ax, double ay) {
  const double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dadd_rn(ay, ay)) {
    const double d = __dsub_rn(h, ay);
    t1 = __dmul_rn(__dsub_rn(__dadd_rn(d, d), ax), ax);
    const double u = __dsub_rn(ax, ay);
    t2 = __dmul_rn(__dsub_rn(d, __dadd_rn(u, u)), d);
  } else {
    const double d = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dadd_rn(d, d), __dsub_rn(ax, __dadd_rn(ay, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, d), ay), ay), __dmul_rn(d, d));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dadd_rn(h, h)));
}

// glibc 2.39 __hypot (x86-64, no FMA), see oracle/fmm_oracle.c orc_hypot.
__device__ __forceinline__ double fmm_hypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000ll);
    return __dadd_rn(x, y);
  }
  x = fabs(x);
  y = fabs(y);
  const double ax = y > x ? y : x;
  const double ay = y > x ? x : y;
  if (ax > 0x1p511) {
    if (__dmul_rn(ax, 0x1p-54) >= ay) return __dadd_rn(ax, ay);
    return __dmul_rn(fmm_hypot_kernel(__dmul_rn(ax, 0x1p-600), __dmul_rn(ay, 0x1p-600)), 0x1p600);
  }
  if (0x1p-459 > ay) {
    if (ax >= __dmul_rn(ay, 0x1p54)) return __dadd_rn(ax, ay);
    return __dmul_rn(fmm_hypot_kernel(__dmul_rn(ax, 0x1p600), __dmul_rn(ay, 0x1p600)), 0x1p-600);
  }
  if (__dmul_rn(ax, 0x1p-54) >= ay) return __dadd_rn(ax, ay);
  return fmm_hypot_kernel(ax, ay);
}

__global__ void hypot_batch_kernel(const double2* __restrict__ xy, uint32_t n,
                                   double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fmm_hypot(xy[i].x, xy[i].y);
}

// ------------------------------------------------------------ pyramid -----
// Radix key of a coordinate: -0.0 -> +0.0 (the reference compares values, so
// the zeros tie and fall back to the index), then IEEE bits -> unsigned order.
__device__ __forceinline__ unsigned long long coord_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(__dadd_rn(v, 0.0));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// keys of coordinate `axis` of points p[0..n), values = identity
__global__ void coord_keys_kernel(const double2* __restrict__ p, uint32_t n, int axis,
                                  unsigned long long* __restrict__ key, uint32_t* __restrict__ id) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 v = p[i];
  key[i] = coord_key(axis ? v.y : v.x);
  id[i] = i;
}

// segment of position i in offsets off[0..nseg] (off[0] = 0, off[nseg] = n).
// Median splits keep source segments balanced (sizes within one of n/nseg),
// so the proportional guess is almost always right: probe it and its
// neighbours first, then fall back to bisection (unbalanced eval segments).
__device__ __forceinline__ uint32_t seg_of(const uint32_t* __restrict__ off, uint32_t nseg,
                                           uint32_t i) {
  const uint32_t n = off[nseg];
  uint32_t g = uint32_t((uint64_t(i) * nseg) / n);
  if (g >= nseg) g = nseg - 1;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (off[g] > i) --g;
    else if (off[g + 1] <= i) ++g;
  }
  if (off[g] <= i && i < off[g + 1]) return g;  // the unique non-empty segment holding i
  uint32_t lo = 0, hi = nseg;  // off[lo] <= i < off[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ double coord(const double2* __restrict__ p, uint32_t i, int axis) {
  const double2 v = p[i];
  return axis ? v.y : v.x;
}

// One split of every segment s of a level (x split of the parents, or y
// split of the halves).  Sources: the first k = ceil(n/2) entries of the
// segment in the list sorted along `axis` go low; split value = the k-th
// coordinate, or fallback[s / fb_div] (the parent centre) for an empty
// segment (geometry.cpp:43-56).  Evals: the entries of the eval list sorted
// along `axis` with coordinate <= split form a prefix (upper bound search).
struct SplitArgs {
  const double2* __restrict__ src;   // source positions (original order)
  const double2* __restrict__ ev;    // eval positions (original order)
  const uint32_t* __restrict__ slist;  // sources sorted along axis within segments
  const uint32_t* __restrict__ elist;  // evals sorted along axis within segments
  const uint32_t* __restrict__ soff;   // [nseg + 1]
  const uint32_t* __restrict__ eoff;   // [nseg + 1]
  const double2* __restrict__ fallback;  // parent centres (level l-1)
  uint32_t fb_div;                     // segment -> parent (1 for x split, 2 for y split)
  uint32_t nseg;
  int axis;
  uint32_t* __restrict__ smid;  // [nseg] first high position
  uint32_t* __restrict__ emid;  // [nseg]
  int* __restrict__ differ;     // non-null: set when emid != smid (eval lists alias sources)
  // fused offsets (null: not written).  x split: the halves' offsets
  // [2 nseg + 1] = (off[s], mid[s]) per parent s; y split: the children's
  // offsets [2 nseg + 1] = (off[s], mid[s]) per half s (children of parent p
  // are halves 2p, 2p+1 split in two) -- child_offsets_kernel's output.
  uint32_t* __restrict__ s_out;
  uint32_t* __restrict__ e_out;
};

__global__ void split_kernel(const SplitArgs a) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.nseg) return;
  const uint32_t b = a.soff[s], e = a.soff[s + 1];
  const uint32_t n = e - b;
  const double2 fb = a.fallback[s / a.fb_div];
  double split = a.axis ? fb.y : fb.x;
  uint32_t mid = b;
  if (n > 0) {
    mid = b + (n + 1) / 2;
    split = coord(a.src, a.slist[mid - 1], a.axis);
  }
  a.smid[s] = mid;
  uint32_t lo = a.eoff[s], hi = a.eoff[s + 1];  // first entry with coord > split
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (coord(a.ev, a.elist[m], a.axis) <= split) lo = m + 1;
    else hi = m;
  }
  a.emid[s] = lo;
  if (a.differ && lo != mid) atomicOr(a.differ, 1);
  if (a.s_out) {
    a.s_out[2 * s] = b;
    a.s_out[2 * s + 1] = mid;
    if (s == a.nseg - 1) a.s_out[2 * a.nseg] = e;
  }
  if (a.e_out) {
    a.e_out[2 * s] = a.eoff[s];
    a.e_out[2 * s + 1] = lo;
    if (s == a.nseg - 1) a.e_out[2 * a.nseg] = a.eoff[a.nseg];
  }
}

// flag[id] = 1 for the entries of list that fall before mid of their segment
__global__ void low_flags_kernel(const uint32_t* __restrict__ list, uint32_t n,
                                 const uint32_t* __restrict__ off, const uint32_t* __restrict__ mid,
                                 uint32_t nseg, uint8_t* __restrict__ flag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t s = seg_of(off, nseg, i);
  flag[list[i]] = i < mid[s] ? 1 : 0;
}

__global__ void gather_flags_kernel(const uint32_t* __restrict__ list, uint32_t n,
                                    const uint8_t* __restrict__ flag, uint32_t* __restrict__ ind) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ind[i] = flag[list[i]];
}

// Stable partition of every segment of `in` by flag (low first) using the
// exclusive scan `scan` of the low indicators.
__global__ void partition_kernel(const uint32_t* __restrict__ in, uint32_t n,
                                 const uint32_t* __restrict__ off, const uint32_t* __restrict__ mid,
                                 uint32_t nseg, const uint32_t* __restrict__ ind,
                                 const uint32_t* __restrict__ scan, uint32_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t s = seg_of(off, nseg, i);
  const uint32_t b = off[s];
  const uint32_t rl = scan[i] - scan[b];
  const uint32_t dst = ind[i] ? b + rl : mid[s] + (i - b - rl);
  out[dst] = in[i];
}

// as partition_kernel, with the low indicator read from the per-id flags
__global__ void partition_flags_kernel(const uint32_t* __restrict__ in, uint32_t n,
                                       const uint32_t* __restrict__ off,
                                       const uint32_t* __restrict__ mid, uint32_t nseg,
                                       const uint8_t* __restrict__ flag,
                                       const uint32_t* __restrict__ scan,
                                       uint32_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t id = in[i];
  const uint32_t s = seg_of(off, nseg, i);
  const uint32_t b = off[s];
  const uint32_t rl = scan[i] - scan[b];
  const uint32_t dst = flag[id] ? b + rl : mid[s] + (i - b - rl);
  out[dst] = id;
}

// Offsets of the children after both splits: per parent p,
// [off[p], ymid[2p]) [ymid[2p], xmid[p]) [xmid[p], ymid[2p+1]) [ymid[2p+1], off[p+1]).
__global__ void child_offsets_kernel(const uint32_t* __restrict__ off,
                                     const uint32_t* __restrict__ xmid,
                                     const uint32_t* __restrict__ ymid, uint32_t np,
                                     uint32_t* __restrict__ half_off, uint32_t* __restrict__ coff) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  if (half_off) {
    half_off[2 * p] = off[p];
    half_off[2 * p + 1] = xmid[p];
    if (p == np - 1) half_off[2 * np] = off[np];
  }
  if (coff) {
    coff[4 * p + 0] = off[p];
    coff[4 * p + 1] = ymid[2 * p];
    coff[4 * p + 2] = xmid[p];
    coff[4 * p + 3] = ymid[2 * p + 1];
    if (p == np - 1) coff[4 * np] = off[np];
  }
}

// make_box (geometry.cpp:69-104) from the first/last entries of the sorted
// segments; empty boxes sit at the parent centre with zero extent.
struct BoxArgs {
  const double2* __restrict__ src;
  const double2* __restrict__ ev;
  const uint32_t* __restrict__ sx;
  const uint32_t* __restrict__ sy;
  const uint32_t* __restrict__ ex;
  const uint32_t* __restrict__ ey;
  const uint32_t* __restrict__ soff;
  const uint32_t* __restrict__ eoff;
  const double2* __restrict__ parent_center;  // null at level 0
  uint32_t nbox;
  double2* __restrict__ center;
  double* __restrict__ hw;
  double* __restrict__ hh;
  double* __restrict__ radius;
};

__device__ __forceinline__ double dmin(double acc, double v) { return v < acc ? v : acc; }
__device__ __forceinline__ double dmax(double acc, double v) { return acc < v ? v : acc; }

__global__ void box_geometry_kernel(const BoxArgs a) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nbox) return;
  const uint32_t sb = a.soff[i], se = a.soff[i + 1], eb = a.eoff[i], ee = a.eoff[i + 1];
  if (sb == se && eb == ee) {
    a.center[i] = a.parent_center ? a.parent_center[i >> 2] : make_double2(0.0, 0.0);
    a.hw[i] = 0.0;
    a.hh[i] = 0.0;
    a.radius[i] = 0.0;
    return;
  }
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double xmin = inf, xmax = -inf, ymin = inf, ymax = -inf;
  if (se > sb) {
    xmin = dmin(xmin, a.src[a.sx[sb]].x);
    xmax = dmax(xmax, a.src[a.sx[se - 1]].x);
    ymin = dmin(ymin, a.src[a.sy[sb]].y);
    ymax = dmax(ymax, a.src[a.sy[se - 1]].y);
  }
  if (ee > eb) {
    xmin = dmin(xmin, a.ev[a.ex[eb]].x);
    xmax = dmax(xmax, a.ev[a.ex[ee - 1]].x);
    ymin = dmin(ymin, a.ev[a.ey[eb]].y);
    ymax = dmax(ymax, a.ev[a.ey[ee - 1]].y);
  }
  a.center[i] = make_double2(__dmul_rn(0.5, __dadd_rn(xmin, xmax)),
                             __dmul_rn(0.5, __dadd_rn(ymin, ymax)));
  const double w = __dmul_rn(0.5, __dsub_rn(xmax, xmin));
  const double h = __dmul_rn(0.5, __dsub_rn(ymax, ymin));
  a.hw[i] = w;
  a.hh[i] = h;
  a.radius[i] = fmm_hypot(w, h);
}

// leaf id of every list entry, scattered to the entry's original index
__global__ void leaf_of_kernel(const uint32_t* __restrict__ list, uint32_t n,
                               const uint32_t* __restrict__ off, uint32_t nseg,
                               uint32_t* __restrict__ leaf_of) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) leaf_of[list[i]] = seg_of(off, nseg, i);
}

// ------------------------------------------------------- connectivity -----
// The reference's theta criterion (geometry.cpp:13-19):
//   max(ra, rb) + theta * min(ra, rb) <= theta * |ca - cb|,  |.| = glibc hypot
__device__ __forceinline__ bool theta_weak_exact(double big, double small, double dx, double dy,
                                                 double theta) {
  const double d = fmm_hypot(dx, dy);
  return __dadd_rn(big, __dmul_rn(theta, small)) <= __dmul_rn(theta, d);
}

// Same decision, bit for bit, at a fraction of the cost: a single-precision
// square root of dx^2 + dy^2 (relative error < 3e-7) settles every candidate
// whose two sides differ by more than 1e-6 relative; only the band around
// equality (and out-of-range magnitudes) runs the restated glibc hypot.
// Soundness: with l = big + theta*small as rounded above, D = |(dx, dy)|
// exactly and a = the fast root, theta*hypot(dx, dy) as rounded lies in
// theta*D*(1 +- 4e-16) while a lies in D*(1 +- 3e-7); so l < theta*a*(1-1e-6)
// implies l <= theta (x) hypot, and l > theta*a*(1+1e-6) implies the
// opposite.
__device__ __forceinline__ bool theta_weak(const double2* __restrict__ c,
                                           const double* __restrict__ r, uint32_t a, uint32_t b,
                                           double theta) {
  const double ra = r[a], rb = r[b];
  const double big = ra < rb ? rb : ra;    // std::max
  const double small = rb < ra ? rb : ra;  // std::min
  const double2 ca = c[a], cb = c[b];
  const double dx = __dsub_rn(ca.x, cb.x), dy = __dsub_rn(ca.y, cb.y);
  const double l = __dadd_rn(big, __dmul_rn(theta, small));
  const double d2 = dx * dx + dy * dy;
  if (d2 > 1e-30 && d2 < 1e30) {
    const double ta = theta * double(sqrtf(float(d2)));
    if (l < ta * (1.0 - 1e-6)) return true;
    if (l > ta * (1.0 + 1e-6)) return false;
  }
  return theta_weak_exact(big, small, dx, dy, theta);
}

// One warp per box a: its candidates are the children 4pq..4pq+3 of its
// parent's strong partners pq, in ascending order (so every row comes out
// sorted, as the reference's); 32 candidates per step, classified by the
// lanes, compacted in order by ballots.  Pass 1 (fill == false) counts;
// pass 2 writes the rows at the scanned offsets.  (A thread per box walked a
// clustered box's thousands of candidates serially: 9 ms of the 1M gauss8
// pipeline.)
template <bool FILL>
__global__ void classify_kernel(const uint32_t* __restrict__ ps_off,
                                const uint32_t* __restrict__ ps_idx, const double2* __restrict__ c,
                                const double* __restrict__ r, uint32_t nbox, double theta,
                                uint32_t* __restrict__ s_cnt, uint32_t* __restrict__ w_cnt,
                                const uint32_t* __restrict__ s_off, const uint32_t* __restrict__ w_off,
                                uint32_t* __restrict__ s_idx, uint32_t* __restrict__ w_idx,
                                uint32_t s_cap = 0xFFFFFFFFu, uint32_t w_cap = 0xFFFFFFFFu,
                                int* __restrict__ overflow = nullptr) {
  const uint32_t a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (a >= nbox) return;  // warp-uniform
  if (!FILL && a == 0 && lane == 0) {  // the exclusive scans' end entries
    s_cnt[nbox] = 0;
    w_cnt[nbox] = 0;
  }
  if (overflow && *overflow) return;  // a coarser level did not fit: lists are invalid
  const uint32_t p = a >> 2;
  uint32_t so = FILL ? s_off[a] : 0, wo = FILL ? w_off[a] : 0;
  // capacity guard: the lists may be filled into buffers sized by a guess
  // before the host has read the counts (a miss is flagged and redone)
  if (FILL && overflow && (uint64_t(s_off[a + 1]) > s_cap || uint64_t(w_off[a + 1]) > w_cap)) {
    if (lane == 0) *overflow = 1;
    return;
  }
  const uint32_t q0 = ps_off[p];
  const uint32_t ncand = 4 * (ps_off[p + 1] - q0);
  const unsigned below = (1u << lane) - 1u;
  uint32_t ns = 0, nw = 0;
  for (uint32_t k0 = 0; k0 < ncand; k0 += 32) {
    const uint32_t k = k0 + lane;
    const bool valid = k < ncand;
    const uint32_t b = valid ? 4 * ps_idx[q0 + (k >> 2)] + (k & 3u) : 0u;
    const bool weak = valid && a != b && theta_weak(c, r, a, b, theta);
    const unsigned mw = __ballot_sync(0xffffffffu, valid && weak);
    const unsigned ms = __ballot_sync(0xffffffffu, valid && !weak);
    if (FILL && valid) {
      if (weak) w_idx[wo + nw + __popc(mw & below)] = b;
      else s_idx[so + ns + __popc(ms & below)] = b;
    }
    nw += __popc(mw);
    ns += __popc(ms);
  }
  if (!FILL && lane == 0) {
    s_cnt[a] = ns;
    w_cnt[a] = nw;
  }
}

}  // namespace fmmcu
