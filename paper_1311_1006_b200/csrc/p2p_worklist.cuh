// fmm-b200 — the P2P work list built on the device.
//
// The near-field kernels consume work items (an eval block of one target
// leaf x a run of its strong list, see P2PItem) and, for leaves whose pair
// work exceeds a budget, partial-sum slots reduced by p2p_finalize_kernel.
// r1 built that list on the host from a host copy of the finest CSR
// (build_worklist, fmmcu.cu): ~1.5 ms of host time at 10M leaves' worth of
// strong lists, on the critical path of the reference-facing launch and,
// after a CSR download, of the device pipeline.  Here the same list -- the
// same items in the same order -- comes from kernels over the device CSR
// (the loop being replaced is the leaf loop of nearfield_run,
// proj/src/backend.cpp:73-89, cut into items):
//
//   (p2p_segments_kernel, run table seg[q] = (first slot, n) per strong entry)
//   wl_leaf_kernel     per leaf: S (sources of its strong list), the last
//                      source slot it reads (-> upload group), pair work, and
//                      the integer lane-cost model of E = 4 / 5 evals per lane
//   (CUB sum)          total pair work -> split budget
//   wl_setup_kernel    E, max_ev and the budget into the device header
//   (CUB radix sort)   leaves stably ordered by group (5-bit key)
//   wl_count_kernel    items / finals / partial evals per leaf, sorted order
//   (CUB scans)        their offsets
//   wl_bounds_kernel   per-group item and final ranges into the header
//   -- one small D2H of the header; the host sizes the buffers --
//   wl_fill_kernel     the items and finals at their offsets
//
// Every count is an integer, so the list is identical run to run (the E
// choice included) and identical to the host builder's.
//
// One warp per leaf, reading the run table coalesced: a clustered tree has
// strong lists of thousands of entries, and one thread walking such a list
// through dependent pt_off[s_idx[q]] gathers took milliseconds (1M gauss8,
// L = 8: 3 ms over the host builder).  The greedy strong-list chunking of a
// split block becomes a warp scan + ballot per chunk of <= 32 entries.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "p2p_kernels.cuh"
#include "p2p_sym.cuh"
#include "p2p_warp.cuh"
#include "p2p_worklist_types.cuh"

namespace fmmcu {

__device__ __forceinline__ unsigned long long wl_lane_cost(uint32_t ntl, unsigned long long S,
                                                           uint32_t E) {
  if (!ntl || !S) return 0ull;
  const uint32_t max_ev = kWarpSlots * E;
  const uint32_t nblk = (ntl + max_ev - 1) / max_ev;
  const uint32_t nt = (ntl + nblk - 1) / nblk;
  const uint32_t G = (nt + E - 1) / E;
  const uint32_t K = 32 / G;
  return (unsigned long long)nblk * E * ((S + K - 1) / K);
}

constexpr unsigned kFull = 0xffffffffu;

// Over every leaf of the job (the E choice and the split budget are
// whole-job quantities, as in the host builder, so a shard's items equal the
// full job's items of its leaves); key / val / S only for leaves in [lb, le).
// One warp per leaf.
static __global__ void wl_leaf_kernel(const uint32_t* __restrict__ pt_off,
                                      const uint32_t* __restrict__ ev_off,
                                      const uint32_t* __restrict__ s_off,
                                      const uint2* __restrict__ seg, uint32_t nl, uint32_t lb,
                                      uint32_t le, const WlGroups g, uint32_t* __restrict__ key,
                                      uint32_t* __restrict__ val,
                                      unsigned long long* __restrict__ S_out,
                                      unsigned long long* __restrict__ work,
                                      WlHead* __restrict__ head) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned long long c4 = 0, c5 = 0;
  if (t < nl) {
    unsigned long long S = 0;
    uint32_t need = lane == 0 ? pt_off[t + 1] : 0u;
    for (uint32_t q = s_off[t] + lane; q < s_off[t + 1]; q += 32) {
      const uint2 r = seg[q];
      S += r.y;
      need = max(need, r.x + r.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      S += __shfl_xor_sync(kFull, S, o);
      need = max(need, __shfl_xor_sync(kFull, need, o));
    }
    if (lane == 0) {
      const uint32_t ntl = ev_off[t + 1] - ev_off[t];
      work[t] = (unsigned long long)ntl * S;
      c4 = wl_lane_cost(ntl, S, 4);
      c5 = wl_lane_cost(ntl, S, 5);
      if (t >= lb && t < le) {
        uint32_t k = 0;
        while (k + 1 < g.K && g.slot_end[k] < need) ++k;
        const uint32_t i = t - lb;
        key[i] = k;
        val[i] = i;
        S_out[i] = S;
      }
    }
  }
  // integer sums over the block's leaves: the E choice does not depend on
  // the summation order
  __shared__ unsigned long long s4[8], s5[8];
  const uint32_t w = threadIdx.x >> 5;
  if (lane == 0) {
    s4[w] = c4;
    s5[w] = c5;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a4 = 0, a5 = 0;
    for (uint32_t i = 0; i < (blockDim.x >> 5); ++i) {
      a4 += s4[i];
      a5 += s5[i];
    }
    if (a4 | a5) {
      atomicAdd(&head->cost4, a4);
      atomicAdd(&head->cost5, a5);
    }
  }
}

// force_e: 0 = model, else 4 / 5 (FMMCU_P2P_E)
static __global__ void wl_setup_kernel(WlHead* head, int force_e) {
  const uint32_t E = force_e == 4 || force_e == 5 ? uint32_t(force_e)
                                                 : (head->cost5 < head->cost4 ? 5u : 4u);
  head->E = E;
  head->max_ev = kWarpSlots * E;
  const unsigned long long b = head->total_work / (148ull * 16ull);
  head->budget = b > (1ull << 16) ? b : (1ull << 16);
}

// Items of leaf t, by the whole warp (the host builder's leaf_items,
// fmmcu.cu): eval blocks of <= max_ev evals, balanced; a block whose pair
// work exceeds the budget (and has > 1 strong entry), or whose list exceeds
// 32 entries, is cut greedily into strong-list chunks -- entries are added
// while the chunk is still empty of sources or stays within budget / nt
// sources, at most 32 per chunk -- with partial slots summed by
// p2p_finalize_kernel.  Lane 0 writes; counts only when it/fin are null.
// Returns the counts in every lane.
__device__ __forceinline__ void wl_leaf_items(uint32_t t, const uint32_t* __restrict__ ev_off,
                                              const uint32_t* __restrict__ s_off,
                                              const uint2* __restrict__ seg,
                                              unsigned long long S, uint32_t max_ev,
                                              unsigned long long budget, P2PItem* it,
                                              P2PFinal* fin, uint32_t pbase, uint32_t& n_items,
                                              uint32_t& n_fins, uint32_t& n_pev) {
  const uint32_t lane = threadIdx.x & 31;
  n_items = n_fins = n_pev = 0;
  const uint32_t ntl = ev_off[t + 1] - ev_off[t];
  const uint32_t sb0 = s_off[t], sb1 = s_off[t + 1];
  const uint32_t nblk = (ntl + max_ev - 1) / max_ev;
  for (uint32_t b = 0, e0 = 0; b < nblk; ++b) {
    const uint32_t nt = (ntl - e0) / (nblk - b) + ((ntl - e0) % (nblk - b) ? 1u : 0u);
    const uint32_t evb = ev_off[t] + e0;
    e0 += nt;
    const unsigned long long pairs = (unsigned long long)nt * S;
    if ((pairs <= budget || sb1 - sb0 <= 1) && sb1 - sb0 <= uint32_t(kWarpMaxEntries) &&
        S <= 0xFFFFFFFFull) {
      if (it && lane == 0) it[n_items] = P2PItem{t, evb, nt, sb0, sb1, uint32_t(S), kNoSelf, 0};
      ++n_items;
      continue;
    }
    const unsigned long long spc = budget / nt > 0 ? budget / nt : 1ull;
    const uint32_t base = pbase + n_pev;
    uint32_t n_chunks = 0;
    // The entries' source counts sit in a 96-entry window in registers
    // (lane-distributed thirds [wq, wq+32), [wq+32, wq+64), [wq+64, wq+96)),
    // refilled a third ahead, so a step of this sequential greedy waits on
    // shuffles, not on a global load (clustered leaves run ~750 steps)
    uint32_t wq = sb0;
    auto ld = [&](uint32_t from) -> uint32_t {
      const uint32_t qq = from + lane;
      return qq < sb1 ? seg[qq].y : 0u;
    };
    uint32_t w0 = ld(wq), w1 = ld(wq + 32), w2 = ld(wq + 64);
    for (uint32_t q = sb0; q < sb1;) {
      const uint32_t qq = q + lane;
      const uint32_t d = q - wq;  // < 32
      const uint32_t from = (d + lane) & 31u;
      const uint32_t a0 = __shfl_sync(kFull, w0, from), a1 = __shfl_sync(kFull, w1, from);
      const unsigned long long n = qq < sb1 ? (d + lane < 32 ? a0 : a1) : 0ull;
      unsigned long long incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(kFull, incl, o);
        if (lane >= uint32_t(o)) incl += v;
      }
      // the lanes taken form a prefix: the chunk is empty of sources before
      // the entry, or the entry keeps it within spc sources
      const bool take = qq < sb1 && (incl - n == 0 || incl <= spc);
      const uint32_t len = __popc(__ballot_sync(kFull, take));  // >= 1: lane 0 always takes
      const unsigned long long acc = __shfl_sync(kFull, incl, len - 1);
      if (it && lane == 0)
        it[n_items] = P2PItem{t, evb, nt, q, q + len, uint32_t(acc), pbase + n_pev, 0};
      ++n_items;
      n_pev += nt;
      ++n_chunks;
      q += len;
      if (q - wq >= 32) {  // slide the window by a third
        w0 = w1;
        w1 = w2;
        wq += 32;
        w2 = ld(wq + 64);
      }
    }
    if (fin && lane == 0) fin[n_fins] = P2PFinal{evb, nt, base, n_chunks};
    ++n_fins;
  }
}

// counts in sorted (group) order: cnt[pos] = {items, fins, pevals}; one warp
// per position
static __global__ void wl_count_kernel(const uint32_t* __restrict__ ev_off,
                                       const uint32_t* __restrict__ s_off,
                                       const uint2* __restrict__ seg, uint32_t lb, uint32_t np,
                                       const uint32_t* __restrict__ val_sorted,
                                       const unsigned long long* __restrict__ S,
                                       const WlHead* __restrict__ head,
                                       uint32_t* __restrict__ ci, uint32_t* __restrict__ cf,
                                       uint32_t* __restrict__ cp) {
  const uint32_t pos = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (pos > np) return;
  if (pos == np) {  // the exclusive scans run over np + 1 entries
    if (lane == 0) ci[np] = cf[np] = cp[np] = 0;
    return;
  }
  const uint32_t i = val_sorted[pos];
  uint32_t a, b, c;
  wl_leaf_items(lb + i, ev_off, s_off, seg, S[i], head->max_ev, head->budget, nullptr, nullptr, 0,
                a, b, c);
  if (lane == 0) {
    ci[pos] = a;
    cf[pos] = b;
    cp[pos] = c;
  }
}

// group k = sorted positions [grp_pos[k], grp_pos[k+1]); header ranges
static __global__ void wl_bounds_kernel(const uint32_t* __restrict__ key_sorted, uint32_t np,
                                        uint32_t K, const uint32_t* __restrict__ io,
                                        const uint32_t* __restrict__ fo,
                                        const uint32_t* __restrict__ po, WlHead* __restrict__ head) {
  const uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos > np) return;
  // groups starting at pos: (key[pos-1], key[pos]]  (pos == np closes the rest)
  const int k0 = pos == 0 ? -1 : int(key_sorted[pos - 1]);
  const int k1 = pos == np ? int(K) : int(key_sorted[pos]);
  for (int k = k0 + 1; k <= k1; ++k) {
    head->grp_item[k] = io[pos];
    head->grp_fin[k] = fo[pos];
  }
  if (pos == np) {
    head->n_items = io[np];
    head->n_fins = fo[np];
    head->n_pevals = po[np];
  }
}

// one warp per position
static __global__ void wl_fill_kernel(const uint32_t* __restrict__ ev_off,
                                      const uint32_t* __restrict__ s_off,
                                      const uint2* __restrict__ seg, uint32_t lb, uint32_t np,
                                      const uint32_t* __restrict__ val_sorted,
                                      const unsigned long long* __restrict__ S,
                                      const WlHead* __restrict__ head,
                                      const uint32_t* __restrict__ io,
                                      const uint32_t* __restrict__ fo,
                                      const uint32_t* __restrict__ po, P2PItem* __restrict__ items,
                                      P2PFinal* __restrict__ fins) {
  const uint32_t pos = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (pos >= np) return;
  const uint32_t i = val_sorted[pos];
  uint32_t a, b, c;
  wl_leaf_items(lb + i, ev_off, s_off, seg, S[i], head->max_ev, head->budget, items + io[pos],
                fins + fo[pos], po[pos], a, b, c);
}

// Grouped symmetric list: per upload group k, its first item and first leaf
// position (positions in group order), from the sorted group keys.
static __global__ void wls_bounds_kernel(const uint32_t* __restrict__ key_sorted, uint32_t np,
                                         uint32_t K, const uint32_t* __restrict__ blk,
                                         WlHead* __restrict__ head) {
  const uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos > np) return;
  const int k0 = pos == 0 ? -1 : int(key_sorted[pos - 1]);
  const int k1 = pos == np ? int(K) : int(key_sorted[pos]);
  for (int k = k0 + 1; k <= k1; ++k) {
    head->grp_item[k] = blk[pos];
    head->grp_fin[k] = pos;
  }
}

// ---------------------------------------------------------------------------
// Symmetric (mutual-kernel) work list on the device: the host builder
// build_sym_worklist (fmmcu.cu) restated as kernels, same entries, items and
// contribution slots.  Item = eval block of leaf t; its entries are t's
// strong partners B outside the range or B >= t, ordered runs (B == t is
// the self run) first, then the symmetric ones (B > t inside the range),
// each in strong-list order.  Partners B < t inside the range are skipped:
// B's items cover the pair.  One warp per leaf.

struct WlSymHead {
  unsigned long long ent, items, slots;  // totals (from the scans)
  uint32_t bad;                          // a leaf does not qualify
  uint32_t pad;
  unsigned long long ncl;  // contribution-list entries: sum of eval blocks x symmetric entries
};

static __global__ void wls_count_kernel(const uint32_t* __restrict__ ev_off,
                                        const uint32_t* __restrict__ s_off,
                                        const uint32_t* __restrict__ s_idx,
                                        const uint2* __restrict__ seg, uint32_t lb, uint32_t le,
                                        const WlHead* __restrict__ head,
                                        uint32_t* __restrict__ n_ent, uint32_t* __restrict__ n_blk,
                                        unsigned long long* __restrict__ ssym,
                                        unsigned long long* __restrict__ sord,
                                        unsigned long long* __restrict__ n_slot,
                                        WlSymHead* __restrict__ sh,
                                        const uint32_t* __restrict__ grp,
                                        const uint32_t* __restrict__ order) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // output position
  const uint32_t np = le - lb;
  if (p > np) return;
  if (p == np) {  // the exclusive scans run over np + 1 entries
    if (lane == 0) n_ent[np] = n_blk[np] = 0, n_slot[np] = 0ull;
    return;
  }
  const uint32_t i = order ? order[p] : p;  // grouped: positions in group order
  const uint32_t t = lb + i;
  uint32_t n = 0, nsym = 0;
  unsigned long long so = 0, ss = 0;
  for (uint32_t q = s_off[t] + lane; q < s_off[t + 1]; q += 32) {
    const uint32_t B = s_idx[q];
    // grouped: symmetric only inside the upload group
    const bool inr = B >= lb && B < le && (!grp || grp[B - lb] == grp[i]);
    if (inr && B < t) continue;
    ++n;
    if (inr && B > t) {
      ss += seg[q].y;
      ++nsym;
    } else {
      so += seg[q].y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n += __shfl_xor_sync(kFull, n, o);
    nsym += __shfl_xor_sync(kFull, nsym, o);
    so += __shfl_xor_sync(kFull, so, o);
    ss += __shfl_xor_sync(kFull, ss, o);
  }
  if (lane == 0) {
    const uint32_t max_ev = head->max_ev;
    const uint32_t ntl = ev_off[t + 1] - ev_off[t];
    const uint32_t nb = ntl ? (ntl + max_ev - 1) / max_ev : 0u;
    if (n > uint32_t(kSymMaxEntries) || so + ss >= (1ull << 31)) atomicOr(&sh->bad, 1u);
    else if (n > uint32_t(kWarpMaxEntries)) atomicOr(&sh->bad, 2u);  // needs entry rounds
    n_ent[p] = n;
    n_blk[p] = nb;
    ssym[p] = ss;
    sord[p] = so;
    n_slot[p] = (unsigned long long)nb * ss;
    // each symmetric entry B of t puts t's nb eval blocks on B's list
    if (nsym && nb) atomicAdd(&sh->ncl, (unsigned long long)nb * nsym);
  }
}

static __global__ void wls_fill_kernel(const uint32_t* __restrict__ pt_off,
                                       const uint32_t* __restrict__ ev_off,
                                       const uint32_t* __restrict__ s_off,
                                       const uint32_t* __restrict__ s_idx,
                                       const uint2* __restrict__ seg, uint32_t lb, uint32_t le,
                                       const WlHead* __restrict__ head,
                                       const uint32_t* __restrict__ ent,
                                       const uint32_t* __restrict__ blk,
                                       const unsigned long long* __restrict__ ssym,
                                       const unsigned long long* __restrict__ sord,
                                       const unsigned long long* __restrict__ slots,
                                       uint4* __restrict__ sym_seg, P2PItem* __restrict__ items,
                                       uint4* __restrict__ sym_info,
                                       const uint32_t* __restrict__ grp,
                                       const uint32_t* __restrict__ order,
                                       uint2* __restrict__ sym_cnt) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // position
  const uint32_t np = le - lb;
  if (p > np) return;
  if (p == np) {
    if (lane == 0 && !order) sym_info[np] = make_uint4(ent[np], blk[np], uint32_t(slots[np]), 0u);
    return;
  }
  const uint32_t i = order ? order[p] : p;
  const uint32_t t = lb + i;
  const unsigned below = (1u << lane) - 1u;
  // entries: ordered runs first, then symmetric, each in strong-list order
  uint32_t o = ent[p];
  for (int pass = 0; pass < 2; ++pass) {
    for (uint32_t q0 = s_off[t]; q0 < s_off[t + 1]; q0 += 32) {
      const uint32_t q = q0 + lane;
      bool take = false;
      uint32_t kind = kRunOrdered, B = 0;
      if (q < s_off[t + 1]) {
        B = s_idx[q];
        const bool inr = B >= lb && B < le && (!grp || grp[B - lb] == grp[i]);
        const bool sym = inr && B > t;
        take = !(inr && B < t) && (sym == (pass == 1));
        kind = sym ? kRunSym : (B == t ? kRunSelf : kRunOrdered);
      }
      const unsigned m = __ballot_sync(kFull, take);
      if (take) {
        const uint2 r = seg[q];
        sym_seg[o + __popc(m & below)] = make_uint4(r.x, r.y, kind, 0u);
      }
      o += __popc(m);
    }
  }
  if (lane == 0) {
    const uint32_t ntl = ev_off[t + 1] - ev_off[t];
    const uint32_t nb = blk[p + 1] - blk[p];
    const unsigned long long ss = ssym[p], so = sord[p];
    for (uint32_t b = 0, e0 = 0; b < nb; ++b) {
      const uint32_t nt = (ntl - e0) / (nb - b) + ((ntl - e0) % (nb - b) ? 1u : 0u);
      items[blk[p] + b] = P2PItem{t, ev_off[t] + e0, nt, ent[p], ent[p + 1], uint32_t(so + ss),
                                  uint32_t(slots[p] + (unsigned long long)b * ss), uint32_t(so)};
      e0 += nt;
    }
    // per leaf (leaf order): first entry / item / slot, symmetric sources;
    // grouped lists also need the counts (consecutive leaves are not
    // consecutive positions)
    sym_info[i] = make_uint4(ent[p], blk[p], uint32_t(slots[p]), uint32_t(ss));
    if (sym_cnt) sym_cnt[i] = make_uint2(ent[p + 1] - ent[p], nb);
  }
  (void)pt_off;
  (void)head;
}

}  // namespace fmmcu
