// fmm-b200 — host driver of the device-built P2P work list (p2p_worklist.cuh).
//
// The job's finest CSR is already on the device (c->d_pt, d_ev, d_soff,
// d_sidx).  The kernels derive the same items / finals as the host builder
// (build_worklist, fmmcu.cu) over the leaf range [lb, le), grouped by upload
// chunk when g.K > 1; one ~400-byte header read sizes the item, final and
// partial buffers.  The loop being cut into items is the leaf loop of the
// reference nearfield_run (proj/src/backend.cpp:73-89).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <cstdlib>
#include <functional>

#include "fmmcu_internal.cuh"
#include "p2p_worklist.cuh"

namespace fmmcu::detail {

namespace {
inline uint32_t nblocks(uint64_t n, uint32_t tb) { return uint32_t((n + tb - 1) / tb); }
}  // namespace

// Shared first half of both device builders: the run table, the per-leaf
// sums over every leaf of the job (keys / S for [lb, le)), the total pair
// work, and E / max_ev / the split budget in the header.  nk counts launches.
int wl_prepare(fmmcu_ctx* c, uint32_t lb, uint32_t le, const WlGroups& g, cudaStream_t s,
               int& nk, size_t& need) {

  const uint32_t np = le - lb;
  const uint32_t nl = c->n_leaves;
  const uint32_t K = g.K ? g.K : 1u;
  if (K > uint32_t(kWlMaxGroups)) return set_err(c, FMMCU_EINVAL, "too many upload groups");
  if (lb > le || le > nl) return set_err(c, FMMCU_EINVAL, "leaf range outside the job");
  CU_TRY(c, c->d_wl_head.ensure(sizeof(WlHead)));
  CU_TRY(c, c->h_wl_head.ensure(sizeof(WlHead)));
  const size_t n1 = size_t(np) + 1;
  CU_TRY(c, c->d_wl_key.ensure(n1 * 8));
  CU_TRY(c, c->d_wl_val.ensure(n1 * 8));
  CU_TRY(c, c->d_wl_S.ensure(n1 * 8));
  CU_TRY(c, c->d_wl_work.ensure((size_t(nl) + 1) * 8));
  CU_TRY(c, c->d_wl_cnt.ensure(n1 * 12));
  CU_TRY(c, c->d_wl_off.ensure(n1 * 12));
  WlHead* head = c->d_wl_head.as<WlHead>();
  uint32_t* key = c->d_wl_key.as<uint32_t>();
  uint32_t* key2 = key + n1;
  uint32_t* val = c->d_wl_val.as<uint32_t>();
  uint32_t* val2 = val + n1;
  auto* S = c->d_wl_S.as<unsigned long long>();
  auto* work = c->d_wl_work.as<unsigned long long>();
  uint32_t* ci = c->d_wl_cnt.as<uint32_t>();
  uint32_t* io = c->d_wl_off.as<uint32_t>();
  CU_TRY(c, cudaMemsetAsync(head, 0, sizeof(WlHead), s));
  const uint32_t* pt = c->d_pt.as<uint32_t>();
  const uint32_t* ev = c->d_ev.as<uint32_t>();
  const uint32_t* so = c->d_soff.as<uint32_t>();
  const uint32_t* si = c->d_sidx.as<uint32_t>();
  // run table first: the work-list kernels read it coalesced
  const uint32_t nnz = c->n_strong;
  CU_TRY(c, c->d_seg.ensure(size_t(std::max(nnz, 1u)) * 8));
  const uint2* seg = c->d_seg.as<uint2>();
  if (nnz) {
    p2p_segments_kernel<<<nblocks(nnz, 256), 256, 0, s>>>(si, pt, nnz, c->d_seg.as<uint2>());
    ++nk;
  }
  if (nl) {
    wl_leaf_kernel<<<nblocks(uint64_t(nl) * 32, 256), 256, 0, s>>>(pt, ev, so, seg, nl, lb, le, g,
                                                                  key, val, S, work, head);
    ++nk;
  }
  // pair work of the whole job (split budget) and of the range (pair count);
  // integer sums: order-independent
  size_t tb = 0;
  need = 0;
  CU_TRY(c, cub::DeviceReduce::Sum(nullptr, tb, work, &head->total_work, int64_t(nl), s));
  need = tb;
  CU_TRY(c, cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, val, val2, int64_t(np), 0, 5,
                                            s));
  need = std::max(need, tb);
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(nullptr, tb, ci, io, int64_t(n1), s));
  need = std::max(need, tb);
  CU_TRY(c, c->d_cubtmp.ensure(need));
  tb = need;
  CU_TRY(c, cub::DeviceReduce::Sum(c->d_cubtmp.p, tb, work, &head->total_work, int64_t(nl), s));
  tb = need;
  CU_TRY(c, cub::DeviceReduce::Sum(c->d_cubtmp.p, tb, work + lb, &head->range_work, int64_t(np),
                                   s));
  const char* fe = std::getenv("FMMCU_P2P_E");
  wl_setup_kernel<<<1, 1, 0, s>>>(head, fe ? std::atoi(fe) : 0);
  ++nk;
  return FMMCU_OK;
}

int build_worklist_dev(fmmcu_ctx* c, uint32_t lb, uint32_t le, const WlGroups& g,
                       cudaStream_t s, const std::function<void()>& while_waiting) {
  const uint32_t np = le - lb;
  const uint32_t K = g.K ? g.K : 1u;
  int nk = 0;
  size_t need = 0;
  if (int rc = wl_prepare(c, lb, le, g, s, nk, need)) return rc;
  const size_t n1 = size_t(np) + 1;
  WlHead* head = c->d_wl_head.as<WlHead>();
  uint32_t* key = c->d_wl_key.as<uint32_t>();
  uint32_t* key2 = key + n1;
  uint32_t* val = c->d_wl_val.as<uint32_t>();
  uint32_t* val2 = val + n1;
  auto* S = c->d_wl_S.as<unsigned long long>();
  uint32_t* ci = c->d_wl_cnt.as<uint32_t>();
  uint32_t* cf = ci + n1;
  uint32_t* cp = cf + n1;
  uint32_t* io = c->d_wl_off.as<uint32_t>();
  uint32_t* fo = io + n1;
  uint32_t* po = fo + n1;
  const uint32_t* ev = c->d_ev.as<uint32_t>();
  const uint32_t* so = c->d_soff.as<uint32_t>();
  const uint2* seg = c->d_seg.as<uint2>();
  size_t tb = 0;
  // leaves stably ordered by group (K == 1: ascending leaves, no sort)
  const uint32_t* ks = key;
  const uint32_t* vs = val;
  if (K > 1 && np) {
    tb = need;
    CU_TRY(c, cub::DeviceRadixSort::SortPairs(c->d_cubtmp.p, tb, key, key2, val, val2,
                                              int64_t(np), 0, 5, s));
    ks = key2;
    vs = val2;
  }
  wl_count_kernel<<<nblocks(uint64_t(n1) * 32, 256), 256, 0, s>>>(ev, so, seg, lb, np, vs, S, head,
                                                                  ci, cf, cp);
  ++nk;
  for (int q = 0; q < 3; ++q) {
    tb = need;
    CU_TRY(c, cub::DeviceScan::ExclusiveSum(c->d_cubtmp.p, tb, ci + q * n1, io + q * n1,
                                            int64_t(n1), s));
  }
  wl_bounds_kernel<<<nblocks(n1, 256), 256, 0, s>>>(ks, np, K, io, fo, po, head);
  ++nk;
  CU_TRY(c, cudaMemcpyAsync(c->h_wl_head.p, head, sizeof(WlHead), cudaMemcpyDeviceToHost, s));
  if (while_waiting) while_waiting();  // host work overlapping the list build
  CU_TRY(c, cudaStreamSynchronize(s));
  const WlHead h = *c->h_wl_head.as<WlHead>();
  // the ordering key and val arrays stay valid for the fill
  CU_TRY(c, c->d_items.ensure(size_t(std::max(h.n_items, 1u)) * sizeof(P2PItem)));
  CU_TRY(c, c->d_fin.ensure(size_t(std::max(h.n_fins, 1u)) * sizeof(P2PFinal)));
  CU_TRY(c, c->d_partial.ensure(size_t(std::max(h.n_pevals, 1u)) * 16));
  if (np) {
    wl_fill_kernel<<<nblocks(uint64_t(np) * 32, 256), 256, 0, s>>>(
        ev, so, seg, lb, np, vs, S, head, io, fo, po, c->d_items.as<P2PItem>(),
        c->d_fin.as<P2PFinal>());
    ++nk;
  }
  CU_TRY(c, cudaGetLastError());
  c->launches += uint64_t(nk);
  c->warp_e = int(h.E);
  c->warp_items = true;
  c->sym_items = false;
  c->grouped = K > 1;
  c->partial_evals = h.n_pevals;
  c->dev_wl = true;
  c->dev_wl_lb = lb;
  c->dev_wl_le = le;
  c->dev_list = true;
  c->dev_list_total = h.range_work;
  c->dev_grp_item.assign(h.grp_item, h.grp_item + K + 1);
  c->dev_grp_fin.assign(h.grp_fin, h.grp_fin + K + 1);
  return FMMCU_OK;
}

// Symmetric (mutual-kernel) list over [lb, le) on the device (the host
// build_sym_worklist restated, same entries / items / slots), plus the
// per-leaf contribution lists of p2p_sym_finalize_kernel.  Returns -1 when
// the job does not qualify (a leaf with more than 32 entries, or too many
// contribution slots): the caller then builds the ordinary list.  Two small
// header reads synchronize `s`.
//
// Upload groups (gp->K > 1, the overlapped launch): a pair is symmetric only
// when both leaves are in the same group (the group of a leaf is the upload
// chunk of the last source slot its strong list reads, wl_leaf_kernel), so
// group k's items read chunks <= k only and its finalize needs only its own
// items; cross-group partners run as ordered pairs from both sides.  Items
// are laid out in group order (a stable sort of the leaves by group, as
// build_worklist_dev); c->dev_grp_item / dev_grp_fin hold each group's
// first item and first leaf position, and the positions -> leaves map stays
// in d_wl_val for the finalize.
int build_sym_worklist_dev(fmmcu_ctx* c, uint32_t lb, uint32_t le, cudaStream_t s,
                           const WlGroups* gp) {
  const uint32_t np = le - lb;
  WlGroups g{};
  g.K = 1;
  if (gp) g = *gp;
  const uint32_t K = g.K ? g.K : 1u;
  const bool grouped = K > 1;
  int nk = 0;
  size_t need = 0;
  if (int rc = wl_prepare(c, lb, le, g, s, nk, need)) return rc;
  const size_t n1 = size_t(np) + 1;
  WlHead* head = c->d_wl_head.as<WlHead>();
  // grouped: leaves stably ordered by group; grp = group per leaf (leaf order)
  const uint32_t* grp = nullptr;
  const uint32_t* order = nullptr;
  const uint32_t* key_sorted = nullptr;
  if (grouped && np) {
    uint32_t* key = c->d_wl_key.as<uint32_t>();
    uint32_t* val = c->d_wl_val.as<uint32_t>();
    size_t tb = need;
    CU_TRY(c, cub::DeviceRadixSort::SortPairs(c->d_cubtmp.p, tb, key, key + n1, val, val + n1,
                                              int64_t(np), 0, 5, s));
    grp = key;
    key_sorted = key + n1;
    order = val + n1;
  }
  auto rup = [](size_t b) { return (b + 255) & ~size_t(255); };
  CU_TRY(c, c->d_wls.ensure(256 + 4 * rup(n1 * 4) + 4 * rup(n1 * 8)));
  char* base = c->d_wls.as<char>();
  auto* sh = reinterpret_cast<WlSymHead*>(base);
  char* p = base + 256;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  auto* n_ent = reinterpret_cast<uint32_t*>(take(n1 * 4));
  auto* n_blk = reinterpret_cast<uint32_t*>(take(n1 * 4));
  auto* ssym = reinterpret_cast<unsigned long long*>(take(n1 * 8));
  auto* sord = reinterpret_cast<unsigned long long*>(take(n1 * 8));
  auto* n_slot = reinterpret_cast<unsigned long long*>(take(n1 * 8));
  auto* ent = reinterpret_cast<uint32_t*>(take(n1 * 4));
  auto* blk = reinterpret_cast<uint32_t*>(take(n1 * 4));
  auto* slot = reinterpret_cast<unsigned long long*>(take(n1 * 8));
  if (size_t(p - base) > c->d_wls.cap) return set_err(c, FMMCU_EINVAL, "sym scratch layout");
  CU_TRY(c, cudaMemsetAsync(sh, 0, sizeof(WlSymHead), s));
  const uint32_t* pt = c->d_pt.as<uint32_t>();
  const uint32_t* ev = c->d_ev.as<uint32_t>();
  const uint32_t* so = c->d_soff.as<uint32_t>();
  const uint32_t* si = c->d_sidx.as<uint32_t>();
  const uint2* seg = c->d_seg.as<uint2>();
  wls_count_kernel<<<nblocks(uint64_t(n1) * 32, 256), 256, 0, s>>>(ev, so, si, seg, lb, le, head,
                                                                  n_ent, n_blk, ssym, sord, n_slot,
                                                                  sh, grp, order);
  ++nk;
  size_t tb = 0;
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(nullptr, tb, n_slot, slot, int64_t(n1), s));
  need = std::max(need, tb);
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(nullptr, tb, n_ent, ent, int64_t(n1), s));
  need = std::max(need, tb);
  CU_TRY(c, c->d_cubtmp.ensure(need));
  tb = need;
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(c->d_cubtmp.p, tb, n_ent, ent, int64_t(n1), s));
  tb = need;
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(c->d_cubtmp.p, tb, n_blk, blk, int64_t(n1), s));
  tb = need;
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(c->d_cubtmp.p, tb, n_slot, slot, int64_t(n1), s));
  if (grouped && np) {
    wls_bounds_kernel<<<nblocks(n1, 256), 256, 0, s>>>(key_sorted, np, K, blk, head);
    ++nk;
  }
  // totals + the qualification flag + the header (E)
  CU_TRY(c, c->h_wl_head.ensure(sizeof(WlHead) + 64));
  auto* hh = c->h_wl_head.as<char>();
  CU_TRY(c, cudaMemcpyAsync(hh, head, sizeof(WlHead), cudaMemcpyDeviceToHost, s));
  auto* tot = reinterpret_cast<uint64_t*>(hh + sizeof(WlHead));
  for (int q = 0; q < 6; ++q) tot[q] = 0;  // 4-byte copies land in the low halves
  CU_TRY(c, cudaMemcpyAsync(&tot[0], ent + np, 4, cudaMemcpyDeviceToHost, s));
  CU_TRY(c, cudaMemcpyAsync(&tot[1], blk + np, 4, cudaMemcpyDeviceToHost, s));
  CU_TRY(c, cudaMemcpyAsync(&tot[2], slot + np, 8, cudaMemcpyDeviceToHost, s));
  CU_TRY(c, cudaMemcpyAsync(&tot[3], &sh->bad, 4, cudaMemcpyDeviceToHost, s));
  CU_TRY(c, cudaMemcpyAsync(&tot[5], &sh->ncl, 8, cudaMemcpyDeviceToHost, s));
  CU_TRY(c, cudaStreamSynchronize(s));
  const WlHead h = *reinterpret_cast<const WlHead*>(hh);
  const uint64_t n_entries = tot[0], n_items = tot[1], n_slots = tot[2];
  c->launches += uint64_t(nk);
  if ((tot[3] & 1u) || n_slots > 0xFFFFFFF0ull || n_items > 0xFFFFFFF0ull ||
      tot[5] > 0xFFFFFFF0ull)
    return -1;
  CU_TRY(c, c->d_symseg.ensure(std::max<uint64_t>(n_entries, 1) * 16));
  CU_TRY(c, c->d_items.ensure(std::max<uint64_t>(n_items, 1) * sizeof(P2PItem)));
  CU_TRY(c, c->d_syminfo.ensure(n1 * 16));
  CU_TRY(c, c->d_contrib.ensure(std::max<uint64_t>(n_slots, 1) * 16));
  CU_TRY(c, c->d_tgt.ensure(size_t(std::max(c->n_eval, 1u)) * 16));
  uint2* cnt = nullptr;
  if (grouped) {
    CU_TRY(c, c->d_symcnt.ensure(n1 * 8));
    cnt = c->d_symcnt.as<uint2>();
  }
  wls_fill_kernel<<<nblocks(uint64_t(n1) * 32, 256), 256, 0, s>>>(
      pt, ev, so, si, seg, lb, le, head, ent, blk, ssym, sord, slot, c->d_symseg.as<uint4>(),
      c->d_items.as<P2PItem>(), c->d_syminfo.as<uint4>(), grp, order, cnt);
  c->launches += 1;
  // per-leaf contribution lists (count, scan, fill), as stage_csr
  CU_TRY(c, c->d_cloff.ensure(n1 * 4));
  CU_TRY(c, c->d_clcnt.ensure(n1 * 4));
  CU_TRY(c, cudaMemsetAsync(c->d_clcnt.p, 0, n1 * 4, s));
  const uint32_t gb = (np + 7) / 8;
  if (np)
    p2p_sym_lists_kernel<false><<<gb, 256, 0, s>>>(lb, np, pt, so, si, c->d_syminfo.as<uint4>(),
                                                   c->d_symseg.as<uint4>(),
                                                   c->d_clcnt.as<uint32_t>(), nullptr, nullptr,
                                                   grp, cnt);
  tb = 0;
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(nullptr, tb, c->d_clcnt.as<uint32_t>(),
                                          c->d_cloff.as<uint32_t>(), int64_t(n1), s));
  CU_TRY(c, c->d_cubtmp.ensure(tb));
  CU_TRY(c, cub::DeviceScan::ExclusiveSum(c->d_cubtmp.p, tb, c->d_clcnt.as<uint32_t>(),
                                          c->d_cloff.as<uint32_t>(), int64_t(n1), s));
  // cl_base sized from the count kernel's total (no second header read)
  const uint32_t ncl = uint32_t(tot[5]);
  CU_TRY(c, c->d_clbase.ensure(size_t(std::max(ncl, 1u)) * 4));
  if (np)
    p2p_sym_lists_kernel<true><<<gb, 256, 0, s>>>(lb, np, pt, so, si, c->d_syminfo.as<uint4>(),
                                                  c->d_symseg.as<uint4>(), nullptr,
                                                  c->d_cloff.as<uint32_t>(),
                                                  c->d_clbase.as<uint32_t>(), grp, cnt);
  CU_TRY(c, cudaGetLastError());
  c->launches += 3;
  c->sym_grouped = grouped;
  if (grouped) {
    c->dev_grp_item.assign(h.grp_item, h.grp_item + K + 1);
    c->dev_grp_fin.assign(h.grp_fin, h.grp_fin + K + 1);  // first leaf positions
  } else {
    c->dev_grp_item.assign({0u, uint32_t(n_items)});
    c->dev_grp_fin.assign({0u, np});
  }
  c->sym_order = order;
  c->warp_e = int(h.E);
  c->warp_items = true;
  c->sym_items = true;
  c->sym_lb = lb;
  c->sym_le = le;
  c->sym_slots = n_slots;
  c->sym_n_items = uint32_t(n_items);
  c->sym_rounds = (tot[3] & 2u) != 0;
  c->grouped = grouped;
  c->partial_evals = 0;
  c->dev_wl = false;
  c->dev_list = true;
  c->dev_list_total = h.range_work;
  return FMMCU_OK;
}

}  // namespace fmmcu::detail

namespace fmmcu::detail {

// The finest CSR of a device-resident tree (pt_off, ev_off, strong_off,
// strong_idx) staged for the P2P kernels without a host round trip: copied
// into the context's staging on stream `w`, the run table and the work list
// built there (one header read synchronizes `w` only), `done` recorded on
// `w`.  The eval records (which need the permuted evals) are the caller's.
int stage_csr_dev(fmmcu_ctx* c, const uint32_t* pt, const uint32_t* ev, const uint32_t* so,
                  const uint32_t* si, uint32_t nl, uint32_t nnz, uint32_t ne, cudaStream_t w,
                  cudaEvent_t done, bool want_sym) {
  c->n_leaves = nl;
  CU_TRY(c, c->d_pt.ensure(size_t(nl + 1) * 4));
  CU_TRY(c, c->d_ev.ensure(size_t(nl + 1) * 4));
  CU_TRY(c, c->d_soff.ensure(size_t(nl + 1) * 4));
  CU_TRY(c, c->d_sidx.ensure(size_t(std::max(nnz, 1u)) * 4));
  CU_TRY(c, c->d_out.ensure(size_t(std::max(ne, 1u)) * 16));
  CU_TRY(c, c->d_evr.ensure(size_t(std::max(ne, 1u)) * 32));
  CU_TRY(c, c->d_hits.ensure(8));
  CU_TRY(c, c->d_counter.ensure(8));
  CU_TRY(c, c->h_hits.ensure(8));
  CU_TRY(c, cudaMemcpyAsync(c->d_pt.p, pt, size_t(nl + 1) * 4, cudaMemcpyDeviceToDevice, w));
  CU_TRY(c, cudaMemcpyAsync(c->d_ev.p, ev, size_t(nl + 1) * 4, cudaMemcpyDeviceToDevice, w));
  CU_TRY(c, cudaMemcpyAsync(c->d_soff.p, so, size_t(nl + 1) * 4, cudaMemcpyDeviceToDevice, w));
  if (nnz)
    CU_TRY(c, cudaMemcpyAsync(c->d_sidx.p, si, size_t(nnz) * 4, cudaMemcpyDeviceToDevice, w));
  c->n_strong = nnz;
  c->n_eval = ne;
  int rc_sym = -1;
  if (want_sym) {  // mutual kernel; falls back to the ordered list
    rc_sym = build_sym_worklist_dev(c, 0, nl, w);
    if (rc_sym != FMMCU_OK && rc_sym != -1) return rc_sym;
  }
  if (rc_sym != FMMCU_OK) {
    WlGroups g{};
    g.K = 1;
    if (int rc = build_worklist_dev(c, 0, nl, g, w)) return rc;
  }
  CU_TRY(c, cudaEventRecord(done, w));
  CU_TRY(c, cudaGetLastError());
  c->staged = true;
  return FMMCU_OK;
}

}  // namespace fmmcu::detail
