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

#include "fmmcu_internal.cuh"
#include "p2p_worklist.cuh"

namespace fmmcu::detail {

namespace {
inline uint32_t nblocks(uint64_t n, uint32_t tb) { return uint32_t((n + tb - 1) / tb); }
}  // namespace

int build_worklist_dev(fmmcu_ctx* c, uint32_t lb, uint32_t le, const WlGroups& g,
                       cudaStream_t s) {
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
  uint32_t* cf = ci + n1;
  uint32_t* cp = cf + n1;
  uint32_t* io = c->d_wl_off.as<uint32_t>();
  uint32_t* fo = io + n1;
  uint32_t* po = fo + n1;
  CU_TRY(c, cudaMemsetAsync(head, 0, sizeof(WlHead), s));
  const uint32_t* pt = c->d_pt.as<uint32_t>();
  const uint32_t* ev = c->d_ev.as<uint32_t>();
  const uint32_t* so = c->d_soff.as<uint32_t>();
  const uint32_t* si = c->d_sidx.as<uint32_t>();
  int nk = 0;
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
  size_t tb = 0, need = 0;
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
  c->dev_wl_total = h.range_work;
  c->dev_grp_item.assign(h.grp_item, h.grp_item + K + 1);
  c->dev_grp_fin.assign(h.grp_fin, h.grp_fin + K + 1);
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
                  cudaEvent_t done) {
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
  WlGroups g{};
  g.K = 1;
  c->n_strong = nnz;
  if (int rc = build_worklist_dev(c, 0, nl, g, w)) return rc;
  CU_TRY(c, cudaEventRecord(done, w));
  CU_TRY(c, cudaGetLastError());
  c->staged = true;
  return FMMCU_OK;
}

}  // namespace fmmcu::detail
