// fmm-b200 — header / grouping records of the device-built P2P work list
// (p2p_worklist.cuh), shared with the host code that launches it.
#pragma once

#include <cstdint>

namespace fmmcu {

constexpr int kWlMaxGroups = 32;

// device-written, host-read summary of a device work list
struct WlHead {
  unsigned long long cost4, cost5;  // lane-cost model sums (choose E)
  unsigned long long total_work;    // sum of n_evals * S over every leaf of the job
  unsigned long long range_work;    // ... over the range [lb, le)
  unsigned long long budget;        // pair work per item before a block splits
  uint32_t E, max_ev;
  uint32_t n_items, n_fins, n_pevals, pad;
  uint32_t grp_item[kWlMaxGroups + 1];
  uint32_t grp_fin[kWlMaxGroups + 1];
};

struct WlGroups {
  uint32_t K;                          // upload groups (1: everything resident)
  uint32_t slot_end[kWlMaxGroups];     // group k holds source slots below slot_end[k]
};

}  // namespace fmmcu
