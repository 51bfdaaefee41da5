// fmm-b200 — arguments of the batched M2L (m2l_kernels.cuh; launched by
// fmmcu::detail::m2l_run in fmmcu.cu for both the C-ABI M2L and the device
// pipeline).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fmmcu {

constexpr int kM2LMaxP = 96;  // largest order of the warp kernel (and the C ABI)

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
  // work items of the register kernel (m2l_run): {target, first partner,
  // end partner, partial slot or ~0u = the target's only item}
  const uint4* __restrict__ items;
  const uint32_t* __restrict__ n_items;  // device count
  double2* __restrict__ partial;         // [slots][p+1] sums of split lists
};

}  // namespace fmmcu
