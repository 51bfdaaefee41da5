// fmm-b200 — the B200 near-field backend (BackendKind::cuda).
//
// A NearFieldBackend (reference backend.hpp:48-57) that forwards the job to
// libfmmcuda.so through the C ABI of include/fmm_cuda.h.  Concurrent: launch
// packs + enqueues and returns, finish blocks on a CUDA event (no spinning,
// so the OpenMP far field keeps every core) and rethrows device failures.
// With several devices the target leaves are split into contiguous,
// pair-work-balanced ranges, one per device; every device holds all sources
// (replicated) and returns only its slice of the potentials.
#pragma once

#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "fmm/backend.hpp"
#include "fmm/engine.hpp"
#include "fmm/geometry.hpp"

struct fmmcu_ctx;

namespace fmm {

class CudaBackend final : public NearFieldBackend {
 public:
  explicit CudaBackend(const CudaSettings& cs);
  ~CudaBackend() override;
  CudaBackend(const CudaBackend&) = delete;
  CudaBackend& operator=(const CudaBackend&) = delete;

  bool concurrent() const override { return true; }
  const char* name() const override { return "cuda"; }
  void launch(const NearFieldJob& job, std::vector<cplx>& out) override;
  NearFieldStats finish() override;

  const CudaSettings& settings() const { return cs_; }

  // Batched M2L on the first device (see include/fmm_cuda.h fmmcu_m2l_job).
  // Asynchronous; m2l_finish fills `out` ([n_targets][p+1]) and throws
  // SingularConfiguration on coincident centres.
  void m2l_launch(int p, Kernel kernel, const std::vector<cplx>& centers,
                  const std::vector<cplx>& coeffs, const std::vector<std::uint32_t>& target_box,
                  const std::vector<std::uint32_t>& weak_off,
                  const std::vector<std::uint32_t>& weak_idx, std::vector<cplx>& out);
  std::uint64_t m2l_finish(double* seconds = nullptr);
  // The same on flat arrays in the context's page-locked buffers
  // (fmmcu_m2l_host_buffers): the caller flattens straight into them, the
  // launch DMAs them in place and the sums land in `out` ([n_targets][p+1]).
  struct M2LBuffers {
    cplx* centers = nullptr;  // [n_boxes]
    cplx* coeffs = nullptr;   // [n_boxes][p+1]
    cplx* out = nullptr;      // [n_targets][p+1]
    std::uint32_t* target_box = nullptr;
    std::uint32_t* weak_off = nullptr;
    std::uint32_t* weak_idx = nullptr;
  };
  M2LBuffers m2l_buffers(std::uint32_t n_boxes, int p, std::uint32_t n_targets, std::uint64_t nnz);
  void m2l_launch(int p, Kernel kernel, std::uint32_t n_boxes, std::uint32_t n_targets,
                  const M2LBuffers& b);
  // Downward pass on the device (fmmcu_m2l_downward): launch with
  // keep_on_device = true, then the L2L chain runs on the device and the
  // finest level's locals land in finest_out ([boxes of the finest level][p+1],
  // rows of boxes with a target slot) at m2l_finish.
  void m2l_launch_keep(int p, Kernel kernel, std::uint32_t n_boxes, std::uint32_t n_targets,
                       const M2LBuffers& b);
  void m2l_downward(int n_levels, const std::uint32_t* level_base, const std::int32_t* target_of,
                    cplx* finest_out);

  // The whole FmmEngine::evaluate on the first device (fmmcu_fmm_evaluate):
  // potentials in the original eval order, counters, device phase times.
  struct DeviceEval {
    WorkCounters counters;
    double t_upload = 0, t_tree = 0, t_connect = 0, t_p2m_upward = 0, t_m2l = 0, t_p2p = 0,
           t_device = 0, t_far_wait = 0;
  };
  DeviceEval fmm_evaluate(const SourceSet& sources, const EvalSet& evals, int n_levels,
                          double theta, int p, Kernel kernel, const Smoother& smoother,
                          std::vector<cplx>& out);

  // The pyramid and the theta-connectivity built on the first device
  // (fmmcu_tree_build; bit-exact with build_pyramid / build_connectivity)
  // and read back into the host structures the CPU far field uses.
  void device_tree(const SourceSet& sources, const EvalSet& evals, int n_levels, double theta,
                   Pyramid& pyr, Connectivity& conn);

  std::uint64_t kernel_launches() const;

 private:
  CudaSettings cs_;
  std::vector<fmmcu_ctx*> ctx_;
  bool inflight_ = false;
  std::thread fill_;  // zero fill of the caller's near-field vector (launch -> finish)
  // flattened job (must outlive the device work)
  std::vector<std::uint32_t> pt_off_, ev_off_, s_off_, s_idx_;
};

}  // namespace fmm
