// The reference-side binding of the B200 near field: a NearFieldBackend of
// kind `cuda` written against the UNMODIFIED reference interface
// (proj/include/fmm/backend.hpp:48-57), calling libfmmcuda.so through its C
// ABI (include/fmm_cuda.h).  This is the class INTEGRATION.md §A tells a
// maintainer to add; integration/patch_reference.py applies the three small
// edits that register it (BackendKind::cuda, backend_from_string/to_string,
// make_backend) to a scratch copy of the reference sources, and
// oracle/Makefile compiles that copy together with this file into
// oracle/_ref/libfmmref_cuda.so, so the tests can run the reference's OWN
// FmmEngine::evaluate (engine.cpp:208-347) with the GPU near field.
//
// No CUDA header is needed: the job is flattened into the CSR arrays of
// fmmcu_p2p_job (finest MBox point/eval ranges, LevelConn::strong), and
// std::complex<double> vectors pass as interleaved doubles.
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fmm/backend.hpp"
#include "fmm_cuda.h"

namespace fmm {

namespace {

class RefCudaBackend final : public NearFieldBackend {
 public:
  RefCudaBackend() {
    if (fmmcu_create(&ctx_, 0) != FMMCU_OK) {
      const std::string msg = ctx_ ? fmmcu_last_error(ctx_) : "no context";
      if (ctx_) fmmcu_destroy(ctx_);
      ctx_ = nullptr;
      throw BackendError("cuda", msg);
    }
  }
  ~RefCudaBackend() override {
    if (inflight_) {
      std::uint64_t p = 0;
      double s = 0.0;
      fmmcu_p2p_finish(ctx_, &p, &s);  // drain before the buffers go
    }
    fmmcu_destroy(ctx_);
  }
  bool concurrent() const override { return true; }
  const char* name() const override { return "cuda"; }

  void launch(const NearFieldJob& job, std::vector<cplx>& out) override {
    const std::vector<MBox>& fine = job.pyramid->finest();
    const auto& strong = job.finest->strong;
    const std::uint32_t nl = static_cast<std::uint32_t>(fine.size());
    pt_off_.resize(nl + 1);
    ev_off_.resize(nl + 1);
    s_off_.resize(nl + 1);
    s_idx_.clear();
    for (std::uint32_t i = 0; i < nl; ++i) {
      pt_off_[i] = fine[i].point_begin;
      ev_off_[i] = fine[i].eval_begin;
      s_off_[i] = static_cast<std::uint32_t>(s_idx_.size());
      s_idx_.insert(s_idx_.end(), strong[i].begin(), strong[i].end());
    }
    pt_off_[nl] = nl ? fine[nl - 1].point_end : 0;
    ev_off_[nl] = nl ? fine[nl - 1].eval_end : 0;
    s_off_[nl] = static_cast<std::uint32_t>(s_idx_.size());
    out.assign(job.eval_y->size(), cplx(0.0, 0.0));
    fmmcu_p2p_job cj{};
    cj.n_leaves = nl;
    cj.n_src = static_cast<std::uint32_t>(job.src_z->size());
    cj.n_eval = static_cast<std::uint32_t>(job.eval_y->size());
    cj.pt_off = pt_off_.data();
    cj.ev_off = ev_off_.data();
    cj.strong_off = s_off_.data();
    cj.strong_idx = s_idx_.data();
    cj.perm = job.pyramid->perm.data();
    cj.src_z = reinterpret_cast<const double*>(job.src_z->data());
    cj.src_m = reinterpret_cast<const double*>(job.src_m->data());
    cj.eval_y = reinterpret_cast<const double*>(job.eval_y->data());
    cj.eval_sid = (job.eval_sid && !job.eval_sid->empty()) ? job.eval_sid->data() : nullptr;
    cj.kernel = job.kernel == Kernel::harmonic ? FMMCU_KERNEL_HARMONIC : FMMCU_KERNEL_LOG;
    cj.smoother = job.smoother.kind == Smoother::Kind::none       ? FMMCU_SMOOTH_NONE
                  : job.smoother.kind == Smoother::Kind::gaussian ? FMMCU_SMOOTH_GAUSSIAN
                                                                   : FMMCU_SMOOTH_PLUMMER;
    cj.delta = job.smoother.delta;
    cj.mode = FMMCU_MODE_FAST;
    cj.leaf_begin = 0;
    cj.leaf_end = nl;
    cj.out = reinterpret_cast<double*>(out.data());
    const int rc = fmmcu_p2p_launch(ctx_, &cj);
    if (rc != FMMCU_OK) {
      if (rc == FMMCU_EINVAL) throw InvalidInput(std::string("cuda: ") + fmmcu_last_error(ctx_));
      throw std::runtime_error(std::string("cuda: ") + fmmcu_last_error(ctx_));
    }
    inflight_ = true;
  }

  NearFieldStats finish() override {
    NearFieldStats st;
    inflight_ = false;
    if (fmmcu_p2p_finish(ctx_, &st.pair_evals, &st.seconds) != FMMCU_OK)
      throw std::runtime_error(std::string("cuda: ") + fmmcu_last_error(ctx_));
    return st;  // the engine wraps throws as BackendError (engine.cpp:294-311)
  }

 private:
  fmmcu_ctx* ctx_ = nullptr;
  bool inflight_ = false;
  std::vector<std::uint32_t> pt_off_, ev_off_, s_off_, s_idx_;  // finest-level CSR
};

}  // namespace

// Declared by the patch in backend.hpp; called from make_backend's new case.
std::unique_ptr<NearFieldBackend> make_cuda_backend() { return std::make_unique<RefCudaBackend>(); }

}  // namespace fmm
