// fmm-b200 — CudaBackend: NearFieldBackend -> libfmmcuda.so C ABI.
//
// Flattens the reference NearFieldJob (backend.hpp:27-37) into the CSR
// arrays of fmmcu_p2p_job, shards target leaves across devices by pair
// work, and maps C-ABI status codes onto the reference error taxonomy
// (types.hpp:62-92): launch/finish failures surface as exceptions that the
// engine wraps as BackendError("nearfield launch" | "nearfield", ...)
// (engine.cpp:294-311); coincident M2L centres as SingularConfiguration.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <sys/mman.h>

#include <algorithm>
#include <cstdint>
#include <thread>
#include <stdexcept>

#include "fmm/cuda_backend.hpp"
#include "fmm_cuda.h"
#include "host_util.hpp"

namespace fmm {

using detail::resize_huge;

namespace {

[[noreturn]] void raise(fmmcu_ctx* c, int rc, const char* what) {
  const std::string msg = std::string(what) + ": " + (c ? fmmcu_last_error(c) : "no context");
  if (rc == FMMCU_ESINGULAR) throw SingularConfiguration(msg);
  if (rc == FMMCU_EINVAL) throw InvalidInput(msg);
  throw std::runtime_error(msg);
}

}  // namespace

CudaBackend::CudaBackend(const CudaSettings& cs) : cs_(cs) {
  if (cs_.devices.empty()) cs_.devices.push_back(0);
  for (int d : cs_.devices) {
    fmmcu_ctx* c = nullptr;
    const int rc = fmmcu_create(&c, d);
    if (rc != FMMCU_OK) {
      const std::string msg = std::string("cuda backend: ") + (c ? fmmcu_last_error(c) : "");
      if (c) fmmcu_destroy(c);
      for (fmmcu_ctx* o : ctx_) fmmcu_destroy(o);
      ctx_.clear();
      throw BackendError("cuda init", msg);
    }
    ctx_.push_back(c);
  }
}

CudaBackend::~CudaBackend() {
  if (fill_.joinable()) fill_.join();
  if (inflight_) {
    for (fmmcu_ctx* c : ctx_) {
      std::uint64_t p;
      double s;
      fmmcu_p2p_finish(c, &p, &s);
    }
  }
  for (fmmcu_ctx* c : ctx_) fmmcu_destroy(c);
}

CudaBackend::DeviceEval CudaBackend::fmm_evaluate(const SourceSet& sources, const EvalSet& evals,
                                                  int n_levels, double theta, int p,
                                                  Kernel kernel, const Smoother& smoother,
                                                  std::vector<cplx>& out) {
  if (inflight_) throw InvalidState("cuda backend: evaluate while a near field is in flight");
  if (sources.size() > 0xFFFFFFFFull || evals.size() > 0xFFFFFFFFull)
    throw InvalidInput("device pipeline: more than 2^32 points");
  // The result vector is value-initialised (the API returns a std::vector);
  // its 16 B/eval zero fill + first-touch page faults run on a helper thread
  // while the device pipeline works, and the potentials are copied in once
  // it has finished.  reserve() fixes the storage, so data() stays valid.
  // A result that already has the right size (evaluate_into) is overwritten
  // in place: no allocation, no zero fill.
  const bool reuse = !out.empty() && out.size() == evals.size();
  if (!reuse) {
    out.clear();
    out.reserve(evals.size());
  }
  // started once the pipeline has read the inputs (the host then only waits
  // on the device), so the fill does not compete with the upload staging
  std::thread zero_fill;
  struct Hook {
    std::thread* t;
    std::vector<cplx>* out;
    std::size_t n;
  } hook{&zero_fill, &out, evals.size()};
  fmmcu_fmm_job j{};
  j.n_src = std::uint32_t(sources.size());
  j.n_eval = std::uint32_t(evals.size());
  j.src_z = reinterpret_cast<const double*>(sources.z.data());
  j.src_m = reinterpret_cast<const double*>(sources.m.data());
  j.eval_y = evals.size() ? reinterpret_cast<const double*>(evals.y.data()) : nullptr;
  j.eval_sid = evals.source_id.empty() ? nullptr : evals.source_id.data();
  j.n_levels = n_levels;
  j.theta = theta;
  j.p = p;
  j.kernel = kernel == Kernel::harmonic ? FMMCU_KERNEL_HARMONIC : FMMCU_KERNEL_LOG;
  j.smoother = smoother.kind == Smoother::Kind::none       ? FMMCU_SMOOTH_NONE
               : smoother.kind == Smoother::Kind::gaussian ? FMMCU_SMOOTH_GAUSSIAN
                                                           : FMMCU_SMOOTH_PLUMMER;
  j.delta = smoother.delta;
  j.out = reuse ? reinterpret_cast<double*>(out.data()) : nullptr;  // direct D2H if page-locked
  j.inputs_consumed = [](void* arg) {
    auto* h = static_cast<Hook*>(arg);
    *h->t = std::thread([out = h->out, n = h->n] { resize_huge(*out, n); });
  };
  j.inputs_consumed_arg = &hook;
  if (reuse) j.inputs_consumed = nullptr;
  fmmcu_fmm_stats st{};
  using TClock = std::chrono::steady_clock;
  const auto t0 = TClock::now();
  int rc = fmmcu_fmm_launch(ctx_[0], &j);
  const auto t1 = TClock::now();
  if (zero_fill.joinable()) zero_fill.join();
  else if (!reuse) resize_huge(out, evals.size());
  const auto t2 = TClock::now();
  if (rc == FMMCU_OK)
    rc = fmmcu_fmm_finish(ctx_[0], evals.size() ? reinterpret_cast<double*>(out.data()) : nullptr,
                          &st);
  if (std::getenv("FMMCU_TRACE")) {
    auto ms = [](TClock::time_point a, TClock::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    std::fprintf(stderr, "[fmm] launch %.3f ms, result fill join %.3f ms, finish %.3f ms\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, TClock::now()));
  }
  if (rc != FMMCU_OK) raise(ctx_[0], rc, "device pipeline");
  DeviceEval d;
  d.counters.p2p_pairs = st.p2p_pairs;
  d.counters.m2l_ops = st.m2l_ops;
  d.counters.p2m_points = st.p2m_points;
  d.counters.l2p_points = st.l2p_points;
  d.t_upload = st.t_upload;
  d.t_tree = st.t_tree;
  d.t_connect = st.t_connect;
  d.t_p2m_upward = st.t_p2m_upward;
  d.t_m2l = st.t_m2l;
  d.t_p2p = st.t_p2p;
  d.t_device = st.t_device;
  d.t_far_wait = st.t_far_wait;
  return d;
}

std::uint64_t CudaBackend::kernel_launches() const {
  std::uint64_t n = 0;
  for (fmmcu_ctx* c : ctx_) n += fmmcu_kernel_launches(c);
  return n;
}

void CudaBackend::launch(const NearFieldJob& job, std::vector<cplx>& out) {
  if (inflight_) throw InvalidState("cuda backend: launch while a job is in flight");
  const std::vector<MBox>& fine = job.pyramid->finest();
  const std::uint32_t nl = std::uint32_t(fine.size());
  const std::uint32_t ne = std::uint32_t(job.eval_y->size());
  // zero fill (huge pages) on a helper thread; joined in finish() before the
  // device results are copied in
  out.clear();
  out.reserve(ne);
  fill_ = std::thread([&out, ne] { resize_huge(out, ne); });

  pt_off_.resize(nl + 1);
  ev_off_.resize(nl + 1);
  s_off_.resize(nl + 1);
  for (std::uint32_t i = 0; i < nl; ++i) {
    pt_off_[i] = fine[i].point_begin;
    ev_off_[i] = fine[i].eval_begin;
  }
  pt_off_[nl] = nl ? fine[nl - 1].point_end : 0;
  ev_off_[nl] = nl ? fine[nl - 1].eval_end : 0;
  std::uint32_t nnz = 0;
  for (std::uint32_t i = 0; i < nl; ++i) {
    s_off_[i] = nnz;
    nnz += std::uint32_t(job.finest->strong[i].size());
  }
  s_off_[nl] = nnz;
  s_idx_.resize(nnz);
  for (std::uint32_t i = 0; i < nl; ++i)
    std::copy(job.finest->strong[i].begin(), job.finest->strong[i].end(), s_idx_.begin() + s_off_[i]);

  // Contiguous target-leaf shards balanced by pair work n_evals * |strong sources|.
  const std::size_t nd = ctx_.size();
  std::vector<std::uint32_t> cut(nd + 1, 0);
  cut[nd] = nl;
  if (nd > 1) {
    std::vector<double> pre(nl + 1, 0.0);
    for (std::uint32_t i = 0; i < nl; ++i) {
      double s = 0;
      for (std::uint32_t q = s_off_[i]; q < s_off_[i + 1]; ++q)
        s += fine[s_idx_[q]].point_end - fine[s_idx_[q]].point_begin;
      pre[i + 1] = pre[i] + s * (fine[i].eval_end - fine[i].eval_begin);
    }
    for (std::size_t d = 1; d < nd; ++d) {
      const double want = pre[nl] * double(d) / double(nd);
      cut[d] = std::uint32_t(std::lower_bound(pre.begin(), pre.end(), want) - pre.begin());
      cut[d] = std::max(cut[d], cut[d - 1]);
    }
  }

  fmmcu_p2p_job j{};
  j.n_leaves = nl;
  j.n_src = std::uint32_t(job.src_z->size());
  j.n_eval = ne;
  j.pt_off = pt_off_.data();
  j.ev_off = ev_off_.data();
  j.strong_off = s_off_.data();
  j.strong_idx = s_idx_.data();
  j.perm = job.pyramid->perm.data();
  j.src_z = reinterpret_cast<const double*>(job.src_z->data());
  j.src_m = reinterpret_cast<const double*>(job.src_m->data());
  j.eval_y = reinterpret_cast<const double*>(job.eval_y->data());
  j.eval_sid = (job.eval_sid && !job.eval_sid->empty()) ? job.eval_sid->data() : nullptr;
  j.kernel = job.kernel == Kernel::harmonic ? FMMCU_KERNEL_HARMONIC : FMMCU_KERNEL_LOG;
  j.smoother = job.smoother.kind == Smoother::Kind::none      ? FMMCU_SMOOTH_NONE
               : job.smoother.kind == Smoother::Kind::gaussian ? FMMCU_SMOOTH_GAUSSIAN
                                                               : FMMCU_SMOOTH_PLUMMER;
  j.delta = job.smoother.delta;
  j.mode = cs_.exact ? FMMCU_MODE_EXACT : FMMCU_MODE_FAST;
  j.out = reinterpret_cast<double*>(out.data());
  for (std::size_t d = 0; d < nd; ++d) {
    j.leaf_begin = cut[d];
    j.leaf_end = cut[d + 1];
    const int rc = fmmcu_p2p_launch(ctx_[d], &j);
    if (rc != FMMCU_OK) {
      if (fill_.joinable()) fill_.join();
      for (std::size_t q = 0; q < d; ++q) {
        std::uint64_t p;
        double s;
        fmmcu_p2p_finish(ctx_[q], &p, &s);
      }
      raise(ctx_[d], rc, "cuda near field launch");
    }
  }
  inflight_ = true;
}

NearFieldStats CudaBackend::finish() {
  if (!inflight_) return NearFieldStats{};
  inflight_ = false;
  if (fill_.joinable()) fill_.join();
  NearFieldStats st;
  int bad = FMMCU_OK;
  fmmcu_ctx* bad_ctx = nullptr;
  for (fmmcu_ctx* c : ctx_) {
    std::uint64_t pairs = 0;
    double secs = 0;
    const int rc = fmmcu_p2p_finish(c, &pairs, &secs);
    if (rc != FMMCU_OK && bad == FMMCU_OK) {
      bad = rc;
      bad_ctx = c;
    }
    st.pair_evals += pairs;
    st.seconds = std::max(st.seconds, secs);
  }
  if (bad != FMMCU_OK) raise(bad_ctx, bad, "cuda near field");
  return st;
}

void CudaBackend::m2l_launch(int p, Kernel kernel, const std::vector<cplx>& centers,
                             const std::vector<cplx>& coeffs,
                             const std::vector<std::uint32_t>& target_box,
                             const std::vector<std::uint32_t>& weak_off,
                             const std::vector<std::uint32_t>& weak_idx, std::vector<cplx>& out) {
  out.assign(target_box.size() * std::size_t(p + 1), cplx(0, 0));
  fmmcu_m2l_job j{};
  j.p = p;
  j.kernel = kernel == Kernel::harmonic ? FMMCU_KERNEL_HARMONIC : FMMCU_KERNEL_LOG;
  j.n_boxes = std::uint32_t(centers.size());
  j.centers = reinterpret_cast<const double*>(centers.data());
  j.coeffs = reinterpret_cast<const double*>(coeffs.data());
  j.n_targets = std::uint32_t(target_box.size());
  j.target_box = target_box.data();
  j.weak_off = weak_off.data();
  j.weak_idx = weak_idx.data();
  j.out = reinterpret_cast<double*>(out.data());
  const int rc = fmmcu_m2l_launch(ctx_[0], &j);
  if (rc != FMMCU_OK) raise(ctx_[0], rc, "cuda m2l launch");
}

void CudaBackend::device_tree(const SourceSet& sources, const EvalSet& evals, int n_levels,
                              double theta, Pyramid& pyr, Connectivity& conn) {
  if (inflight_) throw InvalidState("cuda backend: tree build while a near field is in flight");
  if (sources.size() == 0) throw InvalidInput("build_pyramid: empty source set");
  if (sources.size() > 0xFFFFFFFFull || evals.size() > 0xFFFFFFFFull)
    throw InvalidInput("device tree: more than 2^32 points");
  fmmcu_ctx* c = ctx_[0];
  fmmcu_fmm_job j{};
  j.n_src = std::uint32_t(sources.size());
  j.n_eval = std::uint32_t(evals.size());
  j.src_z = reinterpret_cast<const double*>(sources.z.data());
  j.src_m = nullptr;
  j.eval_y = evals.size() ? reinterpret_cast<const double*>(evals.y.data()) : nullptr;
  j.eval_sid = evals.source_id.empty() ? nullptr : evals.source_id.data();
  j.n_levels = n_levels;
  j.theta = theta;
  j.p = 1;
  using TClock = std::chrono::steady_clock;
  const auto t0 = TClock::now();
  int rc = fmmcu_tree_build(c, &j);
  if (rc != FMMCU_OK) raise(c, rc, "cuda tree build");
  const auto t1 = TClock::now();
  const int L = n_levels;
  pyr = Pyramid{};
  pyr.n_levels = L;
  pyr.levels.resize(L);
  conn = Connectivity{};
  conn.levels.resize(L);
  std::vector<double> f64;
  std::vector<std::uint32_t> u32, off, idx;
  for (int l = 0; l < L; ++l) {
    std::uint32_t nb = 0;
    if ((rc = fmmcu_fmm_tree_level(c, l, &nb, nullptr, nullptr)) != FMMCU_OK) raise(c, rc, "tree");
    f64.resize(std::size_t(nb) * 5);
    u32.resize(std::size_t(nb) * 4);
    if ((rc = fmmcu_fmm_tree_level(c, l, &nb, f64.data(), u32.data())) != FMMCU_OK)
      raise(c, rc, "tree");
    std::vector<MBox>& boxes = pyr.levels[l];
    boxes.resize(nb);
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < std::int64_t(nb); ++i) {
      MBox& b = boxes[i];
      b.center = cplx(f64[5 * i], f64[5 * i + 1]);
      b.half_width = f64[5 * i + 2];
      b.half_height = f64[5 * i + 3];
      b.radius = f64[5 * i + 4];
      b.level = l;
      b.index_in_level = std::uint32_t(i);
      b.point_begin = u32[4 * i];
      b.point_end = u32[4 * i + 1];
      b.eval_begin = u32[4 * i + 2];
      b.eval_end = u32[4 * i + 3];
    }
    for (int weak = 0; weak < 2; ++weak) {
      std::uint64_t nnz = 0;
      if ((rc = fmmcu_fmm_tree_lists(c, l, weak, &nnz, nullptr, nullptr)) != FMMCU_OK)
        raise(c, rc, "tree");
      off.resize(std::size_t(nb) + 1);
      idx.resize(std::max<std::uint64_t>(nnz, 1));
      if ((rc = fmmcu_fmm_tree_lists(c, l, weak, &nnz, off.data(), idx.data())) != FMMCU_OK)
        raise(c, rc, "tree");
      auto& rows = weak ? conn.levels[l].weak : conn.levels[l].strong;
      rows.resize(nb);
#pragma omp parallel for schedule(static)
      for (std::int64_t i = 0; i < std::int64_t(nb); ++i)
        rows[i].assign(idx.begin() + off[i], idx.begin() + off[i + 1]);
    }
  }
  pyr.perm.resize(sources.size());
  pyr.eval_perm.resize(evals.size());
  if ((rc = fmmcu_fmm_tree_perm(c, pyr.perm.data(), evals.size() ? pyr.eval_perm.data() : nullptr)) !=
      FMMCU_OK)
    raise(c, rc, "tree");
  if (std::getenv("FMM_TRACE"))
    std::fprintf(stderr, "[fmm] device tree: build %.2f ms, read back + host lists %.2f ms\n",
                 std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(TClock::now() - t1).count());
}

CudaBackend::M2LBuffers CudaBackend::m2l_buffers(std::uint32_t n_boxes, int p,
                                                 std::uint32_t n_targets, std::uint64_t nnz) {
  fmmcu_m2l_buffers hb{};
  const int rc = fmmcu_m2l_host_buffers(ctx_[0], n_boxes, p, n_targets, nnz, &hb);
  if (rc != FMMCU_OK) raise(ctx_[0], rc, "cuda m2l buffers");
  M2LBuffers b;
  b.centers = reinterpret_cast<cplx*>(hb.centers);
  b.coeffs = reinterpret_cast<cplx*>(hb.coeffs);
  b.out = reinterpret_cast<cplx*>(hb.out);
  b.target_box = hb.target_box;
  b.weak_off = hb.weak_off;
  b.weak_idx = hb.weak_idx;
  return b;
}

void CudaBackend::m2l_launch(int p, Kernel kernel, std::uint32_t n_boxes, std::uint32_t n_targets,
                             const M2LBuffers& b) {
  fmmcu_m2l_job j{};
  j.p = p;
  j.kernel = kernel == Kernel::harmonic ? FMMCU_KERNEL_HARMONIC : FMMCU_KERNEL_LOG;
  j.n_boxes = n_boxes;
  j.centers = reinterpret_cast<const double*>(b.centers);
  j.coeffs = reinterpret_cast<const double*>(b.coeffs);
  j.n_targets = n_targets;
  j.target_box = b.target_box;
  j.weak_off = b.weak_off;
  j.weak_idx = b.weak_idx;
  j.out = reinterpret_cast<double*>(b.out);
  const int rc = fmmcu_m2l_launch(ctx_[0], &j);
  if (rc != FMMCU_OK) raise(ctx_[0], rc, "cuda m2l launch");
}

void CudaBackend::m2l_launch_keep(int p, Kernel kernel, std::uint32_t n_boxes,
                                  std::uint32_t n_targets, const M2LBuffers& b) {
  fmmcu_m2l_job j{};
  j.p = p;
  j.kernel = kernel == Kernel::harmonic ? FMMCU_KERNEL_HARMONIC : FMMCU_KERNEL_LOG;
  j.n_boxes = n_boxes;
  j.centers = reinterpret_cast<const double*>(b.centers);
  j.coeffs = reinterpret_cast<const double*>(b.coeffs);
  j.n_targets = n_targets;
  j.target_box = b.target_box;
  j.weak_off = b.weak_off;
  j.weak_idx = b.weak_idx;
  j.out = nullptr;  // the sums stay on the device for m2l_downward
  const int rc = fmmcu_m2l_launch(ctx_[0], &j);
  if (rc != FMMCU_OK) raise(ctx_[0], rc, "cuda m2l launch");
}

void CudaBackend::m2l_downward(int n_levels, const std::uint32_t* level_base,
                               const std::int32_t* target_of, cplx* finest_out) {
  fmmcu_l2l_job j{};
  j.n_levels = n_levels;
  j.level_base = level_base;
  j.target_of = target_of;
  j.finest_out = reinterpret_cast<double*>(finest_out);
  const int rc = fmmcu_m2l_downward(ctx_[0], &j);
  if (rc != FMMCU_OK) raise(ctx_[0], rc, "cuda m2l downward");
}

std::uint64_t CudaBackend::m2l_finish(double* seconds) {
  std::uint64_t ops = 0;
  double s = 0;
  const int rc = fmmcu_m2l_finish(ctx_[0], &ops, &s);
  if (seconds) *seconds = s;
  if (rc != FMMCU_OK) raise(ctx_[0], rc, "cuda m2l");
  return ops;
}

}  // namespace fmm
