// fmm-b200 — FMM evaluation pipeline (host orchestration).
//
// Semantics of the reference proj/src/engine.cpp:19-347: partition
// (pyramid + connectivity + permutation) -> P2M -> serial M2M -> launch the
// near field -> downward pass (L2L + M2L, fixed per-box accumulation order)
// -> join -> assembly (near + L2P), with the same PhaseTimings / WorkCounters
// and the observer hook the autotuner hangs on.
//
// B200 additions:
//  * BackendKind::cuda runs the near field on the GPU(s) concurrently with
//    the CPU downward pass (cpu_wait = time blocked in finish()).
//  * FmmConfig::m2l_on_device offloads every M2L of every level in one
//    batched launch that overlaps the device P2P; the host keeps the cheap
//    L2L chain and adds the device M2L sums per box (local = L2L(parent) +
//    sum_w M2L(w)).  m2l_ops is identical to the CPU path.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>

#include "fmm/cuda_backend.hpp"
#include "fmm/engine.hpp"
#include "host_util.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace fmm {

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

Expansion fresh(cplx center, Expansion::Kind kind, Kernel kernel, int p) {
  Expansion e;
  e.center = center;
  e.kind = kind;
  e.kernel = kernel;
  e.coeffs.assign(std::size_t(p) + 1, cplx(0, 0));
  return e;
}

// P2M on every non-empty finest box (engine.cpp:37-59 / :244-265).
void p2m_finest(const Pyramid& pyr, const std::vector<cplx>& zp, const std::vector<cplx>& mp,
                Kernel kernel, int p, int threads, std::vector<Expansion>& fexp) {
  const std::vector<MBox>& fine = pyr.finest();
#pragma omp parallel for schedule(dynamic) num_threads(threads)
  for (std::int64_t i = 0; i < std::int64_t(fine.size()); ++i) {
    const MBox& b = fine[i];
    if (b.n_points() == 0) continue;
    fexp[i] = p2m(b.center, std::span<const cplx>(zp.data() + b.point_begin, b.n_points()),
                  std::span<const cplx>(mp.data() + b.point_begin, b.n_points()), kernel, p);
  }
}

// Serial M2M chain: parent = sum of its shifted children (engine.cpp:61-80).
void m2m_chain(const Pyramid& pyr, Kernel kernel, int p, ExpansionPyramid& out) {
  for (int l = pyr.finest_level() - 1; l >= 0; --l) {
    for (std::size_t i = 0; i < pyr.levels[l].size(); ++i) {
      const MBox& b = pyr.levels[l][i];
      if (b.n_points() == 0) continue;
      Expansion& acc = out.levels[l][i];
      acc = fresh(b.center, Expansion::Kind::outgoing, kernel, p);
      for (std::size_t c = 4 * i; c < 4 * i + 4; ++c) {
        const Expansion& kid = out.levels[l + 1][c];
        if (kid.coeffs.empty()) continue;
        const Expansion moved = m2m(kid, b.center);
        for (int k = 0; k <= p; ++k) acc.coeffs[k] += moved.coeffs[k];
      }
    }
  }
}

struct Downward {
  const Pyramid& pyr;
  const Connectivity& conn;
  const ExpansionPyramid& out;
  ExpansionPyramid& loc;
  Kernel kernel;
  int p;
};

// Local of one box: L2L from the parent (l >= 2), then M2L from each weak
// partner with content, ascending (engine.cpp:96-114).
void local_of(Downward& d, int l, std::uint32_t i, std::uint64_t& ops) {
  const MBox& b = d.pyr.levels[l][i];
  if (b.n_evals() == 0) return;
  Expansion& me = d.loc.levels[l][i];
  me = fresh(b.center, Expansion::Kind::ingoing, d.kernel, d.p);
  if (l >= 2) {
    const Expansion& up = d.loc.levels[l - 1][i / 4];
    if (!up.coeffs.empty()) l2l_add(up, me);
  }
  for (std::uint32_t w : d.conn.levels[l].weak[i]) {
    const Expansion& src = d.out.levels[l][w];
    if (src.coeffs.empty()) continue;
    m2l_add(src, me);
    ++ops;
  }
}

void subtree(Downward& d, int l, std::uint32_t i, std::uint64_t& ops) {
  if (l + 1 >= d.pyr.n_levels || d.pyr.levels[l][i].n_evals() == 0) return;
  for (std::uint32_t c = 4 * i; c < 4 * i + 4; ++c) {
    local_of(d, l + 1, c, ops);
    subtree(d, l + 1, c, ops);
  }
}

ExpansionPyramid empty_like(const Pyramid& pyr) {
  ExpansionPyramid e;
  e.levels.resize(pyr.n_levels);
  for (int l = 0; l < pyr.n_levels; ++l) e.levels[l].resize(pyr.levels[l].size());
  return e;
}

// Device M2L (hybrid path): every level's expansions and weak lists are
// flattened in parallel straight into the backend's page-locked buffers
// (DMA'd in place), the batched M2L runs on the device (m2l_reg_kernel) while
// the CPU waits on nothing else, and the host L2L chain adds the sums.
struct DeviceM2L {
  CudaBackend::M2LBuffers b;
  std::uint32_t n_boxes = 0, n_targets = 0;
  std::vector<std::uint32_t> level_base;  // global id of box 0 of level l
  std::vector<std::int64_t> slot;         // global box id -> target row (-1 if none)
  // device downward pass (default; FMM_HOST_L2L=1: L2L on the host): the
  // finest level's locals land in b.out, row = finest box index
  bool device_l2l = false;
  std::vector<std::int32_t> target_of;    // slot as int32 for fmmcu_m2l_downward
};

void device_m2l_launch(CudaBackend& be, const Pyramid& pyr, const Connectivity& conn,
                       const ExpansionPyramid& out, Kernel kernel, int p, int threads,
                       DeviceM2L& dm) {
  static const bool trace = std::getenv("FMM_TRACE") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[fmm]   m2l flatten: %-16s %.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  const int L = pyr.n_levels;
  dm.level_base.assign(L + 1, 0);
  for (int l = 0; l < L; ++l)
    dm.level_base[l + 1] = dm.level_base[l] + std::uint32_t(pyr.levels[l].size());
  const std::uint32_t nb = dm.level_base[L];
  const std::size_t P1 = std::size_t(p) + 1;
  // Global box g = level_base[l] + i.  One parallel region per pass over
  // all levels' boxes: nonempty flags (a byte per box: the weak-list scans
  // then read bytes, not Expansion objects), then per target its nonempty
  // weak partners; prefix sums (serial, cheap); then the fill.
  auto level_of = [&](std::uint32_t g) {
    return int(std::upper_bound(dm.level_base.begin(), dm.level_base.end(), g) -
               dm.level_base.begin()) - 1;
  };
  std::vector<std::uint32_t> tcnt(std::size_t(nb) + 1, 0), wcnt(std::size_t(nb) + 1, 0);
  std::vector<std::uint8_t> nonempty(nb);
  std::uint32_t n_empty = 0;
#pragma omp parallel num_threads(threads)
  {
#pragma omp for schedule(static) reduction(+ : n_empty)
    for (std::int64_t g = 0; g < std::int64_t(nb); ++g) {
      const int l = level_of(std::uint32_t(g));
      nonempty[g] = out.levels[l][std::uint32_t(g) - dm.level_base[l]].coeffs.empty() ? 0 : 1;
      n_empty += nonempty[g] ? 0u : 1u;
    }
    // (every box has sources -- uniform inputs -- : the weak lists are taken
    // whole, no per-partner test)
#pragma omp for schedule(static)
    for (std::int64_t g = dm.level_base[std::min(1, L)]; g < std::int64_t(nb); ++g) {
      const int l = level_of(std::uint32_t(g));
      const std::uint32_t base = dm.level_base[l], i = std::uint32_t(g) - base;
      if (pyr.levels[l][i].n_evals() == 0) continue;
      const std::vector<std::uint32_t>& wl = conn.levels[l].weak[i];
      std::uint32_t k = std::uint32_t(wl.size());
      if (n_empty) {
        k = 0;
        for (std::uint32_t w : wl) k += nonempty[base + w];
      }
      tcnt[g + 1] = 1;
      wcnt[g + 1] = k;
    }
  }
  for (std::uint32_t g = 0; g < nb; ++g) {
    tcnt[g + 1] += tcnt[g];
    wcnt[g + 1] += wcnt[g];
  }
  mark("count + prefix");
  dm.n_boxes = nb;
  dm.n_targets = tcnt[nb];
  static const bool host_l2l = std::getenv("FMM_HOST_L2L") != nullptr;
  dm.device_l2l = !host_l2l && L >= 2;
  const std::uint32_t n_fin = dm.level_base[L] - dm.level_base[L - 1];
  // out holds the sums ([n_targets][p+1]) or, with the device downward
  // pass, the finest locals ([n_fin][p+1])
  dm.b = be.m2l_buffers(nb, p, dm.device_l2l ? std::max(dm.n_targets, n_fin) : dm.n_targets,
                        wcnt[nb]);
  dm.slot.assign(nb, -1);
  dm.target_of.resize(nb);
  const CudaBackend::M2LBuffers& b = dm.b;
  b.weak_off[0] = 0;
#pragma omp parallel for schedule(static) num_threads(threads)
  for (std::int64_t gg = 0; gg < std::int64_t(nb); ++gg) {
    const std::uint32_t g = std::uint32_t(gg);
    const int l = level_of(g);
    const std::uint32_t base = dm.level_base[l], i = g - base;
    b.centers[g] = pyr.levels[l][i].center;
    const Expansion& e = out.levels[l][i];
    cplx* dst = b.coeffs + std::size_t(g) * P1;
    if (nonempty[g]) std::copy(e.coeffs.begin(), e.coeffs.end(), dst);
    else std::fill(dst, dst + P1, cplx(0, 0));
    if (tcnt[g + 1] == tcnt[g]) {  // not a target
      dm.target_of[g] = -1;
      continue;
    }
    const std::uint32_t t = tcnt[g];
    dm.slot[g] = std::int64_t(t);
    dm.target_of[g] = std::int32_t(t);
    b.target_box[t] = g;
    std::uint32_t o = wcnt[g];
    if (n_empty) {
      for (std::uint32_t w : conn.levels[l].weak[i])
        if (nonempty[base + w]) b.weak_idx[o++] = base + w;
    } else {
      for (std::uint32_t w : conn.levels[l].weak[i]) b.weak_idx[o++] = base + w;
    }
    b.weak_off[t + 1] = o;
  }
  mark("fill");
  if (!dm.device_l2l) {
    be.m2l_launch(p, kernel, nb, dm.n_targets, b);
    return;
  }
  be.m2l_launch_keep(p, kernel, nb, dm.n_targets, b);
  mark("launch");
  be.m2l_downward(L, dm.level_base.data(), dm.target_of.data(), b.out);
  mark("downward");
}

// Host half of the device downward pass: L2L chain + device M2L sums.
ExpansionPyramid device_m2l_assemble(const Pyramid& pyr, const DeviceM2L& dm, Kernel kernel,
                                     int p, int threads) {
  ExpansionPyramid loc = empty_like(pyr);
  const std::size_t P1 = std::size_t(p) + 1;
  for (int l = 1; l < pyr.n_levels; ++l) {
    const std::int64_t n = std::int64_t(pyr.levels[l].size());
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
    for (std::int64_t i = 0; i < n; ++i) {
      const MBox& b = pyr.levels[l][i];
      if (b.n_evals() == 0) continue;
      Expansion& me = loc.levels[l][i];
      me = fresh(b.center, Expansion::Kind::ingoing, kernel, p);
      if (l >= 2) {
        const Expansion& up = loc.levels[l - 1][i / 4];
        if (!up.coeffs.empty()) l2l_add(up, me);
      }
      const std::int64_t row = dm.slot[dm.level_base[l] + std::uint32_t(i)];
      const cplx* s = dm.b.out + std::size_t(row) * P1;
      for (std::size_t k = 0; k < P1; ++k) me.coeffs[k] += s[k];
    }
  }
  return loc;
}

}  // namespace

int FmmConfig::expansion_order() const {
  if (p_override > 0) return std::min(p_override, kMaxOrder);
  return choose_p(p_rule, tol, theta, p_calibration);
}

// engine.cpp:24-35 (closed forms for a uniform unit square)
CostEstimate estimate_cost(double n, int n_levels, double theta, int p) {
  if (!(n > 0) || n_levels < 1 || !(theta > 0.0 && theta < 1.0) || p < 1)
    throw InvalidParameter("estimate_cost: invalid parameters");
  const double leaves = std::pow(4.0, n_levels - 1);
  const double ring = M_PI * std::pow((1.0 + theta) / theta, 2.0);
  const double pp = double(p) * p;
  CostEstimate c;
  c.c_p2p = n * n / (2.0 * leaves) * ring;
  c.c_m2l = 1.5 * leaves * pp * ring;
  c.c_m2m = (4.0 / 3.0) * leaves * pp;
  c.c_p2m = n * p;
  return c;
}

ExpansionPyramid upward_pass(const Pyramid& pyr, const std::vector<cplx>& src_z_perm,
                             const std::vector<cplx>& src_m_perm, Kernel kernel, int p,
                             int threads, WorkCounters* counters) {
  ExpansionPyramid out = empty_like(pyr);
  p2m_finest(pyr, src_z_perm, src_m_perm, kernel, p, threads, out.levels[pyr.finest_level()]);
  if (counters) counters->p2m_points += src_z_perm.size();
  m2m_chain(pyr, kernel, p, out);
  return out;
}

// engine.cpp:127-169: serial breadth-first walk to the split level, then one
// OpenMP task per split-level subtree (no shared mutable state).
ExpansionPyramid downward_pass(const Pyramid& pyr, const Connectivity& conn,
                               const ExpansionPyramid& outgoing, int p, int task_split_level,
                               int threads, WorkCounters* counters) {
  ExpansionPyramid loc = empty_like(pyr);
  Kernel kernel = outgoing.levels[0][0].kernel;
  if (outgoing.levels[0][0].coeffs.empty()) kernel = Kernel::harmonic;
  Downward d{pyr, conn, outgoing, loc, kernel, p};
  const int split = std::max(0, std::min(task_split_level, pyr.n_levels - 1));
  std::uint64_t ops = 0;
  for (int l = 1; l <= split; ++l)
    for (std::uint32_t i = 0; i < pyr.levels[l].size(); ++i) local_of(d, l, i, ops);
  const std::uint32_t roots = std::uint32_t(pyr.levels[split].size());
  if (threads > 1 && split < pyr.n_levels - 1) {
#pragma omp parallel num_threads(threads)
#pragma omp single
    for (std::uint32_t i = 0; i < roots; ++i) {
#pragma omp task firstprivate(i)
      {
        std::uint64_t mine = 0;
        subtree(d, split, i, mine);
#pragma omp atomic
        ops += mine;
      }
    }
  } else {
    for (std::uint32_t i = 0; i < roots; ++i) subtree(d, split, i, ops);
  }
  if (counters) counters->m2l_ops += ops;
  return loc;
}

namespace {

void permute_inputs(const Pyramid& pyr, const SourceSet& s, const EvalSet& e, int threads,
                    std::vector<cplx>& zp, std::vector<cplx>& mp, std::vector<cplx>& yp,
                    std::vector<std::int64_t>& sidp) {
  // huge pages, populated from all cores: the value-initialising resize of
  // four 80-160 MB vectors was ~200 ms of page faults at 10M
  detail::resize_huge(zp, s.size());
  detail::resize_huge(mp, s.size());
#pragma omp parallel for schedule(static) num_threads(threads)
  for (std::int64_t i = 0; i < std::int64_t(s.size()); ++i) {
    zp[i] = s.z[pyr.perm[i]];
    mp[i] = s.m[pyr.perm[i]];
  }
  detail::resize_huge(yp, e.size());
  sidp.clear();
  if (!e.source_id.empty()) detail::resize_huge(sidp, e.size());
#pragma omp parallel for schedule(static) num_threads(threads)
  for (std::int64_t i = 0; i < std::int64_t(e.size()); ++i) {
    yp[i] = e.y[pyr.eval_perm[i]];
    if (!sidp.empty()) sidp[i] = e.source_id[pyr.eval_perm[i]];
  }
}

}  // namespace

// engine.cpp:171-194
std::vector<cplx> nearfield_eval(NearFieldBackend& backend, const Pyramid& pyr,
                                 const Connectivity& conn, const SourceSet& sources,
                                 const EvalSet& evals, Kernel kernel, const Smoother& smoother) {
  std::vector<cplx> zp, mp, yp;
  std::vector<std::int64_t> sidp;
  permute_inputs(pyr, sources, evals, 1, zp, mp, yp, sidp);
  NearFieldJob job{&pyr, &conn.finest(), &zp, &mp, &yp, &sidp, kernel, smoother, 1};
  std::vector<cplx> near;
  backend.launch(job, near);
  backend.finish();
  std::vector<cplx> out(evals.size());
  for (std::size_t i = 0; i < evals.size(); ++i) out[pyr.eval_perm[i]] = near[i];
  return out;
}

FmmEngine::FmmEngine(FmmConfig cfg) : cfg_(std::move(cfg)), backend_kind_(cfg_.backend) {
  backend_ = make_backend(cfg_.backend, cfg_.throttle, cfg_.cuda);
}

FmmEngine::~FmmEngine() = default;

void FmmEngine::set_config(const FmmConfig& cfg) {
  const bool devices_changed = cfg.backend == BackendKind::cuda &&
                               (cfg.cuda.devices != cfg_.cuda.devices || cfg.cuda.exact != cfg_.cuda.exact);
  if (cfg.backend != backend_kind_ || devices_changed) {
    backend_ = make_backend(cfg.backend, cfg.throttle, cfg.cuda);
    backend_kind_ = cfg.backend;
  }
  cfg_ = cfg;
}

EvalResult FmmEngine::evaluate(const SourceSet& sources, const EvalSet& evals) {
  EvalResult res;
  evaluate_into(sources, evals, res);
  return res;
}

void FmmEngine::evaluate_into(const SourceSet& sources, const EvalSet& evals, EvalResult& res) {
  if (!(cfg_.theta > 0.0 && cfg_.theta < 1.0)) throw InvalidParameter("evaluate: theta outside (0,1)");
  if (cfg_.n_levels < 1) throw InvalidParameter("evaluate: n_levels < 1");
  if (cfg_.worker_threads < 1) throw InvalidParameter("evaluate: worker_threads < 1");
  if (cfg_.p_override <= 0 && !(cfg_.tol > 0.0 && cfg_.tol < 1.0))
    throw InvalidParameter("evaluate: tol outside (0,1)");
  if (sources.size() == 0) throw InvalidInput("evaluate: empty source set");
  if (cfg_.m2l_on_device && cfg_.backend != BackendKind::cuda)
    throw InvalidParameter("evaluate: m2l_on_device requires the cuda backend");

  if (cfg_.device_pipeline && cfg_.backend != BackendKind::cuda)
    throw InvalidParameter("evaluate: device_pipeline requires the cuda backend");

  res.timings = PhaseTimings{};
  res.counters = WorkCounters{};
  res.p = cfg_.expansion_order();
  const int p = res.p;
  const int threads = cfg_.worker_threads;
  PhaseTimings& T = res.timings;
  const auto t_start = Clock::now();

  if (cfg_.device_pipeline) {
    // everything on the first device (fmmcu_fmm_evaluate); the reference's
    // phase split is reported from device event spans
    auto* cb = dynamic_cast<CudaBackend*>(backend_.get());
    CudaBackend::DeviceEval d;
    try {
      d = cb->fmm_evaluate(sources, evals, cfg_.n_levels, cfg_.theta, p, cfg_.kernel,
                           cfg_.smoother, res.potentials);
    } catch (const SingularConfiguration&) {
      throw;
    } catch (const InvalidInput&) {
      throw;
    } catch (const std::exception& e) {
      throw BackendError("device pipeline", e.what());
    }
    res.counters = d.counters;
    T.t_partition = d.t_upload + d.t_tree + d.t_connect;
    T.t_p2m = d.t_p2m_upward;
    T.t_upward = 0.0;
    T.t_m2l = d.t_m2l;
    T.t_p2p = d.t_p2p;
    T.t_total = since(t_start);
    T.t_q = T.t_partition + T.t_p2m + T.t_upward +
            std::max(0.0, d.t_device - T.t_partition - std::max(T.t_p2p, T.t_p2m + T.t_m2l));
    // The reference's wait signal (engine.cpp:312) is the time the far field
    // spent waiting on the near field. Here both branches run on the device,
    // so it is the far stream's idle tail before the P2P ends (device
    // events): positive when the near field is longer, zero otherwise, the
    // sign AT3a steers the level count by (autotune.cpp:155).
    T.cpu_wait = d.t_far_wait;
    if (observer_) observer_(*this, res);
    return;
  }

  // ---- partition ------------------------------------------------------------
  // (device_tree: the same pyramid and lists built on the GPU and read back)
  Pyramid pyr;
  Connectivity conn;
  if (cfg_.device_tree && cfg_.backend == BackendKind::cuda) {
    auto* cb = dynamic_cast<CudaBackend*>(backend_.get());
    try {
      cb->device_tree(sources, evals, cfg_.n_levels, cfg_.theta, pyr, conn);
    } catch (const InvalidInput&) {
      throw;
    } catch (const std::exception& e) {
      throw BackendError("device tree", e.what());
    }
  } else {
    pyr = build_pyramid(sources, evals, cfg_.n_levels, threads);
    conn = build_connectivity(pyr, cfg_.theta);
  }
  std::vector<cplx> zp, mp, yp;
  std::vector<std::int64_t> sidp;
  const double t_tree = since(t_start);
  permute_inputs(pyr, sources, evals, threads, zp, mp, yp, sidp);
  T.t_partition = since(t_start);
  static const bool trace_part = std::getenv("FMM_TRACE") != nullptr;
  if (trace_part)
    std::fprintf(stderr, "[fmm] partition: tree + lists %.2f ms, permute %.2f ms\n", 1e3 * t_tree,
                 1e3 * (T.t_partition - t_tree));

  // ---- upward -------------------------------------------------------------
  const auto t_p2m = Clock::now();
  ExpansionPyramid outgoing = empty_like(pyr);
  p2m_finest(pyr, zp, mp, cfg_.kernel, p, threads, outgoing.levels[pyr.finest_level()]);
  res.counters.p2m_points += sources.size();
  T.t_p2m = since(t_p2m);
  const auto t_up = Clock::now();
  m2m_chain(pyr, cfg_.kernel, p, outgoing);
  T.t_upward = since(t_up);

  // ---- near field || downward ----------------------------------------------
  NearFieldJob job{&pyr, &conn.finest(), &zp, &mp, &yp, &sidp, cfg_.kernel, cfg_.smoother, threads};
  std::vector<cplx> near;
  try {
    backend_->launch(job, near);
  } catch (const std::exception& e) {
    throw BackendError("nearfield launch", e.what());
  }

  const auto t_m2l = Clock::now();
  ExpansionPyramid locals;
  DeviceM2L dm;  // (device downward pass: the finest locals stay in dm.b.out)
  if (cfg_.m2l_on_device) {
    auto* cb = dynamic_cast<CudaBackend*>(backend_.get());
    static const bool trace = std::getenv("FMM_TRACE") != nullptr;
    try {
      device_m2l_launch(*cb, pyr, conn, outgoing, cfg_.kernel, p, threads, dm);
      const double t_fl = since(t_m2l);
      double dev_s = 0.0;
      res.counters.m2l_ops += cb->m2l_finish(&dev_s);
      if (trace)
        std::fprintf(stderr, "[fmm] hybrid m2l: flatten+launch %.2f ms, finish at %.2f ms "
                     "(device span %.2f ms)\n", 1e3 * t_fl, 1e3 * since(t_m2l), 1e3 * dev_s);
    } catch (const SingularConfiguration&) {
      try {
        backend_->finish();
      } catch (...) {
      }
      throw;
    } catch (const std::exception& e) {
      try {
        backend_->finish();
      } catch (...) {
      }
      throw BackendError("m2l", e.what());
    }
    if (!dm.device_l2l) {
      locals = device_m2l_assemble(pyr, dm, cfg_.kernel, p, threads);
      if (trace)
        std::fprintf(stderr, "[fmm] hybrid m2l: assembled at %.2f ms\n", 1e3 * since(t_m2l));
    }
  } else {
    locals = downward_pass(pyr, conn, outgoing, p, cfg_.task_split_level, threads, &res.counters);
  }
  T.t_m2l = since(t_m2l);

  const auto t_join = Clock::now();
  NearFieldStats nf;
  try {
    nf = backend_->finish();
  } catch (const std::exception& e) {
    throw BackendError("nearfield", e.what());
  }
  T.cpu_wait = backend_->concurrent() ? since(t_join) : 0.0;
  T.t_p2p = nf.seconds;
  res.counters.p2p_pairs += nf.pair_evals;

  // ---- assembly (engine.cpp:316-339) -----------------------------------------
  const auto t_asm = Clock::now();
  const std::vector<MBox>& fine = pyr.finest();
  res.potentials.resize(evals.size());
  std::uint64_t l2p = 0;
  if (dm.device_l2l) {
    // the finest locals from the device downward pass, flat ([box][p+1]);
    // Horner exactly as eval_local (expansion.cpp)
    const cplx* fl = dm.b.out;
    const std::int32_t* tof = dm.target_of.data() + dm.level_base[pyr.finest_level()];
    const std::size_t P1 = std::size_t(p) + 1;
#pragma omp parallel for schedule(dynamic) reduction(+ : l2p) num_threads(threads)
    for (std::int64_t i = 0; i < std::int64_t(fine.size()); ++i) {
      const MBox& b = fine[i];
      const bool far = tof[i] >= 0;
      const cplx* c = fl + std::size_t(i) * P1;
      for (std::uint32_t e = b.eval_begin; e < b.eval_end; ++e) {
        cplx v = near[e];
        if (far) {
          const cplx d = yp[e] - b.center;
          cplx s(0, 0);
          for (int k = p; k >= 0; --k) s = s * d + c[k];
          v = near[e] + s;
        }
        res.potentials[pyr.eval_perm[e]] = v;
      }
      if (far) l2p += b.n_evals();
    }
  } else {
    const std::vector<Expansion>& floc = locals.levels[pyr.finest_level()];
#pragma omp parallel for schedule(dynamic) reduction(+ : l2p) num_threads(threads)
    for (std::int64_t i = 0; i < std::int64_t(fine.size()); ++i) {
      const MBox& b = fine[i];
      const Expansion& loc = floc[i];
      const bool far = !loc.coeffs.empty();
      for (std::uint32_t e = b.eval_begin; e < b.eval_end; ++e) {
        const cplx v = far ? near[e] + eval_local(loc, yp[e]) : near[e];
        res.potentials[pyr.eval_perm[e]] = v;
      }
      if (far) l2p += b.n_evals();
    }
  }
  res.counters.l2p_points += l2p;
  const double t_assembly = since(t_asm);
  T.t_q = T.t_partition + T.t_p2m + T.t_upward + t_assembly;
  T.t_total = since(t_start);
  if (observer_) observer_(*this, res);
  return;
}

}  // namespace fmm
