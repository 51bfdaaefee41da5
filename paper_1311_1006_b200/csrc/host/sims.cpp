// fmm-b200 — vortex-sheet driver (reference proj/src/sims.cpp:13-89).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "fmm/sims.hpp"
#include "fmm_cuda.h"

namespace fmm::sims {

namespace {

// 1 / (2 pi i) = -i / (2 pi)
const cplx kOneOverTwoPiI = cplx(0.0, -1.0) / (2.0 * M_PI);

void use_vortex_kernel(FmmEngine& engine, double delta) {
  FmmConfig cfg = engine.config();
  const bool same = cfg.kernel == Kernel::harmonic &&
                    cfg.smoother.kind == Smoother::Kind::gaussian && cfg.smoother.delta == delta;
  if (same) return;
  cfg.kernel = Kernel::harmonic;
  cfg.smoother = Smoother::gaussian(delta);
  engine.set_config(cfg);
}

// Per-thread step buffers.  With the cuda backend their storage is
// page-locked (fmmcu_pin_host) so the device pipeline DMAs the sources and
// the potentials in place; unpinned before any reallocation and at thread
// exit.
struct StepBuffers {
  SourceSet src;
  EvalSet ev;
  EvalResult r;
  void* p[4] = {};
  std::size_t b[4] = {};
  std::int64_t ids_n = -1;  // ev.source_id holds 0..ids_n-1
  ~StepBuffers() { unpin(); }
  void unpin() {
    for (int i = 0; i < 4; ++i) {
      if (p[i]) fmmcu_unpin_host(p[i]);
      p[i] = nullptr;
      b[i] = 0;
    }
  }
  void pin() {
    void* ptr[4] = {src.z.data(), src.m.data(), ev.y.data(), r.potentials.data()};
    const std::size_t bytes[4] = {src.z.size() * 16, src.m.size() * 16, ev.y.size() * 16,
                                  r.potentials.size() * 16};
    for (int i = 0; i < 4; ++i) {
      if (p[i] == ptr[i] && b[i] == bytes[i]) continue;
      if (p[i]) fmmcu_unpin_host(p[i]);
      p[i] = nullptr;
      b[i] = 0;
      if (bytes[i] >= (std::size_t(1) << 20) && fmmcu_pin_host(ptr[i], bytes[i]) == FMMCU_OK) {
        p[i] = ptr[i];
        b[i] = bytes[i];
      }
    }
  }
};

}  // namespace

double smoother(double r, double delta) {
  if (!(delta > 0.0)) throw InvalidParameter("smoother: delta must be > 0");
  if (r < 0.0) throw InvalidParameter("smoother: r must be >= 0");
  return 1.0 - std::exp(-(r * r) / (delta * delta));
}

double VortexSystem::total_circulation() const {
  return std::accumulate(gamma.begin(), gamma.end(), 0.0);
}

VortexSystem init_shear_layer(int n, double aspect, double gamma) {
  if (n < 2 || n % 2 != 0) throw InvalidParameter("init_shear_layer: n must be even and >= 2");
  if (!(aspect > 0.0)) throw InvalidParameter("init_shear_layer: aspect must be > 0");
  // rows: even, divides n, near sqrt(n / aspect)
  int rows = int(std::lround(std::sqrt(double(n) / aspect)));
  rows = std::max(2, rows - rows % 2);
  while (n % rows != 0) rows -= 2;
  const int cols = n / rows;
  const double width = aspect, height = 1.0;
  VortexSystem sys;
  sys.pos.reserve(n);
  sys.gamma.reserve(n);
  for (int r = 0; r < rows / 2; ++r) {
    const double y_low = -0.5 * height + (r + 0.5) * height / rows;
    const double y_high = -0.5 * height + (r + rows / 2 + 0.5) * height / rows;
    for (int c = 0; c < cols; ++c) {
      const double x = -0.5 * width + (c + 0.5) * width / cols;
      sys.pos.emplace_back(x, y_low);
      sys.gamma.push_back(-gamma);
      sys.pos.emplace_back(x, y_high);
      sys.gamma.push_back(gamma);
    }
  }
  sys.delta = 2.0 * width / cols;
  sys.dt = 0.5 * height / rows;
  return sys;
}

namespace {
// Sources / self evals of the system in the thread's step buffers, then one
// evaluation into B.r (shared by vortex_velocities and vortex_step).
StepBuffers& evaluate_system(const VortexSystem& sys, FmmEngine& engine, bool prefilled = false) {
  use_vortex_kernel(engine, sys.delta);
  // Time stepping evaluates one problem size over and over: the sources, the
  // (self) evals and the result live in per-thread buffers that are refilled
  // in parallel, and evaluate_into() reuses the result storage.  Same values
  // as building them afresh (reference sims.cpp:66-84).
  thread_local StepBuffers tl;
  // plain references: inside the OpenMP regions a thread_local name would
  // denote each worker's own (empty) copy
  StepBuffers& B = tl;
  SourceSet& src = B.src;
  EvalSet& ev = B.ev;
  EvalResult& r = B.r;
  const std::int64_t n = std::int64_t(sys.size());
  const bool cuda = engine.config().backend == BackendKind::cuda;
  if (!cuda || src.z.capacity() < std::size_t(n) || r.potentials.capacity() < std::size_t(n))
    B.unpin();  // never free registered storage
  src.z.resize(n);
  src.m.resize(n);
  ev.y.resize(n);
  // the ids are 0..n-1 every step: rewritten only when the size changes
  const bool ids = B.ids_n != n || ev.source_id.size() != std::size_t(n);
  ev.source_id.resize(n);
  if (cuda) {
    r.potentials.resize(n);  // evaluate_into keeps storage of the right size
    B.pin();
  }
  int64_t* sid = ev.source_id.data();
  // prefilled (vortex_steps): the previous step's update already wrote the
  // positions into src.z / ev.y, and the strengths have not changed
  if (!prefilled || ids) {
#pragma omp parallel for schedule(static)
    for (std::int64_t k = 0; k < n; ++k) {
      src.z[k] = sys.pos[k];
      src.m[k] = sys.gamma[k] * kOneOverTwoPiI;
      ev.y[k] = sys.pos[k];
      if (ids) sid[k] = k;
    }
  }
  B.ids_n = n;
  engine.evaluate_into(src, ev, r);
  return B;
}
}  // namespace

std::vector<cplx> vortex_velocities(const VortexSystem& sys, FmmEngine& engine, EvalResult* info) {
  if (sys.size() == 0) return {};
  if (sys.size() == 1) {
    if (info) *info = EvalResult{};
    return {cplx(0, 0)};
  }
  const EvalResult& r = evaluate_system(sys, engine).r;
  const std::int64_t n = std::int64_t(sys.size());
  std::vector<cplx> v(n);
#pragma omp parallel for schedule(static)
  for (std::int64_t k = 0; k < n; ++k) v[k] = std::conj(r.potentials[k]);
  if (info) *info = r;
  return v;
}

// steps x vortex_step with the next step's inputs written by the update
// (pos, src.z and ev.y in one pass; the strengths are constant): the system
// is not visible between the steps, so nothing else can change it.
void vortex_steps(VortexSystem& sys, FmmEngine& engine, int steps) {
  if (sys.size() < 2 || steps <= 0) return;
  const std::int64_t n = std::int64_t(sys.size());
  for (int s = 0; s < steps; ++s) {
    StepBuffers& B = evaluate_system(sys, engine, s > 0);
    const cplx* pot = B.r.potentials.data();
    cplx* z = B.src.z.data();
    cplx* y = B.ev.y.data();
#pragma omp parallel for schedule(static)
    for (std::int64_t k = 0; k < n; ++k) {
      const cplx p = sys.pos[k] + sys.dt * std::conj(pot[k]);
      sys.pos[k] = p;
      z[k] = p;
      y[k] = p;
    }
  }
}

// euler_step(sys, vortex_velocities(sys, engine)) without the velocity
// vector (a fresh 16 B/vortex allocation, zero-filled by one thread, every
// step): pos += dt * conj(potential), the same arithmetic.
void vortex_step(VortexSystem& sys, FmmEngine& engine) {
  if (sys.size() < 2) return;  // one vortex: zero velocity
  static const bool trace = std::getenv("FMM_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  const EvalResult& r = evaluate_system(sys, engine).r;
  const auto t1 = std::chrono::steady_clock::now();
  const std::int64_t n = std::int64_t(sys.size());
  const cplx* pot = r.potentials.data();
#pragma omp parallel for schedule(static)
  for (std::int64_t k = 0; k < n; ++k) sys.pos[k] += sys.dt * std::conj(pot[k]);
  if (trace) {
    const auto t2 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[fmm] vortex step: fill+evaluate %.2f ms (t_total %.2f), update %.2f ms\n",
                 ms(t0, t1), 1e3 * r.timings.t_total, ms(t1, t2));
  }
}

void euler_step(VortexSystem& sys, const std::vector<cplx>& velocities) {
  if (velocities.size() != sys.size()) throw InvalidInput("euler_step: velocity count mismatch");
  const std::int64_t n = std::int64_t(sys.size());
#pragma omp parallel for schedule(static)
  for (std::int64_t k = 0; k < n; ++k) sys.pos[k] += sys.dt * velocities[k];
}

}  // namespace fmm::sims
