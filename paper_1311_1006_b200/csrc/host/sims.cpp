// fmm-b200 — vortex-sheet driver (reference proj/src/sims.cpp:13-89).
#include <cmath>
#include <numeric>

#include "fmm/sims.hpp"

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

std::vector<cplx> vortex_velocities(const VortexSystem& sys, FmmEngine& engine, EvalResult* info) {
  if (sys.size() == 0) return {};
  if (sys.size() == 1) {
    if (info) *info = EvalResult{};
    return {cplx(0, 0)};
  }
  use_vortex_kernel(engine, sys.delta);
  SourceSet src;
  src.z = sys.pos;
  src.m.resize(sys.size());
  for (std::size_t k = 0; k < sys.size(); ++k) src.m[k] = sys.gamma[k] * kOneOverTwoPiI;
  EvalResult r = engine.evaluate(src, EvalSet::self_of(src));
  std::vector<cplx> v(sys.size());
  for (std::size_t k = 0; k < v.size(); ++k) v[k] = std::conj(r.potentials[k]);
  if (info) *info = std::move(r);
  return v;
}

void euler_step(VortexSystem& sys, const std::vector<cplx>& velocities) {
  if (velocities.size() != sys.size()) throw InvalidInput("euler_step: velocity count mismatch");
  for (std::size_t k = 0; k < sys.size(); ++k) sys.pos[k] += sys.dt * velocities[k];
}

}  // namespace fmm::sims
