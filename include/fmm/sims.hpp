// fmm-b200 — vortex-sheet driver (the config-5 workload).
//
// Restates the vortex part of the reference proj/include/fmm/sims.hpp:12-36
// (sims.cpp:25-89).  The galaxy and cylinder drivers (sims.hpp:38-106) are
// out of scope: they are not on the near-field hot path and the cylinder
// needs Eigen.
#pragma once

#include <vector>

#include "fmm/engine.hpp"

namespace fmm::sims {

// 1 - exp(-r^2/delta^2); delta > 0, r >= 0 (sims.cpp:25-29).
double smoother(double r, double delta);

struct VortexSystem {
  std::vector<cplx> pos;
  std::vector<double> gamma;
  double delta = 0.05;
  double dt = 0.01;

  std::size_t size() const { return pos.size(); }
  double total_circulation() const;
};

// Shear layer on an aspect:1 lattice, lower half -gamma, upper +gamma,
// mirror rows interleaved so the circulation sums to exactly zero.
VortexSystem init_shear_layer(int n, double aspect, double gamma);

// conj of the smoothed harmonic potential of all other vortices
// (m_k = gamma_k / (2 pi i)); reconfigures the engine's kernel/smoother.
std::vector<cplx> vortex_velocities(const VortexSystem& sys, FmmEngine& engine,
                                    EvalResult* info = nullptr);

void euler_step(VortexSystem& sys, const std::vector<cplx>& velocities);

// euler_step(sys, vortex_velocities(sys, engine)) fused: same positions,
// without materialising the velocity vector (time-stepping drivers).
void vortex_step(VortexSystem& sys, FmmEngine& engine);
// `steps` vortex_step calls, each update also writing the next step's
// inputs (same positions, one pass less per step).
void vortex_steps(VortexSystem& sys, FmmEngine& engine, int steps);

}  // namespace fmm::sims
