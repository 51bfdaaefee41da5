// fmm-b200 — balanced pyramid and θ-connectivity (host, kept on the CPU).
//
// Contract: reference proj/src/geometry.cpp:13-216 / geometry.hpp:55-74.
// Output is bit-identical to the reference (tests/test_host_geometry.py):
//  * the low half of every split is the first ceil(n/2) points in the
//    strict total order (coordinate, original index) -- a set, so it does
//    not depend on the selection algorithm (reference: nth_element on perm,
//    geometry.cpp:44-63);
//  * evaluation points are split stably by `coord <= split value`
//    (geometry.cpp:60-61), so eval_perm is ascending inside every leaf;
//  * box extents/centres/radii use the same arithmetic (geometry.cpp:66-102);
//  * leaf-internal source order is ascending original index
//    (geometry.cpp:154-161).
// Implementation differs: points travel as contiguous {x, y, index}
// records so selection and partitioning stream through memory instead of
// gathering coordinates through the permutation, the two y-splits of a
// parent run in parallel, and connectivity is built per child box in
// parallel (each list emerges sorted; no post-sort).
#include <algorithm>
#include <cmath>
#include <limits>

#include "fmm/geometry.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace fmm {

bool theta_criterion(const MBox& a, const MBox& b, double theta) {
  if (!(theta > 0.0 && theta < 1.0))
    throw InvalidParameter("theta_criterion: theta outside (0,1)");
  const double r_big = std::max(a.radius, b.radius);
  const double r_small = std::min(a.radius, b.radius);
  const double dist = std::abs(a.center - b.center);
  return r_big + theta * r_small <= theta * dist;
}

namespace {

struct Rec {
  double x, y;
  std::uint32_t id;
};

inline double along(const Rec& r, bool x_axis) { return x_axis ? r.x : r.y; }

// Selects the low half of recs[b,e) in place; returns the split position
// and the split coordinate (fallback when the range is empty).
struct Cut {
  std::uint32_t mid;
  double value;
};

Cut select_low_half(std::vector<Rec>& recs, std::uint32_t b, std::uint32_t e, bool x_axis,
                    double fallback) {
  if (e == b) return {b, fallback};
  const std::uint32_t k = (e - b + 1) / 2;
  auto less = [x_axis](const Rec& p, const Rec& q) {
    const double cp = along(p, x_axis), cq = along(q, x_axis);
    if (cp != cq) return cp < cq;
    return p.id < q.id;
  };
  Rec* base = recs.data();
  std::nth_element(base + b, base + b + (k - 1), base + e, less);
  return {b + k, along(recs[b + k - 1], x_axis)};
}

// Stable two-way partition of evs[b,e) by coord <= value; returns the
// boundary.  tmp[b,e) is this range's private scratch.
std::uint32_t split_evals(std::vector<Rec>& evs, std::vector<Rec>& tmp, std::uint32_t b,
                          std::uint32_t e, bool x_axis, double value) {
  std::uint32_t lo = b, hi = 0;
  for (std::uint32_t i = b; i < e; ++i) {
    const Rec r = evs[i];
    if (along(r, x_axis) <= value)
      evs[lo++] = r;
    else
      tmp[b + hi++] = r;
  }
  std::copy(tmp.begin() + b, tmp.begin() + b + hi, evs.begin() + lo);
  return lo;
}

void fill_box(MBox& box, const std::vector<Rec>& src, const std::vector<Rec>& evs, cplx fallback) {
  if (box.point_begin == box.point_end && box.eval_begin == box.eval_end) {
    box.center = fallback;
    box.half_width = box.half_height = box.radius = 0.0;
    return;
  }
  double x0 = std::numeric_limits<double>::infinity(), x1 = -x0, y0 = x0, y1 = -x0;
  for (std::uint32_t i = box.point_begin; i < box.point_end; ++i) {
    x0 = std::min(x0, src[i].x);
    x1 = std::max(x1, src[i].x);
    y0 = std::min(y0, src[i].y);
    y1 = std::max(y1, src[i].y);
  }
  for (std::uint32_t i = box.eval_begin; i < box.eval_end; ++i) {
    x0 = std::min(x0, evs[i].x);
    x1 = std::max(x1, evs[i].x);
    y0 = std::min(y0, evs[i].y);
    y1 = std::max(y1, evs[i].y);
  }
  box.center = cplx(0.5 * (x0 + x1), 0.5 * (y0 + y1));
  box.half_width = 0.5 * (x1 - x0);
  box.half_height = 0.5 * (y1 - y0);
  box.radius = std::hypot(box.half_width, box.half_height);
}

}  // namespace

Pyramid build_pyramid(const SourceSet& sources, const EvalSet& evals, int n_levels, int threads) {
  if (n_levels < 1) throw InvalidParameter("build_pyramid: n_levels must be >= 1");
  if (sources.size() == 0) throw InvalidInput("build_pyramid: empty source set");
  for (const cplx& z : sources.z)
    if (!std::isfinite(z.real()) || !std::isfinite(z.imag()))
      throw InvalidInput("build_pyramid: non-finite source position");
  for (const cplx& y : evals.y)
    if (!std::isfinite(y.real()) || !std::isfinite(y.imag()))
      throw InvalidInput("build_pyramid: non-finite eval position");
  if (threads < 1) threads = 1;

  const std::uint32_t ns = static_cast<std::uint32_t>(sources.size());
  const std::uint32_t ne = static_cast<std::uint32_t>(evals.size());
  std::vector<Rec> src(ns), evs(ne);
#pragma omp parallel for schedule(static) num_threads(threads)
  for (std::int64_t i = 0; i < std::int64_t(ns); ++i)
    src[i] = Rec{sources.z[i].real(), sources.z[i].imag(), std::uint32_t(i)};
#pragma omp parallel for schedule(static) num_threads(threads)
  for (std::int64_t i = 0; i < std::int64_t(ne); ++i)
    evs[i] = Rec{evals.y[i].real(), evals.y[i].imag(), std::uint32_t(i)};

  Pyramid pyr;
  pyr.n_levels = n_levels;
  pyr.levels.resize(n_levels);
  MBox root;
  root.point_end = ns;
  root.eval_end = ne;
  fill_box(root, src, evs, cplx(0, 0));
  pyr.levels[0].push_back(root);

  std::vector<Rec> scratch(ne);
  for (int l = 1; l < n_levels; ++l) {
    const std::vector<MBox>& up = pyr.levels[l - 1];
    std::vector<MBox>& kids = pyr.levels[l];
    kids.resize(up.size() * 4);
    const std::int64_t np = std::int64_t(up.size());
    // Few huge parents near the root: parallelise inside the parent (the
    // two y-splits); many parents deeper down: parallelise across parents.
    const bool inner = np < threads;
#pragma omp parallel for schedule(dynamic) num_threads(threads) if (!inner)
    for (std::int64_t pi = 0; pi < np; ++pi) {
      const MBox& par = up[pi];
      const Cut cx = select_low_half(src, par.point_begin, par.point_end, true, par.center.real());
      const std::uint32_t emx =
          split_evals(evs, scratch, par.eval_begin, par.eval_end, true, cx.value);
      Cut cyl{}, cyh{};
      std::uint32_t emyl = 0, emyh = 0;
#pragma omp parallel sections num_threads(2) if (inner)
      {
#pragma omp section
        {
          cyl = select_low_half(src, par.point_begin, cx.mid, false, par.center.imag());
          emyl = split_evals(evs, scratch, par.eval_begin, emx, false, cyl.value);
        }
#pragma omp section
        {
          cyh = select_low_half(src, cx.mid, par.point_end, false, par.center.imag());
          emyh = split_evals(evs, scratch, emx, par.eval_end, false, cyh.value);
        }
      }
      const std::uint32_t pb[5] = {par.point_begin, cyl.mid, cx.mid, cyh.mid, par.point_end};
      const std::uint32_t eb[5] = {par.eval_begin, emyl, emx, emyh, par.eval_end};
      for (int c = 0; c < 4; ++c) {
        MBox& kid = kids[4 * pi + c];
        kid.level = l;
        kid.index_in_level = std::uint32_t(4 * pi + c);
        kid.point_begin = pb[c];
        kid.point_end = pb[c + 1];
        kid.eval_begin = eb[c];
        kid.eval_end = eb[c + 1];
        fill_box(kid, src, evs, par.center);
      }
    }
  }

  // Canonical (ascending original index) order of sources inside each leaf.
  const std::vector<MBox>& fine = pyr.levels.back();
  pyr.perm.resize(ns);
  pyr.eval_perm.resize(ne);
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
  for (std::int64_t i = 0; i < std::int64_t(fine.size()); ++i) {
    const MBox& b = fine[i];
    for (std::uint32_t k = b.point_begin; k < b.point_end; ++k) pyr.perm[k] = src[k].id;
    std::sort(pyr.perm.begin() + b.point_begin, pyr.perm.begin() + b.point_end);
    for (std::uint32_t k = b.eval_begin; k < b.eval_end; ++k) pyr.eval_perm[k] = evs[k].id;
  }
  return pyr;
}

LevelConn classify_level(const LevelConn& parent, const Pyramid& pyramid, int level,
                         double theta) {
  LevelConn out;
  if (level == 0) {
    out.strong.assign(1, std::vector<std::uint32_t>{0});
    out.weak.resize(1);
    return out;
  }
  if (level < 1 || level >= pyramid.n_levels)
    throw InvalidParameter("classify_level: level out of range");
  if (!(theta > 0.0 && theta < 1.0))
    throw InvalidParameter("theta_criterion: theta outside (0,1)");
  const std::vector<MBox>& boxes = pyramid.levels[level];
  const std::int64_t n = std::int64_t(boxes.size());
  out.strong.resize(n);
  out.weak.resize(n);
  // Child a of parent p meets every child b of every q strongly connected
  // to p.  q ascends and b = 4q..4q+3 ascends, so both lists come out
  // sorted; the θ test is symmetric, so the lists are symmetric.
#pragma omp parallel for schedule(dynamic, 256)
  for (std::int64_t a = 0; a < n; ++a) {
    const std::uint32_t p = std::uint32_t(a / 4);
    const auto& nbrs = parent.strong[p];
    auto& s = out.strong[a];
    auto& w = out.weak[a];
    s.reserve(nbrs.size() * 4);
    for (std::uint32_t q : nbrs) {
      for (std::uint32_t b = 4 * q; b < 4 * q + 4; ++b) {
        if (b == std::uint32_t(a)) {
          s.push_back(b);
          continue;
        }
        const MBox& A = boxes[a];
        const MBox& B = boxes[b];
        const double r_big = std::max(A.radius, B.radius);
        const double r_small = std::min(A.radius, B.radius);
        if (r_big + theta * r_small <= theta * std::abs(A.center - B.center))
          w.push_back(b);
        else
          s.push_back(b);
      }
    }
  }
  return out;
}

Connectivity build_connectivity(const Pyramid& pyramid, double theta) {
  Connectivity c;
  c.levels.resize(pyramid.n_levels);
  c.levels[0] = classify_level(LevelConn{}, pyramid, 0, theta);
  for (int l = 1; l < pyramid.n_levels; ++l)
    c.levels[l] = classify_level(c.levels[l - 1], pyramid, l, theta);
  return c;
}

}  // namespace fmm
