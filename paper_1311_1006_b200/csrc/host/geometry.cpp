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
// parallel (each list emerges sorted; no post-sort).  The few huge boxes
// near the root are split one at a time with every step parallel: a
// sample-bracketed parallel selection, a parallel stable eval split and
// parallel extents (10M points: the two top levels 1.2 s -> see DESIGN).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <memory>
#include <sys/mman.h>

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

// Uninitialised record storage (no serial zero fill of ~240 MB per array at
// 10M; the pages are first touched by the parallel fills), on transparent
// huge pages.
class RecBuf {
 public:
  RecBuf() = default;
  explicit RecBuf(std::size_t n) { resize(n); }
  void resize(std::size_t n) {
    p_.reset(n ? new Rec[n] : nullptr);  // default-initialised: no zeroing
    n_ = n;
    const std::size_t bytes = n * sizeof(Rec);
    constexpr std::uintptr_t kHuge = std::uintptr_t(2) << 20;
    if (bytes >= 2 * kHuge) {
      const auto b = reinterpret_cast<std::uintptr_t>(p_.get());
      const std::uintptr_t a0 = (b + kHuge - 1) & ~(kHuge - 1), a1 = (b + bytes) & ~(kHuge - 1);
      if (a1 > a0) madvise(reinterpret_cast<void*>(a0), a1 - a0, MADV_HUGEPAGE);
    }
  }
  std::size_t size() const { return n_; }
  Rec* data() { return p_.get(); }
  const Rec* data() const { return p_.get(); }
  Rec* begin() { return p_.get(); }
  Rec& operator[](std::size_t i) { return p_[i]; }
  const Rec& operator[](std::size_t i) const { return p_[i]; }

 private:
  std::unique_ptr<Rec[]> p_;
  std::size_t n_ = 0;
};

// Selects the low half of recs[b,e) in place; returns the split position
// and the split coordinate (fallback when the range is empty).
struct Cut {
  std::uint32_t mid;
  double value;
};

Cut select_low_half(RecBuf& recs, std::uint32_t b, std::uint32_t e, bool x_axis,
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
std::uint32_t split_evals(RecBuf& evs, RecBuf& tmp, std::uint32_t b,
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

void fill_box(MBox& box, const RecBuf& src, const RecBuf& evs, cplx fallback) {
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

// ---- parallel versions for the few huge boxes near the root --------------
// (a box of n >= kParMin points; below that, one thread per box).  They give
// the same SETS, split values, eval order and extents as the serial helpers,
// so the pyramid is unchanged (the low half is a set; evals split stably).
constexpr std::uint32_t kParMin = 1u << 18;

std::uint32_t par_min_size() {
  static const std::uint32_t v = [] {
    const char* s = std::getenv("FMM_PAR_SELECT_MIN");  // tests force the parallel path
    return s ? std::uint32_t(std::strtoul(s, nullptr, 10)) : kParMin;
  }();
  return v;
}

// Low half of recs[b,e) by a sample-bracketed parallel partition: two
// pivots from a sorted sample bracket the median rank; one parallel pass
// scatters [< lo | between | > hi] through tmp, and nth_element finishes
// inside the (small) middle bucket.  Falls back to the serial selection if
// the sample missed the rank.
Cut select_low_half_par(RecBuf& recs, RecBuf& tmp, std::uint32_t b,
                        std::uint32_t e, bool x_axis, double fallback, int threads) {
  const std::uint32_t n = e - b;
  if (n < par_min_size() || threads < 2 || n < 4096) return select_low_half(recs, b, e, x_axis, fallback);
  auto less = [x_axis](const Rec& p, const Rec& q) {
    const double cp = along(p, x_axis), cq = along(q, x_axis);
    if (cp != cq) return cp < cq;
    return p.id < q.id;
  };
  const std::uint32_t k = (n + 1) / 2, r = k - 1;
  constexpr int S = 4096, D = 96;
  std::vector<Rec> smp(S);
  for (int i = 0; i < S; ++i) smp[i] = recs[b + std::uint32_t(std::uint64_t(i) * n / S)];
  std::sort(smp.begin(), smp.end(), less);
  const int at = int(std::uint64_t(r) * S / n);
  const Rec plo = smp[std::max(0, at - D)], phi = smp[std::min(S - 1, at + D)];
  const int T = threads;
  const std::uint64_t per = (std::uint64_t(n) + T - 1) / T;
  std::vector<std::uint64_t> c(3 * std::size_t(T) + 3, 0);  // [t] lt, mid, gt
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    const std::uint64_t i0 = b + std::min<std::uint64_t>(n, t * per);
    const std::uint64_t i1 = b + std::min<std::uint64_t>(n, (t + 1) * per);
    std::uint64_t lt = 0, gt = 0;
    for (std::uint64_t i = i0; i < i1; ++i) {
      if (less(recs[i], plo)) ++lt;
      else if (less(phi, recs[i])) ++gt;
    }
    c[3 * t] = lt;
    c[3 * t + 1] = (i1 - i0) - lt - gt;
    c[3 * t + 2] = gt;
  }
  std::uint64_t L = 0, M = 0;
  for (int t = 0; t < T; ++t) L += c[3 * t], M += c[3 * t + 1];
  if (!(L <= r && r < L + M)) return select_low_half(recs, b, e, x_axis, fallback);
  std::vector<std::uint64_t> o(3 * std::size_t(T), 0);  // per-thread output starts
  {
    std::uint64_t ol = b, om = b + L, og = b + L + M;
    for (int t = 0; t < T; ++t) {
      o[3 * t] = ol, ol += c[3 * t];
      o[3 * t + 1] = om, om += c[3 * t + 1];
      o[3 * t + 2] = og, og += c[3 * t + 2];
    }
  }
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    const std::uint64_t i0 = b + std::min<std::uint64_t>(n, t * per);
    const std::uint64_t i1 = b + std::min<std::uint64_t>(n, (t + 1) * per);
    std::uint64_t pl = o[3 * t], pm = o[3 * t + 1], pg = o[3 * t + 2];
    for (std::uint64_t i = i0; i < i1; ++i) {
      const Rec v = recs[i];
      if (less(v, plo)) tmp[pl++] = v;
      else if (less(phi, v)) tmp[pg++] = v;
      else tmp[pm++] = v;
    }
  }
#pragma omp parallel for schedule(static) num_threads(T)
  for (std::int64_t i = b; i < std::int64_t(e); ++i) recs[i] = tmp[i];
  Rec* base = recs.data();
  std::nth_element(base + b + L, base + b + r, base + b + L + M, less);
  return {b + k, along(recs[b + k - 1], x_axis)};
}

// split_evals over a huge range: per-thread counts, then every record goes
// through tmp to its stable place (lows first), and back.
std::uint32_t split_evals_par(RecBuf& evs, RecBuf& tmp, std::uint32_t b,
                              std::uint32_t e, bool x_axis, double value, int threads) {
  const std::uint32_t n = e - b;
  if (n < par_min_size() || threads < 2) return split_evals(evs, tmp, b, e, x_axis, value);
  const int T = threads;
  const std::uint64_t per = (std::uint64_t(n) + T - 1) / T;
  std::vector<std::uint64_t> lo(std::size_t(T) + 1, 0);
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    const std::uint64_t i0 = b + std::min<std::uint64_t>(n, t * per);
    const std::uint64_t i1 = b + std::min<std::uint64_t>(n, (t + 1) * per);
    std::uint64_t cnt = 0;
    for (std::uint64_t i = i0; i < i1; ++i) cnt += along(evs[i], x_axis) <= value ? 1 : 0;
    lo[t + 1] = cnt;
  }
  for (int t = 0; t < T; ++t) lo[t + 1] += lo[t];
  const std::uint64_t nlo = lo[T];
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    const std::uint64_t i0 = b + std::min<std::uint64_t>(n, t * per);
    const std::uint64_t i1 = b + std::min<std::uint64_t>(n, (t + 1) * per);
    std::uint64_t pl = b + lo[t], ph = b + nlo + ((i0 - b) - lo[t]);
    for (std::uint64_t i = i0; i < i1; ++i) {
      const Rec v = evs[i];
      if (along(v, x_axis) <= value) tmp[pl++] = v;
      else tmp[ph++] = v;
    }
  }
#pragma omp parallel for schedule(static) num_threads(T)
  for (std::int64_t i = b; i < std::int64_t(e); ++i) evs[i] = tmp[i];
  return std::uint32_t(b + nlo);
}

// fill_box with the extents reduced over all threads (huge boxes)
void fill_box_par(MBox& box, const RecBuf& src, const RecBuf& evs,
                  cplx fallback, int threads) {
  const std::uint32_t n = (box.point_end - box.point_begin) + (box.eval_end - box.eval_begin);
  if (n < par_min_size() || threads < 2) return fill_box(box, src, evs, fallback);
  if (box.point_begin == box.point_end && box.eval_begin == box.eval_end) {
    box.center = fallback;
    box.half_width = box.half_height = box.radius = 0.0;
    return;
  }
  // per-thread partial extents combined in thread order with the serial
  // helper's std::min / std::max: ties (+0.0 / -0.0) resolve as in index order
  const int T = threads;
  std::vector<double> part(4 * std::size_t(T));
  const std::uint64_t np = box.point_end - box.point_begin, ne = box.eval_end - box.eval_begin;
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    double a0 = std::numeric_limits<double>::infinity(), a1 = -a0, b0 = a0, b1 = -a0;
    const std::uint64_t s0 = box.point_begin + np * t / T, s1 = box.point_begin + np * (t + 1) / T;
    for (std::uint64_t i = s0; i < s1; ++i) {
      a0 = std::min(a0, src[i].x);
      a1 = std::max(a1, src[i].x);
      b0 = std::min(b0, src[i].y);
      b1 = std::max(b1, src[i].y);
    }
    part[4 * t] = a0, part[4 * t + 1] = a1, part[4 * t + 2] = b0, part[4 * t + 3] = b1;
  }
  double x0 = std::numeric_limits<double>::infinity(), x1 = -x0, y0 = x0, y1 = -x0;
  for (int t = 0; t < T; ++t) {
    x0 = std::min(x0, part[4 * t]);
    x1 = std::max(x1, part[4 * t + 1]);
    y0 = std::min(y0, part[4 * t + 2]);
    y1 = std::max(y1, part[4 * t + 3]);
  }
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    double a0 = std::numeric_limits<double>::infinity(), a1 = -a0, b0 = a0, b1 = -a0;
    const std::uint64_t s0 = box.eval_begin + ne * t / T, s1 = box.eval_begin + ne * (t + 1) / T;
    for (std::uint64_t i = s0; i < s1; ++i) {
      a0 = std::min(a0, evs[i].x);
      a1 = std::max(a1, evs[i].x);
      b0 = std::min(b0, evs[i].y);
      b1 = std::max(b1, evs[i].y);
    }
    part[4 * t] = a0, part[4 * t + 1] = a1, part[4 * t + 2] = b0, part[4 * t + 3] = b1;
  }
  for (int t = 0; t < T; ++t) {
    x0 = std::min(x0, part[4 * t]);
    x1 = std::max(x1, part[4 * t + 1]);
    y0 = std::min(y0, part[4 * t + 2]);
    y1 = std::max(y1, part[4 * t + 3]);
  }
  box.center = cplx(0.5 * (x0 + x1), 0.5 * (y0 + y1));
  box.half_width = 0.5 * (x1 - x0);
  box.half_height = 0.5 * (y1 - y0);
  box.radius = std::hypot(box.half_width, box.half_height);
}

}  // namespace

Pyramid build_pyramid(const SourceSet& sources, const EvalSet& evals, int n_levels, int threads) {
  const auto t_setup = std::chrono::steady_clock::now();
  if (n_levels < 1) throw InvalidParameter("build_pyramid: n_levels must be >= 1");
  if (sources.size() == 0) throw InvalidInput("build_pyramid: empty source set");
  if (threads < 1) threads = 1;
  bool fin_s = true, fin_e = true;
#pragma omp parallel for schedule(static) num_threads(threads) reduction(&& : fin_s)
  for (std::int64_t i = 0; i < std::int64_t(sources.size()); ++i)
    fin_s = fin_s && std::isfinite(sources.z[i].real()) && std::isfinite(sources.z[i].imag());
  if (!fin_s) throw InvalidInput("build_pyramid: non-finite source position");
#pragma omp parallel for schedule(static) num_threads(threads) reduction(&& : fin_e)
  for (std::int64_t i = 0; i < std::int64_t(evals.size()); ++i)
    fin_e = fin_e && std::isfinite(evals.y[i].real()) && std::isfinite(evals.y[i].imag());
  if (!fin_e) throw InvalidInput("build_pyramid: non-finite eval position");

  const std::uint32_t ns = static_cast<std::uint32_t>(sources.size());
  const std::uint32_t ne = static_cast<std::uint32_t>(evals.size());
  RecBuf src(ns), evs(ne);
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
  fill_box_par(root, src, evs, cplx(0, 0), threads);
  pyr.levels[0].push_back(root);

  RecBuf scratch(ne), src_tmp;
  if (threads > 1 && ns >= par_min_size()) src_tmp.resize(ns);
  static const bool trace = std::getenv("FMM_TRACE") != nullptr;
  auto tl = std::chrono::steady_clock::now();
  if (trace)
    std::fprintf(stderr, "[fmm] host pyramid setup: %.1f ms\n",
                 std::chrono::duration<double, std::milli>(tl - t_setup).count());
  for (int l = 1; l < n_levels; ++l) {
    if (trace && l > 1) {
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[fmm] host pyramid level %d: %.1f ms\n", l - 1,
                   std::chrono::duration<double, std::milli>(now - tl).count());
      tl = now;
    }
    const std::vector<MBox>& up = pyr.levels[l - 1];
    std::vector<MBox>& kids = pyr.levels[l];
    kids.resize(up.size() * 4);
    const std::int64_t np = std::int64_t(up.size());
    const bool inner = np < threads;
    auto place = [&](std::int64_t pi, const MBox& par, const std::uint32_t* pb,
                     const std::uint32_t* eb, bool par_fill) {
      for (int c = 0; c < 4; ++c) {
        MBox& kid = kids[4 * pi + c];
        kid.level = l;
        kid.index_in_level = std::uint32_t(4 * pi + c);
        kid.point_begin = pb[c];
        kid.point_end = pb[c + 1];
        kid.eval_begin = eb[c];
        kid.eval_end = eb[c + 1];
        if (par_fill) fill_box_par(kid, src, evs, par.center, threads);
        else fill_box(kid, src, evs, par.center);
      }
    };
    if (inner) {
      // Few huge parents near the root: one parent at a time, each step
      // (selection, eval split, extents) parallel over all threads.
      for (std::int64_t pi = 0; pi < np; ++pi) {
        const MBox& par = up[pi];
        const Cut cx = select_low_half_par(src, src_tmp, par.point_begin, par.point_end, true,
                                           par.center.real(), threads);
        const std::uint32_t emx =
            split_evals_par(evs, scratch, par.eval_begin, par.eval_end, true, cx.value, threads);
        const Cut cyl = select_low_half_par(src, src_tmp, par.point_begin, cx.mid, false,
                                            par.center.imag(), threads);
        const std::uint32_t emyl =
            split_evals_par(evs, scratch, par.eval_begin, emx, false, cyl.value, threads);
        const Cut cyh = select_low_half_par(src, src_tmp, cx.mid, par.point_end, false,
                                            par.center.imag(), threads);
        const std::uint32_t emyh =
            split_evals_par(evs, scratch, emx, par.eval_end, false, cyh.value, threads);
        const std::uint32_t pb[5] = {par.point_begin, cyl.mid, cx.mid, cyh.mid, par.point_end};
        const std::uint32_t eb[5] = {par.eval_begin, emyl, emx, emyh, par.eval_end};
        place(pi, par, pb, eb, true);
      }
      continue;
    }
    // many parents deeper down: parallelise across parents
#pragma omp parallel for schedule(dynamic) num_threads(threads)
    for (std::int64_t pi = 0; pi < np; ++pi) {
      const MBox& par = up[pi];
      const Cut cx = select_low_half(src, par.point_begin, par.point_end, true, par.center.real());
      const std::uint32_t emx =
          split_evals(evs, scratch, par.eval_begin, par.eval_end, true, cx.value);
      const Cut cyl = select_low_half(src, par.point_begin, cx.mid, false, par.center.imag());
      const std::uint32_t emyl = split_evals(evs, scratch, par.eval_begin, emx, false, cyl.value);
      const Cut cyh = select_low_half(src, cx.mid, par.point_end, false, par.center.imag());
      const std::uint32_t emyh = split_evals(evs, scratch, emx, par.eval_end, false, cyh.value);
      const std::uint32_t pb[5] = {par.point_begin, cyl.mid, cx.mid, cyh.mid, par.point_end};
      const std::uint32_t eb[5] = {par.eval_begin, emyl, emx, emyh, par.eval_end};
      place(pi, par, pb, eb, false);
    }
  }

  if (trace)
    std::fprintf(stderr, "[fmm] host pyramid levels done: %.1f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_setup)
                     .count());
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
  static const bool trace = std::getenv("FMM_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  Connectivity c;
  c.levels.resize(pyramid.n_levels);
  c.levels[0] = classify_level(LevelConn{}, pyramid, 0, theta);
  for (int l = 1; l < pyramid.n_levels; ++l)
    c.levels[l] = classify_level(c.levels[l - 1], pyramid, l, theta);
  if (trace)
    std::fprintf(stderr, "[fmm] host connectivity: %.1f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                     .count());
  return c;
}

}  // namespace fmm
