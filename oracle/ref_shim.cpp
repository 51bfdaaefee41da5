// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim around the *unmodified* reference library (`atfmm`, compiled from
// /root/reference/proj/src/{geometry,expansion,backend,engine,autotune,csv}.cpp
// by oracle/Makefile into oracle/_ref/libfmmref.so).  It exists so that the
// Python tests, the golden-fixture generator and bench.py's reference arm can
// drive the reference's own code path through ctypes:
//
//   fmmref_tree_*      -> fmm::build_pyramid / build_connectivity   (geometry.cpp:106-216)
//   fmmref_nearfield   -> fmm::nearfield_run (serial or OpenMP pool) (backend.cpp:73-89)
//   fmmref_evaluate    -> fmm::FmmEngine::evaluate                   (engine.cpp:208-347)
//   fmmref_m2l_add     -> fmm::m2l_add                               (expansion.cpp:188-269)
//   fmmref_kernel_term -> fmm::kernel_term                           (expansion.cpp:90-92)
//
// Everything here is glue written for this repo; no reference source is
// copied.  Input generators restate tools/atfmm.cpp:70-86 (make_distribution)
// and tests/test_util.hpp:10-23 (random_sources) with the same std:: engines.

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "fmm/autotune.hpp"
#include "fmm/engine.hpp"

using fmm::cplx;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const fmm::InvalidParameter*>(&e)) return 1;
  if (dynamic_cast<const fmm::InvalidInput*>(&e)) return 2;
  if (dynamic_cast<const fmm::SingularConfiguration*>(&e)) return 3;
  if (dynamic_cast<const fmm::BackendError*>(&e)) return 4;
  return 9;
}

fmm::SourceSet make_sources(const double* z, const double* m, int64_t n) {
  fmm::SourceSet s;
  s.z.resize(n);
  s.m.resize(n);
  std::memcpy(s.z.data(), z, sizeof(double) * 2 * n);
  std::memcpy(s.m.data(), m, sizeof(double) * 2 * n);
  return s;
}

fmm::EvalSet make_evals(const double* y, const int64_t* sid, int64_t n) {
  fmm::EvalSet e;
  e.y.resize(n);
  if (n) std::memcpy(e.y.data(), y, sizeof(double) * 2 * n);
  if (sid) e.source_id.assign(sid, sid + n);
  return e;
}

struct RefTree {
  fmm::SourceSet src;
  fmm::EvalSet ev;
  fmm::Pyramid pyr;
  fmm::Connectivity conn;
};

fmm::Smoother make_smoother(int kind, double delta) {
  if (kind == 1) return fmm::Smoother::gaussian(delta);
  if (kind == 2) return fmm::Smoother::plummer(delta);
  return fmm::Smoother::none();
}

}  // namespace

extern "C" {

const char* fmmref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- inputs --
// kind 0: uniform (atfmm.cpp:70-86, x,y,m_re ~ U(0,1), m_im = 0)
// kind 1: "line" band (atfmm.cpp:79-80)
// kind 2: 8 Gaussian clusters (SURVEY.md §8(d) config 3 definition)
// kind 3: testutil::random_sources(n, seed, 1.0, positive=false) (test_util.hpp:10-23)
// kind 4: testutil::random_sources(n, seed, 1.0, positive=true)
void fmmref_make_distribution(int kind, int64_t n, uint64_t seed, double* z, double* m) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  if (kind == 3 || kind == 4) {
    const bool pos = kind == 4;
    std::uniform_real_distribution<double> um(pos ? 0.1 : -1.0, 1.0);
    for (int64_t i = 0; i < n; ++i) {
      z[2 * i] = uni(rng);
      z[2 * i + 1] = uni(rng);
      if (pos) {
        m[2 * i] = um(rng);
        m[2 * i + 1] = 0.0;
      } else {
        m[2 * i] = um(rng);
        m[2 * i + 1] = um(rng);
      }
    }
    return;
  }
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int64_t i = 0; i < n; ++i) {
    if (kind == 1) {
      z[2 * i] = uni(rng);
      z[2 * i + 1] = 0.005 * uni(rng);
    } else if (kind == 2) {
      const int c = static_cast<int>(i % 8);
      const double g1 = gauss(rng);
      const double g2 = gauss(rng);
      z[2 * i] = 0.15 + 0.1 * c + 0.02 * g1;
      z[2 * i + 1] = 0.5 + 0.3 * std::sin(static_cast<double>(c)) + 0.02 * g2;
    } else {
      z[2 * i] = uni(rng);
      z[2 * i + 1] = uni(rng);
    }
    m[2 * i] = uni(rng);
    m[2 * i + 1] = 0.0;
  }
}

// ------------------------------------------------------------------ tree --
void* fmmref_tree_build(const double* z, const double* m, int64_t n_src, const double* y,
                        const int64_t* sid, int64_t n_eval, int n_levels, double theta,
                        int threads) {
  try {
    auto t = std::make_unique<RefTree>();
    t->src = make_sources(z, m, n_src);
    t->ev = make_evals(y, sid, n_eval);
    t->pyr = fmm::build_pyramid(t->src, t->ev, n_levels, threads);
    t->conn = fmm::build_connectivity(t->pyr, theta);
    return t.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void fmmref_tree_free(void* h) { delete static_cast<RefTree*>(h); }

int64_t fmmref_tree_nboxes(void* h, int level) {
  return static_cast<int64_t>(static_cast<RefTree*>(h)->pyr.levels[level].size());
}

// f64: 5 per box (cx, cy, half_width, half_height, radius)
// u32: 4 per box (point_begin, point_end, eval_begin, eval_end)
void fmmref_tree_boxes(void* h, int level, double* f64, uint32_t* u32) {
  const auto& boxes = static_cast<RefTree*>(h)->pyr.levels[level];
  for (std::size_t i = 0; i < boxes.size(); ++i) {
    const fmm::MBox& b = boxes[i];
    f64[5 * i + 0] = b.center.real();
    f64[5 * i + 1] = b.center.imag();
    f64[5 * i + 2] = b.half_width;
    f64[5 * i + 3] = b.half_height;
    f64[5 * i + 4] = b.radius;
    u32[4 * i + 0] = b.point_begin;
    u32[4 * i + 1] = b.point_end;
    u32[4 * i + 2] = b.eval_begin;
    u32[4 * i + 3] = b.eval_end;
  }
}

void fmmref_tree_perm(void* h, uint32_t* perm, uint32_t* eperm) {
  const auto& p = static_cast<RefTree*>(h)->pyr;
  std::memcpy(perm, p.perm.data(), sizeof(uint32_t) * p.perm.size());
  if (!p.eval_perm.empty())
    std::memcpy(eperm, p.eval_perm.data(), sizeof(uint32_t) * p.eval_perm.size());
}

int64_t fmmref_tree_nnz(void* h, int level, int weak) {
  const auto& lc = static_cast<RefTree*>(h)->conn.levels[level];
  const auto& lists = weak ? lc.weak : lc.strong;
  int64_t n = 0;
  for (const auto& v : lists) n += static_cast<int64_t>(v.size());
  return n;
}

void fmmref_tree_lists(void* h, int level, int weak, uint32_t* off, uint32_t* idx) {
  const auto& lc = static_cast<RefTree*>(h)->conn.levels[level];
  const auto& lists = weak ? lc.weak : lc.strong;
  uint32_t k = 0;
  for (std::size_t i = 0; i < lists.size(); ++i) {
    off[i] = k;
    for (uint32_t v : lists[i]) idx[k++] = v;
  }
  off[lists.size()] = k;
}

// Reference near field over the tree's finest level (backend.cpp:73-89).
// Only target leaves in [leaf_begin, leaf_end) are evaluated: the others get
// their eval range emptied in a private copy of the pyramid, so near_box()
// skips them (backend.cpp:44) -- this is how bench.py times a bounded sample
// of a large workload on the reference's own loop.  out: permuted eval order.
int fmmref_tree_nearfield(void* h, int kernel, int smoother, double delta, int parallel,
                          int threads, int64_t leaf_begin, int64_t leaf_end, double* out,
                          uint64_t* pairs, double* seconds) {
  try {
    RefTree* t = static_cast<RefTree*>(h);
    const auto& pyr = t->pyr;
    const std::size_t ns = t->src.size(), ne = t->ev.size();
    std::vector<cplx> zp(ns), mp(ns), yp(ne);
    std::vector<int64_t> sidp;
    for (std::size_t i = 0; i < ns; ++i) {
      zp[i] = t->src.z[pyr.perm[i]];
      mp[i] = t->src.m[pyr.perm[i]];
    }
    if (!t->ev.source_id.empty()) sidp.resize(ne);
    for (std::size_t i = 0; i < ne; ++i) {
      yp[i] = t->ev.y[pyr.eval_perm[i]];
      if (!sidp.empty()) sidp[i] = t->ev.source_id[pyr.eval_perm[i]];
    }
    const int64_t nleaf = static_cast<int64_t>(pyr.finest().size());
    const fmm::Pyramid* use = &pyr;
    fmm::Pyramid masked;
    if (leaf_begin > 0 || leaf_end < nleaf) {
      masked.n_levels = pyr.n_levels;
      masked.levels = pyr.levels;  // box geometry is unused by near_box except ranges
      masked.perm = pyr.perm;
      masked.eval_perm = pyr.eval_perm;
      auto& fine = masked.levels.back();
      for (int64_t i = 0; i < nleaf; ++i)
        if (i < leaf_begin || i >= leaf_end) fine[i].eval_end = fine[i].eval_begin;
      use = &masked;
    }
    fmm::NearFieldJob job{use, &t->conn.finest(), &zp, &mp, &yp, &sidp,
                          kernel ? fmm::Kernel::logarithmic : fmm::Kernel::harmonic,
                          make_smoother(smoother, delta), threads};
    std::vector<cplx> near;
    fmm::NearFieldStats st = fmm::nearfield_run(job, near, parallel != 0);
    if (out && ne) std::memcpy(out, near.data(), sizeof(double) * 2 * ne);
    *pairs = st.pair_evals;
    *seconds = st.seconds;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ------------------------------------------------- near field from CSR ----
// The reference nearfield_run (backend.cpp:73-89) over a finest level given
// as CSR arrays (the same arrays the product's C ABI takes), so bench.py can
// time the reference's own loop on exactly the device workload without
// rebuilding the reference tree.  The pyramid is a one-level shell holding
// the leaf ranges; near_box() reads nothing else (backend.cpp:41-69).
struct RefNF {
  fmm::Pyramid pyr;
  fmm::LevelConn conn;
  std::vector<cplx> zp, mp, yp;
  std::vector<int64_t> sidp;
  std::vector<uint32_t> ev_begin;  // unmasked eval ranges
  std::vector<uint32_t> ev_end;
};

void* fmmref_nf_create(uint32_t n_leaves, const uint32_t* pt_off, const uint32_t* ev_off,
                       const uint32_t* s_off, const uint32_t* s_idx, const uint32_t* perm,
                       uint32_t n_src, uint32_t n_eval, const double* zp, const double* mp,
                       const double* yp, const int64_t* sidp) {
  auto h = std::make_unique<RefNF>();
  h->pyr.n_levels = 1;
  h->pyr.levels.resize(1);
  auto& fine = h->pyr.levels[0];
  fine.resize(n_leaves);
  h->ev_begin.resize(n_leaves);
  h->ev_end.resize(n_leaves);
  for (uint32_t i = 0; i < n_leaves; ++i) {
    fine[i].point_begin = pt_off[i];
    fine[i].point_end = pt_off[i + 1];
    fine[i].eval_begin = h->ev_begin[i] = ev_off[i];
    fine[i].eval_end = h->ev_end[i] = ev_off[i + 1];
  }
  h->pyr.perm.assign(perm, perm + n_src);
  h->conn.strong.resize(n_leaves);
  for (uint32_t i = 0; i < n_leaves; ++i) h->conn.strong[i].assign(s_idx + s_off[i], s_idx + s_off[i + 1]);
  h->zp.resize(n_src);
  h->mp.resize(n_src);
  h->yp.resize(n_eval);
  std::memcpy(h->zp.data(), zp, sizeof(double) * 2 * n_src);
  std::memcpy(h->mp.data(), mp, sizeof(double) * 2 * n_src);
  if (n_eval) std::memcpy(h->yp.data(), yp, sizeof(double) * 2 * n_eval);
  if (sidp) h->sidp.assign(sidp, sidp + n_eval);
  return h.release();
}

void fmmref_nf_free(void* h) { delete static_cast<RefNF*>(h); }

int fmmref_nf_run(void* hv, int kernel, int smoother, double delta, int parallel, int threads,
                  int64_t leaf_begin, int64_t leaf_end, double* out, uint64_t* pairs,
                  double* seconds) {
  try {
    RefNF* h = static_cast<RefNF*>(hv);
    auto& fine = h->pyr.levels[0];
    const int64_t n = static_cast<int64_t>(fine.size());
    for (int64_t i = 0; i < n; ++i) {
      const bool in = i >= leaf_begin && i < leaf_end;
      fine[i].eval_begin = h->ev_begin[i];
      fine[i].eval_end = in ? h->ev_end[i] : h->ev_begin[i];
    }
    fmm::NearFieldJob job{&h->pyr, &h->conn, &h->zp, &h->mp, &h->yp, &h->sidp,
                          kernel ? fmm::Kernel::logarithmic : fmm::Kernel::harmonic,
                          make_smoother(smoother, delta), threads};
    std::vector<cplx> near;
    const fmm::NearFieldStats st = fmm::nearfield_run(job, near, parallel != 0);
    if (out && !near.empty()) std::memcpy(out, near.data(), sizeof(double) * 2 * near.size());
    *pairs = st.pair_evals;
    *seconds = st.seconds;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ------------------------------------------------------------- evaluate --
// cfg_f: theta, tol, p_calibration, delta
// cfg_i: n_levels, kernel, p_rule(0 formula,1 table), p_override, backend(0 serial,1 pool),
//        worker_threads, task_split_level, smoother kind
// timings: 8 (PhaseTimings order), counters: 4 (WorkCounters order)
int fmmref_evaluate(const double* z, const double* m, int64_t n_src, const double* y,
                    const int64_t* sid, int64_t n_eval, const double* cfg_f, const int* cfg_i,
                    double* out, double* timings, uint64_t* counters, int* p_out) {
  try {
    fmm::FmmConfig cfg;
    cfg.theta = cfg_f[0];
    cfg.tol = cfg_f[1];
    cfg.p_calibration = cfg_f[2];
    cfg.n_levels = cfg_i[0];
    cfg.kernel = cfg_i[1] ? fmm::Kernel::logarithmic : fmm::Kernel::harmonic;
    cfg.p_rule = cfg_i[2] ? fmm::PRule::table : fmm::PRule::formula;
    cfg.p_override = cfg_i[3];
    cfg.backend = cfg_i[4] ? fmm::BackendKind::pool : fmm::BackendKind::serial;
    cfg.worker_threads = cfg_i[5];
    cfg.task_split_level = cfg_i[6];
    cfg.smoother = make_smoother(cfg_i[7], cfg_f[3]);
    fmm::SourceSet s = make_sources(z, m, n_src);
    fmm::EvalSet e = make_evals(y, sid, n_eval);
    fmm::FmmEngine eng(cfg);
    fmm::EvalResult r = eng.evaluate(s, e);
    if (out && n_eval) std::memcpy(out, r.potentials.data(), sizeof(double) * 2 * n_eval);
    const auto& t = r.timings;
    const double tv[8] = {t.t_partition, t.t_p2m, t.t_upward, t.t_m2l,
                          t.t_p2p,       t.t_q,   t.t_total,  t.cpu_wait};
    if (timings) std::memcpy(timings, tv, sizeof tv);
    if (counters) {
      counters[0] = r.counters.p2p_pairs;
      counters[1] = r.counters.m2l_ops;
      counters[2] = r.counters.p2m_points;
      counters[3] = r.counters.l2p_points;
    }
    if (p_out) *p_out = r.p;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ------------------------------------------------------------ operators --
int fmmref_m2l_add(int p, int kernel, const double* src_center, const double* coeffs,
                   const double* tgt_center, double* local) {
  try {
    fmm::Expansion out;
    out.center = cplx(src_center[0], src_center[1]);
    out.kernel = kernel ? fmm::Kernel::logarithmic : fmm::Kernel::harmonic;
    out.coeffs.resize(p + 1);
    std::memcpy(out.coeffs.data(), coeffs, sizeof(double) * 2 * (p + 1));
    fmm::Expansion loc;
    loc.center = cplx(tgt_center[0], tgt_center[1]);
    loc.kind = fmm::Expansion::Kind::ingoing;
    loc.kernel = out.kernel;
    loc.coeffs.resize(p + 1);
    std::memcpy(loc.coeffs.data(), local, sizeof(double) * 2 * (p + 1));
    fmm::m2l_add(out, loc);
    std::memcpy(local, loc.coeffs.data(), sizeof(double) * 2 * (p + 1));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int fmmref_p2m(int p, int kernel, const double* center, const double* z, const double* m,
               int64_t n, double* coeffs) {
  try {
    std::vector<cplx> zz(n), mm(n);
    std::memcpy(zz.data(), z, sizeof(double) * 2 * n);
    std::memcpy(mm.data(), m, sizeof(double) * 2 * n);
    fmm::Expansion e = fmm::p2m(cplx(center[0], center[1]), zz, mm,
                                kernel ? fmm::Kernel::logarithmic : fmm::Kernel::harmonic, p);
    std::memcpy(coeffs, e.coeffs.data(), sizeof(double) * 2 * (p + 1));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void fmmref_kernel_term(int kernel, const double* y, const double* x, const double* m,
                        double* out) {
  cplx r = fmm::kernel_term(kernel ? fmm::Kernel::logarithmic : fmm::Kernel::harmonic,
                            cplx(y[0], y[1]), cplx(x[0], x[1]), cplx(m[0], m[1]));
  out[0] = r.real();
  out[1] = r.imag();
}

// Batched kernel_term for the divdc3 pin: out[i] = kernel_term(harmonic, y_i, x_i, m_i)
void fmmref_kernel_term_batch(int kernel, int64_t n, const double* y, const double* x,
                              const double* m, double* out) {
  for (int64_t i = 0; i < n; ++i) fmmref_kernel_term(kernel, y + 2 * i, x + 2 * i, m + 2 * i, out + 2 * i);
}

double fmmref_smoother_factor(int kind, double delta, double r) {
  return fmm::smoother_factor(make_smoother(kind, delta), r);
}

int fmmref_choose_p(int rule, double tol, double theta, double calibration) {
  try {
    return fmm::choose_p(rule ? fmm::PRule::table : fmm::PRule::formula, tol, theta, calibration);
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

void fmmref_estimate_cost(double n, int nl, double theta, int p, double* out4) {
  fmm::CostEstimate c = fmm::estimate_cost(n, nl, theta, p);
  out4[0] = c.c_p2p;
  out4[1] = c.c_m2l;
  out4[2] = c.c_m2m;
  out4[3] = c.c_p2m;
}

// ------------------------------------------------------------ autotuner --
// Controller parity driver: feeds `n` measurements and records params after
// each step.  meas: n x 3 (time, cpu_wait, has_wait); out: n x 2 (theta, nl)
int fmmref_controller_run(int kind, const double* ccfg_f, const int* ccfg_i, double theta0,
                          int nl0, uint64_t seed, int64_t n, const double* meas, double* out,
                          int* events) {
  try {
    fmm::ControllerConfig cc;
    cc.theta_min = ccfg_f[0];
    cc.theta_max = ccfg_f[1];
    cc.base_thetastep = ccfg_f[2];
    cc.cap = ccfg_f[3];
    cc.nl_min = ccfg_i[0];
    cc.nl_max = ccfg_i[1];
    cc.theta_every = ccfg_i[2];
    cc.nl_every = ccfg_i[3];
    cc.filter_window = ccfg_i[4];
    cc.init_fiblength = ccfg_i[5];
    cc.max_fiblength = ccfg_i[6];
    fmm::Controller ctl(static_cast<fmm::TunerKind>(kind), cc, {theta0, nl0}, seed);
    for (int64_t i = 0; i < n; ++i) {
      fmm::Measurement mm{static_cast<int>(i + 1), meas[3 * i], meas[3 * i + 1],
                          meas[3 * i + 2] != 0.0};
      fmm::Params p = ctl.step(mm);
      out[2 * i] = p.theta;
      out[2 * i + 1] = p.n_levels;
      const fmm::StepEvent& ev = ctl.last_event();
      events[3 * i] = static_cast<int>(ev.proposed);
      events[3 * i + 1] = ev.move_dir;
      events[3 * i + 2] = ev.accepted;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
