// TEST GLUE for the reference-side binding (not product): a C entry point
// that runs the REFERENCE's FmmEngine::evaluate (engine.cpp:208-347,
// compiled from the patched scratch copy) with the backend named by string
// through the reference's own backend_from_string -- "serial", "pool" or the
// added "cuda" (integration/cuda_backend_ref.cpp over libfmmcuda.so).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "fmm/engine.hpp"

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* refcu_last_error() { return g_err.c_str(); }

// cfg_f: theta, tol; cfg_i: n_levels, p_rule (0 formula, 1 table), worker_threads
// timings: 8 (PhaseTimings order), counters: 4 (WorkCounters order)
// returns 0, or 1 InvalidParameter, 2 InvalidInput, 3 Singular, 4 BackendError, 9 other
int refcu_evaluate(const char* backend, const double* z, const double* m, int64_t n,
                   const int64_t* sid, const double* cfg_f, const int* cfg_i, double* out,
                   double* timings, uint64_t* counters, char* backend_name, int name_len) {
  try {
    fmm::FmmConfig cfg;
    cfg.theta = cfg_f[0];
    cfg.tol = cfg_f[1];
    cfg.n_levels = cfg_i[0];
    cfg.p_rule = cfg_i[1] ? fmm::PRule::table : fmm::PRule::formula;
    cfg.worker_threads = cfg_i[2];
    cfg.backend = fmm::backend_from_string(backend);
    fmm::SourceSet s;
    s.z.resize(n);
    s.m.resize(n);
    std::memcpy(s.z.data(), z, sizeof(double) * 2 * n);
    std::memcpy(s.m.data(), m, sizeof(double) * 2 * n);
    fmm::EvalSet e;
    e.y = s.z;
    if (sid) e.source_id.assign(sid, sid + n);
    fmm::FmmEngine eng(cfg);
    if (backend_name && name_len > 0) {
      std::strncpy(backend_name, fmm::to_string(cfg.backend), size_t(name_len) - 1);
      backend_name[name_len - 1] = 0;
    }
    fmm::EvalResult r = eng.evaluate(s, e);
    if (!eng.backend_concurrent() && cfg.backend == fmm::BackendKind::cuda) return 9;
    std::memcpy(out, r.potentials.data(), sizeof(double) * 2 * n);
    const auto& t = r.timings;
    const double tv[8] = {t.t_partition, t.t_p2m, t.t_upward, t.t_m2l,
                          t.t_p2p,       t.t_q,   t.t_total,  t.cpu_wait};
    std::memcpy(timings, tv, sizeof tv);
    counters[0] = r.counters.p2p_pairs;
    counters[1] = r.counters.m2l_ops;
    counters[2] = r.counters.p2m_points;
    counters[3] = r.counters.l2p_points;
    return 0;
  } catch (const fmm::InvalidParameter& e) {
    g_err = e.what();
    return 1;
  } catch (const fmm::InvalidInput& e) {
    g_err = e.what();
    return 2;
  } catch (const fmm::SingularConfiguration& e) {
    g_err = e.what();
    return 3;
  } catch (const fmm::BackendError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

}  // extern "C"
