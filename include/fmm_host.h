/*
 * fmm-b200 — flat C ABI of the C++ host library (libfmm.so) for bindings
 * (Python ctypes in paper_1311_1006_b200/, or any FFI).  It exposes the
 * reference's public C++ surface (the include/fmm headers) with plain pointers:
 *
 *   fmmh_tree_*         build_pyramid / build_connectivity   (geometry.hpp:59-74)
 *   fmmh_tree_nearfield NearFieldBackend launch+finish        (backend.hpp:48-63)
 *   fmmh_engine_*       FmmEngine / FmmConfig / EvalResult    (engine.hpp:14-118)
 *   fmmh_controller_run Controller::step                      (autotune.hpp:73-121)
 *   fmmh_vortex_run     sims::init_shear_layer/vortex_velocities/euler_step
 *
 * Status codes mirror the reference exceptions: 0 ok, 1 InvalidParameter,
 * 2 InvalidInput, 3 SingularConfiguration, 4 BackendError, 5 InvalidState /
 * NoMeasurement, 9 other; the message is fmmh_last_error() (thread-local).
 *
 * Config vectors:
 *   cfg_f[6] = theta, tol, p_calibration, smoother delta, throttle latency_s,
 *              throttle throughput
 *   cfg_i[11] = n_levels, kernel (0 harmonic, 1 log), p_rule (0 formula,
 *              1 table), p_override, backend (0 serial, 1 pool, 2 throttled,
 *              3 cuda), worker_threads, task_split_level, smoother kind
 *              (0 none, 1 gaussian, 2 plummer), cuda exact (0/1),
 *              m2l_on_device (0/1), device_pipeline (0/1)
 *   timings[8] = PhaseTimings in declaration order; counters[4] = WorkCounters.
 */
#ifndef FMM_HOST_H_
#define FMM_HOST_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char *fmmh_last_error(void);
/* Status of the last failing call on this thread (for handle-returning calls). */
int fmmh_last_status(void);

/* Synthetic inputs: 0 uniform (x,y,m_re ~ U(0,1)), 1 line band, 2 eight
 * Gaussian clusters, 3 random complex strengths U(-1,1)^2, 4 positive real
 * strengths U(0.1,1).  std::mt19937_64(seed) as the reference CLI/tests. */
void fmmh_make_distribution(int kind, int64_t n, uint64_t seed, double *z, double *m);

void *fmmh_tree_build(const double *z, const double *m, int64_t n_src, const double *y,
                      const int64_t *sid, int64_t n_eval, int n_levels, double theta,
                      int threads);
void fmmh_tree_free(void *tree);
int64_t fmmh_tree_nboxes(void *tree, int level);
void fmmh_tree_boxes(void *tree, int level, double *f64, uint32_t *u32);
void fmmh_tree_perm(void *tree, uint32_t *perm, uint32_t *eval_perm);
int64_t fmmh_tree_nnz(void *tree, int level, int weak);
void fmmh_tree_lists(void *tree, int level, int weak, uint32_t *off, uint32_t *idx);
int fmmh_tree_nearfield(void *tree, int backend, const int *devices, int n_devices, int exact,
                        int kernel, int smoother, double delta, int threads, double *out,
                        uint64_t *pairs, double *seconds);

void *fmmh_engine_create(const double *cfg_f, const int *cfg_i, const int *devices,
                         int n_devices);
int fmmh_engine_set_config(void *engine, const double *cfg_f, const int *cfg_i,
                           const int *devices, int n_devices);
int fmmh_engine_evaluate(void *engine, const double *z, const double *m, int64_t n_src,
                         const double *y, const int64_t *sid, int64_t n_eval, double *out,
                         double *timings, uint64_t *counters, int *p);
uint64_t fmmh_engine_kernel_launches(void *engine);
void fmmh_engine_free(void *engine);

int fmmh_controller_run(int kind, const double *ccfg_f, const int *ccfg_i, double theta0,
                        int nl0, uint64_t seed, int64_t n, const double *meas, double *out,
                        int *events);

/* Vortex sheet, `steps` Euler steps, optional tuner (0 none .. 4 at3b).
 * trace: steps x 8 = t_total, t_m2l, t_p2p, t_q, cpu_wait, theta, n_levels,
 * p2p_pairs; final_pos (2n doubles) may be NULL. */
int fmmh_vortex_run(int n, double aspect, int steps, int tuner, double cap, uint64_t seed,
                    const double *cfg_f, const int *cfg_i, const int *devices, int n_devices,
                    double *trace, double *final_pos);

int fmmh_m2l_add(int p, int kernel, const double *src_center, const double *coeffs,
                 const double *tgt_center, double *local);
int fmmh_p2m(int p, int kernel, const double *center, const double *z, const double *m,
             int64_t n, double *coeffs);
int fmmh_choose_p(int rule, double tol, double theta, double calibration);
int fmmh_estimate_cost(double n, int n_levels, double theta, int p, double *out4);
int fmmh_p2p_direct(const double *z, const double *m, int64_t n_src, const double *y,
                    const int64_t *sid, int64_t n_eval, int kernel, int smoother, double delta,
                    double *out);

#ifdef __cplusplus
}
#endif
#endif /* FMM_HOST_H_ */
