/*
 * fmm-b200 — C ABI of the B200 near-field library (libfmmcuda.so, sm_100a).
 *
 * Plain pointers and sizes only.  This is the boundary the reference's
 * near-field plug-in interface binds to:
 *
 *   reference (proj/include/fmm/backend.hpp)      this ABI
 *   -------------------------------------------   ------------------------------
 *   NearFieldBackend::launch(job, out)  :53-55    fmmcu_p2p_launch
 *   NearFieldBackend::finish()          :56       fmmcu_p2p_finish
 *   NearFieldJob                        :27-37    fmmcu_p2p_job (CSR-flattened)
 *   NearFieldStats                      :39-42    pair_evals / seconds outputs
 *   m2l_add (expansion.hpp:60, called at
 *            engine.cpp:108-113)                  fmmcu_m2l_launch / _finish
 *   l2l_add chain of the downward pass
 *            (engine.cpp:96-114)                  fmmcu_m2l_downward
 *   errors thrown as BackendError /
 *   SingularConfiguration (types.hpp:70-78)       int status + fmmcu_last_error
 *
 * The C++ class fmm::CudaBackend (backend kind "cuda") is a thin wrapper
 * that flattens the job, calls these entry points and rethrows failures.
 * Every function returns FMMCU_OK (0) or an FMMCU_E* code; the message is in
 * fmmcu_last_error(ctx).  There is no CPU fallback: a missing device is an
 * error (FMMCU_ECUDA).
 */
#ifndef FMM_CUDA_H_
#define FMM_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMMCU_OK 0
#define FMMCU_EINVAL 1    /* bad argument (InvalidParameter / InvalidInput) */
#define FMMCU_ECUDA 2     /* CUDA runtime failure or no device */
#define FMMCU_ESINGULAR 4 /* M2L with coincident centres (SingularConfiguration) */
#define FMMCU_ENOMEM 5    /* device or pinned allocation failed */
#define FMMCU_ESTATE 6    /* call out of order (finish without launch, ...) */
#define FMMCU_ENCCL 7     /* NCCL unavailable or a collective failed */

#define FMMCU_IPC_HANDLE_BYTES 64  /* cudaIpcMemHandle_t */
#define FMMCU_NCCL_ID_BYTES 128    /* ncclUniqueId */

#define FMMCU_KERNEL_HARMONIC 0 /* -m / (y - x)     (expansion.cpp:90-92) */
#define FMMCU_KERNEL_LOG 1      /*  m * log(y - x) */

#define FMMCU_SMOOTH_NONE 0     /* expansion.cpp:78-88 */
#define FMMCU_SMOOTH_GAUSSIAN 1 /* 1 - exp(-r^2/delta^2) */
#define FMMCU_SMOOTH_PLUMMER 2  /* r / sqrt(delta^2 + r^2) */

#define FMMCU_MODE_FAST 0  /* FP64, rcp+Newton, FMA; <= 1e-12 normwise of the reference */
#define FMMCU_MODE_EXACT 1 /* bit-compatible: restated __divdc3, reference order */

typedef struct fmmcu_ctx fmmcu_ctx;

/* One near-field evaluation (reference NearFieldJob, backend.hpp:27-37),
 * flattened.  Leaf i of the finest level owns permuted sources
 * [pt_off[i], pt_off[i+1]) and permuted evals [ev_off[i], ev_off[i+1])
 * (MBox::point_begin/end, eval_begin/end, geometry.hpp:22-23 — contiguous at
 * the finest level); its strong list (LevelConn::strong, geometry.hpp:44-47,
 * self included, ascending) is strong_idx[strong_off[i] .. strong_off[i+1]).
 * Complex arrays are interleaved (re, im) doubles, i.e. the bytes of
 * std::vector<std::complex<double>>. */
typedef struct {
  uint32_t n_leaves;
  uint32_t n_src;
  uint32_t n_eval;
  const uint32_t *pt_off;     /* [n_leaves + 1] */
  const uint32_t *ev_off;     /* [n_leaves + 1] */
  const uint32_t *strong_off; /* [n_leaves + 1] */
  const uint32_t *strong_idx; /* [strong_off[n_leaves]] */
  const uint32_t *perm;       /* [n_src]  Pyramid::perm (self-skip compares perm[j] to eval_sid) */
  const double *src_z;        /* [2 n_src]  permuted source positions */
  const double *src_m;        /* [2 n_src]  permuted strengths */
  const double *eval_y;       /* [2 n_eval] permuted eval positions */
  const int64_t *eval_sid;    /* [n_eval] permuted source ids, -1 = none; NULL = no ids */
  int kernel;                 /* FMMCU_KERNEL_* */
  int smoother;               /* FMMCU_SMOOTH_* */
  double delta;
  int mode;                   /* FMMCU_MODE_* */
  uint32_t leaf_begin;        /* target-leaf shard [leaf_begin, leaf_end); 0,n_leaves = all */
  uint32_t leaf_end;
  double *out;                /* [2 n_eval] host; slots of the shard's evals are written */
} fmmcu_p2p_job;

/* M2L sums for every (target box, weak partner) pair of every level
 * (downward pass, engine.cpp:96-114): out[t] = sum over weak_idx of
 * m2l_add(outgoing[src], local about centers[target_box[t]]), partners in
 * ascending order.  Box ids are global (all levels concatenated). */
typedef struct {
  int p;                      /* expansion order, <= 96 */
  int kernel;                 /* FMMCU_KERNEL_* */
  uint32_t n_boxes;           /* global box count */
  const double *centers;      /* [2 n_boxes] */
  const double *coeffs;       /* [2 (p+1) n_boxes] outgoing coefficients */
  uint32_t n_targets;
  const uint32_t *target_box; /* [n_targets] */
  const uint32_t *weak_off;   /* [n_targets + 1] */
  const uint32_t *weak_idx;   /* [weak_off[n_targets]] */
  double *out;                /* [2 (p+1) n_targets] host */
} fmmcu_m2l_job;

/* ---- context ---------------------------------------------------------- */
int fmmcu_create(fmmcu_ctx **ctx, int device);
void fmmcu_destroy(fmmcu_ctx *ctx);
const char *fmmcu_last_error(const fmmcu_ctx *ctx);
int fmmcu_device_count(int *count);

/* ---- reference-facing near field (host buffers) ------------------------- */
/* Asynchronous: packs the job into pinned staging, enqueues H2D, the P2P
 * kernels and the D2H of the shard's potentials, and returns.  All job
 * pointers must stay valid until fmmcu_p2p_finish returns. */
int fmmcu_p2p_launch(fmmcu_ctx *ctx, const fmmcu_p2p_job *job);
/* Blocks (without spinning) until the launched job completed, scatters the
 * potentials into job->out and reports NearFieldStats: pair_evals (exact,
 * reference counting) and seconds (launch start -> results on host). */
int fmmcu_p2p_finish(fmmcu_ctx *ctx, uint64_t *pair_evals, double *seconds);

/* Page-lock caller memory (cudaHostRegister).  When job->out of
 * fmmcu_p2p_launch is page-locked, the potentials are copied straight into it
 * slice by slice instead of through pinned staging + a host copy in finish. */
int fmmcu_host_register(fmmcu_ctx *ctx, void *ptr, uint64_t bytes);
int fmmcu_host_unregister(fmmcu_ctx *ctx, void *ptr);
/* The same without a context (portable registration, every context sees it):
 * used by owners of long-lived host buffers, e.g. the engine handle of
 * include/fmm_host.h that keeps its SourceSet / EvalSet / EvalResult between
 * evaluations, so the device pipeline DMAs them in place. */
int fmmcu_pin_host(void *ptr, uint64_t bytes);
int fmmcu_unpin_host(void *ptr);

/* ---- device-resident near field (benchmarks, multi-GPU sharding) -------- */
/* Uploads and packs the job's inputs once (synchronous); they stay resident. */
int fmmcu_p2p_stage(fmmcu_ctx *ctx, const fmmcu_p2p_job *job);
/* Enqueues only the P2P kernels over [leaf_begin, leaf_end) of the staged
 * job on the context stream; potentials stay on the device (permuted eval
 * order, double2).  *launches receives the number of kernels enqueued. */
int fmmcu_p2p_run_staged(fmmcu_ctx *ctx, uint32_t leaf_begin, uint32_t leaf_end, int mode,
                         int *launches);
/* Device pointer to the staged potentials ([2 n_eval] doubles). */
int fmmcu_p2p_device_out(fmmcu_ctx *ctx, double **dptr);
/* Make subsequent runs write potentials into caller-owned device memory
 * ([2 n_eval] doubles on this context's device, e.g. a torch tensor that is
 * then all-gathered with NCCL); NULL restores the internal buffer. */
int fmmcu_p2p_bind_device_out(fmmcu_ctx *ctx, double *dptr);
/* Synchronous D2H of potentials [eval_begin, eval_end) of the last run. */
int fmmcu_p2p_copy_out(fmmcu_ctx *ctx, double *host, uint32_t eval_begin, uint32_t eval_end);
/* Pair count of the last run (exact; waits for it). */
int fmmcu_p2p_pairs(fmmcu_ctx *ctx, uint64_t *pair_evals);
/* Pair work of leaves [0, n) of the staged job, prefix-summed on the host
 * ([n_leaves + 1] uint64, before self-skips) -- for work-balanced shards. */
int fmmcu_p2p_work_prefix(fmmcu_ctx *ctx, uint64_t *prefix);
/* Use an external stream (cudaStream_t) for subsequent work; NULL = own. */
int fmmcu_set_stream(fmmcu_ctx *ctx, void *stream);
int fmmcu_synchronize(fmmcu_ctx *ctx);

/* ---- M2L on the device --------------------------------------------------- */
/* Asynchronous.  Inputs in page-locked memory (fmmcu_m2l_host_buffers,
 * fmmcu_host_register) are DMA'd in place, and a page-locked job->out
 * receives the sums straight from the device; other memory is staged. */
int fmmcu_m2l_launch(fmmcu_ctx *ctx, const fmmcu_m2l_job *job);
int fmmcu_m2l_finish(fmmcu_ctx *ctx, uint64_t *m2l_ops, double *seconds);
/* Page-locked host arrays sized for one M2L job, owned by the context and
 * valid until the next call or fmmcu_destroy (grown, never shrunk).  A caller
 * that flattens its expansions and interaction lists straight into them (the
 * hybrid engine path) saves the staging copies of fmmcu_m2l_launch. */
typedef struct {
  double *centers, *coeffs, *out;
  uint32_t *target_box, *weak_off, *weak_idx;
} fmmcu_m2l_buffers;
int fmmcu_m2l_host_buffers(fmmcu_ctx *ctx, uint32_t n_boxes, int p, uint32_t n_targets,
                           uint64_t nnz, fmmcu_m2l_buffers *bufs);
/* Downward pass on the device after fmmcu_m2l_launch with job->out = NULL
 * (the sums then stay on the device): level by level, the local expansion of
 * every box with a target slot = l2l_add(parent local) (expansion.cpp,
 * levels >= 2) + its M2L sum, as the reference's downward pass
 * (engine.cpp:96-114); the locals of the finest level's boxes go to
 * finest_out (row = box index within the finest level; rows of boxes without
 * a slot are not written).  Completes with fmmcu_m2l_finish. */
typedef struct {
  int n_levels;
  const uint32_t *level_base; /* [n_levels + 1] first global box id per level */
  const int32_t *target_of;   /* [n_boxes] target slot of each box, or -1 */
  double *finest_out;         /* [2 (p+1) boxes of the finest level] host */
} fmmcu_l2l_job;
int fmmcu_m2l_downward(fmmcu_ctx *ctx, const fmmcu_l2l_job *job);

/* ---- the whole FMM evaluation on one device ------------------------------
 * FmmEngine::evaluate (reference engine.cpp:208-347) with every phase on the
 * GPU: median-split pyramid and theta connectivity (bit-exact with
 * build_pyramid / build_connectivity, geometry.cpp:106-216), P2M, M2M, the
 * batched M2L, L2L, the P2P near field and near + L2P assembly.  Inputs and
 * the output are in the caller's original order (like evaluate()). */
typedef struct {
  uint32_t n_src;
  uint32_t n_eval;
  const double *src_z;       /* [2 n_src]  source positions */
  const double *src_m;       /* [2 n_src]  strengths */
  const double *eval_y;      /* [2 n_eval] eval positions */
  const int64_t *eval_sid;   /* [n_eval] source id of each eval (-1 none), or NULL */
  int n_levels;
  double theta;
  int p;                     /* expansion order (FmmConfig::expansion_order) */
  int kernel;                /* FMMCU_KERNEL_* */
  int smoother;              /* FMMCU_SMOOTH_* (near field only, as the reference) */
  double delta;
  double *out;               /* [2 n_eval] potentials, original eval order */
  /* optional: called once every input has been read (staged for upload, or
   * handed to the DMA engines when page-locked), before fmmcu_fmm_launch
   * returns -- on the launching thread, or on the helper thread that stages
   * the masses while the pyramid builds.  From then on the host only drives
   * the device, so the caller can prepare its result buffer without
   * competing for memory bandwidth with the staging copies.  The input arrays
   * must stay unchanged until fmmcu_fmm_launch returns. */
  void (*inputs_consumed)(void *arg);
  void *inputs_consumed_arg;
} fmmcu_fmm_job;

typedef struct {
  uint64_t p2p_pairs, m2l_ops, p2m_points, l2p_points; /* WorkCounters */
  double t_upload;      /* H2D of the inputs (device span, s) */
  double t_tree;        /* pyramid build */
  double t_connect;     /* connectivity + permutation/packing */
  double t_p2m_upward;  /* P2M + M2M chain (far stream) */
  double t_m2l;         /* M2L + L2L (far stream) */
  double t_p2p;         /* near-field kernels */
  double t_device;      /* first H2D .. potentials on the host */
  double t_total;       /* host wall time of the call */
  uint64_t h2d_bytes, d2h_bytes;
  /* the device analogue of the reference's cpu_wait (engine.cpp:312): how
   * long the far chain (P2M..M2L+L2L, far stream) sat finished before the
   * near field (P2P, main stream) ended, i.e. max(0, near end - far end) on
   * the device clock.  > 0 means the near field is the longer branch, which
   * is exactly what the reference's positive wait tells AT3a
   * (autotune.cpp:155: more levels). */
  double t_far_wait;
} fmmcu_fmm_stats;

int fmmcu_fmm_evaluate(fmmcu_ctx *ctx, const fmmcu_fmm_job *job, fmmcu_fmm_stats *stats);
/* The same call split in two: launch returns once the potentials' D2H is
 * enqueued; finish waits and writes them to `out` ([2 n_eval] doubles) chunk
 * by chunk as they land.  When job->out is page-locked (fmmcu_host_register)
 * the D2H lands in it directly, so it is written asynchronously after launch
 * returns and finish only waits (pass the same pointer to finish).  Page-
 * locked inputs are DMA'd in place.  A job with ids and n_eval == n_src is
 * built speculatively as self-evaluation; launch verifies the speculation
 * before it returns and re-runs without it if the evals are not the sources
 * (results are identical either way). */
int fmmcu_fmm_launch(fmmcu_ctx *ctx, const fmmcu_fmm_job *job);
int fmmcu_fmm_finish(fmmcu_ctx *ctx, double *out, fmmcu_fmm_stats *stats);
/* Only the pyramid and the theta-connectivity of the job (bit-exact with
 * build_pyramid / build_connectivity, geometry.cpp:106-216) on the device,
 * synchronously; src_m may be NULL.  Read the tree back with
 * fmmcu_fmm_tree_level / _perm / _lists (the hybrid engine's device_tree). */
int fmmcu_tree_build(fmmcu_ctx *ctx, const fmmcu_fmm_job *job);
/* The device-built pyramid / connectivity of the last fmmcu_fmm_evaluate
 * (parity checks).  Box layout as fmmh_tree_boxes: f64[5 n] = centre x, y,
 * half width, half height, radius; u32[4 n] = point and eval ranges. */
int fmmcu_fmm_tree_level(fmmcu_ctx *ctx, int level, uint32_t *n_boxes, double *f64,
                         uint32_t *u32);
int fmmcu_fmm_tree_perm(fmmcu_ctx *ctx, uint32_t *perm, uint32_t *eval_perm);
/* nnz of the level's strong (weak = 0) or weak (weak = 1) lists; off [n+1]
 * and idx [nnz] filled when non-NULL. */
int fmmcu_fmm_tree_lists(fmmcu_ctx *ctx, int level, int weak, uint64_t *nnz, uint32_t *off,
                         uint32_t *idx);

/* ---- diagnostics --------------------------------------------------------- */
/* Device restatement of glibc hypot (box radii / theta distances), batched. */
int fmmcu_hypot_batch(fmmcu_ctx *ctx, const double *xy, uint32_t n, double *out);
/* Kernels launched by this context since creation (evidence counter). */
uint64_t fmmcu_kernel_launches(const fmmcu_ctx *ctx);
/* Host<->device bytes moved by the last fmmcu_p2p_launch (H2D: packed
 * sources, evals, self map, CSR and work list; D2H: potentials + counter). */
int fmmcu_last_transfer_bytes(const fmmcu_ctx *ctx, uint64_t *h2d, uint64_t *d2h);
/* Shape of the staged fast work list: *symmetric = 1 when the mutual kernel
 * runs (self-evaluation: each leaf pair once), *evals_per_lane = E. */
int fmmcu_p2p_kernel_info(const fmmcu_ctx *ctx, int *symmetric, int *evals_per_lane);
/* Measured FP64 FMA throughput of this device (TFLOP/s, DFMA = 2 flops). */
int fmmcu_fp64_peak(fmmcu_ctx *ctx, double *tflops);

/* ---- multi-GPU: target-leaf shards, one process (rank) per GPU ----------
 * (replaces the per-leaf loop of backend.cpp:73-89 split over
 * ranks; the only exchange is the potentials' gather, backend.cpp:41-69 has
 * no cross-leaf reduction.)  Each rank stages its shard with
 * fmmcu_p2p_stage(job with leaf_begin/leaf_end) -- halo-only: just the
 * sources its strong lists read cross PCIe -- and runs
 * fmmcu_p2p_run_staged over its range.  The slices reach the root either
 *  (a) fused into the kernels' stores: the root exports its staged output
 *      buffer, every other rank maps it and binds it as its output, so the
 *      shard's potentials are written into the root's HBM over NVLink while
 *      the kernels run (no collective, no extra pass); or
 *  (b) with NCCL: one grouped ncclSend / ncclRecv of each rank's eval slice
 *      [eval_cuts[r], eval_cuts[r+1]) into the root's output at the same
 *      offset, enqueued on the context stream behind the kernels.
 * The root's potentials are complete once every rank's stream has passed
 * its kernels (a) or the gather (b). */
/* (a) root: IPC handle (FMMCU_IPC_HANDLE_BYTES) of its staged output buffer */
int fmmcu_p2p_out_ipc_handle(fmmcu_ctx *ctx, void *handle);
/* (a) other ranks: write subsequent runs' potentials into the root's buffer
 * (NULL unmaps and restores the context's own output). */
int fmmcu_p2p_bind_peer_out(fmmcu_ctx *ctx, const void *handle);
/* (b) NCCL (libnccl.so.2 loaded at run time): a unique id on one rank
 * (FMMCU_NCCL_ID_BYTES, shared out of band), then every rank joins. */
int fmmcu_nccl_unique_id(void *id);
int fmmcu_nccl_init(fmmcu_ctx *ctx, const void *id, int rank, int world);
/* (b) gather the ranks' eval slices of the staged output into the root's,
 * in place (eval_cuts: [world + 1] permuted-eval offsets). */
int fmmcu_nccl_gather_out(fmmcu_ctx *ctx, int root, const uint32_t *eval_cuts);

#ifdef __cplusplus
}
#endif
#endif /* FMM_CUDA_H_ */
