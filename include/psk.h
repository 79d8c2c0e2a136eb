/*
 * psk.h -- C-ABI of the B200 parallel Kalman filter / smoother library
 * (libpsk.so).  Plain pointers and sizes only; no torch / C++ types.
 *
 * This is the drop-in boundary for the reference's parallel drivers:
 *   psk_pkf   replaces parascan::pkf_run   (reference: proj/core/include/
 *             parascan/kalman_par.hpp:111-119)
 *   psk_prts  replaces parascan::prts_run  (kalman_par.hpp:156-179)
 *   psk_ptfs  replaces parascan::ptfs_run  (kalman_par.hpp:207-238)
 * with the executor slot `Backend&` (backend.hpp:39-44) filled by a psk
 * context, the scan selector `ScanSpec` (scan.hpp:32-44) passed as
 * (alg, sengupta_n), and the `Lgssm<S>` / `Measurements<S>` containers
 * (lgssm.hpp:29-45) passed as per-step arrays (psk_model).  The C++ shim
 * include/parascan_b200/cuda_backend.hpp wraps these entry points in the
 * reference's own signatures; INTEGRATION.md shows the bindings.
 *
 * Threading: a context serialises its calls (like PoolBackend, which must
 * not be driven by two callers at once, backend.hpp:82-88); distinct contexts
 * may be used from different threads.  Errors are reported by status code
 * and psk_last_error() (thread-local message), mirroring the reference
 * exception types (mat.hpp:21-32, scan.hpp:28-30).
 */
#ifndef PSK_H
#define PSK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the C++ shim maps them onto the reference exceptions */
typedef enum {
  PSK_OK = 0,
  PSK_E_DIM = 1,      /* DimensionMismatch       (mat.hpp:21-23)  */
  PSK_E_CONTRACT = 2, /* ContractViolation       (scan.hpp:28-30) */
  PSK_E_NOT_PD = 3,   /* NotPositiveDefinite     (mat.hpp:24-26)  */
  PSK_E_SINGULAR = 4, /* SingularMatrix          (mat.hpp:27-29)  */
  PSK_E_CUDA = 5,     /* CUDA runtime failure / no device          */
  PSK_E_NCCL = 6,     /* collective failure                        */
  PSK_E_ARG = 7,      /* bad argument (null pointer, bad enum)     */
  PSK_E_ALLOC = 8     /* out of device / pinned memory             */
} psk_status;

/* ScanAlg (scan.hpp:32-39) in the reference order, plus the new
 * single-pass decoupled look-back scan appended after SenguptaB. */
typedef enum {
  PSK_SEQUENTIAL = 0,
  PSK_HILLIS_STEELE = 1,
  PSK_BLELLOCH = 2,
  PSK_INPLACE_LAFI = 3,
  PSK_SENGUPTA_A = 4,
  PSK_SENGUPTA_B = 5,
  PSK_DECOUPLED_LOOKBACK = 6
} psk_alg;

typedef enum { PSK_F32 = 0, PSK_F64 = 1 } psk_dtype;
typedef enum { PSK_HOST = 0, PSK_DEVICE = 1 } psk_space;

/* Execution mode of a context.
 *  PSK_MODE_FAST  (default): chunked kernels -- each thread folds `chunk`
 *      consecutive steps into a scan element, the chunk elements are scanned
 *      with the selected ScanAlg, and a per-chunk pass writes the outputs.
 *      chunk = 1 is the paper's one-element-per-step formulation; chunk = 0
 *      (default) picks the chunk length per call so that the chunks exactly
 *      fill "waves" waves of co-resident threads.
 *  PSK_MODE_EXACT: the reference's level-by-level scan kernels
 *      (scan.hpp:198-444) with the reference's operation order and no FMA
 *      contraction -- bitwise equal to the reference CPU path. */
typedef enum { PSK_MODE_FAST = 0, PSK_MODE_EXACT = 1 } psk_mode;

/* Lgssm<S> + Measurements<S> (lgssm.hpp:29-45).  Field k of F/u/Q is the
 * transition k -> k+1 (F[0] acts on the prior); H/d/R/y[k] belong to the
 * measurement of step k+1 (lgssm.hpp:5-8).  Each field is an array of
 * row-major per-step blocks; `*_stride` is the distance between consecutive
 * steps in scalars: -1 = dense (block size), 0 = time-invariant broadcast.
 * All pointers live in `space`; bases and strides must keep 16-byte
 * alignment for device inputs (host inputs are repacked). */
typedef struct {
  uint64_t t;
  int32_t nx, ny;
  int32_t dtype; /* psk_dtype */
  int32_t space; /* psk_space */
  const void *f, *u, *q, *h, *d, *r, *y;
  int64_t f_stride, u_stride, q_stride, h_stride, d_stride, r_stride,
      y_stride;
  const void* prior_mean; /* [nx]     */
  const void* prior_cov;  /* [nx][nx] */
} psk_model;

typedef struct psk_ctx psk_ctx;

/* Create a context bound to CUDA device `device` (no host fallback: fails
 * with PSK_E_CUDA when no device is present). */
int psk_create(psk_ctx** ctx, int device);
/* A context over several devices (devices[0..ndev), repeats allowed: two
 * entries of one GPU are two streams of it).  On it psk_pkf / psk_prts shard
 * the time axis over the devices (shard reduce, exchange of the shard
 * elements by peer copies over NVLink, fold, finish -- the single-process
 * form of distributed.py), psk_ptfs runs the forward filter on the first half
 * of the devices and the backward filter on the second half, each
 * time-sharded (ptfs_run's devices, kalman_par.hpp:207-211, extended from
 * {1, 2} to halves), and the batch calls give each device a contiguous share
 * of the series.  Host inputs are copied shard by shard by the device that
 * owns the shard.  Calls are synchronous; dimensions without shard phases
 * (nx or ny > 4), exact mode and series shorter than the shard count run on
 * the first device.  Replaces: tools/bench_main.cpp:125-128 devices check. */
int psk_create_multi(psk_ctx** ctx, const int* devices, int ndev);
/* number of devices of a context (1 for psk_create) */
int psk_num_devices(psk_ctx* ctx);
int psk_destroy(psk_ctx* ctx);
/* Mode and tuning: mode (psk_mode), chunk length (>= 1, or 0 = auto) */
int psk_set_mode(psk_ctx* ctx, int mode);
int psk_set_chunk(psk_ctx* ctx, int chunk);
/* Named tuning options of the fast path:
 *   "chunk"     steps folded per thread, 0 = auto (same as psk_set_chunk)
 *   "waves"     auto chunk: the chunks fill this many waves of co-resident
 *               threads (default: 4 in FP64, 3 in FP32)
 *   "async"     1: psk_pkf / psk_prts / psk_ptfs return once their work is
 *               queued on the context's stream (outputs valid when the stream
 *               completes; errors are reported by psk_sync); default 0 =
 *               synchronous, like the reference's drivers
 *   "batch_streams"  sub-streams of psk_pkf_batch / psk_prts_batch (1..64,
 *               default 4)
 *   "shard_async"  1: the shard phases before psk_shard_smoother_finish and
 *               the folds return without synchronising the stream (errors
 *               are reported by the smoother finish); default 0
 *   "tile"      1 (default): state dimensions with a register-tiled warp
 *               instantiation (nx = 16, ny = 8) run it; 0: the runtime-
 *               dimension warp kernels (A/B comparisons)
 *   "dlb_trace" 1: diagnostics -- per-phase timestamps of every decoupled
 *               look-back scan of this context are appended to the file
 *               $PSK_DLB_TRACE (tools/dlb_trace.py); synchronises each scan
 * Returns PSK_E_ARG for an unknown key or value. */
int psk_set_option(psk_ctx* ctx, const char* key, int64_t value);
/* Wait for the context's queued work and report the first device error since
 * the last synchronising call (async mode). */
int psk_sync(psk_ctx* ctx);
/* Run on this CUDA stream (cudaStream_t as void*; NULL = context stream).
 * The entry points are synchronous: outputs are valid on return. */
int psk_set_stream(psk_ctx* ctx, void* stream);
/* The stream the context currently runs on (its own stream unless one was set
 * with psk_set_stream), so callers can order their own work against it. */
int psk_get_stream(psk_ctx* ctx, void** stream);

/* Parallel Kalman filter (Alg. 5).  mean[T][nx], cov[T][nx][nx] in
 * model->space, model->dtype. */
int psk_pkf(psk_ctx* ctx, const psk_model* model, int alg,
            uint64_t sengupta_n, void* mean, void* cov);
/* Parallel RTS smoother (Alg. 6): filter + reversed smoother scan. */
int psk_prts(psk_ctx* ctx, const psk_model* model, int alg,
             uint64_t sengupta_n, void* mean, void* cov);
/* Parallel two-filter smoother (Alg. 7).  The forward scan runs on
 * ctx_fwd and the reversed (shifted-element) scan on ctx_bwd; with
 * devices == 2 and contexts on different GPUs the two scans run
 * concurrently and the backward (eta, J) are moved to the forward device.
 * devices must be 1 or 2 (bench_main.cpp:125-128); the numbers do not
 * depend on it (test_kalman_par.cpp:209-227). */
int psk_ptfs(psk_ctx* ctx_fwd, psk_ctx* ctx_bwd, int devices,
             const psk_model* model, int alg, uint64_t sengupta_n, void* mean,
             void* cov);

/* Batches of independent series (no reference counterpart; SURVEY.md 8(f)
 * row 2, BASELINE configs[4]): series i is models[i] with outputs means[i],
 * covs[i] (each series its own T, dims, dtype, space, strides -- e.g.
 * time-invariant per-series models with stride-0 fields).  Every series is
 * validated before any work is queued; the series then run on
 * "batch_streams" (option, default 4) sub-streams of the context's stream,
 * so series too short to fill the GPU alone overlap.  Synchronous unless the
 * context is in async mode; on a failure the first failing series' status is
 * returned (series after it are not run). */
int psk_pkf_batch(psk_ctx* ctx, const psk_model* models, int count, int alg,
                  uint64_t sengupta_n, void* const* means, void* const* covs);
int psk_prts_batch(psk_ctx* ctx, const psk_model* models, int count, int alg,
                   uint64_t sengupta_n, void* const* means, void* const* covs);

/* ---- time-sharded PRTS: one process per GPU (paper_2511_10363_b200/
 * distributed.py).  A shard is the steps [lo, hi) of a
 * T-step series, passed as a DEVICE-space psk_model with t = hi - lo.  Unless
 * the shard contains step T-1, its f/u/q arrays carry one more transition at
 * local index t (needed by the smoother element of step hi-1).
 *   flags: PSK_SHARD_FIRST  lo == 0 (the first step absorbs the prior)
 *          PSK_SHARD_LAST   hi == T
 * Element and state buffers are device arrays in model->dtype:
 *   filter element    3 nx^2 + 2 nx scalars (A | b | C | eta | J), row-major
 *   smoother element  2 nx^2 + nx   scalars (E | g | L)
 *   state             nx + nx^2     scalars (mean | cov)
 * A reduce call leaves the shard's scanned chunk elements in the context for
 * the following finish call.  The only cross-GPU data are the shard elements
 * (gathered by the caller, e.g. an NCCL all_gather) and their folds. */
#define PSK_SHARD_FIRST 1
#define PSK_SHARD_LAST 2
/* PKF shards (and the forward half of a sharded PTFS): the filter finish
 * writes the shard's filtered stats to mean / cov and reports errors */
#define PSK_SHARD_FILTERED 4
/* filter pass, part 1: local element build + scan; elem_out = shard total */
int psk_shard_filter_reduce(psk_ctx* ctx, const psk_model* shard, int flags,
                            int alg, uint64_t sengupta_n, void* elem_out);
/* filter pass, part 2: filtered stats of the shard from carry_state (the
 * filtered state before the shard; NULL for the FIRST shard) */
int psk_shard_filter_finish(psk_ctx* ctx, const psk_model* shard, int flags,
                            const void* carry_state, void* mean, void* cov);
/* smoother pass, part 1: mean/cov hold the shard's filtered stats;
 * elem_out = the shard's suffix smoothing element */
int psk_shard_smoother_reduce(psk_ctx* ctx, const psk_model* shard, int flags,
                              int alg, uint64_t sengupta_n, const void* mean,
                              const void* cov, void* elem_out);
/* smoother pass, part 2: smoothed stats written in place over mean/cov from
 * carry_state (the smoothed state after the shard; NULL for the LAST shard) */
int psk_shard_smoother_finish(psk_ctx* ctx, const psk_model* shard, int flags,
                              const void* carry_state, void* mean, void* cov);
/* prefix fold e_0 (x) ... (x) e_{count-1} of gathered filter elements (the
 * first contains a_1) -> filtered state; suffix fold of smoother elements
 * (the last contains a_T) -> smoothed state.  Device buffers, on ctx. */
int psk_fold_filter(psk_ctx* ctx, int dtype, int nx, const void* elems,
                    int count, void* state_out);
int psk_fold_smoother(psk_ctx* ctx, int dtype, int nx, const void* elems,
                      int count, void* state_out);

/* ---- time-sharded PTFS (ptfs_run on disjoint GPU halves, kalman_par.hpp:
 * 207-238): the forward filter runs as a sharded PKF
 * (PSK_SHARD_FILTERED) on one half of the GPUs while the backward filter runs
 * sharded on the other half, shard for shard over the same step ranges.  A
 * backward shard carries one extra step of EVERY field (slot i holds the
 * element of step i+1, kalman_par.hpp:63-89) unless it is the LAST.
 *   backward reduce: shifted elements + reverse scan; elem_out = the shard's
 *     backward total (filter element, later steps on the right);
 *   psk_fold_backward: e_0 (x) ... (x) e_{count-1} of the LATER shards'
 *     totals -> (eta | J), nx + nx^2 scalars (the backward information of
 *     every step after the shard);
 *   backward finish: from carry (eta | J; NULL for the LAST shard) and the
 *     shard's filtered stats fmean / fcov (device, from the forward half),
 *     the smoothed stats (two-filter combination, kalman_seq.hpp:239-260). */
int psk_shard_backward_reduce(psk_ctx* ctx, const psk_model* shard, int flags,
                              int alg, uint64_t sengupta_n, void* elem_out);
int psk_fold_backward(psk_ctx* ctx, int dtype, int nx, const void* elems,
                      int count, void* info_out);
int psk_shard_backward_finish(psk_ctx* ctx, const psk_model* shard, int flags,
                              const void* carry_info, const void* fmean,
                              const void* fcov, void* mean, void* cov);

/* Per-kernel device time of the last call, for roofline accounting:
 * fills up to `cap` entries of names[i] (static strings) / ms[i]; returns
 * the number of recorded kernels (recording enabled by psk_set_profile). */
int psk_set_profile(psk_ctx* ctx, int enable);
int psk_last_profile(psk_ctx* ctx, const char** names, float* ms, int cap);

/* Number of this library's kernels launched by the last call. */
int64_t psk_last_launch_count(psk_ctx* ctx);

/* Pinned (page-locked, portable) host memory for HOST-space models and
 * outputs: the input / output copies of a call then run at full PCIe speed
 * instead of staging through pageable buffers.  The C++ shim's marshalling
 * (include/parascan_b200/cuda_backend.hpp) packs the reference containers
 * into such a buffer.  bytes = 0 yields NULL; psk_host_free(NULL) is a no-op. */
int psk_host_alloc(void** p, size_t bytes);
int psk_host_free(void* p);

/* Thread-local message of the last failing call on this thread. */
const char* psk_last_error(void);
/* Library version string. */
const char* psk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PSK_H */
