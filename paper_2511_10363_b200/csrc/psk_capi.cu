// psk_capi.cu -- the C-ABI (include/psk.h): contexts, validation with the
// reference's contract semantics, host<->device marshalling, dispatch to the
// fast or exact device path, and status mapping.  There is no host compute
// path: every numeric result comes from the CUDA kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/psk.h"
#include "psk_common.cuh"
#include "psk_exact.h"
#include "psk_plan.hpp"

using namespace psk;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

const char* cuda_msg(cudaError_t e) { return cudaGetErrorString(e); }

}  // namespace

struct psk_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int mode = PSK_MODE_FAST;
  long long chunk = 0;  // 0: auto (whole waves of chunks)
  int waves = 0;        // waves of chunks for the auto chunk length (0: per precision)
  int tile = 1;         // register-tiled kernels for their (nx, ny) (option "tile")
  int shard_async = 0;  // shard phases 0-2 and folds return without a host sync
  int async = 0;        // drivers return once queued; psk_sync reports errors
  unsigned* d_err = nullptr;
  std::mutex mu;
  ExactLaunch launch;
  std::vector<void*> allocs;   // per-call device allocations
  std::vector<void*> persist;  // sharded-run scratch kept between calls
  void* shard_scratch = nullptr;
  int shard_dtype = -1;
  int shard_alg = 6;
  uint64_t shard_sn = 1;
  std::vector<std::pair<const char*, float>> profile;
  // batched calls: series i runs on sub[i % batch_streams]
  int batch_streams = 4;
  std::vector<cudaStream_t> sub;
  std::vector<cudaEvent_t> sub_ev;  // fork (index 0) / join events
  // multi-device context (psk_create_multi): one member context per device
  // entry; the time axis is sharded over them
  std::vector<psk_ctx*> members;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void* ctx_alloc(size_t bytes, void* c) {
  psk_ctx* ctx = static_cast<psk_ctx*>(c);
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  if (cudaMallocAsync(&p, bytes, ctx->stream) != cudaSuccess) return nullptr;
  ctx->allocs.push_back(p);
  return p;
}
void ctx_free_all(psk_ctx* ctx) {
  for (void* p : ctx->allocs) cudaFreeAsync(p, ctx->stream);
  ctx->allocs.clear();
}
void* ctx_alloc_persist(size_t bytes, void* c) {
  psk_ctx* ctx = static_cast<psk_ctx*>(c);
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  if (cudaMallocAsync(&p, bytes, ctx->stream) != cudaSuccess) return nullptr;
  ctx->persist.push_back(p);
  return p;
}
void ctx_free_persist(psk_ctx* ctx) {
  for (void* p : ctx->persist) cudaFreeAsync(p, ctx->stream);
  ctx->persist.clear();
}

inline bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// per-field description used for marshalling
struct Field {
  const void* src;
  int64_t stride;  // in scalars, after resolving -1
  long long block; // scalars per step
  const char* name;
};

// dst[k * dp + b] = src[k * sp + b] for b < bytes, k < rows (4-byte units:
// every block and pitch here is a multiple of sizeof(float))
__global__ void k_repitch(unsigned* dst, long long dp, const unsigned* src, long long sp,
                          int words, long long rows) {
  const long long n = rows * words;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long k = i / words;
    const int w = (int)(i - k * words);
    dst[k * dp + w] = src[k * sp + w];
  }
}
cudaError_t repitch(void* dst, size_t dpitch, const void* src, size_t spitch, size_t bytes,
                    long long rows, cudaStream_t stream) {
  const int words = (int)(bytes / 4);
  const long long n = rows * words;
  const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 32);
  k_repitch<<<grid < 1 ? 1 : grid, 256, 0, stream>>>(
      static_cast<unsigned*>(dst), (long long)(dpitch / 4), static_cast<const unsigned*>(src),
      (long long)(spitch / 4), words, rows);
  return cudaGetLastError();
}

// Resolve a model into a device ModelView<S>: device inputs are used in place
// when 16-byte aligned, host (or misaligned) inputs are packed into dense
// device arrays (time-invariant fields keep a single block, stride 0).
template <typename S>
int prepare_model(psk_ctx* ctx, const psk_model* m, ModelView<S>& v, int extra_fuq = 0,
                  bool force_copy = false, bool extra_all = false) {
  const long long T = (long long)m->t;
  const int nx = m->nx, ny = m->ny;
  Field f[7] = {{m->f, m->f_stride, (long long)nx * nx, "f"},
                {m->u, m->u_stride, nx, "u"},
                {m->q, m->q_stride, (long long)nx * nx, "q"},
                {m->h, m->h_stride, (long long)ny * nx, "h"},
                {m->d, m->d_stride, ny, "d"},
                {m->r, m->r_stride, (long long)ny * ny, "r"},
                {m->y, m->y_stride, ny, "y"}};
  const S* outp[7];
  long long outs[7];
  // `force_copy`: device inputs that live on another GPU (two-context PTFS)
  // are staged like host inputs; cudaMemcpyDefault resolves every pair.
  const bool host = m->space == PSK_HOST || force_copy;
  for (int i = 0; i < 7; ++i) {
    if (!f[i].src) return fail(PSK_E_ARG, std::string("null model field ") + f[i].name);
    long long st = f[i].stride < 0 ? f[i].block : f[i].stride;
    const size_t bb = sizeof(S) * (size_t)f[i].block;
    // Device arrays are used in place when the TMA stage (psk_stage.cuh) can
    // read them: 16-byte aligned base, per-step pitch a multiple of 16 bytes,
    // and blocks that are whole 16-byte rows (the stage reads rounded rows).
    // Dense blocks of 4 / 8 bytes (d, y at small ny in FP32, ...) are used as
    // they are too: the stage groups 16 / bytes consecutive steps per row.
    const bool small_dense = bb < 16 && 16 % bb == 0 && (size_t)st * sizeof(S) == bb;
    const bool dense_ok = !host && (reinterpret_cast<uintptr_t>(f[i].src) % 16) == 0 &&
                          ((bb % 16 == 0 && ((size_t)st * sizeof(S)) % 16 == 0) ||
                           small_dense || st == 0);
    if (dense_ok) {
      outp[i] = static_cast<const S*>(f[i].src);
      outs[i] = st;
      continue;
    }
    // pack: one block if broadcast, else T blocks (plus the boundary
    // transition of a sharded run for f/u/q) at a 16-byte-rounded pitch
    const long long nblk =
        st == 0 ? 1
                : (T > 0 ? T : 1) + ((extra_all || i == 0 || i == 1 || i == 2) ? extra_fuq : 0);
    // small dense blocks keep their dense pitch (grouped rows), the rest is
    // rounded up to whole 16-byte rows
    const size_t pb = (bb < 16 && 16 % bb == 0) ? bb : (bb + 15) / 16 * 16;
    S* dst = static_cast<S*>(ctx_alloc(pb * (size_t)nblk, ctx));
    if (!dst) return fail(PSK_E_ALLOC, "device allocation failed (model)");
    const cudaMemcpyKind kind = cudaMemcpyDefault;
    cudaError_t e = cudaSuccess;
    const size_t sp = st == 0 ? bb : sizeof(S) * (size_t)st;  // source pitch (bytes)
    if (st != 0 && pb == bb && sp == bb) {
      e = cudaMemcpyAsync(dst, f[i].src, bb * (size_t)nblk, kind, ctx->stream);
    } else if (st == 0 || nblk == 1) {
      e = cudaMemcpyAsync(dst, f[i].src, bb, kind, ctx->stream);
    } else {
      // re-pitch on the device (a 2-D memcpy with rows of a few bytes runs
      // far below HBM speed: 3.7 ms for the two 8-byte FP32 fields at 2^24)
      const void* src = f[i].src;
      if (host) {  // dense H2D of the source span first
        void* tmp = ctx_alloc(sp * (size_t)nblk, ctx);
        if (!tmp) return fail(PSK_E_ALLOC, "device allocation failed (model staging)");
        e = cudaMemcpyAsync(tmp, src, sp * (size_t)(nblk - 1) + bb, kind, ctx->stream);
        src = tmp;
      }
      if (e == cudaSuccess) e = repitch(dst, pb, src, sp, bb, nblk, ctx->stream);
    }
    if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("model copy: ") + cuda_msg(e));
    outp[i] = dst;
    outs[i] = st == 0 ? 0 : (long long)(pb / sizeof(S));
  }
  // prior
  const void* pm = m->prior_mean;
  const void* pc = m->prior_cov;
  if (!pm || !pc) return fail(PSK_E_ARG, "null prior");
  S* prior = static_cast<S*>(ctx_alloc(sizeof(S) * (size_t)(nx + nx * nx + 8), ctx));
  if (!prior) return fail(PSK_E_ALLOC, "device allocation failed (prior)");
  // prior mean at [0, nx) rounded up to a 16-byte boundary, cov after it
  const int moff = (int)((sizeof(S) * nx + 15) / 16 * 16 / sizeof(S));
  S* pcov = prior + moff;
  const cudaMemcpyKind kind = cudaMemcpyDefault;
  cudaError_t e1 = cudaMemcpyAsync(prior, pm, sizeof(S) * nx, kind, ctx->stream);
  cudaError_t e2 = cudaMemcpyAsync(pcov, pc, sizeof(S) * nx * nx, kind, ctx->stream);
  if (e1 != cudaSuccess || e2 != cudaSuccess)
    return fail(PSK_E_CUDA, "prior copy failed");
  v.f = outp[0]; v.u = outp[1]; v.q = outp[2]; v.h = outp[3];
  v.d = outp[4]; v.r = outp[5]; v.y = outp[6];
  v.sf = outs[0]; v.su = outs[1]; v.sq = outs[2]; v.sh = outs[3];
  v.sd = outs[4]; v.sr = outs[5]; v.sy = outs[6];
  v.m0 = prior;
  v.p0 = pcov;
  v.t = T;
  v.nx = nx;
  v.ny = ny;
  v.prior_first = 1;
  v.last_step = T - 1;
  if (host || force_copy) ctx->launch.mark("h2d_inputs");  // profile: copy span
  return PSK_OK;
}

// The reference's contract checks (scan.hpp:450-483 on padded_len,
// kalman_par.hpp:22-25), evaluated on the reference's own series length so
// the error behaviour does not depend on the device formulation.
int check_contract(int alg, uint64_t sengupta_n, uint64_t t) {
  if (alg < 0 || alg > PSK_DECOUPLED_LOOKBACK)
    return fail(PSK_E_ARG, "unknown scan algorithm");
  const unsigned long long n =
      (alg == PSK_SEQUENTIAL || alg == PSK_DECOUPLED_LOOKBACK) ? t : next_pow2(t);
  if (n == 0) return fail(PSK_E_CONTRACT, "scan of empty series");
  if (n == 1) return PSK_OK;
  if (alg == PSK_SENGUPTA_B && (sengupta_n < 2 || !is_pow2(sengupta_n)))
    return fail(PSK_E_CONTRACT, "sengupta_n must be a power of 2, >= 2");
  return PSK_OK;
}

template <typename S>
int run_typed(psk_ctx* ctx, const psk_model* m, int method, int alg,
              uint64_t sengupta_n, void* mean, void* cov) {
  const long long T = (long long)m->t;
  const int nx = m->nx;
  ModelView<S> v;
  int st = prepare_model<S>(ctx, m, v);
  if (st) return st;
  // outputs: device-resident and aligned are written in place
  const bool host = m->space == PSK_HOST;
  const size_t mb = sizeof(S) * (size_t)T * nx, cb = sizeof(S) * (size_t)T * nx * nx;
  S* dmean = static_cast<S*>(mean);
  S* dcov = static_cast<S*>(cov);
  const bool tmp_out = host || !aligned16(mean) || !aligned16(cov);
  if (tmp_out) {
    dmean = static_cast<S*>(ctx_alloc(mb + 16, ctx));
    dcov = static_cast<S*>(ctx_alloc(cb + 16, ctx));
    if (!dmean || !dcov) return fail(PSK_E_ALLOC, "device allocation failed (outputs)");
  }
  ExactLaunch& L = ctx->launch;
  bool done = false;  // served by a fast (register-resident or wide) path
  if (ctx->mode == PSK_MODE_FAST && fast_supported<S>(m->nx, m->ny)) {
    FastArgs a;
    a.method = method;
    a.alg = alg;
    a.sengupta_n = sengupta_n;
    a.chunk = ctx->chunk;
    a.waves = ctx->waves;
    st = fast_run<S>(L, v, a, dmean, dcov, ctx_alloc, ctx);
    if (st == 2) return fail(PSK_E_CONTRACT, "chunk scan contract violation");
    if (st == 8) return fail(PSK_E_ALLOC, "device allocation failed (scan)");
    if (st) return fail(PSK_E_CUDA, "fast path failed");
    done = true;
  }
  if (!done && ctx->mode == PSK_MODE_FAST) {
    // dims without a register-resident instantiation: warp-per-chunk kernels
    FastArgs a;
    a.method = method;
    a.alg = alg;
    a.sengupta_n = sengupta_n;
    a.chunk = ctx->chunk;
    a.waves = ctx->waves;
    a.tile = ctx->tile;
    st = wide_run<S>(L, v, a, dmean, dcov, ctx_alloc, ctx);
    if (st == 2) return fail(PSK_E_CONTRACT, "chunk scan contract violation");
    if (st == 8) return fail(PSK_E_ALLOC, "device allocation failed (wide scan)");
    if (st > 0) return fail(PSK_E_CUDA, "wide fast path failed");
    done = st == 0;
  }
  if (!done) {
    if (alg == PSK_DECOUPLED_LOOKBACK) {
      if (ctx->mode != PSK_MODE_FAST)
        return fail(PSK_E_CONTRACT,
                    "decoupled look-back is a fast-path scan (not in the "
                    "reference's level-by-level set)");
      alg = PSK_INPLACE_LAFI;  // fast mode, uncovered request (wide PTFS)
    }
    const unsigned long long n = alg == PSK_SEQUENTIAL ? T : next_pow2(T);
    ScanPlan plan = make_scan_plan(alg, sengupta_n, (long long)n);
    if (plan.status) return fail(PSK_E_CONTRACT, plan.why);
    const size_t fs = (size_t)(3 * nx * nx + 2 * nx);
    S* el0 = static_cast<S*>(ctx_alloc(sizeof(S) * fs * n, ctx));
    S* el1 = static_cast<S*>(ctx_alloc(sizeof(S) * fs * (plan.cap1 ? plan.cap1 : 1), ctx));
    S* el2 = static_cast<S*>(ctx_alloc(sizeof(S) * fs * (plan.cap2 ? plan.cap2 : 1), ctx));
    S* bel0 = method == 2 ? static_cast<S*>(ctx_alloc(sizeof(S) * fs * n, ctx)) : el0;
    if (!el0 || !el1 || !el2 || !bel0) return fail(PSK_E_ALLOC, "device allocation failed (exact)");
    exact_run<S>(L, v, method, plan, el0, el1, el2, bel0, dmean, dcov);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("kernel launch: ") + cuda_msg(e));
  if (tmp_out && T > 0) {
    const cudaMemcpyKind kind = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    cudaMemcpyAsync(mean, dmean, mb, kind, ctx->stream);
    cudaMemcpyAsync(cov, dcov, cb, kind, ctx->stream);
    ctx->launch.mark(host ? "d2h_outputs" : "d2d_outputs");
  }
  return PSK_OK;
}

int run_entry(psk_ctx* ctx, const psk_model* m, int method, int alg,
              uint64_t sengupta_n, void* mean, void* cov) {
  // argument and contract validation first (host-only, no device needed),
  // then the context
  if (!m) return fail(PSK_E_ARG, "null model");
  if (m->nx < 1 || m->nx > 16 || m->ny < 1 || m->ny > 16)
    return fail(PSK_E_DIM, "mat dims");  // Mat requires 1..kMaxDim (mat.hpp:19, 326)
  if (m->dtype != PSK_F32 && m->dtype != PSK_F64) return fail(PSK_E_ARG, "bad dtype");
  if (m->space != PSK_HOST && m->space != PSK_DEVICE) return fail(PSK_E_ARG, "bad space");
  int st = check_contract(alg, sengupta_n, m->t);
  if (st) return st;
  if (m->t > 0 && (!mean || !cov)) return fail(PSK_E_ARG, "null output");
  if (!ctx) return fail(PSK_E_ARG, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg(ctx->device);
  ctx->launch.stream = ctx->stream;
  ctx->launch.err = ctx->d_err;
  // "async" mode: the call returns once its work is queued on the stream;
  // the device error word accumulates and the per-kernel event spans are
  // kept until psk_sync reports them
  ctx->launch.start(ctx->async != 0);
  if (!ctx->async) cudaMemsetAsync(ctx->d_err, 0, sizeof(unsigned), ctx->stream);
  st = m->dtype == PSK_F64 ? run_typed<double>(ctx, m, method, alg, sengupta_n, mean, cov)
                           : run_typed<float>(ctx, m, method, alg, sengupta_n, mean, cov);
  if (ctx->async) {
    ctx_free_all(ctx);  // stream-ordered frees
    if (st) return st;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("kernel launch: ") + cuda_msg(e));
    return PSK_OK;
  }
  unsigned herr = 0;
  cudaMemcpyAsync(&herr, ctx->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream);
  ctx_free_all(ctx);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (st) return st;
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("execution: ") + cuda_msg(e));
  ctx->profile.clear();
  if (ctx->launch.profile && ctx->launch.evs.size() > 1) {
    for (size_t i = 0; i + 1 < ctx->launch.evs.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->launch.evs[i], ctx->launch.evs[i + 1]);
      ctx->profile.emplace_back(ctx->launch.names[i], ms);
    }
  }
  if (herr & kErrNotPD) return fail(PSK_E_NOT_PD, "cholesky pivot");
  if (herr & kErrSingular) return fail(PSK_E_SINGULAR, "lu zero pivot");
  return PSK_OK;
}

// A batch of independent series: every series is
// validated first, then series i is queued on the context's sub-stream
// i % batch_streams (forked from and joined back into the context's stream),
// so short series that do not fill the GPU alone run concurrently.  One
// synchronisation at the end (none in async mode).
int batch_entry(psk_ctx* ctx, const psk_model* ms, int count, int method, int alg,
                uint64_t sengupta_n, void* const* means, void* const* covs) {
  if (count < 0) return fail(PSK_E_ARG, "negative batch count");
  if (count > 0 && (!ms || !means || !covs)) return fail(PSK_E_ARG, "null batch array");
  for (int i = 0; i < count; ++i) {
    const psk_model* m = &ms[i];
    if (m->nx < 1 || m->nx > 16 || m->ny < 1 || m->ny > 16) return fail(PSK_E_DIM, "mat dims");
    if (m->dtype != PSK_F32 && m->dtype != PSK_F64) return fail(PSK_E_ARG, "bad dtype");
    if (m->space != PSK_HOST && m->space != PSK_DEVICE) return fail(PSK_E_ARG, "bad space");
    const int st = check_contract(alg, sengupta_n, m->t);
    if (st) return st;
    if (m->t > 0 && (!means[i] || !covs[i])) return fail(PSK_E_ARG, "null output");
  }
  if (!ctx) return fail(PSK_E_ARG, "null context");
  if (count == 0) return PSK_OK;
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg(ctx->device);
  const int k = std::max(1, std::min(count, ctx->batch_streams));
  while ((int)ctx->sub.size() < k) {
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
      return fail(PSK_E_CUDA, "batch stream creation failed");
    ctx->sub.push_back(s);
  }
  while ((int)ctx->sub_ev.size() < k + 1) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return fail(PSK_E_CUDA, "batch event creation failed");
    ctx->sub_ev.push_back(e);
  }
  cudaStream_t main = ctx->stream;
  const bool prof = ctx->launch.profile;
  ctx->launch.profile = false;  // event spans across streams are not per-kernel times
  ctx->launch.err = ctx->d_err;
  ctx->launch.stream = main;
  ctx->launch.start(ctx->async != 0);
  if (!ctx->async) cudaMemsetAsync(ctx->d_err, 0, sizeof(unsigned), main);
  cudaEventRecord(ctx->sub_ev[0], main);
  for (int j = 0; j < k; ++j) cudaStreamWaitEvent(ctx->sub[j], ctx->sub_ev[0], 0);
  int st = PSK_OK;
  long long launches = 0;
  for (int i = 0; i < count && st == PSK_OK; ++i) {
    ctx->stream = ctx->sub[i % k];
    ctx->launch.stream = ctx->stream;
    ctx->launch.launches = 0;
    const psk_model* m = &ms[i];
    st = m->dtype == PSK_F64
             ? run_typed<double>(ctx, m, method, alg, sengupta_n, means[i], covs[i])
             : run_typed<float>(ctx, m, method, alg, sengupta_n, means[i], covs[i]);
    launches += ctx->launch.launches;
    ctx_free_all(ctx);  // stream-ordered on the series' stream
  }
  for (int j = 0; j < k; ++j) {
    cudaEventRecord(ctx->sub_ev[j + 1], ctx->sub[j]);
    cudaStreamWaitEvent(main, ctx->sub_ev[j + 1], 0);
  }
  ctx->stream = main;
  ctx->launch.stream = main;
  ctx->launch.launches = launches;
  ctx->launch.profile = prof;
  if (st) {
    cudaStreamSynchronize(main);
    return st;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("kernel launch: ") + cuda_msg(e));
  if (ctx->async) return PSK_OK;
  unsigned herr = 0;
  cudaMemcpyAsync(&herr, ctx->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, main);
  e = cudaStreamSynchronize(main);
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("execution: ") + cuda_msg(e));
  ctx->profile.clear();
  if (herr & kErrNotPD) return fail(PSK_E_NOT_PD, "cholesky pivot");
  if (herr & kErrSingular) return fail(PSK_E_SINGULAR, "lu zero pivot");
  return PSK_OK;
}

// ---- time-sharded phases --------------------------------------------------
// phases: 0 filter reduce + scan, 1 filter finish, 2 smoother reduce + scan,
// 3 smoother finish (PRTS, or PKF with PSK_SHARD_FILTERED: phase 1 writes the
// filtered stats); 4 backward reduce + reverse scan, 5 backward finish fused
// with the two-filter combination (the backward half of a sharded PTFS, whose
// forward states arrive as dense filtered stats fmean / fcov)
template <typename S>
int shard_typed(psk_ctx* ctx, const psk_model* m, int flags, int phase, int alg,
                uint64_t sn, void* mean, void* cov, const void* carry, void* elem_out,
                const void* fmean = nullptr, const void* fcov = nullptr) {
  ModelView<S> v;
  const int extra = (flags & PSK_SHARD_LAST) ? 0 : 1;
  const bool bwd = phase == 4 || phase == 5;
  // the backward pass reads element a(step i+1) at slot i: a shard that does
  // not end the series carries one extra step of every field
  int st = prepare_model<S>(ctx, m, v, extra, false, bwd);
  if (st) return st;
  v.prior_first = (flags & PSK_SHARD_FIRST) ? 1 : 0;
  v.last_step = (flags & PSK_SHARD_LAST) ? (long long)m->t - 1 : -1;
  FastArgs a;
  a.method = bwd ? 2 : ((flags & PSK_SHARD_FILTERED) ? 0 : 1);
  a.alg = alg;
  a.sengupta_n = sn;
  a.chunk = ctx->chunk;
  a.waves = ctx->waves;
  if (phase != 0 && phase != 2 && phase != 4) {  // finishes reuse the reduce's scan spec
    a.alg = ctx->shard_alg;
    a.sengupta_n = ctx->shard_sn;
  } else {
    ctx->shard_alg = alg;
    ctx->shard_sn = sn;
  }
  if (phase == 0 || phase == 4) {
    ctx_free_persist(ctx);
    if (ctx->shard_scratch) {
      if (ctx->shard_dtype == PSK_F64) fast_shard_release<double>(ctx->shard_scratch);
      else fast_shard_release<float>(ctx->shard_scratch);
      ctx->shard_scratch = nullptr;
    }
    ctx->shard_dtype = m->dtype;
  } else if (!ctx->shard_scratch || ctx->shard_dtype != m->dtype) {
    return fail(PSK_E_ARG, "finish without a matching reduce on this context");
  }
  st = fast_shard_phase<S>(ctx->launch, v, a, phase, &ctx->shard_scratch,
                           static_cast<S*>(mean), static_cast<S*>(cov),
                           static_cast<const S*>(carry), static_cast<S*>(elem_out),
                           ctx_alloc_persist, ctx, static_cast<const S*>(fmean),
                           static_cast<const S*>(fcov));
  if (st == 2) return fail(PSK_E_CONTRACT, "chunk scan contract violation");
  if (st == 8) return fail(PSK_E_ALLOC, "device allocation failed (shard scan)");
  if (st) return fail(PSK_E_CUDA, "shard phase failed");
  return PSK_OK;
}

int finish_call(psk_ctx* ctx, int st) {
  unsigned herr = 0;
  cudaMemcpyAsync(&herr, ctx->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream);
  ctx_free_all(ctx);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (st) return st;
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("execution: ") + cuda_msg(e));
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("kernel launch: ") + cuda_msg(e));
  ctx->profile.clear();
  if (ctx->launch.profile && ctx->launch.evs.size() > 1) {
    for (size_t i = 0; i + 1 < ctx->launch.evs.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->launch.evs[i], ctx->launch.evs[i + 1]);
      ctx->profile.emplace_back(ctx->launch.names[i], ms);
    }
  }
  if (herr & kErrNotPD) return fail(PSK_E_NOT_PD, "cholesky pivot");
  if (herr & kErrSingular) return fail(PSK_E_SINGULAR, "lu zero pivot");
  return PSK_OK;
}

int shard_entry(psk_ctx* ctx, const psk_model* m, int flags, int phase, int alg, uint64_t sn,
                void* mean, void* cov, const void* carry, void* elem_out,
                const void* fmean = nullptr, const void* fcov = nullptr) {
  if (!m) return fail(PSK_E_ARG, "null model");
  if (flags & ~(PSK_SHARD_FIRST | PSK_SHARD_LAST | PSK_SHARD_FILTERED))
    return fail(PSK_E_ARG, "unknown shard flags");
  if (m->nx < 1 || m->nx > 16 || m->ny < 1 || m->ny > 16) return fail(PSK_E_DIM, "mat dims");
  if (m->dtype != PSK_F32 && m->dtype != PSK_F64) return fail(PSK_E_ARG, "bad dtype");
  if (m->space != PSK_DEVICE) return fail(PSK_E_ARG, "sharded runs take device-space shards");
  if (phase == 0 || phase == 2 || phase == 4) {
    int st = check_contract(alg, sn, m->t);
    if (st) return st;
  }
  if (m->t == 0) return fail(PSK_E_CONTRACT, "empty shard");
  if (!mean || !cov) return fail(PSK_E_ARG, "null stats buffer");
  if ((phase == 0 || phase == 2 || phase == 4) && !elem_out)
    return fail(PSK_E_ARG, "null element output");
  if (phase == 1 && !(flags & PSK_SHARD_FIRST) && !carry)
    return fail(PSK_E_ARG, "non-first shard needs the carried filtered state");
  if (phase == 3 && !(flags & PSK_SHARD_LAST) && !carry)
    return fail(PSK_E_ARG, "non-last shard needs the carried smoothed state");
  if (phase == 5 && !(flags & PSK_SHARD_LAST) && !carry)
    return fail(PSK_E_ARG, "non-last shard needs the carried backward information");
  if (phase == 5 && (!fmean || !fcov))
    return fail(PSK_E_ARG, "backward finish needs the shard's filtered stats");
  if (!ctx) return fail(PSK_E_ARG, "null context");
  if (!ctx->members.empty()) return fail(PSK_E_ARG, "shard phases take a single-device context");
  if (ctx->mode != PSK_MODE_FAST) return fail(PSK_E_ARG, "sharded runs use the fast path");
  const bool ok = m->dtype == PSK_F64 ? fast_supported<double>(m->nx, m->ny)
                                      : fast_supported<float>(m->nx, m->ny);
  if (!ok) return fail(PSK_E_DIM, "no fast-path instantiation for these dimensions");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg(ctx->device);
  ctx->launch.stream = ctx->stream;
  ctx->launch.err = ctx->d_err;
  ctx->launch.start(ctx->async != 0);
  // "shard_async": the phases before the smoother finish return without a
  // host synchronisation (the error word accumulates and is checked by the
  // final phase), so a rank's phases and its NCCL exchanges stay queued on
  // the stream back to back; "async": no phase synchronises (psk_sync does)
  // the final phases (smoother finish, PKF filter finish, backward finish)
  // synchronise and report the device errors of the whole sequence
  const bool final_phase = phase == 3 || phase == 5 || (phase == 1 && (flags & PSK_SHARD_FILTERED));
  const bool defer = (ctx->shard_async && !final_phase) || ctx->async;
  if (!ctx->async && (!ctx->shard_async || phase == 0 || phase == 4))
    cudaMemsetAsync(ctx->d_err, 0, sizeof(unsigned), ctx->stream);
  int st = m->dtype == PSK_F64
               ? shard_typed<double>(ctx, m, flags, phase, alg, sn, mean, cov, carry, elem_out,
                                     fmean, fcov)
               : shard_typed<float>(ctx, m, flags, phase, alg, sn, mean, cov, carry, elem_out,
                                    fmean, fcov);
  if (defer) {
    ctx_free_all(ctx);
    if (st) return st;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("kernel launch: ") + cuda_msg(e));
    return PSK_OK;
  }
  return finish_call(ctx, st);
}

int fold_entry(psk_ctx* ctx, int kind, int dtype, int nx, const void* elems, int count,
               void* out) {
  if (!ctx) return fail(PSK_E_ARG, "null context");
  if (!ctx->members.empty()) return fail(PSK_E_ARG, "folds take a single-device context");
  if (dtype != PSK_F32 && dtype != PSK_F64) return fail(PSK_E_ARG, "bad dtype");
  if (!elems || !out || count < 1) return fail(PSK_E_ARG, "bad fold arguments");
  if (nx < 1 || nx > 4) return fail(PSK_E_DIM, "fold supports nx 1..4");
  if (kind < 0 || kind > 2) return fail(PSK_E_ARG, "bad fold kind");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard dg(ctx->device);
  ctx->launch.stream = ctx->stream;
  ctx->launch.err = ctx->d_err;
  ctx->launch.start(ctx->async != 0);
  if (!ctx->shard_async && !ctx->async)
    cudaMemsetAsync(ctx->d_err, 0, sizeof(unsigned), ctx->stream);
  int st = dtype == PSK_F64
               ? fast_fold<double>(ctx->launch, kind, nx, static_cast<const double*>(elems),
                                   count, static_cast<double*>(out))
               : fast_fold<float>(ctx->launch, kind, nx, static_cast<const float*>(elems),
                                  count, static_cast<float*>(out));
  if (st) st = fail(PSK_E_ARG, "fold failed");
  if (ctx->shard_async || ctx->async) {  // see shard_entry
    if (st) return st;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("kernel launch: ") + cuda_msg(e));
    return PSK_OK;
  }
  return finish_call(ctx, st);
}

template <typename S>
int ptfs_two_typed(psk_ctx* cf, psk_ctx* cb, const psk_model* m, int alg, uint64_t sn,
                   void* mean, void* cov) {
  const long long T = (long long)m->t;
  const int nx = m->nx;
  ModelView<S> va, vb;
  int st;
  // device-space inputs that live on another GPU than a context are staged
  // like host inputs on that context (no peer access is assumed)
  auto foreign = [&](int dev) {
    if (m->space != PSK_DEVICE) return false;
    cudaPointerAttributes at{};
    const void* fields[9] = {m->f, m->u, m->q, m->h, m->d, m->r, m->y, m->prior_mean,
                             m->prior_cov};
    for (const void* p : fields) {
      if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (at.type == cudaMemoryTypeDevice && at.device != dev) return true;
    }
    return false;
  };
  {
    DeviceGuard dg(cb->device);
    st = prepare_model<S>(cb, m, vb, 0, foreign(cb->device));
    if (st) return st;
  }
  DeviceGuard dg(cf->device);
  st = prepare_model<S>(cf, m, va, 0, foreign(cf->device));
  if (st) return st;
  const bool host = m->space == PSK_HOST;
  const size_t mb = sizeof(S) * (size_t)T * nx, cb_ = sizeof(S) * (size_t)T * nx * nx;
  S* dmean = static_cast<S*>(mean);
  S* dcov = static_cast<S*>(cov);
  // device outputs on another GPU than the forward context are written
  // through a staging buffer on it (cudaMemcpyDefault resolves the pair)
  bool out_foreign = false;
  if (!host) {
    for (void* p : {mean, cov}) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, p) == cudaSuccess) {
        if (at.type == cudaMemoryTypeDevice && at.device != cf->device) out_foreign = true;
      } else {
        cudaGetLastError();
      }
    }
  }
  const bool tmp_out = host || out_foreign || !aligned16(mean) || !aligned16(cov);
  if (tmp_out) {
    dmean = static_cast<S*>(ctx_alloc(mb + 16, cf));
    dcov = static_cast<S*>(ctx_alloc(cb_ + 16, cf));
    if (!dmean || !dcov) return fail(PSK_E_ALLOC, "device allocation failed (outputs)");
  }
  FastArgs a;
  a.method = 2;
  a.alg = alg;
  a.sengupta_n = sn;
  a.chunk = cf->chunk;
  a.waves = cf->waves;
  st = fast_ptfs2<S>(cf->launch, va, cf->device, cb->launch, vb, cb->device, a, dmean, dcov,
                     ctx_alloc, cf, ctx_alloc, cb);
  cudaSetDevice(cf->device);
  if (st == 2) return fail(PSK_E_CONTRACT, "chunk scan contract violation");
  if (st == 8) return fail(PSK_E_ALLOC, "device allocation failed (scan)");
  if (st) return fail(PSK_E_CUDA, "two-context PTFS failed");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("kernel launch: ") + cuda_msg(e));
  if (tmp_out) {
    cudaMemcpyAsync(mean, dmean, mb, cudaMemcpyDefault, cf->stream);
    cudaMemcpyAsync(cov, dcov, cb_, cudaMemcpyDefault, cf->stream);
  }
  return PSK_OK;
}

int ptfs_two(psk_ctx* cf, psk_ctx* cb, const psk_model* m, int alg, uint64_t sn, void* mean,
             void* cov) {
  if (m->nx < 1 || m->nx > 16 || m->ny < 1 || m->ny > 16) return fail(PSK_E_DIM, "mat dims");
  if (m->dtype != PSK_F32 && m->dtype != PSK_F64) return fail(PSK_E_ARG, "bad dtype");
  if (m->space != PSK_HOST && m->space != PSK_DEVICE) return fail(PSK_E_ARG, "bad space");
  int st = check_contract(alg, sn, m->t);
  if (st) return st;
  if (!mean || !cov) return fail(PSK_E_ARG, "null output");
  // one caller at a time per context (like PoolBackend); lock in address
  // order so two concurrent two-context calls cannot deadlock
  psk_ctx* lo = cf < cb ? cf : cb;
  psk_ctx* hi = cf < cb ? cb : cf;
  std::lock_guard<std::mutex> l1(lo->mu);
  std::lock_guard<std::mutex> l2(hi->mu);
  for (psk_ctx* c : {cf, cb}) {
    DeviceGuard dg(c->device);
    c->launch.stream = c->stream;
    c->launch.err = c->d_err;
    c->launch.start();
    cudaMemsetAsync(c->d_err, 0, sizeof(unsigned), c->stream);
  }
  st = m->dtype == PSK_F64 ? ptfs_two_typed<double>(cf, cb, m, alg, sn, mean, cov)
                           : ptfs_two_typed<float>(cf, cb, m, alg, sn, mean, cov);
  unsigned herr[2] = {0, 0};
  cudaError_t e = cudaSuccess;
  int i = 0;
  for (psk_ctx* c : {cf, cb}) {
    DeviceGuard dg(c->device);
    cudaMemcpyAsync(&herr[i++], c->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream);
    ctx_free_all(c);
    const cudaError_t ec = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) e = ec;
  }
  if (st) return st;
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("execution: ") + cuda_msg(e));
  for (psk_ctx* c : {cf, cb}) {  // per-kernel timing of each context
    c->profile.clear();
    if (c->launch.profile && c->launch.evs.size() > 1)
      for (size_t k = 0; k + 1 < c->launch.evs.size(); ++k) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->launch.evs[k], c->launch.evs[k + 1]);
        c->profile.emplace_back(c->launch.names[k], ms);
      }
  }
  const unsigned herr_all = herr[0] | herr[1];
  if (herr_all & kErrNotPD) return fail(PSK_E_NOT_PD, "cholesky pivot");
  if (herr_all & kErrSingular) return fail(PSK_E_SINGULAR, "lu zero pivot");
  return PSK_OK;
}


// ---- multi-device contexts (psk_create_multi) --------------------------------
// One host thread drives G member contexts (one per device entry; repeated
// devices are separate streams of one GPU).  PKF / PRTS shard the time axis
// over the members exactly like distributed.py does over processes -- reduce,
// exchange of the shard elements, fold, finish -- with the exchange done by
// peer copies between the members' devices (cudaMemcpyPeerAsync over NVLink /
// NVSwitch once peer access is enabled; a plain device copy for repeated
// devices) ordered by events, so no member ever waits on the host.  PTFS runs
// the forward filter time-sharded on the first half of the members and the
// backward filter time-sharded on the second half, concurrently; the forward
// filtered stats of each shard are the only per-step data that cross devices
// (kalman_par.hpp:207-238).  Host inputs are copied shard
// by shard by the member that owns the shard (every GPU on its own PCIe
// link).  Results do not depend on G beyond rounding.

inline void peer_enable(int dev, int peer) {
  if (dev == peer) return;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, dev, peer) != cudaSuccess || !can) {
    cudaGetLastError();
    return;
  }
  DeviceGuard dg(dev);
  if (cudaDeviceEnablePeerAccess(peer, 0) != cudaSuccess) cudaGetLastError();
}

inline long long shard_lo(long long t, int g, int G) {
  const long long base = t / G, rem = t % G;
  return g * base + std::min<long long>(g, rem);
}

// steps [lo, lo + n) of a model (pointers advanced by lo steps)
psk_model model_slice(const psk_model* m, long long lo, long long n) {
  psk_model v = *m;
  const size_t es = m->dtype == PSK_F64 ? 8 : 4;
  const long long nx = m->nx, ny = m->ny;
  const void** fp[7] = {&v.f, &v.u, &v.q, &v.h, &v.d, &v.r, &v.y};
  const int64_t st[7] = {m->f_stride, m->u_stride, m->q_stride, m->h_stride,
                         m->d_stride, m->r_stride, m->y_stride};
  const long long blk[7] = {nx * nx, nx, nx * nx, ny * nx, ny, ny * ny, ny};
  for (int i = 0; i < 7; ++i) {
    const long long s = st[i] < 0 ? blk[i] : st[i];
    *fp[i] = static_cast<const char*>(*fp[i]) + (size_t)(lo * s) * es;
  }
  v.t = (uint64_t)n;
  return v;
}

// Stage a shard on member c (device arrays; in place when the inputs already
// live there) and describe it as a device-space psk_model.  `extra`: one more
// step of f/u/q (or of every field with `all`) past the shard.
template <typename S>
int stage_shard(psk_ctx* c, const psk_model* sv, int extra, bool all, psk_model* out) {
  bool foreign = false;
  if (sv->space == PSK_DEVICE) {
    const void* fields[9] = {sv->f, sv->u, sv->q, sv->h, sv->d, sv->r, sv->y, sv->prior_mean,
                             sv->prior_cov};
    for (const void* p : fields) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (at.type == cudaMemoryTypeDevice && at.device != c->device) foreign = true;
    }
  }
  ModelView<S> v;
  const int st = prepare_model<S>(c, sv, v, extra, foreign, all);
  if (st) return st;
  *out = *sv;
  out->space = PSK_DEVICE;
  out->f = v.f; out->u = v.u; out->q = v.q; out->h = v.h; out->d = v.d; out->r = v.r;
  out->y = v.y;
  out->f_stride = v.sf; out->u_stride = v.su; out->q_stride = v.sq; out->h_stride = v.sh;
  out->d_stride = v.sd; out->r_stride = v.sr; out->y_stride = v.sy;
  out->prior_mean = v.m0;
  out->prior_cov = v.p0;
  return PSK_OK;
}

struct MultiEvents {  // one event per member, recorded / waited per exchange
  std::vector<cudaEvent_t> ev;
  explicit MultiEvents(const std::vector<psk_ctx*>& ms) : ev(ms.size(), nullptr) {
    for (size_t i = 0; i < ms.size(); ++i) {
      DeviceGuard dg(ms[i]->device);
      cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    }
  }
  ~MultiEvents() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
};

// gather the packed elements of members `from` (in order) into member c's
// buffer `dst`, after their producers' events
template <typename S>
void gather_elems(psk_ctx* c, S* dst, const std::vector<psk_ctx*>& ms, const std::vector<S*>& el,
                  MultiEvents& evs, const std::vector<int>& from, size_t es) {
  for (size_t k = 0; k < from.size(); ++k) {
    const int i = from[k];
    cudaStreamWaitEvent(c->stream, evs.ev[i], 0);
    cudaMemcpyPeerAsync(dst + k * es, c->device, el[i], ms[i]->device, es * sizeof(S), c->stream);
  }
}

template <typename S>
int multi_typed(psk_ctx* ctx, const psk_model* m, int method, int alg, uint64_t sn, void* mean,
                void* cov) {
  std::vector<psk_ctx*> ms = ctx->members;
  const int nx = m->nx;
  const long long T = (long long)m->t;
  const size_t FS = 3 * nx * nx + 2 * nx, SS = 2 * nx * nx + nx, ST = nx + nx * nx;
  const size_t es = sizeof(S);
  int G = (int)ms.size();
  if (method == 2) G = G / 2 * 2;  // PTFS: two halves
  const int H = method == 2 ? G / 2 : G;  // shards
  if ((long long)H > T) return -1;        // fewer steps than shards: one member runs it
  MultiEvents evs(ms);
  std::vector<psk_model> sm(G);
  std::vector<S*> el(G, nullptr), dm(G, nullptr), dc(G, nullptr), carry(G, nullptr);
  std::vector<long long> lo(G), n(G);
  std::vector<int> flags(G);
  int st = PSK_OK;
  auto shard_of = [&](int g) { return method == 2 ? g % H : g; };
  for (int g = 0; g < G && !st; ++g) {  // stage the shards, allocate
    psk_ctx* c = ms[g];
    DeviceGuard dg(c->device);
    const int i = shard_of(g);
    lo[g] = shard_lo(T, i, H);
    n[g] = shard_lo(T, i + 1, H) - lo[g];
    const bool last = i == H - 1;
    flags[g] = (i == 0 ? PSK_SHARD_FIRST : 0) | (last ? PSK_SHARD_LAST : 0);
    const bool bwd = method == 2 && g >= H;
    if (method != 1 && !bwd) flags[g] |= PSK_SHARD_FILTERED;
    const psk_model sv = model_slice(m, lo[g], n[g]);
    st = stage_shard<S>(c, &sv, last ? 0 : 1, bwd, &sm[g]);
    if (st) break;
    el[g] = static_cast<S*>(ctx_alloc(es * FS * (size_t)std::max(G, 1), c));
    dm[g] = static_cast<S*>(ctx_alloc(es * (size_t)(n[g] * nx), c));
    dc[g] = static_cast<S*>(ctx_alloc(es * (size_t)(n[g] * nx * nx), c));
    carry[g] = static_cast<S*>(ctx_alloc(es * (ST + 16), c));
    if (!el[g] || !dm[g] || !dc[g] || !carry[g]) st = fail(PSK_E_ALLOC, "multi-device scratch");
  }
  auto phase = [&](int g, int ph, const S* cy, const S* fm, const S* fc) {
    psk_ctx* c = ms[g];
    DeviceGuard dg(c->device);
    return shard_typed<S>(c, &sm[g], flags[g], ph, alg, sn, dm[g], dc[g], cy, el[g], fm, fc);
  };
  auto record = [&](int g) {
    DeviceGuard dg(ms[g]->device);
    cudaEventRecord(evs.ev[g], ms[g]->stream);
  };
  // ---- forward filter (members [0, H)): reduce, gather + prefix fold, finish
  for (int g = 0; g < H && !st; ++g) {
    st = phase(g, 0, nullptr, nullptr, nullptr);
    record(g);
  }
  for (int g = 1; g < H && !st; ++g) {
    psk_ctx* c = ms[g];
    DeviceGuard dg(c->device);
    std::vector<int> from;
    for (int i = 0; i < g; ++i) from.push_back(i);
    S* gbuf = static_cast<S*>(ctx_alloc(es * FS * (size_t)g, c));
    if (!gbuf) st = fail(PSK_E_ALLOC, "multi-device gather");
    if (st) break;
    gather_elems<S>(c, gbuf, ms, el, evs, from, FS);
    if (fast_fold<S>(c->launch, 0, nx, gbuf, g, carry[g])) st = fail(PSK_E_ARG, "fold failed");
  }
  for (int g = 0; g < H && !st; ++g) {
    st = phase(g, 1, g > 0 ? carry[g] : nullptr, nullptr, nullptr);
    record(g);
  }
  if (method == 1) {  // ---- RTS smoother: reduce, gather + suffix fold, finish
    for (int g = 0; g < G && !st; ++g) {
      st = phase(g, 2, nullptr, nullptr, nullptr);
      record(g);
    }
    for (int g = 0; g < G - 1 && !st; ++g) {
      psk_ctx* c = ms[g];
      DeviceGuard dg(c->device);
      std::vector<int> from;
      for (int i = g + 1; i < G; ++i) from.push_back(i);
      S* gbuf = static_cast<S*>(ctx_alloc(es * SS * from.size(), c));
      if (!gbuf) st = fail(PSK_E_ALLOC, "multi-device gather");
      if (st) break;
      gather_elems<S>(c, gbuf, ms, el, evs, from, SS);
      if (fast_fold<S>(c->launch, 1, nx, gbuf, (int)from.size(), carry[g]))
        st = fail(PSK_E_ARG, "fold failed");
    }
    for (int g = 0; g < G && !st; ++g)
      st = phase(g, 3, g < G - 1 ? carry[g] : nullptr, nullptr, nullptr);
  } else if (method == 2) {  // ---- backward filter on members [H, 2H)
    for (int g = H; g < G && !st; ++g) {
      st = phase(g, 4, nullptr, nullptr, nullptr);
      record(g);
    }
    for (int g = H; g < G && !st; ++g) {
      psk_ctx* c = ms[g];
      DeviceGuard dg(c->device);
      std::vector<int> from;
      for (int i = g + 1; i < G; ++i) from.push_back(i);
      if (!from.empty()) {
        S* gbuf = static_cast<S*>(ctx_alloc(es * FS * from.size(), c));
        if (!gbuf) st = fail(PSK_E_ALLOC, "multi-device gather");
        if (st) break;
        gather_elems<S>(c, gbuf, ms, el, evs, from, FS);
        if (fast_fold<S>(c->launch, 2, nx, gbuf, (int)from.size(), carry[g]))
          st = fail(PSK_E_ARG, "fold failed");
      }
      // the forward half's filtered stats of this shard
      const int f = g - H;
      S* fm = static_cast<S*>(ctx_alloc(es * (size_t)(n[g] * nx), c));
      S* fc = static_cast<S*>(ctx_alloc(es * (size_t)(n[g] * nx * nx), c));
      if (!fm || !fc) st = fail(PSK_E_ALLOC, "multi-device forward states");
      if (st) break;
      cudaStreamWaitEvent(c->stream, evs.ev[f], 0);
      cudaMemcpyPeerAsync(fm, c->device, dm[f], ms[f]->device, es * (size_t)(n[g] * nx),
                          c->stream);
      cudaMemcpyPeerAsync(fc, c->device, dc[f], ms[f]->device, es * (size_t)(n[g] * nx * nx),
                          c->stream);
      c->launch.count("ptfs_forward_states_peer_copy");
      st = phase(g, 5, from.empty() ? nullptr : carry[g], fm, fc);
    }
  }
  // ---- outputs: every shard's stats into the caller's buffer (any memory)
  const int o0 = method == 2 ? H : 0;
  for (int g = o0; g < o0 + H && !st; ++g) {
    psk_ctx* c = ms[g];
    DeviceGuard dg(c->device);
    cudaMemcpyAsync(static_cast<char*>(mean) + es * (size_t)(lo[g] * nx), dm[g],
                    es * (size_t)(n[g] * nx), cudaMemcpyDefault, c->stream);
    cudaMemcpyAsync(static_cast<char*>(cov) + es * (size_t)(lo[g] * nx * nx), dc[g],
                    es * (size_t)(n[g] * nx * nx), cudaMemcpyDefault, c->stream);
  }
  return st;
}

int multi_entry(psk_ctx* ctx, const psk_model* m, int method, int alg, uint64_t sn, void* mean,
                void* cov) {
  if (!m) return fail(PSK_E_ARG, "null model");
  if (m->nx < 1 || m->nx > 16 || m->ny < 1 || m->ny > 16) return fail(PSK_E_DIM, "mat dims");
  if (m->dtype != PSK_F32 && m->dtype != PSK_F64) return fail(PSK_E_ARG, "bad dtype");
  if (m->space != PSK_HOST && m->space != PSK_DEVICE) return fail(PSK_E_ARG, "bad space");
  int st = check_contract(alg, sn, m->t);
  if (st) return st;
  if (m->t > 0 && (!mean || !cov)) return fail(PSK_E_ARG, "null output");
  std::vector<psk_ctx*> ms = ctx->members;
  const bool fast = ctx->mode == PSK_MODE_FAST &&
                    (m->dtype == PSK_F64 ? fast_supported<double>(m->nx, m->ny)
                                         : fast_supported<float>(m->nx, m->ny));
  const int G = (int)ms.size();
  if (!fast || G < 2 || (method == 2 && G < 2) || m->t < 2) {
    // a single member runs it (dims without shard phases, exact mode, tiny
    // series): the numbers do not depend on the placement
    if (method == 2) return psk_ptfs(ms[0], ms[0], 1, m, alg, sn, mean, cov);
    return run_entry(ms[0], m, method, alg, sn, mean, cov);
  }
  std::lock_guard<std::mutex> lk0(ctx->mu);
  std::vector<psk_ctx*> order = ms;  // lock members in address order
  std::sort(order.begin(), order.end());
  order.erase(std::unique(order.begin(), order.end()), order.end());
  std::vector<std::unique_lock<std::mutex>> locks;
  for (psk_ctx* c : order) locks.emplace_back(c->mu);
  for (psk_ctx* c : order) {
    DeviceGuard dg(c->device);
    c->launch.stream = c->stream;
    c->launch.err = c->d_err;
    c->launch.start();
    cudaMemsetAsync(c->d_err, 0, sizeof(unsigned), c->stream);
  }
  st = m->dtype == PSK_F64 ? multi_typed<double>(ctx, m, method, alg, sn, mean, cov)
                           : multi_typed<float>(ctx, m, method, alg, sn, mean, cov);
  if (st == -1) {  // fewer steps than shards
    locks.clear();
    if (method == 2) return psk_ptfs(ms[0], ms[0], 1, m, alg, sn, mean, cov);
    return run_entry(ms[0], m, method, alg, sn, mean, cov);
  }
  unsigned herr_all = 0;
  cudaError_t e = cudaSuccess;
  long long launches = 0;
  std::vector<unsigned> herr(order.size(), 0);
  for (size_t i = 0; i < order.size(); ++i) {
    psk_ctx* c = order[i];
    DeviceGuard dg(c->device);
    cudaMemcpyAsync(&herr[i], c->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream);
    ctx_free_all(c);
  }
  for (size_t i = 0; i < order.size(); ++i) {
    psk_ctx* c = order[i];
    DeviceGuard dg(c->device);
    const cudaError_t ec = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) e = ec;
    herr_all |= herr[i];
    launches += c->launch.launches;
  }
  ctx->launch.launches = launches;
  if (st) return st;
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("execution: ") + cuda_msg(e));
  if (herr_all & kErrNotPD) return fail(PSK_E_NOT_PD, "cholesky pivot");
  if (herr_all & kErrSingular) return fail(PSK_E_SINGULAR, "lu zero pivot");
  return PSK_OK;
}

// A batch on a multi-device context: contiguous shares of the series per
// member (BASELINE configs[4] batch sharding, no exchange), all members
// queued before any waits.
int multi_batch_entry(psk_ctx* ctx, const psk_model* ms_, int count, int method, int alg,
                      uint64_t sn, void* const* means, void* const* covs) {
  std::vector<psk_ctx*> ms = ctx->members;
  const int G = (int)ms.size();
  std::vector<int> was(G);
  int st = PSK_OK;
  for (int g = 0; g < G && !st; ++g) {
    const long long a = shard_lo(count, g, G), b = shard_lo(count, g + 1, G);
    if (b == a) continue;
    was[g] = ms[g]->async;
    ms[g]->async = 1;
    st = batch_entry(ms[g], ms_ + a, (int)(b - a), method, alg, sn, means + a, covs + a);
    ms[g]->async = was[g];
  }
  int st2 = PSK_OK;
  for (int g = 0; g < G; ++g) {
    const int s2 = psk_sync(ms[g]);
    if (!st2) st2 = s2;
  }
  return st ? st : st2;
}
}  // namespace

extern "C" {

int psk_create(psk_ctx** out, int device) {
  if (!out) return fail(PSK_E_ARG, "null ctx out");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(PSK_E_CUDA, std::string("no CUDA device: ") + cuda_msg(e));
  if (device < 0 || device >= n) return fail(PSK_E_ARG, "device index out of range");
  auto* c = new psk_ctx;
  c->device = device;
  DeviceGuard dg(device);
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&c->d_err, sizeof(unsigned)) != cudaSuccess) {
    delete c;
    return fail(PSK_E_CUDA, "context setup failed");
  }
  c->stream = c->own_stream;
  // keep freed scratch in the pool between calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return PSK_OK;
}

int psk_create_multi(psk_ctx** out, const int* devices, int ndev) {
  if (!out) return fail(PSK_E_ARG, "null ctx out");
  *out = nullptr;
  if (!devices || ndev < 1 || ndev > 64) return fail(PSK_E_ARG, "devices: 1..64 entries");
  std::vector<psk_ctx*> ms;
  for (int i = 0; i < ndev; ++i) {
    psk_ctx* c = nullptr;
    const int st = psk_create(&c, devices[i]);
    if (st) {
      for (psk_ctx* x : ms) psk_destroy(x);
      return st;
    }
    ms.push_back(c);
  }
  for (int i = 0; i < ndev; ++i)  // NVLink P2P between every pair of members
    for (int j = 0; j < ndev; ++j) peer_enable(devices[i], devices[j]);
  auto* c = new psk_ctx;
  c->device = devices[0];
  c->own_stream = nullptr;
  c->stream = ms[0]->stream;
  c->d_err = nullptr;
  c->members = std::move(ms);
  *out = c;
  return PSK_OK;
}

int psk_destroy(psk_ctx* c) {
  if (!c) return PSK_OK;
  if (!c->members.empty()) {
    for (psk_ctx* m : c->members) psk_destroy(m);
    delete c;
    return PSK_OK;
  }
  {
    DeviceGuard dg(c->device);
    ctx_free_persist(c);
    if (c->shard_scratch) {
      if (c->shard_dtype == PSK_F64) fast_shard_release<double>(c->shard_scratch);
      else fast_shard_release<float>(c->shard_scratch);
    }
    cudaStreamSynchronize(c->stream);
    c->launch.start();  // releases events
    for (auto s : c->sub) cudaStreamDestroy(s);
    for (auto e : c->sub_ev) cudaEventDestroy(e);
    cudaFree(c->d_err);
    if (c->launch.dlb_trace) cudaFree(c->launch.dlb_trace);
    cudaStreamDestroy(c->own_stream);
  }
  delete c;
  return PSK_OK;
}

int psk_set_mode(psk_ctx* c, int mode) {
  if (!c) return fail(PSK_E_ARG, "null context");
  if (mode != PSK_MODE_FAST && mode != PSK_MODE_EXACT) return fail(PSK_E_ARG, "bad mode");
  c->mode = mode;
  for (psk_ctx* m : c->members) m->mode = mode;
  return PSK_OK;
}

int psk_set_chunk(psk_ctx* c, int chunk) {
  if (!c) return fail(PSK_E_ARG, "null context");
  if (chunk < 0) return fail(PSK_E_ARG, "chunk must be >= 1 (or 0 = auto)");
  c->chunk = chunk;
  for (psk_ctx* m : c->members) m->chunk = chunk;
  return PSK_OK;
}

int psk_set_option(psk_ctx* c, const char* key, int64_t value) {
  if (!c || !key) return fail(PSK_E_ARG, "null context or key");
  if (!c->members.empty()) {  // a multi-device context: every member
    const std::string k(key);
    if (k == "async" || k == "shard_async")
      return fail(PSK_E_ARG, "multi-device calls are synchronous");
    for (psk_ctx* m : c->members) {
      const int st = psk_set_option(m, key, value);
      if (st) return st;
    }
    if (k == "chunk") c->chunk = value;
    return PSK_OK;
  }
  const std::string k(key);
  if (k == "chunk") {
    if (value < 0) return fail(PSK_E_ARG, "chunk must be >= 1 (or 0 = auto)");
    c->chunk = value;
  } else if (k == "async") {
    if (value != 0 && value != 1) return fail(PSK_E_ARG, "async must be 0 or 1");
    c->async = (int)value;
  } else if (k == "shard_async") {
    if (value != 0 && value != 1) return fail(PSK_E_ARG, "shard_async must be 0 or 1");
    c->shard_async = (int)value;
  } else if (k == "batch_streams") {
    if (value < 1 || value > 64) return fail(PSK_E_ARG, "batch_streams must be 1..64");
    c->batch_streams = (int)value;
  } else if (k == "dlb_trace") {
    // diagnostics: per-phase stamps of every DLB scan of this context are
    // appended to $PSK_DLB_TRACE (default dlb_trace.bin); synchronises
    if (value != 0 && value != 1) return fail(PSK_E_ARG, "dlb_trace must be 0 or 1");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    if (value && !c->launch.dlb_trace) {
      const long long cap = 65536;
      if (cudaMalloc(&c->launch.dlb_trace, sizeof(unsigned long long) * 8 * cap) != cudaSuccess)
        return fail(PSK_E_ALLOC, "trace buffer");
      c->launch.dlb_trace_cap = cap;
      const char* path = std::getenv("PSK_DLB_TRACE");
      c->launch.dlb_trace_path = path ? path : "dlb_trace.bin";
    } else if (!value && c->launch.dlb_trace) {
      cudaStreamSynchronize(c->stream);
      cudaFree(c->launch.dlb_trace);
      c->launch.dlb_trace = nullptr;
      c->launch.dlb_trace_cap = 0;
    }
  } else if (k == "tile") {
    if (value != 0 && value != 1) return fail(PSK_E_ARG, "tile must be 0 or 1");
    c->tile = (int)value;
  } else if (k == "waves") {
    if (value < 1 || value > 1024) return fail(PSK_E_ARG, "waves must be 1..1024");
    c->waves = (int)value;
  } else {
    return fail(PSK_E_ARG, "unknown option " + k);
  }
  return PSK_OK;
}

int psk_sync(psk_ctx* c) {
  if (!c) return fail(PSK_E_ARG, "null context");
  if (!c->members.empty()) {
    int st = PSK_OK;
    for (psk_ctx* m : c->members) {
      const int s2 = psk_sync(m);
      if (!st) st = s2;
    }
    return st;
  }
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  unsigned herr = 0;
  cudaMemcpyAsync(&herr, c->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream);
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  cudaMemsetAsync(c->d_err, 0, sizeof(unsigned), c->stream);
  // per-kernel spans of every call since the last synchronisation
  c->profile.clear();
  auto drain = [&](std::vector<cudaEvent_t>& evs, std::vector<const char*>& names) {
    for (size_t i = 0; i + 1 < evs.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, evs[i], evs[i + 1]);
      c->profile.emplace_back(names[i], ms);
    }
    for (auto ev : evs) cudaEventDestroy(ev);
    evs.clear();
    names.clear();
  };
  for (auto& p : c->launch.pending) drain(p.first, p.second);
  c->launch.pending.clear();
  drain(c->launch.evs, c->launch.names);
  if (e != cudaSuccess) return fail(PSK_E_CUDA, std::string("execution: ") + cuda_msg(e));
  if (herr & kErrNotPD) return fail(PSK_E_NOT_PD, "cholesky pivot");
  if (herr & kErrSingular) return fail(PSK_E_SINGULAR, "lu zero pivot");
  return PSK_OK;
}

int psk_set_stream(psk_ctx* c, void* stream) {
  if (!c) return fail(PSK_E_ARG, "null context");
  if (!c->members.empty()) return fail(PSK_E_ARG, "a multi-device context runs on its members' streams");
  c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
  return PSK_OK;
}

int psk_get_stream(psk_ctx* c, void** stream) {
  if (!c || !stream) return fail(PSK_E_ARG, "null context or stream out");
  *stream = static_cast<void*>(c->stream);
  return PSK_OK;
}

int psk_set_profile(psk_ctx* c, int enable) {
  if (!c) return fail(PSK_E_ARG, "null context");
  c->launch.profile = enable != 0;
  return PSK_OK;
}

int psk_last_profile(psk_ctx* c, const char** names, float* ms, int cap) {
  if (!c) return fail(PSK_E_ARG, "null context");
  const int n = (int)c->profile.size();
  for (int i = 0; i < n && i < cap; ++i) {
    if (names) names[i] = c->profile[i].first;
    if (ms) ms[i] = c->profile[i].second;
  }
  return n;
}

int64_t psk_last_launch_count(psk_ctx* c) { return c ? c->launch.launches : -1; }

int psk_pkf(psk_ctx* c, const psk_model* m, int alg, uint64_t sn, void* mean, void* cov) {
  if (c && !c->members.empty()) return multi_entry(c, m, 0, alg, sn, mean, cov);
  return run_entry(c, m, 0, alg, sn, mean, cov);
}
int psk_prts(psk_ctx* c, const psk_model* m, int alg, uint64_t sn, void* mean, void* cov) {
  if (c && !c->members.empty()) return multi_entry(c, m, 1, alg, sn, mean, cov);
  return run_entry(c, m, 1, alg, sn, mean, cov);
}
int psk_ptfs(psk_ctx* cf, psk_ctx* cb, int devices, const psk_model* m, int alg, uint64_t sn,
             void* mean, void* cov) {
  if (cf && !cf->members.empty()) {
    // a multi-device forward context: the two filters on its member halves
    // (devices = 1 keeps the whole smoother on the first member)
    if (devices == 1) return psk_ptfs(cf->members[0], cf->members[0], 1, m, alg, sn, mean, cov);
    return multi_entry(cf, m, 2, alg, sn, mean, cov);
  }
  if (cb && !cb->members.empty()) return fail(PSK_E_ARG, "multi-device backward context");
  if (devices != 1 && devices != 2) return fail(PSK_E_ARG, "devices must be 1 or 2");
  if (!cb) cb = cf;
  // devices == 2 with a second context: forward filter on ctx_fwd and the
  // backward reduce + scan on ctx_bwd, concurrently.
  // Anything the split does not cover runs on the forward context alone; the
  // numbers do not depend on the placement (test_kalman_par.cpp:209-227).
  if (devices == 2 && cb != cf && m && cf && cf->mode == PSK_MODE_FAST &&
      cb->mode == PSK_MODE_FAST && m->t > 0 &&
      (m->dtype == PSK_F64 ? fast_supported<double>(m->nx, m->ny)
                           : fast_supported<float>(m->nx, m->ny)))
    return ptfs_two(cf, cb, m, alg, sn, mean, cov);
  return run_entry(cf, m, 2, alg, sn, mean, cov);
}

int psk_shard_filter_reduce(psk_ctx* c, const psk_model* m, int flags, int alg, uint64_t sn,
                            void* elem_out) {
  // mean/cov are not touched by a reduce; pass the element buffer to pass
  // the null checks
  return shard_entry(c, m, flags, 0, alg, sn, elem_out, elem_out, nullptr, elem_out);
}
int psk_shard_filter_finish(psk_ctx* c, const psk_model* m, int flags, const void* carry,
                            void* mean, void* cov) {
  return shard_entry(c, m, flags, 1, 0, 1, mean, cov, carry, nullptr);
}
int psk_shard_smoother_reduce(psk_ctx* c, const psk_model* m, int flags, int alg, uint64_t sn,
                              const void* mean, const void* cov, void* elem_out) {
  return shard_entry(c, m, flags, 2, alg, sn, const_cast<void*>(mean), const_cast<void*>(cov),
                     nullptr, elem_out);
}
int psk_shard_smoother_finish(psk_ctx* c, const psk_model* m, int flags, const void* carry,
                              void* mean, void* cov) {
  return shard_entry(c, m, flags, 3, 0, 1, mean, cov, carry, nullptr);
}
int psk_shard_backward_reduce(psk_ctx* c, const psk_model* m, int flags, int alg, uint64_t sn,
                              void* elem_out) {
  return shard_entry(c, m, flags, 4, alg, sn, elem_out, elem_out, nullptr, elem_out);
}
int psk_shard_backward_finish(psk_ctx* c, const psk_model* m, int flags, const void* carry,
                              const void* fmean, const void* fcov, void* mean, void* cov) {
  return shard_entry(c, m, flags, 5, 0, 1, mean, cov, carry, nullptr, fmean, fcov);
}
int psk_fold_backward(psk_ctx* c, int dtype, int nx, const void* elems, int count, void* out) {
  return fold_entry(c, 2, dtype, nx, elems, count, out);
}
int psk_fold_filter(psk_ctx* c, int dtype, int nx, const void* elems, int count, void* out) {
  return fold_entry(c, 0, dtype, nx, elems, count, out);
}
int psk_fold_smoother(psk_ctx* c, int dtype, int nx, const void* elems, int count, void* out) {
  return fold_entry(c, 1, dtype, nx, elems, count, out);
}

int psk_pkf_batch(psk_ctx* c, const psk_model* ms, int count, int alg, uint64_t sn,
                  void* const* means, void* const* covs) {
  if (c && !c->members.empty()) return multi_batch_entry(c, ms, count, 0, alg, sn, means, covs);
  return batch_entry(c, ms, count, 0, alg, sn, means, covs);
}
int psk_prts_batch(psk_ctx* c, const psk_model* ms, int count, int alg, uint64_t sn,
                   void* const* means, void* const* covs) {
  if (c && !c->members.empty()) return multi_batch_entry(c, ms, count, 1, alg, sn, means, covs);
  return batch_entry(c, ms, count, 1, alg, sn, means, covs);
}

int psk_num_devices(psk_ctx* c) {
  if (!c) return fail(PSK_E_ARG, "null context");
  return c->members.empty() ? 1 : (int)c->members.size();
}

int psk_host_alloc(void** p, size_t bytes) {
  if (!p) return fail(PSK_E_ARG, "null pointer out");
  *p = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(PSK_E_CUDA, std::string("no CUDA device: ") + cuda_msg(e));
  if (bytes == 0) return PSK_OK;
  e = cudaHostAlloc(p, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(PSK_E_ALLOC, std::string("pinned host allocation: ") + cuda_msg(e));
  }
  return PSK_OK;
}

int psk_host_free(void* p) {
  if (!p) return PSK_OK;
  const cudaError_t e = cudaFreeHost(p);
  return e == cudaSuccess ? PSK_OK : fail(PSK_E_CUDA, std::string("cudaFreeHost: ") + cuda_msg(e));
}

const char* psk_last_error(void) { return g_last_error.c_str(); }
const char* psk_version(void) { return "psk-b200 0.1.0 (sm_100a)"; }

}  // extern "C"
