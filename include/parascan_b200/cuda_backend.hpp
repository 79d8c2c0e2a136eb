// cuda_backend.hpp -- drop-in C++ shim over the psk C-ABI for callers of the
// reference library (parascan).  Include it after (or instead of) the
// reference's kalman_par.hpp; then
//
//     parascan::CudaBackend be(/*device=*/0);
//     auto sm = parascan::prts_run(model, ys, parascan::ScanSpec{alg, n}, be);
//
// resolves to the overloads below (exact match on CudaBackend& beats the
// reference templates' derived-to-base conversion to Backend&), so call sites
// only swap the backend object.  Replaces, with unchanged signatures:
//   pkf_run   kalman_par.hpp:111-119
//   prts_run  kalman_par.hpp:156-179
//   ptfs_run  kalman_par.hpp:207-238
// Status codes map back onto the reference exception types (mat.hpp:21-32,
// scan.hpp:28-30).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include "parascan/backend.hpp"
#include "parascan/lgssm.hpp"
#include "parascan/mat.hpp"
#include "parascan/scan.hpp"
#include "psk.h"
#include "parascan_b200/host_parallel.hpp"

namespace parascan {

// ScanAlg value of the new single-pass decoupled look-back scan (appended
// after SenguptaB so the reference's values and names stay stable).
inline constexpr ScanAlg kDecoupledLookback = static_cast<ScanAlg>(PSK_DECOUPLED_LOOKBACK);

namespace psk_detail {
[[noreturn]] inline void throw_status(int st) {
  const std::string msg = psk_last_error();
  switch (st) {
    case PSK_E_DIM: throw DimensionMismatch(msg);
    case PSK_E_CONTRACT: throw ContractViolation(msg);
    case PSK_E_NOT_PD: throw NotPositiveDefinite(msg);
    case PSK_E_SINGULAR: throw SingularMatrix(msg);
    case PSK_E_ALLOC: throw std::bad_alloc();
    default: throw std::runtime_error("psk: " + msg);
  }
}
inline void check(int st) {
  if (st != PSK_OK) throw_status(st);
}
}  // namespace psk_detail

namespace psk_detail {

// ---- host marshalling ------------------------------
// The reference containers are per-step heap objects (lgssm.hpp:29-45,
// GaussianStats lgssm.hpp:18-21): packing them into the C-ABI's per-field
// arrays and building the output vector are memory-bound host loops that the
// reference runs on one thread (probe: 5.7 s pack + 1.8 s unpack at 2^22).
// Here both are split over the host cores by step range, and the packed
// inputs / raw outputs live in PINNED buffers owned by the backend (reused
// across calls), so the device copies run at full PCIe speed.

// A growable pinned host buffer (psk_host_alloc); contents are scratch.
class Pinned {
 public:
  Pinned() = default;
  ~Pinned() { psk_host_free(p_); }
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
  void* reserve(std::size_t bytes) {
    if (bytes > cap_) {
      psk_host_free(p_);
      p_ = nullptr;
      cap_ = 0;
      check(psk_host_alloc(&p_, bytes));
      cap_ = bytes;
    }
    return p_;
  }

 private:
  void* p_ = nullptr;
  std::size_t cap_ = 0;
};

}  // namespace psk_detail

// The Backend& executor slot (backend.hpp:39-44) filled by a psk context on
// one CUDA device.  Host closures cannot run on the device, so run() throws.
// The backend also owns the pinned staging of the marshalling layer.
class CudaBackend final : public Backend {
 public:
  explicit CudaBackend(int device = 0, int mode = PSK_MODE_FAST, int chunk = 0) {
    psk_detail::check(psk_create(&ctx_, device));
    psk_detail::check(psk_set_mode(ctx_, mode));
    psk_detail::check(psk_set_chunk(ctx_, chunk));
  }
  // several GPUs (psk_create_multi): pkf_run / prts_run shard the time axis
  // over them, ptfs_run(m, ys, spec, be, be, devices > 1) runs the forward and
  // backward filters on the two halves, each time-sharded
  explicit CudaBackend(const std::vector<int>& devices, int mode = PSK_MODE_FAST,
                       int chunk = 0) {
    psk_detail::check(psk_create_multi(&ctx_, devices.data(), int(devices.size())));
    psk_detail::check(psk_set_mode(ctx_, mode));
    psk_detail::check(psk_set_chunk(ctx_, chunk));
  }
  int devices() const { return psk_num_devices(ctx_); }
  ~CudaBackend() override { psk_destroy(ctx_); }
  CudaBackend(const CudaBackend&) = delete;
  CudaBackend& operator=(const CudaBackend&) = delete;

  void run(const Launch&) override {
    throw ContractViolation("CudaBackend runs only the parallel Kalman drivers");
  }
  unsigned workers() const override { return 1; }
  psk_ctx* ctx() const { return ctx_; }
  psk_detail::Pinned& staging_in() { return in_; }
  psk_detail::Pinned& staging_out() { return out_; }

 private:
  psk_ctx* ctx_ = nullptr;
  psk_detail::Pinned in_, out_;
};

namespace psk_detail {

template <typename S>
constexpr int dtype_of() {
  static_assert(std::is_same_v<S, float> || std::is_same_v<S, double>,
                "the CUDA path supports float and double");
  return std::is_same_v<S, double> ? PSK_F64 : PSK_F32;
}

// shape checks of one step's block: the reference's mat_mul / mat_add reject
// mismatched operands with DimensionMismatch (mat.hpp:61-63); the packer
// memcpys raw blocks, so it checks every block before reading it
template <typename S>
inline bool block_dims_ok(const Mat<S>& a, std::size_t r, std::size_t c) {
  return std::size_t(a.rows()) == r && std::size_t(a.cols()) == c;
}
template <typename S>
inline bool block_dims_ok(const Vec<S>& a, std::size_t r, std::size_t) {
  return std::size_t(a.len()) == r;
}

// scalars of the packed per-field arrays of a model (16-byte aligned fields)
template <typename S>
std::size_t packed_size(const Lgssm<S>& m) {
  const std::size_t nx = std::size_t(m.nx), ny = std::size_t(m.ny), t = m.t;
  const std::size_t blk[9] = {nx * nx, nx, nx * nx, ny * nx, ny, ny * ny, ny, nx, nx * nx};
  const std::size_t align = 16 / sizeof(S);
  std::size_t total = 0;
  for (int i = 0; i < 9; ++i) {
    const std::size_t n = i < 7 ? blk[i] * t : blk[i];
    total += (n + align - 1) / align * align;
  }
  return total;
}

// Lgssm<S> (per-step std::vector<Mat>) -> per-field dense arrays at `base`
// (packed_size(m) scalars; one field after another, 16-byte aligned)
template <typename S>
psk_model pack_into(const Lgssm<S>& m, const Measurements<S>& ys, S* base) {
  const std::size_t nx = std::size_t(m.nx), ny = std::size_t(m.ny), t = m.t;
  if (m.f.size() != t || m.u.size() != t || m.q.size() != t || m.h.size() != t ||
      m.d.size() != t || m.r.size() != t || ys.size() != t)
    throw DimensionMismatch("model / measurement length");
  if (!block_dims_ok(m.prior_mean, nx, 1) || !block_dims_ok(m.prior_cov, nx, nx))
    throw DimensionMismatch("prior dims");
  const std::size_t blk[9] = {nx * nx, nx, nx * nx, ny * nx, ny, ny * ny, ny, nx, nx * nx};
  std::size_t off[9], total = 0;
  const std::size_t align = 16 / sizeof(S);
  for (int i = 0; i < 9; ++i) {
    off[i] = total;
    const std::size_t n = i < 7 ? blk[i] * t : blk[i];
    total += (n + align - 1) / align * align;
  }
  parallel_for(t, 1 << 14, [&](std::size_t lo, std::size_t hi) {
    auto put = [&](int i, const auto& src, std::size_t r, std::size_t c) {
      S* dst = base + off[i];
      const std::size_t b = blk[i];
      for (std::size_t k = lo; k < hi; ++k) {
        if (!block_dims_ok(src[k], r, c))
          throw DimensionMismatch("step " + std::to_string(k) + ": block dims");
        std::memcpy(dst + k * b, src[k].view().d, sizeof(S) * b);
      }
    };
    put(0, m.f, nx, nx);
    put(1, m.u, nx, 1);
    put(2, m.q, nx, nx);
    put(3, m.h, ny, nx);
    put(4, m.d, ny, 1);
    put(5, m.r, ny, ny);
    put(6, ys, ny, 1);
  });
  std::memcpy(base + off[7], m.prior_mean.view().d, sizeof(S) * nx);
  std::memcpy(base + off[8], m.prior_cov.view().d, sizeof(S) * nx * nx);
  psk_model md{};
  md.t = t;
  md.nx = m.nx;
  md.ny = m.ny;
  md.dtype = dtype_of<S>();
  md.space = PSK_HOST;
  const void** fp[7] = {&md.f, &md.u, &md.q, &md.h, &md.d, &md.r, &md.y};
  for (int i = 0; i < 7; ++i) *fp[i] = base + off[i];
  md.f_stride = md.u_stride = md.q_stride = md.h_stride = md.d_stride =
      md.r_stride = md.y_stride = -1;
  md.prior_mean = base + off[7];
  md.prior_cov = base + off[8];
  return md;
}

// the same into the backend's pinned input buffer
template <typename S>
psk_model pack(const Lgssm<S>& m, const Measurements<S>& ys, Pinned& buf) {
  return pack_into(m, ys, static_cast<S*>(buf.reserve(sizeof(S) * (packed_size(m) + 1))));
}

// The output vector<GaussianStats<S>> of t steps with every step's Vec / Mat
// allocated (by the worker that will fill it: first-touch locality).  The
// per-step heap objects are the reference's return type (lgssm.hpp:18-21);
// allocating 2 t of them is the single largest host cost of a drop-in call,
// so call() builds them on a separate thread while it packs the inputs and
// the device runs.
template <typename S>
std::vector<GaussianStats<S>> alloc_stats(std::size_t t, int nx) {
  std::vector<GaussianStats<S>> out(t);
  parallel_for(t, 1 << 13, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t k = lo; k < hi; ++k) {
      out[k].mean = Vec<S>(nx);
      out[k].cov = Mat<S>(nx, nx);
    }
  });
  return out;
}
// raw outputs mean[T][nx], cov[T][nx][nx] -> the allocated per-step objects
template <typename S>
void fill_stats(std::vector<GaussianStats<S>>& out, const S* mean, const S* cov, int nx) {
  const std::size_t n = std::size_t(nx);
  parallel_for(out.size(), 1 << 13, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t k = lo; k < hi; ++k) {
      std::memcpy(out[k].mean.view().d, mean + k * n, sizeof(S) * n);
      std::memcpy(out[k].cov.data(), cov + k * n * n, sizeof(S) * n * n);
    }
  });
}
template <typename S>
std::vector<GaussianStats<S>> unpack(const S* mean, const S* cov, std::size_t t, int nx) {
  std::vector<GaussianStats<S>> out = alloc_stats<S>(t, nx);
  fill_stats(out, mean, cov, nx);
  return out;
}

inline void check_dims(int nx, int ny) {
  if (nx < 1 || nx > kMaxDim || ny < 1 || ny > kMaxDim) throw DimensionMismatch("mat dims");
}

// vector<GaussianStats> outputs: raw results land in the pinned output buffer
// The output objects are allocated on a helper thread while this thread
// packs the inputs and the device computes (pack -> H2D -> kernels -> D2H);
// only the copy into them remains after the call.
template <typename S, class F>
std::vector<GaussianStats<S>> call(const Lgssm<S>& m, const Measurements<S>& ys,
                                   CudaBackend& be, F&& f) {
  check_dims(m.nx, m.ny);
  std::vector<GaussianStats<S>> out;
  std::thread alloc([&] { out = alloc_stats<S>(m.t, m.nx); });
  struct Join {
    std::thread& th;
    ~Join() {
      if (th.joinable()) th.join();
    }
  } join{alloc};
  const psk_model md = pack(m, ys, be.staging_in());
  const std::size_t nm = m.t * std::size_t(m.nx), nc = nm * std::size_t(m.nx);
  const std::size_t mb = (sizeof(S) * nm + 15) / 16 * 16;
  char* o = static_cast<char*>(be.staging_out().reserve(mb + sizeof(S) * nc + 16));
  S* mean = reinterpret_cast<S*>(o);
  S* cov = reinterpret_cast<S*>(o + mb);
  check(f(md, mean, cov));
  alloc.join();
  fill_stats(out, mean, cov, m.nx);
  return out;
}

// caller-owned SoA outputs (mean[T][nx], cov[T][nx][nx], host memory)
template <typename S, class F>
void call_into(const Lgssm<S>& m, const Measurements<S>& ys, CudaBackend& be, S* mean, S* cov,
               F&& f) {
  check_dims(m.nx, m.ny);
  const psk_model md = pack(m, ys, be.staging_in());
  check(f(md, mean, cov));
}

}  // namespace psk_detail

// PKF, Alg. 5 (kalman_par.hpp:111-119)
template <typename S>
std::vector<GaussianStats<S>> pkf_run(const Lgssm<S>& m, const Measurements<S>& ys,
                                      const ScanSpec& spec, CudaBackend& be) {
  return psk_detail::call(m, ys, be, [&](const psk_model& md, S* mean, S* cov) {
    return psk_pkf(be.ctx(), &md, int(spec.alg), spec.sengupta_n, mean, cov);
  });
}

// PRTS, Alg. 6 (kalman_par.hpp:156-179)
template <typename S>
std::vector<GaussianStats<S>> prts_run(const Lgssm<S>& m, const Measurements<S>& ys,
                                       const ScanSpec& spec, CudaBackend& be) {
  return psk_detail::call(m, ys, be, [&](const psk_model& md, S* mean, S* cov) {
    return psk_prts(be.ctx(), &md, int(spec.alg), spec.sengupta_n, mean, cov);
  });
}

// PTFS, Alg. 7 (kalman_par.hpp:207-238)
template <typename S>
std::vector<GaussianStats<S>> ptfs_run(const Lgssm<S>& m, const Measurements<S>& ys,
                                       const ScanSpec& spec, CudaBackend& be_fwd,
                                       CudaBackend& be_bwd, int devices = 1) {
  return psk_detail::call(m, ys, be_fwd, [&](const psk_model& md, S* mean, S* cov) {
    return psk_ptfs(be_fwd.ctx(), be_bwd.ctx(), devices, &md, int(spec.alg),
                    spec.sengupta_n, mean, cov);
  });
}

// SoA-output overloads (no reference counterpart):
// the smoothed / filtered stats go straight into caller-owned host arrays
// mean[T][nx] and cov[T][nx][nx] (pinned memory copies at full speed) --
// no per-step heap objects are built.
template <typename S>
void pkf_run(const Lgssm<S>& m, const Measurements<S>& ys, const ScanSpec& spec,
             CudaBackend& be, S* mean, S* cov) {
  psk_detail::call_into(m, ys, be, mean, cov, [&](const psk_model& md, S* mo, S* co) {
    return psk_pkf(be.ctx(), &md, int(spec.alg), spec.sengupta_n, mo, co);
  });
}
template <typename S>
void prts_run(const Lgssm<S>& m, const Measurements<S>& ys, const ScanSpec& spec,
              CudaBackend& be, S* mean, S* cov) {
  psk_detail::call_into(m, ys, be, mean, cov, [&](const psk_model& md, S* mo, S* co) {
    return psk_prts(be.ctx(), &md, int(spec.alg), spec.sengupta_n, mo, co);
  });
}
template <typename S>
void ptfs_run(const Lgssm<S>& m, const Measurements<S>& ys, const ScanSpec& spec,
              CudaBackend& be_fwd, CudaBackend& be_bwd, int devices, S* mean, S* cov) {
  psk_detail::call_into(m, ys, be_fwd, mean, cov, [&](const psk_model& md, S* mo, S* co) {
    return psk_ptfs(be_fwd.ctx(), be_bwd.ctx(), devices, &md, int(spec.alg), spec.sengupta_n,
                    mo, co);
  });
}

}  // namespace parascan
