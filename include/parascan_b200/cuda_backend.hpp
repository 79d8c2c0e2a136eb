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

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "parascan/backend.hpp"
#include "parascan/lgssm.hpp"
#include "parascan/mat.hpp"
#include "parascan/scan.hpp"
#include "psk.h"

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

// The Backend& executor slot (backend.hpp:39-44) filled by a psk context on
// one CUDA device.  Host closures cannot run on the device, so run() throws.
class CudaBackend final : public Backend {
 public:
  explicit CudaBackend(int device = 0, int mode = PSK_MODE_FAST, int chunk = 0) {
    psk_detail::check(psk_create(&ctx_, device));
    psk_detail::check(psk_set_mode(ctx_, mode));
    psk_detail::check(psk_set_chunk(ctx_, chunk));
  }
  ~CudaBackend() override { psk_destroy(ctx_); }
  CudaBackend(const CudaBackend&) = delete;
  CudaBackend& operator=(const CudaBackend&) = delete;

  void run(const Launch&) override {
    throw ContractViolation("CudaBackend runs only the parallel Kalman drivers");
  }
  unsigned workers() const override { return 1; }
  psk_ctx* ctx() const { return ctx_; }

 private:
  psk_ctx* ctx_ = nullptr;
};

namespace psk_detail {

template <typename S>
constexpr int dtype_of() {
  static_assert(std::is_same_v<S, float> || std::is_same_v<S, double>,
                "the CUDA path supports float and double");
  return std::is_same_v<S, double> ? PSK_F64 : PSK_F32;
}

// Lgssm<S> (per-step std::vector<Mat>) -> dense per-step host arrays
template <typename S>
struct Packed {
  std::vector<S> f, u, q, h, d, r, y, m0, p0;
  psk_model model{};
};

template <typename S, class M>
void pack_mats(std::vector<S>& out, const std::vector<M>& src, std::size_t block) {
  out.resize(src.size() * block);
  for (std::size_t k = 0; k < src.size(); ++k)
    for (std::size_t i = 0; i < block; ++i)
      out[k * block + i] = src[k].view().d[i];
}

template <typename S>
Packed<S> pack(const Lgssm<S>& m, const Measurements<S>& ys) {
  Packed<S> p;
  const std::size_t nx = std::size_t(m.nx), ny = std::size_t(m.ny);
  if (m.f.size() != m.t || m.u.size() != m.t || m.q.size() != m.t || m.h.size() != m.t ||
      m.d.size() != m.t || m.r.size() != m.t || ys.size() != m.t)
    throw DimensionMismatch("model / measurement length");
  pack_mats(p.f, m.f, nx * nx);
  pack_mats(p.u, m.u, nx);
  pack_mats(p.q, m.q, nx * nx);
  pack_mats(p.h, m.h, ny * nx);
  pack_mats(p.d, m.d, ny);
  pack_mats(p.r, m.r, ny * ny);
  pack_mats(p.y, ys, ny);
  p.m0.assign(m.prior_mean.view().d, m.prior_mean.view().d + nx);
  p.p0.assign(m.prior_cov.view().d, m.prior_cov.view().d + nx * nx);
  psk_model& md = p.model;
  md.t = m.t;
  md.nx = m.nx;
  md.ny = m.ny;
  md.dtype = dtype_of<S>();
  md.space = PSK_HOST;
  md.f = p.f.data(); md.u = p.u.data(); md.q = p.q.data(); md.h = p.h.data();
  md.d = p.d.data(); md.r = p.r.data(); md.y = p.y.data();
  md.f_stride = md.u_stride = md.q_stride = md.h_stride = md.d_stride =
      md.r_stride = md.y_stride = -1;
  md.prior_mean = p.m0.data();
  md.prior_cov = p.p0.data();
  return p;
}

template <typename S>
std::vector<GaussianStats<S>> unpack(const std::vector<S>& mean,
                                     const std::vector<S>& cov, std::size_t t, int nx) {
  std::vector<GaussianStats<S>> out;
  out.reserve(t);
  for (std::size_t k = 0; k < t; ++k) {
    GaussianStats<S> g{Vec<S>(nx), Mat<S>(nx, nx)};
    for (int i = 0; i < nx; ++i) g.mean[i] = mean[k * nx + i];
    std::memcpy(g.cov.data(), cov.data() + k * nx * nx, sizeof(S) * nx * nx);
    out.push_back(std::move(g));
  }
  return out;
}

template <typename S, class F>
std::vector<GaussianStats<S>> call(const Lgssm<S>& m, const Measurements<S>& ys, F&& f) {
  if (m.nx < 1 || m.nx > kMaxDim || m.ny < 1 || m.ny > kMaxDim)
    throw DimensionMismatch("mat dims");
  Packed<S> p = pack(m, ys);
  std::vector<S> mean(m.t * std::size_t(m.nx) + 1), cov(m.t * std::size_t(m.nx * m.nx) + 1);
  check(f(p.model, mean.data(), cov.data()));
  return unpack(mean, cov, m.t, m.nx);
}

}  // namespace psk_detail

// PKF, Alg. 5 (kalman_par.hpp:111-119)
template <typename S>
std::vector<GaussianStats<S>> pkf_run(const Lgssm<S>& m, const Measurements<S>& ys,
                                      const ScanSpec& spec, CudaBackend& be) {
  return psk_detail::call(m, ys, [&](const psk_model& md, S* mean, S* cov) {
    return psk_pkf(be.ctx(), &md, int(spec.alg), spec.sengupta_n, mean, cov);
  });
}

// PRTS, Alg. 6 (kalman_par.hpp:156-179)
template <typename S>
std::vector<GaussianStats<S>> prts_run(const Lgssm<S>& m, const Measurements<S>& ys,
                                       const ScanSpec& spec, CudaBackend& be) {
  return psk_detail::call(m, ys, [&](const psk_model& md, S* mean, S* cov) {
    return psk_prts(be.ctx(), &md, int(spec.alg), spec.sengupta_n, mean, cov);
  });
}

// PTFS, Alg. 7 (kalman_par.hpp:207-238)
template <typename S>
std::vector<GaussianStats<S>> ptfs_run(const Lgssm<S>& m, const Measurements<S>& ys,
                                       const ScanSpec& spec, CudaBackend& be_fwd,
                                       CudaBackend& be_bwd, int devices = 1) {
  return psk_detail::call(m, ys, [&](const psk_model& md, S* mean, S* cov) {
    return psk_ptfs(be_fwd.ctx(), be_bwd.ctx(), devices, &md, int(spec.alg),
                    spec.sengupta_n, mean, cov);
  });
}

}  // namespace parascan
