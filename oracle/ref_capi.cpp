// ref_capi.cpp -- plain-C entry points over the UNMODIFIED reference headers
// (/root/reference/proj/core/include/parascan), compiled by oracle/Makefile
// into oracle/_ref/libparascan_ref.so.  TEST / BASELINE INFRASTRUCTURE ONLY:
// used by tests/ to pin the oracle restatement and by bench.py's
// `--impl reference` / cpu_baseline legs to time the reference's own CPU
// path.  No reference source is copied; this file only marshals flat arrays
// into the reference's Lgssm / Measurements containers and back.
//
// Layout of every flat array: see oracle/psk_oracle.h.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <vector>

#include "parascan/backend.hpp"
#include "parascan/kalman_elems.hpp"
#include "parascan/kalman_par.hpp"
#include "parascan/kalman_seq.hpp"
#include "parascan/lgssm.hpp"
#include "parascan/model_gen.hpp"
#include "parascan/scan.hpp"

using namespace parascan;

namespace {

template <typename S>
struct Flat {
  std::size_t t;
  int nx, ny;
  const S *f, *u, *q, *h, *d, *r, *y, *m0, *p0;
};

template <typename S>
Mat<S> to_mat(const S* p, int r, int c) {
  Mat<S> m(r, c);
  std::memcpy(m.data(), p, sizeof(S) * r * c);
  return m;
}
template <typename S>
Vec<S> to_vec(const S* p, int n) {
  Vec<S> v(n);
  for (int i = 0; i < n; ++i) v[i] = p[i];
  return v;
}

template <typename S>
struct Built {
  Lgssm<S> m;
  Measurements<S> ys;
};

template <typename S>
Built<S> build(const Flat<S>& fl) {
  Built<S> b;
  const int nx = fl.nx, ny = fl.ny;
  b.m.t = fl.t;
  b.m.nx = nx;
  b.m.ny = ny;
  for (std::size_t k = 0; k < fl.t; ++k) {
    b.m.f.push_back(to_mat(fl.f + k * nx * nx, nx, nx));
    b.m.u.push_back(to_vec(fl.u + k * nx, nx));
    b.m.q.push_back(to_mat(fl.q + k * nx * nx, nx, nx));
    b.m.h.push_back(to_mat(fl.h + k * ny * nx, ny, nx));
    b.m.d.push_back(to_vec(fl.d + k * ny, ny));
    b.m.r.push_back(to_mat(fl.r + k * ny * ny, ny, ny));
    if (fl.y) b.ys.push_back(to_vec(fl.y + k * ny, ny));
  }
  b.m.prior_mean = to_vec(fl.m0, nx);
  b.m.prior_cov = to_mat(fl.p0, nx, nx);
  return b;
}

template <typename S>
void put_stats(const std::vector<GaussianStats<S>>& st, int nx, S* mean,
               S* cov) {
  for (std::size_t k = 0; k < st.size(); ++k) {
    for (int i = 0; i < nx; ++i) mean[k * nx + i] = st[k].mean[i];
    std::memcpy(cov + k * nx * nx, st[k].cov.data(), sizeof(S) * nx * nx);
  }
}

// exception -> status code (include/psk.h values)
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const DimensionMismatch&) {
    return 1;
  } catch (const ContractViolation&) {
    return 2;
  } catch (const NotPositiveDefinite&) {
    return 3;
  } catch (const SingularMatrix&) {
    return 4;
  } catch (const std::bad_alloc&) {
    return 8;
  } catch (...) {
    return 9;
  }
}

ScanSpec spec_of(int alg, std::size_t sn) {
  return ScanSpec{static_cast<ScanAlg>(alg), sn};
}

template <typename S>
void put_felem(const FilterElement<S>& e, int nx, S* out) {
  const int n2 = nx * nx;
  std::memcpy(out, e.a.data(), sizeof(S) * n2);
  for (int i = 0; i < nx; ++i) out[n2 + i] = e.b[i];
  std::memcpy(out + n2 + nx, e.c.data(), sizeof(S) * n2);
  for (int i = 0; i < nx; ++i) out[2 * n2 + nx + i] = e.eta[i];
  std::memcpy(out + 2 * n2 + 2 * nx, e.jmat.data(), sizeof(S) * n2);
}
template <typename S>
FilterElement<S> get_felem(const S* p, int nx) {
  const int n2 = nx * nx;
  return FilterElement<S>{to_mat(p, nx, nx), to_vec(p + n2, nx),
                          to_mat(p + n2 + nx, nx, nx),
                          to_vec(p + 2 * n2 + nx, nx),
                          to_mat(p + 2 * n2 + 2 * nx, nx, nx)};
}
template <typename S>
void put_selem(const SmootherElement<S>& e, int nx, S* out) {
  const int n2 = nx * nx;
  std::memcpy(out, e.e.data(), sizeof(S) * n2);
  for (int i = 0; i < nx; ++i) out[n2 + i] = e.g[i];
  std::memcpy(out + n2 + nx, e.l.data(), sizeof(S) * n2);
}
template <typename S>
SmootherElement<S> get_selem(const S* p, int nx) {
  const int n2 = nx * nx;
  return SmootherElement<S>{to_mat(p, nx, nx), to_vec(p + n2, nx),
                            to_mat(p + n2 + nx, nx, nx)};
}

// Persistent model for timing loops (marshalling excluded from timings).
struct Handle {
  bool f64;
  Built<double> bd;
  Built<float> bf;
};

}  // namespace

#define PSR_DEFINE(S, SFX)                                                    \
  extern "C" int psr_kf_run_##SFX(const Flat<S>* fl, S* mean, S* cov) {       \
    return guarded([&] {                                                      \
      auto b = build(*fl);                                                    \
      put_stats(kf_run(b.m, b.ys), fl->nx, mean, cov);                        \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_rts_run_##SFX(const Flat<S>* fl, S* mean, S* cov) {      \
    return guarded([&] {                                                      \
      auto b = build(*fl);                                                    \
      put_stats(rts_run(b.m, kf_run(b.m, b.ys)), fl->nx, mean, cov);          \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_tfs_run_##SFX(const Flat<S>* fl, S* mean, S* cov) {      \
    return guarded([&] {                                                      \
      auto b = build(*fl);                                                    \
      put_stats(tfs_run(b.m, b.ys), fl->nx, mean, cov);                       \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_bif_run_##SFX(const Flat<S>* fl, S* eta, S* jm) {        \
    return guarded([&] {                                                      \
      auto b = build(*fl);                                                    \
      auto info = bif_run(b.m, b.ys);                                         \
      const int nx = fl->nx;                                                  \
      for (std::size_t k = 0; k < info.size(); ++k) {                         \
        for (int i = 0; i < nx; ++i) eta[k * nx + i] = info[k].eta[i];        \
        std::memcpy(jm + k * nx * nx, info[k].jmat.data(),                    \
                    sizeof(S) * nx * nx);                                     \
      }                                                                       \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_pkf_run_##SFX(const Flat<S>* fl, int alg,                \
                                   std::size_t sn, unsigned threads, S* mean, \
                                   S* cov) {                                  \
    return guarded([&] {                                                      \
      auto b = build(*fl);                                                    \
      PoolBackend be(threads);                                                \
      put_stats(pkf_run(b.m, b.ys, spec_of(alg, sn), be), fl->nx, mean,      \
                cov);                                                         \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_prts_run_##SFX(const Flat<S>* fl, int alg,               \
                                    std::size_t sn, unsigned threads,         \
                                    S* mean, S* cov) {                        \
    return guarded([&] {                                                      \
      auto b = build(*fl);                                                    \
      PoolBackend be(threads);                                                \
      put_stats(prts_run(b.m, b.ys, spec_of(alg, sn), be), fl->nx, mean,     \
                cov);                                                         \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_ptfs_run_##SFX(const Flat<S>* fl, int alg,               \
                                    std::size_t sn, unsigned threads,         \
                                    int devices, S* mean, S* cov) {           \
    return guarded([&] {                                                      \
      auto b = build(*fl);                                                    \
      PoolBackend be1(threads), be2(threads);                                 \
      put_stats(ptfs_run(b.m, b.ys, spec_of(alg, sn), be1,                    \
                         devices == 2 ? be2 : be1, devices),                  \
                fl->nx, mean, cov);                                           \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_make_filter_element_##SFX(const Flat<S>* fl,             \
                                               std::size_t k, S* out) {       \
    return guarded([&] {                                                      \
      auto b = build(*fl);                                                    \
      put_felem(make_filter_element(b.m, k, b.ys[k - 1]), fl->nx, out);       \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_filter_combine_##SFX(int nx, const S* l, const S* r,     \
                                          S* out) {                           \
    return guarded([&] {                                                      \
      put_felem(filter_combine(get_felem(l, nx), get_felem(r, nx)), nx, out); \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_make_smoother_element_##SFX(                             \
      const Flat<S>* fl, const S* fm, const S* fc, std::size_t k, S* out) {   \
    return guarded([&] {                                                      \
      auto b = build(*fl);                                                    \
      GaussianStats<S> st{to_vec(fm, fl->nx), to_mat(fc, fl->nx, fl->nx)};    \
      put_selem(make_smoother_element(b.m, st, k, fl->t), fl->nx, out);       \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_smoother_combine_##SFX(int nx, const S* l, const S* r,   \
                                            S* out) {                         \
    return guarded([&] {                                                      \
      put_selem(smoother_combine(get_selem(l, nx), get_selem(r, nx)), nx,     \
                out);                                                         \
    });                                                                       \
  }                                                                           \
  extern "C" int psr_tf_combine_##SFX(int nx, const S* x, const S* p,         \
                                      const S* eta, const S* jm, S* ox,       \
                                      S* op) {                                \
    return guarded([&] {                                                      \
      GaussianStats<S> fs{to_vec(x, nx), to_mat(p, nx, nx)};                  \
      InfoStats<S> in{to_vec(eta, nx), to_mat(jm, nx, nx)};                   \
      auto o = tf_combine(fs, in);                                            \
      for (int i = 0; i < nx; ++i) ox[i] = o.mean[i];                         \
      std::memcpy(op, o.cov.data(), sizeof(S) * nx * nx);                     \
    });                                                                       \
  }

PSR_DEFINE(double, d)
PSR_DEFINE(float, f)

// ---- generators --------------------------------------------------------
extern "C" int psr_gen_model(std::uint64_t seed, int nx, int ny, std::size_t t,
                             double* f, double* u, double* q, double* h,
                             double* d, double* r, double* m0, double* p0) {
  return guarded([&] {
    auto m = gen_model(seed, nx, ny, t);
    for (std::size_t k = 0; k < t; ++k) {
      std::memcpy(f + k * nx * nx, m.f[k].data(), sizeof(double) * nx * nx);
      for (int i = 0; i < nx; ++i) u[k * nx + i] = m.u[k][i];
      std::memcpy(q + k * nx * nx, m.q[k].data(), sizeof(double) * nx * nx);
      std::memcpy(h + k * ny * nx, m.h[k].data(), sizeof(double) * ny * nx);
      for (int i = 0; i < ny; ++i) d[k * ny + i] = m.d[k][i];
      std::memcpy(r + k * ny * ny, m.r[k].data(), sizeof(double) * ny * ny);
    }
    for (int i = 0; i < nx; ++i) m0[i] = m.prior_mean[i];
    std::memcpy(p0, m.prior_cov.data(), sizeof(double) * nx * nx);
  });
}
extern "C" int psr_simulate_data(const Flat<double>* fl, std::uint64_t seed,
                                 double* y) {
  return guarded([&] {
    auto b = build(*fl);
    auto ys = simulate_data(b.m, seed);
    for (std::size_t k = 0; k < ys.size(); ++k)
      for (int i = 0; i < fl->ny; ++i) y[k * fl->ny + i] = ys[k][i];
  });
}

// ---- int64 scans (scan.hpp Int64Elems) ---------------------------------
extern "C" int psr_int64_scan(std::size_t n, std::int64_t* v, int alg,
                              std::size_t sn, int reverse) {
  return guarded([&] {
    Int64Elems e(n);
    for (std::size_t i = 0; i < n; ++i) e[i] = v[i];
    SerialBackend be;
    if (reverse)
      scan_reverse(spec_of(alg, sn), e, be);
    else
      scan_forward(spec_of(alg, sn), e, be);
    for (std::size_t i = 0; i < n; ++i) v[i] = e[i];
  });
}
extern "C" int psr_count_work_and_span(int alg, std::size_t sn, std::size_t t,
                                       std::uint64_t* work,
                                       std::uint64_t* span) {
  return guarded([&] {
    auto ws = count_work_and_span(spec_of(alg, sn), t);
    *work = ws.work;
    *span = ws.span_levels;
  });
}

// ---- timing handles: build the reference containers once, time the run --
extern "C" void* psr_handle_create_d(const Flat<double>* fl, int as_f32) {
  try {
    auto* h = new Handle;
    h->f64 = !as_f32;
    h->bd = build(*fl);
    if (as_f32) {
      h->bf.m = convert_model<float>(h->bd.m);
      h->bf.ys = convert_measurements<float>(h->bd.ys);
      h->bd = Built<double>{};
    }
    return h;
  } catch (...) {
    return nullptr;
  }
}
extern "C" void psr_handle_destroy(void* h) { delete static_cast<Handle*>(h); }

// method: 0 seq KF+RTS (1 core), 1 pkf, 2 prts, 3 ptfs (devices=1),
//         4 seq KF only; returns wall seconds of one run, <0 on error
template <typename S>
static double time_one(const Built<S>& b, int method, int alg, std::size_t sn,
                       PoolBackend& be) {
  const auto t0 = std::chrono::steady_clock::now();
  std::size_t sink = 0;
  switch (method) {
    case 0: sink += rts_run(b.m, kf_run(b.m, b.ys)).size(); break;
    case 1: sink += pkf_run(b.m, b.ys, spec_of(alg, sn), be).size(); break;
    case 2: sink += prts_run(b.m, b.ys, spec_of(alg, sn), be).size(); break;
    case 3: sink += ptfs_run(b.m, b.ys, spec_of(alg, sn), be, be, 1).size(); break;
    case 4: sink += kf_run(b.m, b.ys).size(); break;
    default: return -1.0;
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (sink != b.m.t) return -2.0;
  return std::chrono::duration<double>(t1 - t0).count();
}
extern "C" double psr_handle_time(void* hv, int method, int alg,
                                  std::size_t sn, unsigned threads) {
  try {
    auto* h = static_cast<Handle*>(hv);
    PoolBackend be(threads);
    return h->f64 ? time_one(h->bd, method, alg, sn, be)
                  : time_one(h->bf, method, alg, sn, be);
  } catch (...) {
    return -3.0;
  }
}
