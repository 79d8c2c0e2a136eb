// model_gen_par.hpp -- the reference's random model generator, parallel over
// steps.
//
// gen_model (reference model_gen.hpp:104-158) draws every per-step matrix
// from its own counter-mode stream seeded by stream_seed(seed, step, role)
// (model_gen.hpp:27-31), so the steps are independent: gen_model_par fills
// contiguous step ranges on the host cores with the reference's own per-step
// code (gen_detail::GaussianStream, qr_qfactor, random_spd) and is
// BIT-IDENTICAL to gen_model for every seed (tests/test_model_gen_par.py).
// The measurement series (simulate_data, model_gen.hpp:161-209) is an
// ancestral recursion and stays sequential.  Probe: gen_model takes 12.6 s
// single-threaded at T = 2^22.
#pragma once

#include "parascan/model_gen.hpp"
#include "parascan_b200/host_parallel.hpp"

namespace parascan {

inline Lgssm<double> gen_model_par(std::uint64_t seed, int nx, int ny, std::size_t t) {
  using namespace gen_detail;
  Lgssm<double> m;
  m.t = t;
  m.nx = nx;
  m.ny = ny;
  m.f.resize(t);
  m.u.resize(t);
  m.q.resize(t);
  m.h.resize(t);
  m.d.resize(t);
  m.r.resize(t);
  psk_detail::parallel_for(t, 4096, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t k = lo; k < hi; ++k) {
      {
        GaussianStream g(stream_seed(seed, k, kRoleF));
        Mat<double> raw(nx, nx);
        g.fill(raw.view());
        Mat<double> q(nx, nx);
        qr_qfactor(q.view(), raw.view());
        for (int i = 0; i < nx * nx; ++i) q.data()[i] *= 0.99;
        m.f[k] = std::move(q);
      }
      {
        GaussianStream g(stream_seed(seed, k, kRoleU));
        Vec<double> u(nx);
        g.fill(u.view());
        m.u[k] = std::move(u);
      }
      {
        GaussianStream g(stream_seed(seed, k, kRoleQ));
        m.q[k] = random_spd(g, nx);
      }
      {
        GaussianStream g(stream_seed(seed, k, kRoleH));
        Mat<double> h(ny, nx);
        g.fill(h.view());
        m.h[k] = std::move(h);
      }
      {
        GaussianStream g(stream_seed(seed, k, kRoleD));
        Vec<double> d(ny);
        g.fill(d.view());
        m.d[k] = std::move(d);
      }
      {
        GaussianStream g(stream_seed(seed, k, kRoleR));
        m.r[k] = random_spd(g, ny);
      }
    }
  });
  {
    GaussianStream g(stream_seed(seed, 0, kRolePriorMean));
    m.prior_mean = Vec<double>(nx);
    g.fill(m.prior_mean.view());
  }
  {
    GaussianStream g(stream_seed(seed, 0, kRolePriorCov));
    m.prior_cov = random_spd(g, nx);
  }
  return m;
}

}  // namespace parascan
