// dropin_check.cpp -- the C++ drop-in exercised end to end (test
// infrastructure, run by tests/test_gpu_dropin.py on the GPU box).
//
// A reference user's program: the UNMODIFIED reference headers
// (/root/reference/proj/core/include, model generator, drivers, PoolBackend)
// plus include/parascan_b200/cuda_backend.hpp.  The same call sites run once
// with the reference's PoolBackend and once with parascan::CudaBackend -- the
// only change a caller makes -- and the program prints the max relative
// error (bench.hpp:216-237 metric) of every GPU result against the
// reference's own result on the same inputs.  Exit 0 iff all are within the
// FP64 gate (1e-9), and the reference's exception types come back from the
// GPU path (a non-PD S: NotPositiveDefinite; an empty SenguptaB threshold:
// ContractViolation).
#include <cmath>
#include <cstdio>
#include <vector>

#include "parascan/kalman_par.hpp"
#include "parascan/model_gen.hpp"
#include "parascan_b200/cuda_backend.hpp"

using namespace parascan;

static double rel_err(const std::vector<GaussianStats<double>>& a,
                      const std::vector<GaussianStats<double>>& b) {
  double e = 0;
  for (std::size_t k = 0; k < a.size(); ++k) {
    const auto am = a[k].mean.view(), bm = b[k].mean.view();
    for (int i = 0; i < am.rows; ++i)
      e = std::fmax(e, std::fabs(am(i, 0) - bm(i, 0)) / (1 + std::fabs(bm(i, 0))));
    const auto ac = a[k].cov.view(), bc = b[k].cov.view();
    for (int i = 0; i < ac.rows; ++i)
      for (int j = 0; j < ac.cols; ++j)
        e = std::fmax(e, std::fabs(ac(i, j) - bc(i, j)) / (1 + std::fabs(bc(i, j))));
  }
  return a.size() == b.size() ? e : 1e300;
}

int main() {
  int bad = 0;
  PoolBackend pool(4);
  CudaBackend gpu(0), gpu2(0);
  CudaBackend exact(0, PSK_MODE_EXACT);
  const int dims[][2] = {{4, 2}, {3, 1}, {8, 4}};
  for (const auto& d : dims) {
    const Lgssm<double> m = gen_model(11, d[0], d[1], 1500);
    const Measurements<double> ys = simulate_data(m, 12);
    for (ScanAlg alg : {ScanAlg::InplaceLaFi, ScanAlg::Blelloch, ScanAlg::SenguptaB}) {
      const ScanSpec spec{alg, 16};
      const double e1 = rel_err(prts_run(m, ys, spec, gpu), prts_run(m, ys, spec, pool));
      const double e2 = rel_err(pkf_run(m, ys, spec, gpu), pkf_run(m, ys, spec, pool));
      const double e3 = rel_err(ptfs_run(m, ys, spec, gpu, gpu2, 2),
                                ptfs_run(m, ys, spec, pool, pool, 2));
      // exact mode: the reference's own operation order, bitwise
      const double e4 = rel_err(prts_run(m, ys, spec, exact), prts_run(m, ys, spec, pool));
      std::printf("nx=%d ny=%d alg=%s prts %.3e pkf %.3e ptfs %.3e exact-prts %.3e\n", d[0],
                  d[1], to_string(alg), e1, e2, e3, e4);
      if (!(e1 < 1e-9 && e2 < 1e-9 && e3 < 1e-9 && e4 == 0.0)) ++bad;
    }
    const double ed = rel_err(prts_run(m, ys, ScanSpec{kDecoupledLookback, 1}, gpu),
                              prts_run(m, ys, ScanSpec{ScanAlg::InplaceLaFi, 1}, pool));
    std::printf("nx=%d ny=%d alg=decoupled_lookback prts %.3e\n", d[0], d[1], ed);
    if (!(ed < 1e-9)) ++bad;
  }
  // multi-device backends (psk_create_multi): the time axis sharded over the
  // members, PTFS on two halves; on a one-GPU box the members are streams of
  // GPU 0 (the exchange is then a same-device peer copy)
  for (const std::vector<int> devs : {std::vector<int>{0, 0}, std::vector<int>{0, 0, 0, 0},
                                      std::vector<int>{0, 0, 0}}) {
    CudaBackend multi(devs);
    const Lgssm<double> m = gen_model(31, 4, 2, 2500);
    const Measurements<double> ys = simulate_data(m, 32);
    for (ScanAlg alg : {kDecoupledLookback, ScanAlg::InplaceLaFi}) {
      const ScanSpec spec{alg, 16};
      const ScanSpec rspec{ScanAlg::InplaceLaFi, 16};
      const double e1 = rel_err(prts_run(m, ys, spec, multi), prts_run(m, ys, rspec, pool));
      const double e2 = rel_err(pkf_run(m, ys, spec, multi), pkf_run(m, ys, rspec, pool));
      const double e3 = rel_err(ptfs_run(m, ys, spec, multi, multi, multi.devices()),
                                ptfs_run(m, ys, rspec, pool, pool, 2));
      std::printf("multi-device x%d alg=%s prts %.3e pkf %.3e ptfs(halves) %.3e\n",
                  multi.devices(), alg == kDecoupledLookback ? "decoupled_lookback" : to_string(alg),
                  e1, e2, e3);
      if (!(e1 < 1e-9 && e2 < 1e-9 && e3 < 1e-9)) ++bad;
    }
  }
  // SoA-output overloads (caller-owned arrays) == the vector<GaussianStats> path
  {
    const Lgssm<double> m = gen_model(21, 4, 2, 3000);
    const Measurements<double> ys = simulate_data(m, 22);
    const ScanSpec spec{kDecoupledLookback, 1};
    const auto v = prts_run(m, ys, spec, gpu);
    std::vector<double> mean(m.t * 4), cov(m.t * 16);
    prts_run(m, ys, spec, gpu, mean.data(), cov.data());
    double e = 0;
    for (std::size_t k = 0; k < m.t; ++k) {
      for (int i = 0; i < 4; ++i) e = std::fmax(e, std::fabs(mean[k * 4 + i] - v[k].mean[i]));
      for (int i = 0; i < 16; ++i) e = std::fmax(e, std::fabs(cov[k * 16 + i] - v[k].cov.data()[i]));
    }
    std::printf("SoA-output prts vs vector prts: max |diff| %.3e\n", e);
    if (e != 0.0) ++bad;
    // f32 through the shim against the reference's f32 PoolBackend result
    const auto m32 = convert_model<float>(m);
    const auto ys32 = convert_measurements<float>(ys);
    const auto g32 = prts_run(m32, ys32, ScanSpec{ScanAlg::InplaceLaFi, 1}, gpu);
    const auto r32 = prts_run(m32, ys32, ScanSpec{ScanAlg::InplaceLaFi, 1}, pool);
    double e32 = 0;
    for (std::size_t k = 0; k < m.t; ++k)
      for (int i = 0; i < 16; ++i)
        e32 = std::fmax(e32, std::fabs(double(g32[k].cov.data()[i]) - r32[k].cov.data()[i]) /
                                 (1 + std::fabs(r32[k].cov.data()[i])));
    std::printf("f32 prts cov vs reference f32: %.3e\n", e32);
    if (!(e32 < 1e-2)) ++bad;  // the reference's f32 gate (bench.hpp rel_err_tolerance)
  }
  // error behaviour
  {
    Lgssm<double> m = gen_model(3, 4, 2, 50);
    const Measurements<double> ys = simulate_data(m, 4);
    bool threw = false;
    try {
      prts_run(m, ys, ScanSpec{ScanAlg::SenguptaB, 3}, gpu);
    } catch (const ContractViolation&) {
      threw = true;
    }
    std::printf("SenguptaB n=3 -> ContractViolation: %s\n", threw ? "yes" : "no");
    if (!threw) ++bad;
    m.r[10] = Mat<double>(2, 2);
    m.r[10].view()(0, 0) = -1e3;
    m.r[10].view()(1, 1) = -1e3;
    threw = false;
    try {
      pkf_run(m, ys, ScanSpec{ScanAlg::InplaceLaFi, 1}, gpu);
    } catch (const NotPositiveDefinite&) {
      threw = true;
    }
    std::printf("indefinite S -> NotPositiveDefinite: %s\n", threw ? "yes" : "no");
    if (!threw) ++bad;
    // a malformed step block: the reference rejects it in mat_mul
    // (DimensionMismatch, mat.hpp:61-63); so must the packer
    Lgssm<double> mb = gen_model(5, 4, 2, 40);
    const Measurements<double> ysb = simulate_data(mb, 6);
    mb.h[7] = Mat<double>(3, 4);
    bool ref_threw = false;
    threw = false;
    try {
      prts_run(mb, ysb, ScanSpec{ScanAlg::InplaceLaFi, 1}, pool);
    } catch (const DimensionMismatch&) {
      ref_threw = true;
    }
    try {
      prts_run(mb, ysb, ScanSpec{ScanAlg::InplaceLaFi, 1}, gpu);
    } catch (const DimensionMismatch&) {
      threw = true;
    }
    std::printf("malformed H block -> DimensionMismatch: reference %s, CudaBackend %s\n",
                ref_threw ? "yes" : "no", threw ? "yes" : "no");
    if (!threw || !ref_threw) ++bad;
  }
  std::printf("%s\n", bad ? "DROPIN FAIL" : "DROPIN OK");
  return bad ? 1 : 0;
}
