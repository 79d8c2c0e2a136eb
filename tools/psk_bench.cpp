// psk_bench.cpp -- the reference's benchmark workbench with the CUDA backend
// (SURVEY.md 8(f) row 3): a CLI11-free driver mirroring `bench run / verify /
// speedup` (reference tools/bench_main.cpp:163-250) that emits rows in the
// reference's tidy CSV schema (bench.hpp:108-188:
// method,alg,T,precision,metric,value,seed,threads,devices), so GPU results
// sit next to the reference's own CPU rows.
//
// It is a reference user's program: the UNMODIFIED reference headers (model
// generator gen_model -- run step-parallel by include/parascan_b200/
// model_gen_par.hpp, bit-identical -- / simulate_data, the sequential f64 oracle kf_run /
// rts_run, the timing protocol time_run, max_rel_err, CSV writer) plus
// include/parascan_b200/cuda_backend.hpp.  Built by tools/Makefile into
// tools/_bin/psk_bench (the reference headers exist only in the build
// container; the binary travels to the GPU box prebuilt).
//
// Per (T, method, alg) cell with --backend cuda (default) the rows are
//   max_rel_err       vs the f64 sequential kf_run / rts_run (bench.hpp:222-260)
//   wall_median_s     the drop-in call through the shim: marshalling of the
//                     reference containers + H2D + kernels + D2H + unpack
//   device_median_s   the kernels alone (psk per-kernel event spans)
//   steps_per_s       T / wall_median_s
//   device_steps_per_s  T / device_median_s
//   hbm_frac          compulsory bytes per step (SURVEY.md 8(d) fused figures:
//                     PKF M + O, PRTS M + 3 O + |F, Q, u|, PTFS 2 M + 3 O
//                     scalars, M = model scalars, O = nx + nx^2) x T /
//                     device time / --peak-gbs
//   fp_frac           (nx = 4, ny = 2 only) counted flops at c = 2 (SURVEY.md
//                     8(d): PKF 3555, PRTS 5073, PTFS 7444 per step) x T /
//                     device time / --peak-tflops
// `threads` = host threads of the marshalling layer; `devices` = GPUs.
// --backend pool runs the reference's own PoolBackend(threads) instead
// (max_rel_err + wall_median_s, the reference's rows).
//
// usage: psk_bench run|verify|speedup [--seed S] [--nx N] [--ny N] [--T t]...
//        [--methods m...] [--algs a...|all] [--precision f32|f64] [--runs R]
//        [--warmup W] [--threads P] [--devices D] [--sengupta-n N] [--out f.csv]
//        [--gate] [--backend cuda|pool] [--mode fast|exact] [--device d]
//        [--model gen|cv] [--peak-gbs G] [--peak-tflops F]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "parascan/bench.hpp"
#include "parascan/kalman_par.hpp"
#include "parascan/kalman_seq.hpp"
#include "parascan/model_gen.hpp"
#include "parascan_b200/cuda_backend.hpp"
#include "parascan_b200/model_gen_par.hpp"

using namespace parascan;

namespace {

struct Opts {
  std::string cmd;
  std::uint64_t seed = 0;
  int nx = 4, ny = 2;
  std::vector<std::size_t> t_grid;
  std::vector<std::string> methods = {"pkf", "prts", "ptfs", "seq_kf"};
  std::vector<std::string> algs = {"decoupled_lookback"};
  std::string precision = "f64";
  int runs = 12, warmup = 2;
  unsigned threads = 0;
  int devices = 1;
  std::size_t sengupta_n = 16;
  std::string out;
  bool gate = false;
  std::string backend = "cuda", mode = "fast", model = "gen";
  int device = 0;
  double peak_gbs = 6547.5, peak_tflops = 0;
};

std::optional<Method> parse_method(const std::string& s) {
  if (s == "pkf") return Method::PKF;
  if (s == "prts") return Method::PRTS;
  if (s == "ptfs") return Method::PTFS;
  if (s == "seq_kf") return Method::SEQ_KF;
  if (s == "seq_rts") return Method::SEQ_RTS;
  if (s == "seq_tfs") return Method::SEQ_TFS;
  return std::nullopt;
}

// the reference's labels (scan.hpp:46-56) + the appended look-back scan
std::optional<ScanAlg> parse_alg(const std::string& s) {
  if (s == "seqscan") return ScanAlg::Sequential;
  if (s == "hillis_steele") return ScanAlg::HillisSteele;
  if (s == "blelloch") return ScanAlg::Blelloch;
  if (s == "inplace_lafi") return ScanAlg::InplaceLaFi;
  if (s == "sengupta_a") return ScanAlg::SenguptaA;
  if (s == "sengupta_b") return ScanAlg::SenguptaB;
  if (s == "decoupled_lookback") return kDecoupledLookback;
  return std::nullopt;
}
std::string alg_label(ScanAlg a) {
  return a == kDecoupledLookback ? std::string("decoupled_lookback") : std::string(to_string(a));
}

int usage(const char* why) {
  std::cerr << "psk_bench: " << why
            << "\nusage: psk_bench run|verify|speedup [--seed S] [--nx N] [--ny N] [--T t]..."
               " [--methods m...] [--algs a...|all] [--precision f32|f64] [--runs R]"
               " [--warmup W] [--threads P] [--devices D] [--sengupta-n N] [--out f.csv]"
               " [--gate] [--backend cuda|pool] [--mode fast|exact] [--device d]"
               " [--model gen|cv] [--peak-gbs G] [--peak-tflops F]\n";
  return 2;
}

// multi-value options take every following token that is not a flag
int parse(int argc, char** argv, Opts& o) {
  if (argc < 2) return usage("missing subcommand");
  o.cmd = argv[1];
  if (o.cmd != "run" && o.cmd != "verify" && o.cmd != "speedup") return usage("bad subcommand");
  bool methods_set = false, algs_set = false;
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto one = [&]() -> std::string {
      if (i + 1 >= argc) throw std::invalid_argument("missing value for " + k);
      return argv[++i];
    };
    auto many = [&]() {
      std::vector<std::string> v;
      while (i + 1 < argc && std::strncmp(argv[i + 1], "--", 2) != 0) v.push_back(argv[++i]);
      if (v.empty()) throw std::invalid_argument("missing value for " + k);
      return v;
    };
    if (k == "--seed") o.seed = std::stoull(one());
    else if (k == "--nx") o.nx = std::stoi(one());
    else if (k == "--ny") o.ny = std::stoi(one());
    else if (k == "--T") for (auto& s : many()) o.t_grid.push_back(std::stoull(s));
    else if (k == "--methods") {
      if (!methods_set) o.methods.clear();
      methods_set = true;
      for (auto& s : many()) o.methods.push_back(s);
    } else if (k == "--algs") {
      if (!algs_set) o.algs.clear();
      algs_set = true;
      for (auto& s : many()) o.algs.push_back(s);
    }
    else if (k == "--precision") o.precision = one();
    else if (k == "--runs") o.runs = std::stoi(one());
    else if (k == "--warmup") o.warmup = std::stoi(one());
    else if (k == "--threads") o.threads = unsigned(std::stoul(one()));
    else if (k == "--devices") o.devices = std::stoi(one());
    else if (k == "--sengupta-n") o.sengupta_n = std::stoull(one());
    else if (k == "--out") o.out = one();
    else if (k == "--gate") o.gate = true;
    else if (k == "--backend") o.backend = one();
    else if (k == "--mode") o.mode = one();
    else if (k == "--device") o.device = std::stoi(one());
    else if (k == "--model") o.model = one();
    else if (k == "--peak-gbs") o.peak_gbs = std::stod(one());
    else if (k == "--peak-tflops") o.peak_tflops = std::stod(one());
    else return usage(("unknown option " + k).c_str());
  }
  if (o.t_grid.empty()) o.t_grid = {64, 256, 1024};
  if (!algs_set && o.backend == "pool") o.algs = {"inplace_lafi"};  // the reference's default
  if (o.nx < 1 || o.nx > 16 || o.ny < 1 || o.ny > 16) return usage("nx, ny in 1..16");
  if (o.precision != "f32" && o.precision != "f64") return usage("precision f32|f64");
  if (o.runs <= o.warmup || o.warmup < 0) return usage("need runs > warmup >= 0");
  if (o.devices != 1 && o.devices != 2) return usage("devices must be 1 or 2");
  if (o.backend != "cuda" && o.backend != "pool") return usage("backend cuda|pool");
  if (o.mode != "fast" && o.mode != "exact") return usage("mode fast|exact");
  if (o.model != "gen" && o.model != "cv") return usage("model gen|cv");
  if (o.threads == 0) {
    if (const char* e = std::getenv("PARASCAN_THREADS")) o.threads = unsigned(std::atol(e));
    if (o.threads == 0) o.threads = o.backend == "cuda" ? psk_detail::host_threads() : 1;
  }
  if (o.peak_tflops <= 0) o.peak_tflops = o.precision == "f64" ? 34.2 : 72.55;  // tools/peak.py
  return 0;
}

// SURVEY.md 8(d) synthetic tracking model: damped 2-D constant velocity
// (rho_p = 0.99, rho_v = 0.95, dt = 0.1, q = 1, R = 0.25 I), written per step;
// measurements from the reference's simulate_data
Lgssm<double> cv_model(std::size_t t) {
  const double dt = 0.1, rp = 0.99, rv = 0.95;
  Mat<double> F(4, 4), Q(4, 4), H(2, 4), R(2, 2);
  F(0, 0) = F(1, 1) = rp;
  F(2, 2) = F(3, 3) = rv;
  F(0, 2) = F(1, 3) = dt;
  for (int i = 0; i < 2; ++i) {
    Q(i, i) = dt * dt * dt / 3;
    Q(i, i + 2) = Q(i + 2, i) = dt * dt / 2;
    Q(i + 2, i + 2) = dt;
    H(i, i) = 1;
    R(i, i) = 0.25;
  }
  Lgssm<double> m;
  m.nx = 4;
  m.ny = 2;
  m.t = t;
  m.f.assign(t, F);
  m.q.assign(t, Q);
  m.h.assign(t, H);
  m.r.assign(t, R);
  m.u.assign(t, Vec<double>(4));
  m.d.assign(t, Vec<double>(2));
  m.prior_mean = Vec<double>(4);
  m.prior_mean[2] = 1;
  m.prior_mean[3] = -1;
  m.prior_cov = Mat<double>::identity(4);
  return m;
}

double median(std::vector<double> v, int warmup) { return median_after_warmup(std::move(v), warmup); }

struct Cell {
  double err = 0, wall = 0, dev = 0;
};

// device time of the last call: the kernel spans, without the copy marks
double device_seconds(psk_ctx* c) {
  const char* names[64];
  float ms[64];
  const int n = psk_last_profile(c, names, ms, 64);
  double s = 0;
  for (int i = 0; i < n && i < 64; ++i)
    if (std::strstr(names[i], "h2d") == nullptr && std::strstr(names[i], "d2h") == nullptr &&
        std::strstr(names[i], "d2d") == nullptr)
      s += ms[i];
  return s * 1e-3;
}

template <typename S>
Cell run_cell(const Opts& o, Method method, ScanAlg alg, const Lgssm<S>& m,
              const Measurements<S>& ys, const std::vector<GaussianStats<double>>& ref,
              CudaBackend* be, CudaBackend* be2, PoolBackend* pool, int runs, int warmup) {
  const ScanSpec spec{alg, o.sengupta_n};
  const bool seq = method == Method::SEQ_KF || method == Method::SEQ_RTS ||
                   method == Method::SEQ_TFS;
  double dev_last = 0;
  auto call = [&]() -> std::vector<GaussianStats<S>> {
    if (seq || pool) return bench_detail::run_method(method, m, ys, spec, *pool, o.devices);
    std::vector<GaussianStats<S>> r;
    switch (method) {
      case Method::PKF: r = pkf_run(m, ys, spec, *be); dev_last = device_seconds(be->ctx()); break;
      case Method::PRTS: r = prts_run(m, ys, spec, *be); dev_last = device_seconds(be->ctx()); break;
      default:
        r = ptfs_run(m, ys, spec, *be, *be2, o.devices);
        dev_last = std::max(device_seconds(be->ctx()), device_seconds(be2->ctx()));
    }
    return r;
  };
  Cell c;
  c.err = bench_detail::max_rel_err(call(), ref);
  std::vector<double> walls, devs;
  for (int i = 0; i < runs; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    call();
    const auto t1 = std::chrono::steady_clock::now();
    walls.push_back(std::chrono::duration<double>(t1 - t0).count());
    devs.push_back(dev_last);
  }
  c.wall = median(walls, warmup);
  c.dev = median(devs, warmup);
  return c;
}

std::size_t model_scalars(int nx, int ny) {
  return std::size_t(2 * nx * nx + nx + ny * nx + ny + ny * ny + ny);
}

}  // namespace

int main(int argc, char** argv) {
  Opts o;
  try {
    if (int rc = parse(argc, argv, o)) return rc;
  } catch (const std::exception& e) {
    return usage(e.what());
  }
  std::vector<Method> methods;
  for (auto& s : o.methods) {
    auto m = parse_method(s);
    if (!m) return usage(("unknown method " + s).c_str());
    methods.push_back(*m);
  }
  std::vector<ScanAlg> algs;
  for (auto& s : o.algs) {
    if (s == "all") {
      algs = {ScanAlg::Sequential, ScanAlg::HillisSteele, ScanAlg::Blelloch, ScanAlg::InplaceLaFi,
              ScanAlg::SenguptaA, ScanAlg::SenguptaB};
      if (o.backend == "cuda") algs.push_back(kDecoupledLookback);
      break;
    }
    auto a = parse_alg(s);
    if (!a) return usage(("unknown scan algorithm " + s).c_str());
    if (*a == kDecoupledLookback && o.backend == "pool")
      return usage("decoupled_lookback runs on the cuda backend only");
    algs.push_back(*a);
  }
  const bool verify = o.cmd == "verify";
  const int runs = verify ? 1 : o.runs, warmup = verify ? 0 : o.warmup;
  const bool f32 = o.precision == "f32";
  try {
    std::unique_ptr<CudaBackend> be, be2;
    std::unique_ptr<PoolBackend> pool(new PoolBackend(o.backend == "pool" ? o.threads : 1));
    if (o.backend == "cuda") {
      const int mode = o.mode == "fast" ? PSK_MODE_FAST : PSK_MODE_EXACT;
      be.reset(new CudaBackend(o.device, mode));
      if (o.devices == 2) {  // a second GPU for the backward pass when present
        try {
          be2.reset(new CudaBackend(o.device + 1, mode));
        } catch (const std::exception&) {
          be2.reset();
        }
      }
      if (!be2) be2.reset(new CudaBackend(o.device, mode));
      psk_set_profile(be->ctx(), 1);
      psk_set_profile(be2->ctx(), 1);
      setenv("PSK_HOST_THREADS", std::to_string(o.threads).c_str(), 1);
    }
    std::vector<ResultRow> rows;
    bool gating_failed = false;
    for (std::size_t t : o.t_grid) {
      const Lgssm<double> m = o.model == "cv" ? cv_model(t) : gen_model_par(o.seed, o.nx, o.ny, t);
      const Measurements<double> ys = simulate_data(m, o.seed + 1);
      const auto kf = kf_run(m, ys);
      const auto rts = rts_run(m, kf);
      const auto m32 = convert_model<float>(m);
      const auto ys32 = convert_measurements<float>(ys);
      auto emit_for = [&](Method method, const std::string& alg, const std::string& metric,
                          double v) {
        rows.push_back(ResultRow{to_string(method), alg, t, o.precision, metric, v, o.seed,
                                 o.threads, o.devices});
      };
      if (o.cmd == "speedup") {
        // sequential KF on one core vs the PKF drop-in (bench.hpp:326-359)
        const ScanSpec spec{algs.empty() ? kDecoupledLookback : algs[0], o.sengupta_n};
        double seq_s, par_s;
        if (f32) {
          seq_s = time_run([&] { kf_run(m32, ys32); }, o.runs, o.warmup);
          par_s = o.backend == "cuda" ? time_run([&] { pkf_run(m32, ys32, spec, *be); }, o.runs, o.warmup)
                                      : time_run([&] { pkf_run(m32, ys32, spec, *pool); }, o.runs, o.warmup);
        } else {
          seq_s = time_run([&] { kf_run(m, ys); }, o.runs, o.warmup);
          par_s = o.backend == "cuda" ? time_run([&] { pkf_run(m, ys, spec, *be); }, o.runs, o.warmup)
                                      : time_run([&] { pkf_run(m, ys, spec, *pool); }, o.runs, o.warmup);
        }
        emit_for(Method::PKF, alg_label(spec.alg), "speedup_wall", seq_s / par_s);
        continue;
      }
      for (Method method : methods) {
        const bool seq = method == Method::SEQ_KF || method == Method::SEQ_RTS ||
                         method == Method::SEQ_TFS;
        const std::vector<ScanAlg> cell_algs = seq ? std::vector<ScanAlg>{ScanAlg::Sequential} : algs;
        const auto& ref = bench_detail::oracle_for(method, kf, rts);
        for (ScanAlg alg : cell_algs) {
          const std::string label = seq ? "seq" : alg_label(alg);
          CudaBackend* b = seq ? nullptr : be.get();
          PoolBackend* p = (seq || o.backend == "pool") ? pool.get() : nullptr;
          Cell c = f32 ? run_cell<float>(o, method, alg, m32, ys32, ref, b, be2.get(), p, runs, warmup)
                       : run_cell<double>(o, method, alg, m, ys, ref, b, be2.get(), p, runs, warmup);
          emit_for(method, label, "max_rel_err", c.err);
          if (c.err > rel_err_tolerance(f32 ? Precision::F32 : Precision::F64)) gating_failed = true;
          if (verify) continue;
          emit_for(method, label, "wall_median_s", c.wall);
          emit_for(method, label, "steps_per_s", double(t) / c.wall);
          if (b == nullptr || c.dev <= 0) continue;
          emit_for(method, label, "device_median_s", c.dev);
          emit_for(method, label, "device_steps_per_s", double(t) / c.dev);
          const std::size_t M = model_scalars(o.nx, o.ny), O = std::size_t(o.nx + o.nx * o.nx);
          const std::size_t fqu = std::size_t(2 * o.nx * o.nx + o.nx);
          const std::size_t scal = method == Method::PKF ? M + O
                                   : method == Method::PRTS ? M + 3 * O + fqu
                                                            : 2 * M + 3 * O;
          const double bytes = double(scal) * (f32 ? 4 : 8) * double(t);
          emit_for(method, label, "hbm_frac", bytes / c.dev / (o.peak_gbs * 1e9));
          if (o.nx == 4 && o.ny == 2) {
            const double fl = method == Method::PKF ? 3555 : method == Method::PRTS ? 5073 : 7444;
            emit_for(method, label, "fp_frac", fl * double(t) / c.dev / (o.peak_tflops * 1e12));
          }
        }
      }
    }
    sort_rows(rows);
    if (!o.out.empty()) write_csv(o.out, rows);
    std::cout << kCsvHeader << "\n";
    for (const auto& r : rows) std::cout << format_row(r) << "\n";
    if (verify) return gating_failed ? 1 : 0;
    return (o.gate && gating_failed) ? 1 : 0;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
