/*
 * psk_oracle.c -- CPU restatement of the reference hot path (parascan).
 * TEST INFRASTRUCTURE ONLY; see psk_oracle.h for the contract.  Build with
 * -ffp-contract=off (oracle/Makefile) so results are plain IEEE and bitwise
 * comparable with the reference compiled the same way.
 */
#include "psk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "psk_scan_generic.h"

#define S double
#define SFX d
#define SQRT sqrt
#include "psk_oracle_impl.inc"
#undef S
#undef SFX
#undef SQRT

#define S float
#define SFX f
#define SQRT sqrtf
#include "psk_oracle_impl.inc"
#undef S
#undef SFX
#undef SQRT

/* ---- model_gen.hpp ----------------------------------------------------- */

/* model_gen.hpp:20-25 */
uint64_t pso_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
/* model_gen.hpp:27-31 */
static uint64_t stream_seed(uint64_t seed, uint64_t step, uint64_t role) {
  return pso_splitmix64(pso_splitmix64(seed ^ (step * 0x9e3779b97f4a7c15ull)) ^
                        (role * 0xd1b54a32d192ed03ull));
}
/* model_gen.hpp:33-67: Marsaglia polar over counter-mode splitmix64 */
typedef struct {
  uint64_t state;
  int have;
  double spare;
} gstream;
static void gs_init(gstream* g, uint64_t seed) {
  g->state = seed;
  g->have = 0;
  g->spare = 0;
}
static double gs_uniform(gstream* g) {
  return (double)(pso_splitmix64(g->state++) >> 11) * 0x1.0p-53;
}
static double gs_next(gstream* g) {
  if (g->have) {
    g->have = 0;
    return g->spare;
  }
  double u, v, s;
  do {
    u = 2.0 * gs_uniform(g) - 1.0;
    v = 2.0 * gs_uniform(g) - 1.0;
    s = u * u + v * v;
  } while (s >= 1.0 || s == 0.0);
  const double f = sqrt(-2.0 * log(s) / s);
  g->spare = v * f;
  g->have = 1;
  return u * f;
}
static void gs_fill(gstream* g, double* a, int n) {
  for (int i = 0; i < n; ++i) a[i] = gs_next(g);
}
enum { kRoleF = 0, kRoleU, kRoleQ, kRoleH, kRoleD, kRoleR, kRolePriorMean,
       kRolePriorCov, kRoleStateNoise, kRoleMeasNoise, kRoleInitState };

/* model_gen.hpp:85-97: Xi Xi^T + 1e-6 I */
static void random_spd(gstream* g, int n, double* out) {
  double xi[256], xt[256];
  gs_fill(g, xi, n * n);
  mtrans_d(xt, xi, n, n);
  mmul_d(out, xi, xt, n, n, n);
  for (int i = 0; i < n; ++i) out[i * n + i] += 1e-6;
  msym_d(out, n);
}

/* mat.hpp:271-318: Householder Q factor, diag(R) >= 0 */
static int qr_qfactor(double* out, const double* a, int n) {
  double r[256], v[16];
  mcopy_d(r, a, n, n);
  meye_d(out, n);
  for (int c = 0; c < n; ++c) {
    double norm2 = 0.0;
    for (int i = c; i < n; ++i) norm2 += r[i * n + c] * r[i * n + c];
    if (!(norm2 > 0.0)) return 5;
    double norm = sqrt(norm2);
    double alpha = r[c * n + c] >= 0.0 ? 0.0 - norm : norm;
    for (int i = c; i < n; ++i) v[i] = r[i * n + c];
    v[c] -= alpha;
    double vnorm2 = 0.0;
    for (int i = c; i < n; ++i) vnorm2 += v[i] * v[i];
    if (vnorm2 == 0.0) continue;
    double beta = 2.0 / vnorm2;
    for (int j = c; j < n; ++j) {
      double dot = 0.0;
      for (int i = c; i < n; ++i) dot += v[i] * r[i * n + j];
      double f = beta * dot;
      for (int i = c; i < n; ++i) r[i * n + j] -= f * v[i];
    }
    for (int j = 0; j < n; ++j) {
      double dot = 0.0;
      for (int i = c; i < n; ++i) dot += out[j * n + i] * v[i];
      double f = beta * dot;
      for (int i = c; i < n; ++i) out[j * n + i] -= f * v[i];
    }
  }
  for (int c = 0; c < n; ++c)
    if (r[c * n + c] < 0.0)
      for (int i = 0; i < n; ++i) out[i * n + c] = 0.0 - out[i * n + c];
  return 0;
}

/* model_gen.hpp:101-158 */
int pso_gen_model(uint64_t seed, int nx, int ny, size_t t, double* f,
                  double* u, double* q, double* h, double* d, double* r,
                  double* m0, double* p0) {
  if (nx < 1 || nx > 16 || ny < 1 || ny > 16) return PSO_E_DIM;
  gstream g;
  for (size_t k = 0; k < t; ++k) {
    double raw[256];
    gs_init(&g, stream_seed(seed, k, kRoleF));
    gs_fill(&g, raw, nx * nx);
    double* fk = f + k * nx * nx;
    if (qr_qfactor(fk, raw, nx)) return 5;
    for (int i = 0; i < nx * nx; ++i) fk[i] *= 0.99;
    gs_init(&g, stream_seed(seed, k, kRoleU));
    gs_fill(&g, u + k * nx, nx);
    gs_init(&g, stream_seed(seed, k, kRoleQ));
    random_spd(&g, nx, q + k * nx * nx);
    gs_init(&g, stream_seed(seed, k, kRoleH));
    gs_fill(&g, h + k * ny * nx, ny * nx);
    gs_init(&g, stream_seed(seed, k, kRoleD));
    gs_fill(&g, d + k * ny, ny);
    gs_init(&g, stream_seed(seed, k, kRoleR));
    random_spd(&g, ny, r + k * ny * ny);
  }
  gs_init(&g, stream_seed(seed, 0, kRolePriorMean));
  gs_fill(&g, m0, nx);
  gs_init(&g, stream_seed(seed, 0, kRolePriorCov));
  random_spd(&g, nx, p0);
  return PSO_OK;
}

/* model_gen.hpp:160-209 */
int pso_simulate_data(const pso_model_d* m, uint64_t seed, double* ys) {
  const int nx = m->nx, ny = m->ny;
  double x[16], l[256], z[16], nn[16], xn[16], y[16];
  gstream g;
  gs_init(&g, stream_seed(seed, 0, kRoleInitState));
  if (chol_d(l, m->p0, nx)) return PSO_E_NOT_PD;
  gs_fill(&g, z, nx);
  mmul_d(x, l, z, nx, nx, 1);
  madd_d(x, x, m->m0, nx, 1);
  for (size_t k = 0; k < m->t; ++k) {
    mmul_d(xn, MF(m, k), x, nx, nx, 1);
    madd_d(xn, xn, MU(m, k), nx, 1);
    gs_init(&g, stream_seed(seed, k, kRoleStateNoise));
    if (chol_d(l, MQ(m, k), nx)) return PSO_E_NOT_PD;
    gs_fill(&g, z, nx);
    mmul_d(nn, l, z, nx, nx, 1);
    madd_d(xn, xn, nn, nx, 1);
    mcopy_d(x, xn, nx, 1);
    mmul_d(y, MH(m, k), x, ny, nx, 1);
    madd_d(y, y, MD(m, k), ny, 1);
    gs_init(&g, stream_seed(seed, k, kRoleMeasNoise));
    if (chol_d(l, MR(m, k), ny)) return PSO_E_NOT_PD;
    gs_fill(&g, z, ny);
    mmul_d(nn, l, z, ny, ny, 1);
    madd_d(y, y, nn, ny, 1);
    mcopy_d(ys + k * ny, y, ny, 1);
  }
  return PSO_OK;
}

/* ---- Int64Elems (scan.hpp:87-112) ------------------------------------ */
static void op_i64_combine(const void* ctx, void* dst, const void* l,
                           const void* r) {
  (void)ctx;
  *(int64_t*)dst = *(const int64_t*)l + *(const int64_t*)r;
}
static void op_i64_identity(const void* ctx, void* dst) {
  (void)ctx;
  *(int64_t*)dst = 0;
}
int pso_int64_scan(size_t n, int64_t* v, int alg, size_t sengupta_n,
                   int reverse) {
  pso_ops ops = {op_i64_combine, op_i64_identity, 0};
  pso_handle h = {(char*)v, n, sizeof(int64_t), &ops, reverse};
  return pso_scan_forward(alg, sengupta_n, &h);
}
uint64_t pso_last_scan_work(void) { return g_pso_work; }
uint64_t pso_last_scan_span(void) { return g_pso_span; }
