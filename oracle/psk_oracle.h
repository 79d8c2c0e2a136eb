/*
 * psk_oracle.h -- CPU restatement of the reference (parascan) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2511_10363_b200/,
 * include/, libpsk.so) links or calls this code.  Only tests/, the smoke()
 * check in __graft_entry__.py and the cpu_baseline / --impl reference legs of
 * bench.py may load it, and only as the checker / the timed CPU baseline.
 *
 * Every function restates the reference algorithm in plain C with the same
 * floating-point operation order, so that when compiled with
 * -ffp-contract=off it is bitwise identical to the reference headers compiled
 * the same way (pinned by tests/test_oracle.py against oracle/_ref, which is
 * built from /root/reference by oracle/Makefile, and against the committed
 * golden vectors in tests/golden/).
 *
 * Layout (shared with the C-ABI in include/psk.h): per-step arrays of
 * row-major matrices,
 *   f[T][nx][nx] u[T][nx] q[T][nx][nx] h[T][ny][nx] d[T][ny] r[T][ny][ny]
 *   y[T][ny], prior mean m0[nx], prior cov p0[nx][nx];
 * outputs mean[T][nx], cov[T][nx][nx].  Index convention follows
 * lgssm.hpp:5-8 (F[0] acts on the prior, H[k] belongs to y[k]).
 */
#ifndef PSK_ORACLE_H
#define PSK_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same values as include/psk.h) */
#define PSO_OK 0
#define PSO_E_DIM 1
#define PSO_E_CONTRACT 2
#define PSO_E_NOT_PD 3
#define PSO_E_SINGULAR 4
#define PSO_E_ALLOC 8

/* ScanAlg order of scan.hpp:32-39 */
#define PSO_SEQUENTIAL 0
#define PSO_HILLIS_STEELE 1
#define PSO_BLELLOCH 2
#define PSO_INPLACE_LAFI 3
#define PSO_SENGUPTA_A 4
#define PSO_SENGUPTA_B 5

#define PSO_DECLARE(S, SFX)                                                   \
  typedef struct {                                                            \
    size_t t;                                                                 \
    int nx, ny;                                                               \
    const S *f, *u, *q, *h, *d, *r, *y, *m0, *p0;                             \
    unsigned bcast; /* bit i: field i (f,u,q,h,d,r,y) is one block */         \
  } pso_model_##SFX;                                                          \
  int pso_kf_run_##SFX(const pso_model_##SFX* m, S* mean, S* cov);            \
  int pso_rts_run_##SFX(const pso_model_##SFX* m, const S* fmean,             \
                        const S* fcov, S* mean, S* cov);                      \
  int pso_bif_run_##SFX(const pso_model_##SFX* m, S* eta, S* jmat);           \
  int pso_tfs_run_##SFX(const pso_model_##SFX* m, S* mean, S* cov);           \
  int pso_pkf_run_##SFX(const pso_model_##SFX* m, int alg, size_t sengupta_n, \
                        S* mean, S* cov);                                     \
  int pso_prts_run_##SFX(const pso_model_##SFX* m, int alg,                   \
                         size_t sengupta_n, S* mean, S* cov);                 \
  int pso_ptfs_run_##SFX(const pso_model_##SFX* m, int alg,                   \
                         size_t sengupta_n, S* mean, S* cov);                 \
  /* element-level entry points (tests): element = a|b|c|eta|J packed */      \
  int pso_make_filter_element_##SFX(const pso_model_##SFX* m, size_t k,       \
                                    S* elem);                                 \
  int pso_filter_combine_##SFX(int nx, const S* l, const S* r, S* out);       \
  int pso_make_smoother_element_##SFX(const pso_model_##SFX* m,               \
                                      const S* fmean_k, const S* fcov_k,      \
                                      size_t k, S* elem);                     \
  int pso_smoother_combine_##SFX(int nx, const S* l, const S* r, S* out);     \
  int pso_tf_combine_##SFX(int nx, const S* mean, const S* cov,               \
                           const S* eta, const S* jmat, S* omean, S* ocov);   \
  /* scan of packed filter elements (n slots, padded by caller), forward or \
     reversed, in place */                                                    \
  int pso_filter_scan_##SFX(int nx, size_t n, S* elems, int alg,              \
                            size_t sengupta_n, int reverse);                  \
  int pso_smoother_scan_##SFX(int nx, size_t n, S* elems, int alg,            \
                              size_t sengupta_n, int reverse);

PSO_DECLARE(double, d)
PSO_DECLARE(float, f)

/* model_gen.hpp restatement (double only, as in the reference). Outputs are
 * caller-allocated arrays in the layout above. */
int pso_gen_model(uint64_t seed, int nx, int ny, size_t t, double* f,
                  double* u, double* q, double* h, double* d, double* r,
                  double* m0, double* p0);
int pso_simulate_data(const pso_model_d* m, uint64_t seed, double* y);
uint64_t pso_splitmix64(uint64_t x);

/* int64 scan under addition (scan.hpp:87-112 Int64Elems) -- the reference's
 * own scan-differential handle, used to pin the scan index maps. */
int pso_int64_scan(size_t n, int64_t* v, int alg, size_t sengupta_n,
                   int reverse);
/* number of combine applications performed by the last int64 scan
 * (count_work_and_span, scan.hpp:495-524) */
uint64_t pso_last_scan_work(void);
uint64_t pso_last_scan_span(void);

#ifdef __cplusplus
}
#endif
#endif
