/*
 * Scalar-agnostic restatement of the reference scan kernels (scan.hpp).
 * TEST INFRASTRUCTURE ONLY (see psk_oracle.h).
 *
 * A handle is an array of n packed slots of `slot_bytes` each plus an
 * operator table; `rev` implements the Reversed<E> adapter of
 * scan.hpp:149-177 (logical i -> physical n-1-i, operands flipped).
 */
#ifndef PSK_SCAN_GENERIC_H
#define PSK_SCAN_GENERIC_H
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  /* dst = l (x) r ; alias-safe (dst may be l or r) */
  void (*combine)(const void* ctx, void* dst, const void* l, const void* r);
  void (*set_identity)(const void* ctx, void* dst);
  const void* ctx;
} pso_ops;

typedef struct {
  char* data;
  size_t n;
  size_t slot_bytes;
  const pso_ops* ops;
  int rev;
} pso_handle;

/* work/span tally of scan.hpp:495-524 (count_work_and_span) */
static uint64_t g_pso_work, g_pso_span, g_pso_launch_work;
static void pso_launch_begin(void) { g_pso_launch_work = 0; }
static void pso_launch_end(void) {
  g_pso_work += g_pso_launch_work;
  if (g_pso_launch_work) ++g_pso_span;
}

static char* pso_slot(const pso_handle* h, size_t i) {
  size_t p = h->rev ? h->n - 1 - i : i;
  return h->data + p * h->slot_bytes;
}

/* H::combine(dst, l, li, r, ri) through the adapter */
static void pso_hcombine(pso_handle* dst, size_t di, const pso_handle* l,
                         size_t li, const pso_handle* r, size_t ri) {
  ++g_pso_launch_work;
  if (!dst->rev)
    dst->ops->combine(dst->ops->ctx, pso_slot(dst, di), pso_slot(l, li),
                      pso_slot(r, ri));
  else /* Reversed::combine flips operands, scan.hpp:164-167 */
    dst->ops->combine(dst->ops->ctx, pso_slot(dst, di), pso_slot(r, ri),
                      pso_slot(l, li));
}
static void pso_hassign(pso_handle* dst, size_t di, const pso_handle* src,
                        size_t si) {
  memcpy(pso_slot(dst, di), pso_slot(src, si), dst->slot_bytes);
}
static void pso_hidentity(pso_handle* h, size_t i) {
  h->ops->set_identity(h->ops->ctx, pso_slot(h, i));
}
static int pso_make_like(const pso_handle* h, size_t n, pso_handle* out) {
  out->n = n;
  out->slot_bytes = h->slot_bytes;
  out->ops = h->ops;
  out->rev = h->rev;
  out->data = (char*)calloc(n ? n : 1, h->slot_bytes);
  return out->data ? 0 : -1;
}

static int pso_is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }
static size_t pso_next_pow2(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}
static unsigned pso_log2_exact(size_t n) {
  unsigned l = 0;
  while (((size_t)1 << l) < n) ++l;
  return l;
}

/* scan.hpp:198-210 */
static void pso_seq(pso_handle* a) {
  size_t n = a->n;
  if (n <= 1) return;
  pso_launch_begin();
  for (size_t i = 0; i + 1 < n; ++i) pso_hcombine(a, i + 1, a, i, a, i + 1);
  pso_launch_end();
}

/* scan.hpp:214-259: Hillis-Steele on [base, base+n) with ping-pong */
static int pso_hs_segment(pso_handle* buf, size_t base, size_t n) {
  if (n <= 1) return 0;
  pso_handle aux;
  if (pso_make_like(buf, n, &aux)) return -1;
  pso_handle *cur = buf, *nxt = &aux;
  size_t cur_base = base, nxt_base = 0;
  unsigned levels = pso_log2_exact(n);
  for (unsigned d = 0; d < levels; ++d) {
    size_t delta = (size_t)1 << d;
    pso_launch_begin();
    for (size_t i = 0; i < n; ++i) {
      if (i >= delta)
        pso_hcombine(nxt, nxt_base + i, cur, cur_base + i - delta, cur,
                     cur_base + i);
      else
        pso_hassign(nxt, nxt_base + i, cur, cur_base + i);
    }
    pso_launch_end();
    pso_handle* t = cur;
    cur = nxt;
    nxt = t;
    size_t tb = cur_base;
    cur_base = nxt_base;
    nxt_base = tb;
  }
  if (cur != buf)
    for (size_t i = 0; i < n; ++i) pso_hassign(buf, base + i, cur, cur_base + i);
  free(aux.data);
  return 0;
}

/* scan.hpp:261-279 */
static void pso_upsweep(pso_handle* a, size_t n) {
  unsigned levels = pso_log2_exact(n);
  for (unsigned d = 0; d < levels; ++d) {
    size_t d1 = (size_t)1 << d, d2 = d1 << 1;
    pso_launch_begin();
    for (size_t m = 0; m < n / d2; ++m) {
      size_t j = m * d2 + d1 - 1, kk = m * d2 + d2 - 1;
      pso_hcombine(a, kk, a, j, a, kk);
    }
    pso_launch_end();
  }
}

/* scan.hpp:281-341 */
static int pso_blelloch(pso_handle* a) {
  size_t n = a->n;
  if (n <= 1) return 0;
  unsigned levels = pso_log2_exact(n);
  pso_handle orig, tmp;
  if (pso_make_like(a, n, &orig)) return -1;
  for (size_t i = 0; i < n; ++i) pso_hassign(&orig, i, a, i);
  pso_upsweep(a, n);
  pso_hidentity(a, n - 1);
  if (pso_make_like(a, n / 2, &tmp)) {
    free(orig.data);
    return -1;
  }
  for (unsigned d = levels; d-- > 0;) {
    size_t d1 = (size_t)1 << d, d2 = d1 << 1;
    pso_launch_begin();
    for (size_t m = 0; m < n / d2; ++m) {
      size_t j = m * d2 + d1 - 1, kk = m * d2 + d2 - 1;
      pso_hassign(&tmp, m, a, j);
      pso_hassign(a, j, a, kk);
      pso_hcombine(a, kk, a, kk, &tmp, m);
    }
    pso_launch_end();
  }
  pso_launch_begin();
  for (size_t i = 0; i < n; ++i) pso_hcombine(a, i, a, i, &orig, i);
  pso_launch_end();
  free(orig.data);
  free(tmp.data);
  return 0;
}

/* scan.hpp:343-367 */
static void pso_lafi(pso_handle* a) {
  size_t n = a->n;
  if (n <= 1) return;
  unsigned levels = pso_log2_exact(n);
  pso_upsweep(a, n);
  for (unsigned d = levels; d-- > 0;) {
    size_t d1 = (size_t)1 << d, d2 = d1 << 1, blocks = n / d2;
    if (blocks <= 1) continue;
    pso_launch_begin();
    for (size_t m = 0; m + 1 < blocks; ++m) {
      size_t i = (m + 1) * d2 - 1, j = i + d1;
      pso_hcombine(a, j, a, i, a, j);
    }
    pso_launch_end();
  }
}

/* scan.hpp:369-444 */
static int pso_sengupta(pso_handle* a, size_t threshold_n) {
  size_t n = a->n;
  if (n <= 1) return 0;
  if (threshold_n >= n) return pso_hs_segment(a, 0, n);
  unsigned levels = pso_log2_exact(n);
  unsigned dstar = levels - pso_log2_exact(threshold_n);
  size_t off[65];
  memset(off, 0, sizeof off);
  size_t total = 0;
  for (unsigned d = 1; d <= dstar; ++d) {
    off[d] = total;
    total += n >> d;
  }
  pso_handle arena;
  if (pso_make_like(a, total, &arena)) return -1;
  for (unsigned d = 1; d <= dstar; ++d) {
    size_t dst_off = off[d], src_off = d == 1 ? 0 : off[d - 1];
    pso_handle* src = d == 1 ? a : &arena;
    pso_launch_begin();
    for (size_t m = 0; m < (n >> d); ++m)
      pso_hcombine(&arena, dst_off + m, src, src_off + 2 * m, src,
                   src_off + 2 * m + 1);
    pso_launch_end();
  }
  if (pso_hs_segment(&arena, off[dstar], n >> dstar)) {
    free(arena.data);
    return -1;
  }
  for (unsigned d = dstar; d-- > 0;) {
    size_t dst_off = d == 0 ? 0 : off[d], par_off = off[d + 1];
    pso_handle* dst = d == 0 ? a : &arena;
    pso_launch_begin();
    for (size_t m = 0; m < (n >> d); ++m) {
      if (m == 0) continue;
      if ((m & 1) == 0)
        pso_hcombine(dst, dst_off + m, &arena, par_off + m / 2 - 1, dst,
                     dst_off + m);
      else
        pso_hassign(dst, dst_off + m, &arena, par_off + (m - 1) / 2);
    }
    pso_launch_end();
  }
  free(arena.data);
  return 0;
}

/* scan.hpp:450-483 (+ scan_reverse 486-490 through h->rev) */
static int pso_scan_forward(int alg, size_t sengupta_n, pso_handle* a) {
  size_t n = a->n;
  g_pso_work = g_pso_span = 0;
  if (n == 0) return 2; /* ContractViolation: scan of empty series */
  if (n == 1) return 0;
  if (alg == 0) {
    pso_seq(a);
    return 0;
  }
  if (!pso_is_pow2(n)) return 2;
  switch (alg) {
    case 1: return pso_hs_segment(a, 0, n) ? 8 : 0;
    case 2: return pso_blelloch(a) ? 8 : 0;
    case 3: pso_lafi(a); return 0;
    case 4: return pso_sengupta(a, 1) ? 8 : 0;
    case 5:
      if (sengupta_n < 2 || !pso_is_pow2(sengupta_n)) return 2;
      return pso_sengupta(a, sengupta_n) ? 8 : 0;
    default: return 2;
  }
}

#endif
