// psk_plan.hpp -- host-side planner for level-by-level scans.
//
// Produces the sequence of levels (one kernel launch each) that the
// reference's scan kernels execute (scan.hpp:198-444), plus the sizes of the
// scratch buffers they need.  The same plan drives the exact path (over T
// elements, reference operation order) and the fast path's scan of chunk
// elements.  Contract checks mirror scan_forward (scan.hpp:450-483).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "psk_common.cuh"

namespace psk {

struct ScanPlan {
  std::vector<LevelDesc> levels;
  long long n = 0;        // logical size of buffer 0
  long long cap1 = 0;     // slots of buffer 1 (aux / orig / arena)
  long long cap2 = 0;     // slots of buffer 2 (tmp / HS aux inside Sengupta)
  int status = 0;         // 0 ok, 2 contract violation
  std::string why;
};

inline bool is_pow2(unsigned long long n) { return n && !(n & (n - 1)); }
inline unsigned long long next_pow2(unsigned long long n) {
  unsigned long long p = 1;
  while (p < n) p <<= 1;
  return p;
}
inline unsigned log2_exact(unsigned long long n) {
  unsigned l = 0;
  while ((1ull << l) < n) ++l;
  return l;
}

namespace plan_detail {
inline LevelDesc lv(int kind, int a, int b, int c, long long count,
                    long long p0 = 0, long long p1 = 0, long long p2 = 0) {
  LevelDesc d;
  d.kind = kind;
  d.bufA = a;
  d.bufB = b;
  d.bufC = c;
  d.count = count;
  d.p0 = p0;
  d.p1 = p1;
  d.p2 = p2;
  return d;
}
// scan.hpp:214-259: HS on [base, base+n) of buffer `buf`, ping-pong with
// buffer `aux` (>= n slots)
inline void hs_segment(ScanPlan& p, int buf, long long base, long long n,
                       int aux) {
  if (n <= 1) return;
  int cur = buf, nxt = aux;
  long long cb = base, nb = 0;
  const unsigned levels = log2_exact(n);
  for (unsigned d = 0; d < levels; ++d) {
    p.levels.push_back(lv(kLvHS, cur, nxt, 0, n, cb, nb, 1ll << d));
    std::swap(cur, nxt);
    std::swap(cb, nb);
  }
  if (cur != buf) p.levels.push_back(lv(kLvCopy, buf, cur, 0, n, base, cb));
}
inline void upsweep(ScanPlan& p, long long n) {
  const unsigned levels = log2_exact(n);
  for (unsigned d = 0; d < levels; ++d) {
    long long d1 = 1ll << d, d2 = d1 << 1;
    p.levels.push_back(lv(kLvUp, 0, 0, 0, n / d2, d1, d2));
  }
}
}  // namespace plan_detail

// alg: psk_alg values 0..5 (DLB is not level-by-level)
inline ScanPlan make_scan_plan(int alg, unsigned long long sengupta_n,
                               long long n) {
  using namespace plan_detail;
  ScanPlan p;
  p.n = n;
  if (n == 0) {
    p.status = 2;
    p.why = "scan of empty series";
    return p;
  }
  if (n == 1) return p;
  if (alg == 0) {
    p.levels.push_back(lv(kLvSeqChain, 0, 0, 0, n - 1));
    return p;
  }
  if (!is_pow2((unsigned long long)n)) {
    p.status = 2;
    p.why = "parallel scan length not a power of 2";
    return p;
  }
  switch (alg) {
    case 1:  // Hillis-Steele, scan.hpp:450-483 -> 214-259
      p.cap1 = n;
      hs_segment(p, 0, 0, n, 1);
      break;
    case 2: {  // Blelloch, scan.hpp:281-341
      const unsigned levels = log2_exact(n);
      p.cap1 = n;      // orig
      p.cap2 = n / 2;  // tmp
      p.levels.push_back(lv(kLvCopy, 1, 0, 0, n, 0, 0));
      upsweep(p, n);
      p.levels.push_back(lv(kLvIdentity, 0, 0, 0, 1, n - 1));
      for (unsigned d = levels; d-- > 0;) {
        long long d1 = 1ll << d, d2 = d1 << 1;
        p.levels.push_back(lv(kLvBlDown, 0, 2, 0, n / d2, d1, d2));
      }
      p.levels.push_back(lv(kLvBlFinal, 0, 1, 0, n));
      break;
    }
    case 3: {  // in-place Ladner-Fischer, scan.hpp:343-367
      const unsigned levels = log2_exact(n);
      upsweep(p, n);
      for (unsigned d = levels; d-- > 0;) {
        long long d1 = 1ll << d, d2 = d1 << 1, blocks = n / d2;
        if (blocks <= 1) continue;
        p.levels.push_back(lv(kLvLafiDown, 0, 0, 0, blocks - 1, d1, d2));
      }
      break;
    }
    case 4:
    case 5: {  // Sengupta hybrid, scan.hpp:369-444
      unsigned long long tn = 1;
      if (alg == 5) {
        tn = sengupta_n;
        if (tn < 2 || !is_pow2(tn)) {
          p.status = 2;
          p.why = "sengupta_n must be a power of 2, >= 2";
          return p;
        }
      }
      if (tn >= (unsigned long long)n) {
        p.cap1 = n;
        hs_segment(p, 0, 0, n, 1);
        break;
      }
      const unsigned levels = log2_exact(n);
      const unsigned dstar = levels - log2_exact(tn);
      std::vector<long long> off(dstar + 1, 0);
      long long total = 0;
      for (unsigned d = 1; d <= dstar; ++d) {
        off[d] = total;
        total += n >> d;
      }
      p.cap1 = total;  // arena
      for (unsigned d = 1; d <= dstar; ++d) {
        long long dst_off = off[d], src_off = d == 1 ? 0 : off[d - 1];
        int src = d == 1 ? 0 : 1;
        p.levels.push_back(
            lv(kLvSgReduce, 1, src, 0, n >> d, dst_off, src_off));
      }
      p.cap2 = n >> dstar;  // HS aux for the top segment
      hs_segment(p, 1, off[dstar], n >> dstar, 2);
      for (unsigned d = dstar; d-- > 0;) {
        long long dst_off = d == 0 ? 0 : off[d], par_off = off[d + 1];
        int dst = d == 0 ? 0 : 1;
        p.levels.push_back(lv(kLvSgDist, dst, 1, 0, n >> d, dst_off, par_off));
      }
      break;
    }
    default:
      p.status = 2;
      p.why = "unknown scan algorithm";
  }
  return p;
}

}  // namespace psk
