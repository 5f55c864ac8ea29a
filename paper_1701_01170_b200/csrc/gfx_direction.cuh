// Direction-optimisation arithmetic, bit-identical to the reference's Python
// floats (reference direction.py:52-70):
//   m_f = n_f * m / n
//   m_u = n_u * (mu_edge_based ? m : n) / (n - n_u)   (+inf when n_u >= n)
// Python evaluates int*int exactly and int/int as a correctly rounded true
// division; div_round() reproduces that for any operands whose product fits
// in 127 bits, so host and device replicas agree with CPython bit for bit.
#pragma once

#include <math.h>
#include <stdint.h>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

namespace gfx {

// correctly rounded (nearest-even) num/den for num >= 0, den > 0
__host__ __device__ inline double div_round(unsigned __int128 num, unsigned long long den) {
  if (num == 0) return 0.0;
  const unsigned __int128 two53 = (unsigned __int128)1 << 53;
  if (num < two53 && den < (1ull << 53)) return (double)(unsigned long long)num / (double)den;
  // bit lengths
  int la = 0;
  for (unsigned __int128 t = num; t; t >>= 1) ++la;
  int lb = 0;
  for (unsigned long long t = den; t; t >>= 1) ++lb;
  // choose k so that q = floor(num * 2^k / den) has 55 or 56 bits
  int k = 55 - (la - lb);
  unsigned __int128 a = num, b = den;
  if (k >= 0) a <<= k; else b <<= -k;
  unsigned __int128 q = a / b;
  unsigned __int128 r = a - q * b;
  // normalise q to exactly 55 bits (2 guard bits beyond 53)
  int extra = 0;
  while ((q >> 55) != 0) {  // q has > 55 bits
    if (q & 1) r = 1;       // fold into sticky
    q >>= 1;
    ++extra;
  }
  unsigned long long mant = (unsigned long long)(q >> 2);
  unsigned low2 = (unsigned)(q & 3);
  bool sticky = r != 0;
  if (low2 > 2 || (low2 == 2 && (sticky || (mant & 1)))) ++mant;
  return ldexp((double)mant, 2 - k + extra);
}

struct DirEstimate {
  double m_f, m_u;
};

__host__ __device__ inline DirEstimate estimate_mf_mu(long long n, long long m, long long n_f,
                                                      long long n_u, int mu_edge_based) {
  DirEstimate e;
  e.m_f = div_round((unsigned __int128)n_f * (unsigned long long)m, (unsigned long long)n);
  if (n_u >= n) {
    e.m_u = INFINITY;
  } else {
    unsigned long long num = mu_edge_based ? (unsigned long long)m : (unsigned long long)n;
    e.m_u = div_round((unsigned __int128)n_u * num, (unsigned long long)(n - n_u));
  }
  return e;
}

// mode: 0 push, 1 pull
__host__ __device__ inline int decide_direction(int mode, DirEstimate e, double do_a, double do_b) {
  if (mode == 0) return (e.m_f > e.m_u * do_a) ? 1 : 0;
  return (e.m_f < e.m_u * do_b) ? 0 : 1;
}

}  // namespace gfx
