// kog2_gen.cuh — counter-based random-matrix generator on the device.
// generate<T>(cfg, index) of /root/reference/proj/include/kogsvd2/harness.hpp
// (lines 114-186) bit for bit, plus the KOG_REGIME_RANGED extension used for
// BASELINE configs 2-5 (include/kog2.h documents the rule).
#pragma once

#include "kog2_svd2.cuh"

namespace kog2 {

// mix64 (harness.hpp:114-118)
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Stream (harness.hpp:120-128)
struct Stream {
  unsigned long long s;
  __device__ __forceinline__ Stream(unsigned long long seed, unsigned long long index)
      : s(mix64(seed + 0x9e3779b97f4a7c15ull * (index + 1))) {}
  __device__ __forceinline__ unsigned long long next() {
    s += 0x9e3779b97f4a7c15ull;
    return mix64(s);
  }
};

// u % m, the reference's 64-bit modulo (harness.hpp:152), without a 64-bit
// division: with M = floor((2^64 - 1) / m) (precomputed on the host),
// 2^64/m - 1 <= M < 2^64/m, so q~ = floor(u M / 2^64) is floor(u/m) or one
// less and u - q~ m lies in [0, 2m): one conditional subtraction is exact
struct UMod {
  unsigned long long m, magic;
};
inline UMod umod_of(unsigned long long m) { return UMod{m, m ? ~0ull / m : 0ull}; }
__device__ __forceinline__ unsigned long long umod(unsigned long long u, const UMod& d) {
  const unsigned long long r = u - __umul64hi(u, d.magic) * d.m;
  return r >= d.m ? r - d.m : r;
}

// POD mirror of the generator fields of kog_run_config, passed by value, with
// the ranged draw's exponent window resolved for T (harness.hpp:157-166)
struct GenCfg {
  unsigned long long seed;
  int shape, regime;
  int lo, hi;  // bullet [e_mu, e_nu - 2], sigma [e_mu + varsigma, e_nu - 2], ranged [elo, ehi]
  UMod range;  // hi - lo + 1
  int tail_lo, tail_hi;
  UMod tail_range, tail_mod;
  unsigned zero_mask_rule;
};

template <class T>
inline GenCfg gen_cfg_of(const kog_run_config* c) {
  GenCfg g;
  g.seed = c->seed;
  g.shape = c->shape;
  g.regime = c->regime;
  g.lo = c->regime == KOG_REGIME_BULLET  ? FP<T>::emin
         : c->regime == KOG_REGIME_SIGMA ? FP<T>::emin + c->varsigma
                                         : c->elo;
  g.hi = c->regime == KOG_REGIME_RANGED ? c->ehi : FP<T>::emax - 2;
  g.range = umod_of(static_cast<unsigned long long>(g.hi - g.lo + 1));
  g.tail_lo = c->tail_lo;
  g.tail_hi = c->tail_hi;
  g.tail_range = umod_of(static_cast<unsigned long long>(c->tail_hi - c->tail_lo + 1));
  g.tail_mod = umod_of(c->tail_mod);
  g.zero_mask_rule = c->zero_mask_rule;
  return g;
}

template <class T>
__device__ __forceinline__ T gen_ranged(Stream& st, int elo, const UMod& range) {  // harness.hpp:150-156
  constexpr int p = FP<T>::p;
  const unsigned long long u = st.next();
  const int e = elo + static_cast<int>(umod(u, range));
  const T f = T(1) + scalbn_t(static_cast<T>(st.next() >> (64 - (p - 1))), 1 - p);
  const T v = scalbn_t(f, e);
  return (u >> 63) ? -v : v;
}

template <class T>
__device__ __forceinline__ T gen_circ(Stream& st) {  // harness.hpp:145-149
  const unsigned long long u = st.next();
  const T m = static_cast<T>(static_cast<double>(u >> 11) * 0x1p-53);
  return (u & 1) ? -m : m;
}

template <class T>
__device__ __forceinline__ T gen_element(Stream& st, const GenCfg& c) {  // harness.hpp:157-166
  if (c.regime == KOG_REGIME_CIRC) return gen_circ<T>(st);
  if (c.regime == KOG_REGIME_RANGED && c.tail_mod.m != 0) {
    const unsigned long long t = st.next();
    if (umod(t, c.tail_mod) == 0) return gen_ranged<T>(st, c.tail_lo, c.tail_range);
  }
  return gen_ranged<T>(st, c.lo, c.range);  // bullet, sigma, ranged
}

template <class T>
__device__ __forceinline__ T gen_nonzero(Stream& st, const GenCfg& c) {  // harness.hpp:167-171
  T v = gen_element<T>(st, c);
  while (v == T(0)) v = gen_element<T>(st, c);
  return v;
}

// generate<T> (harness.hpp:139-186) + zero-mask extension
template <class T>
__device__ __forceinline__ Mat<T> generate(const GenCfg& c, unsigned long long index) {
  Stream st(c.seed, index);
  Mat<T> g;
  if (c.shape == KOG_SHAPE_TRI) {
    g.g11 = gen_nonzero<T>(st, c);
    g.g12 = gen_element<T>(st, c);
    g.g21 = T(0);
    g.g22 = gen_nonzero<T>(st, c);
  } else {
    g.g11 = gen_element<T>(st, c);
    g.g12 = gen_element<T>(st, c);
    g.g21 = gen_element<T>(st, c);
    g.g22 = gen_element<T>(st, c);
  }
  if (c.regime == KOG_REGIME_RANGED && c.zero_mask_rule) {
    const unsigned long long z = st.next();
    if ((z & 7) == 0) {
      const unsigned m = static_cast<unsigned>(z >> 3) & 15u;
      if (m & 1) g.g11 = T(0);
      if (m & 2) g.g21 = T(0);
      if (m & 4) g.g12 = T(0);
      if (m & 8) g.g22 = T(0);
    }
  }
  return g;
}

}  // namespace kog2
