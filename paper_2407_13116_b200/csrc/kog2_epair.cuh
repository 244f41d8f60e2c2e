// kog2_epair.cuh — exponent-mantissa pairs 2^e * f on the device.
// Semantics: /root/reference/proj/include/kogsvd2/epair.hpp (cited per
// function).  Where the reference throws std::domain_error, the device code
// sets bit 0 of the caller's `err` word and returns the value the reference
// would have produced had the check been absent (callers report the bit).
#pragma once

#include "kog2_fp.cuh"

namespace kog2 {

// EPair<T> (epair.hpp:16-46)
template <class T>
struct EPair {
  int e;  // |e| < 2^30 on every path (sigma exponents lie in [-3171, 1024])
  T f;  // 0, or |f| in [1,2)
};

template <class T>
__device__ __forceinline__ EPair<T> ep_zero() {
  return EPair<T>{0, T(0)};
}

// EPair(ee, ff): normalising constructor (epair.hpp:23-36)
// zero / subnormal / non-finite mantissas (rare; out of line)
template <class T>
static __device__ __noinline__ EPair<T> ep_make_rare(int ee, T ff) {
  KOG2_RARE(5);
  if (ff == T(0) || !is_finite(ff)) return EPair<T>{0, T(0)};
  return EPair<T>{ee + ilogb_nz(ff), mant_nz(ff)};
}
__device__ __forceinline__ EPair<double> ep_make_(int ee, double ff, unsigned& err) {
  const int h = hiw(ff), e = bexp(h);
  if (normal_bexp(e)) return EPair<double>{ee + e - 1023, sethi(ff, (h & 0x800fffff) | 0x3ff00000)};
  if (ff == 0.0) return EPair<double>{0, 0.0};  // canonical zero
  if (e == 0x7ff) err |= 1u;  // the reference throws on a NaN/inf mantissa
  return ep_make_rare<double>(ee, ff);  // subnormal
}
// binary32: through the (always normal) double, without branches for zero and
// subnormal mantissas; NaN/inf set err (the reference throws)
__device__ __forceinline__ EPair<float> ep_make_(int ee, float ff, unsigned& err) {
  const int b = __float_as_int(ff);
  if (bexpf(b) == 0xff) err |= 1u;
  const bool z = (b & 0x7fffffff) == 0 || bexpf(b) == 0xff;
  return z ? EPair<float>{0, 0.0f} : EPair<float>{ee + ilogb_nz(ff), mant_nz(ff)};
}
template <class T>
__device__ __forceinline__ EPair<T> ep_make(int ee, T ff, unsigned& err) {
  return ep_make_(ee, ff, err);
}

// value() (epair.hpp:40)
template <class T>
__device__ __forceinline__ T ep_value(const EPair<T>& x) {
  return assemble(x.e, x.f);
}

// require_positive_finite (epair.hpp:49-53)
template <class T>
__device__ __forceinline__ void ep_require_positive_finite(T x, T y, unsigned& err) {
  if (!(x > T(0)) || !(y > T(0)) || !is_finite(x) || !is_finite(y)) err |= 1u;
}

// oplus (epair.hpp:56-64): overflow-avoiding addition of positive finite scalars
template <class T>
__device__ __forceinline__ EPair<T> oplus(T x, T y, unsigned& err) {
  ep_require_positive_finite(x, y, err);
  const T z = x + y;
  if (z <= FP<T>::norm_max()) return ep_make<T>(0, z, err);
  const T zh = T(0.5) * x + T(0.5) * y;
  return ep_make<T>(1, zh, err);
}

// ominus (epair.hpp:66-77): underflow-avoiding subtraction
template <class T>
__device__ __forceinline__ EPair<T> ominus(T x, T y, unsigned& err) {
  ep_require_positive_finite(x, y, err);
  if (x == y) return ep_zero<T>();
  const T z = x - y;
  if (fabs(z) >= FP<T>::norm_min()) return ep_make<T>(0, z, err);
  const int ex = static_cast<int>(split(x).e), ey = static_cast<int>(split(y).e);
  const int c = FP<T>::emin + FP<T>::p - 1 - (ex < ey ? ex : ey);
  const T zs = assemble(c, x) - assemble(c, y);
  return ep_make<T>(-c, zs, err);
}

// operator* (epair.hpp:79-82)
template <class T>
__device__ __forceinline__ EPair<T> ep_mul(const EPair<T>& x, const EPair<T>& y, unsigned& err) {
  return ep_make<T>(x.e + y.e, x.f * y.f, err);
}

// operator/ (epair.hpp:84-88)
template <class T>
__device__ __forceinline__ EPair<T> ep_div(const EPair<T>& x, const EPair<T>& y, unsigned& err) {
  if (y.f == T(0)) err |= 1u;
  return ep_make<T>(x.e - y.e, div_rn(x.f, y.f), err);
}

// abs / neg (epair.hpp:90-102)
template <class T>
__device__ __forceinline__ EPair<T> ep_abs(const EPair<T>& x) {
  return EPair<T>{x.e, fabs(x.f)};
}
template <class T>
__device__ __forceinline__ EPair<T> ep_neg(const EPair<T>& x) {
  return EPair<T>{x.e, -x.f};
}

// scale2 (epair.hpp:104-110): exact multiplication by 2^k
template <class T>
__device__ __forceinline__ EPair<T> scale2(int k, const EPair<T>& x) {
  EPair<T> r = x;
  if (r.f != T(0)) r.e += k;
  return r;
}

// recip (epair.hpp:112-116)
template <class T>
__device__ __forceinline__ EPair<T> ep_recip(const EPair<T>& x, unsigned& err) {
  if (x.f == T(0)) err |= 1u;
  return ep_make<T>(-x.e, T(1) / x.f, err);
}

// less (epair.hpp:118-127): strict value order on the fields
template <class T>
__device__ __forceinline__ bool ep_less(const EPair<T>& x, const EPair<T>& y) {
  const int sx = (x.f > T(0)) - (x.f < T(0));
  const int sy = (y.f > T(0)) - (y.f < T(0));
  if (sx != sy) return sx < sy;
  if (sx == 0) return false;
  if (x.e != y.e) return sx > 0 ? x.e < y.e : x.e > y.e;
  return x.f < y.f;
}

}  // namespace kog2
