// kog2_svd2.cuh — the enhanced 2x2 Kogbetliantz SVD on the device, one
// thread per matrix.  Semantics (operation sequence, branch structure, sign
// conventions) follow /root/reference/proj/include/kogsvd2/classify.hpp and
// svd2.hpp, cited per function; results are bit-identical to the reference.
#pragma once

#include "../../include/kog2.h"
#include "kog2_epair.cuh"

namespace kog2 {

// Matrix2<T> (classify.hpp:14-19), row-major g11, g12, g21, g22
template <class T>
struct Mat {
  T g11, g12, g21, g22;
};

template <class T>
__device__ __forceinline__ bool all_finite(const Mat<T>& g) {  // classify.hpp:21-25
  return is_finite(g.g11) && is_finite(g.g12) && is_finite(g.g21) && is_finite(g.g22);
}

// ------------------------------------------------------------------ classify
#define KOG2_EXP_SENTINEL (-9223372036854775807ll - 1)  // kExpSentinel (classify.hpp:27)

struct TypeInfo {  // classify.hpp:29-35
  unsigned t;
  int s_type;
  int s;
  long long e_G;
};

__device__ __forceinline__ int scale_type_of(unsigned t) {  // classify.hpp:37-42
  // {0,1,2,4,6,8,9} -> 0, 15 -> 2, the rest -> 1, as a 16-entry bit table
  if (t == 15) return 2;
  return ((0x0357u >> t) & 1u) ? 0 : 1;
}

// classify (classify.hpp:44-58); err bit 0 <- non-finite element
template <class T>
__device__ __forceinline__ TypeInfo classify(const Mat<T>& g, unsigned& err) {
  if (!all_finite(g)) err |= 1u;
  TypeInfo info;
  info.t = (g.g11 != T(0) ? 1u : 0u) | (g.g21 != T(0) ? 2u : 0u) | (g.g12 != T(0) ? 4u : 0u) |
           (g.g22 != T(0) ? 8u : 0u);
  info.s_type = scale_type_of(info.t);
  // e_G: max floor(lg|g_ij|) over the nonzero elements (iteration order is
  // irrelevant for a max)
  int eg = -0x7fffffff;
  if (g.g11 != T(0)) eg = max(eg, ilogb_nz(g.g11));
  if (g.g21 != T(0)) eg = max(eg, ilogb_nz(g.g21));
  if (g.g12 != T(0)) eg = max(eg, ilogb_nz(g.g12));
  if (g.g22 != T(0)) eg = max(eg, ilogb_nz(g.g22));
  info.e_G = info.t == 0 ? KOG2_EXP_SENTINEL : static_cast<long long>(eg);
  info.s = info.t == 0 ? 0 : FP<T>::emax - eg - info.s_type;
  return info;
}

// nonzero pattern only (the re-classification in svd2.hpp:616 reads .t)
template <class T>
__device__ __forceinline__ unsigned type_of(const Mat<T>& g) {
  return (g.g11 != T(0) ? 1u : 0u) | (g.g21 != T(0) ? 2u : 0u) | (g.g12 != T(0) ? 4u : 0u) |
         (g.g22 != T(0) ? 8u : 0u);
}

// prescale (classify.hpp:60-78)
template <class T>
__device__ __forceinline__ Mat<T> prescale(const Mat<T>& g, int s, bool& inexact) {
  Mat<T> gp{assemble(s, g.g11), assemble(s, g.g12), assemble(s, g.g21), assemble(s, g.g22)};
  inexact = false;
  if (s < 0)
    inexact = assemble(-s, gp.g11) != g.g11 || assemble(-s, gp.g12) != g.g12 ||
              assemble(-s, gp.g21) != g.g21 || assemble(-s, gp.g22) != g.g22;
  return gp;
}

// ----------------------------------------------------------------- SignPerm
// signed permutation (svd2.hpp:21-48): exactly one +-1 per row and column
struct SP {
  int m00, m01, m10, m11;
};
__device__ __forceinline__ SP sp_identity() { return SP{1, 0, 0, 1}; }
__device__ __forceinline__ SP sp_exchange() { return SP{0, 1, 1, 0}; }
__device__ __forceinline__ SP sp_row_signs(int s0, int s1) { return SP{s0, 0, 0, s1}; }
__device__ __forceinline__ SP sp_mul(const SP& a, const SP& b) {
  return SP{a.m00 * b.m00 + a.m01 * b.m10, a.m00 * b.m01 + a.m01 * b.m11,
            a.m10 * b.m00 + a.m11 * b.m10, a.m10 * b.m01 + a.m11 * b.m11};
}
__device__ __forceinline__ SP sp_t(const SP& a) { return SP{a.m00, a.m10, a.m01, a.m11}; }
template <class T>
__device__ __forceinline__ Mat<T> sp_mat(const SP& a) {  // as_matrix: zeros are +0
  return Mat<T>{T(a.m00), T(a.m01), T(a.m10), T(a.m11)};
}

// x * T(s) for s = +-1: exact; equal to a conditional sign flip on non-NaN x
__device__ __forceinline__ double sgnmul(int s, double x) {  // s = +-1: flip the sign bit
  return sethi(x, hiw(x) ^ (s & 0x80000000));
}
__device__ __forceinline__ float sgnmul(int s, float x) {
  return __int_as_float(__float_as_int(x) ^ (s & 0x80000000));
}

// apply_left (svd2.hpp:50-67): s * g, error-free.  Each row of s has one
// nonzero (+-1) entry: the source row and sign are selected, not branched on.
template <class T>
__device__ __forceinline__ Mat<T> apply_left(const SP& s, const Mat<T>& g) {
  const bool a0 = s.m00 != 0, a1 = s.m10 != 0;
  const int k0 = a0 ? s.m00 : s.m01, k1 = a1 ? s.m10 : s.m11;
  return Mat<T>{sgnmul(k0, a0 ? g.g11 : g.g21), sgnmul(k0, a0 ? g.g12 : g.g22), sgnmul(k1, a1 ? g.g11 : g.g21),
                sgnmul(k1, a1 ? g.g12 : g.g22)};
}

// apply_right (svd2.hpp:69-86): g * s, error-free (source column selected)
template <class T>
__device__ __forceinline__ Mat<T> apply_right(const Mat<T>& g, const SP& s) {
  const bool a0 = s.m00 != 0, a1 = s.m01 != 0;
  const int k0 = a0 ? s.m00 : s.m10, k1 = a1 ? s.m01 : s.m11;
  return Mat<T>{sgnmul(k0, a0 ? g.g11 : g.g12), sgnmul(k1, a1 ? g.g11 : g.g12), sgnmul(k0, a0 ? g.g21 : g.g22),
                sgnmul(k1, a1 ? g.g21 : g.g22)};
}

// Options (svd2.hpp:122-132).  Kernels pass either a compile-time constant
// (the default options: branches fold away) or the runtime value.
struct Opt {
  bool hcr;  // hypot_is_cr
  bool omd;  // ominus_for_d
  int wc;    // wide_channel: KOG_WIDE_WIDER_TYPE / KOG_WIDE_KAHAN_DET
};

// ------------------------------------------------------------- result + trace
struct Trace {  // BranchTrace (svd2.hpp:108-120), packed as in include/kog2.h
  unsigned bits;
};

template <class T>
struct Result {  // Svd2Result<T> (svd2.hpp:134-140)
  Mat<T> u, v;
  EPair<T> sigma1, sigma2;
  int s;
  unsigned flags;  // trace bits + KOG_F_DOMAIN_ERROR; sign bits added at store
};

__device__ __forceinline__ unsigned tr_path(unsigned p) { return p << KOG_F_PATH_SHIFT; }
__device__ __forceinline__ unsigned tr_t2p(unsigned b) { return b << KOG_F_T2P_SHIFT; }

// ------------------------------------------------------------ phase 1
// svd_simple (svd2.hpp:145-182): t' ~ 9, exact SVD by permutations and signs
template <class T>
__device__ __forceinline__ void svd_simple(const Mat<T>& a, int s, unsigned t, unsigned flags,
                                           Result<T>& out) {
  flags |= tr_path(KOG_PATH_SIMPLE);
  SP pu = sp_identity(), pv = sp_identity();
  if (t == 2 || t == 6) pu = sp_exchange();
  else if (t == 4) pv = sp_exchange();
  else if (t == 8) pu = pv = sp_exchange();
  Mat<T> d = apply_right(apply_left(sp_t(pu), a), pv);
  if (fabs(d.g11) < fabs(d.g22)) {
    pu = sp_mul(pu, sp_exchange());
    pv = sp_mul(pv, sp_exchange());
    d = apply_right(apply_left(sp_exchange(), d), sp_exchange());
  }
  const SP sg = sp_row_signs(sign_bit(d.g11) ? -1 : 1, sign_bit(d.g22) ? -1 : 1);
  out.u = sp_mat<T>(sp_mul(pu, sg));
  out.v = sp_mat<T>(pv);
  unsigned err = 0;
  out.sigma1 = scale2(-s, ep_make<T>(0, fabs(d.g11), err));
  out.sigma2 = scale2(-s, ep_make<T>(0, fabs(d.g22), err));
  out.s = s;
  out.flags = flags | (err ? KOG_F_DOMAIN_ERROR : 0u);
}

// Rot / rot_from_tan_sec (svd2.hpp:186-195)
template <class T>
__device__ __forceinline__ Mat<T> rot_mat(T tan, T sec) {
  const T c = div_rn(T(1), sec), s = div_rn(tan, sec);
  return Mat<T>{c, -s, s, c};
}

// svd_mono (svd2.hpp:199-244): t' ~ 3 or 5, one Givens rotation
template <class T>
__device__ __forceinline__ void svd_mono(const Mat<T>& gp, int s, unsigned t, unsigned flags,
                                         Result<T>& out) {
  unsigned err = 0;
  out.s = s;
  if (t == 3 || t == 12) {
    flags |= tr_path(KOG_PATH_MONO_COL);
    const SP pv = t == 12 ? sp_exchange() : sp_identity();
    Mat<T> a = apply_right(gp, pv);
    const SP su = sp_row_signs(sign_bit(a.g11) ? -1 : 1, sign_bit(a.g21) ? -1 : 1);
    a = apply_left(su, a);
    const bool swap = a.g11 < a.g21;
    const SP pu = swap ? sp_exchange() : sp_identity();
    a = apply_left(pu, a);
    const T tan = div_rn(a.g21, a.g11);
    const T sec = sec_from_tan(tan);
    const T sig1 = hypot_cr(a.g11, a.g21);
    const Mat<T> uth = rot_mat(tan, sec);
    out.u = apply_left(su, apply_left(pu, uth));
    out.v = sp_mat<T>(pv);
    out.sigma1 = scale2(-s, ep_make<T>(0, sig1, err));
  } else {
    flags |= tr_path(KOG_PATH_MONO_ROW);
    const SP pu = t == 10 ? sp_exchange() : sp_identity();
    Mat<T> a = apply_left(sp_t(pu), gp);
    const SP sv = sp_row_signs(sign_bit(a.g11) ? -1 : 1, sign_bit(a.g12) ? -1 : 1);
    a = apply_right(a, sv);
    const bool swap = a.g11 < a.g12;
    const SP pvo = swap ? sp_exchange() : sp_identity();
    a = apply_right(a, pvo);
    const T tan = div_rn(a.g12, a.g11);
    const T sec = sec_from_tan(tan);
    const T sig1 = hypot_cr(a.g11, a.g12);
    const Mat<T> vth = rot_mat(tan, sec);
    out.u = sp_mat<T>(pu);
    out.v = apply_left(sv, apply_left(pvo, vth));
    out.sigma1 = scale2(-s, ep_make<T>(0, sig1, err));
  }
  out.sigma2 = ep_zero<T>();
  out.flags = flags | (err ? KOG_F_DOMAIN_ERROR : 0u);
}

// ------------------------------------------------------------ phase 2
// triangularize13 (svd2.hpp:251-271): t' ~ 13, error-free positive triangle
template <class T>
struct Tri13 {
  Mat<T> r;
  SP uplus, vplus;
};
template <class T>
__device__ __forceinline__ Tri13<T> triangularize13(const Mat<T>& gp, unsigned t) {
  const bool row_swap = t == 14 || t == 11;
  const bool col_swap = t == 7 || t == 11;
  const SP pu = row_swap ? sp_exchange() : sp_identity();
  const SP pv = col_swap ? sp_exchange() : sp_identity();
  Mat<T> a = apply_right(apply_left(sp_t(pu), gp), pv);
  const int s11 = sign_bit(a.g11) ? -1 : 1;
  a = apply_left(sp_row_signs(s11, 1), a);
  const int s12 = sign_bit(a.g12) ? -1 : 1;
  a = apply_right(a, sp_row_signs(1, s12));
  const int s22 = sign_bit(a.g22) ? -1 : 1;
  a = apply_left(sp_row_signs(1, s22), a);
  return Tri13<T>{a, sp_mul(pu, sp_row_signs(s11, s22)), sp_mul(pv, sp_row_signs(1, s12))};
}

// wide_dot2_div (svd2.hpp:275-321): fl(FL(FL(ab+cd)/q1)/q2), FL >= 2p bits.
// All four factors and q1 are nonzero finite on every call site (t' = 15).
template <class T>
__device__ __forceinline__ T wide_dot2_div(T a, T b, T c, T d, T q1, T q2, int WC) {
  const int la = ilogb_nz(a), lb = ilogb_nz(b), lc = ilogb_nz(c), ld = ilogb_nz(d);
  const int sa = la + lb;
  const int sb = lc + ld;
  const int scale = sa > sb ? sa : sb;
  const int guard = WC == KOG_WIDE_KAHAN_DET ? FP<T>::p + 20 : 120;
  T a1 = scalbn_t(a, -la);
  T b1 = scalbn_t(b, -(lb + (scale - sa)));
  T c1 = scalbn_t(c, -lc);
  T d1 = scalbn_t(d, -(ld + (scale - sb)));
  if (scale - sa > guard) a1 = b1 = T(0);
  if (scale - sb > guard) c1 = d1 = T(0);
  const int kq = ilogb_nz(q1);
  const T qs = scalbn_t(q1, -kq);
  if (WC == KOG_WIDE_KAHAN_DET) {
    const T w = c1 * d1;
    const T e = fma(c1, d1, -w);
    const T f = fma(a1, b1, w);
    return div_rn(scalbn_t(div_rn(f + e, qs), scale - kq), q2);
  }
  if (FP<T>::p == 24) {
    const double num = static_cast<double>(a1) * static_cast<double>(b1) +
                       static_cast<double>(c1) * static_cast<double>(d1);
    return div_rn(scalbn_t(static_cast<T>(div_rn(num, static_cast<double>(qs))), scale - kq), q2);
  } else {
    double p1, e1, p2, e2;
    two_prod(static_cast<double>(a1), static_cast<double>(b1), p1, e1);
    two_prod(static_cast<double>(c1), static_cast<double>(d1), p2, e2);
    double s1, s2, t1, t2;
    two_sum(p1, p2, s1, s2);
    two_sum(e1, e2, t1, t2);
    s2 += t1;
    fast_two_sum(s1, s2, s1, s2);
    s2 += t2;
    fast_two_sum(s1, s2, s1, s2);
    const double qd = static_cast<double>(qs);
    const double h = div_rn(s1, qd);
    const double rem = fma(-h, qd, s1) + s2;
    return div_rn(static_cast<T>(scalbn_d(h + div_rn(rem, qd), scale - kq)), q2);
  }
}

// Urv15 (svd2.hpp:325-337)
template <class T>
struct Urv15 {
  bool col_swap, row_swap;
  int sr0, sr1;
  Mat<T> gppp;
  T tan_theta, sec_theta;
  T r11, r12_raw, r22_raw;
  int s12, s22;
  Mat<T> r;
  bool ext_is_r22;
  int next;  // 0 triangular, 1 diagonal, 2 row
};

// urv15 (svd2.hpp:339-384): fully pivoted URV of a matrix with no zeros
template <class T>
__device__ __forceinline__ Urv15<T> urv15(const Mat<T>& gp, const Opt& o) {
  Urv15<T> out;
  const T w1 = hypot_cr(gp.g11, gp.g21);
  const T w2 = hypot_cr(gp.g12, gp.g22);
  out.col_swap = w1 < w2;
  Mat<T> a = out.col_swap ? Mat<T>{gp.g12, gp.g11, gp.g22, gp.g21} : gp;
  const T w1p = out.col_swap ? w2 : w1;
  out.sr0 = sign_bit(a.g11) ? -1 : 1;
  out.sr1 = sign_bit(a.g21) ? -1 : 1;
  a = apply_left(sp_row_signs(out.sr0, out.sr1), a);
  out.row_swap = a.g11 < a.g21;
  if (out.row_swap) a = Mat<T>{a.g21, a.g22, a.g11, a.g12};
  out.gppp = a;

  out.tan_theta = div_rn(a.g21, a.g11);
  out.sec_theta = sec_from_tan(out.tan_theta);
  out.r11 = w1p;
  const bool same_sign = sign_bit(a.g12) == sign_bit(a.g22);
  if (same_sign) {
    out.r12_raw = div_rn(fma(a.g22, out.tan_theta, a.g12), out.sec_theta);
    out.r22_raw = wide_dot2_div<T>(a.g22, a.g11, -a.g12, a.g21, a.g11, out.sec_theta, o.wc);
    out.ext_is_r22 = true;
  } else {
    out.r22_raw = div_rn(fma(-a.g12, out.tan_theta, a.g22), out.sec_theta);
    out.r12_raw = wide_dot2_div<T>(a.g12, a.g11, a.g22, a.g21, a.g11, out.sec_theta, o.wc);
    out.ext_is_r22 = false;
  }
  out.s12 = 1;
  out.s22 = 1;
  out.r = Mat<T>{T(0), T(0), T(0), T(0)};
  if (out.r12_raw == T(0)) {
    out.next = 1;
    return out;
  }
  if (out.r22_raw == T(0)) {
    out.next = 2;
    return out;
  }
  out.s12 = sign_bit(out.r12_raw) ? -1 : 1;
  const T r22p = sgnmul(out.s12, out.r22_raw);
  out.s22 = sign_bit(r22p) ? -1 : 1;
  out.r = Mat<T>{out.r11, fabs(out.r12_raw), T(0), fabs(out.r22_raw)};
  out.next = 0;
  return out;
}

// ------------------------------------------------------------ phase 3
// std::max(a, b) exactly: (a < b) ? b : a (keeps a on ties and NaN)
template <class T>
__device__ __forceinline__ T std_max(T a, T b) {
  return (a < b) ? b : a;
}

// tan2phi (svd2.hpp:389-426), Alg. 1; rt.g11 >= rt.g22 > 0, rt.g12 > 0
template <class T>
__device__ __forceinline__ T tan2phi(T r11, T r12, T r22, bool t13, const Opt& o, unsigned& branch,
                                     unsigned& err) {
  if (r11 == r22) {
    branch = KOG_T2P_DIAG_EQUAL;
    return div_rn(T(2) * r22, r12);
  }
  if (r12 == r22) {
    branch = KOG_T2P_OFFDIAG_EQUAL;
    const EPair<T> num = scale2(1, ep_mul(ep_make<T>(0, r12, err), ep_make<T>(0, r22, err), err));
    return ep_value(ep_div(num, ep_mul(ep_make<T>(0, r11, err), ep_make<T>(0, r11, err), err), err));
  }
  if (t13 && div_rn(r11, r12) < FP<T>::unit_roundoff()) {
    branch = KOG_T2P_SMALL_RATIO;
    return div_rn(T(2) * r22, r12);
  }
  if (!o.hcr) {
    branch = KOG_T2P_FALLBACK;
    if (r11 > r12) {
      const T x = div_rn(r12, r11), y = div_rn(r22, r11);
      return div_rn((T(2) * x) * y, std_max(fma(x - y, x + y, T(1)), T(0)));
    }
    const T x = div_rn(r11, r12), y = div_rn(r22, r12);
    return div_rn(T(2) * y, std_max(fma(x - y, x + y, T(1)), T(0)));
  }
  const T h = hypot_cr(r11, r12);
  if (h == r22) {
    branch = KOG_T2P_GENERAL_INF;
    return FP<T>::inf();
  }
  branch = KOG_T2P_GENERAL;
  const EPair<T> sum = oplus(h, r22, err);
  const EPair<T> dif = o.omd ? ominus(h, r22, err) : ep_make<T>(0, h - r22, err);
  const EPair<T> num = scale2(1, ep_mul(ep_make<T>(0, r12, err), ep_make<T>(0, r22, err), err));
  return ep_value(ep_div(num, ep_mul(dif, sum, err), err));
}

// TriSvd (svd2.hpp:428-436)
template <class T>
struct TriSvd {
  T tan_phi, sec_phi, cos_phi, sin_phi;
  T tan_psi, sec_psi, cos_psi, sin_psi;
  EPair<T> sig1, sig2;
  bool sigma_swapped, tanpsi_inf;
  unsigned t2p;
  T t2f;
};

// tri_svd (svd2.hpp:438-474), Alg. 2
template <class T>
__device__ __forceinline__ TriSvd<T> tri_svd(T r11, T r12, T r22, bool t13, const Opt& o, unsigned& err) {
  TriSvd<T> out;
  out.t2p = KOG_T2P_NONE;
  const T t2f = tan2phi<T>(r11, r12, r22, t13, o, out.t2p, err);
  out.t2f = t2f;
  out.tan_phi = tan_from_double_angle(t2f);
  out.sec_phi = sec_from_tan(out.tan_phi);
  out.cos_phi = div_rn(T(1), out.sec_phi);
  out.sin_phi = div_rn(out.tan_phi, out.sec_phi);

  const EPair<T> r11p = ep_make<T>(0, r11, err), r22p = ep_make<T>(0, r22, err);
  const T t = fma(r22, out.tan_phi, r12);
  out.tan_psi = div_rn(t, r11);
  if (is_inf(out.tan_psi)) {
    out.tanpsi_inf = true;
    const EPair<T> tp = ep_make<T>(0, t, err);
    const EPair<T> cos_pair = ep_div(r11p, tp, err);
    out.cos_psi = ep_value(cos_pair);
    out.sin_psi = T(1);
    out.sec_psi = FP<T>::inf();
    out.sig1 = tp;
    out.sig2 = ep_mul(r22p, cos_pair, err);
  } else {
    out.tanpsi_inf = false;
    out.sec_psi = sec_from_tan(out.tan_psi);
    out.cos_psi = div_rn(T(1), out.sec_psi);
    out.sin_psi = div_rn(out.tan_psi, out.sec_psi);
    const EPair<T> ratio = ep_div(ep_make<T>(0, out.sec_phi, err), ep_make<T>(0, out.sec_psi, err), err);
    out.sig1 = ep_div(r11p, ratio, err);
    out.sig2 = ep_mul(r22p, ratio, err);
  }
  out.sigma_swapped = false;
  if (ep_less(out.sig1, out.sig2)) {
    const EPair<T> tmp = out.sig1;
    out.sig1 = out.sig2;
    out.sig2 = tmp;
    out.sigma_swapped = true;
  }
  return out;
}

// compose_left (svd2.hpp:476-515): single-rotation form of the left factor
template <class T>
__device__ __forceinline__ void compose_left(T tan_phi_bold, T tan_theta, bool minus_form, T& rc,
                                             T& rs) {
  T tanchi;
  bool beyond_quarter;
  if (is_inf(tan_phi_bold)) {
    tanchi = div_rn(minus_form ? T(1) : T(-1), tan_theta);
    beyond_quarter = !minus_form;
  } else {
    const T num = minus_form ? tan_phi_bold - tan_theta : tan_phi_bold + tan_theta;
    const T den = minus_form ? fma(tan_phi_bold, tan_theta, T(1)) : fma(-tan_phi_bold, tan_theta, T(1));
    if (is_inf(den)) {
      const T q = div_rn(T(1), tan_theta);
      tanchi = sign_bit(den) ? -fabs(q) : fabs(q);  // std::copysign(1/tan_theta, den)
    } else {
      tanchi = div_rn(num, den);
    }
    beyond_quarter = !minus_form && den < T(0);
  }
  if (is_inf(tanchi)) {
    rc = T(0);
    rs = sign_bit(tanchi) ? T(-1) : T(1);
  } else {
    const T sec = sec_from_tan(tanchi);
    rc = div_rn(T(1), sec);
    rs = div_rn(tanchi, sec);
  }
  if (beyond_quarter) {
    rc = -rc;
    rs = -rs;
  }
}

// LeftFactor (svd2.hpp:537-545)
template <class T>
struct LeftFactor {
  bool composed;
  SP uplus;
  int sr0, sr1;
  bool row_swap;
  T tan_theta;
  int s22;
};

// assemble_svd (svd2.hpp:547-598)
template <class T>
__device__ __forceinline__ void assemble_svd(const Mat<T>& r, const LeftFactor<T>& left,
                                             const SP& vplus, int s, bool t13, const Opt& o,
                                             unsigned flags, Result<T>& out) {
  const bool diag_swap = r.g11 < r.g22;
  if (diag_swap) flags |= KOG_F_DIAG_SWAP;
  const T a11 = diag_swap ? r.g22 : r.g11;
  const T a22 = diag_swap ? r.g11 : r.g22;
  unsigned err = 0;
  const TriSvd<T> ts = tri_svd<T>(a11, r.g12, a22, t13, o, err);
  flags |= tr_t2p(ts.t2p);
  if (ts.tanpsi_inf) flags |= KOG_F_TANPSI_INF;
  if (ts.sigma_swapped) flags |= KOG_F_SIGMA_SWAP;

  const Mat<T> vrot = diag_swap ? Mat<T>{ts.sin_phi, ts.cos_phi, ts.cos_phi, -ts.sin_phi}
                                : Mat<T>{ts.cos_psi, -ts.sin_psi, ts.sin_psi, ts.cos_psi};
  Mat<T> v = apply_left(vplus, vrot);

  Mat<T> u;
  if (!left.composed) {
    const Mat<T> urot = diag_swap ? Mat<T>{ts.sin_psi, ts.cos_psi, ts.cos_psi, -ts.sin_psi}
                                  : Mat<T>{ts.cos_phi, -ts.sin_phi, ts.sin_phi, ts.cos_phi};
    u = apply_left(left.uplus, urot);
  } else {
    const T tan_phi_bold = diag_swap ? div_rn(T(1), ts.tan_psi) : ts.tan_phi;
    const bool minus_form = left.s22 < 0;
    if (minus_form) flags |= KOG_F_COMPOSE_MINUS;
    T cc, cs;
    compose_left(tan_phi_bold, left.tan_theta, minus_form, cc, cs);
    Mat<T> m{cc, -cs, cs, cc};
    if (diag_swap) m = Mat<T>{m.g11, -m.g12, m.g21, -m.g22};
    if (minus_form) m = Mat<T>{m.g11, m.g12, -m.g21, -m.g22};
    if (left.row_swap) m = Mat<T>{m.g21, m.g22, m.g11, m.g12};
    u = apply_left(sp_row_signs(left.sr0, left.sr1), m);
  }

  if (ts.sigma_swapped) {
    u = Mat<T>{u.g12, u.g11, u.g22, u.g21};
    v = Mat<T>{v.g12, v.g11, v.g22, v.g21};
  }
  out.u = u;
  out.v = v;
  out.sigma1 = scale2(-s, ts.sig1);
  out.sigma2 = scale2(-s, ts.sig2);
  out.s = s;
  out.flags = flags | (err ? KOG_F_DOMAIN_ERROR : 0u);
}

// svd2 driver (svd2.hpp:603-687)
template <class T>
__device__ __forceinline__ void svd2(const Mat<T>& g, const Opt& o, Result<T>& out) {
  unsigned err = 0;
  const TypeInfo info = classify(g, err);
  unsigned flags = (info.t << KOG_F_TYPE_INIT_SHIFT) | (err ? KOG_F_DOMAIN_ERROR : 0u);

  if (info.s_type == 0) {
    flags |= info.t << KOG_F_TYPE_SCALED_SHIFT;
    svd_simple(g, 0, info.t, flags, out);
    return;
  }

  bool inexact;
  const Mat<T> gp = prescale(g, info.s, inexact);
  if (inexact) flags |= KOG_F_PRESCALE_INEXACT;
  const unsigned t1 = type_of(gp);
  flags |= t1 << KOG_F_TYPE_SCALED_SHIFT;

  if (scale_type_of(t1) == 0) {
    svd_simple(gp, info.s, t1, flags, out);
    return;
  }
  if (t1 == 3 || t1 == 12 || t1 == 5 || t1 == 10) {
    svd_mono(gp, info.s, t1, flags, out);
    return;
  }
  // Both triangular routes (t' ~ 13 and the non-degenerate t' = 15) end in the
  // same assemble_svd (svd2.hpp:627, 647); it is called from one site here so
  // a warp mixing the two routes runs the triangular SVD once, converged.
  Mat<T> r;
  LeftFactor<T> left;
  SP vplus;
  bool t13;
  Urv15<T> urv;
  if (t1 != 15) {
    flags |= tr_path(KOG_PATH_TRI13);
    const Tri13<T> tri = triangularize13(gp, t1);
    r = tri.r;
    left.composed = false;
    left.uplus = tri.uplus;
    left.sr0 = left.sr1 = 1;
    left.row_swap = false;
    left.tan_theta = T(0);
    left.s22 = 1;
    vplus = tri.vplus;
    t13 = true;
    urv.next = 0;
  } else {
    urv = urv15<T>(gp, o);
    if (urv.col_swap) flags |= KOG_F_URV_COL_SWAP;
    if (urv.row_swap) flags |= KOG_F_URV_ROW_SWAP;
    flags |= tr_path(KOG_PATH_URV15);
    r = urv.r;
    left.composed = true;
    left.uplus = sp_identity();
    left.sr0 = urv.sr0;
    left.sr1 = urv.sr1;
    left.row_swap = urv.row_swap;
    left.tan_theta = urv.tan_theta;
    left.s22 = urv.s22;
    vplus = sp_mul(urv.col_swap ? sp_exchange() : sp_identity(), sp_row_signs(1, urv.s12));
    t13 = false;
  }
  if (urv.next == 0) {
    assemble_svd<T>(r, left, vplus, info.s, t13, o, flags, out);
    return;
  }

  // degenerate triangle (svd2.hpp:650-686)
  flags &= ~(7u << KOG_F_PATH_SHIFT);
  const SP pu = urv.row_swap ? sp_exchange() : sp_identity();
  const SP s1 = sp_row_signs(urv.sr0, urv.sr1);
  const SP pv = urv.col_swap ? sp_exchange() : sp_identity();
  const Mat<T> uth = rot_mat(urv.tan_theta, urv.sec_theta);
  const Mat<T> uleft = apply_left(s1, apply_left(pu, uth));
  out.s = info.s;
  if (urv.next == 1) {
    flags |= tr_path(KOG_PATH_URV15_TO_DIAG);
    T d1 = urv.r11, d2 = urv.r22_raw;
    const bool ord_swap = fabs(d1) < fabs(d2);
    if (ord_swap) {
      const T tmp = d1;
      d1 = d2;
      d2 = tmp;
    }
    const SP ps = ord_swap ? sp_exchange() : sp_identity();
    const SP sg = sp_row_signs(sign_bit(d1) ? -1 : 1, sign_bit(d2) ? -1 : 1);
    out.u = apply_right(apply_right(uleft, ps), sg);
    out.v = sp_mat<T>(sp_mul(pv, ps));
    out.sigma1 = scale2(-info.s, ep_make<T>(0, fabs(d1), err));
    out.sigma2 = scale2(-info.s, ep_make<T>(0, fabs(d2), err));
  } else {
    flags |= tr_path(KOG_PATH_URV15_TO_ROW);
    const SP sv2 = sp_row_signs(1, sign_bit(urv.r12_raw) ? -1 : 1);
    T a = urv.r11, b = fabs(urv.r12_raw);
    const bool ord_swap = a < b;
    if (ord_swap) {
      const T tmp = a;
      a = b;
      b = tmp;
    }
    const SP pvo = ord_swap ? sp_exchange() : sp_identity();
    const T tan = div_rn(b, a);
    const T sec = sec_from_tan(tan);
    const Mat<T> vth = rot_mat(tan, sec);
    out.u = uleft;
    out.v = apply_left(pv, apply_left(sv2, apply_left(pvo, vth)));
    out.sigma1 = scale2(-info.s, ep_make<T>(0, hypot_cr(urv.r11, urv.r12_raw), err));
    out.sigma2 = ep_zero<T>();
  }
  out.flags = flags | (err ? KOG_F_DOMAIN_ERROR : 0u);
}

}  // namespace kog2
