// kog2_lean.cuh — the "separated" case of svd2's t' = 15 route (binary64,
// default Options), where every hypot and secant of the reference's sequence
// (svd2.hpp:339-384 urv15, 438-474 tri_svd, 485-515 compose_left) takes its
// own early-out and most quotients are divisions by 1.
//
// On inputs whose exponents are spread over hundreds of binades (configs 3
// and 5: e uniform in [-500, 500]) about 90% of the full matrices are like
// this: the two entries of the pivot column lie 28 binades or more apart (the
// other column's too, or it is clearly the smaller one), so do r11 and r12,
// and tan(2 phi), tan(psi) and the composed tangent are below 2^-27.  Then,
// with the same bits as the reference:
//   * hypot_cr(a, b) = max(|a|, |b|) (fpcore.hpp:150 and hypot_args, kog2_fp.cuh);
//   * sec(theta) = sec(phi) = sec(psi) = sec(chi) = hypot_cr(t, 1) = 1 for |t| < 2^-27
//     (1 <= sqrt(1 + t^2) < 1 + 2^-55, half an ulp of 1 is 2^-53), so every x / sec
//     is x / 1 = x, cos = 1 / 1 = 1 and sin = tan;
//   * tan(phi) = tan(2 phi) / (1 + 1) = RN(tan(2 phi) / 2) (fpcore.hpp:192-196);
//   * sec(phi) / sec(psi) = 1 as a pair (0, 1.0): sigma1 = r11 / 1 and sigma2 = r22 * 1
//     are the pairs of r11 and r22 themselves (epair.hpp:79-88), and r11 > r22
//     means no sigma exchange;
//   * compose_left's denominator fma(-+tan(phi), tan(theta), 1) is exactly 1
//     (|tan(phi) tan(theta)| < 2^-55), so tan(chi) = (tan(phi) +- tan(theta)) / 1.
// What is left is the pivoting, tan(theta) = a21 / a11, the fma element, the
// wide-channel element (wide_dot2_div without its division by sec(theta) = 1),
// tan(2 phi) on pairs, tan(psi) = t / r11 — three quotients by a11 = r11 on one
// shared reciprocal and one significand quotient.  Each condition is tested on
// the computed values; a lane that fails any of them (or meets anything the
// fast path defers) returns false and is recomputed by svd2_fast, so a lane
// that returns true went through exactly the reference's operation sequence.
#pragma once

#include "kog2_fast.cuh"

namespace kog2 {
namespace fast {

// -x on the integer pipe (the compiler's DADD -RZ, -x takes an FP64 issue slot)
__device__ __forceinline__ double neg_i(double x) { return sethi(x, hiw(x) ^ static_cast<int>(0x80000000u)); }
__device__ __forceinline__ bool below_2m27(double x) {  // 0 <= x < 2^-27 on a non-negative finite x
  return hiw(x) < 0x3e400000;
}

__device__ __forceinline__ bool svd2_lean(const Mat<double>& gi, Result<double>& out) {
  const int k11 = hiw(gi.g11), k12 = hiw(gi.g12), k21 = hiw(gi.g21), k22 = hiw(gi.g22);
  const int h11 = k11 & 0x7fffffff, h12 = k12 & 0x7fffffff, h21 = k21 & 0x7fffffff, h22 = k22 & 0x7fffffff;
  const int hmax = max(max(h11, h12), max(h21, h22)), hmin = min(min(h11, h12), min(h21, h22));
  // classify (classify.hpp:44-58): four normal nonzero entries (t = 15, s_type = 2)
  // and s = e_nu - e_G - 2 >= 0, so prescale (classify.hpp:67-78) is exact
  bool bad = hmin < 0x00100000 || hmax >= (2045 << 20);
  const int s = 2044 - (hmax >> 20);
  const int sh = s << 20;
  // urv15's column norms (svd2.hpp:343-344): the early-out of hypot_args (high
  // words 28 binades or more apart) — the norm is the column's larger entry
  const int d1 = h11 - h21, d2 = h12 - h22;
  // The pivot column's norm must be its larger entry.  The OTHER column's norm only decides the column
  // exchange (w1 < w2, svd2.hpp:345): a column whose entries lie within 28 binades of each other may stay if it
  // surely is not the pivot column — its correctly rounded norm is at most sqrt 2 (1 + 2^-53) times its larger
  // entry, and that is below the other column's larger entry (= norm) when the high words are 2^20 apart (a
  // factor 2 (1 - 2^-20) or more), so comparing the larger entries decides w1 < w2 as the norms would.
  const bool near1 = abs(d1) < (28 << 20), near2 = abs(d2) < (28 << 20);
  const int m1 = max(h11, h21), m2 = max(h12, h22);
  bad |= (near1 & (near2 | (m2 - m1 < (1 << 20)))) | (near2 & (m1 - m2 < (1 << 20)));  // (no short circuits: no branches)
  const bool lo1 = d1 < 0, lo2 = d2 < 0;  // the column's larger entry sits in row 1
  const bool col_swap = fabs(lo1 ? gi.g21 : gi.g11) < fabs(lo2 ? gi.g22 : gi.g12);
  // the pivot column (cx, cy) and the other one (ox, oy); row signs make the
  // pivot column positive, the row exchange brings its larger entry on top
  const double cx = col_swap ? gi.g12 : gi.g11, cy = col_swap ? gi.g22 : gi.g21;
  const double ox = col_swap ? gi.g11 : gi.g12, oy = col_swap ? gi.g21 : gi.g22;
  const int kcx = hiw(cx), kcy = hiw(cy);
  const int sr0 = kcx >> 31 | 1, sr1 = kcy >> 31 | 1;  // -1 for a negative entry, else 1
  const bool row_swap = col_swap ? lo2 : lo1;
  const double px = sethi(cx, (kcx & 0x7fffffff) + sh), py = sethi(cy, (kcy & 0x7fffffff) + sh);
  const double qx = sethi(ox, (hiw(ox) ^ (kcx & 0x80000000)) + sh), qy = sethi(oy, (hiw(oy) ^ (kcy & 0x80000000)) + sh);
  const double a11 = row_swap ? py : px, a21 = row_swap ? px : py;
  const double a12 = row_swap ? qy : qx, a22 = row_swap ? qx : qy;
  // tan(theta) = a21 / a11 < 2^-27 (the entries are 28 binades apart on their
  // high words: a21 / a11 <= 2^-28 (1 + 2^-20)), so sec(theta) = 1
  const DivBy da = div_prep(a11);
  bool ok;
  const double tth = div_rn_fast(a21, da, ok);
  bad |= !ok;
  const bool same = ((hiw(a12) ^ hiw(a22)) & 0x80000000) == 0;
  // the fma element: x / sec(theta) = x / 1
  const double fe = same ? fma(a22, tth, a12) : fma(-a12, tth, a22);
  // wide_dot2_div (svd2.hpp:281-321) of (A a11 + C a21) / a11 / 1, as wide_n
  double we;
  {
    const double A = same ? a22 : a12, C = same ? neg_i(a12) : a22;
    const int la = bexp(hiw(A)), lb = bexp(hiw(a11)), lc = bexp(hiw(C)), ld = bexp(hiw(a21));  // biased
    const int sa = la + lb, sb = lc + ld;
    const int scale = max(sa, sb);
    const double a1 = mant_n(A), c1 = mant_n(C);
    const double b1 = sethi(a11, (hiw(a11) & 0x800fffff) | ((1023 - (scale - sa)) << 20));
    const double d1m = sethi(a21, (hiw(a21) & 0x800fffff) | ((1023 - (scale - sb)) << 20));
    const bool za = scale - sa > 120, zc = scale - sb > 120;
    double p1, e1, p2, e2;
    two_prod(za ? 0.0 : a1, za ? 0.0 : b1, p1, e1);
    two_prod(zc ? 0.0 : c1, zc ? 0.0 : d1m, p2, e2);
    double s1, s2, t1, t2;
    two_sum(p1, p2, s1, s2);
    two_sum(e1, e2, t1, t2);
    s2 += t1;
    fast_two_sum(s1, s2, s1, s2);
    s2 += t2;
    fast_two_sum(s1, s2, s1, s2);
    // q1 = a11: its significand and reciprocal are da's
    const DivBy dq{static_cast<unsigned>(hiw(da.ym)), da.ym, da.r};
    const double h = div_rn_fast(s1, dq, ok);
    bad |= !ok;
    const double rem = fma(-h, da.ym, s1) + s2;
    const bool z = rem == 0.0;
    const double q = div_rn_fast(z ? da.ym : rem, dq, ok);
    bad |= !ok;
    const double qz = z ? __hiloint2double(hiw(rem) & 0x80000000, 0) : q;  // rem / qs, qs > 0
    // scale - kq in unbiased terms: (scale - 2046) - (lb - 1023)
    we = scal_n(h + qz, scale - lb - 1023, bad);
  }
  const double r12_raw = same ? fe : we, r22_raw = same ? we : fe;
  const bool minus = ((hiw(r12_raw) ^ hiw(r22_raw)) & 0x80000000) != 0;  // s22 < 0
  const double r11 = a11, r12 = fabs(r12_raw), r22 = fabs(r22_raw);
  // assemble_svd (svd2.hpp:547-598) without the diagonal exchange; tan2phi's
  // general branch (svd2.hpp:389-426) with hypot(r11, r12) = max(r11, r12)
  bad |= !(r11 > r22) || r12 == r22;
  const int hr11 = hiw(r11), hr12 = hiw(r12);
  bad |= abs(hr11 - hr12) < (28 << 20);
  const double h = hr11 < hr12 ? r12 : r11;
  const double zs = h + r22;
  bad |= zs > FP<double>::norm_max();
  const EPair<double> sum = ep_nz(0, zs);
  const EPair<double> dif = ep_n(0, h - r22, bad);
  const EPair<double> p12 = ep_n(0, r12, bad), p22 = ep_n(0, r22, bad);  // zero or subnormal elements leave
  EPair<double> num = ep_mul_n(p12, p22, bad);
  num.e += 1;
  const double t2f = ep_value_nz(ep_div_n(num, ep_mul_n(dif, sum, bad), bad));
  bad |= !below_2m27(t2f);
  const double tphi = t2f * 0.5;
  const double t = fma(r22, tphi, r12);
  const double tpsi = div_rn_fast(t, da, ok);
  bad |= !ok || !below_2m27(tpsi);
  // compose_left (svd2.hpp:485-515): tan_phi_bold = tan(phi)
  const double cnum = minus ? tphi - tth : tphi + tth;
  const double cden = fma(minus ? tphi : -tphi, tth, 1.0);
  const int hcn = hiw(cnum) & 0x7fffffff;
  bad |= cden != 1.0 || static_cast<unsigned>(hcn - 0x00100000) >= static_cast<unsigned>(0x3e400000 - 0x00100000);
  const double sn = cnum;  // tan(chi) / 1
  Mat<double> m{1.0, neg_i(sn), sn, 1.0};
  if (minus) m = Mat<double>{m.g11, m.g12, neg_i(m.g21), neg_i(m.g22)};
  if (row_swap) m = Mat<double>{m.g21, m.g22, m.g11, m.g12};
  out.u = Mat<double>{sgnmul(sr0, m.g11), sgnmul(sr0, m.g12), sgnmul(sr1, m.g21), sgnmul(sr1, m.g22)};
  const int s12 = hiw(r12_raw) >> 31 | 1;
  const SP vplus = sp_mul(col_swap ? sp_exchange() : sp_identity(), sp_row_signs(1, s12));
  out.v = apply_left(vplus, Mat<double>{1.0, neg_i(tpsi), tpsi, 1.0});
  out.sigma1 = EPair<double>{bexp(hr11) - 1023 - s, mant_n(r11)};
  out.sigma2 = EPair<double>{p22.e - s, p22.f};
  out.s = s;
  out.flags = (15u << KOG_F_TYPE_INIT_SHIFT) | (15u << KOG_F_TYPE_SCALED_SHIFT) | tr_path(KOG_PATH_URV15) |
              tr_t2p(KOG_T2P_GENERAL) | (col_swap ? KOG_F_URV_COL_SWAP : 0u) | (row_swap ? KOG_F_URV_ROW_SWAP : 0u) |
              (minus ? KOG_F_COMPOSE_MINUS : 0u);
  return !bad;
}

}  // namespace fast
}  // namespace kog2
