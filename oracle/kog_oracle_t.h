/*
 * TEST INFRASTRUCTURE ONLY.  Type-generic body of the C oracle, included by
 * kog_oracle.c once per working precision with
 *   T (double|float), SUF (f64|f32), KP (significand bits), KEMAX, KEMIN, KF32 (0|1).
 * Every function restates the reference routine it cites (paths relative to
 * /root/reference/proj/include/kogsvd2/); where the reference throws, the
 * restatement sets *err and continues.
 */
#define CAT2(a, b) a##_##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, SUF)

typedef struct {
  int64_t e;
  T f;
} FN(pair);
typedef struct {
  T g11, g12, g21, g22;
} FN(mat);

static T FN(norm_max)(void) { return KF32 ? (T)FLT_MAX : (T)DBL_MAX; }
static T FN(norm_min)(void) { return KF32 ? (T)FLT_MIN : (T)DBL_MIN; }
static T FN(uround)(void) { return KF32 ? (T)0x1p-24 : (T)0x1p-53; }
static T FN(scalbn)(T x, int n) { return KF32 ? (T)scalbnf((float)x, n) : (T)scalbn((double)x, n); }
static int FN(ilogb)(T x) { return KF32 ? ilogbf((float)x) : ilogb((double)x); }
static T FN(fma)(T a, T b, T c) { return KF32 ? (T)fmaf((float)a, (float)b, (float)c) : (T)fma(a, b, c); }
static T FN(sqrt)(T x) { return KF32 ? (T)sqrtf((float)x) : (T)sqrt((double)x); }
static T FN(fabs)(T x) { return KF32 ? (T)fabsf((float)x) : (T)fabs((double)x); }
static T FN(copysign)(T a, T b) { return KF32 ? (T)copysignf((float)a, (float)b) : (T)copysign(a, b); }

/* split (fpcore.hpp:41-47) */
static void FN(split)(T x, int64_t* e, T* f) {
  if (x == (T)0 || !isfinite(x)) {
    *e = 0;
    *f = x;
    return;
  }
  int be;
  const T fr = KF32 ? (T)frexpf((float)x, &be) : (T)frexp((double)x, &be);
  *e = (int64_t)be - 1;
  *f = fr + fr;
}

/* assemble (fpcore.hpp:51-55) */
static T FN(assemble)(int64_t e, T f) {
  const long ce = (long)(e < -100000 ? -100000 : (e > 100000 ? 100000 : e));
  return KF32 ? (T)scalblnf((float)f, ce) : (T)scalbln((double)f, ce);
}

/* hypot_cr (fpcore.hpp:140-188) */
static T FN(hypot)(T a, T b) {
  if (isinf(a) || isinf(b)) return (T)INFINITY;
  if (isnan(a) || isnan(b)) return a + b;
  T big = FN(fabs)(a), small = FN(fabs)(b);
  if (big < small) {
    const T t = big;
    big = small;
    small = t;
  }
  if (small == (T)0) return big;
  const int ea = FN(ilogb)(big), eb = FN(ilogb)(small);
  if (ea - eb >= KP + 2) return big;
  const double as = (double)FN(scalbn)(big, -ea), bs = (double)FN(scalbn)(small, -ea);
  double x1, x2, y1, y2;
  if (KF32) {
    x1 = as * as;
    y1 = bs * bs;
    x2 = y2 = 0.0;
  } else {
    ora_two_prod(as, as, &x1, &x2);
    ora_two_prod(bs, bs, &y1, &y2);
  }
  double s1, s2;
  ora_two_sum(x1, y1, &s1, &s2);
  const double slo = (x2 + y2) + s2;
  const double z0 = sqrt(s1);
  double zq, zqe;
  ora_two_prod(z0, z0, &zq, &zqe);
  const double resid = ((s1 - zq) - zqe) + slo;
  const double zdd = z0 + resid / (z0 + z0);
  const double s4[5] = {x1, x2, y1, y2, -4.0};
  const int cmp4 = ora_exact_sum_sign(s4, 5);
  const int tg_floor = (KEMIN - (KP - 1)) - ea;
  double zs;
  if (cmp4 == 0)
    zs = 2.0;
  else if (cmp4 < 0)
    zs = ora_round_sqrt_on_grid(x1, x2, y1, y2, zdd, tg_floor > (1 - KP) ? tg_floor : (1 - KP), 1.0, 2.0);
  else
    zs = ora_round_sqrt_on_grid(x1, x2, y1, y2, zdd, tg_floor > (2 - KP) ? tg_floor : (2 - KP), 2.0, 3.0);
  return FN(scalbn)((T)zs, ea);
}

/* tan_from_double_angle / sec_from_tan (fpcore.hpp:190-201) */
static T FN(tan2)(T t2) {
  if (isinf(t2)) return FN(copysign)((T)1, t2);
  return t2 / ((T)1 + FN(hypot)(t2, (T)1));
}
static T FN(sec)(T t) { return FN(hypot)(t, (T)1); }

/* EPair constructor (epair.hpp:23-36) */
static FN(pair) FN(pmake)(int64_t ee, T ff, int* err) {
  FN(pair) r = {0, (T)0};
  if (isnan(ff) || isinf(ff)) {
    *err = 1;
    return r;
  }
  if (ff == (T)0) return r;
  int64_t se;
  T sf;
  FN(split)(ff, &se, &sf);
  r.e = ee + se;
  r.f = sf;
  return r;
}
static T FN(pvalue)(FN(pair) x) { return FN(assemble)(x.e, x.f); }
static void FN(req_pos)(T x, T y, int* err) {
  if (!(x > (T)0) || !(y > (T)0) || !isfinite(x) || !isfinite(y)) *err = 1;
}
/* oplus / ominus (epair.hpp:56-77) */
static FN(pair) FN(oplus)(T x, T y, int* err) {
  FN(req_pos)(x, y, err);
  const T z = x + y;
  if (z <= FN(norm_max)()) return FN(pmake)(0, z, err);
  const T zh = (T)0.5 * x + (T)0.5 * y;
  return FN(pmake)(1, zh, err);
}
static FN(pair) FN(ominus)(T x, T y, int* err) {
  FN(pair) zero = {0, (T)0};
  FN(req_pos)(x, y, err);
  if (x == y) return zero;
  const T z = x - y;
  if (FN(fabs)(z) >= FN(norm_min)()) return FN(pmake)(0, z, err);
  int64_t ex, ey;
  T fx, fy;
  FN(split)(x, &ex, &fx);
  FN(split)(y, &ey, &fy);
  const int64_t c = KEMIN + KP - 1 - (ex < ey ? ex : ey);
  const T zs = FN(assemble)(c, x) - FN(assemble)(c, y);
  return FN(pmake)(-c, zs, err);
}
/* *, /, scale2, recip, less (epair.hpp:79-127) */
static FN(pair) FN(pmul)(FN(pair) x, FN(pair) y, int* err) { return FN(pmake)(x.e + y.e, x.f * y.f, err); }
static FN(pair) FN(pdiv)(FN(pair) x, FN(pair) y, int* err) {
  if (y.f == (T)0) {
    *err = 1;
    FN(pair) z = {0, (T)0};
    return z;
  }
  return FN(pmake)(x.e - y.e, x.f / y.f, err);
}
static FN(pair) FN(pscale2)(int64_t k, FN(pair) x) {
  if (x.f != (T)0) x.e += k;
  return x;
}
static FN(pair) FN(precip)(FN(pair) x, int* err) {
  if (x.f == (T)0) {
    *err = 1;
    return x;
  }
  return FN(pmake)(-x.e, (T)1 / x.f, err);
}
static int FN(pless)(FN(pair) x, FN(pair) y) {
  const int sx = (x.f > (T)0) - (x.f < (T)0);
  const int sy = (y.f > (T)0) - (y.f < (T)0);
  if (sx != sy) return sx < sy;
  if (sx == 0) return 0;
  if (x.e != y.e) return sx > 0 ? x.e < y.e : x.e > y.e;
  return x.f < y.f;
}

/* classify / prescale (classify.hpp:44-78) */
static int FN(all_finite)(FN(mat) g) {
  return isfinite(g.g11) && isfinite(g.g12) && isfinite(g.g21) && isfinite(g.g22);
}
static unsigned FN(pattern)(FN(mat) g) {
  return (g.g11 != (T)0 ? 1u : 0u) | (g.g21 != (T)0 ? 2u : 0u) | (g.g12 != (T)0 ? 4u : 0u) |
         (g.g22 != (T)0 ? 8u : 0u);
}
static ora_info FN(classify)(FN(mat) g, int* err) {
  ora_info info;
  if (!FN(all_finite)(g)) *err = 1;
  info.t = FN(pattern)(g);
  info.s_type = ora_scale_type(info.t);
  info.e_G = INT64_MIN;
  const T v[4] = {g.g11, g.g21, g.g12, g.g22};
  for (int k = 0; k < 4; ++k)
    if (v[k] != (T)0) {
      int64_t e;
      T f;
      FN(split)(v[k], &e, &f);
      if (info.e_G == INT64_MIN || e > info.e_G) info.e_G = e;
    }
  info.s = info.e_G == INT64_MIN ? 0 : KEMAX - info.e_G - info.s_type;
  return info;
}
static FN(mat) FN(prescale)(FN(mat) g, int64_t s, int* inexact) {
  FN(mat) r = {FN(assemble)(s, g.g11), FN(assemble)(s, g.g12), FN(assemble)(s, g.g21), FN(assemble)(s, g.g22)};
  *inexact = 0;
  if (s < 0)
    *inexact = FN(assemble)(-s, r.g11) != g.g11 || FN(assemble)(-s, r.g12) != g.g12 ||
               FN(assemble)(-s, r.g21) != g.g21 || FN(assemble)(-s, r.g22) != g.g22;
  return r;
}

/* signed permutations applied to matrices (svd2.hpp:50-86) */
static FN(mat) FN(left)(ora_sp s, FN(mat) g) {
  FN(mat) r;
  if (s.m[0][0] != 0) {
    r.g11 = (T)s.m[0][0] * g.g11;
    r.g12 = (T)s.m[0][0] * g.g12;
  } else {
    r.g11 = (T)s.m[0][1] * g.g21;
    r.g12 = (T)s.m[0][1] * g.g22;
  }
  if (s.m[1][0] != 0) {
    r.g21 = (T)s.m[1][0] * g.g11;
    r.g22 = (T)s.m[1][0] * g.g12;
  } else {
    r.g21 = (T)s.m[1][1] * g.g21;
    r.g22 = (T)s.m[1][1] * g.g22;
  }
  return r;
}
static FN(mat) FN(right)(FN(mat) g, ora_sp s) {
  FN(mat) r;
  if (s.m[0][0] != 0) {
    r.g11 = g.g11 * (T)s.m[0][0];
    r.g21 = g.g21 * (T)s.m[0][0];
  } else {
    r.g11 = g.g12 * (T)s.m[1][0];
    r.g21 = g.g22 * (T)s.m[1][0];
  }
  if (s.m[0][1] != 0) {
    r.g12 = g.g11 * (T)s.m[0][1];
    r.g22 = g.g21 * (T)s.m[0][1];
  } else {
    r.g12 = g.g12 * (T)s.m[1][1];
    r.g22 = g.g22 * (T)s.m[1][1];
  }
  return r;
}
static FN(mat) FN(spmat)(ora_sp s) {
  FN(mat) r = {(T)s.m[0][0], (T)s.m[0][1], (T)s.m[1][0], (T)s.m[1][1]};
  return r;
}
static FN(mat) FN(rot)(T tan, T sec) {  /* rot_from_tan_sec (svd2.hpp:192-195) */
  const T c = (T)1 / sec, s = tan / sec;
  FN(mat) r = {c, -s, s, c};
  return r;
}

typedef struct {
  FN(mat) u, v;
  FN(pair) s1, s2;
  int64_t s;
  uint32_t flags;
  int err;
} FN(res);

/* svd_simple (svd2.hpp:145-182) */
static void FN(simple)(FN(mat) a, int64_t s, unsigned t, uint32_t flags, FN(res) * out) {
  ora_sp pu = ora_sp_id(), pv = ora_sp_id();
  if (t == 2 || t == 6)
    pu = ora_sp_x();
  else if (t == 4)
    pv = ora_sp_x();
  else if (t == 8)
    pu = pv = ora_sp_x();
  FN(mat) d = FN(right)(FN(left)(ora_sp_t(pu), a), pv);
  if (FN(fabs)(d.g11) < FN(fabs)(d.g22)) {
    pu = ora_sp_mul(pu, ora_sp_x());
    pv = ora_sp_mul(pv, ora_sp_x());
    d = FN(right)(FN(left)(ora_sp_x(), d), ora_sp_x());
  }
  const ora_sp sg = ora_sp_rows(signbit(d.g11) ? -1 : 1, signbit(d.g22) ? -1 : 1);
  out->u = FN(spmat)(ora_sp_mul(pu, sg));
  out->v = FN(spmat)(pv);
  out->s1 = FN(pscale2)(-s, FN(pmake)(0, FN(fabs)(d.g11), &out->err));
  out->s2 = FN(pscale2)(-s, FN(pmake)(0, FN(fabs)(d.g22), &out->err));
  out->s = s;
  out->flags = flags | ((uint32_t)KOG_PATH_SIMPLE << KOG_F_PATH_SHIFT);
}

/* svd_mono (svd2.hpp:199-244) */
static void FN(mono)(FN(mat) gp, int64_t s, unsigned t, uint32_t flags, FN(res) * out) {
  FN(pair) zero = {0, (T)0};
  out->s = s;
  if (t == 3 || t == 12) {
    const ora_sp pv = t == 12 ? ora_sp_x() : ora_sp_id();
    FN(mat) a = FN(right)(gp, pv);
    const ora_sp su = ora_sp_rows(signbit(a.g11) ? -1 : 1, signbit(a.g21) ? -1 : 1);
    a = FN(left)(su, a);
    const ora_sp pu = a.g11 < a.g21 ? ora_sp_x() : ora_sp_id();
    a = FN(left)(pu, a);
    const T tan = a.g21 / a.g11;
    const T sec = FN(sec)(tan);
    const T sig1 = FN(hypot)(a.g11, a.g21);
    out->u = FN(left)(su, FN(left)(pu, FN(rot)(tan, sec)));
    out->v = FN(spmat)(pv);
    out->s1 = FN(pscale2)(-s, FN(pmake)(0, sig1, &out->err));
    out->flags = flags | ((uint32_t)KOG_PATH_MONO_COL << KOG_F_PATH_SHIFT);
  } else {
    const ora_sp pu = t == 10 ? ora_sp_x() : ora_sp_id();
    FN(mat) a = FN(left)(ora_sp_t(pu), gp);
    const ora_sp sv = ora_sp_rows(signbit(a.g11) ? -1 : 1, signbit(a.g12) ? -1 : 1);
    a = FN(right)(a, sv);
    const ora_sp pvo = a.g11 < a.g12 ? ora_sp_x() : ora_sp_id();
    a = FN(right)(a, pvo);
    const T tan = a.g12 / a.g11;
    const T sec = FN(sec)(tan);
    const T sig1 = FN(hypot)(a.g11, a.g12);
    out->u = FN(spmat)(pu);
    out->v = FN(left)(sv, FN(left)(pvo, FN(rot)(tan, sec)));
    out->s1 = FN(pscale2)(-s, FN(pmake)(0, sig1, &out->err));
    out->flags = flags | ((uint32_t)KOG_PATH_MONO_ROW << KOG_F_PATH_SHIFT);
  }
  out->s2 = zero;
}

/* triangularize13 (svd2.hpp:257-271) */
static void FN(tri13)(FN(mat) gp, unsigned t, FN(mat) * r, ora_sp* uplus, ora_sp* vplus) {
  const ora_sp pu = (t == 14 || t == 11) ? ora_sp_x() : ora_sp_id();
  const ora_sp pv = (t == 7 || t == 11) ? ora_sp_x() : ora_sp_id();
  FN(mat) a = FN(right)(FN(left)(ora_sp_t(pu), gp), pv);
  const int s11 = signbit(a.g11) ? -1 : 1;
  a = FN(left)(ora_sp_rows(s11, 1), a);
  const int s12 = signbit(a.g12) ? -1 : 1;
  a = FN(right)(a, ora_sp_rows(1, s12));
  const int s22 = signbit(a.g22) ? -1 : 1;
  a = FN(left)(ora_sp_rows(1, s22), a);
  *r = a;
  *uplus = ora_sp_mul(pu, ora_sp_rows(s11, s22));
  *vplus = ora_sp_mul(pv, ora_sp_rows(1, s12));
}

/* wide_dot2_div (svd2.hpp:281-321) */
static T FN(wide)(T a, T b, T c, T d, T q1, T q2, int kahan) {
  const int sa = FN(ilogb)(a) + FN(ilogb)(b);
  const int sb = FN(ilogb)(c) + FN(ilogb)(d);
  const int scale = sa > sb ? sa : sb;
  const int guard = kahan ? KP + 20 : 120;
  T a1 = FN(scalbn)(a, -FN(ilogb)(a));
  T b1 = FN(scalbn)(b, -(FN(ilogb)(b) + (scale - sa)));
  T c1 = FN(scalbn)(c, -FN(ilogb)(c));
  T d1 = FN(scalbn)(d, -(FN(ilogb)(d) + (scale - sb)));
  if (scale - sa > guard) a1 = b1 = (T)0;
  if (scale - sb > guard) c1 = d1 = (T)0;
  const T qs = FN(scalbn)(q1, -FN(ilogb)(q1));
  const int kq = FN(ilogb)(q1);
  if (kahan) {
    const T w = c1 * d1;
    const T e = FN(fma)(c1, d1, -w);
    const T f = FN(fma)(a1, b1, w);
    return FN(scalbn)((f + e) / qs, scale - kq) / q2;
  }
  if (KF32) {
    const double num = (double)a1 * (double)b1 + (double)c1 * (double)d1;
    return FN(scalbn)((T)(num / (double)qs), scale - kq) / q2;
  } else {
    double p1, e1, p2, e2, s1, s2, t1, t2;
    ora_two_prod((double)a1, (double)b1, &p1, &e1);
    ora_two_prod((double)c1, (double)d1, &p2, &e2);
    ora_two_sum(p1, p2, &s1, &s2);
    ora_two_sum(e1, e2, &t1, &t2);
    s2 += t1;
    ora_fast_two_sum(s1, s2, &s1, &s2);
    s2 += t2;
    ora_fast_two_sum(s1, s2, &s1, &s2);
    const double h = s1 / (double)qs;
    const double rem = fma(-h, (double)qs, s1) + s2;
    return (T)scalbn(h + rem / (double)qs, scale - kq) / q2;
  }
}

typedef struct {
  int col_swap, row_swap, sr0, sr1, s12, s22, ext_is_r22, next;
  FN(mat) gppp, r;
  T tan_theta, sec_theta, r11, r12_raw, r22_raw;
} FN(urv);

/* urv15 (svd2.hpp:339-384) */
static FN(urv) FN(urv15)(FN(mat) gp, const kog_options* o) {
  FN(urv) u;
  memset(&u, 0, sizeof u);
  u.sec_theta = (T)1;
  const T w1 = FN(hypot)(gp.g11, gp.g21), w2 = FN(hypot)(gp.g12, gp.g22);
  u.col_swap = w1 < w2;
  FN(mat) a = gp;
  if (u.col_swap) {
    FN(mat) sw = {gp.g12, gp.g11, gp.g22, gp.g21};
    a = sw;
  }
  const T w1p = u.col_swap ? w2 : w1;
  u.sr0 = signbit(a.g11) ? -1 : 1;
  u.sr1 = signbit(a.g21) ? -1 : 1;
  a = FN(left)(ora_sp_rows(u.sr0, u.sr1), a);
  u.row_swap = a.g11 < a.g21;
  if (u.row_swap) {
    FN(mat) sw = {a.g21, a.g22, a.g11, a.g12};
    a = sw;
  }
  u.gppp = a;
  u.tan_theta = a.g21 / a.g11;
  u.sec_theta = FN(sec)(u.tan_theta);
  u.r11 = w1p;
  if (signbit(a.g12) == signbit(a.g22)) {
    u.r12_raw = FN(fma)(a.g22, u.tan_theta, a.g12) / u.sec_theta;
    u.r22_raw = FN(wide)(a.g22, a.g11, -a.g12, a.g21, a.g11, u.sec_theta, o->wide_channel);
    u.ext_is_r22 = 1;
  } else {
    u.r22_raw = FN(fma)(-a.g12, u.tan_theta, a.g22) / u.sec_theta;
    u.r12_raw = FN(wide)(a.g12, a.g11, a.g22, a.g21, a.g11, u.sec_theta, o->wide_channel);
    u.ext_is_r22 = 0;
  }
  u.s12 = u.s22 = 1;
  if (u.r12_raw == (T)0) {
    u.next = 1;
    return u;
  }
  if (u.r22_raw == (T)0) {
    u.next = 2;
    return u;
  }
  u.s12 = signbit(u.r12_raw) ? -1 : 1;
  u.s22 = signbit((T)u.s12 * u.r22_raw) ? -1 : 1;
  FN(mat) r = {u.r11, FN(fabs)(u.r12_raw), (T)0, FN(fabs)(u.r22_raw)};
  u.r = r;
  u.next = 0;
  return u;
}

/* tan2phi (svd2.hpp:389-426) */
static T FN(tan2phi)(T r11, T r12, T r22, int t13, const kog_options* o, unsigned* br, int* err) {
  if (r11 == r22) {
    *br = KOG_T2P_DIAG_EQUAL;
    return ((T)2 * r22) / r12;
  }
  if (r12 == r22) {
    *br = KOG_T2P_OFFDIAG_EQUAL;
    const FN(pair) num = FN(pscale2)(1, FN(pmul)(FN(pmake)(0, r12, err), FN(pmake)(0, r22, err), err));
    return FN(pvalue)(FN(pdiv)(num, FN(pmul)(FN(pmake)(0, r11, err), FN(pmake)(0, r11, err), err), err));
  }
  if (t13 && r11 / r12 < FN(uround)()) {
    *br = KOG_T2P_SMALL_RATIO;
    return ((T)2 * r22) / r12;
  }
  if (!o->hypot_is_cr) {
    *br = KOG_T2P_FALLBACK;
    T x, y, den;
    if (r11 > r12) {
      x = r12 / r11;
      y = r22 / r11;
      den = FN(fma)(x - y, x + y, (T)1);
      den = den < (T)0 ? (T)0 : den; /* std::max(den, 0) */
      return (((T)2 * x) * y) / den;
    }
    x = r11 / r12;
    y = r22 / r12;
    den = FN(fma)(x - y, x + y, (T)1);
    den = den < (T)0 ? (T)0 : den;
    return ((T)2 * y) / den;
  }
  const T h = FN(hypot)(r11, r12);
  if (h == r22) {
    *br = KOG_T2P_GENERAL_INF;
    return (T)INFINITY;
  }
  *br = KOG_T2P_GENERAL;
  const FN(pair) sum = FN(oplus)(h, r22, err);
  const FN(pair) dif = o->ominus_for_d ? FN(ominus)(h, r22, err) : FN(pmake)(0, h - r22, err);
  const FN(pair) num = FN(pscale2)(1, FN(pmul)(FN(pmake)(0, r12, err), FN(pmake)(0, r22, err), err));
  return FN(pvalue)(FN(pdiv)(num, FN(pmul)(dif, sum, err), err));
}

typedef struct {
  T tan_phi, sec_phi, cos_phi, sin_phi, tan_psi, sec_psi, cos_psi, sin_psi, t2f;
  FN(pair) sig1, sig2;
  int sigma_swapped, tanpsi_inf;
  unsigned t2p;
} FN(tri);

/* tri_svd (svd2.hpp:438-474) */
static FN(tri) FN(tri_svd)(T r11, T r12, T r22, int t13, const kog_options* o, int* err) {
  FN(tri) out;
  memset(&out, 0, sizeof out);
  out.t2p = KOG_T2P_NONE;
  out.t2f = FN(tan2phi)(r11, r12, r22, t13, o, &out.t2p, err);
  out.tan_phi = FN(tan2)(out.t2f);
  out.sec_phi = FN(sec)(out.tan_phi);
  out.cos_phi = (T)1 / out.sec_phi;
  out.sin_phi = out.tan_phi / out.sec_phi;
  const FN(pair) r11p = FN(pmake)(0, r11, err), r22p = FN(pmake)(0, r22, err);
  const T t = FN(fma)(r22, out.tan_phi, r12);
  out.tan_psi = t / r11;
  if (isinf(out.tan_psi)) {
    out.tanpsi_inf = 1;
    const FN(pair) tp = FN(pmake)(0, t, err);
    const FN(pair) cp = FN(pdiv)(r11p, tp, err);
    out.cos_psi = FN(pvalue)(cp);
    out.sin_psi = (T)1;
    out.sec_psi = (T)INFINITY;
    out.sig1 = tp;
    out.sig2 = FN(pmul)(r22p, cp, err);
  } else {
    out.sec_psi = FN(sec)(out.tan_psi);
    out.cos_psi = (T)1 / out.sec_psi;
    out.sin_psi = out.tan_psi / out.sec_psi;
    const FN(pair) ratio = FN(pdiv)(FN(pmake)(0, out.sec_phi, err), FN(pmake)(0, out.sec_psi, err), err);
    out.sig1 = FN(pdiv)(r11p, ratio, err);
    out.sig2 = FN(pmul)(r22p, ratio, err);
  }
  if (FN(pless)(out.sig1, out.sig2)) {
    const FN(pair) tmp = out.sig1;
    out.sig1 = out.sig2;
    out.sig2 = tmp;
    out.sigma_swapped = 1;
  }
  return out;
}

/* compose_left (svd2.hpp:485-515) */
static void FN(compose)(T tpb, T tth, int minus, T* rc, T* rs) {
  T tanchi;
  int beyond;
  if (isinf(tpb)) {
    tanchi = (minus ? (T)1 : (T)-1) / tth;
    beyond = !minus;
  } else {
    const T num = minus ? tpb - tth : tpb + tth;
    const T den = minus ? FN(fma)(tpb, tth, (T)1) : FN(fma)(-tpb, tth, (T)1);
    tanchi = isinf(den) ? FN(copysign)((T)1 / tth, den) : num / den;
    beyond = !minus && den < (T)0;
  }
  T c, s;
  if (isinf(tanchi)) {
    c = (T)0;
    s = FN(copysign)((T)1, tanchi);
  } else {
    const T sec = FN(sec)(tanchi);
    c = (T)1 / sec;
    s = tanchi / sec;
  }
  if (beyond) {
    c = -c;
    s = -s;
  }
  *rc = c;
  *rs = s;
}

/* assemble_svd (svd2.hpp:547-598) */
static void FN(assemble_svd)(FN(mat) r, int composed, ora_sp uplus, int sr0, int sr1, int row_swap, T tan_theta,
                             int s22, ora_sp vplus, int64_t s, int t13, const kog_options* o, uint32_t flags,
                             FN(res) * out) {
  const int diag_swap = r.g11 < r.g22;
  if (diag_swap) flags |= KOG_F_DIAG_SWAP;
  const FN(tri) ts = diag_swap ? FN(tri_svd)(r.g22, r.g12, r.g11, t13, o, &out->err)
                               : FN(tri_svd)(r.g11, r.g12, r.g22, t13, o, &out->err);
  flags |= ts.t2p << KOG_F_T2P_SHIFT;
  if (ts.tanpsi_inf) flags |= KOG_F_TANPSI_INF;
  if (ts.sigma_swapped) flags |= KOG_F_SIGMA_SWAP;
  FN(mat) vrot;
  if (diag_swap) {
    FN(mat) m = {ts.sin_phi, ts.cos_phi, ts.cos_phi, -ts.sin_phi};
    vrot = m;
  } else {
    FN(mat) m = {ts.cos_psi, -ts.sin_psi, ts.sin_psi, ts.cos_psi};
    vrot = m;
  }
  FN(mat) v = FN(left)(vplus, vrot), u;
  if (!composed) {
    FN(mat) urot;
    if (diag_swap) {
      FN(mat) m = {ts.sin_psi, ts.cos_psi, ts.cos_psi, -ts.sin_psi};
      urot = m;
    } else {
      FN(mat) m = {ts.cos_phi, -ts.sin_phi, ts.sin_phi, ts.cos_phi};
      urot = m;
    }
    u = FN(left)(uplus, urot);
  } else {
    const T tpb = diag_swap ? (T)1 / ts.tan_psi : ts.tan_phi;
    const int minus = s22 < 0;
    if (minus) flags |= KOG_F_COMPOSE_MINUS;
    T cc, cs;
    FN(compose)(tpb, tan_theta, minus, &cc, &cs);
    FN(mat) m = {cc, -cs, cs, cc};
    if (diag_swap) {
      m.g12 = -m.g12;
      m.g22 = -m.g22;
    }
    if (minus) {
      m.g21 = -m.g21;
      m.g22 = -m.g22;
    }
    if (row_swap) m = FN(left)(ora_sp_x(), m);
    u = FN(left)(ora_sp_rows(sr0, sr1), m);
  }
  if (ts.sigma_swapped) {
    FN(mat) uu = {u.g12, u.g11, u.g22, u.g21}, vv = {v.g12, v.g11, v.g22, v.g21};
    u = uu;
    v = vv;
  }
  out->u = u;
  out->v = v;
  out->s1 = FN(pscale2)(-s, ts.sig1);
  out->s2 = FN(pscale2)(-s, ts.sig2);
  out->s = s;
  out->flags = flags;
}

/* svd2 driver (svd2.hpp:603-687) */
static FN(res) FN(svd2)(FN(mat) g, const kog_options* o) {
  FN(res) out;
  memset(&out, 0, sizeof out);
  const ora_info info = FN(classify)(g, &out.err);
  uint32_t flags = info.t << KOG_F_TYPE_INIT_SHIFT;
  if (info.s_type == 0) {
    FN(simple)(g, 0, info.t, flags | (info.t << KOG_F_TYPE_SCALED_SHIFT), &out);
    return out;
  }
  int inexact;
  const FN(mat) gp = FN(prescale)(g, info.s, &inexact);
  if (inexact) flags |= KOG_F_PRESCALE_INEXACT;
  const unsigned t1 = FN(pattern)(gp);
  flags |= t1 << KOG_F_TYPE_SCALED_SHIFT;
  if (ora_scale_type(t1) == 0) {
    FN(simple)(gp, info.s, t1, flags, &out);
    return out;
  }
  if (t1 == 3 || t1 == 12 || t1 == 5 || t1 == 10) {
    FN(mono)(gp, info.s, t1, flags, &out);
    return out;
  }
  if (t1 != 15) {
    FN(mat) r;
    ora_sp up, vp;
    FN(tri13)(gp, t1, &r, &up, &vp);
    FN(assemble_svd)(r, 0, up, 1, 1, 0, (T)0, 1, vp, info.s, 1, o,
                     flags | ((uint32_t)KOG_PATH_TRI13 << KOG_F_PATH_SHIFT), &out);
    return out;
  }
  const FN(urv) u = FN(urv15)(gp, o);
  if (u.col_swap) flags |= KOG_F_URV_COL_SWAP;
  if (u.row_swap) flags |= KOG_F_URV_ROW_SWAP;
  const ora_sp pu = u.row_swap ? ora_sp_x() : ora_sp_id();
  const ora_sp s1 = ora_sp_rows(u.sr0, u.sr1);
  const ora_sp pv = u.col_swap ? ora_sp_x() : ora_sp_id();
  if (u.next == 0) {
    FN(assemble_svd)(u.r, 1, ora_sp_id(), u.sr0, u.sr1, u.row_swap, u.tan_theta, u.s22,
                     ora_sp_mul(pv, ora_sp_rows(1, u.s12)), info.s, 0, o,
                     flags | ((uint32_t)KOG_PATH_URV15 << KOG_F_PATH_SHIFT), &out);
    return out;
  }
  const FN(mat) uleft = FN(left)(s1, FN(left)(pu, FN(rot)(u.tan_theta, u.sec_theta)));
  out.s = info.s;
  if (u.next == 1) {
    flags |= (uint32_t)KOG_PATH_URV15_TO_DIAG << KOG_F_PATH_SHIFT;
    T d1 = u.r11, d2 = u.r22_raw;
    const int ord = FN(fabs)(d1) < FN(fabs)(d2);
    if (ord) {
      const T tmp = d1;
      d1 = d2;
      d2 = tmp;
    }
    const ora_sp ps = ord ? ora_sp_x() : ora_sp_id();
    const ora_sp sg = ora_sp_rows(signbit(d1) ? -1 : 1, signbit(d2) ? -1 : 1);
    out.u = FN(right)(FN(right)(uleft, ps), sg);
    out.v = FN(spmat)(ora_sp_mul(pv, ps));
    out.s1 = FN(pscale2)(-info.s, FN(pmake)(0, FN(fabs)(d1), &out.err));
    out.s2 = FN(pscale2)(-info.s, FN(pmake)(0, FN(fabs)(d2), &out.err));
  } else {
    flags |= (uint32_t)KOG_PATH_URV15_TO_ROW << KOG_F_PATH_SHIFT;
    const ora_sp sv2 = ora_sp_rows(1, signbit(u.r12_raw) ? -1 : 1);
    T a = u.r11, b = FN(fabs)(u.r12_raw);
    const int ord = a < b;
    if (ord) {
      const T tmp = a;
      a = b;
      b = tmp;
    }
    const ora_sp pvo = ord ? ora_sp_x() : ora_sp_id();
    const T tan = b / a;
    const T sec = FN(sec)(tan);
    out.u = uleft;
    out.v = FN(left)(pv, FN(left)(sv2, FN(left)(pvo, FN(rot)(tan, sec))));
    out.s1 = FN(pscale2)(-info.s, FN(pmake)(0, FN(hypot)(u.r11, u.r12_raw), &out.err));
    FN(pair) zero = {0, (T)0};
    out.s2 = zero;
  }
  out.flags = flags;
  return out;
}

/* ---------------------------------------------------- oracle.hpp in ExtFloat */
static ora_emat FN(emat_from)(FN(mat) g) {
  ora_emat r = {ora_ext_from((double)g.g11), ora_ext_from((double)g.g12), ora_ext_from((double)g.g21),
                ora_ext_from((double)g.g22)};
  return r;
}

/* svd2_ext (oracle.hpp:102-238) */
static ora_extsvd FN(svd2_ext)(FN(mat) g) {
  ora_extsvd out;
  memset(&out, 0, sizeof out);
  int err = 0;
  const ora_info info = FN(classify)(g, &err);
  const unsigned t = info.t;
  if (ora_scale_type(t) == 0) {
    ora_sp pu = ora_sp_id(), pv = ora_sp_id();
    if (t == 2 || t == 6) pu = ora_sp_x();
    if (t == 4) pv = ora_sp_x();
    if (t == 8) pu = pv = ora_sp_x();
    FN(mat) d = FN(right)(FN(left)(ora_sp_t(pu), g), pv);
    if (FN(fabs)(d.g11) < FN(fabs)(d.g22)) {
      pu = ora_sp_mul(pu, ora_sp_x());
      pv = ora_sp_mul(pv, ora_sp_x());
      d = FN(right)(FN(left)(ora_sp_x(), d), ora_sp_x());
    }
    const ora_sp sg = ora_sp_rows(signbit(d.g11) ? -1 : 1, signbit(d.g22) ? -1 : 1);
    out.sigma1 = ora_ext_from((double)FN(fabs)(d.g11));
    out.sigma2 = ora_ext_from((double)FN(fabs)(d.g22));
    out.u = ora_ext_sp(ora_sp_mul(pu, sg));
    out.v = ora_ext_sp(pv);
    return out;
  }
  if (t == 3 || t == 12 || t == 5 || t == 10) {
    const int col = t == 3 || t == 12;
    ora_sp pu = ora_sp_id(), pv = ora_sp_id();
    FN(mat) a = g;
    if (t == 12) {
      pv = ora_sp_x();
      a = FN(right)(a, pv);
    }
    if (t == 10) {
      pu = ora_sp_x();
      a = FN(left)(ora_sp_t(pu), a);
    }
    const T x = a.g11, y = col ? a.g21 : a.g12;
    const ora_sp sgn = ora_sp_rows(signbit(x) ? -1 : 1, signbit(y) ? -1 : 1);
    const T ax = FN(fabs)(x), ay = FN(fabs)(y);
    const int sw = ax < ay;
    const ora_ext hi = ora_ext_from((double)(sw ? ay : ax)), lo = ora_ext_from((double)(sw ? ax : ay));
    out.sigma1 = ora_ext_hypot(hi, lo);
    const ora_emat rot = ora_ext_rot_tan(ora_ext_div(lo, hi));
    const ora_sp ord = sw ? ora_sp_x() : ora_sp_id();
    memset(&out.sigma2, 0, sizeof out.sigma2);
    const ora_emat lhs = ora_emat_mul(ora_ext_sp(sgn), ora_ext_sp(ord));
    if (col) {
      out.u = ora_emat_mul(lhs, rot);
      out.v = ora_ext_sp(pv);
    } else {
      out.u = ora_ext_sp(pu);
      out.v = ora_emat_mul(lhs, rot);
    }
    return out;
  }
  ora_ext r11, r12, r22;
  ora_emat uplus, vplus;
  if (t != 15) {
    FN(mat) r;
    ora_sp up, vp;
    FN(tri13)(g, t, &r, &up, &vp);
    r11 = ora_ext_from((double)r.g11);
    r12 = ora_ext_from((double)r.g12);
    r22 = ora_ext_from((double)r.g22);
    uplus = ora_ext_sp(up);
    vplus = ora_ext_sp(vp);
  } else {
    const ora_ext w1 = ora_ext_hypot(ora_ext_from((double)g.g11), ora_ext_from((double)g.g21));
    const ora_ext w2 = ora_ext_hypot(ora_ext_from((double)g.g12), ora_ext_from((double)g.g22));
    const int col_swap = ora_ext_cmp(w1, w2) < 0;
    FN(mat) a = g;
    if (col_swap) {
      FN(mat) sw = {g.g12, g.g11, g.g22, g.g21};
      a = sw;
    }
    const ora_ext w = col_swap ? w2 : w1;
    const int s0 = signbit(a.g11) ? -1 : 1, s1 = signbit(a.g21) ? -1 : 1;
    a = FN(left)(ora_sp_rows(s0, s1), a);
    const int row_swap = a.g11 < a.g21;
    if (row_swap) {
      FN(mat) sw = {a.g21, a.g22, a.g11, a.g12};
      a = sw;
    }
    const ora_ext e11 = ora_ext_from((double)a.g11), e12 = ora_ext_from((double)a.g12);
    const ora_ext e21 = ora_ext_from((double)a.g21), e22 = ora_ext_from((double)a.g22);
    const ora_ext num12 = ora_ext_add(ora_ext_mul(e12, e11), ora_ext_mul(e22, e21));
    const ora_ext num22 = ora_ext_sub(ora_ext_mul(e22, e11), ora_ext_mul(e12, e21));
    r11 = w;
    r12 = ora_ext_div(num12, w);
    r22 = ora_ext_div(num22, w);
    const int s12 = ora_ext_sign(r12) < 0 ? -1 : 1;
    const int s22 = ora_ext_sign(r12) * ora_ext_sign(r22) < 0 ? -1 : 1;
    r12 = ora_ext_abs(r12);
    r22 = ora_ext_abs(r22);
    const ora_sp pu = row_swap ? ora_sp_x() : ora_sp_id();
    const ora_sp pv = col_swap ? ora_sp_x() : ora_sp_id();
    const ora_emat uth = ora_ext_rot_tan(ora_ext_div(e21, e11));
    uplus = ora_emat_mul(ora_emat_mul(ora_ext_sp(ora_sp_rows(s0, s1)), ora_ext_sp(pu)),
                         ora_emat_mul(uth, ora_ext_sp(ora_sp_rows(1, s22))));
    vplus = ora_ext_sp(ora_sp_mul(pv, ora_sp_rows(1, s12)));
    if (ora_ext_is_zero(r22)) {
      const int ord = ora_ext_cmp(r11, r12) < 0;
      const ora_ext hi = ord ? r12 : r11, lo = ord ? r11 : r12;
      const ora_emat rot = ora_ext_rot_tan(ora_ext_div(lo, hi));
      out.sigma1 = ora_ext_hypot(r11, r12);
      memset(&out.sigma2, 0, sizeof out.sigma2);
      out.u = uplus;
      out.v = ora_emat_mul(vplus, ora_emat_mul(ora_ext_sp(ord ? ora_sp_x() : ora_sp_id()), rot));
      return out;
    }
  }
  const int diag_swap = ora_ext_cmp(r11, r22) < 0;
  const ora_triref ts = ora_tri_ref(diag_swap ? r22 : r11, r12, diag_swap ? r11 : r22);
  out.sigma1 = ts.sigma1;
  out.sigma2 = ts.sigma2;
  ora_emat ut, vt;
  if (!diag_swap) {
    ut = ora_ext_rot(ts.cphi, ts.sphi);
    vt = ora_ext_rot(ts.cpsi, ts.spsi);
  } else {
    ora_emat a = {ts.spsi, ts.cpsi, ts.cpsi, ora_ext_neg(ts.spsi)};
    ora_emat b = {ts.sphi, ts.cphi, ts.cphi, ora_ext_neg(ts.sphi)};
    ut = a;
    vt = b;
  }
  out.u = ora_emat_mul(uplus, ut);
  out.v = ora_emat_mul(vplus, vt);
  return out;
}

/* metrics (oracle.hpp:267-301) */
static ora_metrics FN(metrics)(FN(mat) g, FN(mat) u, FN(mat) v, ora_ext sig1, ora_ext sig2, const ora_extsvd* ref) {
  ora_metrics out;
  memset(&out, 0, sizeof out);
  const ora_emat ge = FN(emat_from)(g), ue = FN(emat_from)(u), ve = FN(emat_from)(v);
  const ora_ext z = ora_ext_zero();
  const ora_emat sig = {sig1, z, z, sig2};
  ora_emat rec = ora_emat_mul(ora_emat_mul(ue, sig), ora_emat_t(ve));
  rec.a11 = ora_ext_sub(ge.a11, rec.a11);
  rec.a12 = ora_ext_sub(ge.a12, rec.a12);
  rec.a21 = ora_ext_sub(ge.a21, rec.a21);
  rec.a22 = ora_ext_sub(ge.a22, rec.a22);
  out.reG = ora_ext_ratio(ora_emat_fnorm(rec), ora_emat_fnorm(ge));
  out.reS1 = ora_relerr(ref->sigma1, sig1);
  out.reS2 = ora_relerr(ref->sigma2, sig2);
  out.reU = ora_ortho_defect(ue);
  out.reV = ora_ortho_defect(ve);
  if (ora_ext_is_zero(ref->sigma2)) {
    out.kappa_inf = !ora_ext_is_zero(ref->sigma1);
    out.kappa2 = ora_ext_zero();
  } else {
    out.kappa2 = ora_ext_div(ref->sigma1, ref->sigma2);
  }
  return out;
}

/* lasv2_ref (lasv2.hpp:22-127) */
static void FN(lasv2)(T f, T g, T h, T* o) {
  const T one = 1, two = 2, four = 4, half = (T)0.5, zero = 0;
  const T eps = FN(uround)();
  T ssmin = 0, ssmax = 0, snr, csr, snl, csl, clt = 0, crt = 0, slt = 0, srt = 0;
  T ft = f, fa = FN(fabs)(ft), ht = h, ha = FN(fabs)(h);
  int pmax = 1;
  const int swap = ha > fa;
  if (swap) {
    T tmp;
    pmax = 3;
    tmp = ft, ft = ht, ht = tmp;
    tmp = fa, fa = ha, ha = tmp;
  }
  const T gt = g, ga = FN(fabs)(gt);
  if (ga == zero) {
    ssmin = ha;
    ssmax = fa;
    clt = one;
    crt = one;
    slt = zero;
    srt = zero;
  } else {
    int gasmal = 1;
    if (ga > fa) {
      pmax = 2;
      if (fa / ga < eps) {
        gasmal = 0;
        ssmax = ga;
        ssmin = ha > one ? fa / (ga / ha) : (fa / ga) * ha;
        clt = one;
        slt = ht / gt;
        srt = one;
        crt = ft / gt;
      }
    }
    if (gasmal) {
      const T d = fa - ha;
      const T l = (d == fa) ? one : d / fa;
      const T m = gt / ft;
      T t = two - l;
      const T mm = m * m, tt = t * t;
      const T s = FN(sqrt)(tt + mm);
      const T r = (l == zero) ? FN(fabs)(m) : FN(sqrt)(l * l + mm);
      const T a = half * (s + r);
      ssmin = ha / a;
      ssmax = fa * a;
      if (mm == zero) {
        if (l == zero)
          t = FN(copysign)(two, ft) * FN(copysign)(one, gt);
        else
          t = gt / FN(copysign)(d, ft) + m / t;
      } else {
        t = (m / (s + t) + m / (r + l)) * (one + a);
      }
      const T ll = FN(sqrt)(t * t + four);
      crt = two / ll;
      srt = t / ll;
      clt = (crt + srt * m) / a;
      slt = (ht / ft) * srt / a;
    }
  }
  if (swap) {
    csl = srt, snl = crt, csr = slt, snr = clt;
  } else {
    csl = clt, snl = slt, csr = crt, snr = srt;
  }
  T tsign = 0;
  if (pmax == 1) tsign = FN(copysign)(one, csr) * FN(copysign)(one, csl) * FN(copysign)(one, f);
  if (pmax == 2) tsign = FN(copysign)(one, snr) * FN(copysign)(one, csl) * FN(copysign)(one, g);
  if (pmax == 3) tsign = FN(copysign)(one, snr) * FN(copysign)(one, snl) * FN(copysign)(one, h);
  ssmax = FN(copysign)(ssmax, tsign);
  ssmin = FN(copysign)(ssmin, tsign * FN(copysign)(one, f) * FN(copysign)(one, h));
  o[0] = ssmin, o[1] = ssmax, o[2] = snr, o[3] = csr, o[4] = snl, o[5] = csl;
}

/* generate<T> (harness.hpp:139-186) + the kog2 extension (include/kog2.h) */
static T FN(ranged)(ora_stream* st, int elo, int ehi) {
  const uint64_t u = ora_next(st);
  const int e = elo + (int)(u % (uint64_t)(ehi - elo + 1));
  const T f = (T)1 + FN(scalbn)((T)(ora_next(st) >> (64 - (KP - 1))), 1 - KP);
  const T v = FN(scalbn)(f, e);
  return (u >> 63) ? -v : v;
}
static T FN(element)(ora_stream* st, const kog_run_config* c) {
  switch (c->regime) {
    case KOG_REGIME_CIRC: {
      const uint64_t u = ora_next(st);
      const T m = (T)((double)(u >> 11) * 0x1p-53);
      return (u & 1) ? -m : m;
    }
    case KOG_REGIME_BULLET:
      return FN(ranged)(st, KEMIN, KEMAX - 2);
    case KOG_REGIME_SIGMA:
      return FN(ranged)(st, KEMIN + c->varsigma, KEMAX - 2);
    default:
      if (c->tail_mod != 0) {
        const uint64_t t = ora_next(st);
        if (t % c->tail_mod == 0) return FN(ranged)(st, c->tail_lo, c->tail_hi);
      }
      return FN(ranged)(st, c->elo, c->ehi);
  }
}
static T FN(nonzero)(ora_stream* st, const kog_run_config* c) {
  T v = FN(element)(st, c);
  while (v == (T)0) v = FN(element)(st, c);
  return v;
}
static FN(mat) FN(generate)(const kog_run_config* c, uint64_t index) {
  ora_stream st = ora_stream_make(c->seed, index);
  FN(mat) g;
  if (c->shape == KOG_SHAPE_TRI) {
    g.g11 = FN(nonzero)(&st, c);
    g.g12 = FN(element)(&st, c);
    g.g21 = (T)0;
    g.g22 = FN(nonzero)(&st, c);
  } else {
    g.g11 = FN(element)(&st, c);
    g.g12 = FN(element)(&st, c);
    g.g21 = FN(element)(&st, c);
    g.g22 = FN(element)(&st, c);
  }
  if (c->regime == KOG_REGIME_RANGED && c->zero_mask_rule) {
    const uint64_t z = ora_next(&st);
    if ((z & 7) == 0) {
      const unsigned m = (unsigned)(z >> 3) & 15u;
      if (m & 1) g.g11 = (T)0;
      if (m & 2) g.g21 = (T)0;
      if (m & 4) g.g12 = (T)0;
      if (m & 8) g.g22 = (T)0;
    }
  }
  return g;
}

static uint32_t FN(sign_flags)(FN(mat) u, FN(mat) v) {
  return (signbit(u.g21) ? KOG_F_SIGN_U21 : 0u) | (signbit(u.g22) ? KOG_F_SIGN_U22 : 0u) |
         (signbit(v.g21) ? KOG_F_SIGN_V21 : 0u) | (signbit(v.g22) ? KOG_F_SIGN_V22 : 0u);
}

/* run_one (harness.hpp:190-222): returns 0, KOG_FAIL_NONFINITE or KOG_FAIL_NAN_METRIC */
static int FN(run_one)(const kog_run_config* c, uint64_t index, ora_stats* st) {
  const FN(mat) g = FN(generate)(c, index);
  const ora_extsvd ref = FN(svd2_ext)(g);
  ora_metrics m;
  if (c->routine == KOG_ROUTINE_KOG) {
    const FN(res) r = FN(svd2)(g, &c->options);
    if (!FN(all_finite)(r.u) || !FN(all_finite)(r.v) || !isfinite(r.s1.f) || !isfinite(r.s2.f))
      return KOG_FAIL_NONFINITE;
    m = FN(metrics)(g, r.u, r.v, ora_ext_from_pair(r.s1.e, (double)r.s1.f), ora_ext_from_pair(r.s2.e, (double)r.s2.f),
                    &ref);
    if (isnan(m.reG) || isnan(m.reS1) || isnan(m.reS2) || isnan(m.reU) || isnan(m.reV)) return KOG_FAIL_NAN_METRIC;
    ora_stats_absorb(st, &m, r.flags, 1);
  } else {
    T o[6];
    FN(lasv2)(g.g11, g.g12, g.g22, o);
    const FN(mat) u = {o[5], -o[4], o[4], o[5]};
    const FN(mat) v = {o[3], -o[2], o[2], o[3]};
    if (!FN(all_finite)(u) || !FN(all_finite)(v) || !isfinite(o[1]) || !isfinite(o[0])) return KOG_FAIL_NONFINITE;
    m = FN(metrics)(g, u, v, ora_ext_from((double)o[1]), ora_ext_from((double)o[0]), &ref);
    if (isnan(m.reG) || isnan(m.reS1) || isnan(m.reS2) || isnan(m.reU) || isnan(m.reV)) return KOG_FAIL_NAN_METRIC;
    ora_stats_absorb(st, &m, 0, 0);
  }
  return 0;
}

#undef FN
#undef CAT
#undef CAT2
