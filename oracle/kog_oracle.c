/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's hot path:
 * fpcore (correctly rounded hypot), epair, classify/prescale, the svd2 phases
 * and driver, extfloat, the ExtFloat oracle and error measures, the seeded
 * generator, ErrorStats and the CSV row.  Paths cited are relative to
 * /root/reference/proj/include/kogsvd2/.  Compiled with -ffp-contract=off
 * (the reference's own requirement, proj/CMakeLists.txt:14-15).
 *
 * This file is the checker, never the product: it is loaded only by tests/,
 * __graft_entry__.smoke() and bench.py's CPU baseline leg.  Parity pinned
 * against oracle/_ref (the reference compiled in place) and tests/golden/.
 */
#define _GNU_SOURCE
#include "kog_oracle.h"

#include <float.h>
#include <inttypes.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static __thread char g_err[512];

/* ------------------------------------------- EFTs (fpcore.hpp:59-95) */
static void ora_two_sum(double a, double b, double* s, double* e) {
  *s = a + b;
  const double bv = *s - a;
  *e = (a - (*s - bv)) + (b - bv);
}
static void ora_fast_two_sum(double a, double b, double* s, double* e) {
  const double ss = a + b;
  *e = (a - ss) + b;
  *s = ss;
}
static void ora_two_prod(double a, double b, double* p, double* e) {
  *p = a * b;
  *e = fma(a, b, -*p);
}

/* exact sign of a sum via a nonoverlapping expansion (fpcore.hpp:78-95) */
static int ora_exact_sum_sign(const double* x, int n) {
  double comp[16];
  int len = 0;
  for (int i = 0; i < n; ++i) {
    double q = x[i];
    int k = 0;
    for (int j = 0; j < len; ++j) {
      double s, err;
      ora_two_sum(q, comp[j], &s, &err);
      if (err != 0.0) comp[k++] = err;
      q = s;
    }
    if (q != 0.0) comp[k++] = q;
    len = k;
  }
  if (len == 0) return 0;
  return (comp[len - 1] > 0.0) - (comp[len - 1] < 0.0);
}

/* round sqrt(x1+x2+y1+y2) onto the grid 2^tg by exact midpoint tests
 * (fpcore.hpp:100-134) */
static double ora_round_sqrt_on_grid(double x1, double x2, double y1, double y2, double z0, int tg, double zlo,
                                     double zhi) {
  const double g = scalbn(1.0, tg);
  double z = nearbyint(scalbn(z0 < zlo ? zlo : (z0 > zhi ? zhi : z0), -tg));
  z = scalbn(z, tg);
  if (z < zlo) z = zlo;
  if (z > zhi) z = zhi;
  for (int iter = 0; iter < 8; ++iter) {
    double zq, zqe;
    ora_two_prod(z, z, &zq, &zqe);
    const double zg = z * g;
    const double g24 = scalbn(1.0, 2 * tg - 2);
    if (z < zhi) {
      const double up[8] = {x1, x2, y1, y2, -zq, -zqe, -zg, -g24};
      const int cu = ora_exact_sum_sign(up, 8);
      if (cu > 0) {
        z += g;
        continue;
      }
      if (cu == 0) return fmod(scalbn(z, -tg), 2.0) == 0.0 ? z : z + g;
    }
    if (z > zlo) {
      const double dn[8] = {x1, x2, y1, y2, -zq, -zqe, zg, -g24};
      const int cd = ora_exact_sum_sign(dn, 8);
      if (cd < 0) {
        z -= g;
        continue;
      }
      if (cd == 0) return fmod(scalbn(z, -tg), 2.0) == 0.0 ? z : z - g;
    }
    break;
  }
  return z;
}

/* -------------------------------------------- classify.hpp helpers */
typedef struct {
  unsigned t;
  int s_type;
  int64_t s, e_G;
} ora_info;

static int ora_scale_type(unsigned t) { /* classify.hpp:37-42 */
  if (t == 15) return 2;
  if (t == 0 || t == 1 || t == 2 || t == 4 || t == 6 || t == 8 || t == 9) return 0;
  return 1;
}

/* -------------------------------------------- SignPerm (svd2.hpp:21-48) */
typedef struct {
  int8_t m[2][2];
} ora_sp;
static ora_sp ora_sp_id(void) {
  ora_sp s = {{{1, 0}, {0, 1}}};
  return s;
}
static ora_sp ora_sp_x(void) {
  ora_sp s = {{{0, 1}, {1, 0}}};
  return s;
}
static ora_sp ora_sp_rows(int a, int b) {
  ora_sp s = {{{(int8_t)a, 0}, {0, (int8_t)b}}};
  return s;
}
static ora_sp ora_sp_mul(ora_sp a, ora_sp b) {
  ora_sp r;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) r.m[i][j] = (int8_t)(a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j]);
  return r;
}
static ora_sp ora_sp_t(ora_sp a) {
  ora_sp r = {{{a.m[0][0], a.m[1][0]}, {a.m[0][1], a.m[1][1]}}};
  return r;
}

/* -------------------------------------------- ExtFloat (extfloat.hpp) */
typedef struct {
  int64_t e;
  double hi, lo;
} ora_ext;
typedef struct {
  ora_ext a11, a12, a21, a22;
} ora_emat;
typedef struct {
  ora_ext sigma1, sigma2;
  ora_emat u, v;
} ora_extsvd;
typedef struct {
  double reG, reS1, reS2, reU, reV;
  ora_ext kappa2;
  int kappa_inf;
} ora_metrics;

static ora_ext ora_ext_zero(void) {
  ora_ext z = {0, 0.0, 0.0};
  return z;
}
static int ora_ext_is_zero(ora_ext a) { return a.hi == 0.0; }
static int ora_ext_sign(ora_ext a) { return (a.hi > 0.0) - (a.hi < 0.0); }

static ora_ext ora_ext_make(int64_t e, double h, double l) { /* extfloat.hpp:33-48 */
  if (h == 0.0) {
    h = l;
    l = 0.0;
  }
  if (h == 0.0) return ora_ext_zero();
  if (fabs(h) < fabs(l)) {
    const double t = h;
    h = l;
    l = t;
  }
  double s, t;
  ora_fast_two_sum(h, l, &s, &t);
  if (s == 0.0) return ora_ext_zero();
  const int k = ilogb(s);
  double tl = scalbn(t, -k);
  if (fabs(tl) < 0x1p-120) tl = 0.0;
  ora_ext r = {e + k, scalbn(s, -k), tl};
  return r;
}
static ora_ext ora_ext_from(double x) { /* extfloat.hpp:52-55 via split */
  ora_ext r = {0, x, 0.0};
  if (x == 0.0 || !isfinite(x)) return r;
  int be;
  const double fr = frexp(x, &be);
  r.e = (int64_t)be - 1;
  r.hi = fr + fr;
  return r;
}
static ora_ext ora_ext_from_pair(int64_t e, double f) { /* extfloat.hpp:58-62 */
  if (f == 0.0) return ora_ext_zero();
  ora_ext r = {e, f, 0.0};
  return r;
}
static ora_ext ora_ext_neg(ora_ext a) {
  ora_ext r = {a.e, -a.hi, -a.lo};
  return r;
}
static ora_ext ora_ext_abs(ora_ext a) { return a.hi < 0 ? ora_ext_neg(a) : a; }
static ora_ext ora_ext_scale2(int64_t k, ora_ext a) {
  if (!ora_ext_is_zero(a)) a.e += k;
  return a;
}
static ora_ext ora_ext_add(ora_ext a, ora_ext b) { /* extfloat.hpp:72-90 */
  if (ora_ext_is_zero(a)) return b;
  if (ora_ext_is_zero(b)) return a;
  const int64_t d = a.e - b.e;
  if (d > 120) return a;
  if (d < -120) return b;
  const ora_ext big = d >= 0 ? a : b, sml = d >= 0 ? b : a;
  const int sh = (int)(d >= 0 ? d : -d);
  const double bh = scalbn(sml.hi, -sh), bl = scalbn(sml.lo, -sh);
  double s1, s2, t1, t2;
  ora_two_sum(big.hi, bh, &s1, &s2);
  ora_two_sum(big.lo, bl, &t1, &t2);
  s2 += t1;
  ora_fast_two_sum(s1, s2, &s1, &s2);
  s2 += t2;
  ora_fast_two_sum(s1, s2, &s1, &s2);
  return ora_ext_make(big.e, s1, s2);
}
static ora_ext ora_ext_sub(ora_ext a, ora_ext b) { return ora_ext_add(a, ora_ext_neg(b)); }
static ora_ext ora_ext_mul(ora_ext a, ora_ext b) { /* extfloat.hpp:96-102 */
  if (ora_ext_is_zero(a) || ora_ext_is_zero(b)) return ora_ext_zero();
  double p, e;
  ora_two_prod(a.hi, b.hi, &p, &e);
  e += a.hi * b.lo + a.lo * b.hi + a.lo * b.lo;
  return ora_ext_make(a.e + b.e, p, e);
}
static ora_ext ora_ext_div(ora_ext a, ora_ext b) { /* extfloat.hpp:104-113 */
  if (ora_ext_is_zero(a)) return ora_ext_zero();
  const double bd = b.hi + b.lo;
  const double q1 = a.hi / bd;
  double p, pe;
  ora_two_prod(q1, b.hi, &p, &pe);
  const double r = ((a.hi - p) - pe) + a.lo - q1 * b.lo;
  return ora_ext_make(a.e - b.e, q1, r / bd);
}
static ora_ext ora_ext_sqrt(ora_ext a) { /* extfloat.hpp:115-134 */
  if (ora_ext_is_zero(a)) return ora_ext_zero();
  int64_t e = a.e;
  double h = a.hi, l = a.lo;
  if (e & 1) {
    h *= 2;
    l *= 2;
    e -= 1;
  }
  const double q1 = sqrt(h + l);
  double p, pe, s1, s2, t1, t2;
  ora_two_prod(q1, q1, &p, &pe);
  ora_two_sum(h, -p, &s1, &s2);
  ora_two_sum(l, -pe, &t1, &t2);
  s2 += t1;
  ora_fast_two_sum(s1, s2, &s1, &s2);
  return ora_ext_make(e / 2, q1, (s1 + (s2 + t2)) / (2 * q1));
}
static int ora_ext_cmp(ora_ext a, ora_ext b) { return ora_ext_sign(ora_ext_sub(a, b)); }
static double ora_ext_to_double(ora_ext a) { /* extfloat.hpp:140-144 */
  const long ce = (long)(a.e < -100000 ? -100000 : (a.e > 100000 ? 100000 : a.e));
  return scalbln(a.hi + a.lo, ce);
}
static ora_ext ora_ext_pow10(int64_t n) { /* extfloat.hpp:146-157 */
  ora_ext base = ora_ext_from(10.0);
  if (n < 0) base = ora_ext_div(ora_ext_from(1.0), base);
  uint64_t k = (uint64_t)(n < 0 ? -n : n);
  ora_ext acc = ora_ext_from(1.0);
  while (k) {
    if (k & 1) acc = ora_ext_mul(acc, base);
    base = ora_ext_mul(base, base);
    k >>= 1;
  }
  return acc;
}

/* ExtMat helpers (oracle.hpp:18-64) */
static ora_emat ora_emat_mul(ora_emat x, ora_emat y) {
  ora_emat r = {ora_ext_add(ora_ext_mul(x.a11, y.a11), ora_ext_mul(x.a12, y.a21)),
                ora_ext_add(ora_ext_mul(x.a11, y.a12), ora_ext_mul(x.a12, y.a22)),
                ora_ext_add(ora_ext_mul(x.a21, y.a11), ora_ext_mul(x.a22, y.a21)),
                ora_ext_add(ora_ext_mul(x.a21, y.a12), ora_ext_mul(x.a22, y.a22))};
  return r;
}
static ora_emat ora_emat_t(ora_emat x) {
  ora_emat r = {x.a11, x.a21, x.a12, x.a22};
  return r;
}
static ora_ext ora_emat_fnorm(ora_emat x) {
  ora_ext s = ora_ext_mul(x.a11, x.a11);
  s = ora_ext_add(s, ora_ext_mul(x.a12, x.a12));
  s = ora_ext_add(s, ora_ext_mul(x.a21, x.a21));
  s = ora_ext_add(s, ora_ext_mul(x.a22, x.a22));
  return ora_ext_sqrt(s);
}
static ora_ext ora_ext_hypot(ora_ext a, ora_ext b) { return ora_ext_sqrt(ora_ext_add(ora_ext_mul(a, a), ora_ext_mul(b, b))); }
static ora_emat ora_ext_rot(ora_ext c, ora_ext s) {
  ora_emat r = {c, ora_ext_neg(s), s, c};
  return r;
}
static ora_emat ora_ext_rot_tan(ora_ext tan) {
  const ora_ext one = ora_ext_from(1.0);
  const ora_ext sec = ora_ext_sqrt(ora_ext_add(ora_ext_mul(tan, tan), one));
  return ora_ext_rot(ora_ext_div(one, sec), ora_ext_div(tan, sec));
}
static ora_emat ora_ext_sp(ora_sp p) {
  ora_emat r = {ora_ext_from((double)p.m[0][0]), ora_ext_from((double)p.m[0][1]), ora_ext_from((double)p.m[1][0]),
                ora_ext_from((double)p.m[1][1])};
  return r;
}

typedef struct {
  ora_ext sigma1, sigma2, cphi, sphi, cpsi, spsi;
} ora_triref;

/* tri_ref (oracle.hpp:66-98) */
static ora_triref ora_tri_ref(ora_ext a, ora_ext b, ora_ext c) {
  ora_triref out;
  const ora_ext one = ora_ext_from(1.0);
  const ora_ext amc = ora_ext_sub(a, c), apc = ora_ext_add(a, c), b2 = ora_ext_mul(b, b);
  const ora_ext dm = ora_ext_add(ora_ext_mul(amc, amc), b2);
  const ora_ext dp = ora_ext_add(ora_ext_mul(apc, apc), b2);
  const ora_ext gap = ora_ext_sqrt(ora_ext_mul(dm, dp));
  const ora_ext tau = ora_ext_add(ora_ext_add(ora_ext_mul(a, a), b2), ora_ext_mul(c, c));
  out.sigma1 = ora_ext_sqrt(ora_ext_scale2(-1, ora_ext_add(tau, gap)));
  out.sigma2 = ora_ext_div(ora_ext_mul(a, c), out.sigma1);
  const ora_ext den = ora_ext_add(ora_ext_mul(amc, apc), b2);
  const ora_ext t2f = ora_ext_div(ora_ext_scale2(1, ora_ext_mul(b, c)), den);
  const ora_ext tphi = ora_ext_div(t2f, ora_ext_add(one, ora_ext_sqrt(ora_ext_add(ora_ext_mul(t2f, t2f), one))));
  const ora_ext sphi = ora_ext_sqrt(ora_ext_add(ora_ext_mul(tphi, tphi), one));
  const ora_ext tpsi = ora_ext_div(ora_ext_add(b, ora_ext_mul(c, tphi)), a);
  const ora_ext spsi = ora_ext_sqrt(ora_ext_add(ora_ext_mul(tpsi, tpsi), one));
  out.cphi = ora_ext_div(one, sphi);
  out.sphi = ora_ext_div(tphi, sphi);
  out.cpsi = ora_ext_div(one, spsi);
  out.spsi = ora_ext_div(tpsi, spsi);
  return out;
}

static double ora_ext_ratio(ora_ext num, ora_ext den) { /* oracle.hpp:251-255 */
  if (ora_ext_is_zero(num)) return 0.0;
  if (ora_ext_is_zero(den)) return INFINITY;
  return ora_ext_to_double(ora_ext_div(num, den));
}
static double ora_ortho_defect(ora_emat q) { /* oracle.hpp:257-263 */
  ora_emat m = ora_emat_mul(ora_emat_t(q), q);
  const ora_ext one = ora_ext_from(1.0);
  m.a11 = ora_ext_sub(m.a11, one);
  m.a22 = ora_ext_sub(m.a22, one);
  return ora_ext_to_double(ora_emat_fnorm(m));
}
static double ora_relerr(ora_ext want, ora_ext got) { /* oracle.hpp:286-289 */
  if (ora_ext_is_zero(want) && ora_ext_is_zero(got)) return 0.0;
  return ora_ext_ratio(ora_ext_abs(ora_ext_sub(want, ora_ext_abs(got))), want);
}

/* -------------------------------------- Stream (harness.hpp:114-128) */
typedef struct {
  uint64_t s;
} ora_stream;
static uint64_t ora_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static ora_stream ora_stream_make(uint64_t seed, uint64_t index) {
  ora_stream st = {ora_mix64(seed + 0x9e3779b97f4a7c15ull * (index + 1))};
  return st;
}
static uint64_t ora_next(ora_stream* st) {
  st->s += 0x9e3779b97f4a7c15ull;
  return ora_mix64(st->s);
}

/* --------------------------- ErrorStats / BranchCounts (harness.hpp:50-106) */
typedef struct {
  double reG, reS1, reS2, reU, reV;
  ora_ext maxKappa2;
  int kappa_inf;
  uint64_t t2p[7], path[7], tanpsi_inf, diag_swap, compose_minus, sigma_swap, prescale_inexact;
} ora_stats;

static void ora_stats_absorb(ora_stats* st, const ora_metrics* m, uint32_t flags, int with_trace) {
  st->reG = fmax(st->reG, m->reG);
  st->reS1 = fmax(st->reS1, m->reS1);
  st->reS2 = fmax(st->reS2, m->reS2);
  st->reU = fmax(st->reU, m->reU);
  st->reV = fmax(st->reV, m->reV);
  if (m->kappa_inf)
    st->kappa_inf = 1;
  else if (ora_ext_cmp(m->kappa2, st->maxKappa2) > 0)
    st->maxKappa2 = m->kappa2;
  if (!with_trace) return;
  ++st->t2p[(flags >> KOG_F_T2P_SHIFT) & 7u];
  ++st->path[(flags >> KOG_F_PATH_SHIFT) & 7u];
  st->tanpsi_inf += (flags & KOG_F_TANPSI_INF) != 0;
  st->diag_swap += (flags & KOG_F_DIAG_SWAP) != 0;
  st->compose_minus += (flags & KOG_F_COMPOSE_MINUS) != 0;
  st->sigma_swap += (flags & KOG_F_SIGMA_SWAP) != 0;
  st->prescale_inexact += (flags & KOG_F_PRESCALE_INEXACT) != 0;
}
static void ora_stats_merge(ora_stats* st, const ora_stats* o) {
  st->reG = fmax(st->reG, o->reG);
  st->reS1 = fmax(st->reS1, o->reS1);
  st->reS2 = fmax(st->reS2, o->reS2);
  st->reU = fmax(st->reU, o->reU);
  st->reV = fmax(st->reV, o->reV);
  st->kappa_inf = st->kappa_inf || o->kappa_inf;
  if (ora_ext_cmp(o->maxKappa2, st->maxKappa2) > 0) st->maxKappa2 = o->maxKappa2;
  for (int i = 0; i < 7; ++i) {
    st->t2p[i] += o->t2p[i];
    st->path[i] += o->path[i];
  }
  st->tanpsi_inf += o->tanpsi_inf;
  st->diag_swap += o->diag_swap;
  st->compose_minus += o->compose_minus;
  st->sigma_swap += o->sigma_swap;
  st->prescale_inexact += o->prescale_inexact;
}

/* ------------------------------------------ the two working precisions */
#define T double
#define SUF f64
#define KP 53
#define KEMAX 1023
#define KEMIN (-1022)
#define KF32 0
#include "kog_oracle_t.h"
#undef T
#undef SUF
#undef KP
#undef KEMAX
#undef KEMIN
#undef KF32

#define T float
#define SUF f32
#define KP 24
#define KEMAX 127
#define KEMIN (-126)
#define KF32 1
#include "kog_oracle_t.h"
#undef T
#undef SUF
#undef KP
#undef KEMAX
#undef KEMIN
#undef KF32

/* ------------------------------------------------------- thread pool */
typedef struct {
  uint64_t n;
  uint64_t next;
  pthread_mutex_t mu;
  void (*body)(void* ctx, uint64_t blk, uint64_t lo, uint64_t hi);
  void* ctx;
} ora_pool;

static void* ora_worker(void* arg) {
  ora_pool* p = (ora_pool*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    const uint64_t b = p->next++;
    pthread_mutex_unlock(&p->mu);
    const uint64_t lo = b * 4096;
    if (lo >= p->n) return NULL;
    const uint64_t hi = lo + 4096 < p->n ? lo + 4096 : p->n;
    p->body(p->ctx, b, lo, hi);
  }
}

/* blocks of 4096 indices over `threads` workers (harness.hpp:226-263) */
static void ora_parallel(uint64_t n, int threads, void (*body)(void*, uint64_t, uint64_t, uint64_t), void* ctx) {
  ora_pool p;
  p.n = n;
  p.next = 0;
  p.body = body;
  p.ctx = ctx;
  pthread_mutex_init(&p.mu, NULL);
  int w = threads > 0 ? threads : (int)kogora_hardware_threads();
  const uint64_t nb = (n + 4095) / 4096;
  if (w < 1) w = 1;
  if ((uint64_t)w > nb && nb > 0) w = (int)nb;
  if (w <= 1) {
    ora_worker(&p);
  } else {
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)w);
    for (int i = 0; i < w; ++i) pthread_create(&tid[i], NULL, ora_worker, &p);
    for (int i = 0; i < w; ++i) pthread_join(tid[i], NULL);
    free(tid);
  }
  pthread_mutex_destroy(&p.mu);
}

/* ============================================================ exported */
const char* kogora_last_error(void) { return g_err; }
unsigned kogora_hardware_threads(void) {
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (unsigned)n : 1u;
}

#define SIMPLE_LOOP(SUF, T)                                                                   \
  int kogora_hypot_##SUF(const T* a, const T* b, T* o, uint64_t n) {                          \
    for (uint64_t i = 0; i < n; ++i) o[i] = hypot_##SUF(a[i], b[i]);                          \
    return 0;                                                                                 \
  }                                                                                           \
  int kogora_split_##SUF(const T* x, int64_t* e, T* f, uint64_t n) {                          \
    for (uint64_t i = 0; i < n; ++i) split_##SUF(x[i], e + i, f + i);                         \
    return 0;                                                                                 \
  }                                                                                           \
  int kogora_assemble_##SUF(const int64_t* e, const T* f, T* o, uint64_t n) {                 \
    for (uint64_t i = 0; i < n; ++i) o[i] = assemble_##SUF(e[i], f[i]);                       \
    return 0;                                                                                 \
  }                                                                                           \
  int kogora_tan2_##SUF(const T* t, T* o, uint64_t n) {                                       \
    for (uint64_t i = 0; i < n; ++i) o[i] = tan2_##SUF(t[i]);                                 \
    return 0;                                                                                 \
  }                                                                                           \
  int kogora_sec_##SUF(const T* t, T* o, uint64_t n) {                                        \
    for (uint64_t i = 0; i < n; ++i) o[i] = sec_##SUF(t[i]);                                  \
    return 0;                                                                                 \
  }                                                                                           \
  int kogora_compose_left_##SUF(const T* tp, const T* tt, const uint8_t* m, T* c, T* s,       \
                                uint64_t n) {                                                 \
    for (uint64_t i = 0; i < n; ++i) compose_##SUF(tp[i], tt[i], m[i] != 0, c + i, s + i);    \
    return 0;                                                                                 \
  }                                                                                           \
  int kogora_lasv2_##SUF(const T* f, const T* g, const T* h, T* o6, uint64_t n) {             \
    for (uint64_t i = 0; i < n; ++i) lasv2_##SUF(f[i], g[i], h[i], o6 + 6 * i);               \
    return 0;                                                                                 \
  }
SIMPLE_LOOP(f64, double)
SIMPLE_LOOP(f32, float)

#define EPAIR_FN(SUF, T)                                                                              \
  int kogora_epair_##SUF(int op, const int64_t* xe, const T* xf, const int64_t* ye, const T* yf,      \
                         int64_t* oe, T* of, uint8_t* st, uint64_t n) {                               \
    for (uint64_t i = 0; i < n; ++i) {                                                                \
      int err = 0;                                                                                    \
      const int64_t xee = xe ? xe[i] : 0, yee = ye ? ye[i] : 0;                                       \
      const T xff = xf[i], yff = yf ? yf[i] : (T)0;                                                   \
      pair_##SUF r = {0, (T)0};                                                                       \
      T val = 0;                                                                                      \
      int value_out = 0;                                                                              \
      switch (op) {                                                                                   \
        case KOG_EPAIR_OPLUS: r = oplus_##SUF(xff, yff, &err); break;                                 \
        case KOG_EPAIR_OMINUS: r = ominus_##SUF(xff, yff, &err); break;                               \
        case KOG_EPAIR_MUL: {                                                                         \
          const pair_##SUF a = pmake_##SUF(xee, xff, &err), b = pmake_##SUF(yee, yff, &err);          \
          r = pmul_##SUF(a, b, &err);                                                                 \
          break;                                                                                      \
        }                                                                                             \
        case KOG_EPAIR_DIV: {                                                                         \
          const pair_##SUF a = pmake_##SUF(xee, xff, &err), b = pmake_##SUF(yee, yff, &err);          \
          r = pdiv_##SUF(a, b, &err);                                                                 \
          break;                                                                                      \
        }                                                                                             \
        case KOG_EPAIR_LESS: {                                                                        \
          const pair_##SUF a = pmake_##SUF(xee, xff, &err), b = pmake_##SUF(yee, yff, &err);          \
          value_out = 1;                                                                              \
          val = pless_##SUF(a, b) ? (T)1 : (T)0;                                                      \
          break;                                                                                      \
        }                                                                                             \
        case KOG_EPAIR_RECIP: r = precip_##SUF(pmake_##SUF(xee, xff, &err), &err); break;             \
        default: r = pmake_##SUF(xee, xff, &err); break;                                              \
      }                                                                                               \
      st[i] = (uint8_t)(err ? 1 : 0);                                                                 \
      oe[i] = err || value_out ? 0 : r.e;                                                             \
      of[i] = err ? (T)0 : (value_out ? val : r.f);                                                   \
    }                                                                                                 \
    return 0;                                                                                         \
  }
EPAIR_FN(f64, double)
EPAIR_FN(f32, float)

#define CLASSIFY_FN(SUF, T, MT)                                                                        \
  int kogora_classify_prescale_##SUF(const MT* in, const kog_classify_out* o, const MT* gp, uint64_t n) { \
    for (uint64_t i = 0; i < n; ++i) {                                                                 \
      const mat_##SUF g = {in->g11[i], in->g12[i], in->g21[i], in->g22[i]};                            \
      int err = 0;                                                                                     \
      const ora_info info = classify_##SUF(g, &err);                                                   \
      o->status[i] = (uint8_t)err;                                                                     \
      if (err) continue;                                                                               \
      o->t[i] = (uint8_t)info.t;                                                                       \
      o->s_type[i] = info.s_type;                                                                      \
      o->s[i] = info.s;                                                                                \
      o->e_G[i] = info.e_G;                                                                            \
      int inexact;                                                                                     \
      const mat_##SUF r = prescale_##SUF(g, info.s, &inexact);                                         \
      o->inexact_underflow[i] = (uint8_t)inexact;                                                      \
      gp->g11[i] = r.g11;                                                                              \
      gp->g12[i] = r.g12;                                                                              \
      gp->g21[i] = r.g21;                                                                              \
      gp->g22[i] = r.g22;                                                                              \
    }                                                                                                  \
    return 0;                                                                                          \
  }
CLASSIFY_FN(f64, double, kog_mat_f64)
CLASSIFY_FN(f32, float, kog_mat_f32)

#define URV_FN(SUF, T, MT, RT)                                                                       \
  int kogora_urv15_##SUF(const MT* g, RT* o, uint64_t n, const kog_options* opt) {                   \
    for (uint64_t i = 0; i < n; ++i) {                                                               \
      const mat_##SUF m = {g->g11[i], g->g12[i], g->g21[i], g->g22[i]};                              \
      const urv_##SUF u = urv15_##SUF(m, opt);                                                       \
      RT* r = o + i;                                                                                 \
      memset(r, 0, sizeof *r);                                                                       \
      r->gppp[0] = u.gppp.g11, r->gppp[1] = u.gppp.g12, r->gppp[2] = u.gppp.g21, r->gppp[3] = u.gppp.g22; \
      r->tan_theta = u.tan_theta, r->sec_theta = u.sec_theta, r->r11 = u.r11;                        \
      r->r12_raw = u.r12_raw, r->r22_raw = u.r22_raw;                                                \
      r->r[0] = u.r.g11, r->r[1] = u.r.g12, r->r[2] = u.r.g21, r->r[3] = u.r.g22;                    \
      r->sr0 = u.sr0, r->sr1 = u.sr1, r->s12 = u.s12, r->s22 = u.s22;                                \
      r->col_swap = (uint8_t)u.col_swap, r->row_swap = (uint8_t)u.row_swap;                          \
      r->ext_is_r22 = (uint8_t)u.ext_is_r22, r->next = (uint8_t)u.next;                              \
    }                                                                                                \
    return 0;                                                                                        \
  }
URV_FN(f64, double, kog_mat_f64, kog_urv15_f64)
URV_FN(f32, float, kog_mat_f32, kog_urv15_f32)

#define TRI_FN(SUF, T, RT)                                                                                 \
  int kogora_tri_svd_##SUF(const T* a, const T* b, const T* c, const uint8_t* t13, RT* o, uint64_t n,     \
                           const kog_options* opt) {                                                       \
    for (uint64_t i = 0; i < n; ++i) {                                                                     \
      int err = 0;                                                                                         \
      const tri_##SUF ts = tri_svd_##SUF(a[i], b[i], c[i], t13[i] != 0, opt, &err);                        \
      RT* r = o + i;                                                                                       \
      memset(r, 0, sizeof *r);                                                                             \
      if (err) {                                                                                           \
        r->status = 1;                                                                                     \
        continue;                                                                                          \
      }                                                                                                    \
      r->t2f = ts.t2f, r->tan_phi = ts.tan_phi, r->sec_phi = ts.sec_phi, r->cos_phi = ts.cos_phi;          \
      r->sin_phi = ts.sin_phi, r->tan_psi = ts.tan_psi, r->sec_psi = ts.sec_psi;                           \
      r->cos_psi = ts.cos_psi, r->sin_psi = ts.sin_psi;                                                    \
      r->sig1_f = ts.sig1.f, r->sig2_f = ts.sig2.f, r->sig1_e = ts.sig1.e, r->sig2_e = ts.sig2.e;          \
      r->sigma_swapped = (uint8_t)ts.sigma_swapped, r->tanpsi_inf = (uint8_t)ts.tanpsi_inf;                \
      r->t2p = (uint8_t)ts.t2p;                                                                            \
    }                                                                                                      \
    return 0;                                                                                              \
  }
TRI_FN(f64, double, kog_trisvd_f64)
TRI_FN(f32, float, kog_trisvd_f32)

#define TRI13_FN(SUF, T, MT)                                                                             \
  int kogora_triangularize13_##SUF(const MT* g, const uint8_t* t, const MT* r, int8_t* up, int8_t* vp,  \
                                   uint64_t n) {                                                         \
    for (uint64_t i = 0; i < n; ++i) {                                                                   \
      const mat_##SUF m = {g->g11[i], g->g12[i], g->g21[i], g->g22[i]};                                  \
      mat_##SUF rr;                                                                                      \
      ora_sp u, v;                                                                                       \
      tri13_##SUF(m, t[i], &rr, &u, &v);                                                                 \
      r->g11[i] = rr.g11, r->g12[i] = rr.g12, r->g21[i] = rr.g21, r->g22[i] = rr.g22;                    \
      for (int k = 0; k < 4; ++k) {                                                                      \
        up[4 * i + k] = u.m[k / 2][k % 2];                                                               \
        vp[4 * i + k] = v.m[k / 2][k % 2];                                                               \
      }                                                                                                  \
    }                                                                                                    \
    return 0;                                                                                            \
  }
TRI13_FN(f64, double, kog_mat_f64)
TRI13_FN(f32, float, kog_mat_f32)

/* threaded SoA svd2 / generate / metrics */
typedef struct {
  const void* in;
  const void* out;
  const kog_options* opt;
  const kog_run_config* cfg;
  uint64_t index0;
} ora_job;

static kog_extfloat ora_c(ora_ext x) {
  kog_extfloat r = {x.e, x.hi, x.lo};
  return r;
}

#define BATCH_FNS(SUF, T, MT, OT)                                                                        \
  static void svd2_body_##SUF(void* ctx, uint64_t blk, uint64_t lo, uint64_t hi) {                       \
    (void)blk;                                                                                           \
    const ora_job* j = (const ora_job*)ctx;                                                              \
    const MT* in = (const MT*)j->in;                                                                     \
    const OT* out = (const OT*)j->out;                                                                   \
    for (uint64_t i = lo; i < hi; ++i) {                                                                 \
      const mat_##SUF g = {in->g11[i], in->g12[i], in->g21[i], in->g22[i]};                              \
      res_##SUF r = svd2_##SUF(g, j->opt);                                                               \
      uint32_t flags = r.flags;                                                                          \
      if (r.err) {                                                                                       \
        memset(&r, 0, sizeof r);                                                                         \
        flags = KOG_F_DOMAIN_ERROR;                                                                      \
      }                                                                                                  \
      out->sig1_f[i] = r.s1.f, out->sig2_f[i] = r.s2.f;                                                  \
      out->sig1_e[i] = (int32_t)r.s1.e, out->sig2_e[i] = (int32_t)r.s2.e;                                \
      out->u11[i] = r.u.g11, out->u12[i] = r.u.g12, out->v11[i] = r.v.g11, out->v12[i] = r.v.g12;        \
      out->s[i] = (int32_t)r.s;                                                                          \
      out->flags[i] = flags | sign_flags_##SUF(r.u, r.v);                                                \
    }                                                                                                    \
  }                                                                                                      \
  int kogora_svd2_##SUF(const MT* in, const OT* out, uint64_t n, const kog_options* opt, int threads) {  \
    kog_options d = {1, 0, 0, 0};                                                                        \
    ora_job j = {in, out, opt ? opt : &d, NULL, 0};                                                      \
    ora_parallel(n, threads, svd2_body_##SUF, &j);                                                       \
    return 0;                                                                                            \
  }                                                                                                      \
  static void gen_body_##SUF(void* ctx, uint64_t blk, uint64_t lo, uint64_t hi) {                        \
    (void)blk;                                                                                           \
    const ora_job* j = (const ora_job*)ctx;                                                              \
    const MT* o = (const MT*)j->out;                                                                     \
    for (uint64_t i = lo; i < hi; ++i) {                                                                 \
      const mat_##SUF g = generate_##SUF(j->cfg, j->index0 + i);                                         \
      o->g11[i] = g.g11, o->g12[i] = g.g12, o->g21[i] = g.g21, o->g22[i] = g.g22;                        \
    }                                                                                                    \
  }                                                                                                      \
  int kogora_generate_##SUF(const kog_run_config* c, uint64_t index0, const MT* o, uint64_t n,            \
                            int threads) {                                                               \
    ora_job j = {NULL, o, NULL, c, index0};                                                              \
    ora_parallel(n, threads, gen_body_##SUF, &j);                                                        \
    return 0;                                                                                            \
  }                                                                                                      \
  int kogora_svd2_ext_##SUF(const MT* g, kog_extsvd* o, uint64_t n) {                                    \
    for (uint64_t i = 0; i < n; ++i) {                                                                   \
      const mat_##SUF m = {g->g11[i], g->g12[i], g->g21[i], g->g22[i]};                                  \
      const ora_extsvd r = svd2_ext_##SUF(m);                                                            \
      o[i].sigma1 = ora_c(r.sigma1), o[i].sigma2 = ora_c(r.sigma2);                                      \
      o[i].u[0] = ora_c(r.u.a11), o[i].u[1] = ora_c(r.u.a12), o[i].u[2] = ora_c(r.u.a21);                \
      o[i].u[3] = ora_c(r.u.a22);                                                                        \
      o[i].v[0] = ora_c(r.v.a11), o[i].v[1] = ora_c(r.v.a12), o[i].v[2] = ora_c(r.v.a21);                \
      o[i].v[3] = ora_c(r.v.a22);                                                                        \
    }                                                                                                    \
    return 0;                                                                                            \
  }                                                                                                      \
  static void met_body_##SUF(void* ctx, uint64_t blk, uint64_t lo, uint64_t hi) {                        \
    (void)blk;                                                                                           \
    const ora_job* j = (const ora_job*)ctx;                                                              \
    const MT* in = (const MT*)j->in;                                                                     \
    kog_metrics* o = (kog_metrics*)j->out;                                                               \
    for (uint64_t i = lo; i < hi; ++i) {                                                                 \
      const mat_##SUF g = {in->g11[i], in->g12[i], in->g21[i], in->g22[i]};                              \
      memset(o + i, 0, sizeof o[i]);                                                                     \
      const ora_extsvd ref = svd2_ext_##SUF(g);                                                          \
      const res_##SUF r = svd2_##SUF(g, j->opt);                                                         \
      if (r.err) {                                                                                       \
        o[i].flags = KOG_F_DOMAIN_ERROR;                                                                 \
        continue;                                                                                        \
      }                                                                                                  \
      uint32_t flags = r.flags;                                                                          \
      if (!all_finite_##SUF(r.u) || !all_finite_##SUF(r.v) || !isfinite(r.s1.f) || !isfinite(r.s2.f))   \
        flags |= KOG_M_NONFINITE_FACTOR;                                                                 \
      const ora_metrics m = metrics_##SUF(g, r.u, r.v, ora_ext_from_pair(r.s1.e, (double)r.s1.f),        \
                                          ora_ext_from_pair(r.s2.e, (double)r.s2.f), &ref);              \
      if (isnan(m.reG) || isnan(m.reS1) || isnan(m.reS2) || isnan(m.reU) || isnan(m.reV))               \
        flags |= KOG_M_NAN_METRIC;                                                                       \
      o[i].reG = m.reG, o[i].reS1 = m.reS1, o[i].reS2 = m.reS2, o[i].reU = m.reU, o[i].reV = m.reV;      \
      o[i].kappa2 = ora_c(m.kappa2);                                                                     \
      o[i].kappa_inf = (uint32_t)m.kappa_inf;                                                            \
      o[i].flags = flags;                                                                                \
    }                                                                                                    \
  }                                                                                                      \
  int kogora_metrics_##SUF(const MT* g, kog_metrics* o, uint64_t n, const kog_options* opt, int threads) { \
    kog_options d = {1, 0, 0, 0};                                                                        \
    ora_job j = {g, o, opt ? opt : &d, NULL, 0};                                                         \
    ora_parallel(n, threads, met_body_##SUF, &j);                                                        \
    return 0;                                                                                            \
  }
BATCH_FNS(f64, double, kog_mat_f64, kog_svd_out_f64)
BATCH_FNS(f32, float, kog_mat_f32, kog_svd_out_f32)

/* run_batch (harness.hpp:226-271) with per-block stats and ordered merge */
typedef struct {
  const kog_run_config* cfg;
  ora_stats* blocks;
  uint64_t* fail;  /* per block: UINT64_MAX or index*4 + reason */
} ora_run;

static void run_body(void* ctx, uint64_t blk, uint64_t lo, uint64_t hi) {
  ora_run* r = (ora_run*)ctx;
  for (uint64_t i = lo; i < hi; ++i) {
    const int why = r->cfg->single_precision ? run_one_f32(r->cfg, i, &r->blocks[blk])
                                              : run_one_f64(r->cfg, i, &r->blocks[blk]);
    if (why) {
      r->fail[blk] = i * 4 + (uint64_t)why;
      return;
    }
  }
}

static void ora_to_c(const ora_stats* s, kog_stats* o) {
  memset(o, 0, sizeof *o);
  o->reG = s->reG, o->reS1 = s->reS1, o->reS2 = s->reS2, o->reU = s->reU, o->reV = s->reV;
  o->max_kappa2 = ora_c(s->maxKappa2);
  o->kappa_inf = (uint64_t)s->kappa_inf;
  for (int i = 0; i < 7; ++i) o->t2p[i] = s->t2p[i], o->path[i] = s->path[i];
  o->tanpsi_inf = s->tanpsi_inf, o->diag_swap = s->diag_swap, o->compose_minus = s->compose_minus;
  o->sigma_swap = s->sigma_swap, o->prescale_inexact = s->prescale_inexact;
  o->fail_key = UINT64_MAX;
}

int kogora_run_batch(const kog_run_config* c, kog_stats* out) {
  const int emin = c->single_precision ? -126 : -1022, emax = c->single_precision ? 127 : 1023;
  if (c->routine == KOG_ROUTINE_LASV2 && c->shape != KOG_SHAPE_TRI) {
    snprintf(g_err, sizeof g_err, "lasv2 accepts triangular inputs only");
    return -1;
  }
  if (c->regime == KOG_REGIME_SIGMA) {
    if (c->varsigma < 1) {
      snprintf(g_err, sizeof g_err, "sigma regime needs varsigma >= 1");
      return -1;
    }
    if (emin + c->varsigma > emax - 2) {
      snprintf(g_err, sizeof g_err, "varsigma exceeds the exponent range");
      return -1;
    }
  }
  const uint64_t nb = (c->count + 4095) / 4096;
  ora_run r;
  r.cfg = c;
  r.blocks = (ora_stats*)calloc(nb ? nb : 1, sizeof(ora_stats));
  r.fail = (uint64_t*)malloc(sizeof(uint64_t) * (nb ? nb : 1));
  for (uint64_t b = 0; b < nb; ++b) r.fail[b] = UINT64_MAX;
  ora_parallel(c->count, c->threads, run_body, &r);
  ora_stats total;
  memset(&total, 0, sizeof total);
  int rc = 0;
  for (uint64_t b = 0; b < nb; ++b) {
    if (r.fail[b] != UINT64_MAX) {
      snprintf(g_err, sizeof g_err, "%s at index %" PRIu64, (r.fail[b] & 3) == 1 ? "non-finite factor" : "NaN metric",
               r.fail[b] / 4);
      rc = -4;
      break;
    }
    ora_stats_merge(&total, &r.blocks[b]);
  }
  ora_to_c(&total, out);
  free(r.blocks);
  free(r.fail);
  return rc;
}

/* ------------------------------------------- CSV row (harness.hpp:276-317) */
/* shortest round-trip decimal, as std::to_chars(double) prints it: the
 * fewest significant digits that round-trip, in whichever of fixed or
 * scientific notation is shorter (fixed on ties) */
static void ora_shortest(double x, char* out, size_t cap) {
  char sci[40];
  int prec;
  for (prec = 1; prec <= 17; ++prec) {
    snprintf(sci, sizeof sci, "%.*e", prec - 1, x);
    if (strtod(sci, NULL) == x) break;
  }
  /* digits and exponent of the scientific form */
  char digits[32];
  int nd = 0, neg = 0;
  const char* p = sci;
  if (*p == '-') {
    neg = 1;
    ++p;
  }
  for (; *p && *p != 'e'; ++p)
    if (*p >= '0' && *p <= '9') digits[nd++] = *p;
  digits[nd] = 0;
  const int exp10 = atoi(p + 1);
  while (nd > 1 && digits[nd - 1] == '0') digits[--nd] = 0;
  /* scientific candidate: d[.ddd]e[+-]XX (at least two exponent digits) */
  char s1[48], s2[400];
  int k = 0;
  if (neg) s1[k++] = '-';
  s1[k++] = digits[0];
  if (nd > 1) {
    s1[k++] = '.';
    for (int i = 1; i < nd; ++i) s1[k++] = digits[i];
  }
  snprintf(s1 + k, sizeof s1 - (size_t)k, "e%c%02d", exp10 < 0 ? '-' : '+', exp10 < 0 ? -exp10 : exp10);
  /* fixed candidate */
  k = 0;
  if (neg) s2[k++] = '-';
  if (exp10 >= 0) {
    for (int i = 0; i <= exp10 || i < nd; ++i) {
      if (i == exp10 + 1) s2[k++] = '.';
      s2[k++] = i < nd ? digits[i] : '0';
    }
  } else {
    s2[k++] = '0';
    s2[k++] = '.';
    for (int i = 0; i < -exp10 - 1; ++i) s2[k++] = '0';
    for (int i = 0; i < nd; ++i) s2[k++] = digits[i];
  }
  s2[k] = 0;
  snprintf(out, cap, "%s", strlen(s2) <= strlen(s1) ? s2 : s1);
}

static void ora_ext_to_decimal(ora_ext a, char* out, size_t cap) { /* extfloat.hpp:159-179 */
  if (ora_ext_is_zero(a)) {
    snprintf(out, cap, "0");
    return;
  }
  const double l10 = (double)a.e * 0.30102999566398119521 + log10(fabs(a.hi + a.lo));
  int64_t d10 = (int64_t)floor(l10);
  const ora_ext m = ora_ext_mul(a, ora_ext_pow10(-d10));
  double md = ora_ext_to_double(m);
  if (fabs(md) >= 10.0) {
    md /= 10.0;
    ++d10;
  } else if (fabs(md) < 1.0) {
    md *= 10.0;
    --d10;
  }
  snprintf(out, cap, "%.17ge%+lld", md, (long long)d10);
}

int kogora_csv_row(const kog_run_config* c, const kog_stats* st, char* buf, size_t cap) {
  char v[5][48], k[64];
  const double vals[5] = {st->reG, st->reS1, st->reS2, st->reU, st->reV};
  for (int i = 0; i < 5; ++i) ora_shortest(vals[i], v[i], sizeof v[i]);
  const ora_ext kap = {st->max_kappa2.e, st->max_kappa2.hi, st->max_kappa2.lo};
  if (st->kappa_inf)
    snprintf(k, sizeof k, "inf");
  else if (kap.e > -1000 && kap.e < 1000)
    ora_shortest(ora_ext_to_double(kap), k, sizeof k);
  else
    ora_ext_to_decimal(kap, k, sizeof k);
  const char* regime = c->regime == KOG_REGIME_CIRC ? "circ"
                       : c->regime == KOG_REGIME_BULLET ? "bullet"
                       : c->regime == KOG_REGIME_SIGMA  ? "sigma"
                                                        : "ranged";
  const int len = snprintf(buf, cap, "%s,%s,%s,%d,%" PRIu64 ",%016" PRIx64 ",%s,%s,%s,%s,%s,%s,%s",
                           c->single_precision ? "single" : "double", c->shape == KOG_SHAPE_TRI ? "tri" : "gen",
                           regime, c->varsigma, c->count, c->seed, c->routine == KOG_ROUTINE_KOG ? "kog" : "lasv2",
                           v[0], v[1], v[2], v[3], v[4], k);
  return (len < 0 || (size_t)len >= cap) ? -1 : len;
}
