// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// oracle/_ref/libkogref.so: the UNMODIFIED reference headers
// (/root/reference/proj/include/kogsvd2, included in place with -I, never
// copied) behind an extern "C" surface shaped like include/kog2.h, but on HOST
// arrays.  Built by oracle/Makefile with the reference's Release flags
// (proj/CMakeLists.txt:8-15: -std=c++20 -O3 -DNDEBUG -ffp-contract=off).
// Used by tests/ to pin the C restatement (oracle/kog_oracle.c) and to generate
// the golden fixtures under tests/golden/, and by bench.py's reference arm.
//
// The only non-reference logic here is (a) packing BranchTrace into the kog2
// flags word, (b) the kog2 generator extension for BASELINE configs 2-5
// (SURVEY.md §8d), written on top of the reference's own Stream
// (harness.hpp:114-128), and (c) thread-pool loops mirroring harness.hpp:226-271.

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "kogsvd2/kogsvd2.hpp"
#include "kog2.h"

using namespace kogsvd2;

namespace {

template <class T>
struct MatT;
template <>
struct MatT<double> { using type = kog_mat_f64; using out = kog_svd_out_f64; };
template <>
struct MatT<float> { using type = kog_mat_f32; using out = kog_svd_out_f32; };

template <class T>
Matrix2<T> load(const typename MatT<T>::type* m, uint64_t i) {
  return Matrix2<T>{m->g11[i], m->g12[i], m->g21[i], m->g22[i]};
}

uint32_t pack_trace(const BranchTrace& t) {
  uint32_t f = 0;
  f |= uint32_t(t.path) << KOG_F_PATH_SHIFT;
  f |= uint32_t(t.t2p) << KOG_F_T2P_SHIFT;
  if (t.tanpsi_inf) f |= KOG_F_TANPSI_INF;
  if (t.diag_swap) f |= KOG_F_DIAG_SWAP;
  if (t.sigma_swap) f |= KOG_F_SIGMA_SWAP;
  if (t.compose_minus) f |= KOG_F_COMPOSE_MINUS;
  if (t.prescale_inexact) f |= KOG_F_PRESCALE_INEXACT;
  if (t.urv_col_swap) f |= KOG_F_URV_COL_SWAP;
  if (t.urv_row_swap) f |= KOG_F_URV_ROW_SWAP;
  f |= uint32_t(t.type_initial) << KOG_F_TYPE_INIT_SHIFT;
  f |= uint32_t(t.type_scaled) << KOG_F_TYPE_SCALED_SHIFT;
  return f;
}

Options to_opt(const kog_options* o) {
  Options r;
  if (o) {
    r.hypot_is_cr = o->hypot_is_cr != 0;
    r.ominus_for_d = o->ominus_for_d != 0;
    r.wide_channel = o->wide_channel ? WideChannel::kahan_det : WideChannel::wider_type;
  }
  return r;
}

template <class F>
void parallel_blocks(uint64_t n, int threads, F&& body) {
  constexpr uint64_t kBlock = 4096;
  const uint64_t nblocks = (n + kBlock - 1) / kBlock;
  int workers = threads;
  if (workers <= 0) workers = int(std::thread::hardware_concurrency());
  if (workers < 1) workers = 1;
  if (uint64_t(workers) > nblocks && nblocks > 0) workers = int(nblocks);
  std::atomic<uint64_t> next{0};
  auto work = [&]() {
    for (;;) {
      const uint64_t b = next.fetch_add(1, std::memory_order_relaxed);
      if (b >= nblocks) return;
      const uint64_t lo = b * kBlock, hi = std::min(n, lo + kBlock);
      body(b, lo, hi);
    }
  };
  if (workers <= 1 || nblocks <= 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int i = 0; i < workers; ++i) pool.emplace_back(work);
    for (auto& t : pool) t.join();
  }
}

template <class T>
int svd2_soa(const typename MatT<T>::type* in, const typename MatT<T>::out* out, uint64_t n,
             const kog_options* o, int threads) {
  const Options opt = to_opt(o);
  std::atomic<int> errors{0};
  parallel_blocks(n, threads, [&](uint64_t, uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      const Matrix2<T> g = load<T>(in, i);
      uint32_t flags = 0;
      Svd2Result<T> r;
      try {
        r = svd2(g, opt);
        flags = pack_trace(r.trace);
      } catch (const std::exception&) {
        flags = KOG_F_DOMAIN_ERROR;
        errors.fetch_add(1);
      }
      if (std::signbit(r.u.g21)) flags |= KOG_F_SIGN_U21;
      if (std::signbit(r.u.g22)) flags |= KOG_F_SIGN_U22;
      if (std::signbit(r.v.g21)) flags |= KOG_F_SIGN_V21;
      if (std::signbit(r.v.g22)) flags |= KOG_F_SIGN_V22;
      out->sig1_f[i] = r.sigma1.f;
      out->sig2_f[i] = r.sigma2.f;
      out->sig1_e[i] = int32_t(r.sigma1.e);
      out->sig2_e[i] = int32_t(r.sigma2.e);
      out->u11[i] = r.u.g11;
      out->u12[i] = r.u.g12;
      out->v11[i] = r.v.g11;
      out->v12[i] = r.v.g12;
      out->s[i] = int32_t(r.s);
      out->flags[i] = flags;
    }
  });
  return errors.load();
}

// ---- kog2 generator extension on the reference Stream -----
RunConfig to_rc(const kog_run_config* c) {
  RunConfig r;
  r.single_precision = c->single_precision != 0;
  r.shape = c->shape == KOG_SHAPE_TRI ? Shape::tri : Shape::gen;
  r.regime = c->regime == KOG_REGIME_CIRC ? Regime::circ
             : c->regime == KOG_REGIME_BULLET ? Regime::bullet
                                                : Regime::sigma;
  r.varsigma = c->varsigma;
  r.count = c->count;
  r.seed = c->seed;
  r.routine = c->routine == KOG_ROUTINE_LASV2 ? Routine::lasv2 : Routine::kog;
  r.threads = c->threads;
  r.options = to_opt(&c->options);
  return r;
}

template <class T>
Matrix2<T> gen_any(const kog_run_config* c, uint64_t index) {
  if (c->regime != KOG_REGIME_RANGED) return generate<T>(to_rc(c), index);
  harness_detail::Stream st(c->seed, index);
  constexpr int p = sig_digits<T>;
  auto ranged = [&](int elo, int ehi) {  // same draw rule as harness.hpp:150-156
    const uint64_t u = st.next();
    const int e = elo + int(u % uint64_t(ehi - elo + 1));
    const T f = T(1) + std::scalbn(T(st.next() >> (64 - (p - 1))), 1 - p);
    const T v = std::scalbn(f, e);
    return (u >> 63) ? -v : v;
  };
  auto element = [&]() {
    if (c->tail_mod != 0) {
      const uint64_t t = st.next();
      if (t % c->tail_mod == 0) return ranged(c->tail_lo, c->tail_hi);
    }
    return ranged(c->elo, c->ehi);
  };
  auto nonzero = [&]() {  // harness.hpp:167-171
    T v = element();
    while (v == T(0)) v = element();
    return v;
  };
  Matrix2<T> g;
  if (c->shape == KOG_SHAPE_TRI) {
    g.g11 = nonzero();
    g.g12 = element();
    g.g21 = T(0);
    g.g22 = nonzero();
  } else {
    g.g11 = element();
    g.g12 = element();
    g.g21 = element();
    g.g22 = element();
  }
  if (c->zero_mask_rule) {
    const uint64_t z = st.next();
    if ((z & 7) == 0) {
      const unsigned m = unsigned(z >> 3) & 15;
      if (m & 1) g.g11 = T(0);
      if (m & 2) g.g21 = T(0);
      if (m & 4) g.g12 = T(0);
      if (m & 8) g.g22 = T(0);
    }
  }
  return g;
}

kog_extfloat to_c(const ExtFloat& x) { return kog_extfloat{x.e, x.hi, x.lo}; }

void stats_to_c(const ErrorStats& s, kog_stats* o) {
  std::memset(o, 0, sizeof *o);
  o->reG = s.reG;
  o->reS1 = s.reS1;
  o->reS2 = s.reS2;
  o->reU = s.reU;
  o->reV = s.reV;
  o->max_kappa2 = to_c(s.maxKappa2);
  o->kappa_inf = s.kappa_inf;
  for (int i = 0; i < 7; ++i) {
    o->t2p[i] = s.counts.t2p[i];
    o->path[i] = s.counts.path[i];
  }
  o->tanpsi_inf = s.counts.tanpsi_inf;
  o->diag_swap = s.counts.diag_swap;
  o->compose_minus = s.counts.compose_minus;
  o->sigma_swap = s.counts.sigma_swap;
  o->prescale_inexact = s.counts.prescale_inexact;
  o->fail_key = UINT64_MAX;
}

ErrorStats stats_from_c(const kog_stats* o) {
  ErrorStats s;
  s.reG = o->reG;
  s.reS1 = o->reS1;
  s.reS2 = o->reS2;
  s.reU = o->reU;
  s.reV = o->reV;
  s.maxKappa2 = ExtFloat{o->max_kappa2.e, o->max_kappa2.hi, o->max_kappa2.lo};
  s.kappa_inf = o->kappa_inf != 0;
  for (int i = 0; i < 7; ++i) {
    s.counts.t2p[i] = o->t2p[i];
    s.counts.path[i] = o->path[i];
  }
  s.counts.tanpsi_inf = o->tanpsi_inf;
  s.counts.diag_swap = o->diag_swap;
  s.counts.compose_minus = o->compose_minus;
  s.counts.sigma_swap = o->sigma_swap;
  s.counts.prescale_inexact = o->prescale_inexact;
  return s;
}

// run_one/run_batch for the extended regime: the reference's own per-matrix
// body (harness.hpp:190-222) over the extended generator.
template <class T>
ErrorStats run_ext(const kog_run_config* c, std::string& fail, uint64_t index0 = 0, uint64_t count = UINT64_MAX) {
  const RunConfig cfg = to_rc(c);
  const uint64_t n = count == UINT64_MAX ? c->count : count;
  constexpr uint64_t kBlock = 4096;
  const uint64_t nblocks = (n + kBlock - 1) / kBlock;
  std::vector<ErrorStats> bs(nblocks);
  std::vector<std::string> bf(nblocks);
  parallel_blocks(n, c->threads, [&](uint64_t b, uint64_t lo, uint64_t hi) {
    for (uint64_t i = index0 + lo; i < index0 + hi; ++i) {
      const Matrix2<T> g = gen_any<T>(c, i);
      const ExtSvd ref = svd2_ext(g);
      auto failmsg = [&](const char* what) {
        using harness_detail::bits_of;
        return std::string(what) + " at index " + std::to_string(i) + ": g = [" + bits_of(g.g11) +
               ", " + bits_of(g.g12) + "; " + bits_of(g.g21) + ", " + bits_of(g.g22) + "]";
      };
      ErrorMetrics m;
      if (cfg.routine == Routine::kog) {
        const Svd2Result<T> r = svd2(g, cfg.options);
        if (!all_finite(r.u) || !all_finite(r.v) || !std::isfinite(r.sigma1.f) ||
            !std::isfinite(r.sigma2.f)) {
          bf[b] = failmsg("non-finite factor");
          return;
        }
        m = metrics(g, r.u, r.v, ext_from(r.sigma1), ext_from(r.sigma2), ref);
        if (std::isnan(m.reG) || std::isnan(m.reS1) || std::isnan(m.reS2) || std::isnan(m.reU) ||
            std::isnan(m.reV)) {
          bf[b] = failmsg("NaN metric");
          return;
        }
        bs[b].absorb(m, &r.trace);
      } else {
        const Lasv2Out<T> r = lasv2_ref(g.g11, g.g12, g.g22);
        const Matrix2<T> u{r.csl, -r.snl, r.snl, r.csl};
        const Matrix2<T> v{r.csr, -r.snr, r.snr, r.csr};
        if (!all_finite(u) || !all_finite(v) || !std::isfinite(r.ssmax) ||
            !std::isfinite(r.ssmin)) {
          bf[b] = failmsg("non-finite factor");
          return;
        }
        m = metrics(g, u, v, ext_from(r.ssmax), ext_from(r.ssmin), ref);
        if (std::isnan(m.reG) || std::isnan(m.reS1) || std::isnan(m.reS2) || std::isnan(m.reU) ||
            std::isnan(m.reV)) {
          bf[b] = failmsg("NaN metric");
          return;
        }
        bs[b].absorb(m, nullptr);
      }
    }
  });
  ErrorStats total;
  for (uint64_t b = 0; b < nblocks; ++b) {
    if (!bf[b].empty()) {
      fail = bf[b];
      return total;
    }
    total.merge(bs[b]);
  }
  return total;
}

thread_local std::string g_err;

template <class T>
void metrics_one(const Matrix2<T>& g, const Options& opt, kog_metrics* o) {
  std::memset(o, 0, sizeof *o);
  try {
    const ExtSvd ref = svd2_ext(g);
    const Svd2Result<T> r = svd2(g, opt);
    o->flags = pack_trace(r.trace);
    if (!all_finite(r.u) || !all_finite(r.v) || !std::isfinite(r.sigma1.f) ||
        !std::isfinite(r.sigma2.f))
      o->flags |= KOG_M_NONFINITE_FACTOR;
    const ErrorMetrics m = metrics(g, r.u, r.v, ext_from(r.sigma1), ext_from(r.sigma2), ref);
    o->reG = m.reG;
    o->reS1 = m.reS1;
    o->reS2 = m.reS2;
    o->reU = m.reU;
    o->reV = m.reV;
    o->kappa2 = to_c(m.kappa2);
    o->kappa_inf = m.kappa_inf;
    if (std::isnan(m.reG) || std::isnan(m.reS1) || std::isnan(m.reS2) || std::isnan(m.reU) ||
        std::isnan(m.reV))
      o->flags |= KOG_M_NAN_METRIC;
  } catch (const std::exception&) {
    o->flags |= KOG_F_DOMAIN_ERROR;
  }
}

template <class T>
void ext_svd_one(const Matrix2<T>& g, kog_extsvd* o) {
  std::memset(o, 0, sizeof *o);
  const ExtSvd r = svd2_ext(g);
  o->sigma1 = to_c(r.sigma1);
  o->sigma2 = to_c(r.sigma2);
  o->u[0] = to_c(r.u.a11);
  o->u[1] = to_c(r.u.a12);
  o->u[2] = to_c(r.u.a21);
  o->u[3] = to_c(r.u.a22);
  o->v[0] = to_c(r.v.a11);
  o->v[1] = to_c(r.v.a12);
  o->v[2] = to_c(r.v.a21);
  o->v[3] = to_c(r.v.a22);
}

template <class T, class Rec>
void urv_one(const Matrix2<T>& g, const Options& opt, Rec* o) {
  std::memset(o, 0, sizeof *o);
  const auto u = urv15(g, opt);
  o->gppp[0] = u.gppp.g11;
  o->gppp[1] = u.gppp.g12;
  o->gppp[2] = u.gppp.g21;
  o->gppp[3] = u.gppp.g22;
  o->tan_theta = u.tan_theta;
  o->sec_theta = u.sec_theta;
  o->r11 = u.r11;
  o->r12_raw = u.r12_raw;
  o->r22_raw = u.r22_raw;
  o->r[0] = u.r.g11;
  o->r[1] = u.r.g12;
  o->r[2] = u.r.g21;
  o->r[3] = u.r.g22;
  o->sr0 = u.sr0;
  o->sr1 = u.sr1;
  o->s12 = u.s12;
  o->s22 = u.s22;
  o->col_swap = u.col_swap;
  o->row_swap = u.row_swap;
  o->ext_is_r22 = u.ext_is_r22;
  o->next = uint8_t(u.next);
}

template <class T, class Rec>
void trisvd_one(T r11, T r12, T r22, bool t13, const Options& opt, Rec* o) {
  std::memset(o, 0, sizeof *o);
  const Matrix2<T> rt{r11, r12, T(0), r22};
  try {
    Tan2PhiBranch br = Tan2PhiBranch::none;
    o->t2f = tan2phi(rt, t13, opt, br);
    const auto ts = tri_svd(rt, t13, opt);
    o->tan_phi = ts.tan_phi;
    o->sec_phi = ts.sec_phi;
    o->cos_phi = ts.cos_phi;
    o->sin_phi = ts.sin_phi;
    o->tan_psi = ts.tan_psi;
    o->sec_psi = ts.sec_psi;
    o->cos_psi = ts.cos_psi;
    o->sin_psi = ts.sin_psi;
    o->sig1_f = ts.sig1.f;
    o->sig2_f = ts.sig2.f;
    o->sig1_e = ts.sig1.e;
    o->sig2_e = ts.sig2.e;
    o->sigma_swapped = ts.sigma_swapped;
    o->tanpsi_inf = ts.tanpsi_inf;
    o->t2p = uint8_t(ts.t2p);
  } catch (const std::exception&) {
    o->status = 1;
  }
}

template <class T>
void epair_one(int op, int64_t xe, T xf, int64_t ye, T yf, int64_t* oe, T* of, uint8_t* st) {
  *st = 0;
  *oe = 0;
  *of = T(0);
  try {
    EPair<T> r;
    switch (op) {
      case KOG_EPAIR_OPLUS: r = oplus(xf, yf); break;
      case KOG_EPAIR_OMINUS: r = ominus(xf, yf); break;
      case KOG_EPAIR_MUL: r = EPair<T>(xe, xf) * EPair<T>(ye, yf); break;
      case KOG_EPAIR_DIV: r = EPair<T>(xe, xf) / EPair<T>(ye, yf); break;
      case KOG_EPAIR_LESS:
        *of = less(EPair<T>(xe, xf), EPair<T>(ye, yf)) ? T(1) : T(0);
        return;
      case KOG_EPAIR_RECIP: r = recip(EPair<T>(xe, xf)); break;
      case KOG_EPAIR_MAKE: r = EPair<T>(xe, xf); break;
      default: *st = 2; return;
    }
    *oe = r.e;
    *of = r.f;
  } catch (const std::exception&) {
    *st = 1;
  }
}

}  // namespace

extern "C" {

const char* kogref_last_error(void) { return g_err.c_str(); }

int kogref_hypot_f64(const double* a, const double* b, double* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) o[i] = hypot_cr(a[i], b[i]);
  return 0;
}
int kogref_hypot_f32(const float* a, const float* b, float* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) o[i] = hypot_cr(a[i], b[i]);
  return 0;
}
int kogref_split_f64(const double* x, int64_t* e, double* f, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    const auto s = split(x[i]);
    e[i] = s.e;
    f[i] = s.f;
  }
  return 0;
}
int kogref_split_f32(const float* x, int64_t* e, float* f, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    const auto s = split(x[i]);
    e[i] = s.e;
    f[i] = s.f;
  }
  return 0;
}
int kogref_assemble_f64(const int64_t* e, const double* f, double* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) o[i] = assemble(e[i], f[i]);
  return 0;
}
int kogref_assemble_f32(const int64_t* e, const float* f, float* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) o[i] = assemble(e[i], f[i]);
  return 0;
}
int kogref_tan2_f64(const double* t, double* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) o[i] = tan_from_double_angle(t[i]);
  return 0;
}
int kogref_tan2_f32(const float* t, float* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) o[i] = tan_from_double_angle(t[i]);
  return 0;
}
int kogref_sec_f64(const double* t, double* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) o[i] = sec_from_tan(t[i]);
  return 0;
}
int kogref_sec_f32(const float* t, float* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) o[i] = sec_from_tan(t[i]);
  return 0;
}
int kogref_epair_f64(int op, const int64_t* xe, const double* xf, const int64_t* ye,
                     const double* yf, int64_t* oe, double* of, uint8_t* st, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    epair_one<double>(op, xe ? xe[i] : 0, xf[i], ye ? ye[i] : 0, yf ? yf[i] : 0.0, oe + i, of + i,
                      st + i);
  return 0;
}
int kogref_epair_f32(int op, const int64_t* xe, const float* xf, const int64_t* ye,
                     const float* yf, int64_t* oe, float* of, uint8_t* st, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    epair_one<float>(op, xe ? xe[i] : 0, xf[i], ye ? ye[i] : 0, yf ? yf[i] : 0.0f, oe + i, of + i,
                     st + i);
  return 0;
}

#define KOGREF_CLASSIFY(T, SUF)                                                            \
  int kogref_classify_prescale_##SUF(const MatT<T>::type* in, const kog_classify_out* o,  \
                                     const MatT<T>::type* gp, uint64_t n) {                \
    for (uint64_t i = 0; i < n; ++i) {                                                     \
      const Matrix2<T> g = load<T>(in, i);                                                 \
      o->status[i] = 0;                                                                    \
      try {                                                                                \
        const TypeInfo info = classify(g);                                                 \
        o->t[i] = info.t;                                                                  \
        o->s_type[i] = info.s_type;                                                        \
        o->s[i] = info.s;                                                                  \
        o->e_G[i] = info.e_G;                                                              \
        const auto pr = prescale(g, info);                                                 \
        o->inexact_underflow[i] = pr.inexact_underflow;                                    \
        gp->g11[i] = pr.gp.g11;                                                            \
        gp->g12[i] = pr.gp.g12;                                                            \
        gp->g21[i] = pr.gp.g21;                                                            \
        gp->g22[i] = pr.gp.g22;                                                            \
      } catch (const std::exception&) {                                                    \
        o->status[i] = 1;                                                                  \
      }                                                                                    \
    }                                                                                      \
    return 0;                                                                              \
  }
KOGREF_CLASSIFY(double, f64)
KOGREF_CLASSIFY(float, f32)

int kogref_urv15_f64(const kog_mat_f64* g, kog_urv15_f64* o, uint64_t n, const kog_options* opt) {
  const Options op = to_opt(opt);
  for (uint64_t i = 0; i < n; ++i) urv_one<double>(load<double>(g, i), op, o + i);
  return 0;
}
int kogref_urv15_f32(const kog_mat_f32* g, kog_urv15_f32* o, uint64_t n, const kog_options* opt) {
  const Options op = to_opt(opt);
  for (uint64_t i = 0; i < n; ++i) urv_one<float>(load<float>(g, i), op, o + i);
  return 0;
}
int kogref_tri_svd_f64(const double* a, const double* b, const double* c, const uint8_t* t13,
                       kog_trisvd_f64* o, uint64_t n, const kog_options* opt) {
  const Options op = to_opt(opt);
  for (uint64_t i = 0; i < n; ++i) trisvd_one<double>(a[i], b[i], c[i], t13[i] != 0, op, o + i);
  return 0;
}
int kogref_tri_svd_f32(const float* a, const float* b, const float* c, const uint8_t* t13,
                       kog_trisvd_f32* o, uint64_t n, const kog_options* opt) {
  const Options op = to_opt(opt);
  for (uint64_t i = 0; i < n; ++i) trisvd_one<float>(a[i], b[i], c[i], t13[i] != 0, op, o + i);
  return 0;
}
int kogref_compose_left_f64(const double* tp, const double* tt, const uint8_t* m, double* c,
                            double* s, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    const auto r = compose_left(tp[i], tt[i], m[i] != 0);
    c[i] = r.c;
    s[i] = r.s;
  }
  return 0;
}
int kogref_compose_left_f32(const float* tp, const float* tt, const uint8_t* m, float* c,
                            float* s, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    const auto r = compose_left(tp[i], tt[i], m[i] != 0);
    c[i] = r.c;
    s[i] = r.s;
  }
  return 0;
}

#define KOGREF_TRI13(T, SUF)                                                                    \
  int kogref_triangularize13_##SUF(const MatT<T>::type* g, const uint8_t* t,                   \
                                   const MatT<T>::type* r, int8_t* up, int8_t* vp, uint64_t n) { \
    for (uint64_t i = 0; i < n; ++i) {                                                          \
      const auto f = triangularize13(load<T>(g, i), t[i]);                                      \
      r->g11[i] = f.r.g11;                                                                      \
      r->g12[i] = f.r.g12;                                                                      \
      r->g21[i] = f.r.g21;                                                                      \
      r->g22[i] = f.r.g22;                                                                      \
      for (int k = 0; k < 4; ++k) {                                                             \
        up[4 * i + k] = f.uplus.m[k / 2][k % 2];                                                \
        vp[4 * i + k] = f.vplus.m[k / 2][k % 2];                                                \
      }                                                                                         \
    }                                                                                           \
    return 0;                                                                                   \
  }
KOGREF_TRI13(double, f64)
KOGREF_TRI13(float, f32)

int kogref_svd2_f64(const kog_mat_f64* in, const kog_svd_out_f64* out, uint64_t n,
                    const kog_options* opt, int threads) {
  return svd2_soa<double>(in, out, n, opt, threads);
}
int kogref_svd2_f32(const kog_mat_f32* in, const kog_svd_out_f32* out, uint64_t n,
                    const kog_options* opt, int threads) {
  return svd2_soa<float>(in, out, n, opt, threads);
}

int kogref_svd2_ext_f64(const kog_mat_f64* g, kog_extsvd* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) ext_svd_one<double>(load<double>(g, i), o + i);
  return 0;
}
int kogref_svd2_ext_f32(const kog_mat_f32* g, kog_extsvd* o, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) ext_svd_one<float>(load<float>(g, i), o + i);
  return 0;
}
int kogref_metrics_f64(const kog_mat_f64* g, kog_metrics* o, uint64_t n, const kog_options* opt,
                       int threads) {
  const Options op = to_opt(opt);
  parallel_blocks(n, threads, [&](uint64_t, uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) metrics_one<double>(load<double>(g, i), op, o + i);
  });
  return 0;
}
int kogref_metrics_f32(const kog_mat_f32* g, kog_metrics* o, uint64_t n, const kog_options* opt,
                       int threads) {
  const Options op = to_opt(opt);
  parallel_blocks(n, threads, [&](uint64_t, uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) metrics_one<float>(load<float>(g, i), op, o + i);
  });
  return 0;
}

int kogref_generate_f64(const kog_run_config* c, uint64_t index0, const kog_mat_f64* o,
                        uint64_t n, int threads) {
  parallel_blocks(n, threads, [&](uint64_t, uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      const auto g = gen_any<double>(c, index0 + i);
      o->g11[i] = g.g11;
      o->g12[i] = g.g12;
      o->g21[i] = g.g21;
      o->g22[i] = g.g22;
    }
  });
  return 0;
}
int kogref_generate_f32(const kog_run_config* c, uint64_t index0, const kog_mat_f32* o,
                        uint64_t n, int threads) {
  parallel_blocks(n, threads, [&](uint64_t, uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      const auto g = gen_any<float>(c, index0 + i);
      o->g11[i] = g.g11;
      o->g12[i] = g.g12;
      o->g21[i] = g.g21;
      o->g22[i] = g.g22;
    }
  });
  return 0;
}

// run_batch_any (harness.hpp:319-321) for the reference regimes; the same
// per-matrix body over the extended generator for KOG_REGIME_RANGED.
// Returns 0, or -1 (invalid config) / -4 (BatchAbort) with the message.
int kogref_run_batch(const kog_run_config* c, kog_stats* out) {
  try {
    ErrorStats st;
    if (c->regime != KOG_REGIME_RANGED) {
      st = run_batch_any(to_rc(c));
    } else {
      std::string fail;
      st = c->single_precision ? run_ext<float>(c, fail) : run_ext<double>(c, fail);
      if (!fail.empty()) {
        g_err = fail;
        return -4;
      }
    }
    stats_to_c(st, out);
    return 0;
  } catch (const BatchAbort& e) {
    g_err = e.what();
    return -4;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  }
}

// the reference's run_one body over indices [index0, index0 + n) in 4096-blocks
// merged in order (harness.hpp:190-271 on a sub-range): one shard of a study
int kogref_run_range(const kog_run_config* c, uint64_t index0, uint64_t n, kog_stats* out) {
  std::string fail;
  const ErrorStats st = c->single_precision ? run_ext<float>(c, fail, index0, n) : run_ext<double>(c, fail, index0, n);
  if (!fail.empty()) {
    g_err = fail;
    return -4;
  }
  stats_to_c(st, out);
  return 0;
}

int kogref_csv_row(const kog_run_config* c, const kog_stats* st, char* buf, size_t cap) {
  RunConfig rc = to_rc(c);
  std::string row = csv_row(rc, stats_from_c(st));
  if (c->regime == KOG_REGIME_RANGED) {  // the extension has no reference name
    const size_t a = row.find(',', row.find(',') + 1) + 1, b = row.find(',', a);
    row.replace(a, b - a, "ranged");
  }
  if (row.size() + 1 > cap) return -1;
  std::memcpy(buf, row.c_str(), row.size() + 1);
  return int(row.size());
}

int kogref_lasv2_f64(const double* f, const double* g, const double* h, double* o6, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    const auto r = lasv2_ref(f[i], g[i], h[i]);
    double* o = o6 + 6 * i;
    o[0] = r.ssmin; o[1] = r.ssmax; o[2] = r.snr; o[3] = r.csr; o[4] = r.snl; o[5] = r.csl;
  }
  return 0;
}
int kogref_lasv2_f32(const float* f, const float* g, const float* h, float* o6, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    const auto r = lasv2_ref(f[i], g[i], h[i]);
    float* o = o6 + 6 * i;
    o[0] = r.ssmin; o[1] = r.ssmax; o[2] = r.snr; o[3] = r.csr; o[4] = r.snl; o[5] = r.csl;
  }
  return 0;
}

unsigned kogref_hardware_threads(void) { return std::thread::hardware_concurrency(); }

}  // extern "C"
