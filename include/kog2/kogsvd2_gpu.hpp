// kogsvd2_gpu.hpp — the per-matrix C++ drop-in for the kogsvd2 library on the
// GPU build ("a C++ shim keeps the reference per-matrix
// signatures ... so that tests and harness code recompile unchanged").
//
// Header-only C++20 over the C-ABI of include/kog2.h (link -lkog2; no CUDA
// headers or runtime needed by the caller).  It works on the reference's OWN
// types — Matrix2, Svd2Result, EPair, BranchTrace, Options, ExtFloat, ExtMat,
// ExtSvd, ErrorMetrics, RunConfig, ErrorStats, BatchAbort — so it is included
// after the reference's umbrella header (compile with -I <kogsvd2>/include and
// -I <kog2>/include):
//
//   #include "kogsvd2/kogsvd2.hpp"        // reference types (and CPU routines)
//   #include "kog2/kogsvd2_gpu.hpp"       // the same routines on the GPU
//   namespace ks = kogsvd2::gpu;          // or kogsvd2 for the CPU build
//   auto r = ks::svd2(kogsvd2::Matrix2<double>{4, 3, 0, 2});
//
// Every reference routine below keeps its per-matrix signature and gains
// std::span / std::vector batch overloads (one device round trip per batch):
//
//   svd2       svd2.hpp:603-604      Svd2Result<T> svd2(const Matrix2<T>&, const Options& = {})
//   hypot_cr   fpcore.hpp:140-141    T hypot_cr(T, T)
//   svd2_ext   oracle.hpp:102-103    ExtSvd svd2_ext(const Matrix2<T>&)
//   generate   harness.hpp:139-141   Matrix2<T> generate(const RunConfig&, uint64_t index)
//   run_batch  harness.hpp:225-226   ErrorStats run_batch<T>(const RunConfig&)
//   run_batch_any                    harness.hpp:319-321
//   csv_row    harness.hpp:290       std::string csv_row(const RunConfig&, const ErrorStats&)
//   metrics    run_one's evaluation of svd2(g) against svd2_ext(g)
//              (harness.hpp:200-208 with oracle.hpp:269-301): ErrorMetrics metrics(const Matrix2<T>&, const Options& = {})
//
// Errors follow the reference: std::domain_error("classify: non-finite
// element") where svd2 would throw (classify.hpp:46), std::invalid_argument
// from validate (harness.hpp:39-48), BatchAbort with the reference's message
// from run_batch (harness.hpp:194-198, 267); a CUDA or argument failure of the
// library throws kogsvd2::gpu::Error carrying kog_last_error().
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../kog2.h"

namespace kogsvd2::gpu {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

namespace detail {

inline void check(int rc, const char* what) {
  if (rc == KOG_OK) return;
  const char* msg = kog_last_error();
  if (rc == KOG_ERR_ABORT) throw BatchAbort(msg ? msg : "");
  if (rc == KOG_ERR_ARG && std::strncmp(msg ? msg : "", "lasv2", 5) == 0) throw std::invalid_argument(msg);
  throw Error(rc, std::string(what) + ": " + (msg ? msg : ""));
}

template <class T>
using KMat = std::conditional_t<std::is_same_v<T, double>, kog_mat_f64, kog_mat_f32>;
template <class T>
using KOut = std::conditional_t<std::is_same_v<T, double>, kog_svd_out_f64, kog_svd_out_f32>;

inline kog_options opts(const Options& o) {
  kog_options k{};
  k.hypot_is_cr = o.hypot_is_cr ? 1 : 0;
  k.ominus_for_d = o.ominus_for_d ? 1 : 0;
  k.wide_channel = o.wide_channel == WideChannel::kahan_det ? KOG_WIDE_KAHAN_DET : KOG_WIDE_WIDER_TYPE;
  return k;
}

inline kog_run_config run_config(const RunConfig& c) {
  kog_run_config k{};
  k.single_precision = c.single_precision ? 1 : 0;
  k.shape = c.shape == Shape::tri ? KOG_SHAPE_TRI : KOG_SHAPE_GEN;
  k.regime = c.regime == Regime::circ ? KOG_REGIME_CIRC : (c.regime == Regime::bullet ? KOG_REGIME_BULLET
                                                                                      : KOG_REGIME_SIGMA);
  k.routine = c.routine == Routine::kog ? KOG_ROUTINE_KOG : KOG_ROUTINE_LASV2;
  k.varsigma = c.varsigma;
  k.count = c.count;
  k.seed = c.seed;
  k.threads = c.threads;
  k.options = opts(c.options);
  return k;
}

inline ExtFloat ext(const kog_extfloat& x) { return ExtFloat{x.e, x.hi, x.lo}; }
inline ExtMat ext_mat(const kog_extfloat* a) { return ExtMat{ext(a[0]), ext(a[1]), ext(a[2]), ext(a[3])}; }

template <class T>
T with_sign(T mag, bool neg) {
  const T a = mag < T(0) || (mag == T(0) && std::signbit(mag)) ? -mag : mag;
  return neg ? -a : a;
}

// the compact SoA record of include/kog2.h back into Svd2Result<T>
template <class T>
Svd2Result<T> expand(T s1f, T s2f, int32_t s1e, int32_t s2e, T u11, T u12, T v11, T v12, int32_t s, uint32_t fl) {
  Svd2Result<T> r;
  r.u = Matrix2<T>{u11, u12, with_sign(u12, fl & KOG_F_SIGN_U21), with_sign(u11, fl & KOG_F_SIGN_U22)};
  r.v = Matrix2<T>{v11, v12, with_sign(v12, fl & KOG_F_SIGN_V21), with_sign(v11, fl & KOG_F_SIGN_V22)};
  r.sigma1.e = s1e;  // already normalised pairs: no re-normalisation
  r.sigma1.f = s1f;
  r.sigma2.e = s2e;
  r.sigma2.f = s2f;
  r.s = s;
  BranchTrace& t = r.trace;
  t.path = static_cast<SvdPath>((fl >> KOG_F_PATH_SHIFT) & 7u);
  t.t2p = static_cast<Tan2PhiBranch>((fl >> KOG_F_T2P_SHIFT) & 7u);
  t.tanpsi_inf = fl & KOG_F_TANPSI_INF;
  t.diag_swap = fl & KOG_F_DIAG_SWAP;
  t.sigma_swap = fl & KOG_F_SIGMA_SWAP;
  t.compose_minus = fl & KOG_F_COMPOSE_MINUS;
  t.prescale_inexact = fl & KOG_F_PRESCALE_INEXACT;
  t.urv_col_swap = fl & KOG_F_URV_COL_SWAP;
  t.urv_row_swap = fl & KOG_F_URV_ROW_SWAP;
  t.type_initial = static_cast<std::uint8_t>((fl >> KOG_F_TYPE_INIT_SHIFT) & 15u);
  t.type_scaled = static_cast<std::uint8_t>((fl >> KOG_F_TYPE_SCALED_SHIFT) & 15u);
  return r;
}

// AoS Matrix2 span -> four SoA arrays
template <class T>
struct Soa {
  std::vector<T> a[4];
  explicit Soa(std::span<const Matrix2<T>> g) {
    for (auto& v : a) v.resize(g.size());
    for (size_t i = 0; i < g.size(); ++i) {
      a[0][i] = g[i].g11;
      a[1][i] = g[i].g12;
      a[2][i] = g[i].g21;
      a[3][i] = g[i].g22;
    }
  }
  KMat<T> mat() { return KMat<T>{a[0].data(), a[1].data(), a[2].data(), a[3].data()}; }
};

inline void require_size(size_t a, size_t b, const char* what) {
  if (a != b) throw std::invalid_argument(std::string(what) + ": output span size differs from input");
}

}  // namespace detail

// ------------------------------------------------------------------ svd2
// svd2 over a batch (svd2.hpp:603-687 per element), one device round trip.
// Throws std::domain_error (classify.hpp:46) if any element is non-finite,
// like the reference's loop would at the first such element.
template <WorkingFloat T>
void svd2(std::span<const Matrix2<T>> g, std::span<Svd2Result<T>> out, const Options& opt = {}) {
  detail::require_size(g.size(), out.size(), "svd2");
  const size_t n = g.size();
  if (n == 0) return;
  detail::Soa<T> in(g);
  std::vector<T> f[6];
  std::vector<int32_t> e[3];
  std::vector<uint32_t> flags(n);
  for (auto& v : f) v.resize(n);
  for (auto& v : e) v.resize(n);
  const detail::KMat<T> m = in.mat();
  const detail::KOut<T> o{f[0].data(), f[1].data(), e[0].data(), e[1].data(), f[2].data(),
                          f[3].data(), f[4].data(), f[5].data(), e[2].data(), flags.data()};
  const kog_options ko = detail::opts(opt);
  if constexpr (std::is_same_v<T, double>)
    detail::check(kog_svd2_host_f64(&m, &o, n, &ko), "kog_svd2_host_f64");
  else
    detail::check(kog_svd2_host_f32(&m, &o, n, &ko), "kog_svd2_host_f32");
  for (size_t i = 0; i < n; ++i) {
    if (flags[i] & KOG_F_DOMAIN_ERROR) throw std::domain_error("classify: non-finite element");
    out[i] = detail::expand<T>(f[0][i], f[1][i], e[0][i], e[1][i], f[2][i], f[3][i], f[4][i], f[5][i], e[2][i],
                               flags[i]);
  }
}

template <WorkingFloat T>
std::vector<Svd2Result<T>> svd2(const std::vector<Matrix2<T>>& g, const Options& opt = {}) {
  std::vector<Svd2Result<T>> out(g.size());
  gpu::svd2<T>(std::span<const Matrix2<T>>(g), std::span<Svd2Result<T>>(out), opt);
  return out;
}

// the reference signature (svd2.hpp:603-604)
template <WorkingFloat T>
Svd2Result<T> svd2(const Matrix2<T>& g, const Options& opt = {}) {
  Svd2Result<T> r;
  gpu::svd2<T>(std::span<const Matrix2<T>>(&g, 1), std::span<Svd2Result<T>>(&r, 1), opt);
  return r;
}

// -------------------------------------------------------------- hypot_cr
template <WorkingFloat T>
void hypot_cr(std::span<const T> a, std::span<const T> b, std::span<T> out) {
  detail::require_size(a.size(), b.size(), "hypot_cr");
  detail::require_size(a.size(), out.size(), "hypot_cr");
  if constexpr (std::is_same_v<T, double>)
    detail::check(kog_hypot_host_f64(a.data(), b.data(), out.data(), a.size()), "kog_hypot_host_f64");
  else
    detail::check(kog_hypot_host_f32(a.data(), b.data(), out.data(), a.size()), "kog_hypot_host_f32");
}

template <WorkingFloat T>
T hypot_cr(T a, T b) {  // fpcore.hpp:140-188
  T r{};
  gpu::hypot_cr<T>(std::span<const T>(&a, 1), std::span<const T>(&b, 1), std::span<T>(&r, 1));
  return r;
}

// -------------------------------------------------------------- svd2_ext
// Throws std::domain_error for a non-finite element (classify.hpp:46).
template <WorkingFloat T>
void svd2_ext(std::span<const Matrix2<T>> g, std::span<ExtSvd> out) {
  detail::require_size(g.size(), out.size(), "svd2_ext");
  const size_t n = g.size();
  if (n == 0) return;
  for (const auto& x : g)
    if (!all_finite(x)) throw std::domain_error("classify: non-finite element");
  detail::Soa<T> in(g);
  std::vector<kog_extsvd> rec(n);
  const detail::KMat<T> m = in.mat();
  if constexpr (std::is_same_v<T, double>)
    detail::check(kog_svd2_ext_host_f64(&m, rec.data(), n), "kog_svd2_ext_host_f64");
  else
    detail::check(kog_svd2_ext_host_f32(&m, rec.data(), n), "kog_svd2_ext_host_f32");
  for (size_t i = 0; i < n; ++i)
    out[i] = ExtSvd{detail::ext(rec[i].sigma1), detail::ext(rec[i].sigma2), detail::ext_mat(rec[i].u),
                    detail::ext_mat(rec[i].v)};
}

template <WorkingFloat T>
ExtSvd svd2_ext(const Matrix2<T>& g) {  // oracle.hpp:102-238
  ExtSvd r;
  gpu::svd2_ext<T>(std::span<const Matrix2<T>>(&g, 1), std::span<ExtSvd>(&r, 1));
  return r;
}

// --------------------------------------------------------------- metrics
// run_one's per-matrix evaluation (harness.hpp:200-204): the ErrorMetrics of
// svd2(g, opt) against svd2_ext(g) (oracle.hpp:269-301).
template <WorkingFloat T>
void metrics(std::span<const Matrix2<T>> g, std::span<ErrorMetrics> out, const Options& opt = {}) {
  detail::require_size(g.size(), out.size(), "metrics");
  const size_t n = g.size();
  if (n == 0) return;
  detail::Soa<T> in(g);
  std::vector<kog_metrics> rec(n);
  const detail::KMat<T> m = in.mat();
  const kog_options ko = detail::opts(opt);
  if constexpr (std::is_same_v<T, double>)
    detail::check(kog_metrics_host_f64(&m, rec.data(), n, &ko), "kog_metrics_host_f64");
  else
    detail::check(kog_metrics_host_f32(&m, rec.data(), n, &ko), "kog_metrics_host_f32");
  for (size_t i = 0; i < n; ++i) {
    if (rec[i].flags & KOG_F_DOMAIN_ERROR) throw std::domain_error("classify: non-finite element");
    ErrorMetrics& r = out[i];
    r.reG = rec[i].reG;
    r.reS1 = rec[i].reS1;
    r.reS2 = rec[i].reS2;
    r.reU = rec[i].reU;
    r.reV = rec[i].reV;
    r.kappa2 = detail::ext(rec[i].kappa2);
    r.kappa_inf = rec[i].kappa_inf != 0;
  }
}

template <WorkingFloat T>
ErrorMetrics metrics(const Matrix2<T>& g, const Options& opt = {}) {
  ErrorMetrics r;
  gpu::metrics<T>(std::span<const Matrix2<T>>(&g, 1), std::span<ErrorMetrics>(&r, 1), opt);
  return r;
}

// -------------------------------------------------------------- generate
template <WorkingFloat T>
void generate(const RunConfig& cfg, std::uint64_t index0, std::span<Matrix2<T>> out) {
  const size_t n = out.size();
  if (n == 0) return;
  std::vector<T> a[4];
  for (auto& v : a) v.resize(n);
  const detail::KMat<T> m{a[0].data(), a[1].data(), a[2].data(), a[3].data()};
  const kog_run_config k = detail::run_config(cfg);
  if constexpr (std::is_same_v<T, double>)
    detail::check(kog_generate_host_f64(&k, index0, &m, n), "kog_generate_host_f64");
  else
    detail::check(kog_generate_host_f32(&k, index0, &m, n), "kog_generate_host_f32");
  for (size_t i = 0; i < n; ++i) out[i] = Matrix2<T>{a[0][i], a[1][i], a[2][i], a[3][i]};
}

template <WorkingFloat T>
Matrix2<T> generate(const RunConfig& cfg, std::uint64_t index) {  // harness.hpp:139-186
  Matrix2<T> g;
  gpu::generate<T>(cfg, index, std::span<Matrix2<T>>(&g, 1));
  return g;
}

// ------------------------------------------------------------- run_batch
inline ErrorStats to_error_stats(const kog_stats& s) {
  ErrorStats st;
  st.reG = s.reG;
  st.reS1 = s.reS1;
  st.reS2 = s.reS2;
  st.reU = s.reU;
  st.reV = s.reV;
  st.maxKappa2 = detail::ext(s.max_kappa2);
  st.kappa_inf = s.kappa_inf != 0;
  for (int i = 0; i < 7; ++i) {
    st.counts.t2p[i] = s.t2p[i];
    st.counts.path[i] = s.path[i];
  }
  st.counts.tanpsi_inf = s.tanpsi_inf;
  st.counts.diag_swap = s.diag_swap;
  st.counts.compose_minus = s.compose_minus;
  st.counts.sigma_swap = s.sigma_swap;
  st.counts.prescale_inexact = s.prescale_inexact;
  return st;
}

// run_batch_any on a kog_run_config (the generator extension of configs 2-5)
inline ErrorStats run_batch(const kog_run_config& k) {
  kog_stats s;
  const int rc = kog_run_batch(&k, &s);
  if (rc == KOG_ERR_ARG) throw std::invalid_argument(kog_last_error());
  detail::check(rc, "kog_run_batch");
  return to_error_stats(s);
}

template <WorkingFloat T>
ErrorStats run_batch(const RunConfig& cfg) {  // harness.hpp:225-271 (the GPU ignores cfg.threads)
  kogsvd2::validate<T>(cfg);
  kog_run_config k = detail::run_config(cfg);
  k.single_precision = std::is_same_v<T, float> ? 1 : 0;
  return gpu::run_batch(k);
}

inline ErrorStats run_batch_any(const RunConfig& cfg) {  // harness.hpp:319-321
  return cfg.single_precision ? gpu::run_batch<float>(cfg) : gpu::run_batch<double>(cfg);
}

// ----------------------------------------------------------------- CSV
inline kog_stats to_kog_stats(const ErrorStats& st) {
  kog_stats s;
  kog_stats_init(&s);
  s.reG = st.reG;
  s.reS1 = st.reS1;
  s.reS2 = st.reS2;
  s.reU = st.reU;
  s.reV = st.reV;
  s.max_kappa2 = kog_extfloat{st.maxKappa2.e, st.maxKappa2.hi, st.maxKappa2.lo};
  s.kappa_inf = st.kappa_inf ? 1 : 0;
  return s;
}

inline std::string csv_header() {  // harness.hpp:286-288
  char buf[256];
  detail::check(kog_csv_header(buf, sizeof buf) < 0 ? KOG_ERR_ARG : KOG_OK, "kog_csv_header");
  return buf;
}

inline std::string csv_row(const RunConfig& cfg, const ErrorStats& st) {  // harness.hpp:290-317
  const kog_run_config k = detail::run_config(cfg);
  const kog_stats s = to_kog_stats(st);
  char buf[512];
  const int len = kog_csv_row(&k, &s, buf, sizeof buf);
  if (len < 0) detail::check(len, "kog_csv_row");
  return std::string(buf, static_cast<size_t>(len));
}

}  // namespace kogsvd2::gpu
