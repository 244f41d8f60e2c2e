// kog2_host.cpp — host side of the C-ABI: error state, options, the
// GPU-backed batch runner (run_batch, harness.hpp:226-271), ErrorStats merge
// (harness.hpp:96-105), the CSV boundary (harness.hpp:276-317, with the
// extended decimal of extfloat.hpp:146-179) and the host-buffer svd2 pipeline.
//
// Nothing here computes a decomposition: every matrix is processed by the
// device kernels in kog2_kernels.cu.  The host ExtFloat arithmetic below only
// formats a condition number for the CSV row and orders two statistics.
// Compiled with -ffp-contract=off so that formatting is bit-identical to the
// reference's.
#include <cuda_runtime.h>

#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <string>
#include <vector>

#include "kog2_internal.h"

namespace {

thread_local std::string g_err;

// ------------------------------------------- host ExtFloat (CSV/merge only)
struct HExt {
  int64_t e;
  double hi, lo;
};

void h_two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bv = s - a;
  e = (a - (s - bv)) + (b - bv);
}
void h_fast_two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  e = (a - s) + b;
}
void h_two_prod(double a, double b, double& p, double& e) {
  p = a * b;
  e = std::fma(a, b, -p);
}

// extfloat.hpp:33-48
HExt h_make(int64_t e, double h, double l) {
  if (h == 0.0) {
    h = l;
    l = 0.0;
  }
  if (h == 0.0) return {0, 0.0, 0.0};
  if (std::fabs(h) < std::fabs(l)) std::swap(h, l);
  double s, t;
  h_fast_two_sum(h, l, s, t);
  if (s == 0.0) return {0, 0.0, 0.0};
  const int k = std::ilogb(s);
  double tl = std::scalbn(t, -k);
  if (std::fabs(tl) < 0x1p-120) tl = 0.0;
  return {e + k, std::scalbn(s, -k), tl};
}
HExt h_from(double x) {  // extfloat.hpp:52-55
  if (x == 0.0 || !std::isfinite(x)) return {0, x, 0.0};
  int be;
  const double fr = std::frexp(x, &be);
  return {static_cast<int64_t>(be) - 1, fr + fr, 0.0};
}
HExt h_neg(const HExt& a) { return {a.e, -a.hi, -a.lo}; }
HExt h_add(const HExt& a, const HExt& b) {  // extfloat.hpp:72-90
  if (a.hi == 0.0) return b;
  if (b.hi == 0.0) return a;
  const int64_t d = a.e - b.e;
  if (d > 120) return a;
  if (d < -120) return b;
  const HExt& big = d >= 0 ? a : b;
  const HExt& sml = d >= 0 ? b : a;
  const int sh = static_cast<int>(d >= 0 ? d : -d);
  const double bh = std::scalbn(sml.hi, -sh), bl = std::scalbn(sml.lo, -sh);
  double s1, s2, t1, t2;
  h_two_sum(big.hi, bh, s1, s2);
  h_two_sum(big.lo, bl, t1, t2);
  s2 += t1;
  h_fast_two_sum(s1, s2, s1, s2);
  s2 += t2;
  h_fast_two_sum(s1, s2, s1, s2);
  return h_make(big.e, s1, s2);
}
int h_cmp(const HExt& a, const HExt& b) {  // extfloat.hpp:136-138
  const HExt d = h_add(a, h_neg(b));
  return (d.hi > 0.0) - (d.hi < 0.0);
}
HExt h_mul(const HExt& a, const HExt& b) {  // extfloat.hpp:96-102
  if (a.hi == 0.0 || b.hi == 0.0) return {0, 0.0, 0.0};
  double p, e;
  h_two_prod(a.hi, b.hi, p, e);
  e += a.hi * b.lo + a.lo * b.hi + a.lo * b.lo;
  return h_make(a.e + b.e, p, e);
}
HExt h_div(const HExt& a, const HExt& b) {  // extfloat.hpp:104-113
  if (a.hi == 0.0) return {0, 0.0, 0.0};
  const double bd = b.hi + b.lo;
  const double q1 = a.hi / bd;
  double p, pe;
  h_two_prod(q1, b.hi, p, pe);
  const double r = ((a.hi - p) - pe) + a.lo - q1 * b.lo;
  const double q2 = r / bd;
  return h_make(a.e - b.e, q1, q2);
}
double h_to_double(const HExt& a) {  // extfloat.hpp:140-144
  const long ce = static_cast<long>(a.e < -100000 ? -100000 : (a.e > 100000 ? 100000 : a.e));
  return std::scalbln(a.hi + a.lo, ce);
}
HExt h_pow10(int64_t n) {  // extfloat.hpp:146-157
  HExt base = h_from(10.0);
  if (n < 0) base = h_div(h_from(1.0), base);
  uint64_t k = static_cast<uint64_t>(n < 0 ? -n : n);
  HExt acc = h_from(1.0);
  while (k) {
    if (k & 1) acc = h_mul(acc, base);
    base = h_mul(base, base);
    k >>= 1;
  }
  return acc;
}
std::string h_to_decimal(const HExt& a) {  // extfloat.hpp:159-179
  if (a.hi == 0.0) return "0";
  const double l10 = static_cast<double>(a.e) * 0.30102999566398119521 + std::log10(std::fabs(a.hi + a.lo));
  int64_t d10 = static_cast<int64_t>(std::floor(l10));
  const HExt m = h_mul(a, h_pow10(-d10));
  double md = h_to_double(m);
  if (std::fabs(md) >= 10.0) {
    md /= 10.0;
    ++d10;
  } else if (std::fabs(md) < 1.0) {
    md *= 10.0;
    --d10;
  }
  char buf[48];
  std::snprintf(buf, sizeof buf, "%.17ge%+lld", md, static_cast<long long>(d10));
  return buf;
}

std::string shortest(double x) {  // harness.hpp:278-282
  char buf[40];
  const auto res = std::to_chars(buf, buf + sizeof buf, x);
  return std::string(buf, res.ptr);
}

int copy_out(const std::string& s, char* buf, size_t cap) {
  if (!buf || s.size() + 1 > cap) return kog2_arg_error("output buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

// --------------------------------------------- host-buffer svd2 pipeline
constexpr uint64_t kChunk = 1ull << 22;  // matrices per pipeline stage
constexpr int kSlots = 3;                // H2D / compute / D2H in flight

template <class T>
struct Slot {
  cudaStream_t st = nullptr;
  T* in[4] = {};
  T* of[6] = {};        // sig1_f sig2_f u11 u12 v11 v12
  int32_t* oi[3] = {};  // sig1_e sig2_e s
  uint32_t* flags = nullptr;
};

template <class T>
struct Pool {
  int dev = -1;
  Slot<T> slot[kSlots];
  bool ready = false;
};

std::mutex g_pool_mu;

template <class T>
void pool_release(Pool<T>& p) {
  for (auto& s : p.slot) {
    if (s.st) cudaStreamSynchronize(s.st), cudaStreamDestroy(s.st);
    s.st = nullptr;
    for (auto& b : s.in) cudaFree(b), b = nullptr;
    for (auto& b : s.of) cudaFree(b), b = nullptr;
    for (auto& b : s.oi) cudaFree(b), b = nullptr;
    cudaFree(s.flags);
    s.flags = nullptr;
  }
  p.ready = false;
}

template <class T>
int pool_get(Pool<T>& p, int dev) {
  if (p.ready && p.dev == dev) return KOG_OK;
  bool ok = true;
  for (auto& s : p.slot) {
    ok = ok && cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking) == cudaSuccess;
    for (auto& b : s.in) ok = ok && cudaMalloc(reinterpret_cast<void**>(&b), kChunk * sizeof(T)) == cudaSuccess;
    for (auto& b : s.of) ok = ok && cudaMalloc(reinterpret_cast<void**>(&b), kChunk * sizeof(T)) == cudaSuccess;
    for (auto& b : s.oi) ok = ok && cudaMalloc(reinterpret_cast<void**>(&b), kChunk * sizeof(int32_t)) == cudaSuccess;
    ok = ok && cudaMalloc(reinterpret_cast<void**>(&s.flags), kChunk * sizeof(uint32_t)) == cudaSuccess;
  }
  if (!ok) {  // release whatever was created; the next call starts over
    const int rc = kog2_cuda_error("svd2_host pipeline streams/buffers");
    pool_release(p);
    return rc;
  }
  p.dev = dev;
  p.ready = true;
  return KOG_OK;
}

template <class T, class MatC, class OutC>
int svd2_host(const MatC* in, const OutC* out, uint64_t n, const kog_options* opt,
              int (*batch)(const MatC*, const OutC*, uint64_t, const kog_options*, void*)) {
  if (!in || !out) return kog2_arg_error("kog_svd2_host: null argument");
  if (n == 0) return KOG_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return kog2_cuda_error("cudaGetDevice");
  static Pool<T> pools[64];
  std::lock_guard<std::mutex> lock(g_pool_mu);
  if (dev < 0 || dev >= 64) return kog2_arg_error("device index out of range");
  Pool<T>& p = pools[dev];
  int rc = pool_get(p, dev);
  if (rc != KOG_OK) return rc;
  const T* hin[4] = {in->g11, in->g12, in->g21, in->g22};
  T* hof[6] = {out->sig1_f, out->sig2_f, out->u11, out->u12, out->v11, out->v12};
  int32_t* hoi[3] = {out->sig1_e, out->sig2_e, out->s};
  const uint64_t nchunks = (n + kChunk - 1) / kChunk;
  // every chunk's kernels take their deferral scratch per call on the slot's
  // stream (kog2_ws.cpp), so overlapping slots share nothing but the device
  for (uint64_t c = 0; c < nchunks && rc == KOG_OK; ++c) {
    Slot<T>& s = p.slot[c % kSlots];
    const uint64_t lo = c * kChunk, len = (n - lo < kChunk) ? n - lo : kChunk;
    for (int k = 0; k < 4 && rc == KOG_OK; ++k)
      if (cudaMemcpyAsync(s.in[k], hin[k] + lo, len * sizeof(T), cudaMemcpyHostToDevice, s.st) != cudaSuccess)
        rc = kog2_cuda_error("cudaMemcpyAsync H2D");
    if (rc != KOG_OK) break;
    MatC dm;
    dm.g11 = s.in[0];
    dm.g12 = s.in[1];
    dm.g21 = s.in[2];
    dm.g22 = s.in[3];
    OutC dout;
    dout.sig1_f = s.of[0];
    dout.sig2_f = s.of[1];
    dout.u11 = s.of[2];
    dout.u12 = s.of[3];
    dout.v11 = s.of[4];
    dout.v12 = s.of[5];
    dout.sig1_e = s.oi[0];
    dout.sig2_e = s.oi[1];
    dout.s = s.oi[2];
    dout.flags = s.flags;
    if ((rc = batch(&dm, &dout, len, opt, s.st)) != KOG_OK) break;
    for (int k = 0; k < 6 && rc == KOG_OK; ++k)
      if (cudaMemcpyAsync(hof[k] + lo, s.of[k], len * sizeof(T), cudaMemcpyDeviceToHost, s.st) != cudaSuccess)
        rc = kog2_cuda_error("cudaMemcpyAsync D2H");
    for (int k = 0; k < 3 && rc == KOG_OK; ++k)
      if (cudaMemcpyAsync(hoi[k] + lo, s.oi[k], len * sizeof(int32_t), cudaMemcpyDeviceToHost, s.st) != cudaSuccess)
        rc = kog2_cuda_error("cudaMemcpyAsync D2H");
    if (rc == KOG_OK &&
        cudaMemcpyAsync(out->flags + lo, s.flags, len * sizeof(uint32_t), cudaMemcpyDeviceToHost, s.st) != cudaSuccess)
      rc = kog2_cuda_error("cudaMemcpyAsync D2H");
  }
  // drain every slot, also after an error: no copy into the caller's host
  // buffers may still be running when this returns
  for (auto& s : p.slot)
    if (cudaStreamSynchronize(s.st) != cudaSuccess && rc == KOG_OK) rc = kog2_cuda_error("cudaStreamSynchronize");
  return rc;
}

// ------------------------------------- host-buffer forms of device routines
// One staged call: device arrays from the workspace pool on a private stream,
// H2D of the inputs, the device entry point, D2H of the outputs, synchronise.
// Used by the per-matrix C++ shim (include/kog2/kogsvd2_gpu.hpp).
struct HostArg {
  const void* host;
  size_t bytes;
};
struct HostOut {
  void* host;
  size_t bytes;
};
template <class F>
int staged(std::initializer_list<HostArg> ins, std::initializer_list<HostOut> outs, F launch) {
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return kog2_cuda_error("cudaStreamCreate");
  std::vector<void*> din, dout;
  int rc = KOG_OK;
  for (const HostArg& a : ins) {
    void* d = kog2_ws_alloc(a.bytes, st);
    if (!d) {
      rc = KOG_ERR_CUDA;
      break;
    }
    din.push_back(d);
    if (cudaMemcpyAsync(d, a.host, a.bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      rc = kog2_cuda_error("cudaMemcpyAsync H2D");
      break;
    }
  }
  for (size_t k = 0; rc == KOG_OK && k < outs.size(); ++k) {
    void* d = kog2_ws_alloc(outs.begin()[k].bytes, st);
    if (!d) rc = KOG_ERR_CUDA;
    else dout.push_back(d);
  }
  if (rc == KOG_OK) rc = launch(din.data(), dout.data(), static_cast<void*>(st));
  for (size_t k = 0; rc == KOG_OK && k < outs.size(); ++k)
    if (cudaMemcpyAsync(outs.begin()[k].host, dout[k], outs.begin()[k].bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = kog2_cuda_error("cudaMemcpyAsync D2H");
  for (void* d : din) kog2_ws_free(d, st);
  for (void* d : dout) kog2_ws_free(d, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && rc == KOG_OK) rc = kog2_cuda_error("cudaStreamSynchronize");
  cudaStreamDestroy(st);
  return rc;
}

template <class T, class MatC>
int hypot_host(const T* a, const T* b, T* out, uint64_t n, int (*fn)(const T*, const T*, T*, uint64_t, void*)) {
  if (n == 0) return KOG_OK;
  if (!a || !b || !out) return kog2_arg_error("kog_hypot_host: null argument");
  const size_t B = n * sizeof(T);
  return staged({{a, B}, {b, B}}, {{out, B}}, [&](void** di, void** dout, void* st) {
    return fn(static_cast<const T*>(di[0]), static_cast<const T*>(di[1]), static_cast<T*>(dout[0]), n, st);
  });
}

template <class T, class MatC>
MatC mat_of(void** d) {
  MatC m;
  m.g11 = static_cast<T*>(d[0]);
  m.g12 = static_cast<T*>(d[1]);
  m.g21 = static_cast<T*>(d[2]);
  m.g22 = static_cast<T*>(d[3]);
  return m;
}

template <class T, class MatC, class Rec, class F>
int per_matrix_host(const MatC* g, Rec* out, uint64_t n, F fn) {
  if (n == 0) return KOG_OK;
  if (!g || !g->g11 || !g->g12 || !g->g21 || !g->g22 || !out) return kog2_arg_error("kog host call: null argument");
  const size_t B = n * sizeof(T);
  return staged({{g->g11, B}, {g->g12, B}, {g->g21, B}, {g->g22, B}}, {{out, n * sizeof(Rec)}},
                [&](void** di, void** dout, void* st) {
                  const MatC m = mat_of<T, MatC>(di);
                  return fn(&m, static_cast<Rec*>(dout[0]), st);
                });
}

template <class T, class MatC>
int generate_host(const kog_run_config* cfg, uint64_t index0, const MatC* out, uint64_t n,
                  int (*fn)(const kog_run_config*, uint64_t, const MatC*, uint64_t, void*)) {
  if (n == 0) return KOG_OK;
  if (!cfg || !out || !out->g11 || !out->g12 || !out->g21 || !out->g22)
    return kog2_arg_error("kog_generate_host: null argument");
  const size_t B = n * sizeof(T);
  return staged({}, {{out->g11, B}, {out->g12, B}, {out->g21, B}, {out->g22, B}},
                [&](void**, void** dout, void* st) {
                  const MatC m = mat_of<T, MatC>(dout);
                  return fn(cfg, index0, &m, n, st);
                });
}

template <class T>
std::string bits_of(T x) {  // harness.hpp:130-135
  char buf[40];
  std::snprintf(buf, sizeof buf, "%a", static_cast<double>(x));
  return buf;
}

}  // namespace

// ------------------------------------------------------------ internal API
static std::atomic<uint64_t> g_launches{0};
void kog2_count_launch(void) { g_launches.fetch_add(1, std::memory_order_relaxed); }
void kog2_set_error(const char* msg) { g_err = msg ? msg : ""; }
int kog2_arg_error(const char* msg) {
  g_err = msg;
  return KOG_ERR_ARG;
}
int kog2_cuda_error(const char* what) {
  const cudaError_t e = cudaGetLastError();
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return KOG_ERR_CUDA;
}
kog_options kog2_default_options(void) {
  kog_options o;
  o.hypot_is_cr = 1;
  o.ominus_for_d = 0;
  o.wide_channel = KOG_WIDE_WIDER_TYPE;
  o.reserved = 0;
  return o;
}

// ------------------------------------------------------------------ C-ABI
extern "C" {

const char* kog_last_error(void) { return g_err.c_str(); }
uint64_t kog_launch_count(void) { return g_launches.load(); }
const char* kog_version(void) { return "kog2 0.1 (sm_100a)"; }

int kog_set_device(int device) {
  if (cudaSetDevice(device) != cudaSuccess) return kog2_cuda_error("cudaSetDevice");
  return KOG_OK;
}

int kog_svd2_host_f64(const kog_mat_f64* in, const kog_svd_out_f64* out, uint64_t n, const kog_options* opt) {
  return svd2_host<double>(in, out, n, opt, &kog_svd2_batch_f64);
}
int kog_svd2_host_f32(const kog_mat_f32* in, const kog_svd_out_f32* out, uint64_t n, const kog_options* opt) {
  return svd2_host<float>(in, out, n, opt, &kog_svd2_batch_f32);
}

int kog_hypot_host_f64(const double* a, const double* b, double* out, uint64_t n) {
  return hypot_host<double, kog_mat_f64>(a, b, out, n, &kog_hypot_batch_f64);
}
int kog_hypot_host_f32(const float* a, const float* b, float* out, uint64_t n) {
  return hypot_host<float, kog_mat_f32>(a, b, out, n, &kog_hypot_batch_f32);
}
int kog_svd2_ext_host_f64(const kog_mat_f64* g, kog_extsvd* out, uint64_t n) {
  return per_matrix_host<double>(g, out, n, [&](const kog_mat_f64* m, kog_extsvd* o, void* st) {
    return kog_svd2_ext_batch_f64(m, o, n, st);
  });
}
int kog_svd2_ext_host_f32(const kog_mat_f32* g, kog_extsvd* out, uint64_t n) {
  return per_matrix_host<float>(g, out, n, [&](const kog_mat_f32* m, kog_extsvd* o, void* st) {
    return kog_svd2_ext_batch_f32(m, o, n, st);
  });
}
int kog_metrics_host_f64(const kog_mat_f64* g, kog_metrics* out, uint64_t n, const kog_options* opt) {
  return per_matrix_host<double>(g, out, n, [&](const kog_mat_f64* m, kog_metrics* o, void* st) {
    return kog_metrics_batch_f64(m, o, n, opt, st);
  });
}
int kog_metrics_host_f32(const kog_mat_f32* g, kog_metrics* out, uint64_t n, const kog_options* opt) {
  return per_matrix_host<float>(g, out, n, [&](const kog_mat_f32* m, kog_metrics* o, void* st) {
    return kog_metrics_batch_f32(m, o, n, opt, st);
  });
}
int kog_generate_host_f64(const kog_run_config* cfg, uint64_t index0, const kog_mat_f64* out, uint64_t n) {
  return generate_host<double>(cfg, index0, out, n, &kog_generate_batch_f64);
}
int kog_generate_host_f32(const kog_run_config* cfg, uint64_t index0, const kog_mat_f32* out, uint64_t n) {
  return generate_host<float>(cfg, index0, out, n, &kog_generate_batch_f32);
}

void kog_stats_init(kog_stats* st) {
  if (!st) return;
  std::memset(st, 0, sizeof *st);
  st->fail_key = UINT64_MAX;
}

// ErrorStats::merge (harness.hpp:96-105)
void kog_stats_merge(kog_stats* st, const kog_stats* o) {
  if (!st || !o) return;
  st->reG = std::fmax(st->reG, o->reG);
  st->reS1 = std::fmax(st->reS1, o->reS1);
  st->reS2 = std::fmax(st->reS2, o->reS2);
  st->reU = std::fmax(st->reU, o->reU);
  st->reV = std::fmax(st->reV, o->reV);
  st->kappa_inf = (st->kappa_inf || o->kappa_inf) ? 1 : 0;
  const HExt a{st->max_kappa2.e, st->max_kappa2.hi, st->max_kappa2.lo};
  const HExt b{o->max_kappa2.e, o->max_kappa2.hi, o->max_kappa2.lo};
  const int c = h_cmp(b, a);
  if (c > 0 || (c == 0 && b.hi != 0.0 && a.hi != 0.0 && o->max_kappa2_index < st->max_kappa2_index)) {
    st->max_kappa2 = o->max_kappa2;
    st->max_kappa2_index = o->max_kappa2_index;
  }
  for (int i = 0; i < 7; ++i) {
    st->t2p[i] += o->t2p[i];
    st->path[i] += o->path[i];
  }
  st->tanpsi_inf += o->tanpsi_inf;
  st->diag_swap += o->diag_swap;
  st->compose_minus += o->compose_minus;
  st->sigma_swap += o->sigma_swap;
  st->prescale_inexact += o->prescale_inexact;
  if (o->fail_key < st->fail_key) st->fail_key = o->fail_key;
}

// validate<T> (harness.hpp:39-48) + the generator extension's own checks
int kog_validate(const kog_run_config* cfg) {
  if (!cfg) return kog2_arg_error("null config");
  const int emin = cfg->single_precision ? -126 : -1022;
  const int emax = cfg->single_precision ? 127 : 1023;
  if (cfg->routine == KOG_ROUTINE_LASV2 && cfg->shape != KOG_SHAPE_TRI)
    return kog2_arg_error("lasv2 accepts triangular inputs only");
  if (cfg->regime == KOG_REGIME_SIGMA) {
    if (cfg->varsigma < 1) return kog2_arg_error("sigma regime needs varsigma >= 1");
    if (emin + cfg->varsigma > emax - 2) return kog2_arg_error("varsigma exceeds the exponent range");
  }
  if (cfg->regime > KOG_REGIME_RANGED || cfg->shape > KOG_SHAPE_GEN || cfg->routine > KOG_ROUTINE_LASV2)
    return kog2_arg_error("unknown shape/regime/routine");
  if (cfg->regime == KOG_REGIME_RANGED) {
    if (cfg->elo > cfg->ehi) return kog2_arg_error("ranged regime needs elo <= ehi");
    if (cfg->tail_mod != 0 && cfg->tail_lo > cfg->tail_hi) return kog2_arg_error("ranged tail needs tail_lo <= tail_hi");
  }
  return KOG_OK;
}

int kog_abort_message(const kog_run_config* cfg, uint64_t fail_key, char* buf, size_t cap) {
  if (!cfg || fail_key == UINT64_MAX) return kog2_arg_error("no failure recorded");
  const uint64_t index = fail_key / 4;
  const unsigned reason = static_cast<unsigned>(fail_key % 4);
  std::string g[4];
  if (cfg->single_precision) {
    float* d = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&d), 4 * sizeof(float)) != cudaSuccess) return kog2_cuda_error("cudaMalloc");
    kog_mat_f32 m{d, d + 1, d + 2, d + 3};
    int rc = kog_generate_batch_f32(cfg, index, &m, 1, nullptr);
    float h[4];
    if (rc == KOG_OK && cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess) rc = kog2_cuda_error("cudaMemcpy");
    cudaFree(d);
    if (rc != KOG_OK) return rc;
    for (int k = 0; k < 4; ++k) g[k] = bits_of(h[k]);
  } else {
    double* d = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&d), 4 * sizeof(double)) != cudaSuccess) return kog2_cuda_error("cudaMalloc");
    kog_mat_f64 m{d, d + 1, d + 2, d + 3};
    int rc = kog_generate_batch_f64(cfg, index, &m, 1, nullptr);
    double h[4];
    if (rc == KOG_OK && cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess) rc = kog2_cuda_error("cudaMemcpy");
    cudaFree(d);
    if (rc != KOG_OK) return rc;
    for (int k = 0; k < 4; ++k) g[k] = bits_of(h[k]);
  }
  // harness.hpp:194-198: "<what> at index <i>: g = [g11, g12; g21, g22]"
  const char* what = reason == KOG_FAIL_NONFINITE ? "non-finite factor" : "NaN metric";
  const std::string msg = std::string(what) + " at index " + std::to_string(index) + ": g = [" + g[0] + ", " +
                          g[1] + "; " + g[2] + ", " + g[3] + "]";
  return copy_out(msg, buf, cap);
}

// run_batch_any (harness.hpp:226-271, 319-321) on the current device
int kog_run_batch(const kog_run_config* cfg, kog_stats* out) {
  if (!cfg || !out) return kog2_arg_error("kog_run_batch: null argument");
  int rc = kog_validate(cfg);
  if (rc != KOG_OK) return rc;
  kog_stats* dev = nullptr;
  rc = kog_study_stats_alloc(&dev);
  if (rc != KOG_OK) return rc;
  constexpr uint64_t kLaunch = 1ull << 27;  // bounded kernel duration
  for (uint64_t lo = 0; lo < cfg->count && rc == KOG_OK; lo += kLaunch) {
    const uint64_t len = cfg->count - lo < kLaunch ? cfg->count - lo : kLaunch;
    rc = kog_study_batch(cfg, lo, len, dev, nullptr);
  }
  if (rc == KOG_OK) {
    if (cudaMemcpy(out, dev, sizeof *out, cudaMemcpyDeviceToHost) != cudaSuccess) rc = kog2_cuda_error("cudaMemcpy(kog_stats)");
  }
  kog_study_stats_free(dev);
  if (rc != KOG_OK) return rc;
  if (out->fail_key != UINT64_MAX) {
    char buf[512];
    if (kog_abort_message(cfg, out->fail_key, buf, sizeof buf) < 0) return KOG_ERR_CUDA;
    g_err = buf;
    return KOG_ERR_ABORT;
  }
  return KOG_OK;
}

int kog_csv_header(char* buf, size_t cap) {
  return copy_out("precision,shape,regime,varsigma,count,seed,routine,reG,reS1,reS2,reU,reV,maxKappa2", buf, cap);
}

// csv_row (harness.hpp:290-317); the extended regime prints as "ranged"
int kog_csv_row(const kog_run_config* cfg, const kog_stats* st, char* buf, size_t cap) {
  if (!cfg || !st) return kog2_arg_error("kog_csv_row: null argument");
  std::string row;
  row += cfg->single_precision ? "single" : "double";
  row += cfg->shape == KOG_SHAPE_TRI ? ",tri" : ",gen";
  row += cfg->regime == KOG_REGIME_CIRC     ? ",circ"
         : cfg->regime == KOG_REGIME_BULLET ? ",bullet"
         : cfg->regime == KOG_REGIME_SIGMA  ? ",sigma"
                                            : ",ranged";
  row += "," + std::to_string(cfg->varsigma);
  row += "," + std::to_string(cfg->count);
  char seedbuf[20];
  std::snprintf(seedbuf, sizeof seedbuf, "%016llx", static_cast<unsigned long long>(cfg->seed));
  row += ",";
  row += seedbuf;
  row += cfg->routine == KOG_ROUTINE_KOG ? ",kog" : ",lasv2";
  row += "," + shortest(st->reG);
  row += "," + shortest(st->reS1);
  row += "," + shortest(st->reS2);
  row += "," + shortest(st->reU);
  row += "," + shortest(st->reV);
  row += ",";
  const HExt k{st->max_kappa2.e, st->max_kappa2.hi, st->max_kappa2.lo};
  if (st->kappa_inf) {
    row += "inf";
  } else if (k.e > -1000 && k.e < 1000) {
    row += shortest(h_to_double(k));
  } else {
    row += h_to_decimal(k);
  }
  return copy_out(row, buf, cap);
}

}  // extern "C"
