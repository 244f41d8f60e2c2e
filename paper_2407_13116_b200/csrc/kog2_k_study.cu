// kog2_k_study.cu — the verification path on the device: svd2_ext
// (oracle.hpp:102-238), the per-matrix error measures (oracle.hpp:267-301),
// and the fused study kernel generate -> svd2_ext -> svd2 | lasv2 ->
// finiteness -> metrics -> ErrorStats absorb (harness.hpp:190-222), reduced
// with warp shuffles, shared memory and order-independent global atomics.
#include <atomic>
#include <cstdlib>

#include "kog2_common.cuh"
#include "kog2_ext.cuh"
#include "kog2_gen.cuh"
#include "kog2_lasv2.cuh"

using namespace kog2;

namespace {

__device__ __forceinline__ kog_extfloat to_c(const Ext& x) { return kog_extfloat{x.e, x.hi, x.lo}; }

template <class T>
__global__ void k_svd2_ext(InP<T> in, kog_extsvd* o, uint64_t n) {
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    ExtSvd r;
    svd2_ext(load_mat(in, i), r);
    kog_extsvd rec;
    rec.sigma1 = to_c(r.sigma1);
    rec.sigma2 = to_c(r.sigma2);
    rec.u[0] = to_c(r.u.a11);
    rec.u[1] = to_c(r.u.a12);
    rec.u[2] = to_c(r.u.a21);
    rec.u[3] = to_c(r.u.a22);
    rec.v[0] = to_c(r.v.a11);
    rec.v[1] = to_c(r.v.a12);
    rec.v[2] = to_c(r.v.a21);
    rec.v[3] = to_c(r.v.a22);
    o[i] = rec;
  }
}

// run_one's per-matrix body (harness.hpp:190-222) without the absorb; returns
// the svd2 flags plus KOG_M_NONFINITE_FACTOR / KOG_M_NAN_METRIC
template <class T>
__device__ __forceinline__ uint32_t run_one_kog(const Mat<T>& g, const Opt& o, Metrics& m) {
  ExtSvd ref;
  ref_sigma<T>(g, ref);  // metrics() reads the singular values only (inline Xf where it applies)
  Result<T> r;
  svd2<T>(g, o, r);
  uint32_t flags = r.flags;
  if (!all_finite(r.u) || !all_finite(r.v) || !is_finite(r.sigma1.f) || !is_finite(r.sigma2.f))
    flags |= KOG_M_NONFINITE_FACTOR;
  metrics(g, r.u, r.v, ext_from_pair(r.sigma1), ext_from_pair(r.sigma2), ref, m);
  if (isnan(m.reG) || isnan(m.reS1) || isnan(m.reS2) || isnan(m.reU) || isnan(m.reV)) flags |= KOG_M_NAN_METRIC;
  return flags;
}

// the decomposition as kog_svd2_batch stored it (compact SoA, include/kog2.h)
// and the reference singular values (k_ref_sigma)
template <class T>
struct SvdBuf {
  const T *sig1_f, *sig2_f;
  const int32_t *sig1_e, *sig2_e;
  const T *u11, *u12, *v11, *v12;
  const uint32_t* flags;
  long long *re1, *re2;
  double *rh1, *rl1, *rh2, *rl2;
};

// svd2_ext's singular values (oracle.hpp:102-238) of a chunk, SoA
template <class T>
#ifndef KOG2_REF_MINB
#define KOG2_REF_MINB 4
#endif
__global__ void __launch_bounds__(kThreads, KOG2_REF_MINB) k_ref_sigma(InP<T> in, SvdBuf<T> b, uint64_t n) {
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    ExtSvd ref;
    svd2_ext<T, false>(load_mat(in, i), ref);
    b.re1[i] = ref.sigma1.e;
    b.rh1[i] = ref.sigma1.hi;
    b.rl1[i] = ref.sigma1.lo;
    b.re2[i] = ref.sigma2.e;
    b.rh2[i] = ref.sigma2.hi;
    b.rl2[i] = ref.sigma2.lo;
  }
}

__device__ __forceinline__ double with_sign(double mag, bool neg) { return neg ? -mag : mag; }
__device__ __forceinline__ float with_sign(float mag, bool neg) { return neg ? -mag : mag; }

// run_one (harness.hpp:190-222) on a decomposition computed by the svd2
// kernels: U and V are expanded exactly (|u22| = |u11|, |u21| = |u12| with the
// stored signs), so the metrics see the reference's own factors
template <class T>
__device__ __forceinline__ uint32_t run_one_buf(const Mat<T>& g, const SvdBuf<T>& b, uint64_t i, Metrics& m) {
  ExtSvd ref;  // metrics() reads the singular values only
#ifndef KOG2_STUDY_REF_KERNEL
  ref_sigma<T>(g, ref);  // computed here (inline Xf) instead of by k_ref_sigma
#else
  ref.sigma1 = Ext{b.re1[i], b.rh1[i], b.rl1[i]};
  ref.sigma2 = Ext{b.re2[i], b.rh2[i], b.rl2[i]};
#endif
  uint32_t flags = b.flags[i];
  const T u11 = b.u11[i], u12 = b.u12[i], v11 = b.v11[i], v12 = b.v12[i];
  const Mat<T> u{u11, u12, with_sign(fabs(u12), flags & KOG_F_SIGN_U21), with_sign(fabs(u11), flags & KOG_F_SIGN_U22)};
  const Mat<T> v{v11, v12, with_sign(fabs(v12), flags & KOG_F_SIGN_V21), with_sign(fabs(v11), flags & KOG_F_SIGN_V22)};
  const EPair<T> s1{b.sig1_e[i], b.sig1_f[i]}, s2{b.sig2_e[i], b.sig2_f[i]};
  if (!all_finite(u) || !all_finite(v) || !is_finite(s1.f) || !is_finite(s2.f)) flags |= KOG_M_NONFINITE_FACTOR;
  metrics(g, u, v, ext_from_pair(s1), ext_from_pair(s2), ref, m);
  if (isnan(m.reG) || isnan(m.reS1) || isnan(m.reS2) || isnan(m.reU) || isnan(m.reV)) flags |= KOG_M_NAN_METRIC;
  return flags;
}

// ------------------------------------------------- the split study
// k_study's per-matrix body is ~9,000 straight-line instructions (150 KB of SASS executed once per matrix):
// every warp streams it through a 32 KB instruction cache, and the kernel runs at the rate its leading warp can
// fetch code (ncu r8: 22% of stall samples `no_instructions`, the GPC instruction cache at 41% of its request
// peak with a 41% hit rate; with 20 warps per SM instead of 16 the same code ran 3x slower, 80% of samples
// `no_instructions`).  The phased study therefore runs the body as separate kernels whose loops stay in the
// instruction cache — the reference singular values in two launches (triangular factor; singular values, their
// errors and kappa_2), the reconstruction error in two (residual norm; ratio), one orthogonality defect per
// launch, the rare lanes off the Xf route — and a last kernel that only reads the pieces and absorbs them; the
// pieces go through nine 8-byte and six 4-byte arrays per chunk.  Same operations on the same values: identical
// statistics ("the split study"; profiles/r14_study_kernels.txt has the history).
struct StudyAux {
  double *reG, *reU, *reV, *reS1, *reS2, *kh, *kl;  // kappa_2 = (ke, kh, kl)
  int32_t* ke;
  double *xh3, *xl3;   // between k_study_urv and k_study_sigma: the third intermediate (the first two in the
  int32_t *xe2, *xe3;  // result slots)
  uint32_t* sflag;  // between urv and sigma: ref_urv_xf's kind; then bit 0: the reference singular values are
                    // finite, bit 1: kappa_inf, and from k_study_whole bit 2: non-finite factor, bit 3: wide exponent
  uint32_t* fin;    // g, u, v and the computed singular values are finite (with bit 0 above: metrics()'s Xf route)
  uint32_t *list, *count;  // the chunk's lanes off that route (k_study_whole's work list)
};

// the factors as run_one_buf expands them
template <class T>
__device__ __forceinline__ Mat<T> factor_of(T q11, T q12, bool neg21, bool neg22) {
  return Mat<T>{q11, q12, with_sign(fabs(q12), neg21), with_sign(fabs(q11), neg22)};
}

// Blocks of 256 threads per SM the split kernels are compiled for.  With their loops in the instruction cache,
// occupancy pays (launch list r11, us per 2^22 chunk at 2 / 3 / 4 blocks: urv 349 / 326 / 314, sigma 391 / 317 /
// 287, recon 459 / 437 / 438) — the opposite of the fused kernel, where more warps only fought over the cache.
#ifndef KOG2_SPLIT_MINB
#define KOG2_SPLIT_MINB 4
#endif
#ifndef KOG2_RATIO_MINB
#define KOG2_RATIO_MINB 5  // (548 -> 524 us per 2^24; the other split kernels spill at 48 registers and lose)
#endif
#ifndef KOG2_ABSORB_MINB
#define KOG2_ABSORB_MINB 4
#endif
// svd2_ext's singular values in two launches.  First the triangular factor (r11, r12, r22) of the lanes on the
// Xf route (ref_urv_xf), kept in the slots the second launch overwrites with its results — or, for the other
// lanes, the singular values themselves from svd2_ext; sflag says which (0 values, 1 factor, 2 factor with
// r22 = 0).
template <class T>
__global__ void __launch_bounds__(kThreads, KOG2_SPLIT_MINB) k_study_urv(InP<T> in, StudyAux a, uint64_t n) {
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    const Mat<T> g = load_mat(in, i);
    Xf x1, x2, x3 = xf_zero();
    int kind = ref_urv_xf(g, x1, x2, x3);
    if (kind == 3) kind = 0;  // the singular values themselves
    else if (kind == 0) {
      ExtSvd ref;
      svd2_ext<T, false>(g, ref);
      x1 = xf_of(ref.sigma1);  // (a finite value's exponent fits; the others are not read as numbers)
      x2 = xf_of(ref.sigma2);
    }
    a.reS1[i] = x1.hi;
    a.reS2[i] = x1.lo;
    a.ke[i] = x1.e;
    a.kh[i] = x2.hi;
    a.kl[i] = x2.lo;
    a.xe2[i] = x2.e;
    a.xh3[i] = x3.hi;
    a.xl3[i] = x3.lo;
    a.xe3[i] = x3.e;
    a.sflag[i] = static_cast<uint32_t>(kind);
  }
}
// then the singular values (ref_tri_xf), their errors and kappa_2
template <class T>
__global__ void __launch_bounds__(kThreads, KOG2_SPLIT_MINB) k_study_sigma(SvdBuf<T> b, StudyAux a, uint64_t n) {
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    const int kind = static_cast<int>(a.sflag[i]);
    Xf ref1{a.ke[i], a.reS1[i], a.reS2[i]}, ref2{a.xe2[i], a.kh[i], a.kl[i]};
    if (kind != 0) {
      const Xf r11 = ref1, r12 = ref2, r22{a.xe3[i], a.xh3[i], a.xl3[i]};
      ref_tri_xf(kind, r11, r12, r22, ref1, ref2);
    }
    const bool rf = is_finite(ref1.hi) && is_finite(ref2.hi) && is_finite(ref1.lo) && is_finite(ref2.lo);
    uint32_t sf = rf ? 1u : 0u;
    if (rf) {  // the singular values' errors and kappa_2 (used by the lanes whose factors are finite too)
      const EPair<T> s1{b.sig1_e[i], b.sig1_f[i]}, s2{b.sig2_e[i], b.sig2_f[i]};
      Metrics m;
      xf_sigma_metrics(xf_of(ext_from_pair(s1)), xf_of(ext_from_pair(s2)), ref1, ref2, m);
      a.reS1[i] = m.reS1;
      a.reS2[i] = m.reS2;
      a.kh[i] = m.kappa2.hi;
      a.kl[i] = m.kappa2.lo;
      a.ke[i] = static_cast<int32_t>(m.kappa2.e);
      sf |= m.kappa_inf ? 2u : 0u;
    }
    a.sflag[i] = sf;
  }
}
// reG of the finite lanes in two launches: which lanes those are and the squared norm of the residual ...
template <class T>
__global__ void __launch_bounds__(kThreads, KOG2_SPLIT_MINB) k_study_recon(InP<T> in, SvdBuf<T> b, StudyAux a, uint64_t n) {
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    const Mat<T> g = load_mat(in, i);
    const uint32_t flags = b.flags[i];
    const Mat<T> u = factor_of<T>(b.u11[i], b.u12[i], flags & KOG_F_SIGN_U21, flags & KOG_F_SIGN_U22);
    const Mat<T> v = factor_of<T>(b.v11[i], b.v12[i], flags & KOG_F_SIGN_V21, flags & KOG_F_SIGN_V22);
    const EPair<T> s1{b.sig1_e[i], b.sig1_f[i]}, s2{b.sig2_e[i], b.sig2_f[i]};
    const bool fin = mat_finite(g) && mat_finite(u) && mat_finite(v) && is_finite(s1.f) && is_finite(s2.f);
    a.fin[i] = fin ? 1u : 0u;
    Xf sq = xf_zero();
    if (fin) sq = xf_recon_sq(g, u, v, xf_of(ext_from_pair(s1)), xf_of(ext_from_pair(s2)));
    a.xh3[i] = sq.hi;
    a.xl3[i] = sq.lo;
    a.xe3[i] = sq.e;
  }
}
// ... then its root over ||G||_F
template <class T>
__global__ void __launch_bounds__(kThreads, KOG2_RATIO_MINB) k_study_ratio(InP<T> in, StudyAux a, uint64_t n) {
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    const Mat<T> g = load_mat(in, i);
    const Xf sq{a.xe3[i], a.xh3[i], a.xl3[i]};
    double r = 0.0;
    if (a.fin[i] != 0) r = xf_recon_ratio(g, sq);
    a.reG[i] = r;
  }
}
// the orthogonality defect of one factor (launched for U and for V) of the finite lanes
// (LIST: this launch — the last one, fin and sflag are final — also collects the lanes off the Xf route)
template <class T, bool LIST>
__global__ void __launch_bounds__(kThreads, KOG2_SPLIT_MINB)
    k_study_ortho(const T* q11, const T* q12, const uint32_t* flags, uint32_t bit21, uint32_t bit22,
                  const uint32_t* fin, double* out, uint64_t n, StudyAux a) {
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    const bool xf_lane = fin[i] != 0;
    if constexpr (LIST) {
      if (!xf_lane || (a.sflag[i] & 1u) == 0) a.list[atomicAdd(a.count, 1u)] = static_cast<uint32_t>(i);
    }
    if (!xf_lane) {
      out[i] = 0.0;  // (not used: k_study_whole writes the lane's metrics)
      continue;
    }
    const uint32_t f = flags[i];
    const Mat<T> q = factor_of<T>(q11[i], q12[i], f & bit21, f & bit22);
#ifdef KOG2_ORTHO_GENERAL  // (the reference's full sequence, for A/B)
    out[i] = xf_ortho(q);
#else
    out[i] = xf_ortho_compact(q.g11, q.g12, q.g21, q.g22);
#endif
  }
}
// metrics() of a lane off the Xf route (something is not finite), whole, on the Ext functions; the reference
// singular values again from svd2_ext (ref_sigma's values, bit for bit)
template <class T>
__device__ __noinline__ void metrics_whole_ext(const Mat<T> g, const Mat<T> u, const Mat<T> v, const EPair<T> s1,
                                               const EPair<T> s2, Metrics& m) {
  ExtSvd ref;
  svd2_ext<T, false>(g, ref);
  metrics_ext<T>(g, u, v, ext_from_pair(s1), ext_from_pair(s2), ref, m);
}
// The lanes off the Xf route (something is not finite; rare): metrics() whole, written into the same slots, so
// that the absorb kernel below only reads (a scan for these lanes inside a kernel holding this code ran at its 152
// registers: 126 us per chunk; the list costs nothing).  sflag afterwards: bit 1 kappa_inf, bit 2 KOG_M_NONFINITE_FACTOR, bit 3
// kappa_2's exponent does not fit 32 bits (its high word is in xe2).
template <class T>
__global__ void __launch_bounds__(kThreads) k_study_whole(InP<T> gin, SvdBuf<T> b, StudyAux a) {
  const uint64_t m_count = *a.count;
  for (uint64_t k = gtid(); k < m_count; k += gstride()) {
    const uint64_t i = a.list[k];
    const uint32_t flags = b.flags[i];
    const EPair<T> s1{b.sig1_e[i], b.sig1_f[i]}, s2{b.sig2_e[i], b.sig2_f[i]};
    const Mat<T> u = factor_of<T>(b.u11[i], b.u12[i], flags & KOG_F_SIGN_U21, flags & KOG_F_SIGN_U22);
    const Mat<T> v = factor_of<T>(b.v11[i], b.v12[i], flags & KOG_F_SIGN_V21, flags & KOG_F_SIGN_V22);
    const bool nonfinite = !all_finite(u) || !all_finite(v) || !is_finite(s1.f) || !is_finite(s2.f);
    Metrics m;
    metrics_whole_ext<T>(load_mat(gin, i), u, v, s1, s2, m);
    a.reG[i] = m.reG;
    a.reS1[i] = m.reS1;
    a.reS2[i] = m.reS2;
    a.reU[i] = m.reU;
    a.reV[i] = m.reV;
    a.kh[i] = m.kappa2.hi;
    a.kl[i] = m.kappa2.lo;
    const int32_t lo = static_cast<int32_t>(m.kappa2.e);
    const bool wide = static_cast<long long>(lo) != m.kappa2.e;
    a.ke[i] = lo;
    if (wide) a.xe2[i] = static_cast<int32_t>(m.kappa2.e >> 32);
    a.sflag[i] = 1u | (m.kappa_inf ? 2u : 0u) | (nonfinite ? 4u : 0u) | (wide ? 8u : 0u);
  }
}
// run_one on the pieces the split kernels left
template <class T>
__device__ __forceinline__ uint32_t run_one_split(const SvdBuf<T>& b, const StudyAux& a, uint64_t i, Metrics& m) {
  uint32_t flags = b.flags[i];
  const uint32_t sf = a.sflag[i];
  m.reG = a.reG[i];
  m.reS1 = a.reS1[i];
  m.reS2 = a.reS2[i];
  m.reU = a.reU[i];
  m.reV = a.reV[i];
  const int32_t ke = a.ke[i];
  long long e = ke;
  if (sf & 8u) e = (static_cast<long long>(a.xe2[i]) << 32) | static_cast<uint32_t>(ke);
  m.kappa2 = Ext{e, a.kh[i], a.kl[i]};
  m.kappa_inf = (sf & 2u) != 0;
  if (sf & 4u) flags |= KOG_M_NONFINITE_FACTOR;
  if (isnan(m.reG) || isnan(m.reS1) || isnan(m.reS2) || isnan(m.reU) || isnan(m.reV)) flags |= KOG_M_NAN_METRIC;
  return flags;
}

template <class T>
__device__ __forceinline__ uint32_t run_one_lasv2(const Mat<T>& g, Metrics& m) {
  ExtSvd ref;
  ref_sigma<T>(g, ref);  // metrics() reads the singular values only (inline Xf where it applies)
  const Lasv2<T> r = lasv2(g.g11, g.g12, g.g22);
  const Mat<T> u{r.csl, -r.snl, r.snl, r.csl};
  const Mat<T> v{r.csr, -r.snr, r.snr, r.csr};
  uint32_t flags = 0;
  if (!all_finite(u) || !all_finite(v) || !is_finite(r.ssmax) || !is_finite(r.ssmin)) flags |= KOG_M_NONFINITE_FACTOR;
  metrics(g, u, v, ext_from(r.ssmax), ext_from(r.ssmin), ref, m);
  if (isnan(m.reG) || isnan(m.reS1) || isnan(m.reS2) || isnan(m.reU) || isnan(m.reV)) flags |= KOG_M_NAN_METRIC;
  return flags;
}

template <class T>
__global__ void k_metrics(InP<T> in, kog_metrics* o, uint64_t n, Opt opt) {
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    Metrics m;
    const uint32_t flags = run_one_kog<T>(load_mat(in, i), opt, m);
    kog_metrics rec;
    rec.reG = m.reG;
    rec.reS1 = m.reS1;
    rec.reS2 = m.reS2;
    rec.reU = m.reU;
    rec.reV = m.reV;
    rec.kappa2 = to_c(m.kappa2);
    rec.kappa_inf = m.kappa_inf;
    rec.flags = flags;
    o[i] = rec;
  }
}

// ----------------------------------------------------------------- study
struct KappaBest {
  Ext k;
  unsigned long long idx;
  bool valid;
};

// (a, ia) beats (b, ib): larger under ext_cmp; ties go to the lower index,
// which is the reference's first-occurrence rule under its in-order absorb
// and block-ordered merge (harness.hpp:92-93, 103, 265-270)
__device__ __forceinline__ bool kappa_better(const Ext& a, unsigned long long ia, const Ext& b,
                                             unsigned long long ib, bool bvalid) {
  if (!bvalid) return true;
  const int c = ext_cmp(a, b);
  return c > 0 || (c == 0 && ia < ib);
}

// the lanes' packed byte counters into the block's 19 shared counts (t2p[7], path[7], then the five flags in
// BranchCounts' order: tanpsi_inf, diag_swap, compose_minus, sigma_swap, prescale_inexact = bits 10, 11, 13, 12, 14)
__device__ __forceinline__ void flush_counts(unsigned* cnt, unsigned long long t2p, unsigned long long path,
                                             unsigned long long fl) {
  const unsigned active = __activemask();
  const bool leader = (threadIdx.x & 31u) == static_cast<unsigned>(__ffs(active) - 1);
#pragma unroll
  for (unsigned k = 0; k < 7; ++k) {
    const unsigned a = __reduce_add_sync(active, static_cast<unsigned>(t2p >> (8u * k)) & 255u);
    const unsigned b = __reduce_add_sync(active, static_cast<unsigned>(path >> (8u * k)) & 255u);
    if (leader && a) atomicAdd(&cnt[k], a);
    if (leader && b) atomicAdd(&cnt[7 + k], b);
  }
  const int slot[5] = {14, 15, 17, 16, 18};
#pragma unroll
  for (unsigned k = 0; k < 5; ++k) {
    const unsigned a = __reduce_add_sync(active, static_cast<unsigned>(fl >> (8u * k)) & 255u);
    if (leader && a) atomicAdd(&cnt[slot[k]], a);
  }
}

// a > b under ext_cmp for the absorb's running maximum.  Positive canonical values (significands in
// [1 - 2^-54, 2)) whose exponents lie two or more apart are ordered by the exponents; the others take the
// subtraction as the reference does.
__device__ __forceinline__ bool kappa_gt(const Ext& a, const Ext& b) {
  if (a.hi > 0.0 && b.hi > 0.0) {
    const long long d = a.e - b.e;
    if (d >= 2) return true;
    if (d <= -2) return false;
  }
  return xf_cmp(xf_of(a), xf_of(b)) > 0;
}

struct BlockPartial {
  kog_extfloat k;
  unsigned long long idx;
  unsigned valid;
  unsigned pad;
};

// the five metrics are +0, positive or +inf on the absorbed path (never -0
// or NaN: ext_ratio and relerr return literal 0.0, NaN aborts the batch), so
// their bit patterns order like the values and fmax == unsigned max
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(__double_as_longlong(v)));
}

#ifndef KOG2_STUDY_MINB
#define KOG2_STUDY_MINB 2  // measured with the inline Xf metrics (phased, cfg5 rule, M matrices/s): 2 -> 1416, 3 -> 863, 4 -> 1263
#endif
#ifndef KOG2_STUDY_THREADS
#define KOG2_STUDY_THREADS 256
#endif
constexpr int kStudyThreads = KOG2_STUDY_THREADS;
template <class T, int ROUTINE, int PHASED>  // PHASED: 0 fused, 1 from the chunk's svd2 buffers, 2 from the split kernels' pieces too
__global__ void __launch_bounds__(kStudyThreads, PHASED == 2 ? KOG2_ABSORB_MINB : KOG2_STUDY_MINB)
    k_study(GenCfg c, uint64_t index0, uint64_t n, Opt opt, kog_stats* stats, BlockPartial* partial, InP<T> gin,
            SvdBuf<T> sb, bool accumulate, StudyAux aux) {
  __shared__ unsigned cnt[19];
  __shared__ double red[5][kStudyThreads / 32];
  __shared__ Ext kred_k[kStudyThreads / 32];
  __shared__ unsigned long long kred_i[kStudyThreads / 32];
  __shared__ int kred_v[kStudyThreads / 32];
  if (threadIdx.x < 19) cnt[threadIdx.x] = 0;
  __syncthreads();

  double mG = 0.0, mS1 = 0.0, mS2 = 0.0, mU = 0.0, mV = 0.0;
  KappaBest kb{ext_zero(), 0ull, false};
  bool kinf = false;
  unsigned long long fail = ~0ull;
  const unsigned lane = threadIdx.x & 31u;
  unsigned long long c_t2p = 0ull, c_path = 0ull, c_fl = 0ull;  // 7 + 7 + 5 counts, one byte each
  unsigned absorbed = 0u;

  for (uint64_t i = gtid(); i < n; i += gstride()) {
    const unsigned long long index = index0 + i;
    Metrics m;
    uint32_t flags;
    if constexpr (PHASED == 2) {
      flags = run_one_split<T>(sb, aux, i, m);
    } else if constexpr (PHASED == 1) {  // generated and decomposed by the earlier launches of this chunk
      flags = run_one_buf<T>(load_mat(gin, i), sb, i, m);
    } else {
      const Mat<T> g = generate<T>(c, index);
      if (ROUTINE == KOG_ROUTINE_KOG)
        flags = run_one_kog<T>(g, opt, m);
      else
        flags = run_one_lasv2<T>(g, m);
    }
    bool ok = true;
    if (flags & KOG_M_NONFINITE_FACTOR) {
      ok = false;
      const unsigned long long key = index * 4ull + KOG_FAIL_NONFINITE;
      if (key < fail) fail = key;
    } else if (flags & KOG_M_NAN_METRIC) {
      ok = false;
      const unsigned long long key = index * 4ull + KOG_FAIL_NAN_METRIC;
      if (key < fail) fail = key;
    }
    if (ok) {  // ErrorStats::absorb (harness.hpp:84-95)
      mG = fmax(mG, m.reG);
      mS1 = fmax(mS1, m.reS1);
      mS2 = fmax(mS2, m.reS2);
      mU = fmax(mU, m.reU);
      mV = fmax(mV, m.reV);
      if (m.kappa_inf) {
        kinf = true;
      } else if (kappa_gt(m.kappa2, kb.k)) {  // kb.k starts at zero like maxKappa2
        kb.k = m.kappa2;  // a lane's indices increase: first occurrence kept
        kb.idx = index;
        kb.valid = true;
      }
    }
    if (ROUTINE == KOG_ROUTINE_KOG) {  // BranchCounts::add (harness.hpp:56-64), into this thread's packed counters
      if (ok) {
        c_t2p += 1ull << (8u * ((flags >> KOG_F_T2P_SHIFT) & 7u));
        c_path += 1ull << (8u * ((flags >> KOG_F_PATH_SHIFT) & 7u));
        // flag bits 10..14, bit j to byte j (the multiplier's five copies put bit j at 8j; no two terms meet)
        c_fl += (static_cast<unsigned long long>((flags >> 10) & 31u) * 0x10204081ull) & 0x0101010101ull;
      }
      if (++absorbed == 255u) {  // (one byte per count; the lanes of a warp get here together)
        flush_counts(cnt, c_t2p, c_path, c_fl);
        c_t2p = c_path = c_fl = 0ull;
        absorbed = 0u;
      }
    }
  }
  if (ROUTINE == KOG_ROUTINE_KOG) flush_counts(cnt, c_t2p, c_path, c_fl);

  // ---- warp reduction (every lane participates)
  for (int off = 16; off > 0; off >>= 1) {
    mG = fmax(mG, __shfl_down_sync(0xffffffffu, mG, off));
    mS1 = fmax(mS1, __shfl_down_sync(0xffffffffu, mS1, off));
    mS2 = fmax(mS2, __shfl_down_sync(0xffffffffu, mS2, off));
    mU = fmax(mU, __shfl_down_sync(0xffffffffu, mU, off));
    mV = fmax(mV, __shfl_down_sync(0xffffffffu, mV, off));
    const unsigned long long of = __shfl_down_sync(0xffffffffu, fail, off);
    if (of < fail) fail = of;
    const int okinf = __shfl_down_sync(0xffffffffu, static_cast<int>(kinf), off);
    kinf = kinf || okinf != 0;
    Ext ok;
    ok.e = __shfl_down_sync(0xffffffffu, kb.k.e, off);
    ok.hi = __shfl_down_sync(0xffffffffu, kb.k.hi, off);
    ok.lo = __shfl_down_sync(0xffffffffu, kb.k.lo, off);
    const unsigned long long oi = __shfl_down_sync(0xffffffffu, kb.idx, off);
    const bool ov = __shfl_down_sync(0xffffffffu, static_cast<int>(kb.valid), off) != 0;
    if (ov && kappa_better(ok, oi, kb.k, kb.idx, kb.valid)) {
      kb.k = ok;
      kb.idx = oi;
      kb.valid = true;
    }
  }
  const unsigned warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = mG;
    red[1][warp] = mS1;
    red[2][warp] = mS2;
    red[3][warp] = mU;
    red[4][warp] = mV;
    kred_k[warp] = kb.k;
    kred_i[warp] = kb.idx;
    kred_v[warp] = kb.valid ? 1 : 0;
    if (fail != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(&stats->fail_key), fail);
    if (kinf) atomicExch(reinterpret_cast<unsigned long long*>(&stats->kappa_inf), 1ull);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v[5];
    for (int k = 0; k < 5; ++k) {
      v[k] = 0.0;
      for (int w = 0; w < kStudyThreads / 32; ++w) v[k] = fmax(v[k], red[k][w]);
    }
    atomic_max_nonneg(&stats->reG, v[0]);
    atomic_max_nonneg(&stats->reS1, v[1]);
    atomic_max_nonneg(&stats->reS2, v[2]);
    atomic_max_nonneg(&stats->reU, v[3]);
    atomic_max_nonneg(&stats->reV, v[4]);
    KappaBest best{ext_zero(), 0ull, false};
    if (accumulate) {  // this block's slot from the earlier chunks of the study (the merge is order-free)
      const BlockPartial old = partial[blockIdx.x];
      if (old.valid) best = KappaBest{Ext{old.k.e, old.k.hi, old.k.lo}, old.idx, true};
    }
    for (int w = 0; w < kStudyThreads / 32; ++w)
      if (kred_v[w] && kappa_better(kred_k[w], kred_i[w], best.k, best.idx, best.valid)) {
        best.k = kred_k[w];
        best.idx = kred_i[w];
        best.valid = true;
      }
    BlockPartial bp;
    bp.k = to_c(best.k);
    bp.idx = best.idx;
    bp.valid = best.valid ? 1u : 0u;
    bp.pad = 0;
    partial[blockIdx.x] = bp;
    if (ROUTINE == KOG_ROUTINE_KOG) {
      for (int k = 0; k < 7; ++k) {
        if (cnt[k]) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->t2p[k]), static_cast<unsigned long long>(cnt[k]));
        if (cnt[7 + k])
          atomicAdd(reinterpret_cast<unsigned long long*>(&stats->path[k]), static_cast<unsigned long long>(cnt[7 + k]));
      }
      unsigned long long* tail = reinterpret_cast<unsigned long long*>(&stats->tanpsi_inf);
      for (int k = 0; k < 5; ++k)
        if (cnt[14 + k]) atomicAdd(tail + k, static_cast<unsigned long long>(cnt[14 + k]));
    }
  }
}

// merge the per-block (kappa, index) slots into stats (one block)
__global__ void k_study_finish(kog_stats* stats, const BlockPartial* partial, int nblocks) {
  __shared__ Ext sk[kThreads];
  __shared__ unsigned long long si[kThreads];
  __shared__ int sv[kThreads];
  KappaBest best{ext_zero(), 0ull, false};
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
    const BlockPartial p = partial[b];
    if (!p.valid) continue;
    const Ext k{p.k.e, p.k.hi, p.k.lo};
    if (kappa_better(k, p.idx, best.k, best.idx, best.valid)) {
      best.k = k;
      best.idx = p.idx;
      best.valid = true;
    }
  }
  sk[threadIdx.x] = best.k;
  si[threadIdx.x] = best.idx;
  sv[threadIdx.x] = best.valid;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < static_cast<int>(blockDim.x); ++t)
      if (sv[t] && kappa_better(sk[t], si[t], best.k, best.idx, best.valid)) {
        best.k = sk[t];
        best.idx = si[t];
        best.valid = true;
      }
    // merge with earlier launches; a zero stored kappa means "none yet"
    const Ext cur{stats->max_kappa2.e, stats->max_kappa2.hi, stats->max_kappa2.lo};
    if (best.valid && kappa_better(best.k, best.idx, cur, stats->max_kappa2_index, !ext_is_zero(cur))) {
      stats->max_kappa2 = to_c(best.k);
      stats->max_kappa2_index = best.idx;
    }
  }
}

template <class T, class MatC>
int launch_metrics(const MatC* g, kog_metrics* o, uint64_t n, const kog_options* opt, cudaStream_t st) {
  if (!mat_ok<T>(g) || !o) return kog2_arg_error("kog_metrics_batch: null argument");
  if (n == 0) return KOG_OK;
  k_metrics<T><<<grid_for(n, 128), 128, 0, st>>>(in_of<T>(g), o, n, opt_of(opt));
  return launched("k_metrics");
}

template <class T, class MatC>
int launch_ext(const MatC* g, kog_extsvd* o, uint64_t n, cudaStream_t st) {
  if (!mat_ok<T>(g) || !o) return kog2_arg_error("kog_svd2_ext_batch: null argument");
  if (n == 0) return KOG_OK;
  k_svd2_ext<T><<<grid_for(n, 128), 128, 0, st>>>(in_of<T>(g), o, n);
  return launched("k_svd2_ext");
}


// ------------------------------------------------------------ study launcher
// Every call owns its scratch: the per-block (kappa, index) slots and, for the
// phased kog study, two chunks of generated matrices and their decompositions
// come from the stream-ordered workspace pool (kog2_ws.cpp) on the caller's
// stream and go back to it after the join, so studies on different streams or
// threads never share a buffer.

#ifndef KOG2_STUDY_STREAMS_DEFAULT
#define KOG2_STUDY_STREAMS_DEFAULT 1  // two consumer streams ran two k_study at once: erratic 500-1500 M/s at 2^31
#endif
#ifndef KOG2_STUDY_BPS_DEFAULT
#define KOG2_STUDY_BPS_DEFAULT 4  // the absorb kernel's resident blocks: one wave, one epilogue per block (r11: 8 -> 168 us, 4 -> 154 us, 16 -> 197 us)
#endif
// grid of the study kernels: at most `per_sm` blocks per SM (grid-stride loops)
int study_grid(uint64_t n, int sms, int per_sm = 8) {
  uint64_t want = (n + kStudyThreads - 1) / kStudyThreads;
  const uint64_t cap = static_cast<uint64_t>(sms) * static_cast<uint64_t>(per_sm);
  return static_cast<int>(want > cap ? cap : want);
}
// streams of the phased study: 0 = everything on the caller's stream, 1 = a
// producer stream and one consumer stream, 2 = a producer and two consumers
// (KOG2_STUDY_STREAMS overrides)
int study_streams_mode() {
  static const int v = [] {
    const char* e = std::getenv("KOG2_STUDY_STREAMS");
    const int x = e ? std::atoi(e) : -1;
    return x >= 0 && x <= 2 ? x : KOG2_STUDY_STREAMS_DEFAULT;
  }();
  return v;
}
// the metrics as separate kernels (default) or inside k_study (KOG2_STUDY_SPLIT=0, for A/B)
bool study_split() {
  static const bool v = [] {
#ifdef KOG2_STUDY_REF_KERNEL
    return false;
#else
    const char* e = std::getenv("KOG2_STUDY_SPLIT");
    return !(e && e[0] == '0');
#endif
  }();
  return v;
}
// the phased k_study's blocks per SM (KOG2_STUDY_BPS overrides, for tuning)
int study_bps() {
  static const int v = [] {
    const char* e = std::getenv("KOG2_STUDY_BPS");
    const int x = e ? std::atoi(e) : 0;
    return x > 0 ? x : KOG2_STUDY_BPS_DEFAULT;
  }();
  return v;
}

// Matrices per chunk of the phased study (kog_study_set_chunk_log2).  2^24 by default: from 2^23 the chunk's svd2
// call takes the two-speed kernel, and the per-chunk launches and tails shrink with the count (study over 2^28
// config-5 matrices, 10^6/s: 2^21 2,580, 2^22 2,676, 2^23 2,821, 2^24 2,887; two chunk buffers of 192 B per
// matrix: 6.4 GB of the 180).
#ifndef KOG2_STUDY_CHUNK_LOG2
#define KOG2_STUDY_CHUNK_LOG2 24
#endif
std::atomic<int> g_study_chunk_log2{KOG2_STUDY_CHUNK_LOG2};

template <class T> struct Abi;
template <> struct Abi<double> {
  using Mat = kog_mat_f64;
  using Out = kog_svd_out_f64;
  static int gen(const kog_run_config* c, uint64_t i0, const Mat* m, uint64_t n, void* st) {
    return kog_generate_batch_f64(c, i0, m, n, st);
  }
  static int svd(const Mat* m, const Out* o, uint64_t n, const kog_options* opt, void* st) {
    return kog_svd2_batch_f64(m, o, n, opt, st);
  }
};
template <> struct Abi<float> {
  using Mat = kog_mat_f32;
  using Out = kog_svd_out_f32;
  static int gen(const kog_run_config* c, uint64_t i0, const Mat* m, uint64_t n, void* st) {
    return kog_generate_batch_f32(c, i0, m, n, st);
  }
  static int svd(const Mat* m, const Out* o, uint64_t n, const kog_options* opt, void* st) {
    return kog_svd2_batch_f32(m, o, n, opt, st);
  }
};

// The kog study in phases per chunk — generate, the svd2 kernels (the
// specialised fast path where the Options allow), then the reference
// singular values + metrics + ErrorStats from the buffers.  Each launch runs
// a fraction of the fused kernel's code (the fused kernel was bound by
// instruction fetch: ~85% "no instruction" stalls), and the buffers cost
// ~200 B of HBM traffic per matrix.
template <class T>
int study_phased_run(const kog_run_config* cfg, uint64_t index0, uint64_t n, kog_stats* stats, int sms,
                     cudaStream_t st, uint64_t C, int nbuf, size_t per, int gmax, char* ws, BlockPartial* part,
                     Kog2SideStreams* side);
template <class T>
int study_phased(const kog_run_config* cfg, uint64_t index0, uint64_t n, kog_stats* stats, int sms, cudaStream_t st) {
  const uint64_t chunk = 1ull << g_study_chunk_log2.load(std::memory_order_relaxed);
  const uint64_t C = n < chunk ? n : chunk;
  const int nbuf = n > C ? 2 : 1;  // two chunk buffers when there is more than one chunk
  // per matrix: nine 8-byte arrays (the split kernels' pieces: five metrics and kappa_2's significand, or the
  // reference singular values of the A/B route), the input and the compact decomposition (10 T), exponents
  // and flags (4 x 4 B), kappa_2's exponent, the two lane marks, two intermediate exponents and the work list (6 x 4 B)
  const size_t per = static_cast<size_t>(C) * (9 * 8 + 10 * sizeof(T) + 10 * sizeof(int32_t));
  const int gmax = study_grid(C, sms, study_bps());
  // one set of per-block kappa slots per consumer stream (concurrent k_study
  // launches never share a slot) after the chunk buffers
  const size_t part_off = (per * nbuf + 255) / 256 * 256;
  const size_t need = part_off + sizeof(BlockPartial) * 2 * gmax + 2 * sizeof(uint32_t);  // + the lists' counters
  char* ws = static_cast<char*>(kog2_ws_alloc(need, st));
  if (!ws) return KOG_ERR_CUDA;
  BlockPartial* part = reinterpret_cast<BlockPartial*>(ws + part_off);
  Kog2SideStreams* side = kog2_side_acquire();
  if (!side) {
    kog2_ws_free(ws, st);
    return KOG_ERR_CUDA;
  }
  const int rc = study_phased_run<T>(cfg, index0, n, stats, sms, st, C, nbuf, per, gmax, ws, part, side);
  // the join (inside) has ordered every side-stream use of ws before this free
  const int frc = kog2_ws_free(ws, st);
  kog2_side_release(side);
  return rc != KOG_OK ? rc : frc;
}

template <class T>
int study_phased_run(const kog_run_config* cfg, uint64_t index0, uint64_t n, kog_stats* stats, int sms,
                     cudaStream_t st, uint64_t C, int nbuf, size_t per, int gmax, char* ws, BlockPartial* part,
                     Kog2SideStreams* side) {
  int rc = KOG_OK;
  const cudaStream_t s_prod = static_cast<cudaStream_t>(side->st[0]);
  const cudaStream_t s_cons[2] = {static_cast<cudaStream_t>(side->st[1]), static_cast<cudaStream_t>(side->st[2])};
  cudaEvent_t ev[8];
  for (int k = 0; k < 8; ++k) ev[k] = static_cast<cudaEvent_t>(side->ev[k]);
  cudaEvent_t* ready = ev;      // [2]
  cudaEvent_t* freed = ev + 2;  // [2]
  cudaEvent_t* join = ev + 4;   // [3]
  cudaEvent_t fork = ev[7];
  struct Bufs {
    typename Abi<T>::Mat gm;
    typename Abi<T>::Out om;
    InP<T> gin;
    SvdBuf<T> sb;
    StudyAux aux;
  } bufs[2];
  for (int k = 0; k < nbuf; ++k) {
    double* rd = reinterpret_cast<double*>(ws + per * k);  // the 8-byte arrays first
    long long* rq = reinterpret_cast<long long*>(rd);
    T* t = reinterpret_cast<T*>(rd + 9 * C);
    int32_t* w = reinterpret_cast<int32_t*>(t + 10 * C);
    // (the split kernels' pieces reuse the reference-sigma arrays of the KOG2_STUDY_REF_KERNEL A/B route)
    bufs[k].aux = StudyAux{rd + 6 * C, rd + 7 * C, rd + 8 * C, rd,        rd + C,    rd + 2 * C, rd + 3 * C,
                           w + 4 * C,  rd + 4 * C, rd + 5 * C, w + 7 * C, w + 8 * C, reinterpret_cast<uint32_t*>(w + 5 * C),
                           reinterpret_cast<uint32_t*>(w + 6 * C), reinterpret_cast<uint32_t*>(w + 9 * C),
                           reinterpret_cast<uint32_t*>(part + 2 * gmax) + k};
    bufs[k].gm = typename Abi<T>::Mat{t, t + C, t + 2 * C, t + 3 * C};
    const typename Abi<T>::Out om{t + 4 * C, t + 5 * C, w,         w + C,     t + 6 * C,
                                  t + 7 * C, t + 8 * C, t + 9 * C, w + 2 * C, reinterpret_cast<uint32_t*>(w + 3 * C)};
    bufs[k].om = om;
    bufs[k].gin = InP<T>{t, t + C, t + 2 * C, t + 3 * C};
    bufs[k].sb = SvdBuf<T>{om.sig1_f, om.sig2_f, om.sig1_e, om.sig2_e, om.u11, om.u12, om.v11,
                           om.v12,    om.flags,  rq,        rq + C,    rd + 2 * C, rd + 3 * C, rd + 4 * C, rd + 5 * C};
  }
  // every slot starts empty, each chunk's blocks merge into their own slot,
  // and k_study_finish merges all slots at the end
  if (cudaMemsetAsync(part, 0, sizeof(BlockPartial) * 2 * gmax, st) != cudaSuccess)
    return kog2_cuda_error("cudaMemsetAsync(study partials)");
  // fork from the caller's stream
  const int mode = study_streams_mode();
  const cudaStream_t prod = mode == 0 ? st : s_prod;
  const cudaStream_t cons[2] = {mode == 0 ? st : s_cons[0], mode == 2 ? s_cons[1] : (mode == 0 ? st : s_cons[0])};
  if (cudaEventRecord(fork, st) != cudaSuccess || cudaStreamWaitEvent(s_prod, fork, 0) != cudaSuccess ||
      cudaStreamWaitEvent(s_cons[0], fork, 0) != cudaSuccess || cudaStreamWaitEvent(s_cons[1], fork, 0) != cudaSuccess)
    return kog2_cuda_error("study fork");
  // on an error after the fork, the join below still runs, so nothing enqueued
  // on a side stream can outlive the workspace freed on st by the caller
  uint64_t c = 0;
  for (uint64_t lo = 0; lo < n && rc == KOG_OK; lo += C, ++c) {
    const uint64_t len = n - lo < C ? n - lo : C;
    const int k = static_cast<int>(c & 1);
    Bufs& bf = bufs[nbuf == 2 ? k : 0];
    cudaStream_t q = cons[k];
    // producer: generate + svd2 into buffer k once its previous consumer is done
    if (c >= 2 && cudaStreamWaitEvent(prod, freed[k], 0) != cudaSuccess) {
      rc = kog2_cuda_error("study wait");
      break;
    }
    if ((rc = Abi<T>::gen(cfg, index0 + lo, &bf.gm, len, prod)) != KOG_OK) break;
    if ((rc = Abi<T>::svd(&bf.gm, &bf.om, len, &cfg->options, prod)) != KOG_OK) break;
    // consumer k: reference sigma + metrics + ErrorStats
    if (cudaEventRecord(ready[k], prod) != cudaSuccess || cudaStreamWaitEvent(q, ready[k], 0) != cudaSuccess) {
      rc = kog2_cuda_error("study chunk handoff");
      break;
    }
#ifdef KOG2_STUDY_REF_KERNEL  // (the separate reference-sigma pass, for A/B)
    k_ref_sigma<T><<<grid_for(len), kThreads, 0, q>>>(bf.gin, bf.sb, len);
    if ((rc = launched("k_ref_sigma")) != KOG_OK) break;
#endif
    const int grid = study_grid(len, sms, study_bps());
    if (study_split()) {
      const int gs = grid_for(len);
      k_study_urv<T><<<gs, kThreads, 0, q>>>(bf.gin, bf.aux, len);
      if ((rc = launched("k_study_urv")) != KOG_OK) break;
      k_study_sigma<T><<<gs, kThreads, 0, q>>>(bf.sb, bf.aux, len);
      if ((rc = launched("k_study_sigma")) != KOG_OK) break;
      k_study_recon<T><<<gs, kThreads, 0, q>>>(bf.gin, bf.sb, bf.aux, len);
      if ((rc = launched("k_study_recon")) != KOG_OK) break;
      k_study_ratio<T><<<gs, kThreads, 0, q>>>(bf.gin, bf.aux, len);
      if ((rc = launched("k_study_ratio")) != KOG_OK) break;
      if (cudaMemsetAsync(bf.aux.count, 0, sizeof(uint32_t), q) != cudaSuccess) {
        rc = kog2_cuda_error("cudaMemsetAsync(study list)");
        break;
      }
      k_study_ortho<T, false><<<gs, kThreads, 0, q>>>(bf.sb.u11, bf.sb.u12, bf.sb.flags, KOG_F_SIGN_U21,
                                                      KOG_F_SIGN_U22, bf.aux.fin, bf.aux.reU, len, bf.aux);
      if ((rc = launched("k_study_ortho")) != KOG_OK) break;
      k_study_ortho<T, true><<<gs, kThreads, 0, q>>>(bf.sb.v11, bf.sb.v12, bf.sb.flags, KOG_F_SIGN_V21,
                                                     KOG_F_SIGN_V22, bf.aux.fin, bf.aux.reV, len, bf.aux);
      if ((rc = launched("k_study_ortho")) != KOG_OK) break;
      k_study_whole<T><<<sms, kThreads, 0, q>>>(bf.gin, bf.sb, bf.aux);
      if ((rc = launched("k_study_whole")) != KOG_OK) break;
      k_study<T, KOG_ROUTINE_KOG, 2><<<grid, kStudyThreads, 0, q>>>(GenCfg{}, index0 + lo, len, Opt{}, stats,
                                                                    part + k * gmax, bf.gin, bf.sb, true, bf.aux);
    } else {
      k_study<T, KOG_ROUTINE_KOG, 1><<<grid, kStudyThreads, 0, q>>>(GenCfg{}, index0 + lo, len, Opt{}, stats,
                                                                    part + k * gmax, bf.gin, bf.sb, true, StudyAux{});
    }
    if ((rc = launched("k_study")) != KOG_OK) break;
    if (cudaEventRecord(freed[k], q) != cudaSuccess) {
      rc = kog2_cuda_error("study chunk release");
      break;
    }
  }
  // join back into the caller's stream
  const cudaStream_t sides[3] = {s_prod, s_cons[0], s_cons[1]};
  for (int k = 0; k < 3; ++k)
    if (cudaEventRecord(join[k], sides[k]) != cudaSuccess || cudaStreamWaitEvent(st, join[k], 0) != cudaSuccess) {
      // cannot order the side streams before the caller's free: drain them
      for (auto q : sides) cudaStreamSynchronize(q);
      return rc != KOG_OK ? rc : kog2_cuda_error("study join");
    }
  if (rc != KOG_OK) return rc;
  k_study_finish<<<1, kThreads, 0, st>>>(stats, part, 2 * gmax);
  return launched("k_study_finish");
}

}  // namespace

extern "C" {

int kog_study_set_chunk_log2(int log2_matrices) {
  const int v = log2_matrices < 16 ? 16 : (log2_matrices > 26 ? 26 : log2_matrices);
  return g_study_chunk_log2.exchange(v);
}

int kog_svd2_ext_batch_f64(const kog_mat_f64* g, kog_extsvd* out, uint64_t n, void* stream) {
  return launch_ext<double>(g, out, n, KOG2_ST(stream));
}
int kog_svd2_ext_batch_f32(const kog_mat_f32* g, kog_extsvd* out, uint64_t n, void* stream) {
  return launch_ext<float>(g, out, n, KOG2_ST(stream));
}
int kog_metrics_batch_f64(const kog_mat_f64* g, kog_metrics* out, uint64_t n, const kog_options* opt, void* stream) {
  return launch_metrics<double>(g, out, n, opt, KOG2_ST(stream));
}
int kog_metrics_batch_f32(const kog_mat_f32* g, kog_metrics* out, uint64_t n, const kog_options* opt, void* stream) {
  return launch_metrics<float>(g, out, n, opt, KOG2_ST(stream));
}

int kog_study_stats_alloc(kog_stats** stats_dev) {
  if (!stats_dev) return kog2_arg_error("kog_study_stats_alloc: null argument");
  if (cudaMalloc(reinterpret_cast<void**>(stats_dev), sizeof(kog_stats)) != cudaSuccess)
    return kog2_cuda_error("cudaMalloc(kog_stats)");
  return kog_study_stats_reset(*stats_dev, nullptr);
}
int kog_study_stats_free(kog_stats* stats_dev) {
  if (stats_dev) cudaFree(stats_dev);
  return KOG_OK;
}
int kog_study_stats_reset(kog_stats* stats_dev, void* stream) {
  if (!stats_dev) return kog2_arg_error("kog_study_stats_reset: null argument");
  kog_stats init;
  kog_stats_init(&init);
  if (cudaMemcpyAsync(stats_dev, &init, sizeof init, cudaMemcpyHostToDevice, KOG2_ST(stream)) != cudaSuccess)
    return kog2_cuda_error("cudaMemcpyAsync(kog_stats)");
  return cudaStreamSynchronize(KOG2_ST(stream)) == cudaSuccess ? KOG_OK : kog2_cuda_error("cudaStreamSynchronize");
}

int kog_study_batch(const kog_run_config* cfg, uint64_t index0, uint64_t n, kog_stats* stats_dev, void* stream) {
  if (!cfg || !stats_dev) return kog2_arg_error("kog_study_batch: null argument");
  if (kog_validate(cfg) != KOG_OK) return KOG_ERR_ARG;
  if (n == 0) return KOG_OK;
  const int sms = kog2_sm_count();
  cudaStream_t st = KOG2_ST(stream);
  if (cfg->routine == KOG_ROUTINE_KOG)
    return cfg->single_precision ? study_phased<float>(cfg, index0, n, stats_dev, sms, st)
                                 : study_phased<double>(cfg, index0, n, stats_dev, sms, st);
  // the lasv2 routine: one fused kernel over the range, per-call block slots
  const int grid = study_grid(n, sms);
  BlockPartial* part = static_cast<BlockPartial*>(kog2_ws_alloc(sizeof(BlockPartial) * grid, st));
  if (!part) return KOG_ERR_CUDA;
  const Opt o = opt_of(&cfg->options);
  if (cfg->single_precision)
    k_study<float, KOG_ROUTINE_LASV2, false><<<grid, kStudyThreads, 0, st>>>(gen_cfg_of<float>(cfg), index0, n, o, stats_dev,
                                                                         part, InP<float>{}, SvdBuf<float>{}, false, StudyAux{});
  else
    k_study<double, KOG_ROUTINE_LASV2, false><<<grid, kStudyThreads, 0, st>>>(gen_cfg_of<double>(cfg), index0, n, o, stats_dev,
                                                                          part, InP<double>{}, SvdBuf<double>{}, false, StudyAux{});
  int rc = launched("k_study");
  if (rc == KOG_OK) {
    k_study_finish<<<1, kThreads, 0, st>>>(stats_dev, part, grid);
    rc = launched("k_study_finish");
  }
  const int frc = kog2_ws_free(part, st);
  return rc != KOG_OK ? rc : frc;
}

}  // extern "C"
