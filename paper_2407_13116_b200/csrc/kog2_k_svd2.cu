// kog2_k_svd2.cu — the hot kernels: batched svd2 (svd2.hpp:603-687) over
// structure-of-arrays device buffers, one thread per matrix, compact result
// layout of include/kog2.h.
//
// The default Options run in two stream-ordered launches:
//   k_svd2_fast  the specialised straight-line path (kog2_fast.cuh) over the
//                whole batch; every lane writes its result, and lanes whose
//                input leaves that path's domain append their index to a
//                compacted list (one warp-aggregated atomic per warp);
//   k_svd2_list  the general algorithm (kog2_svd2.cuh) over the listed
//                indices only, overwriting those results — full warps of
//                deferred work instead of divergent lanes in every warp.
// binary32 with the default Options takes the same two launches (the
// binary32 instantiation of kog2_fast.cuh); other Options run the general
// kernel over the batch.
#include <cstdlib>

#include "kog2_common.cuh"
#include "kog2_fast.cuh"

using namespace kog2;

namespace {

template <class T>
struct OutP {
  T *sig1_f, *sig2_f;
  int32_t *sig1_e, *sig2_e;
  T *u11, *u12, *v11, *v12;
  int32_t* s;
  uint32_t* flags;
};

template <class T>
__device__ __forceinline__ uint32_t sign_flags(const Result<T>& r) {
  uint32_t f = 0;
  if (sign_bit(r.u.g21)) f |= KOG_F_SIGN_U21;
  if (sign_bit(r.u.g22)) f |= KOG_F_SIGN_U22;
  if (sign_bit(r.v.g21)) f |= KOG_F_SIGN_V21;
  if (sign_bit(r.v.g22)) f |= KOG_F_SIGN_V22;
  return f;
}

template <class T, class I>
__device__ __forceinline__ void store_result(const OutP<T>& out, I i, const Result<T>& r) {
  st_cs(out.sig1_f + i, r.sigma1.f);
  st_cs(out.sig2_f + i, r.sigma2.f);
  st_cs(out.sig1_e + i, static_cast<int32_t>(r.sigma1.e));
  st_cs(out.sig2_e + i, static_cast<int32_t>(r.sigma2.e));
  st_cs(out.u11 + i, r.u.g11);
  st_cs(out.u12 + i, r.u.g12);
  st_cs(out.v11 + i, r.v.g11);
  st_cs(out.v12 + i, r.v.g12);
  st_cs(out.s + i, static_cast<int32_t>(r.s));
  st_cs(out.flags + i, r.flags | sign_flags(r));
}

// the general algorithm over the whole batch
template <class T, bool DEF>
__global__ void __launch_bounds__(kThreads, 3) k_svd2(InP<T> in, OutP<T> out, uint64_t n, Opt ropt) {
  const Opt o = DEF ? opt_default() : ropt;
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    const Mat<T> g{ld_cs(in.g11 + i), ld_cs(in.g12 + i), ld_cs(in.g21 + i), ld_cs(in.g22 + i)};
    Result<T> r;
    svd2<T>(g, o, r);
    store_result(out, i, r);
  }
}

// the specialised path; deferred indices go to list[0 .. *count)
#ifndef KOG2_FAST_MINB
#define KOG2_FAST_MINB 2
#endif
#ifndef KOG2_FAST_THREADS
#define KOG2_FAST_THREADS 512  // 512 x 2 blocks/SM measured 0.5% faster than 256 x 4 (12.58 vs 12.64 ms per 2^28 cfg3)
#endif
// binary32 block shape: its kernel needs fewer registers than binary64's;
// 512 x 3 blocks/SM (40 registers, a 24-byte spill) measured best on config 4
// (8.89 ms per 2^28 against 8.92 for 384 x 4 and 256 x 5, 8.97 for 256 x 6,
// 9.29 for 512 x 2; profiles/r9_ab_f32_shape.txt)
#ifndef KOG2_F32_THREADS
#define KOG2_F32_THREADS 512
#endif
#ifndef KOG2_F32_MINB
#define KOG2_F32_MINB 3
#endif
template <class T>
struct FastShape {
  static constexpr int threads = KOG2_FAST_THREADS, minb = KOG2_FAST_MINB;
};
template <>
struct FastShape<float> {
  static constexpr int threads = KOG2_F32_THREADS, minb = KOG2_F32_MINB;
};
template <class T>
__global__ void __launch_bounds__(FastShape<T>::threads, FastShape<T>::minb)
    k_svd2_fast(InP<T> in, OutP<T> out, uint64_t n, uint32_t* list, unsigned* count) {
  const unsigned lane = threadIdx.x & 31u;
  // 32-bit indices: n <= kFastChunk = 2^31 per launch, so i + stride < 2^32
  // (one 32x32->64 multiply-add per array address instead of 64-bit arithmetic)
  const unsigned n32 = static_cast<unsigned>(n), stride = gridDim.x * blockDim.x;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += stride) {
    const Mat<T> g{ld_cs(in.g11 + i), ld_cs(in.g12 + i), ld_cs(in.g21 + i), ld_cs(in.g22 + i)};
    Result<T> r;
    bool bad = false;
    fast::svd2_fast(g, r, bad);
    store_result(out, i, r);
    const unsigned active = __activemask();
    const unsigned m = __ballot_sync(active, bad);
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned base = 0;
      if (static_cast<int>(lane) == leader) base = atomicAdd(count, static_cast<unsigned>(__popc(m)));
      base = __shfl_sync(active, base, leader);
      if (bad) list[base + __popc(m & ((1u << lane) - 1u))] = i;
    }
  }
}

#ifdef KOG2_FAST_TMA
// Experiment (A/B builds only): k_svd2_fast with its input tiles fetched by
// the bulk-copy engine.  Each warp owns a 32-matrix tile per iteration (the
// same indices as k_svd2_fast); lane 0 prefetches the warp's tile two
// iterations ahead into a double-buffered shared-memory slot (four 32-entry
// cp.async.bulk copies completing on the slot's mbarrier), and the lanes read
// their entries from shared memory.  The last, partial tile loads directly.
template <class T>
struct TmaSlot {
  T in[2][4][32];
  unsigned long long mbar[2];
};
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
template <class T>
__device__ __forceinline__ void tma_issue(TmaSlot<T>& S, int b, const InP<T>& in, unsigned t) {
  constexpr unsigned bytes = 32 * sizeof(T);
  const unsigned mb = smem_u32(&S.mbar[b]);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(4 * bytes) : "memory");
  const T* src[4] = {in.g11, in.g12, in.g21, in.g22};
#pragma unroll
  for (int f = 0; f < 4; ++f)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(&S.in[b][f][0])),
                 "l"(src[f] + static_cast<size_t>(t) * 32), "r"(bytes), "r"(mb)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned mb, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(mb),
      "r"(parity)
      : "memory");
}
template <class T>
__global__ void __launch_bounds__(KOG2_FAST_THREADS, KOG2_FAST_MINB)
    k_svd2_fast_tma(InP<T> in, OutP<T> out, uint64_t n, uint32_t* list, unsigned* count) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const unsigned lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  TmaSlot<T>& S = reinterpret_cast<TmaSlot<T>*>(smem_raw)[wib];
  const unsigned n32 = static_cast<unsigned>(n), full = n32 / 32u;
  const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
  const unsigned t0 = blockIdx.x * (blockDim.x >> 5) + wib;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.mbar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.mbar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (t0 < full) tma_issue(S, 0, in, t0);
    if (t0 + nwarps < full) tma_issue(S, 1, in, t0 + nwarps);
  }
  __syncwarp();
  unsigned k = 0;
  for (unsigned t = t0; t * 32u < n32; t += nwarps, ++k) {
    const unsigned i = t * 32u + lane;
    const int b = k & 1;
    Mat<T> g;
    if (t < full) {
      mbar_wait(smem_u32(&S.mbar[b]), (k >> 1) & 1u);
      g = Mat<T>{S.in[b][0][lane], S.in[b][1][lane], S.in[b][2][lane], S.in[b][3][lane]};
      __syncwarp();
      if (lane == 0 && t + 2 * nwarps < full) tma_issue(S, b, in, t + 2 * nwarps);
    } else {
      if (i >= n32) break;
      g = Mat<T>{ld_cs(in.g11 + i), ld_cs(in.g12 + i), ld_cs(in.g21 + i), ld_cs(in.g22 + i)};
    }
    Result<T> r;
    bool bad = false;
    fast::svd2_fast(g, r, bad);
    store_result(out, i, r);
    const unsigned active = __activemask();
    const unsigned m = __ballot_sync(active, bad);
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned base = 0;
      if (static_cast<int>(lane) == leader) base = atomicAdd(count, static_cast<unsigned>(__popc(m)));
      base = __shfl_sync(active, base, leader);
      if (bad) list[base + __popc(m & ((1u << lane) - 1u))] = i;
    }
  }
}
template <class T>
bool tma_ok(const InP<T>& ip) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(ip.g11) | reinterpret_cast<uintptr_t>(ip.g12) |
                      reinterpret_cast<uintptr_t>(ip.g21) | reinterpret_cast<uintptr_t>(ip.g22);
  return (a & 15u) == 0;
}
#endif

// matrices recomputed by k_svd2_list on this device since load (diagnostics:
// kog_svd2_deferred_count)
__device__ unsigned long long g_kog2_deferred_total = 0;

// the general algorithm over the deferred indices (gathered loads/stores)
template <class T>
__global__ void __launch_bounds__(kThreads, 3)
    k_svd2_list(InP<T> in, OutP<T> out, const uint32_t* list, const unsigned* count) {
  const uint64_t cnt = *count;
  if (cnt && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_kog2_deferred_total, static_cast<unsigned long long>(cnt));
  for (uint64_t k = gtid(); k < cnt; k += gstride()) {
    const uint64_t i = list[k];
    const Mat<T> g{in.g11[i], in.g12[i], in.g21[i], in.g22[i]};
    Result<T> r;
    svd2<T>(g, opt_default(), r);
    store_result(out, i, r);
  }
}

constexpr uint64_t kFastChunk = 1ull << 31;  // uint32 deferred indices per launch pair

template <class T, class MatC, class OutC>
int launch_svd2(const MatC* in, const OutC* out, uint64_t n, const kog_options* opt, cudaStream_t st) {
  if (n == 0) return KOG_OK;  // empty batch: nothing is dereferenced
  if (!in || !out) return kog2_arg_error("kog_svd2_batch: null argument");
  const OutP<T> op{out->sig1_f, out->sig2_f, out->sig1_e, out->sig2_e, out->u11,
                   out->u12,    out->v11,    out->v12,    out->s,      out->flags};
  if (!mat_ok<T>(in) || !op.sig1_f || !op.sig2_f || !op.sig1_e || !op.sig2_e || !op.u11 || !op.u12 ||
      !op.v11 || !op.v12 || !op.s || !op.flags)
    return kog2_arg_error("kog_svd2_batch: null array pointer");
  const Opt o = opt_of(opt);
  static const bool general_only = std::getenv("KOG2_SVD2_GENERAL") != nullptr;  // A/B comparisons
  {
    if (opt_is_default(o) && !general_only) {
      // per-call deferral scratch, stream-ordered from the workspace pool: the
      // count (first 256 bytes) and one index per matrix of the largest launch
      // (4 B/matrix against the caller's 96, or 56 for binary32)
      const uint64_t cap = n < kFastChunk ? n : kFastChunk;
      char* ws = static_cast<char*>(kog2_ws_alloc(256 + cap * sizeof(uint32_t), st));
      if (!ws) return KOG_ERR_CUDA;
      unsigned* count = reinterpret_cast<unsigned*>(ws);
      uint32_t* list = reinterpret_cast<uint32_t*>(ws + 256);
      const int sms = kog2_sm_count();
      int rc = KOG_OK;
      for (uint64_t lo = 0; lo < n && rc == KOG_OK; lo += kFastChunk) {
        const uint64_t len = n - lo < kFastChunk ? n - lo : kFastChunk;
        const InP<T> ip{in->g11 + lo, in->g12 + lo, in->g21 + lo, in->g22 + lo};
        const OutP<T> ol{op.sig1_f + lo, op.sig2_f + lo, op.sig1_e + lo, op.sig2_e + lo, op.u11 + lo,
                         op.u12 + lo,    op.v11 + lo,    op.v12 + lo,    op.s + lo,      op.flags + lo};
        if (cudaMemsetAsync(count, 0, sizeof(unsigned), st) != cudaSuccess) {
          rc = kog2_cuda_error("cudaMemsetAsync(defer count)");
          break;
        }
#ifdef KOG2_FAST_TMA
        if (tma_ok(ip)) {
          constexpr int smem = (KOG2_FAST_THREADS / 32) * sizeof(TmaSlot<T>);
          static const bool attr = cudaFuncSetAttribute(k_svd2_fast_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        smem) == cudaSuccess;
          (void)attr;
          k_svd2_fast_tma<T><<<grid_for(len, KOG2_FAST_THREADS), KOG2_FAST_THREADS, smem, st>>>(ip, ol, len, list,
                                                                                               count);
        } else
#endif
          k_svd2_fast<T><<<grid_for(len, FastShape<T>::threads), FastShape<T>::threads, 0, st>>>(ip, ol, len, list,
                                                                                           count);
        if ((rc = launched("k_svd2_fast")) != KOG_OK) break;
        // deferred lanes are rare (none in 2^22-matrix samples of configs 1-5):
        // two blocks per SM drain a list of any length (grid-stride)
        k_svd2_list<T><<<2 * sms, kThreads, 0, st>>>(ip, ol, list, count);
        rc = launched("k_svd2_list");
      }
      const int frc = kog2_ws_free(ws, st);
      return rc != KOG_OK ? rc : frc;
    }
  }
  const int grid = grid_for(n);
  if (opt_is_default(o))
    k_svd2<T, true><<<grid, kThreads, 0, st>>>(in_of<T>(in), op, n, o);
  else
    k_svd2<T, false><<<grid, kThreads, 0, st>>>(in_of<T>(in), op, n, o);
  return launched("k_svd2");
}

}  // namespace

extern "C" {

#ifdef KOG2_FAST_STATS
// debug builds: per-reason counts of lanes that left the fast path (kog2_fast.cuh)
// (out[0..15] = deferral reasons, out[16..31] = rare-path calls, out[32..95] = per-site division events)
int kog2_fast_stats(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_kog2_fast_bad, sizeof(g_kog2_fast_bad)) != cudaSuccess ||
      cudaMemcpyFromSymbol(out + KOG2_R_COUNT, g_kog2_rare, sizeof(g_kog2_rare)) != cudaSuccess)
    return kog2_cuda_error("cudaMemcpyFromSymbol");
  if (cudaMemcpyFromSymbol(out + 32, kog2::fast::g_kog2_div_site, sizeof(kog2::fast::g_kog2_div_site)) != cudaSuccess)
    return kog2_cuda_error("cudaMemcpyFromSymbol");
  if (reset) {
    const unsigned long long z[64] = {};
    cudaMemcpyToSymbol(g_kog2_fast_bad, z, sizeof(g_kog2_fast_bad));
    cudaMemcpyToSymbol(g_kog2_rare, z, sizeof(g_kog2_rare));
    cudaMemcpyToSymbol(kog2::fast::g_kog2_div_site, z, sizeof(kog2::fast::g_kog2_div_site));
  }
  return KOG_OK;
}
#endif

int64_t kog_svd2_deferred_count(void) {
  unsigned long long c = 0;
  if (cudaMemcpyFromSymbol(&c, g_kog2_deferred_total, sizeof c) != cudaSuccess) {
    kog2_cuda_error("cudaMemcpyFromSymbol(deferred total)");
    return -1;
  }
  return static_cast<int64_t>(c);
}

int kog_svd2_batch_f64(const kog_mat_f64* in, const kog_svd_out_f64* out, uint64_t n,
                       const kog_options* opt, void* stream) {
  return launch_svd2<double>(in, out, n, opt, KOG2_ST(stream));
}
int kog_svd2_batch_f32(const kog_mat_f32* in, const kog_svd_out_f32* out, uint64_t n,
                       const kog_options* opt, void* stream) {
  return launch_svd2<float>(in, out, n, opt, KOG2_ST(stream));
}

}  // extern "C"
