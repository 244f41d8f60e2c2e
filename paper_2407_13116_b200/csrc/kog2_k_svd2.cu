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
#include <atomic>
#include <cstdlib>

#include "kog2_common.cuh"
#include "kog2_fast.cuh"
#include "kog2_lean.cuh"

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

// STREAM: evict-first stores (whole sectors written once); the two-speed
// kernel writes a sector's lanes at two moments and keeps the default policy
// so that L2 merges them
template <bool STREAM, class V>
__device__ __forceinline__ void st_out(V* p, V v) {
  if constexpr (STREAM) st_cs(p, v);
  else *p = v;
}
template <bool STREAM = true, class T, class I>
__device__ __forceinline__ void store_result(const OutP<T>& out, I i, const Result<T>& r) {
  st_out<STREAM>(out.sig1_f + i, r.sigma1.f);
  st_out<STREAM>(out.sig2_f + i, r.sigma2.f);
  st_out<STREAM>(out.sig1_e + i, static_cast<int32_t>(r.sigma1.e));
  st_out<STREAM>(out.sig2_e + i, static_cast<int32_t>(r.sigma2.e));
  st_out<STREAM>(out.u11 + i, r.u.g11);
  st_out<STREAM>(out.u12 + i, r.u.g12);
  st_out<STREAM>(out.v11 + i, r.v.g11);
  st_out<STREAM>(out.v12 + i, r.v.g12);
  st_out<STREAM>(out.s + i, static_cast<int32_t>(r.s));
  st_out<STREAM>(out.flags + i, r.flags | sign_flags(r));
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
    k_svd2_fast(InP<T> in, OutP<T> out, uint64_t n, uint32_t* list, unsigned* count, const unsigned* gate) {
  if (gate && *gate == 0u) return;  // k_svd2_lean kept the batch
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

// One matrix through the specialised path (k_svd2_fast's loop body): result
// stored, a deferred lane appended to the list for k_svd2_list.
template <class T, int CLS>
__device__ __forceinline__ void fast_one(const InP<T>& in, const OutP<T>& out, unsigned i, uint32_t* list,
                                         unsigned* count, unsigned lane) {
  const Mat<T> g{in.g11[i], in.g12[i], in.g21[i], in.g22[i]};  // read a moment ago by the lean pass: L2
  Result<T> r;
  bool bad = false;
  fast::svd2_fast<T, CLS>(g, r, bad);
  store_result<false>(out, i, r);
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

// binary64, default Options, large batches: the two-speed kernel.
//
// Each warp walks 32-matrix tiles through svd2_lean (kog2_lean.cuh: the
// separated t' = 15 case, about a third of svd2_fast's instructions) and
// sorts the lanes it does not cover into two queues in the block's shared
// memory, so that the rest of the work runs as full warps on one kind of
// route each:
//   class T  every pattern that goes through a triangle (t = 15, t ~ 13 and the
//            one-row/column patterns that ride along urv15): svd2_fast<3>;
//   class S  svd_simple patterns: svd2_fast<0>.
// The warp whose push takes a queue across a multiple of 32 runs those 32.
// (A single queue ran at 12 of 32 lanes: the queue concentrates the divergent
// lanes, and svd_simple lanes leave at once.  A third queue for t ~ 13, run by
// the whole block in phases to keep its 16 KB of code out of the 32 KB
// instruction cache, cost 14% of the kernel's time for 3% of the matrices in
// barriers, cold code and far-away output sectors; sharing the class T
// instance costs those lanes' warps ~100 more instructions per batch instead.
// profiles/r3_lean_kernel_notes.txt has the numbers of every step.)
// The block's thirty-two warps (one block of 1024 threads per SM) fill a batch
// within a fraction of a tile, so the queued matrices' inputs and the output
// sectors they share with their neighbours are still in L2 when the batch
// runs; with a queue per warp they had long left it.  Queue slots are
// exact-turn words (q_put / q_take below); no warp waits for anything but a
// running warp's next step, no block waits for another, and tiles are handed
// out dynamically, eight consecutive tiles per grab.
// Outputs: a sector must be written whole the first time (a first partial
// write costs a DRAM fill read and a second write-back), so the lanes that are
// queued store their (meaningless) lean result too and their batch overwrites
// it a moment later; the fences order the two stores.  The next tile's inputs
// are copied to shared memory while the current one is computed (cp.async).
// A batch whose 1024-matrix sample says svd2_lean would fail on more than
// about half the matrices sets LeanGlobal::mode and leaves the whole batch to
// k_svd2_fast, launched behind it.
#ifndef KOG2_LEAN_PROBE
#define KOG2_LEAN_PROBE 16
#endif
__device__ __forceinline__ unsigned ld_vol(const unsigned* p) { return *reinterpret_cast<const volatile unsigned*>(p); }
#ifdef KOG2_LEAN_DEBUG
// debug builds: spins are counted per site (in pinned host memory when set, so a hung kernel can be watched)
__device__ unsigned g_lean_dbg[64];
__device__ unsigned* g_lean_host = nullptr;
#define KOG2_SPIN(cond, site, a, b)                                      \
  do {                                                                   \
    unsigned spins_ = 0;                                                 \
    while (cond) {                                                       \
      if ((++spins_ & 0xfffu) == 0u) {                                   \
        atomicAdd(&g_lean_dbg[2 + (site)], 1u);                          \
        if (g_lean_host) {                                               \
          atomicAdd(&g_lean_host[(site)], 1u);                           \
          if ((spins_ >> 12) == 64u) {                                   \
            const unsigned k_ = 16u + 6u * (site);                       \
            g_lean_host[k_] = blockIdx.x;                                \
            g_lean_host[k_ + 1] = threadIdx.x;                           \
            g_lean_host[k_ + 2] = (a);                                   \
            g_lean_host[k_ + 3] = (b);                                   \
          }                                                              \
        }                                                                \
      }                                                                  \
    }                                                                    \
  } while (0)
#else
#define KOG2_SPIN(cond, site, a, b) \
  while (cond) {                    \
  }
#endif
typedef unsigned long long u64;
// Ring slots (multi-producer, multi-consumer, exact turns).  A slot word is
// (state << 32) | index: state 2L = empty, lap L's producer may write; 2L + 1 =
// holds lap L's index; the lap of position p in a ring of 2^k slots is p >> k.
// The producer's wait and write are ONE compare-and-swap: with the store behind
// a wait loop, a lane whose turn has come would sit at the loop's reconvergence
// point until the warp's other lanes leave it — and a lane of another class may
// be waiting for a batch that the warp waiting for THIS entry has yet to run.
// Exact turns matter for the same reason: if a later lap's producer could take a
// freed slot first, the earlier one would wait for a consumer that may in turn
// be waiting for it (seen as a hang with free-for-all slots).  With both, every
// wait is for a running warp's step on a strictly earlier reservation, so the
// waits cannot form a cycle.
__device__ __forceinline__ u64 q_word(unsigned state, unsigned v) { return (static_cast<u64>(state) << 32) | v; }
__device__ __forceinline__ void q_put(u64* slot, unsigned lap, unsigned v, unsigned site) {
  const u64 want = q_word(2u * lap, 0u);
  KOG2_SPIN(atomicCAS(slot, want, q_word(2u * lap + 1u, v)) != want, site, lap, v);
}
__device__ __forceinline__ unsigned q_take(u64* slot, unsigned lap, unsigned site) {
  volatile u64* vs = slot;
  u64 w;
  KOG2_SPIN(static_cast<unsigned>((w = *vs) >> 32) != 2u * lap + 1u, site, lap, 0u);
  *vs = q_word(2u * lap + 2u, 0u);
  return static_cast<unsigned>(w);
}
// launches the sample kept on this kernel (diagnostics: kog_svd2_lean_count)
__device__ unsigned long long g_kog2_lean_total = 0;
// Block shape: one block of 1024 threads per SM.  Thirty-two warps on one set of queues fill a batch twice as
// fast as sixteen (the queued matrices' sectors are younger in L2) and the SM holds one hot code set instead of
// two blocks' worth.  Measured (config 3, ms per 2^28): 256 x 4: 10.65, 512 x 2: 10.51, 1024 x 1: 10.04.
#ifndef KOG2_LEAN_THREADS
#define KOG2_LEAN_THREADS 1024
#endif
#ifndef KOG2_LEAN_MINB
#define KOG2_LEAN_MINB 1
#endif
#ifndef KOG2_LEAN_RINGT
#define KOG2_LEAN_RINGT 512
#endif
#ifndef KOG2_LEAN_CHUNK
#define KOG2_LEAN_CHUNK 8
#endif
constexpr unsigned kLeanWarps = KOG2_LEAN_THREADS / 32;
constexpr unsigned kRingT = KOG2_LEAN_RINGT;  // class T ring, a power of two (512 .. 2048 measured alike)
constexpr unsigned kRingS = 256;              // class S ring
constexpr unsigned kLeanChunk = KOG2_LEAN_CHUNK;  // consecutive tiles per grab (a power of two, even; 4 .. 16 measured alike)
constexpr unsigned kLeanStageBytes = kLeanWarps * 2 * 4 * 32 * sizeof(double);  // dynamic shared memory of k_svd2_lean
struct LeanGlobal {
  unsigned next_chunk;
  unsigned mode;  // 1: the batch goes to k_svd2_fast
};
struct LeanShared {
  u64 slotT[kRingT];
  u64 slotS[kRingS];
  unsigned tail[2];  // reserved positions (free-running): [0] class S, [1] class T
  unsigned done;     // warps out of tiles
};
// The staging buffers (dynamic shared memory: two tiles of 4 x 32 doubles per warp) are addressed as 32-bit
// shared-memory addresses recomputed from %tid on every tile: a pointer kept across the tile loop gets spilled
// around the class calls, and its reload queues behind the tile's cp.async copies (12% of all stall samples).
__device__ __forceinline__ unsigned lean_stage(const void* dyn, unsigned buf) {
  unsigned tid;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));  // (volatile: not hoisted out of the loop)
  return static_cast<unsigned>(__cvta_generic_to_shared(dyn)) + (tid >> 5) * 2048u + buf * 1024u + (tid & 31u) * 8u;
}
__device__ __forceinline__ void lean_fetch(unsigned st, const InP<double>& in, unsigned i, unsigned n32) {
  if (i < n32) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(st), "l"(in.g11 + i) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(st + 256u), "l"(in.g12 + i) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(st + 512u), "l"(in.g21 + i) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(st + 768u), "l"(in.g22 + i) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ double lds_f64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
// The class routes are out-of-line calls: inlined, their register demand pushed
// the tile loop's own state into local memory for the whole loop.  The batch
// pointers travel through shared memory (an ABI call would pass fourteen
// pointers in registers).
struct LeanParams {
  InP<double> in;
  OutP<double> out;
  uint32_t* list;
  unsigned* count;
};
template <int CLS>
__device__ __noinline__ void fast_call(const LeanParams* P, unsigned i, unsigned lane) {
  fast_one<double, CLS>(P->in, P->out, i, P->list, P->count, lane);
}
// run the queued indices [pos, pos + cnt) of a ring, cnt <= 32 (T: class T, else class S)
template <bool T>
__device__ __forceinline__ void lean_batch(LeanShared& S, unsigned pos, unsigned cnt, const LeanParams* P,
                                           unsigned lane) {
  constexpr unsigned ring = T ? kRingT : kRingS;
  u64* slots = T ? S.slotT : S.slotS;
  if (lane < cnt) {
    const unsigned p = pos + lane;
    const unsigned i = q_take(&slots[p & (ring - 1u)], p / ring, T ? 1u : 2u);
    __threadfence_block();
    fast_call<T ? 3 : 0>(P, i, lane);
  }
  __syncwarp();
}
__global__ void __launch_bounds__(KOG2_LEAN_THREADS, KOG2_LEAN_MINB)
    k_svd2_lean(InP<double> in, OutP<double> out, uint64_t n, uint32_t* list, unsigned* count, LeanGlobal* G) {
  __shared__ LeanShared S;
  __shared__ LeanParams SP;
  extern __shared__ __align__(16) unsigned char lean_dyn[];  // the input staging buffers (kLeanStageBytes)
  for (unsigned k = threadIdx.x; k < sizeof(LeanShared) / sizeof(unsigned); k += blockDim.x)
    reinterpret_cast<unsigned*>(&S)[k] = 0u;
  if (threadIdx.x == 0) SP = LeanParams{in, out, list, count};
  const unsigned lane = threadIdx.x & 31u;
  const unsigned n32 = static_cast<unsigned>(n);
  // the sample: every block reads the same KOG2_LEAN_THREADS matrices spread over the batch
  {
    const uint64_t si = (static_cast<uint64_t>(2u * threadIdx.x + 1u) * n) / (2u * KOG2_LEAN_THREADS);
    const Mat<double> g{in.g11[si], in.g12[si], in.g21[si], in.g22[si]};
    const int h11 = hiw(g.g11) & 0x7fffffff, h12 = hiw(g.g12) & 0x7fffffff, h21 = hiw(g.g21) & 0x7fffffff,
              h22 = hiw(g.g22) & 0x7fffffff;
    const int hmax = max(max(h11, h12), max(h21, h22)), hmin = min(min(h11, h12), min(h21, h22));
    const bool sep = hmin >= 0x00100000 && hmax < (2045 << 20) && abs(h11 - h21) >= (28 << 20) &&
                     abs(h12 - h22) >= (28 << 20);
    const int ns = __syncthreads_count(sep);  // (also the barrier behind the initialisation of S)
    // the later tests of svd2_lean fail a few percent more; under ~45% it would not pay
    if ((ns - ns / 16) * 20 < 9 * KOG2_LEAN_THREADS) {
      if (blockIdx.x == 0 && threadIdx.x == 0) G->mode = 1u;
      return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_kog2_lean_total, 1ull);
  }
  // Tiles are handed out eight consecutive tiles (a chunk) at a time from a global counter: warps that run
  // more batches take fewer chunks (static striding measured 6% slower).  The tile loop carries ONE word —
  // the tile base with `direct` (warp-uniform: stop trying svd2_lean) in bit 0; the tile's place in its chunk,
  // its staging buffer and the probe turns follow from the base (chunks start at multiples of 256 matrices),
  // and the next chunk is claimed when it is needed (the round trip, once per eight tiles, hides behind the
  // other warps): loop words that the compiler keeps in local memory around the class calls cost reloads on
  // every tile (one such reload, queued behind the tile's cp.async copies, was 12.6% of all stall samples).
  unsigned bd = 0;
  if (lane == 0) bd = atomicAdd(&G->next_chunk, 1u);
  bd = __shfl_sync(0xffffffffu, bd, 0) * (kLeanChunk * 32u);
  lean_fetch(lean_stage(lean_dyn, 0u), in, bd + lane, n32);
  while ((bd & ~31u) < n32) {
    const unsigned base = bd & ~31u;
    bool direct = (bd & 1u) != 0u;
    const unsigned tk = base >> 5;  // tile number: its low bits are the place in the chunk
    unsigned nbase = base + 32u;
    if ((tk & (kLeanChunk - 1u)) == kLeanChunk - 1u) {  // the chunk's last tile: claim the next chunk
      unsigned c = 0;
      if (lane == 0) c = atomicAdd(&G->next_chunk, 1u);
      nbase = __shfl_sync(0xffffffffu, c, 0) * (kLeanChunk * 32u);  // < 2^32: n <= 2^31, a few chunks per warp beyond
    }
    const unsigned stg = tk & 1u;  // staging buffers alternate (chunks hold an even number of tiles)
    const unsigned sg = lean_stage(lean_dyn, stg);  // this tile's buffer; the other one is 1 KB away
    if (nbase < n32) lean_fetch(sg + 1024u - 2048u * stg, in, nbase + lane, n32);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    const unsigned i = base + lane;
    const bool probe = (tk % KOG2_LEAN_PROBE) == 0;
    bool hard = i < n32;
    bool simple = false;
    if (hard) {
      const Mat<double> g{lds_f64(sg), lds_f64(sg + 256u), lds_f64(sg + 512u), lds_f64(sg + 768u)};
      simple = ((0x0357u >> type_of(g)) & 1u) != 0u;  // s_type = 0 patterns (classify.hpp:37-42)
      // (queued lanes store too: whole sectors at the first touch.  Two store sites rather than one behind a
      // merged Result: the merge cost twenty register moves per tile.)
      if (!direct || probe) {
        Result<double> r;
        hard = !fast::svd2_lean(g, r);
        store_result<false>(out, i, r);
      } else {
        Result<double> r;
        r.u = r.v = g;
        r.sigma1 = r.sigma2 = EPair<double>{0, 0.0};
        r.s = 0;
        r.flags = 0;
        store_result<false>(out, i, r);
      }
      asm volatile("fence.acq_rel.cta;" ::: "memory");  // before the push (lighter than __threadfence_block's fence.sc)
    }
    const unsigned mh = __ballot_sync(0xffffffffu, hard);
    if (probe) direct = __popc(mh) > 20;  // svd2_lean pays below ~2/3 of the lanes failing
    bd = nbase | (direct ? 1u : 0u);
    if (mh == 0u) continue;
    const unsigned ms = __ballot_sync(0xffffffffu, hard && simple);
    const unsigned mt = mh & ~ms;
    // lanes 0 and 1 reserve the positions of classes S and T; a reservation that crosses a multiple of 32
    // makes this warp run the 32 that end there
    unsigned at = 0, end = 0;
    if (lane < 2u) {
      const unsigned cnt = __popc(lane == 0u ? ms : mt);
      if (cnt != 0u) at = atomicAdd(&S.tail[lane], cnt);
      end = at + cnt;
    }
    const unsigned run = __ballot_sync(0xffffffffu, (end >> 5) != (at >> 5));
    const unsigned ps = (__shfl_sync(0xffffffffu, end, 0) & ~31u) - 32u;
    const unsigned pt = (__shfl_sync(0xffffffffu, end, 1) & ~31u) - 32u;
    at = __shfl_sync(0xffffffffu, at, simple ? 0 : 1);
    if (hard) {
      const unsigned at1 = at + __popc((simple ? ms : mt) & ((1u << lane) - 1u));
      // one wait loop for the two rings (each lane its own slot)
      u64* slot = simple ? &S.slotS[at1 & (kRingS - 1u)] : &S.slotT[at1 & (kRingT - 1u)];
      q_put(slot, simple ? at1 / kRingS : at1 / kRingT, i, 8u);
    }
    __syncwarp();
    if (run & 2u) lean_batch<true>(S, pt, 32u, &SP, lane);
    if (run & 1u) lean_batch<false>(S, ps, 32u, &SP, lane);
  }
  // out of tiles: the block's last warp runs the remainders of the two rings (< 32 each) as partial batches
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __threadfence_block();
  unsigned l = 0;
  if (lane == 0) l = atomicAdd(&S.done, 1u) == kLeanWarps - 1u;
  if (!__shfl_sync(0xffffffffu, l, 0)) return;
  __threadfence_block();
  const unsigned tt = ld_vol(&S.tail[1]), ts = ld_vol(&S.tail[0]);
  if (tt & 31u) lean_batch<true>(S, tt & ~31u, tt & 31u, &SP, lane);
  if (ts & 31u) lean_batch<false>(S, ts & ~31u, ts & 31u, &SP, lane);
}
// k_svd2_fast for a batch whose sample sent it back (LeanGlobal::mode)
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
// smaller batches: k_svd2_fast alone.  The two-speed kernel's start (sample, queue set-up) and end (partial
// batches) cost ~30 us: it ties at 2^21 config-3 matrices and is 14% ahead at 2^22 (profiles/r3_lean_sizes.txt),
// but the host pipeline's 2^22-matrix chunks ran 3% slower end to end on it (its extra stream operations per
// chunk; the pipeline is PCIe-bound either way), so the threshold sits above them.  kog_svd2_set_lean_min moves it.
static std::atomic<uint64_t> g_lean_min{1ull << 23};

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
      static const bool no_lean = std::getenv("KOG2_SVD2_NO_LEAN") != nullptr;  // A/B comparisons
      const uint64_t lean_min = g_lean_min.load(std::memory_order_relaxed);
      const bool use_lean = sizeof(T) == sizeof(double) && !no_lean && n >= lean_min;
      const size_t list_bytes = (cap * sizeof(uint32_t) + 255) & ~static_cast<size_t>(255);
      char* ws = static_cast<char*>(kog2_ws_alloc(256 + list_bytes + (use_lean ? sizeof(LeanGlobal) : 0), st));
      if (!ws) return KOG_ERR_CUDA;
      unsigned* count = reinterpret_cast<unsigned*>(ws);
      uint32_t* list = reinterpret_cast<uint32_t*>(ws + 256);
      LeanGlobal* lg = use_lean ? reinterpret_cast<LeanGlobal*>(ws + 256 + list_bytes) : nullptr;
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
        {
          const unsigned* gate = nullptr;
          if constexpr (sizeof(T) == sizeof(double)) {
            if (lg && len >= lean_min) {
              // resident blocks only (tiles are handed out dynamically); k_svd2_fast behind it runs only
              // if the kernel's sample sends the batch back
              if (cudaMemsetAsync(lg, 0, sizeof(LeanGlobal), st) != cudaSuccess) {
                rc = kog2_cuda_error("cudaMemsetAsync(lean queues)");
                break;
              }
              // (function attributes are per device: once per device, not once per process)
              static std::atomic<bool> attr_set[64];
              int dev = 0;
              cudaGetDevice(&dev);
              bool smem_ok = dev >= 0 && dev < 64 && attr_set[dev].load(std::memory_order_acquire);
              if (!smem_ok) {
                smem_ok = cudaFuncSetAttribute(k_svd2_lean, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(kLeanStageBytes)) == cudaSuccess;
                if (smem_ok && dev >= 0 && dev < 64) attr_set[dev].store(true, std::memory_order_release);
              }
              if (!smem_ok) {
                rc = kog2_cuda_error("cudaFuncSetAttribute(k_svd2_lean)");
                break;
              }
              k_svd2_lean<<<sms * KOG2_LEAN_MINB, KOG2_LEAN_THREADS, kLeanStageBytes, st>>>(ip, ol, len, list, count, lg);
              if ((rc = launched("k_svd2_lean")) != KOG_OK) break;
              gate = &lg->mode;
            }
          }
          k_svd2_fast<T><<<grid_for(len, FastShape<T>::threads), FastShape<T>::threads, 0, st>>>(ip, ol, len, list,
                                                                                           count, gate);
        }
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

#ifdef KOG2_LEAN_DEBUG
int kog2_lean_debug_host(unsigned* pinned) {
  return cudaMemcpyToSymbol(g_lean_host, &pinned, sizeof(pinned)) == cudaSuccess ? 0 : -1;
}
int kog2_lean_debug(unsigned* out) {
  return cudaMemcpyFromSymbol(out, g_lean_dbg, sizeof(g_lean_dbg)) == cudaSuccess ? 0 : -1;
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

uint64_t kog_svd2_set_lean_min(uint64_t n) {
  return g_lean_min.exchange(n < (1ull << 16) ? (1ull << 16) : n, std::memory_order_relaxed);
}

int64_t kog_svd2_lean_count(void) {
  unsigned long long c = 0;
  if (cudaMemcpyFromSymbol(&c, g_kog2_lean_total, sizeof c) != cudaSuccess) {
    kog2_cuda_error("cudaMemcpyFromSymbol(lean total)");
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
