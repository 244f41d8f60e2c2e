// kog2_common.cuh — launch helpers and batch-pointer structs shared by the
// kernel translation units (kog2_k_*.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "kog2_internal.h"
#include "kog2_svd2.cuh"

namespace kog2 {

constexpr int kThreads = 256;

// grid for an elementwise launch over n items (grid-stride loops inside)
inline int grid_for(uint64_t n, int threads = kThreads) {
  uint64_t blocks = (n + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(kog2_sm_count()) * 64ull;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  return static_cast<int>(blocks);
}

// count the launch and turn a launch error into a KOG_ERR_CUDA + message
inline int launched(const char* what) {
  kog2_count_launch();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
    kog2_set_error(buf);
    return KOG_ERR_CUDA;
  }
  return KOG_OK;
}

__device__ __forceinline__ uint64_t gtid() {
  return static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
}
__device__ __forceinline__ uint64_t gstride() {
  return static_cast<uint64_t>(gridDim.x) * blockDim.x;
}

// streaming (evict-first) loads/stores for once-touched batch data
__device__ __forceinline__ double ld_cs(const double* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_cs(const float* p) { return __ldcs(p); }
template <class V>
__device__ __forceinline__ void st_cs(V* p, V v) {
  __stcs(p, v);
}

template <class T>
struct InP {
  const T *g11, *g12, *g21, *g22;
};

template <class T, class MatC>
inline bool mat_ok(const MatC* m) {
  return m && m->g11 && m->g12 && m->g21 && m->g22;
}
template <class T, class MatC>
inline InP<T> in_of(const MatC* m) {
  return InP<T>{m->g11, m->g12, m->g21, m->g22};
}

template <class T>
__device__ __forceinline__ Mat<T> load_mat(const InP<T>& in, uint64_t i) {
  return Mat<T>{in.g11[i], in.g12[i], in.g21[i], in.g22[i]};
}

inline Opt opt_of(const kog_options* o) {
  const kog_options d = o ? *o : kog2_default_options();
  return Opt{d.hypot_is_cr != 0, d.ominus_for_d != 0, d.wide_channel ? KOG_WIDE_KAHAN_DET : KOG_WIDE_WIDER_TYPE};
}
inline bool opt_is_default(const Opt& o) { return o.hcr && !o.omd && o.wc == KOG_WIDE_WIDER_TYPE; }
__device__ __forceinline__ Opt opt_default() { return Opt{true, false, KOG_WIDE_WIDER_TYPE}; }

}  // namespace kog2

#define KOG2_ST(s) static_cast<cudaStream_t>(s)
