// kog2_ws.cpp — per-call, stream-ordered device workspace and side-stream
// sets (declarations and rationale in kog2_internal.h).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <vector>

#include "kog2_internal.h"

namespace {

constexpr int kMaxDev = 64;
std::mutex g_ws_mu;
cudaMemPool_t g_pool[kMaxDev] = {};
std::vector<Kog2SideStreams*> g_side_free[kMaxDev];

int pool_for(int dev, cudaMemPool_t& pool) {
  std::lock_guard<std::mutex> lock(g_ws_mu);
  if (g_pool[dev]) {
    pool = g_pool[dev];
    return KOG_OK;
  }
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t p = nullptr;
  if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return kog2_cuda_error("cudaMemPoolCreate(workspace)");
  uint64_t keep = UINT64_MAX;  // never trim at synchronisation points
  if (cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep) != cudaSuccess)
    return kog2_cuda_error("cudaMemPoolSetAttribute(workspace)");
  g_pool[dev] = pool = p;
  return KOG_OK;
}

int current_device(int& dev) {
  if (cudaGetDevice(&dev) != cudaSuccess) return kog2_cuda_error("cudaGetDevice");
  if (dev < 0 || dev >= kMaxDev) return kog2_arg_error("device index out of range");
  return KOG_OK;
}

}  // namespace

void* kog2_ws_alloc(size_t bytes, void* stream) {
  int dev = 0;
  cudaMemPool_t pool = nullptr;
  if (current_device(dev) != KOG_OK || pool_for(dev, pool) != KOG_OK) return nullptr;
  void* p = nullptr;
  if (cudaMallocFromPoolAsync(&p, bytes ? bytes : 1, pool, static_cast<cudaStream_t>(stream)) != cudaSuccess) {
    kog2_cuda_error("cudaMallocFromPoolAsync(workspace)");
    return nullptr;
  }
  return p;
}

int kog2_ws_free(void* p, void* stream) {
  if (!p) return KOG_OK;
  if (cudaFreeAsync(p, static_cast<cudaStream_t>(stream)) != cudaSuccess) return kog2_cuda_error("cudaFreeAsync");
  return KOG_OK;
}

Kog2SideStreams* kog2_side_acquire(void) {
  int dev = 0;
  if (current_device(dev) != KOG_OK) return nullptr;
  {
    std::lock_guard<std::mutex> lock(g_ws_mu);
    if (!g_side_free[dev].empty()) {
      Kog2SideStreams* s = g_side_free[dev].back();
      g_side_free[dev].pop_back();
      return s;
    }
  }
  auto* s = new Kog2SideStreams{};
  s->dev = dev;
  bool ok = true;
  for (auto& q : s->st) {
    cudaStream_t t = nullptr;
    ok = ok && cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking) == cudaSuccess;
    q = t;
  }
  for (auto& e : s->ev) {
    cudaEvent_t t = nullptr;
    ok = ok && cudaEventCreateWithFlags(&t, cudaEventDisableTiming) == cudaSuccess;
    e = t;
  }
  if (!ok) {
    kog2_cuda_error("side streams/events");
    for (auto q : s->st)
      if (q) cudaStreamDestroy(static_cast<cudaStream_t>(q));
    for (auto e : s->ev)
      if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
    delete s;
    return nullptr;
  }
  return s;
}

void kog2_side_release(Kog2SideStreams* s) {
  if (!s) return;
  std::lock_guard<std::mutex> lock(g_ws_mu);
  g_side_free[s->dev].push_back(s);
}

int kog2_sm_count(void) {
  static std::atomic<int> cache[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 148;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) return 148;
  cache[dev].store(v, std::memory_order_relaxed);
  return v;
}
