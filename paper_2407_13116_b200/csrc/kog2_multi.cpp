// kog2_multi.cpp — the multi-GPU study on the C++ host side:
// contiguous index shards, one study per device, and ONE NCCL all-reduce of
// a small packed statistics vector; the host merges the per-rank blocks in
// rank order (ErrorStats::merge, harness.hpp:96-105), so the result is
// bit-identical to kog_run_batch for any number of devices.
//
// Slot layout (int64, MAX all-reduce both reduces and gathers):
//   0..4  bit patterns of reG, reS1, reS2, reU, reV (non-negative doubles, so
//         integer order is value order; oracle.hpp:251-263 never makes -0)
//   5     kappa_inf (MAX = OR)
//   6     2^62 - fail_key, or -1 without a failure (MAX = the lowest key)
//   then one block of 23 fields per rank — kappa e, hi, lo, first index and the
//   19 branch counters — each 64-bit field as two non-negative 32-bit halves;
//   a rank writes only its own block, zeros elsewhere.
//
// NCCL is loaded on first use with dlopen("libnccl.so.2") (the system library,
// or the one a host process such as PyTorch already loaded), so libkog2.so
// itself has no NCCL dependency and single-GPU users never load it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "kog2_internal.h"

namespace {

constexpr int kHead = 7;
constexpr int kPerRank = 4 + 19;
constexpr int64_t kNoFail = -1;
constexpr uint64_t kFailBase = 1ull << 62;

uint64_t u64_of(double x) {
  uint64_t u;
  std::memcpy(&u, &x, sizeof u);
  return u;
}
double f64_of(uint64_t u) {
  double x;
  std::memcpy(&x, &u, sizeof x);
  return x;
}

void rank_fields(const kog_stats& st, uint64_t f[kPerRank]) {
  f[0] = static_cast<uint64_t>(st.max_kappa2.e);
  f[1] = u64_of(st.max_kappa2.hi);
  f[2] = u64_of(st.max_kappa2.lo);
  f[3] = st.max_kappa2_index;
  for (int k = 0; k < 7; ++k) {
    f[4 + k] = st.t2p[k];
    f[11 + k] = st.path[k];
  }
  f[18] = st.tanpsi_inf;
  f[19] = st.diag_swap;
  f[20] = st.compose_minus;
  f[21] = st.sigma_swap;
  f[22] = st.prescale_inexact;
}

// ------------------------------------------------------------ NCCL loader
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return;
    }
    bool ok = true;
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      ok = ok && fp != nullptr;
    };
    sym(n.GetUniqueId, "ncclGetUniqueId");
    sym(n.CommInitRank, "ncclCommInitRank");
    sym(n.CommInitAll, "ncclCommInitAll");
    sym(n.CommDestroy, "ncclCommDestroy");
    sym(n.AllReduce, "ncclAllReduce");
    sym(n.GetErrorString, "ncclGetErrorString");
    n.ok = ok;
    if (!ok) n.why = "libnccl lacks a required symbol";
  });
  return n;
}

int nccl_error(const char* what, ncclResult_t r) {
  const Nccl& n = nccl();
  kog2_set_error((std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "nccl error")).c_str());
  return KOG_ERR_CUDA;
}

int need_nccl() {
  const Nccl& n = nccl();
  if (n.ok) return KOG_OK;
  kog2_set_error(n.why.c_str());
  return KOG_ERR_NODEV;
}

// pack -> device -> ncclAllReduce(MAX, in place) -> host -> unpack, on `st`
int allreduce_slots(ncclComm_t comm, int rank, int world, kog_stats* stats, cudaStream_t st) {
  const size_t ns = kog_stats_slot_count(world);
  std::vector<int64_t> host(ns);
  int rc = kog_stats_pack(stats, rank, world, host.data());
  if (rc != KOG_OK) return rc;
  int64_t* dev = static_cast<int64_t*>(kog2_ws_alloc(ns * sizeof(int64_t), st));
  if (!dev) return KOG_ERR_CUDA;
  if (cudaMemcpyAsync(dev, host.data(), ns * sizeof(int64_t), cudaMemcpyHostToDevice, st) != cudaSuccess)
    rc = kog2_cuda_error("cudaMemcpyAsync(stats slots)");
  if (rc == KOG_OK) {
    const ncclResult_t r = nccl().AllReduce(dev, dev, ns, ncclInt64, ncclMax, comm, st);
    if (r != ncclSuccess) rc = nccl_error("ncclAllReduce", r);
  }
  if (rc == KOG_OK &&
      cudaMemcpyAsync(host.data(), dev, ns * sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = kog2_cuda_error("cudaMemcpyAsync(stats slots)");
  kog2_ws_free(dev, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && rc == KOG_OK) rc = kog2_cuda_error("cudaStreamSynchronize");
  if (rc != KOG_OK) return rc;
  return kog_stats_unpack(host.data(), world, stats);
}

}  // namespace

extern "C" {

size_t kog_stats_slot_count(int world) {
  return world > 0 ? static_cast<size_t>(kHead + 2 * kPerRank * world) : 0;
}

int kog_stats_pack(const kog_stats* st, int rank, int world, int64_t* slots) {
  if (!st || !slots || world < 1 || rank < 0 || rank >= world) return kog2_arg_error("kog_stats_pack: bad argument");
  std::memset(slots, 0, kog_stats_slot_count(world) * sizeof(int64_t));
  const double m[5] = {st->reG, st->reS1, st->reS2, st->reU, st->reV};
  for (int k = 0; k < 5; ++k) slots[k] = static_cast<int64_t>(u64_of(m[k]));
  slots[5] = st->kappa_inf ? 1 : 0;
  slots[6] = st->fail_key == UINT64_MAX ? kNoFail : static_cast<int64_t>(kFailBase - st->fail_key);
  uint64_t f[kPerRank];
  rank_fields(*st, f);
  int64_t* b = slots + kHead + 2 * kPerRank * rank;
  for (int k = 0; k < kPerRank; ++k) {
    b[2 * k] = static_cast<int64_t>(f[k] >> 32);
    b[2 * k + 1] = static_cast<int64_t>(f[k] & 0xffffffffu);
  }
  return KOG_OK;
}

int kog_stats_unpack(const int64_t* slots, int world, kog_stats* out) {
  if (!slots || !out || world < 1) return kog2_arg_error("kog_stats_unpack: bad argument");
  kog_stats total;
  kog_stats_init(&total);
  for (int r = 0; r < world; ++r) {
    const int64_t* b = slots + kHead + 2 * kPerRank * r;
    uint64_t v[kPerRank];
    for (int k = 0; k < kPerRank; ++k)
      v[k] = (static_cast<uint64_t>(b[2 * k]) << 32) | static_cast<uint64_t>(b[2 * k + 1] & 0xffffffff);
    kog_stats part;
    kog_stats_init(&part);
    part.max_kappa2.e = static_cast<int64_t>(v[0]);
    part.max_kappa2.hi = f64_of(v[1]);
    part.max_kappa2.lo = f64_of(v[2]);
    part.max_kappa2_index = v[3];
    for (int k = 0; k < 7; ++k) {
      part.t2p[k] = v[4 + k];
      part.path[k] = v[11 + k];
    }
    part.tanpsi_inf = v[18];
    part.diag_swap = v[19];
    part.compose_minus = v[20];
    part.sigma_swap = v[21];
    part.prescale_inexact = v[22];
    kog_stats_merge(&total, &part);  // rank order = index order
  }
  total.reG = f64_of(static_cast<uint64_t>(slots[0]));
  total.reS1 = f64_of(static_cast<uint64_t>(slots[1]));
  total.reS2 = f64_of(static_cast<uint64_t>(slots[2]));
  total.reU = f64_of(static_cast<uint64_t>(slots[3]));
  total.reV = f64_of(static_cast<uint64_t>(slots[4]));
  total.kappa_inf = slots[5] != 0 ? 1 : 0;
  total.fail_key = slots[6] == kNoFail ? UINT64_MAX : kFailBase - static_cast<uint64_t>(slots[6]);
  *out = total;
  return KOG_OK;
}

void kog_study_shard(uint64_t count, int rank, int world, uint64_t* lo, uint64_t* hi) {
  const uint64_t per = world > 0 ? count / static_cast<uint64_t>(world) : count;
  const uint64_t l = static_cast<uint64_t>(rank) * per;
  if (lo) *lo = l;
  if (hi) *hi = rank == world - 1 ? count : l + per;
}

int kog_nccl_available(void) { return nccl().ok ? 1 : 0; }

int kog_nccl_unique_id(uint8_t* id, size_t cap) {
  if (!id || cap < sizeof(ncclUniqueId)) return kog2_arg_error("kog_nccl_unique_id: buffer too small");
  int rc = need_nccl();
  if (rc != KOG_OK) return rc;
  ncclUniqueId u;
  const ncclResult_t r = nccl().GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_error("ncclGetUniqueId", r);
  std::memcpy(id, &u, sizeof u);
  return KOG_OK;
}

int kog_nccl_comm_init(const uint8_t* id, int world, int rank, void** comm) {
  if (!id || !comm || world < 1 || rank < 0 || rank >= world) return kog2_arg_error("kog_nccl_comm_init: bad argument");
  int rc = need_nccl();
  if (rc != KOG_OK) return rc;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().CommInitRank(&c, world, u, rank);
  if (r != ncclSuccess) return nccl_error("ncclCommInitRank", r);
  *comm = c;
  return KOG_OK;
}

int kog_nccl_comm_destroy(void* comm) {
  if (!comm) return KOG_OK;
  int rc = need_nccl();
  if (rc != KOG_OK) return rc;
  const ncclResult_t r = nccl().CommDestroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? KOG_OK : nccl_error("ncclCommDestroy", r);
}

int kog_study_allreduce(void* comm, int rank, int world, kog_stats* stats, void* stream) {
  if (!comm || !stats) return kog2_arg_error("kog_study_allreduce: null argument");
  int rc = need_nccl();
  if (rc != KOG_OK) return rc;
  return allreduce_slots(static_cast<ncclComm_t>(comm), rank, world, stats, static_cast<cudaStream_t>(stream));
}

int kog_study_multi(const kog_run_config* cfg, const int* devices, int ndev, kog_stats* out, double* device_seconds) {
  if (!cfg || !out || ndev < 1) return kog2_arg_error("kog_study_multi: bad argument");
  int rc = kog_validate(cfg);
  if (rc != KOG_OK) return rc;
  if ((rc = need_nccl()) != KOG_OK) return rc;
  std::vector<int> devs(ndev);
  for (int k = 0; k < ndev; ++k) devs[k] = devices ? devices[k] : k;
  std::vector<ncclComm_t> comms(ndev);
  const ncclResult_t r = nccl().CommInitAll(comms.data(), ndev, devs.data());
  if (r != ncclSuccess) return nccl_error("ncclCommInitAll", r);
  std::vector<int> rcs(ndev, KOG_OK);
  std::vector<std::string> errs(ndev);
  std::vector<kog_stats> res(ndev);
  std::vector<double> secs(ndev, 0.0);
  // one host thread per device (the reference's worker pool, harness.hpp:241-263,
  // with devices for workers and contiguous shards for blocks)
  auto worker = [&](int k) {
    int& wrc = rcs[k];
    if (cudaSetDevice(devs[k]) != cudaSuccess) {
      wrc = kog2_cuda_error("cudaSetDevice");
      errs[k] = kog_last_error();
      return;
    }
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    kog_stats* dstats = nullptr;
    uint64_t lo = 0, hi = 0;
    kog_study_shard(cfg->count, k, ndev, &lo, &hi);
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
      wrc = kog2_cuda_error("stream/event create");
    if (wrc == KOG_OK) wrc = kog_study_stats_alloc(&dstats);
    if (wrc == KOG_OK && cudaEventRecord(e0, st) != cudaSuccess) wrc = kog2_cuda_error("cudaEventRecord");
    constexpr uint64_t kLaunch = 1ull << 27;  // bounded kernel duration, as kog_run_batch
    for (uint64_t a = lo; wrc == KOG_OK && a < hi; a += kLaunch)
      wrc = kog_study_batch(cfg, a, hi - a < kLaunch ? hi - a : kLaunch, dstats, st);
    kog_stats& mine = res[k];
    if (wrc == KOG_OK && cudaMemcpyAsync(&mine, dstats, sizeof mine, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      wrc = kog2_cuda_error("cudaMemcpyAsync(kog_stats)");
    if (wrc == KOG_OK && cudaStreamSynchronize(st) != cudaSuccess) wrc = kog2_cuda_error("cudaStreamSynchronize");
    // every rank takes part in the collective even after a local error
    // (with empty stats), so no peer waits forever
    if (wrc != KOG_OK) kog_stats_init(&mine);
    const int arc = allreduce_slots(comms[k], k, ndev, &mine, st);
    if (wrc == KOG_OK) wrc = arc;
    if (wrc == KOG_OK && (cudaEventRecord(e1, st) != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess))
      wrc = kog2_cuda_error("cudaEventRecord");
    float ms = 0.0f;
    if (wrc == KOG_OK && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess) secs[k] = ms * 1e-3;
    if (wrc != KOG_OK) errs[k] = kog_last_error();
    if (dstats) kog_study_stats_free(dstats);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (st) cudaStreamDestroy(st);
  };
  std::vector<std::thread> pool;
  for (int k = 0; k < ndev; ++k) pool.emplace_back(worker, k);
  for (auto& t : pool) t.join();
  for (auto c : comms) nccl().CommDestroy(c);
  for (int k = 0; k < ndev; ++k)
    if (rcs[k] != KOG_OK) {
      kog2_set_error(errs[k].c_str());
      return rcs[k];
    }
  *out = res[0];  // identical on every rank after the all-reduce
  if (device_seconds) {
    double m = 0.0;
    for (double s : secs) m = s > m ? s : m;  // max over ranks
    *device_seconds = m;
  }
  if (out->fail_key != UINT64_MAX) {
    char buf[512];
    if (kog_abort_message(cfg, out->fail_key, buf, sizeof buf) < 0) return KOG_ERR_CUDA;
    kog2_set_error(buf);
    return KOG_ERR_ABORT;
  }
  return KOG_OK;
}

}  // extern "C"
