// launch.cu -- cached launch configuration for the persistent kernels: the
// dynamic shared-memory attribute is raised once per (kernel, size) and the
// occupancy / SM count are queried once, so an alb_apply costs only the
// kernel launches themselves on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <utility>

namespace alb {

namespace {
std::mutex g_mu;
// keyed by device: the dynamic shared-memory attribute and the occupancy are
// per (device context, function), the SM count per device
std::map<std::tuple<int, const void*, size_t>, int> g_occ;
std::set<std::pair<int, const void*>> g_fn_set;
std::map<int, int> g_sms;
}  // namespace

int persistent_grid(const void* fn, int threads, size_t smem, int n_units) {
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  int& sms = g_sms[dev];
  if (sms == 0 && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    sms = 148;
  const auto key = std::make_tuple(dev, fn, smem);
  auto it = g_occ.find(key);
  int occ;
  if (it == g_occ.end()) {
    // the attribute is per function and device: raise it to the opt-in
    // maximum once, so launches of the same kernel with different smem sizes
    // all stay legal
    if (g_fn_set.insert(std::make_pair(dev, fn)).second) {
      int mx = 0;
      cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, fn);
      const int lim = (mx > 0 ? mx : (int)smem) - (int)fa.sharedSizeBytes;
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, lim) != cudaSuccess)
        cudaGetLastError();  // not sticky: the launch reports any real problem
    }
    occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
    occ = std::max(occ, 1);
    g_occ[key] = occ;
  } else {
    occ = it->second;
  }
  return std::min(n_units, sms * occ);
}

namespace {
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  ~SideStream() {  // at host-thread exit (errors during process teardown are ignored)
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (s) cudaStreamDestroy(s);
  }
};
// kSidePool per (host thread, device), destroyed at thread exit; a caller
// stream always forks to the same pool entry (hash of the stream handle), so
// applies on one stream keep their order while applies on different caller
// streams (two batches in flight) mostly get independent side streams.
// Created by side_init() -- alb_plan_create calls it for plans with label /
// box work, so alb_apply on the plan's thread creates nothing -- or on first
// use from another thread.  If creation fails the side stream is the caller's
// stream itself: label / box work then runs in order on it (correct, not
// overlapped).
constexpr int kSidePool = 4;

SideStream& side_entry(int idx) {
  thread_local SideStream t[64][kSidePool];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  SideStream& r = t[dev & 63][idx];
  if (!r.s) {
    cudaStream_t s = nullptr;
    cudaEvent_t f = nullptr, j = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
        cudaEventCreateWithFlags(&f, cudaEventDisableTiming) == cudaSuccess &&
        cudaEventCreateWithFlags(&j, cudaEventDisableTiming) == cudaSuccess) {
      r.s = s; r.fork = f; r.join = j;
    } else {
      if (f) cudaEventDestroy(f);
      if (s) cudaStreamDestroy(s);
      cudaGetLastError();  // reported as "no side stream" below, not as a launch error
    }
  }
  return r;
}

SideStream& side_stream(cudaStream_t caller) {
  const uintptr_t h = (uintptr_t)caller;
  return side_entry((int)(((h >> 4) ^ (h >> 12)) % kSidePool));
}
}  // namespace

bool side_init() {
  bool ok = true;
  for (int i = 0; i < kSidePool; ++i) ok = side_entry(i).s != nullptr && ok;
  return ok;
}

cudaStream_t side_fork(cudaStream_t s) {
  SideStream& r = side_stream(s);
  if (!r.s) return s;
  cudaEventRecord(r.fork, s);  // failures surface through cudaGetLastError at the end of the apply
  cudaStreamWaitEvent(r.s, r.fork, 0);
  return r.s;
}

void side_join(cudaStream_t s) {
  SideStream& r = side_stream(s);
  if (!r.s || r.s == s) return;
  cudaEventRecord(r.join, r.s);
  cudaStreamWaitEvent(s, r.join, 0);
}

}  // namespace alb
