// launch.cu -- cached launch configuration for the persistent kernels: the
// dynamic shared-memory attribute is raised once per (kernel, size) and the
// occupancy / SM count are queried once, so an alb_apply costs only the
// kernel launches themselves on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <set>
#include <utility>

namespace alb {

namespace {
std::mutex g_mu;
std::map<std::pair<const void*, size_t>, int> g_occ;
std::set<const void*> g_fn_set;
int g_sms = 0;
}  // namespace

int persistent_grid(const void* fn, int threads, size_t smem, int n_units) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      g_sms = 148;
  }
  const auto key = std::make_pair(fn, smem);
  auto it = g_occ.find(key);
  int occ;
  if (it == g_occ.end()) {
    // the attribute is per function: raise it to the opt-in maximum once, so
    // launches of the same kernel with different smem sizes all stay legal
    if (g_fn_set.insert(fn).second) {
      int dev = 0, mx = 0;
      cudaGetDevice(&dev);
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
  return std::min(n_units, g_sms * occ);
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
// created on first use per (host thread, device), destroyed at thread exit
SideStream& side_stream() {
  thread_local SideStream t[64];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& r = t[dev & 63];
  if (!r.s) {
    cudaStreamCreateWithFlags(&r.s, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming);
  }
  return r;
}
}  // namespace

cudaStream_t side_fork(cudaStream_t s) {
  SideStream& r = side_stream();
  cudaEventRecord(r.fork, s);
  cudaStreamWaitEvent(r.s, r.fork, 0);
  return r.s;
}

void side_join(cudaStream_t s) {
  SideStream& r = side_stream();
  cudaEventRecord(r.join, r.s);
  cudaStreamWaitEvent(s, r.join, 0);
}

}  // namespace alb
