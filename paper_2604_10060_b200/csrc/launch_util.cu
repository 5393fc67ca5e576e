// launch_util.cu -- per-device launch state (dynamic shared-memory opt-ins, SM counts, occupancy).
//
// Kernel attributes are per (function, device): one process may drive contexts on several GPUs
// and contexts with different page sizes, so nothing here is cached once per process. A small
// table keyed by (kernel, device[, block, smem]) records what was set / measured; a later request
// for more shared memory raises the attribute again.
#include <map>
#include <mutex>
#include <tuple>

#include "kvc_core.hpp"

namespace kvc {

namespace {
std::mutex g_mu;
std::map<std::pair<const void*, int>, size_t> g_optin;                       // (fn, dev) -> bytes set
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;              // -> blocks per SM
std::map<int, std::pair<int, int>> g_dev;                                    // dev -> (sms, optin)
}  // namespace

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

static std::pair<int, int> dev_props(int dev) {
  auto it = g_dev.find(dev);
  if (it != g_dev.end()) return it->second;
  int sms = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return g_dev[dev] = {sms, optin};
}

int device_sms() {
  std::lock_guard<std::mutex> g(g_mu);
  return dev_props(current_device()).first;
}

int device_smem_optin() {
  std::lock_guard<std::mutex> g(g_mu);
  return dev_props(current_device()).second;
}

bool smem_optin(const void* fn, size_t bytes) {
  std::lock_guard<std::mutex> g(g_mu);
  const int dev = current_device();
  auto it = g_optin.find({fn, dev});
  if (it != g_optin.end() && bytes <= it->second) return true;
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) {
    cudaGetLastError();  // never leave a sticky error behind for an unrelated launch check
    return false;
  }
  // dynamic + static shared memory must fit the per-block opt-in limit
  if (bytes + fa.sharedSizeBytes > static_cast<size_t>(dev_props(dev).second)) return false;
  if (bytes > static_cast<size_t>(fa.maxDynamicSharedSizeBytes)) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
  }
  g_optin[{fn, dev}] = bytes;
  return true;
}

int occupancy(const void* fn, int threads, size_t smem) {
  std::lock_guard<std::mutex> g(g_mu);
  const auto key = std::make_tuple(fn, current_device(), threads, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  per_sm = per_sm < 1 ? 1 : per_sm;
  g_occ[key] = per_sm;
  return per_sm;
}

int auto_page_tokens(int d, bool bf16) {
  int p = 64;
  while (p > 8 && attend_smem_bytes(d, p, bf16) > static_cast<size_t>(device_smem_optin())) p /= 2;
  return p;
}

}  // namespace kvc
