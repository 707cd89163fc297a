// C-ABI plumbing: thread-local error messages, launch accounting, version.
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

namespace smb {
namespace {
thread_local char g_err[512] = {0};
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void clear_error() { g_err[0] = 0; }

void count_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void ensure_dynamic_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, size_t>> done;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : done)
    if (e.first == kernel && e.second >= bytes) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  done.emplace_back(kernel, bytes);
}

int check_launch(const char* what, uint64_t launches) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: CUDA error: %s", what, cudaGetErrorString(e));
    return SMB_ERR_CUDA;
  }
  count_launches(launches);
  return SMB_OK;
}

}  // namespace smb

extern "C" int smb_abi_version(void) { return SMB_ABI_VERSION; }
extern "C" const char* smb_last_error(void) { return smb::g_err; }
extern "C" uint64_t smb_launch_count(void) {
  return smb::g_launches.load(std::memory_order_relaxed);
}
