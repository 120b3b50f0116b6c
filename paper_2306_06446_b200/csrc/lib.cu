// Library-level entry points: version, thread-local error text, device info,
// launch accounting.
#include <atomic>
#include <stdarg.h>

#include "common.cuh"

namespace sa {

static thread_local char g_err[1024] = "";
std::atomic<uint64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int n) { g_launches.fetch_add(uint64_t(n), std::memory_order_relaxed); }

}  // namespace sa

extern "C" {

const char* sa_version(void) { return "shiftadd_b200 0.1.0 (sm_100a)"; }

const char* sa_last_error(void) { return sa::g_err; }

uint64_t sa_launch_count(void) { return sa::g_launches.load(); }

int sa_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    sa::set_error("cudaGetDevice: %s", cudaGetErrorString(e));
    return SA_ERR_CUDA;
  }
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) {
    sa::set_error("cudaGetDeviceProperties: %s", cudaGetErrorString(e));
    return SA_ERR_CUDA;
  }
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return SA_OK;
}

}  // extern "C"
