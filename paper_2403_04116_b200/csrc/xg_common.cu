// Error bookkeeping and version query of libxgauss.
#include <stdio.h>

#include <atomic>

#include "xg_internal.cuh"

namespace xg {

static thread_local char g_last_error[512] = "";

void set_error(const char* what, cudaError_t err) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, cudaGetErrorString(err));
}

void set_error_msg(const char* what) { snprintf(g_last_error, sizeof(g_last_error), "%s", what); }

static std::atomic<unsigned long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace xg

extern "C" {

int32_t xg_abi_version(void) { return XG_ABI_VERSION; }

const char* xg_last_error(void) { return xg::g_last_error; }

uint64_t xg_kernel_launches(void) { return xg::g_launches.load(); }

size_t xg_densify_scratch_bytes(int64_t n) {
  return sizeof(uint32_t) * (size_t)(6 * n + 4) + 256 + ((size_t)((n + 2047) / 2048 + 1) * 8 + 512);
}

}  // extern "C"
