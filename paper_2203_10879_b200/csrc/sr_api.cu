// C-ABI housekeeping: version, last-error string.
#include <stdio.h>
#include <string.h>

#include <atomic>

#include "sr_common.cuh"

static thread_local char g_last_error[512] = "";

int sr_set_cuda_error(cudaError_t e, const char* what) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, cudaGetErrorString(e));
  return SR_ECUDA;
}

static std::atomic<unsigned long long> g_launches{0};

void sr_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void sr_count_launches(unsigned long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

extern "C" unsigned long long sr_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int sr_version(void) { return 1; }

extern "C" const char* sr_last_error(void) { return g_last_error; }
