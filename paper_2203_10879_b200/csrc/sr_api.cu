// C-ABI housekeeping: version, last-error string.
#include <stdio.h>
#include <string.h>

#include "sr_common.cuh"

static thread_local char g_last_error[512] = "";

int sr_set_cuda_error(cudaError_t e, const char* what) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, cudaGetErrorString(e));
  return SR_ECUDA;
}

extern "C" int sr_version(void) { return 1; }

extern "C" const char* sr_last_error(void) { return g_last_error; }
