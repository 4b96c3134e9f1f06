// Library-level C ABI: version, error strings, device facts.
#include <stdio.h>
#include <string.h>

#include "sdb_common.cuh"

namespace sdb {

static thread_local char g_last_cuda_error[256] = "";

int record_cuda_error(cudaError_t e) {
  snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "%s: %s", cudaGetErrorName(e),
           cudaGetErrorString(e));
  return SDB_E_CUDA;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

}  // namespace sdb

extern "C" {

int sdb_version(void) { return 100; }

const char *sdb_strerror(int code) {
  switch (code) {
    case SDB_OK: return "ok";
    case SDB_E_INVALID: return "invalid argument (shape, pointer or size)";
    case SDB_E_UNSUPPORTED: return "unsupported dtype or head_dim for this kernel";
    case SDB_E_WORKSPACE: return "workspace too small";
    case SDB_E_CUDA: return "CUDA launch failed";
    default: return "unknown error";
  }
}

const char *sdb_last_cuda_error(void) { return sdb::g_last_cuda_error; }

}  // extern "C"
