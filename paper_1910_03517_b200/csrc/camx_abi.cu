// Library-level entry points of the camx C ABI.
#include "camx_common.cuh"

extern "C" int camx_abi_version(void) { return CAMX_ABI_VERSION; }

namespace camx {
const char *nccl_error_string(int r);  // camx_comm.cu
}
using camx::nccl_error_string;

extern "C" const char *camx_status_string(int status) {
  switch (status) {
    case CAMX_OK:
      return "ok";
    case CAMX_EINVAL:
      return "invalid argument";
    case CAMX_EALIGN:
      return "pointer alignment not met";
    case CAMX_ENOMEM:
      return "out of memory";
    default:
      break;
  }
  if (status == CAMX_ENONCCL) return "NCCL library (libnccl.so.2) not loadable";
  if (status > CAMX_ENCCL_BASE && status < CAMX_ENONCCL)
    return nccl_error_string(status - CAMX_ENCCL_BASE);
  if (status > 0) return cudaGetErrorString(static_cast<cudaError_t>(status));
  return "unknown camx status";
}

extern "C" int camx_device_sm_count(int32_t *sm_count_out) {
  if (sm_count_out == nullptr) return CAMX_EINVAL;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  int n = 0;
  e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  *sm_count_out = n;
  return CAMX_OK;
}
