// CUDA IPC helpers so one-process-per-GPU ranks can map each other's exchange buffers
// (x_sp / x_tp / flags inside the request workspace) and push over NVLink.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>

#include "capi_internal.h"
#include "ddit.h"

using namespace ddit;

namespace {
typedef CUresult (*PFN_getRange)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_getRange get_range_fn() {
  static PFN_getRange fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_getRange>(p);
  });
  return fn;
}
}  // namespace

extern "C" {

DDIT_API int ddit_ipc_export(const void* ptr, void* handle, uint64_t* offset) {
  PFN_getRange fn = get_range_fn();
  if (!fn) {
    set_error("cuMemGetAddressRange unavailable");
    return DDIT_E_CUDA;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) {
    set_error("cuMemGetAddressRange failed");
    return DDIT_E_CUDA;
  }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) {
    set_error("cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    return DDIT_E_CUDA;
  }
  static_assert(sizeof(h) == 64, "ipc handle size");
  memcpy(handle, &h, sizeof h);
  *offset = reinterpret_cast<uint64_t>(ptr) - static_cast<uint64_t>(base);
  return DDIT_OK;
}

DDIT_API int ddit_ipc_import(const void* handle, uint64_t offset, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    set_error("cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    return DDIT_E_CUDA;
  }
  *ptr = static_cast<char*>(base) + offset;
  return DDIT_OK;
}

DDIT_API int ddit_ipc_close(void* ptr, uint64_t offset) {
  cudaError_t e = cudaIpcCloseMemHandle(static_cast<char*>(ptr) - offset);
  if (e != cudaSuccess) {
    set_error("cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return DDIT_E_CUDA;
  }
  return DDIT_OK;
}

}  // extern "C"
