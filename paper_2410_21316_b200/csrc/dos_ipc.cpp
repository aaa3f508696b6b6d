// dos_ipc.cpp — CUDA IPC for the symmetric full-model buffers of the fused
// all-gather (one process per GPU on one node).  A rank exports the
// allocation that holds its full-model buffer; every other rank maps it once
// and K1 / the copy engine then store straight into it over NVLink.
#include <cuda.h>
#include <cuda_runtime.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>

#include "dos_internal.h"

namespace {

typedef CUresult (*pfn_range)(CUdeviceptr*, size_t*, CUdeviceptr);

pfn_range range_fn() {
  static pfn_range fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (pfn_range) nullptr;
    }
    return reinterpret_cast<pfn_range>(f);
  }();
  return fn;
}

std::mutex g_mu;
std::map<std::string, void*> g_open;  // handle bytes -> mapped base in this process

}  // namespace

extern "C" int dos_ipc_export(const void* dev_ptr, unsigned char handle[64], uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return dos_set_error(DOS_EINVAL, "NULL argument");
  pfn_range fn = range_fn();
  if (!fn) return dos_set_error(DOS_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return dos_set_error(DOS_EINVAL, "pointer %p is not device memory", dev_ptr);
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, 64);
  *offset = (uint64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return DOS_OK;
}

extern "C" int dos_ipc_import(const unsigned char handle[64], uint64_t offset, void** dev_ptr) {
  if (!handle || !dev_ptr) return dos_set_error(DOS_EINVAL, "NULL argument");
  const std::string key(reinterpret_cast<const char*>(handle), 64);
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_open.find(key);
  void* base = nullptr;
  if (it != g_open.end()) {
    base = it->second;
  } else {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    g_open[key] = base;
  }
  *dev_ptr = static_cast<char*>(base) + offset;
  return DOS_OK;
}

extern "C" int dos_ipc_close_all(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& kv : g_open) cudaIpcCloseMemHandle(kv.second);
  g_open.clear();
  return DOS_OK;
}
