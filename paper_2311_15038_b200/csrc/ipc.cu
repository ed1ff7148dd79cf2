// Peer memory between the ranks of one node: the atlas
// "gather to rank 0" becomes the fused pass itself -- every rank's kernel
// stores its slab's atlas rows straight into rank 0's atlas buffers over
// NVLink/NVSwitch (CUDA IPC mapping), so the exchange overlaps the compute tile
// by tile and no separate gather runs.  These entry points export / import a
// device buffer between processes; the kernels are unchanged (a level's
// destination pointer may be a peer mapping).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>
#include <string.h>
#include "ctp_common.cuh"

namespace ctp {

static PFN_cuMemGetAddressRange_v3020 range_fn() {
  static std::once_flag once;
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  return fn;
}

}  // namespace ctp

using namespace ctp;

extern "C" {

int ctp_ipc_export(const void* ptr, uint8_t* handle, int64_t* offset) {
  CTP_REQUIRE(ptr && handle && offset, CTP_E_INVALID, "ctp_ipc_export: null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == CTP_IPC_HANDLE_BYTES, "IPC handle size");
  PFN_cuMemGetAddressRange_v3020 fn = range_fn();
  CTP_REQUIRE(fn != nullptr, CTP_E_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr));
  CTP_REQUIRE(r == CUDA_SUCCESS, CTP_E_CUDA, "cuMemGetAddressRange failed (%d)", (int)r);
  cudaIpcMemHandle_t h;
  CTP_CUDA_CALL(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return CTP_OK;
}

int ctp_ipc_import(const uint8_t* handle, int64_t offset, void** ptr) {
  CTP_REQUIRE(handle && ptr && offset >= 0, CTP_E_INVALID, "ctp_ipc_import: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  CTP_CUDA_CALL(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = static_cast<uint8_t*>(base) + offset;
  return CTP_OK;
}

int ctp_ipc_close(void* ptr, int64_t offset) {
  CTP_REQUIRE(ptr && offset >= 0, CTP_E_INVALID, "ctp_ipc_close: bad arguments");
  CTP_CUDA_CALL(cudaIpcCloseMemHandle(static_cast<uint8_t*>(ptr) - offset));
  return CTP_OK;
}

}  // extern "C"
