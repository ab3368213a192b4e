// dk_device.cu — per-device properties and kernel attributes.
//
// Every value here is per device ordinal: a process may drive several GPUs (dk_set_device),
// and cudaFuncSetAttribute applies to the current device only.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

#include "dk_launch.h"

namespace dk {

namespace {
std::mutex g_mu;
int g_sms[kMaxDevices] = {0};
std::map<std::pair<const void*, int>, int> g_smem;  // (kernel, device) -> opted-in bytes
}  // namespace

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

int num_sms() {
  const int dev = current_device();
  const int slot = dev % kMaxDevices;
  int n = __atomic_load_n(&g_sms[slot], __ATOMIC_ACQUIRE);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 1;
    }
    __atomic_store_n(&g_sms[slot], n, __ATOMIC_RELEASE);
  }
  return n;
}

int smem_optin(const void* fn, size_t bytes) {
  // no shortcut below 48 KB: the limit applies to static + dynamic shared memory
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  int& have = g_smem[{fn, dev}];
  if ((size_t)have >= bytes) return 0;
  const cudaError_t e =
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return (int)e;
  have = (int)bytes;
  return 0;
}

}  // namespace dk
