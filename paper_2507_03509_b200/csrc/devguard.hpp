// Current-device guard: selects a decoder's device for the duration of a
// call and restores the caller's device on exit (one host
// thread may hold decoders on several GPUs).
#pragma once

#include <cuda_runtime.h>

namespace bpdec {

class DeviceGuard {
 public:
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev_) != cudaSuccess) {
      (void)cudaGetLastError();
      prev_ = -1;
    }
    if (prev_ != device) {
      err_ = cudaSetDevice(device);
      if (err_ != cudaSuccess) (void)cudaGetLastError();
    }
  }
  ~DeviceGuard() {
    if (prev_ >= 0) cudaSetDevice(prev_);
  }
  cudaError_t status() const { return err_; }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;

 private:
  int prev_ = -1;
  cudaError_t err_ = cudaSuccess;
};

}  // namespace bpdec
