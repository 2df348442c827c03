// Device allocations of the library.  Release builds: cudaMalloc / cudaFree.
//
// Guard builds (-DBPDEC_GUARD, `make guard` -> libbpdec_guard.so; the
// bounds-checking stand-in for compute-sanitizer, which this GPU pool does
// not allow): every allocation gets a 64 KiB guard zone on each side, the
// whole block (zones and payload) is poisoned with 0xFF bytes (NaN floats,
// -1 integers), and dev_verify() checks that every live allocation's zones
// still hold the poison.  So a kernel that writes out of bounds is caught by
// the next verify (the decode entry points run it before returning), one
// that reads out of bounds or reads memory nothing wrote gets NaN / -1,
// which the parity tests (bit-exact or 1e-4 against the CPU reference) turn
// into a failure or an illegal-address error.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace bpdec {

#ifdef BPDEC_GUARD
constexpr size_t kGuardBytes = 64 * 1024;
// returns cudaErrorUnknown with *where set when a guard zone was overwritten
cudaError_t dev_verify(const char** where);
cudaError_t dev_malloc(void** p, size_t bytes);
cudaError_t dev_free(void* p);
#else
inline cudaError_t dev_verify(const char** where) {
  if (where) *where = nullptr;
  return cudaSuccess;
}
inline cudaError_t dev_malloc(void** p, size_t bytes) { return cudaMalloc(p, bytes); }
inline cudaError_t dev_free(void* p) { return cudaFree(p); }
#endif

}  // namespace bpdec
