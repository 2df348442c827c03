// Guard-zone device allocator of the guard build (see devmem.hpp).  Compiled
// into every build; empty unless BPDEC_GUARD is defined.
#include "devmem.hpp"

#ifdef BPDEC_GUARD
#include <map>
#include <mutex>
#include <vector>

namespace bpdec {
namespace {

struct Block {
  char* base;
  size_t bytes;  // payload
  int device;
};

std::mutex& mu() {
  static std::mutex m;
  return m;
}
std::map<void*, Block>& blocks() {
  static std::map<void*, Block> b;
  return b;
}

bool zone_intact(const char* zone, std::vector<unsigned char>& buf) {
  buf.resize(kGuardBytes);
  if (cudaMemcpy(buf.data(), zone, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
  for (unsigned char c : buf)
    if (c != 0xFF) return false;
  return true;
}

}  // namespace

cudaError_t dev_malloc(void** p, size_t bytes) {
  char* base = nullptr;
  const size_t total = bytes + 2 * kGuardBytes;
  cudaError_t e = cudaMalloc(&base, total);
  if (e != cudaSuccess) return e;
  e = cudaMemset(base, 0xFF, total);
  if (e != cudaSuccess) {
    cudaFree(base);
    return e;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  *p = base + kGuardBytes;
  std::lock_guard<std::mutex> lk(mu());
  blocks()[*p] = Block{base, bytes, dev};
  return cudaSuccess;
}

cudaError_t dev_free(void* p) {
  if (p == nullptr) return cudaSuccess;
  Block b;
  {
    std::lock_guard<std::mutex> lk(mu());
    auto it = blocks().find(p);
    if (it == blocks().end()) return cudaFree(p);
    b = it->second;
    blocks().erase(it);
  }
  return cudaFree(b.base);
}

cudaError_t dev_verify(const char** where) {
  if (where) *where = nullptr;
  std::vector<Block> live;
  {
    std::lock_guard<std::mutex> lk(mu());
    for (const auto& kv : blocks()) live.push_back(kv.second);
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return e;
  std::vector<unsigned char> buf;
  for (const Block& b : live) {
    cudaSetDevice(b.device);
    if (!zone_intact(b.base, buf)) {
      if (where) *where = "guard zone before an allocation overwritten (out-of-bounds write)";
      cudaSetDevice(prev);
      return cudaErrorUnknown;
    }
    if (!zone_intact(b.base + kGuardBytes + b.bytes, buf)) {
      if (where) *where = "guard zone after an allocation overwritten (out-of-bounds write)";
      cudaSetDevice(prev);
      return cudaErrorUnknown;
    }
  }
  cudaSetDevice(prev);
  return cudaSuccess;
}

}  // namespace bpdec
#endif
