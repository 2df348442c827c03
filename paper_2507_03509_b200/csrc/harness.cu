// GPU Monte-Carlo harness ≙ etdec::run_trials (reference
// proj/core/src/channel.cpp:74-156, channel.hpp:40-74): all-zero codeword
// over BI-AWGN, per-trial counter-based noise (sample_block, channel.cpp:44-61),
// punctured positions forced to LLR 0, trials decoded in device-resident
// blocks by the batched decoder, and the stop rule applied to the exact
// trial-index prefix (channel.cpp:124-147) so the statistics do not depend on
// the block size — the analogue of the reference's worker-count invariance.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <deque>
#include <memory>
#include <string>
#include <vector>

#include "decoder.hpp"
#include "devguard.hpp"
#include "devmem.hpp"
#include "harness.hpp"

namespace bpdec {

namespace {

#define HCUDA_OK(expr)                                                                     \
  do {                                                                                     \
    cudaError_t err__ = (expr);                                                            \
    if (err__ != cudaSuccess) {                                                            \
      if (err__ == cudaErrorMemoryAllocation) {                                            \
        (void)cudaGetLastError();                                                          \
        throw OomError(std::string("CUDA out of memory: ") + #expr);                       \
      }                                                                                    \
      throw CudaError(std::string("CUDA error ") + cudaGetErrorString(err__) + " at " + #expr); \
    }                                                                                      \
  } while (0)

__global__ void k_puncture(float* llr, int32_t n, int32_t frames, const int32_t* idx, int32_t count) {
  const long long total = static_cast<long long>(frames) * count;
  for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int f = static_cast<int>(t / count);
    llr[static_cast<size_t>(f) * n + idx[t - static_cast<long long>(f) * count]] = 0.0f;
  }
}

// flag[f] = 1 iff frame f's packed hard decision has any bit set
__global__ void k_any_bit(const uint32_t* bits, int32_t nw, int32_t frames, uint32_t* flag) {
  const int f = blockIdx.x;
  if (f >= frames) return;
  uint32_t acc = 0u;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) acc |= bits[static_cast<size_t>(f) * nw + i];
  acc = __syncthreads_or(acc != 0u);
  if (threadIdx.x == 0) flag[f] = acc ? 1u : 0u;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) { HCUDA_OK(dev_malloc(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T))); }
  ~DevBuf() {
    if (p) dev_free(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace

std::pair<double, double> wilson_interval(int64_t k, int64_t n) {
  // channel.cpp:63-72 (95 %, z = 1.959963984540054)
  constexpr double z = 1.959963984540054;
  const double nn = static_cast<double>(n);
  const double p = static_cast<double>(k) / nn;
  const double z2 = z * z;
  const double denom = 1.0 + z2 / nn;
  const double center = (p + z2 / (2.0 * nn)) / denom;
  const double half = z * std::sqrt(p * (1.0 - p) / nn + z2 / (4.0 * nn * nn)) / denom;
  return {std::max(0.0, center - half), std::min(1.0, center + half)};
}

TrialStats run_trials(GpuDecoder* dec, int32_t n_vars, int32_t n_checks, double snr,
                      const std::vector<int32_t>& punctured, const DecodeParams& p, int64_t min_frame_errors,
                      int64_t max_frames, uint64_t seed, int32_t block) {
  if (min_frame_errors < 1 && max_frames < 1) {
    throw ValidationError("run_trials: stop rule must bound the run (min_frame_errors or max_frames)");
  }
  if (block < 1) throw ValidationError("run_trials: block must be >= 1");
  if (!(snr > 0.0) || !std::isfinite(snr)) throw ValidationError("run_trials: snr must be positive and finite");
  for (int32_t v : punctured) {
    if (v < 0 || v >= n_vars) throw ValidationError("run_trials: punctured index out of range");
  }
  // buffers and helper kernels on the decoder's device (the caller's current
  // device is restored on exit)
  DeviceGuard dg(gpu_decoder_device(dec));
  HCUDA_OK(dg.status());
  const int32_t nw = (n_vars + 31) / 32;
  const size_t B = static_cast<size_t>(block);
  // Pipelined: up to kDepth blocks in flight through the decoder's stream
  // mode (generation + puncturing of block k+1 on a side stream while block
  // k decodes; a block's slow frames share their steps with the next
  // block's), folded strictly in trial order on the host.
  constexpr int kDepth = 3;
  struct Slot {
    DevBuf<float> llr;
    DevBuf<uint32_t> bits;
    DevBuf<int32_t> iters;
    DevBuf<uint8_t> reasons;
    explicit Slot(size_t b, int32_t n, int32_t w) : llr(b * n), bits(b * w), iters(b), reasons(b) {}
  };
  std::vector<std::unique_ptr<Slot>> slots;
  for (int k = 0; k < kDepth; ++k) slots.emplace_back(new Slot(B, n_vars, nw));
  DevBuf<uint32_t> d_flag(B);
  DevBuf<int32_t> d_punct(punctured.size());
  if (!punctured.empty()) {
    HCUDA_OK(cudaMemcpy(d_punct.p, punctured.data(), punctured.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  cudaStream_t gs = nullptr;
  HCUDA_OK(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
  struct StreamGuard {  // closes the decoder's stream (and the side stream) on every exit
    GpuDecoder* dec;
    cudaStream_t gs;
    bool open = false;
    ~StreamGuard() {
      if (open) {
        try {
          gpu_stream_close(dec);
        } catch (...) {
        }
      }
      cudaStreamDestroy(gs);
    }
  } guard{dec, gs};
  gpu_stream_open(dec, p, /*packed=*/true, /*want_bits=*/true, /*want_post=*/false, /*want_q=*/false,
                  static_cast<int32_t>(kDepth * B));
  guard.open = true;
  std::vector<int32_t> it(B);
  std::vector<uint8_t> rs(B);
  std::vector<uint32_t> nz(B);

  TrialStats st;
  st.histogram.assign(static_cast<size_t>(p.d_max) + 1, 0);
  struct InFlight {
    int64_t ticket;
    int32_t nb;
    int slot;
  };
  std::deque<InFlight> inflight;
  int64_t next = 0, folded = 0;
  bool exhausted = false, done = false;
  auto submit = [&](int slot) {
    int64_t bs = block;
    if (max_frames > 0) bs = std::min<int64_t>(bs, max_frames - next);
    if (bs <= 0) {
      exhausted = true;
      return;
    }
    const int32_t nb = static_cast<int32_t>(bs);
    Slot& sl = *slots[slot];
    gpu_sample_frames_device(dec, snr, 0.0, 0.0, 0.0, seed, next, nb, /*all_zero=*/true, sl.llr.p, nullptr, nullptr,
                             gs);
    if (!punctured.empty()) {
      k_puncture<<<256, 256, 0, gs>>>(sl.llr.p, n_vars, nb, d_punct.p, static_cast<int32_t>(punctured.size()));
      HCUDA_OK(cudaGetLastError());
      HCUDA_OK(cudaStreamSynchronize(gs));
    }
    StreamOutputs o;
    o.bits = sl.bits.p;
    o.iterations = sl.iters.p;
    o.reasons = sl.reasons.p;
    inflight.push_back({gpu_stream_submit(dec, nb, sl.llr.p, nullptr, o), nb, slot});
    next += nb;
  };
  for (int k = 0; k < kDepth && !exhausted; ++k) submit(k);
  while (!inflight.empty() && !done) {
    const InFlight f = inflight.front();
    inflight.pop_front();
    gpu_stream_wait(dec, f.ticket);
    const Slot& sl = *slots[f.slot];
    const int32_t nb = f.nb;
    k_any_bit<<<nb, 256, 0, gs>>>(sl.bits.p, nw, nb, d_flag.p);
    HCUDA_OK(cudaGetLastError());
    HCUDA_OK(cudaMemcpyAsync(it.data(), sl.iters.p, nb * sizeof(int32_t), cudaMemcpyDeviceToHost, gs));
    HCUDA_OK(cudaMemcpyAsync(rs.data(), sl.reasons.p, nb, cudaMemcpyDeviceToHost, gs));
    HCUDA_OK(cudaMemcpyAsync(nz.data(), d_flag.p, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, gs));
    HCUDA_OK(cudaStreamSynchronize(gs));
    // fold in trial order; the error target truncates exactly where a serial
    // run would have stopped (channel.cpp:133-147)
    for (int32_t t = 0; t < nb; ++t) {
      ++st.frames;
      st.iteration_sum += it[t];
      ++st.histogram[std::min<size_t>(static_cast<size_t>(it[t]), st.histogram.size() - 1)];
      if (rs[t] == 0) ++st.stops_syndrome;
      else if (rs[t] == 1) ++st.stops_vnr;
      else ++st.stops_max_iter;
      const bool all_zero = nz[t] == 0u;
      if (!all_zero || rs[t] != 0) ++st.frame_errors;
      if (!all_zero && rs[t] == 0) ++st.undetected_errors;
      if (min_frame_errors > 0 && st.frame_errors >= min_frame_errors) {
        done = true;
        break;
      }
    }
    folded += nb;
    if (!done && max_frames > 0 && folded >= max_frames) {
      st.hit_max_frames = true;
      done = true;
    }
    if (!done && !exhausted) submit(f.slot);  // the folded block's buffers take the next block
  }
  // blocks still in flight past the stop are discarded (gpu_stream_close
  // waits for them)
  guard.open = false;
  gpu_stream_close(dec);
  st.fer = static_cast<double>(st.frame_errors) / static_cast<double>(st.frames);
  const auto ci = wilson_interval(st.frame_errors, st.frames);
  st.fer_ci_low = ci.first;
  st.fer_ci_high = ci.second;
  st.d_bar = static_cast<double>(st.iteration_sum) / static_cast<double>(st.frames);
  (void)n_checks;
  return st;
}

}  // namespace bpdec
