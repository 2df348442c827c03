// Host-side interface of the CUDA decoder (no CUDA types; used by c_api.cpp).
#pragma once

#include <cstdint>

#include "code.hpp"

namespace bpdec {

struct DecodeParams {
  int32_t d_max = 100;
  int32_t use_pce = 1;
  int32_t use_vnr = 0;
  int32_t q_mode = 0;  // 0 raw, 1 abs
  float msg_clamp = 30.0f;
};

struct DecodeBuffers {
  int32_t batch = 0;
  const float* llr = nullptr;          // [batch][N]
  const uint32_t* syndrome = nullptr;  // [batch][ceil(M/32)] or null
  bool bits_packed = false;
  void* bits = nullptr;                // u8 [batch][N] or u32 [batch][ceil(N/32)]
  int32_t* iterations = nullptr;
  uint8_t* reasons = nullptr;
  float* posteriors = nullptr;
  double* q_trace = nullptr;
  // observer traces (IterationObserver, decoder.hpp:53-55 of the reference):
  // syndrome_ok of every iteration [batch][d_max] (0/1, 0xff past the stop)
  // and the posteriors of every iteration [batch][d_max][N]
  uint8_t* syn_trace = nullptr;
  float* post_trace = nullptr;
};

// Stream mode: caller-owned output buffers of one submitted batch (host or
// device pointers; any may be null except iterations / reasons).
struct StreamOutputs {
  void* bits = nullptr;
  int32_t* iterations = nullptr;
  uint8_t* reasons = nullptr;
  float* posteriors = nullptr;
  double* q_trace = nullptr;
};

class GpuDecoder;

GpuDecoder* gpu_decoder_create(const Code& code, int device, int max_slots);
void gpu_decoder_destroy(GpuDecoder* dec);
int gpu_decoder_slots(const GpuDecoder* dec);
int gpu_decoder_device(const GpuDecoder* dec);
int64_t gpu_decoder_device_bytes(const GpuDecoder* dec);
void gpu_decode_batch(GpuDecoder* dec, const DecodeParams& p, const DecodeBuffers& b, void* stream);
// snr > 0: fixed SNR; snr <= 0: per-frame beta ~ U[beta_lo, beta_hi] (rate R).
void gpu_sample_frames_device(GpuDecoder* dec, double snr, double beta_lo, double beta_hi, double rate,
                              uint64_t seed, int64_t first_frame, int32_t n_frames, bool all_zero, float* d_llr,
                              uint32_t* d_syndrome, uint32_t* d_x_packed, void* stream);
// Asynchronous H2D of a host batch into one of two staging slots; a later
// decode with the same host pointers and batch uses the staged copy.
void gpu_stage_inputs(GpuDecoder* dec, int32_t batch, const float* llr_host, const uint32_t* syn_host);
// Stream mode: batches submitted back to back decode as one continuous frame
// stream through the decoder's slots (a later batch's frames fill the lanes
// an earlier batch's tail frees); completion per batch ticket.
void gpu_stream_open(GpuDecoder* dec, const DecodeParams& p, bool packed, bool want_bits, bool want_post,
                     bool want_q, int32_t ring_frames);
int64_t gpu_stream_submit(GpuDecoder* dec, int32_t n, const float* llr, const uint32_t* syn, const StreamOutputs& o);
bool gpu_stream_query(GpuDecoder* dec, int64_t ticket);
void gpu_stream_wait(GpuDecoder* dec, int64_t ticket);
void gpu_stream_close(GpuDecoder* dec);
void gpu_stream_timer_reset(GpuDecoder* dec);
double gpu_stream_device_ms(GpuDecoder* dec);
void gpu_set_profiling(GpuDecoder* dec, bool enable);
void gpu_profile(const GpuDecoder* dec, int kernel, double* total_ms, int64_t* launches,
                 double* frame_iterations);
void gpu_reset_profile(GpuDecoder* dec);
int64_t gpu_launch_count(const GpuDecoder* dec);

}  // namespace bpdec
