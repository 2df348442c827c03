// GPU Monte-Carlo harness (≙ etdec::run_trials, channel.hpp:40-74).
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "decoder.hpp"

namespace bpdec {

// ≙ etdec::TrialStats (channel.hpp:47-61); histogram[k] = frames that ran k iterations.
struct TrialStats {
  int64_t frames = 0;
  int64_t frame_errors = 0;
  int64_t undetected_errors = 0;
  double fer = 0.0;
  double fer_ci_low = 0.0;
  double fer_ci_high = 0.0;
  double d_bar = 0.0;
  int64_t iteration_sum = 0;
  std::vector<int64_t> histogram;
  int64_t stops_syndrome = 0;
  int64_t stops_vnr = 0;
  int64_t stops_max_iter = 0;
  bool hit_max_frames = false;
};

// ≙ wilson_interval (channel.cpp:63-72)
std::pair<double, double> wilson_interval(int64_t k, int64_t n);

TrialStats run_trials(GpuDecoder* dec, int32_t n_vars, int32_t n_checks, double snr,
                      const std::vector<int32_t>& punctured, const DecodeParams& p, int64_t min_frame_errors,
                      int64_t max_frames, uint64_t seed, int32_t block);

}  // namespace bpdec
