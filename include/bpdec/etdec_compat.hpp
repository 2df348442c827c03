// etdec_compat.hpp — header-only C++ host layer with the reference's decode
// interface (namespace etdec in /root/reference/proj/core/include/etdec/),
// implemented on top of the C ABI in include/bpdec.h.
//
// A caller of the reference switches by replacing
//     #include <etdec/decoder.hpp>           with   #include <bpdec/etdec_compat.hpp>
//     etdec::                                 with   bpdec::compat::
// and linking libbpdec.so.  Same class names, argument meaning and exception
// classes; the difference is that decode runs on the GPU and there is also a
// batched, syndrome-aware entry point (BpDecoder::decode_batch).
//
//   reference (file:line)                          here
//   ParityCheckMatrix::from_check_lists (pcm.hpp:16) ParityCheckMatrix::from_check_lists
//   load_alist_file / save_alist_file (alist.hpp:21,24)  load_alist_file / save_alist_file
//   lift_protograph (protograph.hpp:31)            lift_protograph
//   active_var_set (pcm.hpp:70)                    active_var_set
//   DecodeConfig / DecodeOutcome / StopReason      same (decoder.hpp:13-36)
//   BpDecoder(code), BpDecoder::decode (decoder.hpp:57-65)  same (+ syndrome overload)
//   decode(code, llr, active, cfg) (decoder.hpp:78-79)      same
//   syndrome_check / vnr_statistic / vnr_should_stop (decoder.hpp:39-45)  same
//   snr_for_beta (channel.hpp:24)                  snr_for_beta
//   ConfigError / IoError / ValidationError (errors.hpp:8-24)  same
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <algorithm>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../bpdec.h"

namespace bpdec::compat {

class ConfigError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ValidationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check_status(int st) {
  if (st == BPDEC_OK) return;
  const std::string msg = bpdec_last_error();
  switch (st) {
    case BPDEC_ERR_CONFIG: throw ConfigError(msg);
    case BPDEC_ERR_IO: throw IoError(msg);
    case BPDEC_ERR_VALIDATION: throw ValidationError(msg);
    default: throw DeviceError(msg);
  }
}

class ParityCheckMatrix {
 public:
  static ParityCheckMatrix from_check_lists(int n_vars, const std::vector<std::vector<int>>& per_check_vars) {
    std::vector<int32_t> ptr(per_check_vars.size() + 1, 0), vars;
    for (size_t c = 0; c < per_check_vars.size(); ++c) {
      vars.insert(vars.end(), per_check_vars[c].begin(), per_check_vars[c].end());
      ptr[c + 1] = static_cast<int32_t>(vars.size());
    }
    bpdec_code* h = nullptr;
    check_status(bpdec_code_from_csr(n_vars, static_cast<int32_t>(per_check_vars.size()), ptr.data(),
                                     vars.empty() ? nullptr : vars.data(), &h));
    return ParityCheckMatrix(h);
  }
  static ParityCheckMatrix adopt(bpdec_code* h) { return ParityCheckMatrix(h); }

  int n_vars() const { return n_vars_; }
  int n_checks() const { return n_checks_; }
  int n_edges() const { return static_cast<int>(n_edges_); }
  double rate() const { return static_cast<double>(n_vars_ - n_checks_) / n_vars_; }
  const bpdec_code* handle() const { return h_.get(); }

 private:
  explicit ParityCheckMatrix(bpdec_code* h) : h_(h, &bpdec_code_destroy) {
    int32_t active = 0;
    check_status(bpdec_code_dims(h, &n_vars_, &n_checks_, &n_edges_, &active));
  }
  std::shared_ptr<bpdec_code> h_;
  int32_t n_vars_ = 0, n_checks_ = 0;
  int64_t n_edges_ = 0;
};

inline ParityCheckMatrix load_alist_file(const std::string& path) {
  bpdec_code* h = nullptr;
  check_status(bpdec_code_load_alist(path.c_str(), &h));
  return ParityCheckMatrix::adopt(h);
}
inline void save_alist_file(const ParityCheckMatrix& code, const std::string& path) {
  check_status(bpdec_code_save_alist(code.handle(), path.c_str()));
}
inline ParityCheckMatrix lift_protograph(const std::vector<std::vector<int>>& base, int z, std::uint64_t seed) {
  if (base.empty() || base.front().empty()) throw ValidationError("protograph lift: empty base matrix");
  const size_t rows = base.size(), cols = base.front().size();
  std::vector<int32_t> flat;
  for (const auto& r : base) {
    if (r.size() != cols) throw ValidationError("protograph lift: ragged base matrix");
    flat.insert(flat.end(), r.begin(), r.end());
  }
  bpdec_code* h = nullptr;
  check_status(bpdec_code_lift_protograph(flat.data(), static_cast<int32_t>(rows), static_cast<int32_t>(cols), z,
                                          seed, &h));
  return ParityCheckMatrix::adopt(h);
}

struct ActiveVarSet {
  std::vector<int> members;
};
inline ActiveVarSet active_var_set(const ParityCheckMatrix& code) {
  int32_t n = 0, m = 0, a = 0;
  int64_t e = 0;
  check_status(bpdec_code_dims(code.handle(), &n, &m, &e, &a));
  ActiveVarSet s;
  s.members.resize(a);
  if (a) check_status(bpdec_code_active_vars(code.handle(), s.members.data()));
  return s;
}

enum class StopReason { kSyndromeSatisfied, kVnrDrop, kMaxIterations };
inline const char* to_string(StopReason r) { return bpdec_stop_reason_name(static_cast<int32_t>(r)); }

struct DecodeConfig {
  int d_max = 100;
  bool use_pce = true;
  bool use_vnr = false;
  double msg_clamp = 30.0;
  int q_mode = BPDEC_Q_RAW;  // extension: BPDEC_Q_ABS for true syndrome mode
};

struct DecodeOutcome {
  std::vector<std::uint8_t> bits;
  int iterations = 0;
  StopReason reason = StopReason::kMaxIterations;
  std::vector<double> q_trace;
  std::vector<double> posteriors;
  bool converged() const { return reason == StopReason::kSyndromeSatisfied; }
};

inline bool syndrome_check(const ParityCheckMatrix& code, std::span<const std::uint8_t> bits) {
  if (bits.size() != static_cast<size_t>(code.n_vars())) {
    throw ValidationError("syndrome_check: bit vector length " + std::to_string(bits.size()) +
                          " does not match n_vars=" + std::to_string(code.n_vars()));
  }
  int32_t ok = 0;
  check_status(bpdec_syndrome_check(code.handle(), bits.data(), nullptr, &ok));
  return ok != 0;
}

inline double vnr_statistic(std::span<const double> posteriors, const ActiveVarSet& active) {
  double q = 0.0;
  for (int v : active.members) q += posteriors[v];
  return q;
}
inline bool vnr_should_stop(double q_k, double q_km1) { return q_k < q_km1; }

// ≙ etdec::ChannelPoint / snr_for_beta (channel.hpp:14-23)
struct ChannelPoint {
  double beta = 0.0;
  double rate = 0.0;
  double snr = 0.0;
  double sigma2 = 0.0;
};
inline ChannelPoint snr_for_beta(double beta, double rate) {
  ChannelPoint p;
  check_status(bpdec_snr_for_beta(beta, rate, &p.snr));
  p.beta = beta;
  p.rate = rate;
  p.sigma2 = 1.0 / p.snr;
  return p;
}

// ≙ etdec::PunctureMask / no_puncture / apply_puncture (puncture.hpp:12-26)
struct PunctureMask {
  std::vector<int> punctured;  // ascending variable indices
  double effective_rate = 0.0;
  bool empty() const { return punctured.empty(); }
};
inline PunctureMask no_puncture(const ParityCheckMatrix& code) {
  PunctureMask m;
  m.effective_rate = code.rate();
  return m;
}
inline PunctureMask apply_puncture(const ParityCheckMatrix& code, double target_rate, std::uint64_t seed) {
  PunctureMask m;
  m.punctured.resize(static_cast<size_t>(code.n_vars()));
  int32_t count = 0;
  check_status(bpdec_code_apply_puncture(code.handle(), target_rate, seed, m.punctured.data(), &count,
                                         &m.effective_rate));
  m.punctured.resize(static_cast<size_t>(count));
  return m;
}

// ≙ etdec::StopRule / TrialStats / wilson_interval (channel.hpp:42-64)
struct StopRule {
  long min_frame_errors = 100;
  long max_frames = 10000;
};
struct TrialStats {
  long frames = 0;
  long frame_errors = 0;
  long undetected_errors = 0;
  double fer = 0.0;
  double fer_ci_low = 0.0;
  double fer_ci_high = 0.0;
  double d_bar = 0.0;
  long long iteration_sum = 0;
  std::map<int, long> iteration_histogram;
  long stops_syndrome = 0;
  long stops_vnr = 0;
  long stops_max_iter = 0;
  bool hit_max_frames = false;
};
inline std::pair<double, double> wilson_interval(long k, long n) {
  double lo = 0.0, hi = 0.0;
  check_status(bpdec_wilson_interval(k, n, &lo, &hi));
  return {lo, hi};
}

// GPU decoder for one code on one device.  Not thread-safe (like the
// reference's BpDecoder, decoder.hpp:47-50); use one per host thread.
class BpDecoder {
 public:
  using IterationObserver =
      std::function<void(int iteration, std::span<const double> posteriors, bool syndrome_ok, double q)>;

  explicit BpDecoder(const ParityCheckMatrix& code, int device = 0, int max_slots = 32) : code_(code) {
    bpdec_decoder* d = nullptr;
    check_status(bpdec_decoder_create(code.handle(), device, max_slots, &d));
    dec_.reset(d);
  }

  // ≙ BpDecoder::decode (decoder.hpp:64-65).  LLRs are rounded to float32.
  // `active` must be active_var_set(code) (the device builds q over the
  // degree>=2 variables); another set throws ValidationError.  The observer
  // receives, per iteration, that iteration's posteriors, the real
  // syndrome_ok (computed every iteration, PCE on or off, decoder.cpp:110-112)
  // and q — replayed from bpdec_decode_batch_traced after the decode.
  DecodeOutcome decode(std::span<const double> llr_in, const ActiveVarSet& active, const DecodeConfig& cfg,
                       const IterationObserver& observer = nullptr, const std::uint32_t* syndrome = nullptr) {
    const int n = code_.n_vars();
    if (llr_in.size() != static_cast<size_t>(n)) {
      throw ValidationError("decode: LLR length " + std::to_string(llr_in.size()) +
                            " does not match n_vars=" + std::to_string(n));
    }
    for (double l : llr_in)
      if (!std::isfinite(l)) throw ValidationError("decode: non-finite input LLR");
    if (!same_active_set(active))
      throw ValidationError("decode: only active_var_set(code) (the degree>=2 variables) is supported as the VNR "
                            "active set");
    std::vector<float> llr(llr_in.begin(), llr_in.end());
    if (!observer) return std::move(decode_batch(1, llr.data(), syndrome, cfg, true)[0]);
    // outcome + syndrome_ok trace, then (deterministic per frame) the
    // posteriors of iterations 1..k with d_max = k: a k x N trace buffer
    bpdec_config c{cfg.d_max, cfg.use_pce ? 1 : 0, cfg.use_vnr ? 1 : 0, cfg.q_mode, cfg.msg_clamp};
    std::vector<std::uint8_t> bits(static_cast<size_t>(n)), syn_ok(static_cast<size_t>(cfg.d_max > 0 ? cfg.d_max : 1));
    std::vector<float> post(static_cast<size_t>(n));
    std::vector<double> qt(syn_ok.size());
    int32_t it = 0;
    std::uint8_t rs = 0;
    check_status(bpdec_decode_batch_traced(dec_.get(), 1, llr.data(), syndrome, &c, 0, bits.data(), &it, &rs,
                                           post.data(), qt.data(), syn_ok.data(), nullptr, nullptr));
    bpdec_config tc{it, 0, 0, cfg.q_mode, cfg.msg_clamp};
    std::vector<float> ptrace(static_cast<size_t>(it) * n);
    int32_t it2 = 0;
    std::uint8_t rs2 = 0;
    check_status(bpdec_decode_batch_traced(dec_.get(), 1, llr.data(), syndrome, &tc, 0, nullptr, &it2, &rs2, nullptr,
                                           nullptr, nullptr, ptrace.data(), nullptr));
    std::vector<double> pk(static_cast<size_t>(n));
    for (int k = 0; k < it; ++k) {
      for (int v = 0; v < n; ++v) pk[v] = ptrace[static_cast<size_t>(k) * n + v];
      observer(k + 1, pk, syn_ok[k] == 1, qt[k]);
    }
    DecodeOutcome o;
    o.bits = std::move(bits);
    o.iterations = it;
    o.reason = static_cast<StopReason>(rs);
    o.q_trace.assign(qt.begin(), qt.begin() + it);
    o.posteriors.assign(post.begin(), post.end());
    return o;
  }

  bpdec_decoder* handle() const { return dec_.get(); }
  const ParityCheckMatrix& code() const { return code_; }

  // Batched, syndrome-aware decode of `batch` frames ([batch][N] float LLRs,
  // [batch][ceil(M/32)] packed syndromes or null).
  std::vector<DecodeOutcome> decode_batch(int batch, const float* llr, const std::uint32_t* syndrome,
                                          const DecodeConfig& cfg, bool want_posteriors = false) {
    const int n = code_.n_vars();
    bpdec_config c{cfg.d_max, cfg.use_pce ? 1 : 0, cfg.use_vnr ? 1 : 0, cfg.q_mode, cfg.msg_clamp};
    std::vector<std::uint8_t> bits(static_cast<size_t>(batch) * n);
    std::vector<int32_t> it(batch);
    std::vector<std::uint8_t> rs(batch);
    std::vector<float> post(want_posteriors ? static_cast<size_t>(batch) * n : 0);
    std::vector<double> qt(static_cast<size_t>(batch) * (cfg.d_max > 0 ? cfg.d_max : 1));
    check_status(bpdec_decode_batch(dec_.get(), batch, llr, syndrome, &c, 0, bits.data(), it.data(), rs.data(),
                                    want_posteriors ? post.data() : nullptr, qt.data(), nullptr));
    std::vector<DecodeOutcome> out(batch);
    for (int b = 0; b < batch; ++b) {
      auto& o = out[b];
      o.bits.assign(bits.begin() + static_cast<size_t>(b) * n, bits.begin() + static_cast<size_t>(b + 1) * n);
      o.iterations = it[b];
      o.reason = static_cast<StopReason>(rs[b]);
      o.q_trace.assign(qt.begin() + static_cast<size_t>(b) * cfg.d_max,
                       qt.begin() + static_cast<size_t>(b) * cfg.d_max + it[b]);
      if (want_posteriors)
        o.posteriors.assign(post.begin() + static_cast<size_t>(b) * n, post.begin() + static_cast<size_t>(b + 1) * n);
    }
    return out;
  }

 private:
  struct Del {
    void operator()(bpdec_decoder* d) const { bpdec_decoder_destroy(d); }
  };
  bool same_active_set(const ActiveVarSet& active) {
    if (!active_valid_) {
      active_ = active_var_set(code_);
      active_valid_ = true;
    }
    return active.members == active_.members;
  }
  ParityCheckMatrix code_;
  std::unique_ptr<bpdec_decoder, Del> dec_;
  ActiveVarSet active_;
  bool active_valid_ = false;
};

// Per-frame results of a batch in packed form (stream / multi-decoder calls).
struct BatchOutcome {
  std::vector<std::uint32_t> bits_packed;  // [batch][ceil(N/32)], bit v of frame b = hard decision of v
  std::vector<int32_t> iterations;
  std::vector<std::uint8_t> reasons;       // StopReason values
  int words_per_frame = 0;
  std::uint8_t bit(int b, int v) const {
    return static_cast<std::uint8_t>((bits_packed[static_cast<size_t>(b) * words_per_frame + (v >> 5)] >> (v & 31)) & 1u);
  }
};

// Stream mode (bpdec_stream_*; no reference counterpart — it replaces the
// per-block loop of run_trials, channel.cpp:90-148): batches submitted back
// to back decode as one continuous frame stream through the decoder's slots.
// The caller's LLR / syndrome arrays must stay valid until the batch is
// waited for.  Closing (destructor) waits for every submitted batch.
class FrameStream {
 public:
  FrameStream(BpDecoder& dec, const DecodeConfig& cfg, int ring_frames = 0)
      : dec_(dec), n_(dec.code().n_vars()), nw_((dec.code().n_vars() + 31) / 32) {
    bpdec_config c{cfg.d_max, cfg.use_pce ? 1 : 0, cfg.use_vnr ? 1 : 0, cfg.q_mode, cfg.msg_clamp};
    check_status(bpdec_stream_open(dec_.handle(), &c, BPDEC_BITS_PACKED, ring_frames, 1, 0, 0));
    open_ = true;
  }
  FrameStream(const FrameStream&) = delete;
  FrameStream& operator=(const FrameStream&) = delete;
  ~FrameStream() {
    if (open_) bpdec_stream_close(dec_.handle());
  }
  std::int64_t submit(int batch, const float* llr, const std::uint32_t* syndrome = nullptr) {
    BatchOutcome o;
    o.words_per_frame = nw_;
    o.bits_packed.assign(static_cast<size_t>(batch) * nw_, 0u);
    o.iterations.assign(batch, 0);
    o.reasons.assign(batch, 0);
    std::int64_t t = -1;
    check_status(bpdec_stream_submit(dec_.handle(), batch, llr, syndrome, o.bits_packed.data(), o.iterations.data(),
                                     o.reasons.data(), nullptr, nullptr, &t));
    pending_.emplace(t, std::move(o));  // vectors keep their buffers when moved
    return t;
  }
  BatchOutcome wait(std::int64_t ticket) {
    check_status(bpdec_stream_wait(dec_.handle(), ticket));
    auto it = pending_.find(ticket);
    if (it == pending_.end()) throw ValidationError("stream: unknown or already collected ticket");
    BatchOutcome o = std::move(it->second);
    pending_.erase(it);
    return o;
  }
  void close() {
    if (open_) {
      open_ = false;
      check_status(bpdec_stream_close(dec_.handle()));
    }
  }

 private:
  BpDecoder& dec_;
  int n_, nw_;
  bool open_ = false;
  std::map<std::int64_t, BatchOutcome> pending_;
};

// Several GPUs of one host (bpdec_multi_*; the strided worker pool of
// run_trials, channel.cpp:98-122): one decoder and host thread per entry of
// `devices` (a device may repeat), frames dealt from a dynamic chunk queue,
// per-frame outputs at their frame index — identical for any device list.
class MultiDecoder {
 public:
  MultiDecoder(const ParityCheckMatrix& code, const std::vector<int>& devices, int slots_per_decoder = 64)
      : code_(code) {
    std::vector<int32_t> dv(devices.begin(), devices.end());
    bpdec_multi* m = nullptr;
    check_status(bpdec_multi_create(code.handle(), dv.data(), static_cast<int32_t>(dv.size()), slots_per_decoder, &m));
    m_.reset(m);
  }
  BatchOutcome decode_batch(int batch, const float* llr, const std::uint32_t* syndrome, const DecodeConfig& cfg,
                            int chunk_frames = 0) {
    const int nw = (code_.n_vars() + 31) / 32;
    BatchOutcome o;
    o.words_per_frame = nw;
    o.bits_packed.assign(static_cast<size_t>(batch) * nw, 0u);
    o.iterations.assign(batch, 0);
    o.reasons.assign(batch, 0);
    bpdec_config c{cfg.d_max, cfg.use_pce ? 1 : 0, cfg.use_vnr ? 1 : 0, cfg.q_mode, cfg.msg_clamp};
    check_status(bpdec_multi_decode_batch(m_.get(), batch, llr, syndrome, &c, BPDEC_BITS_PACKED, o.bits_packed.data(),
                                          o.iterations.data(), o.reasons.data(), nullptr, nullptr, chunk_frames,
                                          nullptr));
    return o;
  }

 private:
  struct Del {
    void operator()(bpdec_multi* m) const { bpdec_multi_destroy(m); }
  };
  ParityCheckMatrix code_;
  std::unique_ptr<bpdec_multi, Del> m_;
};

// Two-edge-type low-rate construction with a core code (FER < 1 family;
// bpdec_code_generate_met_core).
inline ParityCheckMatrix generate_met_core(int n_vars, int n_checks, int n_deg1, const std::vector<int>& core_degrees,
                                           const std::vector<double>& core_probs, int ext_degree, std::uint64_t seed) {
  std::vector<int32_t> d(core_degrees.begin(), core_degrees.end());
  bpdec_code* c = nullptr;
  check_status(bpdec_code_generate_met_core(n_vars, n_checks, n_deg1, static_cast<int32_t>(d.size()), d.data(),
                                            core_probs.data(), ext_degree, seed, &c));
  return ParityCheckMatrix::adopt(c);
}

// ≙ etdec::run_trials (channel.hpp:72-74) on the GPU: trials are decoded in
// device-resident blocks instead of by `workers` threads; the stop rule is
// applied to the exact trial-index prefix, so the statistics equal the
// reference's for any block size.  `workers` only scales the block
// (64 frames per worker, at least 64).
inline TrialStats run_trials(const ParityCheckMatrix& code, const PunctureMask& mask, const ChannelPoint& point,
                             const DecodeConfig& cfg, const StopRule& stop, std::uint64_t master_seed,
                             int workers = 1, int device = 0) {
  const int block = std::max(64, 64 * std::max(1, workers));
  bpdec_decoder* d = nullptr;
  check_status(bpdec_decoder_create(code.handle(), device, block, &d));
  std::unique_ptr<bpdec_decoder, void (*)(bpdec_decoder*)> hold(d, bpdec_decoder_destroy);
  bpdec_config c{cfg.d_max, cfg.use_pce ? 1 : 0, cfg.use_vnr ? 1 : 0, cfg.q_mode, cfg.msg_clamp};
  bpdec_stop_rule r{stop.min_frame_errors, stop.max_frames};
  bpdec_trial_stats st{};
  std::vector<int64_t> hist(static_cast<size_t>(cfg.d_max) + 1, 0);
  check_status(bpdec_run_trials(d, point.snr, mask.punctured.data(), static_cast<int32_t>(mask.punctured.size()), &c,
                                &r, master_seed, block, &st, hist.data()));
  TrialStats t;
  t.frames = st.frames;
  t.frame_errors = st.frame_errors;
  t.undetected_errors = st.undetected_errors;
  t.fer = st.fer;
  t.fer_ci_low = st.fer_ci_low;
  t.fer_ci_high = st.fer_ci_high;
  t.d_bar = st.d_bar;
  t.iteration_sum = st.iteration_sum;
  for (size_t k = 0; k < hist.size(); ++k)
    if (hist[k] > 0) t.iteration_histogram[static_cast<int>(k)] = static_cast<long>(hist[k]);
  t.stops_syndrome = st.stops_syndrome;
  t.stops_vnr = st.stops_vnr;
  t.stops_max_iter = st.stops_max_iter;
  t.hit_max_frames = st.hit_max_frames != 0;
  return t;
}

// ≙ etdec::decode (decoder.hpp:78-79): throwaway decoder.
inline DecodeOutcome decode(const ParityCheckMatrix& code, std::span<const double> llr_in, const ActiveVarSet& active,
                            const DecodeConfig& cfg) {
  BpDecoder d(code);
  return d.decode(llr_in, active, cfg);
}

}  // namespace bpdec::compat
