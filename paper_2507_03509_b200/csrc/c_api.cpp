// C ABI (include/bpdec.h).  Every entry point catches C++ exceptions and maps
// them to bpdec_status codes mirroring the reference's exception classes
// (errors.hpp:8-24); the message is kept per thread for bpdec_last_error().
#include "../../include/bpdec.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <deque>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "code.hpp"
#include "decoder.hpp"
#include "devmem.hpp"
#include "harness.hpp"
#include "rng.hpp"

struct bpdec_code {
  bpdec::Code code;
};
struct bpdec_decoder {
  bpdec::GpuDecoder* impl = nullptr;
  int32_t n_vars = 0;
  int32_t n_checks = 0;
};
// Multi-device decoder: one GpuDecoder per entry of the device list, each
// fed by its own host thread from a shared chunk queue (streams stay open
// between calls while the configuration is unchanged).
struct bpdec_multi {
  std::vector<bpdec::GpuDecoder*> decs;
  std::vector<int32_t> devices;
  int32_t n_vars = 0, n_checks = 0, slots = 0;
  bool open = false;
  bpdec::DecodeParams p{};
  uint32_t flags = 0;
  bool want_bits = false, want_post = false, want_q = false;
  int32_t ring = 0;
  std::vector<int64_t> frames_taken;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
#ifdef BPDEC_GUARD
    // guard build: every entry point ends with the guard-zone check of all
    // live device allocations (devmem.hpp)
    const char* where = nullptr;
    if (bpdec::dev_verify(&where) != cudaSuccess)
      throw bpdec::CudaError(std::string("guard build: ") + (where ? where : "device error during verify"));
#endif
    g_last_error.clear();
    return BPDEC_OK;
  } catch (const bpdec::ConfigError& e) {
    g_last_error = e.what();
    return BPDEC_ERR_CONFIG;
  } catch (const bpdec::IoError& e) {
    g_last_error = e.what();
    return BPDEC_ERR_IO;
  } catch (const bpdec::ValidationError& e) {
    g_last_error = e.what();
    return BPDEC_ERR_VALIDATION;
  } catch (const bpdec::CudaError& e) {
    g_last_error = e.what();
    return BPDEC_ERR_CUDA;
  } catch (const bpdec::OomError& e) {
    g_last_error = e.what();
    return BPDEC_ERR_OOM;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return BPDEC_ERR_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BPDEC_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown error";
    return BPDEC_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (p == nullptr) throw bpdec::ValidationError(std::string("null pointer: ") + what);
}

int host_threads() {
  const unsigned n = std::thread::hardware_concurrency();
  return n == 0 ? 1 : static_cast<int>(n);
}

// ≙ snr_for_beta (channel.cpp:29-42).
double snr_for_beta_impl(double beta, double rate) {
  if (!(beta > 0.0) || beta > 1.0) {
    throw bpdec::ValidationError("snr_for_beta: beta must lie in (0,1], got " + std::to_string(beta));
  }
  if (!(rate > 0.0) || rate >= 1.0) {
    throw bpdec::ValidationError("snr_for_beta: rate must lie in (0,1), got " + std::to_string(rate));
  }
  return std::exp2(2.0 * rate / beta) - 1.0;
}

}  // namespace

extern "C" {

int bpdec_abi_version(void) { return BPDEC_ABI_VERSION; }

const char* bpdec_last_error(void) { return g_last_error.c_str(); }

const char* bpdec_stop_reason_name(int32_t reason) {
  switch (reason) {
    case BPDEC_STOP_SYNDROME: return "syndrome_satisfied";
    case BPDEC_STOP_VNR: return "vnr_drop";
    case BPDEC_STOP_MAX_ITER: return "max_iterations";
    default: return "unknown";
  }
}

int bpdec_code_from_csr(int32_t n_vars, int32_t n_checks, const int32_t* check_ptr,
                        const int32_t* check_vars, bpdec_code** out) {
  return guarded([&] {
    need(out, "out");
    auto* c = new bpdec_code{bpdec::Code::from_csr(n_vars, n_checks, check_ptr, check_vars)};
    *out = c;
  });
}

int bpdec_code_load_alist(const char* path, bpdec_code** out) {
  return guarded([&] {
    need(path, "path");
    need(out, "out");
    *out = new bpdec_code{bpdec::load_alist_file(path)};
  });
}

int bpdec_code_save_alist(const bpdec_code* code, const char* path) {
  return guarded([&] {
    need(code, "code");
    need(path, "path");
    bpdec::save_alist_file(code->code, path);
  });
}

int bpdec_code_lift_protograph(const int32_t* base, int32_t rows, int32_t cols, int32_t z,
                               uint64_t seed, bpdec_code** out) {
  return guarded([&] {
    need(out, "out");
    if (rows <= 0 || cols <= 0) throw bpdec::ValidationError("protograph lift: empty base matrix");
    need(base, "base");
    std::vector<std::vector<int32_t>> b(rows, std::vector<int32_t>(cols));
    for (int32_t r = 0; r < rows; ++r)
      for (int32_t c = 0; c < cols; ++c) b[r][c] = base[static_cast<size_t>(r) * cols + c];
    *out = new bpdec_code{bpdec::lift_protograph(b, z, seed)};
  });
}

int bpdec_code_generate_met(int32_t n_vars, int32_t n_checks, double frac_deg1, int32_t n_classes,
                            const int32_t* degrees, const double* probs, uint64_t seed,
                            bpdec_code** out) {
  return guarded([&] {
    need(out, "out");
    if (n_classes <= 0) throw bpdec::ValidationError("met generator: need at least one degree class");
    need(degrees, "degrees");
    need(probs, "probs");
    std::vector<int32_t> d(degrees, degrees + n_classes);
    std::vector<double> p(probs, probs + n_classes);
    *out = new bpdec_code{bpdec::generate_met(n_vars, n_checks, frac_deg1, d, p, seed)};
  });
}

int bpdec_code_generate_met_core(int32_t n_vars, int32_t n_checks, int32_t n_deg1, int32_t n_classes,
                                 const int32_t* core_degrees, const double* core_probs, int32_t ext_degree,
                                 uint64_t seed, bpdec_code** out) {
  return guarded([&] {
    need(out, "out");
    if (n_classes <= 0) throw bpdec::ValidationError("met core generator: need at least one degree class");
    need(core_degrees, "core_degrees");
    need(core_probs, "core_probs");
    std::vector<int32_t> d(core_degrees, core_degrees + n_classes);
    std::vector<double> p(core_probs, core_probs + n_classes);
    *out = new bpdec_code{bpdec::generate_met_core(n_vars, n_checks, n_deg1, d, p, ext_degree, seed)};
  });
}

void bpdec_code_destroy(bpdec_code* code) { delete code; }

int bpdec_code_dims(const bpdec_code* code, int32_t* n_vars, int32_t* n_checks, int64_t* n_edges,
                    int32_t* n_active) {
  return guarded([&] {
    need(code, "code");
    const auto& h = code->code;
    if (n_vars) *n_vars = h.n_vars;
    if (n_checks) *n_checks = h.n_checks;
    if (n_edges) *n_edges = h.n_edges();
    if (n_active) {
      int32_t k = 0;
      for (int32_t v = 0; v < h.n_vars; ++v) k += h.var_degree(v) >= 2 ? 1 : 0;
      *n_active = k;
    }
  });
}

int bpdec_code_csr(const bpdec_code* code, int32_t* check_ptr, int32_t* check_vars) {
  return guarded([&] {
    need(code, "code");
    const auto& h = code->code;
    if (check_ptr) std::copy(h.check_ptr.begin(), h.check_ptr.end(), check_ptr);
    if (check_vars) std::copy(h.check_vars.begin(), h.check_vars.end(), check_vars);
  });
}

int bpdec_code_active_vars(const bpdec_code* code, int32_t* members) {
  return guarded([&] {
    need(code, "code");
    need(members, "members");
    const auto v = bpdec::active_var_set(code->code);
    std::copy(v.begin(), v.end(), members);
  });
}

int bpdec_code_syndrome(const bpdec_code* code, int32_t n_frames, const uint8_t* bits,
                        uint32_t* syndrome_out) {
  return guarded([&] {
    need(code, "code");
    if (n_frames < 0) throw bpdec::ValidationError("syndrome: n_frames must be non-negative");
    if (n_frames == 0) return;
    need(bits, "bits");
    need(syndrome_out, "syndrome_out");
    const auto& h = code->code;
    const size_t mw = (h.n_checks + 31) / 32;
    for (int32_t f = 0; f < n_frames; ++f) {
      bpdec::compute_syndrome(h, bits + static_cast<size_t>(f) * h.n_vars, syndrome_out + f * mw);
    }
  });
}

int bpdec_syndrome_check(const bpdec_code* code, const uint8_t* bits, const uint32_t* syndrome,
                         int32_t* ok) {
  return guarded([&] {
    need(code, "code");
    need(bits, "bits");
    need(ok, "ok");
    const auto& h = code->code;
    *ok = 1;
    for (int32_t c = 0; c < h.n_checks; ++c) {
      uint32_t p = 0;
      for (int32_t e = h.check_ptr[c]; e < h.check_ptr[c + 1]; ++e) p ^= bits[h.check_vars[e]] & 1u;
      const uint32_t target = syndrome ? (syndrome[c >> 5] >> (c & 31)) & 1u : 0u;
      if (p != target) {
        *ok = 0;
        return;
      }
    }
  });
}

int bpdec_snr_for_beta(double beta, double rate, double* snr) {
  return guarded([&] {
    need(snr, "snr");
    *snr = snr_for_beta_impl(beta, rate);
  });
}

}  // extern "C"

namespace {

// Seeded syndrome-mode frames on the host (threaded).  snr_of(f) gives the
// channel SNR of global frame f.
template <typename SnrOf>
void sample_frames_impl(const bpdec::Code& h, SnrOf snr_of, uint64_t seed, int64_t first_frame, int32_t n_frames,
                        int32_t all_zero, float* llr_out, uint8_t* x_out, uint32_t* syndrome_out, double* snr_out) {
  if (n_frames < 0) throw bpdec::ValidationError("sample: n_frames must be non-negative");
  need(llr_out, "llr_out");
  const int32_t n = h.n_vars;
  const size_t mw = (h.n_checks + 31) / 32;
  auto work = [&](int32_t b) {
    const uint64_t f = static_cast<uint64_t>(first_frame + b);
    // sample_block's arithmetic (channel.cpp:51-58) with the BPSK sign of x.
    const double snr = snr_of(f);
    const double sigma2 = 1.0 / snr;
    const double sigma = std::sqrt(sigma2);
    const double scale = 2.0 / sigma2;
    if (snr_out) snr_out[b] = snr;
    const uint64_t nkey = bpdec::stream_key(bpdec::kNoiseDomain, seed, f);
    const uint64_t xkey = bpdec::stream_key(bpdec::kBitDomain, seed, f);
    std::vector<uint8_t> x(n);
    float* l = llr_out + static_cast<size_t>(b) * n;
    for (int32_t i = 0; i < n; ++i) {
      double u1, u2;
      bpdec::noise_uniforms(nkey, static_cast<uint64_t>(i), &u1, &u2);
      const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
      const unsigned xi = all_zero ? 0u : bpdec::message_bit(xkey, static_cast<uint64_t>(i));
      x[i] = static_cast<uint8_t>(xi);
      l[i] = static_cast<float>(scale * ((xi ? -1.0 : 1.0) + sigma * g));
    }
    if (x_out) std::copy(x.begin(), x.end(), x_out + static_cast<size_t>(b) * n);
    if (syndrome_out) bpdec::compute_syndrome(h, x.data(), syndrome_out + b * mw);
  };
  const int nt = std::max(1, std::min(host_threads(), n_frames));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) {
    pool.emplace_back([&, t] {
      for (int32_t b = t; b < n_frames; b += nt) work(b);
    });
  }
  for (auto& th : pool) th.join();
}

void check_beta_range(double lo, double hi) {
  if (!(lo > 0.0) || hi > 1.0 || hi < lo) {
    throw bpdec::ValidationError("sample: need 0 < beta_lo <= beta_hi <= 1");
  }
}

}  // namespace

extern "C" {

int bpdec_sample_frames(const bpdec_code* code, double snr, uint64_t seed, int64_t first_frame,
                        int32_t n_frames, int32_t all_zero, float* llr_out, uint8_t* x_out,
                        uint32_t* syndrome_out) {
  return guarded([&] {
    need(code, "code");
    if (!(snr > 0.0) || !std::isfinite(snr)) throw bpdec::ValidationError("sample: snr must be positive and finite");
    sample_frames_impl(code->code, [snr](uint64_t) { return snr; }, seed, first_frame, n_frames, all_zero, llr_out,
                       x_out, syndrome_out, nullptr);
  });
}

int bpdec_sample_frames_beta(const bpdec_code* code, double beta_lo, double beta_hi, uint64_t seed,
                             int64_t first_frame, int32_t n_frames, int32_t all_zero, float* llr_out, uint8_t* x_out,
                             uint32_t* syndrome_out, double* snr_out) {
  return guarded([&] {
    need(code, "code");
    check_beta_range(beta_lo, beta_hi);
    const double rate = code->code.rate();
    sample_frames_impl(
        code->code,
        [=](uint64_t f) { return std::exp2(2.0 * rate / bpdec::frame_beta(seed, f, beta_lo, beta_hi)) - 1.0; }, seed,
        first_frame, n_frames, all_zero, llr_out, x_out, syndrome_out, snr_out);
  });
}

int bpdec_decoder_create(const bpdec_code* code, int32_t device, int32_t max_slots,
                         bpdec_decoder** out) {
  return guarded([&] {
    need(code, "code");
    need(out, "out");
    auto* d = new bpdec_decoder;
    try {
      d->impl = bpdec::gpu_decoder_create(code->code, device, max_slots);
    } catch (...) {
      delete d;
      throw;
    }
    d->n_vars = code->code.n_vars;
    d->n_checks = code->code.n_checks;
    *out = d;
  });
}

void bpdec_decoder_destroy(bpdec_decoder* dec) {
  if (!dec) return;
  bpdec::gpu_decoder_destroy(dec->impl);
  delete dec;
}

int bpdec_decoder_slots(const bpdec_decoder* dec, int32_t* slots) {
  return guarded([&] {
    need(dec, "decoder");
    need(slots, "slots");
    *slots = bpdec::gpu_decoder_slots(dec->impl);
  });
}

int bpdec_decoder_device_bytes(const bpdec_decoder* dec, int64_t* bytes) {
  return guarded([&] {
    need(dec, "decoder");
    need(bytes, "bytes");
    *bytes = bpdec::gpu_decoder_device_bytes(dec->impl);
  });
}

}  // extern "C"

namespace {
// DecodeConfig validation (decoder.cpp:56-64) and translation.
bpdec::DecodeParams decode_params(const bpdec_config* cfg) {
  need(cfg, "cfg");
  if (cfg->d_max <= 0) throw bpdec::ValidationError("decode: d_max must be positive");
  if (!(cfg->msg_clamp > 0.0)) throw bpdec::ValidationError("decode: msg_clamp must be positive");
  if (cfg->q_mode != BPDEC_Q_RAW && cfg->q_mode != BPDEC_Q_ABS) throw bpdec::ConfigError("decode: unknown q_mode");
  bpdec::DecodeParams p;
  p.d_max = cfg->d_max;
  p.use_pce = cfg->use_pce ? 1 : 0;
  p.use_vnr = cfg->use_vnr ? 1 : 0;
  p.q_mode = cfg->q_mode;
  p.msg_clamp = static_cast<float>(cfg->msg_clamp);
  return p;
}
}  // namespace

extern "C" {

int bpdec_decode_batch_traced(bpdec_decoder* dec, int32_t batch, const float* llr, const uint32_t* syndrome,
                              const bpdec_config* cfg, uint32_t flags, void* bits_out, int32_t* iterations_out,
                              uint8_t* reason_out, float* posteriors_out, double* q_trace_out,
                              uint8_t* syndrome_ok_trace_out, float* posterior_trace_out, void* stream) {
  return guarded([&] {
    need(dec, "decoder");
    const bpdec::DecodeParams p = decode_params(cfg);
    bpdec::DecodeBuffers b;
    b.batch = batch;
    b.llr = llr;
    b.syndrome = syndrome;
    b.bits_packed = (flags & BPDEC_BITS_PACKED) != 0;
    b.bits = bits_out;
    b.iterations = iterations_out;
    b.reasons = reason_out;
    b.posteriors = posteriors_out;
    b.q_trace = q_trace_out;
    b.syn_trace = syndrome_ok_trace_out;
    b.post_trace = posterior_trace_out;
    bpdec::gpu_decode_batch(dec->impl, p, b, stream);
  });
}

int bpdec_decode_batch(bpdec_decoder* dec, int32_t batch, const float* llr, const uint32_t* syndrome,
                       const bpdec_config* cfg, uint32_t flags, void* bits_out, int32_t* iterations_out,
                       uint8_t* reason_out, float* posteriors_out, double* q_trace_out, void* stream) {
  return guarded([&] {
    need(dec, "decoder");
    const bpdec::DecodeParams p = decode_params(cfg);
    bpdec::DecodeBuffers b;
    b.batch = batch;
    b.llr = llr;
    b.syndrome = syndrome;
    b.bits_packed = (flags & BPDEC_BITS_PACKED) != 0;
    b.bits = bits_out;
    b.iterations = iterations_out;
    b.reasons = reason_out;
    b.posteriors = posteriors_out;
    b.q_trace = q_trace_out;
    bpdec::gpu_decode_batch(dec->impl, p, b, stream);
  });
}

int bpdec_decoder_sample_frames_device(bpdec_decoder* dec, double snr, uint64_t seed, int64_t first_frame,
                                       int32_t n_frames, int32_t all_zero, float* d_llr, uint32_t* d_syndrome,
                                       uint32_t* d_x_packed, void* stream) {
  return guarded([&] {
    need(dec, "decoder");
    need(d_llr, "d_llr");
    if (!(snr > 0.0) || !std::isfinite(snr)) throw bpdec::ValidationError("sample: snr must be positive and finite");
    bpdec::gpu_sample_frames_device(dec->impl, snr, 0.0, 0.0, 0.0, seed, first_frame, n_frames, all_zero != 0, d_llr,
                                    d_syndrome, d_x_packed, stream);
  });
}

int bpdec_decoder_sample_frames_beta_device(bpdec_decoder* dec, double beta_lo, double beta_hi, uint64_t seed,
                                            int64_t first_frame, int32_t n_frames, int32_t all_zero, float* d_llr,
                                            uint32_t* d_syndrome, uint32_t* d_x_packed, void* stream) {
  return guarded([&] {
    need(dec, "decoder");
    need(d_llr, "d_llr");
    check_beta_range(beta_lo, beta_hi);
    const double rate = static_cast<double>(dec->n_vars - dec->n_checks) / dec->n_vars;
    bpdec::gpu_sample_frames_device(dec->impl, 0.0, beta_lo, beta_hi, rate, seed, first_frame, n_frames,
                                    all_zero != 0, d_llr, d_syndrome, d_x_packed, stream);
  });
}

int bpdec_code_apply_puncture(const bpdec_code* code, double target_rate, uint64_t seed, int32_t* punctured_out,
                              int32_t* count, double* effective_rate) {
  return guarded([&] {
    need(code, "code");
    need(count, "count");
    double eff = 0.0;
    const auto v = bpdec::apply_puncture(code->code, target_rate, seed, &eff);
    if (!v.empty()) {
      need(punctured_out, "punctured_out");
      std::copy(v.begin(), v.end(), punctured_out);
    }
    *count = static_cast<int32_t>(v.size());
    if (effective_rate) *effective_rate = eff;
  });
}

int bpdec_wilson_interval(int64_t k, int64_t n, double* lo, double* hi) {
  return guarded([&] {
    if (n <= 0 || k < 0 || k > n) throw bpdec::ValidationError("wilson_interval: need 0 <= k <= n, n > 0");
    const auto ci = bpdec::wilson_interval(k, n);
    if (lo) *lo = ci.first;
    if (hi) *hi = ci.second;
  });
}

int bpdec_run_trials(bpdec_decoder* dec, double snr, const int32_t* punctured, int32_t n_punctured,
                     const bpdec_config* cfg, const bpdec_stop_rule* stop, uint64_t seed, int32_t block,
                     bpdec_trial_stats* stats_out, int64_t* histogram_out) {
  return guarded([&] {
    need(dec, "decoder");
    need(cfg, "cfg");
    need(stop, "stop");
    need(stats_out, "stats_out");
    const bpdec::DecodeParams p = decode_params(cfg);
    std::vector<int32_t> punct;
    if (n_punctured > 0) {
      need(punctured, "punctured");
      punct.assign(punctured, punctured + n_punctured);
    }
    const auto st = bpdec::run_trials(dec->impl, dec->n_vars, dec->n_checks, snr, punct, p, stop->min_frame_errors,
                                      stop->max_frames, seed, block);
    bpdec_trial_stats o{};
    o.frames = st.frames;
    o.frame_errors = st.frame_errors;
    o.undetected_errors = st.undetected_errors;
    o.fer = st.fer;
    o.fer_ci_low = st.fer_ci_low;
    o.fer_ci_high = st.fer_ci_high;
    o.d_bar = st.d_bar;
    o.iteration_sum = st.iteration_sum;
    o.stops_syndrome = st.stops_syndrome;
    o.stops_vnr = st.stops_vnr;
    o.stops_max_iter = st.stops_max_iter;
    o.hit_max_frames = st.hit_max_frames ? 1 : 0;
    *stats_out = o;
    if (histogram_out) std::copy(st.histogram.begin(), st.histogram.end(), histogram_out);
  });
}

int bpdec_decoder_stage_inputs(bpdec_decoder* dec, int32_t batch, const float* llr_host,
                               const uint32_t* syndrome_host) {
  return guarded([&] {
    need(dec, "decoder");
    bpdec::gpu_stage_inputs(dec->impl, batch, llr_host, syndrome_host);
  });
}

int bpdec_decoder_set_profiling(bpdec_decoder* dec, int32_t enable) {
  return guarded([&] {
    need(dec, "decoder");
    bpdec::gpu_set_profiling(dec->impl, enable != 0);
  });
}

int bpdec_decoder_profile(const bpdec_decoder* dec, int32_t kernel, double* total_ms, int64_t* launches,
                          double* frame_iterations) {
  return guarded([&] {
    need(dec, "decoder");
    bpdec::gpu_profile(dec->impl, kernel, total_ms, launches, frame_iterations);
  });
}

int bpdec_decoder_reset_profile(bpdec_decoder* dec) {
  return guarded([&] {
    need(dec, "decoder");
    bpdec::gpu_reset_profile(dec->impl);
  });
}

int bpdec_decoder_launch_count(const bpdec_decoder* dec, int64_t* launches) {
  return guarded([&] {
    need(dec, "decoder");
    need(launches, "launches");
    *launches = bpdec::gpu_launch_count(dec->impl);
  });
}

/* ------------------------------------------------------------ stream mode -- */
int bpdec_stream_open(bpdec_decoder* dec, const bpdec_config* cfg, uint32_t flags, int32_t ring_frames,
                      int32_t want_bits, int32_t want_posteriors, int32_t want_q_trace) {
  return guarded([&] {
    need(dec, "decoder");
    const bpdec::DecodeParams p = decode_params(cfg);
    bpdec::gpu_stream_open(dec->impl, p, (flags & BPDEC_BITS_PACKED) != 0, want_bits != 0, want_posteriors != 0,
                           want_q_trace != 0, ring_frames);
  });
}

int bpdec_stream_submit(bpdec_decoder* dec, int32_t batch, const float* llr, const uint32_t* syndrome,
                        void* bits_out, int32_t* iterations_out, uint8_t* reason_out, float* posteriors_out,
                        double* q_trace_out, int64_t* ticket_out) {
  return guarded([&] {
    need(dec, "decoder");
    need(ticket_out, "ticket_out");
    bpdec::StreamOutputs o;
    o.bits = bits_out;
    o.iterations = iterations_out;
    o.reasons = reason_out;
    o.posteriors = posteriors_out;
    o.q_trace = q_trace_out;
    *ticket_out = bpdec::gpu_stream_submit(dec->impl, batch, llr, syndrome, o);
  });
}

int bpdec_stream_query(bpdec_decoder* dec, int64_t ticket, int32_t* done) {
  return guarded([&] {
    need(dec, "decoder");
    need(done, "done");
    *done = bpdec::gpu_stream_query(dec->impl, ticket) ? 1 : 0;
  });
}

int bpdec_stream_wait(bpdec_decoder* dec, int64_t ticket) {
  return guarded([&] {
    need(dec, "decoder");
    bpdec::gpu_stream_wait(dec->impl, ticket);
  });
}

int bpdec_stream_close(bpdec_decoder* dec) {
  return guarded([&] {
    need(dec, "decoder");
    bpdec::gpu_stream_close(dec->impl);
  });
}

int bpdec_stream_timer_reset(bpdec_decoder* dec) {
  return guarded([&] {
    need(dec, "decoder");
    bpdec::gpu_stream_timer_reset(dec->impl);
  });
}

int bpdec_stream_device_ms(bpdec_decoder* dec, double* ms) {
  return guarded([&] {
    need(dec, "decoder");
    need(ms, "ms");
    *ms = bpdec::gpu_stream_device_ms(dec->impl);
  });
}

/* ------------------------------------------------------------ multi-GPU -- */
int bpdec_multi_create(const bpdec_code* code, const int32_t* devices, int32_t n_devices, int32_t slots_per_decoder,
                       bpdec_multi** out) {
  return guarded([&] {
    need(code, "code");
    need(out, "out");
    if (n_devices <= 0) throw bpdec::ValidationError("multi: need at least one device");
    need(devices, "devices");
    auto* m = new bpdec_multi;
    try {
      for (int32_t i = 0; i < n_devices; ++i) {
        m->decs.push_back(bpdec::gpu_decoder_create(code->code, devices[i], slots_per_decoder));
        m->devices.push_back(devices[i]);
      }
    } catch (...) {
      for (auto* d : m->decs) bpdec::gpu_decoder_destroy(d);
      delete m;
      throw;
    }
    m->n_vars = code->code.n_vars;
    m->n_checks = code->code.n_checks;
    m->slots = bpdec::gpu_decoder_slots(m->decs[0]);
    m->frames_taken.assign(m->decs.size(), 0);
    *out = m;
  });
}

void bpdec_multi_destroy(bpdec_multi* m) {
  if (!m) return;
  for (auto* d : m->decs) {
    try {
      bpdec::gpu_stream_close(d);
    } catch (...) {
    }
    bpdec::gpu_decoder_destroy(d);
  }
  delete m;
}

int bpdec_multi_count(const bpdec_multi* m, int32_t* n_decoders) {
  return guarded([&] {
    need(m, "multi");
    need(n_decoders, "n_decoders");
    *n_decoders = static_cast<int32_t>(m->decs.size());
  });
}

int bpdec_multi_decode_batch(bpdec_multi* m, int32_t batch, const float* llr, const uint32_t* syndrome,
                             const bpdec_config* cfg, uint32_t flags, void* bits_out, int32_t* iterations_out,
                             uint8_t* reason_out, float* posteriors_out, double* q_trace_out, int32_t chunk_frames,
                             int64_t* frames_per_decoder_out) {
  return guarded([&] {
    need(m, "multi");
    const bpdec::DecodeParams p = decode_params(cfg);
    if (batch < 0) throw bpdec::ValidationError("decode: batch must be non-negative");
    if (batch == 0) return;
    need(llr, "llr");
    need(iterations_out, "iterations_out");
    need(reason_out, "reason_out");
    const int nd = static_cast<int>(m->decs.size());
    const int32_t chunk = chunk_frames > 0 ? chunk_frames
                                           : std::max<int32_t>(32, std::min<int32_t>(m->slots, (batch + 4 * nd - 1) / (4 * nd)));
    const bool packed = (flags & BPDEC_BITS_PACKED) != 0;
    const bool wb = bits_out != nullptr, wp = posteriors_out != nullptr, wq = q_trace_out != nullptr;
    const int32_t ring = std::max(3 * chunk, m->slots + 2 * chunk);
    // (re)open the per-decoder streams when the configuration changed
    const bool same = m->open && m->p.d_max == p.d_max && m->p.use_pce == p.use_pce && m->p.use_vnr == p.use_vnr &&
                      m->p.q_mode == p.q_mode && m->p.msg_clamp == p.msg_clamp && m->flags == flags &&
                      m->want_bits == wb && m->want_post == wp && m->want_q == wq && m->ring >= ring;
    if (!same) {
      for (auto* d : m->decs) bpdec::gpu_stream_close(d);
      m->open = false;
      for (auto* d : m->decs) bpdec::gpu_stream_open(d, p, packed, wb, wp, wq, ring);
      m->open = true;
      m->p = p;
      m->flags = flags;
      m->want_bits = wb;
      m->want_post = wp;
      m->want_q = wq;
      m->ring = ring;
    }
    const int64_t nchunks = (static_cast<int64_t>(batch) + chunk - 1) / chunk;
    const size_t N = static_cast<size_t>(m->n_vars), MW = (static_cast<size_t>(m->n_checks) + 31) / 32;
    const size_t row_bits = packed ? (N + 31) / 32 * sizeof(uint32_t) : N;
    std::atomic<int64_t> next{0};
    std::mutex err_mu;
    std::string err;
    int err_kind = 0;
    std::vector<int64_t> taken(nd, 0);
    auto worker = [&](int k) {
      bpdec::GpuDecoder* d = m->decs[k];
      std::deque<int64_t> inflight;
      try {
        for (;;) {
          // two chunks in flight per decoder: the next one's upload overlaps
          // the current one's decode, and its frames fill the tail's lanes
          while (inflight.size() < 2) {
            const int64_t c = next.fetch_add(1);
            if (c >= nchunks) break;
            const size_t f0 = static_cast<size_t>(c) * chunk;
            const int32_t nf = static_cast<int32_t>(std::min<int64_t>(chunk, batch - static_cast<int64_t>(f0)));
            bpdec::StreamOutputs o;
            o.bits = wb ? static_cast<char*>(bits_out) + f0 * row_bits : nullptr;
            o.iterations = iterations_out + f0;
            o.reasons = reason_out + f0;
            o.posteriors = wp ? posteriors_out + f0 * N : nullptr;
            o.q_trace = wq ? q_trace_out + f0 * static_cast<size_t>(p.d_max) : nullptr;
            inflight.push_back(bpdec::gpu_stream_submit(d, nf, llr + f0 * N, syndrome ? syndrome + f0 * MW : nullptr, o));
            taken[k] += nf;
          }
          if (inflight.empty()) break;
          bpdec::gpu_stream_wait(d, inflight.front());
          inflight.pop_front();
        }
      } catch (const bpdec::ValidationError& e) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (err.empty()) err = e.what(), err_kind = 3;
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (err.empty()) err = e.what(), err_kind = 4;
      }
      for (int64_t t : inflight) {  // drain after an error
        try {
          bpdec::gpu_stream_wait(d, t);
        } catch (...) {
        }
      }
    };
    std::vector<std::thread> th;
    for (int k = 0; k < nd; ++k) th.emplace_back(worker, k);
    for (auto& t : th) t.join();
    for (int k = 0; k < nd; ++k) m->frames_taken[k] += taken[k];
    if (frames_per_decoder_out) std::copy(taken.begin(), taken.end(), frames_per_decoder_out);
    if (err_kind == 3) throw bpdec::ValidationError(err);
    if (err_kind) throw bpdec::CudaError(err);
  });
}

}  // extern "C"
