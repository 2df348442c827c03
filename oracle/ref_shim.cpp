// TEST INFRASTRUCTURE — not product code.
//
// extern "C" shim over the UNMODIFIED reference library (etdec_core), compiled
// from the sources where they lie under /root/reference/proj/core by
// oracle/Makefile into oracle/_ref/libetdec_ref.so.  Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference leg load it, as the checker and
// as the CPU baseline ("kind": "reference").
//
// Frames run in the reference's run_trials pattern (channel.cpp:98-122): one
// BpDecoder per std::thread, frames strided over threads.
#include <etdec/alist.hpp>
#include <etdec/channel.hpp>
#include <etdec/decoder.hpp>
#include <etdec/errors.hpp>
#include <etdec/parity_check_matrix.hpp>
#include <etdec/protograph.hpp>
#include <etdec/puncture.hpp>
#include <etdec/rng.hpp>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <thread>
#include <vector>

namespace {

void set_err(char* err, int len, const char* msg) {
  if (err && len > 0) {
    std::strncpy(err, msg, static_cast<size_t>(len) - 1);
    err[len - 1] = '\0';
  }
}

// 1 ConfigError, 2 IoError, 3 ValidationError, 6 other (errors.hpp:8-24)
int classify(const std::exception& e) {
  if (dynamic_cast<const etdec::ConfigError*>(&e)) return 1;
  if (dynamic_cast<const etdec::IoError*>(&e)) return 2;
  if (dynamic_cast<const etdec::ValidationError*>(&e)) return 3;
  return 6;
}

}  // namespace

extern "C" {

void* etref_code_create(int n_vars, int n_checks, const int* check_ptr, const int* check_vars, int* status,
                        char* err, int errlen) {
  try {
    std::vector<std::vector<int>> lists(n_checks);
    for (int c = 0; c < n_checks; ++c) lists[c].assign(check_vars + check_ptr[c], check_vars + check_ptr[c + 1]);
    auto* h = new etdec::ParityCheckMatrix(etdec::ParityCheckMatrix::from_check_lists(n_vars, lists));
    *status = 0;
    return h;
  } catch (const std::exception& e) {
    *status = classify(e);
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void* etref_code_load_alist(const char* path, int* status, char* err, int errlen) {
  try {
    auto* h = new etdec::ParityCheckMatrix(etdec::load_alist_file(path));
    *status = 0;
    return h;
  } catch (const std::exception& e) {
    *status = classify(e);
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

int etref_code_save_alist(const void* code, const char* path) {
  try {
    etdec::save_alist_file(*static_cast<const etdec::ParityCheckMatrix*>(code), path);
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

void* etref_lift_protograph(const int* base, int rows, int cols, int z, uint64_t seed, int* status, char* err,
                            int errlen) {
  try {
    etdec::BaseMatrix b(rows, std::vector<int>(cols));
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < cols; ++c) b[r][c] = base[r * cols + c];
    auto* h = new etdec::ParityCheckMatrix(etdec::lift_protograph(b, z, seed));
    *status = 0;
    return h;
  } catch (const std::exception& e) {
    *status = classify(e);
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void etref_code_destroy(void* code) { delete static_cast<etdec::ParityCheckMatrix*>(code); }

void etref_code_dims(const void* code, int* n_vars, int* n_checks, int* n_edges) {
  const auto& h = *static_cast<const etdec::ParityCheckMatrix*>(code);
  *n_vars = h.n_vars();
  *n_checks = h.n_checks();
  *n_edges = h.n_edges();
}

// CSR copy-out (check_ptr[M+1], check_vars[E]).
void etref_code_csr(const void* code, int* check_ptr, int* check_vars) {
  const auto& h = *static_cast<const etdec::ParityCheckMatrix*>(code);
  check_ptr[0] = 0;
  for (int c = 0; c < h.n_checks(); ++c) {
    const auto vars = h.check_vars(c);
    std::copy(vars.begin(), vars.end(), check_vars + h.edge_begin(c));
    check_ptr[c + 1] = h.edge_begin(c + 1);
  }
}

int etref_decode_batch(const void* code, int batch, const double* llr, int d_max, int use_pce, int use_vnr,
                       double msg_clamp, int threads, uint8_t* bits, int32_t* iterations, uint8_t* reasons,
                       double* posteriors, double* q_trace, char* err, int errlen) {
  const auto& h = *static_cast<const etdec::ParityCheckMatrix*>(code);
  const etdec::ActiveVarSet active = etdec::active_var_set(h);
  etdec::DecodeConfig cfg;
  cfg.d_max = d_max;
  cfg.use_pce = use_pce != 0;
  cfg.use_vnr = use_vnr != 0;
  cfg.msg_clamp = msg_clamp;
  const int n = h.n_vars();
  const int nt = std::max(1, std::min(threads, batch));
  std::vector<int> status(nt, 0);
  std::vector<std::string> msgs(nt);
  auto worker = [&](int w) {
    try {
      etdec::BpDecoder dec(h);
      for (int b = w; b < batch; b += nt) {
        const etdec::DecodeOutcome out =
            dec.decode(std::span<const double>(llr + static_cast<size_t>(b) * n, n), active, cfg);
        if (bits) std::copy(out.bits.begin(), out.bits.end(), bits + static_cast<size_t>(b) * n);
        if (posteriors) std::copy(out.posteriors.begin(), out.posteriors.end(), posteriors + static_cast<size_t>(b) * n);
        iterations[b] = out.iterations;
        reasons[b] = static_cast<uint8_t>(out.reason);
        if (q_trace) {
          double* q = q_trace + static_cast<size_t>(b) * d_max;
          std::fill(q, q + d_max, std::numeric_limits<double>::quiet_NaN());
          std::copy(out.q_trace.begin(), out.q_trace.end(), q);
        }
      }
    } catch (const std::exception& e) {
      status[w] = classify(e);
      msgs[w] = e.what();
    }
  };
  if (nt == 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w) pool.emplace_back(worker, w);
    for (auto& t : pool) t.join();
  }
  for (int w = 0; w < nt; ++w) {
    if (status[w] != 0) {
      set_err(err, errlen, msgs[w].c_str());
      return status[w];
    }
  }
  return 0;
}

// One frame with the IterationObserver attached (decoder.hpp:53-55): records
// per-iteration syndrome_ok and q (observer forces the syndrome computation).
int etref_decode_observed(const void* code, const double* llr, int d_max, int use_pce, int use_vnr,
                          double msg_clamp, int32_t* iterations, uint8_t* reason, uint8_t* syndrome_ok_trace,
                          double* q_trace, int32_t* observer_calls) {
  try {
    const auto& h = *static_cast<const etdec::ParityCheckMatrix*>(code);
    etdec::DecodeConfig cfg{d_max, use_pce != 0, use_vnr != 0, msg_clamp};
    etdec::BpDecoder dec(h);
    int calls = 0;
    auto obs = [&](int it, std::span<const double>, bool ok, double q) {
      syndrome_ok_trace[it - 1] = ok ? 1 : 0;
      q_trace[it - 1] = q;
      ++calls;
    };
    const auto out = dec.decode(std::span<const double>(llr, h.n_vars()), etdec::active_var_set(h), cfg, obs);
    *iterations = out.iterations;
    *reason = static_cast<uint8_t>(out.reason);
    *observer_calls = calls;
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// Same, also recording the observer's posteriors of every iteration
// (post_trace [d_max][n], rows past the stop untouched).
int etref_decode_observed_post(const void* code, const double* llr, int d_max, int use_pce, int use_vnr,
                               double msg_clamp, int32_t* iterations, uint8_t* reason, uint8_t* syndrome_ok_trace,
                               double* q_trace, double* post_trace, int32_t* observer_calls) {
  try {
    const auto& h = *static_cast<const etdec::ParityCheckMatrix*>(code);
    etdec::DecodeConfig cfg{d_max, use_pce != 0, use_vnr != 0, msg_clamp};
    etdec::BpDecoder dec(h);
    int calls = 0;
    const size_t n = static_cast<size_t>(h.n_vars());
    auto obs = [&](int it, std::span<const double> post, bool ok, double q) {
      syndrome_ok_trace[it - 1] = ok ? 1 : 0;
      q_trace[it - 1] = q;
      std::copy(post.begin(), post.end(), post_trace + static_cast<size_t>(it - 1) * n);
      ++calls;
    };
    const auto out = dec.decode(std::span<const double>(llr, h.n_vars()), etdec::active_var_set(h), cfg, obs);
    *iterations = out.iterations;
    *reason = static_cast<uint8_t>(out.reason);
    *observer_calls = calls;
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

int etref_syndrome_check(const void* code, const uint8_t* bits, int n) {
  try {
    return etdec::syndrome_check(*static_cast<const etdec::ParityCheckMatrix*>(code),
                                 std::span<const uint8_t>(bits, n))
               ? 1
               : 0;
  } catch (const std::exception& e) {
    return -classify(e);
  }
}

double etref_snr_for_beta(double beta, double rate) {
  try {
    return etdec::snr_for_beta(beta, rate).snr;
  } catch (const std::exception&) {
    return std::numeric_limits<double>::quiet_NaN();
  }
}

void etref_noise_normal(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  const etdec::NoiseStream ns(seed, stream);
  for (int64_t i = 0; i < count; ++i) out[i] = ns.normal(static_cast<uint64_t>(i));
}

// sample_block on the unpunctured code (channel.cpp:44-61).
void etref_sample_block(double snr, int n, uint64_t seed, uint64_t trial, double* llr) {
  etdec::ChannelPoint p;
  p.snr = snr;
  p.sigma2 = 1.0 / snr;
  etdec::PunctureMask mask;
  const auto blk = etdec::sample_block(p, n, mask, seed, trial);
  std::copy(blk.llrs.begin(), blk.llrs.end(), llr);
}

double etref_vnr_statistic(const double* posteriors, const int* members, int count) {
  etdec::ActiveVarSet a;
  a.members.assign(members, members + count);
  // vnr_statistic indexes posteriors by member id only
  int max_id = 0;
  for (int i = 0; i < count; ++i) max_id = std::max(max_id, members[i]);
  return etdec::vnr_statistic(std::span<const double>(posteriors, static_cast<size_t>(max_id) + 1), a);
}

// apply_puncture (puncture.cpp:16-48): writes positions, returns count (<0: -status)
int etref_apply_puncture(const void* code, double target_rate, uint64_t seed, int* out, double* eff) {
  try {
    const auto m = etdec::apply_puncture(*static_cast<const etdec::ParityCheckMatrix*>(code), target_rate, seed);
    std::copy(m.punctured.begin(), m.punctured.end(), out);
    *eff = m.effective_rate;
    return static_cast<int>(m.punctured.size());
  } catch (const std::exception& e) {
    return -classify(e);
  }
}

// run_trials (channel.cpp:74-156) with its own std::thread workers.
// stats: frames, errors, undetected, iteration_sum, stops_syn, stops_vnr,
// stops_max, hit_max (int64[8]); dstats: fer, ci_lo, ci_hi, d_bar (double[4]).
int etref_run_trials(const void* code, const int* punctured, int n_punct, double beta, int d_max, int use_pce,
                     int use_vnr, double clamp, long min_err, long max_frames, uint64_t seed, int workers,
                     int64_t* stats, double* dstats, int64_t* hist, int hist_len) {
  try {
    const auto& h = *static_cast<const etdec::ParityCheckMatrix*>(code);
    etdec::PunctureMask mask;
    mask.punctured.assign(punctured, punctured + n_punct);
    const auto point = etdec::snr_for_beta(beta, h.rate());
    etdec::DecodeConfig cfg{d_max, use_pce != 0, use_vnr != 0, clamp};
    etdec::StopRule stop{min_err, max_frames};
    const auto st = etdec::run_trials(h, mask, point, cfg, stop, seed, workers);
    stats[0] = st.frames;
    stats[1] = st.frame_errors;
    stats[2] = st.undetected_errors;
    stats[3] = st.iteration_sum;
    stats[4] = st.stops_syndrome;
    stats[5] = st.stops_vnr;
    stats[6] = st.stops_max_iter;
    stats[7] = st.hit_max_frames ? 1 : 0;
    dstats[0] = st.fer;
    dstats[1] = st.fer_ci_low;
    dstats[2] = st.fer_ci_high;
    dstats[3] = st.d_bar;
    for (const auto& [k, v] : st.iteration_histogram)
      if (k >= 0 && k < hist_len) hist[k] = v;
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

}  // extern "C"
