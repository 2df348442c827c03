// C++ host-layer test: the reference-shaped API (include/bpdec/etdec_compat.hpp)
// over libbpdec.so, written the way a reference caller would use etdec.
// Exit code 0 = pass.  Without a GPU, only the host-side parts run and the
// decoder construction must fail with DeviceError (no CPU fallback).
#include <bpdec/etdec_compat.hpp>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

namespace ed = bpdec::compat;

#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      return 1;                                                       \
    }                                                                 \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  // code model + errors (parity_check_matrix.cpp:10-62)
  const auto h = ed::ParityCheckMatrix::from_check_lists(3, {{0, 1, 2}});
  CHECK(h.n_vars() == 3 && h.n_checks() == 1 && h.n_edges() == 3);
  bool threw = false;
  try {
    ed::ParityCheckMatrix::from_check_lists(3, {{0, 0}});
  } catch (const ed::ValidationError&) {
    threw = true;
  }
  CHECK(threw);
  const std::vector<std::uint8_t> ok_word = {1, 1, 0};
  CHECK(ed::syndrome_check(h, ok_word));
  const ed::ChannelPoint pt = ed::snr_for_beta(0.95, 0.1);  // channel.hpp:14-23
  CHECK(std::fabs(pt.snr - 0.15711023728271978) < 1e-15 && pt.beta == 0.95 && pt.rate == 0.1);
  CHECK(std::fabs(pt.sigma2 * pt.snr - 1.0) < 1e-15);
  const auto wi = ed::wilson_interval(0, 10);  // channel.cpp:63-72
  CHECK(wi.first == 0.0 && wi.second > 0.27 && wi.second < 0.28);
  const auto lift = ed::lift_protograph({{3, 3}}, 1024, 1);
  CHECK(lift.n_vars() == 2048 && lift.n_checks() == 1024 && lift.n_edges() == 6144);
  CHECK(ed::active_var_set(lift).members.size() == 2048);
  CHECK(std::strcmp(ed::to_string(ed::StopReason::kVnrDrop), "vnr_drop") == 0);
  // puncturing (puncture.cpp:16-48): round(N - (N-M)/target) degree>=2 positions
  const auto pm = ed::apply_puncture(lift, 0.6, 3);
  CHECK(pm.punctured.size() == static_cast<size_t>(std::lround(2048 - 1024 / 0.6)));
  CHECK(ed::no_puncture(lift).empty() && std::fabs(ed::no_puncture(lift).effective_rate - 0.5) < 1e-15);
  // FER < 1 family generator
  const auto met = ed::generate_met_core(8192, 7373, 5734, {2, 3}, {0.5, 0.5}, 2, 1);
  CHECK(met.n_vars() == 8192 && met.n_checks() == 7373);

  if (!gpu) {
    bool dev_err = false;
    try {
      ed::BpDecoder d(h);
    } catch (const ed::DeviceError&) {
      dev_err = true;
    }
    CHECK(dev_err);
    std::printf("compat_test (host) OK\n");
    return 0;
  }
  // decode on the GPU: SPEC.md:140 known answer
  ed::DecodeConfig cfg;
  cfg.d_max = 1;
  cfg.use_pce = false;
  ed::BpDecoder dec(h);
  const std::vector<double> llr = {2.0, 2.0, -0.5};
  const auto out = dec.decode(llr, ed::active_var_set(h), cfg);
  CHECK(out.iterations == 1 && out.reason == ed::StopReason::kMaxIterations);
  CHECK(std::fabs(out.posteriors[2] - 0.82500274735786427) < 2e-6);
  CHECK(out.bits == std::vector<std::uint8_t>({0, 0, 0}));
  // noiseless frame terminates at iteration 1
  const auto o2 = ed::decode(h, std::vector<double>{50, 50, 50}, ed::active_var_set(h), ed::DecodeConfig{});
  CHECK(o2.iterations == 1 && o2.converged());
  // invalid input -> ValidationError (decoder.cpp:60-62)
  threw = false;
  try {
    dec.decode(std::vector<double>{1.0, NAN, 1.0}, ed::active_var_set(h), cfg);
  } catch (const ed::ValidationError&) {
    threw = true;
  }
  CHECK(threw);
  // Monte-Carlo harness (channel.cpp:74-156): statistics independent of the
  // block size, histogram consistent with the frame count
  ed::DecodeConfig tc;
  tc.d_max = 60;
  tc.use_vnr = true;
  const ed::StopRule rule{20, 200};
  const auto t1 = ed::run_trials(lift, pm, ed::snr_for_beta(0.6, pm.effective_rate), tc, rule, 9, 1);
  const auto t4 = ed::run_trials(lift, pm, ed::snr_for_beta(0.6, pm.effective_rate), tc, rule, 9, 4);
  CHECK(t1.frames > 0 && t1.frames == t4.frames && t1.frame_errors == t4.frame_errors);
  CHECK(t1.iteration_sum == t4.iteration_sum && t1.iteration_histogram == t4.iteration_histogram);
  long hsum = 0;
  for (const auto& kv : t1.iteration_histogram) hsum += kv.second;
  CHECK(hsum == t1.frames && t1.stops_syndrome + t1.stops_vnr + t1.stops_max_iter == t1.frames);
  CHECK(t1.fer >= 0.0 && t1.fer <= 1.0 && t1.fer_ci_low <= t1.fer && t1.fer <= t1.fer_ci_high);
  // stream mode and the multi-decoder give, per frame, the blocking decode's
  // result (frames of the (3,6) lift with seeded Gaussian LLRs)
  {
    const int B = 96, n = lift.n_vars();
    std::vector<float> llrs(static_cast<size_t>(B) * n);
    std::uint64_t st = 0x9e3779b97f4a7c15ull;
    for (auto& v : llrs) {  // Irwin-Hall approximation of N(0.9, 1.3^2), reproducible without <random>
      double acc = 0.0;
      for (int k = 0; k < 4; ++k) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        acc += static_cast<double>(st >> 11) * (1.0 / 9007199254740992.0);
      }
      v = static_cast<float>(0.9 + 1.3 * (acc - 2.0) * std::sqrt(3.0));
    }
    ed::DecodeConfig sc;
    sc.d_max = 80;
    sc.use_vnr = true;
    ed::BpDecoder sd(lift, 0, 64);
    const auto want = sd.decode_batch(B, llrs.data(), nullptr, sc);
    std::vector<ed::BatchOutcome> got;
    {
      ed::FrameStream fs(sd, sc);
      std::vector<std::int64_t> tickets;
      for (int b0 = 0; b0 < B; b0 += 32) tickets.push_back(fs.submit(32, llrs.data() + static_cast<size_t>(b0) * n));
      for (auto t : tickets) got.push_back(fs.wait(t));
    }
    for (int b = 0; b < B; ++b) {
      const auto& g = got[b / 32];
      CHECK(g.iterations[b % 32] == want[b].iterations && g.reasons[b % 32] == static_cast<int>(want[b].reason));
      for (int v = 0; v < n; ++v) CHECK(g.bit(b % 32, v) == want[b].bits[v]);
    }
    ed::MultiDecoder md(lift, {0, 0}, 32);
    const auto mo = md.decode_batch(B, llrs.data(), nullptr, sc, 20);
    for (int b = 0; b < B; ++b) {
      CHECK(mo.iterations[b] == want[b].iterations && mo.reasons[b] == static_cast<int>(want[b].reason));
      for (int v = 0; v < n; ++v) CHECK(mo.bit(b, v) == want[b].bits[v]);
    }
  }
  std::printf("compat_test (gpu) OK\n");
  return 0;
}
