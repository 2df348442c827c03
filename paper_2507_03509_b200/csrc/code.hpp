// Host Tanner-graph model of the decoder (≙ etdec::ParityCheckMatrix,
// reference proj/core/include/etdec/parity_check_matrix.hpp:12-62).
//
// Check-major CSR where the edge id is the CSR slot, plus the var-major CSC
// (var_ptr, var_edges, var_checks) in ascending check order, exactly the
// reference's invariant (parity_check_matrix.cpp:47-60): the variable-node sum
// order of the decoder is ascending check index.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <stdexcept>
#include <string>
#include <vector>

namespace bpdec {

// ≙ etdec::ConfigError / IoError / ValidationError (errors.hpp:8-24); mapped
// to BPDEC_ERR_CONFIG / _IO / _VALIDATION at the C ABI.
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
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class OomError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct Code {
  int32_t n_vars = 0;
  int32_t n_checks = 0;
  std::vector<int32_t> check_ptr;   // M+1
  std::vector<int32_t> check_vars;  // E, edge id = slot
  std::vector<int32_t> var_ptr;     // N+1
  std::vector<int32_t> var_edges;   // E, ascending check order per variable
  std::vector<int32_t> var_checks;  // E, aligned with var_edges

  int64_t n_edges() const { return static_cast<int64_t>(check_vars.size()); }
  int32_t check_degree(int32_t c) const { return check_ptr[c + 1] - check_ptr[c]; }
  int32_t var_degree(int32_t v) const { return var_ptr[v + 1] - var_ptr[v]; }
  // R = (N - M) / N assuming full rank (parity_check_matrix.hpp:23-26).
  double rate() const { return static_cast<double>(n_vars - n_checks) / n_vars; }

  // ≙ from_check_lists (parity_check_matrix.cpp:10-62): same checks, same
  // messages, same error class.
  static Code from_check_lists(int32_t n_vars, const std::vector<std::vector<int32_t>>& lists);
  static Code from_csr(int32_t n_vars, int32_t n_checks, const int32_t* check_ptr,
                       const int32_t* check_vars);
};

// ≙ active_var_set (parity_check_matrix.cpp:64-70): degree >= 2, ascending.
std::vector<int32_t> active_var_set(const Code& code);

// ≙ alist.cpp:78-202 (MacKay layout, 1-based, zero padding ignored on read).
Code load_alist(std::istream& in);
Code load_alist_file(const std::string& path);
void save_alist(const Code& code, std::ostream& out);
void save_alist_file(const Code& code, const std::string& path);

// ≙ lift_protograph (protograph.cpp:52-101).
Code lift_protograph(const std::vector<std::vector<int32_t>>& base, int32_t z, uint64_t seed);

// BASELINE.json code construction (see code.cpp for the exact rule).
Code generate_met(int32_t n_vars, int32_t n_checks, double frac_deg1,
                  const std::vector<int32_t>& degrees, const std::vector<double>& probs,
                  uint64_t seed);

// Two-edge-type low-rate construction with a core code (see code.cpp).
Code generate_met_core(int32_t n_vars, int32_t n_checks, int32_t n_deg1, const std::vector<int32_t>& core_degrees,
                       const std::vector<double>& core_probs, int32_t ext_degree, uint64_t seed);

// ≙ apply_puncture (puncture.cpp:16-48): round(N - (N-M)/target) positions
// drawn uniformly (partial Fisher-Yates, SplitMixEngine(seed)) from the
// degree>=2 variables, ascending.  Returns the positions; *effective_rate set.
std::vector<int32_t> apply_puncture(const Code& code, double target_rate, uint64_t seed, double* effective_rate);

// s = H x, packed LSB-first into ceil(M/32) words.
void compute_syndrome(const Code& code, const uint8_t* bits, uint32_t* syndrome);

}  // namespace bpdec
