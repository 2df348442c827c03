// Host code model: validation, alist I/O, protograph lift and the BASELINE
// multi-edge-style generator.  See code.hpp for the reference mapping.
#include "code.hpp"

#include <algorithm>
#include <cerrno>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>
#include <unordered_set>

#include "rng.hpp"

namespace bpdec {

namespace {

// Builds the var-major CSC from the check-major CSR in ascending check order
// (parity_check_matrix.cpp:47-60).
void build_csc(Code& h) {
  const int64_t e_total = h.n_edges();
  h.var_ptr.assign(static_cast<size_t>(h.n_vars) + 1, 0);
  for (int64_t e = 0; e < e_total; ++e) ++h.var_ptr[h.check_vars[e] + 1];
  for (int32_t v = 0; v < h.n_vars; ++v) h.var_ptr[v + 1] += h.var_ptr[v];
  h.var_edges.resize(e_total);
  h.var_checks.resize(e_total);
  std::vector<int32_t> cursor(h.var_ptr.begin(), h.var_ptr.end() - 1);
  for (int32_t c = 0; c < h.n_checks; ++c) {
    for (int32_t e = h.check_ptr[c]; e < h.check_ptr[c + 1]; ++e) {
      const int32_t v = h.check_vars[e];
      h.var_edges[cursor[v]] = e;
      h.var_checks[cursor[v]] = c;
      ++cursor[v];
    }
  }
}

void check_dims(int64_t n_vars, int64_t n_checks) {
  if (n_vars <= 0) throw ValidationError("parity-check matrix: n_vars must be positive");
  if (n_checks < 1 || n_checks >= n_vars) {
    throw ValidationError(
        "parity-check matrix: rate (n_vars-n_checks)/n_vars must lie in (0,1), got n_vars=" +
        std::to_string(n_vars) + " n_checks=" + std::to_string(n_checks));
  }
}

}  // namespace

Code Code::from_check_lists(int32_t n_vars, const std::vector<std::vector<int32_t>>& lists) {
  const int64_t n_checks = static_cast<int64_t>(lists.size());
  check_dims(n_vars, n_checks);
  std::vector<int32_t> ptr(n_checks + 1, 0);
  std::vector<int32_t> vars;
  size_t total = 0;
  for (const auto& l : lists) total += l.size();
  if (total > static_cast<size_t>(INT32_MAX)) throw ValidationError("parity-check matrix: too many edges");
  vars.reserve(total);
  for (int64_t c = 0; c < n_checks; ++c) {
    vars.insert(vars.end(), lists[c].begin(), lists[c].end());
    ptr[c + 1] = static_cast<int32_t>(vars.size());
  }
  return from_csr(n_vars, static_cast<int32_t>(n_checks), ptr.data(), vars.data());
}

Code Code::from_csr(int32_t n_vars, int32_t n_checks, const int32_t* check_ptr,
                    const int32_t* check_vars) {
  check_dims(n_vars, n_checks);
  if (check_ptr == nullptr) throw ValidationError("parity-check matrix: null check_ptr");
  if (check_ptr[0] != 0) throw ValidationError("parity-check matrix: check_ptr[0] must be 0");
  for (int32_t c = 0; c < n_checks; ++c) {
    if (check_ptr[c + 1] < check_ptr[c]) {
      throw ValidationError("parity-check matrix: check_ptr not monotone at check " + std::to_string(c));
    }
  }
  const int64_t e_total = check_ptr[n_checks];
  if (e_total > 0 && check_vars == nullptr) throw ValidationError("parity-check matrix: null check_vars");
  Code h;
  h.n_vars = n_vars;
  h.n_checks = n_checks;
  h.check_ptr.assign(check_ptr, check_ptr + n_checks + 1);
  h.check_vars.assign(check_vars, check_vars + e_total);
  // Range and duplicate validation per check (parity_check_matrix.cpp:23-44).
  std::vector<int32_t> stamp(n_vars, -1);
  for (int32_t c = 0; c < n_checks; ++c) {
    for (int32_t e = check_ptr[c]; e < check_ptr[c + 1]; ++e) {
      const int32_t v = check_vars[e];
      if (v < 0 || v >= n_vars) {
        throw ValidationError("parity-check matrix: variable index " + std::to_string(v) +
                              " out of range in check " + std::to_string(c));
      }
      if (stamp[v] == c) {
        throw ValidationError("parity-check matrix: duplicate edge (" + std::to_string(c) + "," +
                              std::to_string(v) + ")");
      }
      stamp[v] = c;
    }
  }
  build_csc(h);
  return h;
}

std::vector<int32_t> active_var_set(const Code& code) {
  std::vector<int32_t> members;
  for (int32_t v = 0; v < code.n_vars; ++v) {
    if (code.var_degree(v) >= 2) members.push_back(v);
  }
  return members;
}

// ------------------------------------------------------------------ alist --

namespace {

[[noreturn]] void alist_fail(int line, const std::string& what) {
  throw ValidationError("alist line " + std::to_string(line) + ": " + what);
}

struct AlistLine {
  int number;
  std::vector<long> values;
};

std::vector<AlistLine> tokenize(std::istream& in) {
  std::vector<AlistLine> lines;
  std::string raw;
  int number = 0;
  while (std::getline(in, raw)) {
    ++number;
    if (!raw.empty() && raw.back() == '\r') raw.pop_back();
    AlistLine line{number, {}};
    std::istringstream ss(raw);
    std::string tok;
    while (ss >> tok) {
      char* end = nullptr;
      errno = 0;
      const long v = std::strtol(tok.c_str(), &end, 10);
      if (end == tok.c_str() || *end != '\0' || errno == ERANGE) {
        alist_fail(number, "expected integer, got '" + tok + "'");
      }
      line.values.push_back(v);
    }
    lines.push_back(std::move(line));
  }
  return lines;
}

// Header and degree sections may wrap over lines (alist.cpp:56-74).
std::vector<std::pair<long, int>> take_values(const std::vector<AlistLine>& lines, size_t& idx,
                                              size_t count, const char* what) {
  std::vector<std::pair<long, int>> out;
  while (out.size() < count) {
    if (idx >= lines.size()) {
      alist_fail(lines.empty() ? 1 : lines.back().number,
                 std::string("unexpected end of file while reading ") + what);
    }
    const AlistLine& l = lines[idx++];
    if (l.values.size() > count - out.size()) alist_fail(l.number, std::string("too many entries in ") + what);
    for (long v : l.values) out.emplace_back(v, l.number);
  }
  return out;
}

}  // namespace

Code load_alist(std::istream& in) {
  const auto lines = tokenize(in);
  size_t idx = 0;
  const auto header = take_values(lines, idx, 2, "header");
  const long n = header[0].first, m = header[1].first;
  if (n < 1 || m < 1) alist_fail(header[0].second, "malformed header: dimensions must be positive");
  if (m >= n) {
    alist_fail(header[0].second,
               "malformed header: n_checks must be smaller than n_vars for a code of rate in (0,1)");
  }
  if (n > INT32_MAX) alist_fail(header[0].second, "malformed header: n_vars too large");
  const auto maxima = take_values(lines, idx, 2, "maximum degrees");
  if (maxima[0].first < 0 || maxima[1].first < 0) alist_fail(maxima[0].second, "malformed header: negative maximum degree");
  const auto vdeg = take_values(lines, idx, static_cast<size_t>(n), "variable degrees");
  const auto cdeg = take_values(lines, idx, static_cast<size_t>(m), "check degrees");
  for (const auto& [d, ln] : vdeg) {
    if (d < 0 || d > maxima[0].first) {
      alist_fail(ln, "variable degree " + std::to_string(d) + " outside [0," + std::to_string(maxima[0].first) + "]");
    }
  }
  for (const auto& [d, ln] : cdeg) {
    if (d < 0 || d > maxima[1].first) {
      alist_fail(ln, "check degree " + std::to_string(d) + " outside [0," + std::to_string(maxima[1].first) + "]");
    }
  }
  // One node per line; zero entries are padding (alist.cpp:108-140).
  auto adjacency = [&](long count, long limit, const std::vector<std::pair<long, int>>& deg,
                       const char* what, std::vector<int>* line_of) {
    std::vector<std::vector<int32_t>> adj(count);
    line_of->assign(count, 0);
    for (long k = 0; k < count; ++k) {
      if (idx >= lines.size()) {
        alist_fail(lines.empty() ? 1 : lines.back().number,
                   std::string("unexpected end of file while reading ") + what);
      }
      const AlistLine& l = lines[idx++];
      (*line_of)[k] = l.number;
      auto& entries = adj[k];
      for (long v : l.values) {
        if (v == 0) continue;
        if (v < 1 || v > limit) {
          alist_fail(l.number, "index " + std::to_string(v) + " out of range [1," + std::to_string(limit) + "]");
        }
        const int32_t zb = static_cast<int32_t>(v - 1);
        if (std::find(entries.begin(), entries.end(), zb) != entries.end()) {
          alist_fail(l.number, "duplicate edge: index " + std::to_string(v) + " repeated");
        }
        entries.push_back(zb);
      }
      if (static_cast<long>(entries.size()) != deg[k].first) {
        alist_fail(l.number, std::string(what) + " entry count " + std::to_string(entries.size()) +
                                 " does not match declared degree " + std::to_string(deg[k].first));
      }
    }
    return adj;
  };
  std::vector<int> vline, cline;
  const auto var_lists = adjacency(n, m, vdeg, "variable adjacency", &vline);
  const auto check_lists = adjacency(m, n, cdeg, "check adjacency", &cline);
  // The two directions must describe the same edge set (alist.cpp:147-162).
  std::vector<std::vector<int32_t>> from_vars(m);
  for (long v = 0; v < n; ++v) {
    for (int32_t c : var_lists[v]) from_vars[c].push_back(static_cast<int32_t>(v));
  }
  for (long c = 0; c < m; ++c) {
    auto a = from_vars[c];
    auto b = check_lists[c];
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    if (a != b) {
      alist_fail(cline[c], "adjacency mismatch: check " + std::to_string(c + 1) +
                               " disagrees with the variable-side lists");
    }
  }
  return Code::from_check_lists(static_cast<int32_t>(n), check_lists);
}

Code load_alist_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open alist file: " + path);
  return load_alist(in);
}

void save_alist(const Code& h, std::ostream& out) {
  int32_t max_v = 0, max_c = 0;
  for (int32_t v = 0; v < h.n_vars; ++v) max_v = std::max(max_v, h.var_degree(v));
  for (int32_t c = 0; c < h.n_checks; ++c) max_c = std::max(max_c, h.check_degree(c));
  out << h.n_vars << ' ' << h.n_checks << '\n' << max_v << ' ' << max_c << '\n';
  for (int32_t v = 0; v < h.n_vars; ++v) out << h.var_degree(v) << (v + 1 == h.n_vars ? '\n' : ' ');
  for (int32_t c = 0; c < h.n_checks; ++c) out << h.check_degree(c) << (c + 1 == h.n_checks ? '\n' : ' ');
  for (int32_t v = 0; v < h.n_vars; ++v) {
    for (int32_t k = h.var_ptr[v]; k < h.var_ptr[v + 1]; ++k) {
      if (k != h.var_ptr[v]) out << ' ';
      out << h.var_checks[k] + 1;
    }
    out << '\n';
  }
  for (int32_t c = 0; c < h.n_checks; ++c) {
    for (int32_t e = h.check_ptr[c]; e < h.check_ptr[c + 1]; ++e) {
      if (e != h.check_ptr[c]) out << ' ';
      out << h.check_vars[e] + 1;
    }
    out << '\n';
  }
}

void save_alist_file(const Code& code, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot open alist file for writing: " + path);
  save_alist(code, out);
  if (!out) throw IoError("write failed: " + path);
}

// -------------------------------------------------------- protograph lift --

Code lift_protograph(const std::vector<std::vector<int32_t>>& base, int32_t z, uint64_t seed) {
  if (z < 1) throw ValidationError("protograph lift: lifting factor must be >= 1");
  if (base.empty() || base.front().empty()) throw ValidationError("protograph lift: empty base matrix");
  const size_t rows = base.size(), cols = base.front().size();
  for (const auto& row : base) {
    if (row.size() != cols) throw ValidationError("protograph lift: ragged base matrix");
    for (int32_t m : row) {
      if (m < 0) throw ValidationError("protograph lift: negative multiplicity");
    }
  }
  // Cells in row-major order draw `mult` distinct circulant shifts from one
  // SplitMix stream (rejecting repeats within a cell, bounded retries); each
  // shift s connects lifted check r*z+k to variable c*z+(k+s) mod z
  // (protograph.cpp:68-93).
  SplitMixEngine rng(seed);
  std::vector<std::vector<int32_t>> checks(rows * z);
  for (size_t r = 0; r < rows; ++r) {
    for (size_t c = 0; c < cols; ++c) {
      const int32_t mult = base[r][c];
      if (mult == 0) continue;
      std::vector<int32_t> shifts;
      long budget = 256 + 64L * z;
      while (static_cast<int32_t>(shifts.size()) < mult) {
        if (--budget < 0) {
          throw ValidationError("protograph lift: cannot avoid parallel edges for base cell (" +
                                std::to_string(r) + "," + std::to_string(c) + ") with multiplicity " +
                                std::to_string(mult) + " at Z=" + std::to_string(z) +
                                " (lifting factor too small)");
        }
        const int32_t s = static_cast<int32_t>(rng.bounded(static_cast<uint64_t>(z)));
        if (std::find(shifts.begin(), shifts.end(), s) == shifts.end()) shifts.push_back(s);
      }
      for (int32_t s : shifts) {
        for (int32_t k = 0; k < z; ++k) {
          checks[r * z + k].push_back(static_cast<int32_t>(c * z + (k + s) % z));
        }
      }
    }
  }
  return Code::from_check_lists(static_cast<int32_t>(cols * z), checks);
}

// ------------------------------------------------------ BASELINE generator --
//
// Rule (recorded in DESIGN.md):
//  * N1 = floor(f1*N + 0.5) degree-1 variables, the LAST N1 indices; variable
//    (N-N1+j) joins check (M-N1+j), an identity block on the last checks.
//  * The first N_hi = N-N1 variables take degree classes in listed order:
//    n_i = floor(N_hi*p_i + 0.5) for all but the last class, which takes the
//    remainder.
//  * High-degree sockets (variable v repeated deg(v) times, ascending) are
//    matched to the check socket list k mod M (k = 0..E_hi-1; near-regular
//    over all checks) after a Fisher-Yates shuffle driven by
//    SplitMixEngine(seed).  A socket that repeats a check of its variable is
//    swapped with a random other socket until neither variable holds a
//    duplicate (bounded retries).
//  * Each check's variable list is sorted ascending.
Code generate_met(int32_t n_vars, int32_t n_checks, double frac_deg1,
                  const std::vector<int32_t>& degrees, const std::vector<double>& probs,
                  uint64_t seed) {
  check_dims(n_vars, n_checks);
  if (degrees.empty() || degrees.size() != probs.size()) {
    throw ValidationError("met generator: degree and probability lists must be non-empty and aligned");
  }
  if (!(frac_deg1 >= 0.0) || frac_deg1 >= 1.0) throw ValidationError("met generator: frac_deg1 must lie in [0,1)");
  const int64_t n1 = static_cast<int64_t>(std::floor(frac_deg1 * n_vars + 0.5));
  if (n1 > n_checks) throw ValidationError("met generator: more degree-1 variables than checks");
  const int64_t n_hi = n_vars - n1;
  std::vector<int64_t> counts(degrees.size());
  int64_t assigned = 0;
  for (size_t i = 0; i + 1 < degrees.size(); ++i) {
    if (degrees[i] < 2) throw ValidationError("met generator: high-degree classes need degree >= 2");
    counts[i] = static_cast<int64_t>(std::floor(n_hi * probs[i] + 0.5));
    assigned += counts[i];
  }
  if (degrees.back() < 2) throw ValidationError("met generator: high-degree classes need degree >= 2");
  counts.back() = n_hi - assigned;
  if (counts.back() < 0) throw ValidationError("met generator: class proportions exceed 1");
  std::vector<int32_t> vdeg(n_hi);
  {
    int64_t v = 0;
    for (size_t i = 0; i < degrees.size(); ++i) {
      if (degrees[i] > n_checks) throw ValidationError("met generator: degree exceeds n_checks");
      for (int64_t k = 0; k < counts[i]; ++k) vdeg[v++] = degrees[i];
    }
  }
  std::vector<int64_t> sock_ptr(n_hi + 1, 0);
  for (int64_t v = 0; v < n_hi; ++v) sock_ptr[v + 1] = sock_ptr[v] + vdeg[v];
  const int64_t e_hi = sock_ptr[n_hi];
  if (e_hi + n1 > INT32_MAX) throw ValidationError("met generator: too many edges");
  std::vector<int32_t> owner(e_hi);
  for (int64_t v = 0; v < n_hi; ++v) {
    for (int64_t k = sock_ptr[v]; k < sock_ptr[v + 1]; ++k) owner[k] = static_cast<int32_t>(v);
  }
  std::vector<int32_t> cs(e_hi);
  for (int64_t k = 0; k < e_hi; ++k) cs[k] = static_cast<int32_t>(k % n_checks);
  SplitMixEngine rng(seed);
  for (int64_t i = e_hi - 1; i > 0; --i) {
    const int64_t j = static_cast<int64_t>(rng.bounded(static_cast<uint64_t>(i + 1)));
    std::swap(cs[i], cs[j]);
  }
  auto holds = [&](int32_t v, int32_t check, int64_t except) {
    for (int64_t k = sock_ptr[v]; k < sock_ptr[v + 1]; ++k) {
      if (k != except && cs[k] == check) return true;
    }
    return false;
  };
  if (e_hi > 0) {
    for (int64_t v = 0; v < n_hi; ++v) {
      for (int64_t k = sock_ptr[v]; k < sock_ptr[v + 1]; ++k) {
        if (!holds(static_cast<int32_t>(v), cs[k], k)) continue;
        long budget = 1L << 20;
        for (;;) {
          if (--budget < 0) throw ValidationError("met generator: cannot remove duplicate edges");
          const int64_t k2 = static_cast<int64_t>(rng.bounded(static_cast<uint64_t>(e_hi)));
          const int32_t w = owner[k2];
          if (w == v) continue;
          if (holds(static_cast<int32_t>(v), cs[k2], k)) continue;
          if (holds(w, cs[k], k2)) continue;
          std::swap(cs[k], cs[k2]);
          break;
        }
      }
    }
  }
  std::vector<int32_t> cdeg(n_checks, 0);
  for (int64_t k = 0; k < e_hi; ++k) ++cdeg[cs[k]];
  for (int64_t j = 0; j < n1; ++j) ++cdeg[n_checks - n1 + j];
  std::vector<int32_t> ptr(n_checks + 1, 0);
  for (int32_t c = 0; c < n_checks; ++c) ptr[c + 1] = ptr[c] + cdeg[c];
  std::vector<int32_t> vars(ptr[n_checks]);
  std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
  for (int64_t k = 0; k < e_hi; ++k) vars[fill[cs[k]]++] = owner[k];
  for (int64_t j = 0; j < n1; ++j) {
    const int32_t c = static_cast<int32_t>(n_checks - n1 + j);
    vars[fill[c]++] = static_cast<int32_t>(n_hi + j);
  }
  for (int32_t c = 0; c < n_checks; ++c) std::sort(vars.begin() + ptr[c], vars.begin() + ptr[c + 1]);
  return Code::from_csr(n_vars, n_checks, ptr.data(), vars.data());
}

// Two-edge-type low-rate construction (a multi-edge-type code in the sense
// of SURVEY §8f#2; new, not in the reference).  Variables: core 0..nc-1,
// degree-1 nc..N-1 (nc = N - n1).  Checks: core 0..Mc-1 (Mc = M - n1), which
// hold only type-1 edges of core variables, and extension checks Mc+j, which
// hold ext_degree type-2 edges of core variables plus the degree-1 variable
// nc+j.  Every codeword restricted to the core variables is a codeword of
// the core code, so its minimum distance is not capped by the degree-1
// block (the BASELINE construction has distance ~4: a degree-3 variable and
// the degree-1 variables of its checks).
//   type 1: core class counts round(nc * p_i) (remainder in the last class),
//           classes in variable order; check sockets k mod Mc after a
//           SplitMix Fisher-Yates shuffle; duplicates repaired by swaps.
//   type 2: socket i belongs to extension check Mc + i / ext_degree; its
//           variable is i mod nc after a Fisher-Yates shuffle of those
//           (same engine, continued), so type-2 degrees differ by <= 1;
//           duplicates within a check repaired by swaps.
Code generate_met_core(int32_t n_vars, int32_t n_checks, int32_t n_deg1, const std::vector<int32_t>& core_degrees,
                       const std::vector<double>& core_probs, int32_t ext_degree, uint64_t seed) {
  check_dims(n_vars, n_checks);
  if (core_degrees.empty() || core_degrees.size() != core_probs.size())
    throw ValidationError("met core generator: degree and probability lists must be non-empty and aligned");
  if (n_deg1 <= 0 || n_deg1 >= n_checks || n_deg1 >= n_vars)
    throw ValidationError("met core generator: need 0 < n_deg1 < min(n_checks, n_vars)");
  const int32_t nc = n_vars - n_deg1, mc = n_checks - n_deg1, n1 = n_deg1;
  if (ext_degree < 1 || ext_degree > nc)
    throw ValidationError("met core generator: ext_degree must lie in [1, number of core variables]");
  std::vector<int64_t> counts(core_degrees.size());
  int64_t assigned = 0;
  for (size_t i = 0; i < core_degrees.size(); ++i) {
    if (core_degrees[i] < 1 || core_degrees[i] > mc)
      throw ValidationError("met core generator: core degrees must lie in [1, number of core checks]");
    if (i + 1 < core_degrees.size()) {
      counts[i] = static_cast<int64_t>(std::floor(nc * core_probs[i] + 0.5));
      assigned += counts[i];
    }
  }
  counts.back() = nc - assigned;
  if (counts.back() < 0) throw ValidationError("met core generator: class proportions exceed 1");
  SplitMixEngine rng(seed);
  // ---- type 1: core variables x core checks
  std::vector<int64_t> sp(static_cast<size_t>(nc) + 1, 0);
  {
    int64_t v = 0;
    for (size_t i = 0; i < core_degrees.size(); ++i)
      for (int64_t k = 0; k < counts[i]; ++k, ++v) sp[v + 1] = sp[v] + core_degrees[i];
  }
  const int64_t e1 = sp[nc];
  const int64_t e2 = static_cast<int64_t>(n1) * ext_degree;
  if (e1 + e2 + n1 > INT32_MAX) throw ValidationError("met core generator: too many edges");
  std::vector<int32_t> own1(e1), cs1(e1);
  for (int32_t v = 0; v < nc; ++v)
    for (int64_t k = sp[v]; k < sp[v + 1]; ++k) own1[k] = v;
  for (int64_t k = 0; k < e1; ++k) cs1[k] = static_cast<int32_t>(k % mc);
  for (int64_t i = e1 - 1; i > 0; --i) std::swap(cs1[i], cs1[rng.bounded(static_cast<uint64_t>(i + 1))]);
  auto holds1 = [&](int32_t v, int32_t c, int64_t except) {
    for (int64_t k = sp[v]; k < sp[v + 1]; ++k)
      if (k != except && cs1[k] == c) return true;
    return false;
  };
  for (int64_t k = 0; k < e1; ++k) {
    const int32_t v = own1[k];
    if (!holds1(v, cs1[k], k)) continue;
    for (long budget = 1L << 20;; ) {
      if (--budget < 0) throw ValidationError("met core generator: cannot remove duplicate type-1 edges");
      const int64_t k2 = static_cast<int64_t>(rng.bounded(static_cast<uint64_t>(e1)));
      const int32_t w = own1[k2];
      if (w == v || holds1(v, cs1[k2], k) || holds1(w, cs1[k], k2)) continue;
      std::swap(cs1[k], cs1[k2]);
      break;
    }
  }
  // ---- type 2: core variables x extension checks (ext_degree sockets each)
  std::vector<int32_t> own2(e2);
  for (int64_t i = 0; i < e2; ++i) own2[i] = static_cast<int32_t>(i % nc);
  for (int64_t i = e2 - 1; i > 0; --i) std::swap(own2[i], own2[rng.bounded(static_cast<uint64_t>(i + 1))]);
  auto in_check2 = [&](int64_t i, int32_t v) {  // another socket of i's check holds v
    const int64_t b = (i / ext_degree) * ext_degree;
    for (int64_t k = b; k < b + ext_degree; ++k)
      if (k != i && own2[k] == v) return true;
    return false;
  };
  for (int64_t i = 0; i < e2; ++i) {
    if (!in_check2(i, own2[i])) continue;
    for (long budget = 1L << 20;; ) {
      if (--budget < 0) throw ValidationError("met core generator: cannot remove duplicate type-2 edges");
      const int64_t i2 = static_cast<int64_t>(rng.bounded(static_cast<uint64_t>(e2)));
      if (i2 / ext_degree == i / ext_degree || in_check2(i, own2[i2]) || in_check2(i2, own2[i])) continue;
      std::swap(own2[i], own2[i2]);
      break;
    }
  }
  // ---- CSR (check lists ascending)
  std::vector<int32_t> ptr(static_cast<size_t>(n_checks) + 1, 0);
  for (int64_t k = 0; k < e1; ++k) ++ptr[cs1[k] + 1];
  for (int32_t j = 0; j < n1; ++j) ptr[mc + j + 1] = ext_degree + 1;
  for (int32_t c = 0; c < n_checks; ++c) ptr[c + 1] += ptr[c];
  std::vector<int32_t> vars(ptr[n_checks]);
  std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
  for (int64_t k = 0; k < e1; ++k) vars[fill[cs1[k]]++] = own1[k];
  for (int64_t i = 0; i < e2; ++i) vars[fill[mc + i / ext_degree]++] = own2[i];
  for (int32_t j = 0; j < n1; ++j) vars[fill[mc + j]++] = nc + j;
  for (int32_t c = 0; c < n_checks; ++c) std::sort(vars.begin() + ptr[c], vars.begin() + ptr[c + 1]);
  return Code::from_csr(n_vars, n_checks, ptr.data(), vars.data());
}

std::vector<int32_t> apply_puncture(const Code& code, double target_rate, uint64_t seed, double* effective_rate) {
  const double rate = code.rate();
  if (target_rate >= 1.0) throw ValidationError("puncture: target rate must be below 1");
  if (target_rate < rate - 1e-12) {
    throw ValidationError("puncture: target rate " + std::to_string(target_rate) + " is below the code rate " +
                          std::to_string(rate) + "; puncturing can only raise the rate");
  }
  const int32_t n = code.n_vars, m = code.n_checks;
  const long count = std::lround(n - (n - m) / target_rate);
  if (count <= 0) {
    if (effective_rate) *effective_rate = rate;
    return {};
  }
  std::vector<int32_t> eligible;
  for (int32_t v = 0; v < n; ++v)
    if (code.var_degree(v) >= 2) eligible.push_back(v);
  if (count > static_cast<long>(eligible.size())) {
    throw ValidationError("puncture: need " + std::to_string(count) + " positions but only " +
                          std::to_string(eligible.size()) + " variables of degree >= 2 are eligible");
  }
  // k distinct draws from [0, n_eligible): partial Fisher-Yates in draw order
  SplitMixEngine rng(seed);
  const uint32_t pool_n = static_cast<uint32_t>(eligible.size());
  std::vector<uint32_t> pool(pool_n);
  for (uint32_t i = 0; i < pool_n; ++i) pool[i] = i;
  std::vector<int32_t> out(count);
  for (long i = 0; i < count; ++i) {
    const uint64_t j = static_cast<uint64_t>(i) + rng.bounded(pool_n - static_cast<uint64_t>(i));
    std::swap(pool[i], pool[j]);
    out[i] = eligible[pool[i]];
  }
  std::sort(out.begin(), out.end());
  if (effective_rate) *effective_rate = static_cast<double>(n - m) / static_cast<double>(n - count);
  return out;
}

void compute_syndrome(const Code& code, const uint8_t* bits, uint32_t* syndrome) {
  const int32_t words = (code.n_checks + 31) / 32;
  std::fill(syndrome, syndrome + words, 0u);
  for (int32_t c = 0; c < code.n_checks; ++c) {
    uint32_t p = 0;
    for (int32_t e = code.check_ptr[c]; e < code.check_ptr[c + 1]; ++e) p ^= bits[code.check_vars[e]] & 1u;
    syndrome[c >> 5] |= p << (c & 31);
  }
}

}  // namespace bpdec
