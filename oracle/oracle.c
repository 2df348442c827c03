/*
 * TEST INFRASTRUCTURE — CPU oracle, never shipped or measured as the product.
 *
 * Plain-C restatement of the reference decode path (arXiv 2507.03509,
 * /root/reference/proj/core/src/decoder.cpp:50-129) extended to syndrome mode,
 * used only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 *
 * Pinning (tests/test_oracle.py): variant ORC_REF_DOUBLE with s = 0 equals the
 * compiled reference bit for bit (bits, iterations, reason, posteriors,
 * q trace); with s = Hx it equals reference(L * (1-2x)) XOR x (sign
 * equivalence); the SPEC/Appendix-B known-answer values are checked too.
 *
 * Variants
 *   ORC_REF_DOUBLE  double, tanh/atanh with prefix/suffix products — the
 *                   reference's arithmetic, operation for operation.
 *   ORC_PHI_FLOAT   float32 phi-domain algorithm of the CUDA kernels
 *                   (decoder.cu): degree-2 pass-through, degree-1 v2c =
 *                   clamp(llr), per-check order "edges to degree>=2 variables
 *                   first, then degree-1 edges", phi evaluated in double and
 *                   rounded — the GPU algorithm with ideal phi.
 *   ORC_T_FLOAT     the same float32 algorithm in the t domain of the CUDA
 *                   kernels (phi.cuh): t = e^-|m| (double exp, rounded),
 *                   outputs -ln of the float fraction n/d of the prefix /
 *                   suffix (+)-sums, a (+) b = (a + b) / (1 + ab) — the
 *                   shipped GPU algorithm with ideal exp / ln.
 * Build with -ffp-contract=off (no FMA contraction; the reference's Release
 * build on x86-64 has none either).
 */
#include "oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double clampd(double x, double c) { return fmin(c, fmax(-c, x)); }
static float clampf_(float x, float c) { return fminf(c, fmaxf(-c, x)); }

/* uint32 words, LSB first */
static int syn_bit(const uint32_t* s, int c) { return s ? (int)((s[c >> 5] >> (c & 31)) & 1u) : 0; }

/* CSC in ascending check order (parity_check_matrix.cpp:47-60) */
static void build_csc(int n, int m, const int* cp, const int* cv, int* vp, int* ve) {
  int* cur;
  int c, e, v;
  memset(vp, 0, sizeof(int) * (size_t)(n + 1));
  for (e = 0; e < cp[m]; ++e) vp[cv[e] + 1]++;
  for (v = 0; v < n; ++v) vp[v + 1] += vp[v];
  cur = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  memcpy(cur, vp, sizeof(int) * (size_t)n);
  for (c = 0; c < m; ++c)
    for (e = cp[c]; e < cp[c + 1]; ++e) ve[cur[cv[e]]++] = e;
  free(cur);
}

/* ------------------------------------------------ ORC_REF_DOUBLE variant -- */
static int decode_ref_double(int n, int m, const int* cp, const int* cv, const double* llr,
                             const uint32_t* syn, const orc_config* cfg, uint8_t* bits, int32_t* iters,
                             int32_t* reason, double* post_out, double* q_trace) {
  const int E = cp[m];
  int *vp, *ve, *deg;
  double *v2c, *c2v, *th, *prefix, *post;
  uint8_t* hb;
  int maxdeg = 0, c, e, v, j, it;
  double q_prev = 0.0;
  const double clamp = cfg->msg_clamp;
  int stop = 2, last = 0;

  vp = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  ve = (int*)malloc(sizeof(int) * (size_t)(E > 0 ? E : 1));
  deg = (int*)malloc(sizeof(int) * (size_t)n);
  v2c = (double*)malloc(sizeof(double) * (size_t)(E > 0 ? E : 1));
  c2v = (double*)malloc(sizeof(double) * (size_t)(E > 0 ? E : 1));
  th = (double*)malloc(sizeof(double) * (size_t)(E > 0 ? E : 1));
  post = (double*)malloc(sizeof(double) * (size_t)n);
  hb = (uint8_t*)malloc((size_t)n);
  build_csc(n, m, cp, cv, vp, ve);
  for (v = 0; v < n; ++v) deg[v] = vp[v + 1] - vp[v];
  for (c = 0; c < m; ++c)
    if (cp[c + 1] - cp[c] > maxdeg) maxdeg = cp[c + 1] - cp[c];
  prefix = (double*)malloc(sizeof(double) * (size_t)(maxdeg + 1));

  /* v2c[e] = llr[var(e)], unclamped (decoder.cpp:69-73) */
  for (e = 0; e < E; ++e) v2c[e] = llr[cv[e]];

  for (it = 1; it <= cfg->d_max; ++it) {
    double q = 0.0;
    int ok = 0;
    /* check update (decoder.cpp:82-96), times (1 - 2 s_c) in syndrome mode */
    for (c = 0; c < m; ++c) {
      const int b = cp[c], d = cp[c + 1] - cp[c];
      double suffix = 1.0;
      const int flip = syn_bit(syn, c);
      if (d == 0) continue;
      prefix[0] = 1.0;
      for (j = 0; j < d; ++j) {
        th[b + j] = tanh(0.5 * v2c[b + j]);
        prefix[j + 1] = prefix[j] * th[b + j];
      }
      for (j = d - 1; j >= 0; --j) {
        const double r = clampd(2.0 * atanh(prefix[j] * suffix), clamp);
        c2v[b + j] = flip ? -r : r;
        suffix *= th[b + j];
      }
    }
    /* variable update (decoder.cpp:99-105) */
    for (v = 0; v < n; ++v) {
      double p = llr[v];
      int k;
      for (k = vp[v]; k < vp[v + 1]; ++k) p += c2v[ve[k]];
      post[v] = p;
      hb[v] = p < 0.0 ? 1 : 0;
      for (k = vp[v]; k < vp[v + 1]; ++k) v2c[ve[k]] = clampd(p - c2v[ve[k]], clamp);
    }
    /* q over degree>=2 variables, ascending (decoder.cpp:32-36) */
    for (v = 0; v < n; ++v)
      if (deg[v] >= 2) q += cfg->q_mode == ORC_Q_ABS ? fabs(post[v]) : post[v];
    if (q_trace) q_trace[it - 1] = q;
    if (cfg->use_pce) {
      ok = 1;
      for (c = 0; c < m && ok; ++c) {
        int par = syn_bit(syn, c);
        for (e = cp[c]; e < cp[c + 1]; ++e) par ^= hb[cv[e]];
        if (par) ok = 0;
      }
    }
    last = it;
    if (cfg->use_pce && ok) {
      stop = 0;
      break;
    }
    if (cfg->use_vnr && it >= 2 && q < q_prev) {
      stop = 1;
      break;
    }
    q_prev = q;
  }
  *iters = last;
  *reason = stop;
  if (bits) memcpy(bits, hb, (size_t)n);
  if (post_out) memcpy(post_out, post, sizeof(double) * (size_t)n);
  free(vp); free(ve); free(deg); free(v2c); free(c2v); free(th); free(post); free(hb); free(prefix);
  return 0;
}

/* ------------------------------------------------- ORC_PHI_FLOAT variant -- */
/* phi(x) = -ln tanh(x/2) = log1p(2/expm1(x)); phi(0) = inf, phi(inf) = 0 */
static float phi_ideal(float x) { return (float)log1p(2.0 / expm1((double)x)); }

/* t domain: fraction (n, d) (+) t and fraction (+) fraction (float) */
static void tf_add(float* n, float* d, float t) {
  const float nn = *n + t * *d, dd = *d + t * *n;
  *n = nn;
  *d = dd;
}

static int decode_phi_float(int n, int m, const int* cp, const int* cv, const double* llr_d,
                            const uint32_t* syn, const orc_config* cfg, int tdom, uint8_t* bits, int32_t* iters,
                            int32_t* reason, double* post_out, double* q_trace) {
  const int E = cp[m];
  int *vp, *ve, *deg, *ord;
  float *c2v, *post, *llr, *msg, *ph, *pre, *out, *lv;
  uint8_t* hb;
  int maxdeg = 0, c, e, v, j, it, stop = 2, last = 0;
  double q_prev = 0.0;
  const float clamp = (float)cfg->msg_clamp;

  vp = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  ve = (int*)malloc(sizeof(int) * (size_t)(E > 0 ? E : 1));
  deg = (int*)malloc(sizeof(int) * (size_t)n);
  c2v = (float*)calloc((size_t)(E > 0 ? E : 1), sizeof(float));
  post = (float*)malloc(sizeof(float) * (size_t)n);
  llr = (float*)malloc(sizeof(float) * (size_t)n);
  hb = (uint8_t*)malloc((size_t)n);
  build_csc(n, m, cp, cv, vp, ve);
  for (v = 0; v < n; ++v) {
    deg[v] = vp[v + 1] - vp[v];
    llr[v] = (float)llr_d[v];
    post[v] = llr[v];
  }
  for (c = 0; c < m; ++c)
    if (cp[c + 1] - cp[c] > maxdeg) maxdeg = cp[c + 1] - cp[c];
  ord = (int*)malloc(sizeof(int) * (size_t)(maxdeg + 1));
  msg = (float*)malloc(sizeof(float) * (size_t)(maxdeg + 1));
  ph = (float*)malloc(sizeof(float) * (size_t)(maxdeg + 1));
  pre = (float*)malloc(sizeof(float) * (size_t)(maxdeg + 1));
  out = (float*)malloc(sizeof(float) * (size_t)(maxdeg + 1));
  lv = (float*)malloc(sizeof(float) * (size_t)(maxdeg + 1));

  for (it = 1; it <= cfg->d_max; ++it) {
    double q = 0.0;
    int ok = 1;
    for (c = 0; c < m; ++c) {
      const int b = cp[c], d = cp[c + 1] - cp[c];
      unsigned par = (unsigned)syn_bit(syn, c);
      int k = 0;
      float run = 0.0f, suf = 0.0f;
      if (d == 0) {
        if (par) ok = 0;
        continue;
      }
      /* edges to degree>=2 variables first, then degree-1 edges (CSR order within each) */
      for (e = b; e < b + d; ++e)
        if (deg[cv[e]] >= 2) ord[k++] = e;
      for (e = b; e < b + d; ++e)
        if (deg[cv[e]] == 1) ord[k++] = e;
      for (j = 0; j < d; ++j) {
        const int ee = ord[j], vv = cv[ee];
        float mm;
        if (deg[vv] >= 2) {
          mm = it == 1 ? llr[vv] : clampf_(post[vv] - c2v[ee], clamp);
        } else {
          lv[j] = llr[vv];
          mm = it == 1 ? llr[vv] : clampf_(llr[vv], clamp);
        }
        msg[j] = mm;
        par ^= signbit(mm) ? 1u : 0u;
      }
      if (d == 1) {
        out[0] = clamp;
      } else if (d == 2) {
        out[0] = fminf(fabsf(msg[1]), clamp);
        out[1] = fminf(fabsf(msg[0]), clamp);
      } else if (tdom) {
        /* ph = t, pre = prefix fraction numerators, lv-free scratch in out */
        float pn = 0.0f, pd = 1.0f, sn = 0.0f, sd = 1.0f;
        for (j = 0; j < d; ++j) ph[j] = (float)exp(-(double)fabsf(msg[j]));
        for (j = 0; j < d; ++j) { /* out[j] <- prefix over 0..j-1, kept as (pre, out) = (n, d) */
          pre[j] = pn;
          out[j] = pd;
          tf_add(&pn, &pd, ph[j]);
        }
        for (j = d - 1; j >= 0; --j) {
          const float nn = pre[j] * sd + out[j] * sn, dd = out[j] * sd + pre[j] * sn;
          out[j] = nn == dd ? 0.0f : fminf(fabsf((float)log((double)dd / (double)nn)), clamp);
          tf_add(&sn, &sd, ph[j]);
        }
      } else {
        for (j = 0; j < d; ++j) {
          ph[j] = phi_ideal(fabsf(msg[j]));
          pre[j] = run;
          run += ph[j];
        }
        for (j = d - 1; j >= 0; --j) {
          out[j] = fminf(phi_ideal(pre[j] + suf), clamp);
          suf += ph[j];
        }
      }
      for (j = 0; j < d; ++j) {
        const int ee = ord[j], vv = cv[ee];
        const unsigned s = par ^ (signbit(msg[j]) ? 1u : 0u);
        const float o = s ? -out[j] : out[j];
        c2v[ee] = o;
        if (deg[vv] == 1) {
          post[vv] = lv[j] + o;
        }
      }
    }
    for (v = 0; v < n; ++v) {
      int kk;
      float p;
      if (deg[v] < 2) {
        if (deg[v] == 0) post[v] = llr[v];
        hb[v] = post[v] < 0.0f ? 1 : 0;
        continue;
      }
      p = llr[v];
      for (kk = vp[v]; kk < vp[v + 1]; ++kk) p += c2v[ve[kk]];
      post[v] = p;
      hb[v] = p < 0.0f ? 1 : 0;
      q += cfg->q_mode == ORC_Q_ABS ? fabs((double)p) : (double)p;
    }
    if (q_trace) q_trace[it - 1] = q;
    if (cfg->use_pce) {
      for (c = 0; c < m && ok; ++c) {
        int par = syn_bit(syn, c);
        for (e = cp[c]; e < cp[c + 1]; ++e) par ^= hb[cv[e]];
        if (par) ok = 0;
      }
    }
    last = it;
    if (cfg->use_pce && ok) {
      stop = 0;
      break;
    }
    if (cfg->use_vnr && it >= 2 && q < q_prev) {
      stop = 1;
      break;
    }
    q_prev = q;
  }
  *iters = last;
  *reason = stop;
  if (bits) memcpy(bits, hb, (size_t)n);
  if (post_out)
    for (v = 0; v < n; ++v) post_out[v] = (double)post[v];
  free(vp); free(ve); free(deg); free(c2v); free(post); free(llr); free(hb);
  free(ord); free(msg); free(ph); free(pre); free(out); free(lv);
  return 0;
}

int orc_decode(int n_vars, int n_checks, const int* check_ptr, const int* check_vars, const double* llr,
               const uint32_t* syndrome, const orc_config* cfg, int variant, uint8_t* bits, int32_t* iterations,
               int32_t* reason, double* posteriors, double* q_trace) {
  int v;
  if (n_vars <= 0 || n_checks < 1 || n_checks >= n_vars) return 3;
  if (cfg->d_max <= 0 || !(cfg->msg_clamp > 0.0)) return 3; /* decoder.cpp:63-64 */
  for (v = 0; v < n_vars; ++v)
    if (!isfinite(llr[v])) return 3; /* decoder.cpp:60-62 */
  if (variant == ORC_REF_DOUBLE)
    return decode_ref_double(n_vars, n_checks, check_ptr, check_vars, llr, syndrome, cfg, bits, iterations, reason,
                             posteriors, q_trace);
  if (variant == ORC_PHI_FLOAT || variant == ORC_T_FLOAT)
    return decode_phi_float(n_vars, n_checks, check_ptr, check_vars, llr, syndrome, cfg, variant == ORC_T_FLOAT,
                            bits, iterations, reason, posteriors, q_trace);
  return 1;
}

/* ------------------------------------------------------------ channel -- */
/* SplitMix64 finaliser and counter keys (reference rng.hpp:15-30, 85-99) */
static uint64_t sm64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t mixk(uint64_t key, uint64_t word) { return sm64(key ^ sm64(word)); }
static double u01(uint64_t w) { return ((double)(w >> 11) + 0.5) * 0x1.0p-53; }

double orc_snr_for_beta(double beta, double rate) {
  if (!(beta > 0.0) || beta > 1.0 || !(rate > 0.0) || rate >= 1.0) return NAN;
  return exp2(2.0 * rate / beta) - 1.0; /* channel.cpp:39 */
}

double orc_noise_normal(uint64_t seed, uint64_t stream, uint64_t i) {
  const uint64_t key = mixk(mixk(0x243f6a8885a308d3ULL, seed), stream);
  const double a = u01(sm64(key ^ sm64(2 * i)));
  const double b = u01(sm64(key ^ sm64(2 * i + 1)));
  return sqrt(-2.0 * log(a)) * cos(2.0 * 3.141592653589793 * b);
}

int orc_message_bit(uint64_t seed, uint64_t frame, uint64_t i) {
  const uint64_t key = mixk(mixk(0x13198a2e03707344ULL, seed), frame);
  return (int)(sm64(key ^ sm64(i)) >> 63);
}

void orc_sample_frame(int n, double snr, uint64_t seed, uint64_t frame, int all_zero, float* llr, uint8_t* x) {
  const double sigma2 = 1.0 / snr, sigma = sqrt(sigma2), scale = 2.0 / sigma2;
  int i;
  for (i = 0; i < n; ++i) {
    const int xi = all_zero ? 0 : orc_message_bit(seed, frame, (uint64_t)i);
    const double g = orc_noise_normal(seed, frame, (uint64_t)i);
    llr[i] = (float)(scale * ((xi ? -1.0 : 1.0) + sigma * g));
    if (x) x[i] = (uint8_t)xi;
  }
}
