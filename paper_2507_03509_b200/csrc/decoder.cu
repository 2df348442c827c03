// B200 (sm_100a) batched flooding sum-product LDPC decoder with PCE/VNR early
// termination — the hot path of reference proj/core/src/decoder.cpp:50-129.
//
// Layout.  Frames in flight occupy "slots"; 32 slots form a
// group and every per-item array is stored [group][item][32 lanes], so one
// warp handles one check (or variable) for 32 frames and every access —
// including the random Tanner-graph gathers — moves whole 128-byte lines.
// Variables are split into
//   H : degree != 1 (degree >= 2 first = the VNR set 𝒱, then degree 0)
//   D1: degree-1 variables, stored in the order of their (single) check.
// State per slot: channel LLRs (llr_h, llr_d), the posterior of every
// degree>=2 variable (post), and the check->variable message of every edge
// that touches a degree>=2 variable (c2v).  Degree-1 edges keep no message
// state: their variable->check message is clamp(llr) (the reference's
// clamp((llr + c2v) - c2v), decoder.cpp:100-104, without the double rounding
// residue) and their posterior llr + c2v is formed inside the check kernel.
// The c2v of a check with one degree>=2 and one degree-1 edge is a constant
// of the frame; after its first iteration it is not re-read or rewritten.
// A VNR batch's last few live frames run in a narrow group ([row][16] or
// [row][8] inside the group's block, lane-folded kernels; rix()).
//
// One decoding step = one flooding iteration for every active slot:
//   k_check     check-node update (decoder.cpp:82-96) + degree-1 posteriors,
//               hard bits and the degree-1 part of the syndrome
//   k_var       variable-node update (decoder.cpp:99-105) for degree>=2
//               variables, hard bits, per-tile q partial sums (:32-36, :107)
//   k_decide    bit-sliced parity of every check vs the target syndrome
//               (decoder.cpp:19-30), the fixed-order q^(k) reduction, and
//               the PCE -> VNR -> d_max decision per frame (:114-123)
//   k_turnover  outputs of frames that stopped this step (:126-128) and
//               the next queued frames streamed into the freed slots
//   k_compact   tail compaction of the live frames into fewer groups, and
//               the move of a last group's few live frames into a narrow
//               (16 / 8-lane) group
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <type_traits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "decoder.hpp"
#include "devguard.hpp"
#include "devmem.hpp"
#include "phi.cuh"
#include "rng.hpp"

namespace bpdec {

namespace {

#define CUDA_OK(expr)                                                                        \
  do {                                                                                       \
    cudaError_t err__ = (expr);                                                              \
    if (err__ != cudaSuccess) {                                                              \
      if (err__ == cudaErrorMemoryAllocation) {                                              \
        (void)cudaGetLastError();                                                            \
        throw OomError(std::string("CUDA out of memory: ") + #expr);                         \
      }                                                                                      \
      throw CudaError(std::string("CUDA error ") + cudaGetErrorString(err__) + " at " + #expr); \
    }                                                                                        \
  } while (0)

constexpr int kLanes = 32;
constexpr int kVarWarps = 4;    // warps per k_var block
constexpr int kQTile = 64;     // variables per k_var tile and q partial sum (code-fixed order)
constexpr int kThreads = 256;
constexpr int kCheckThreads = 128;  // k_check blocks: 4 warps (per-warp smem ring)
enum KernelId { kCheck = 0, kVar = 1, kSyn = 2, kTerm = 3, kTurnover = 4, kCompact = 5, kSnapshot = 6, kTrace = 7, kNumKernels = 8 };
// (kSyn = k_decide; kTerm is kept for the profiling ABI and stays 0)
#ifndef BPDEC_CHECK_MINB
#define BPDEC_CHECK_MINB 5
#endif
#ifndef BPDEC_SPLIT_MAXD
#define BPDEC_SPLIT_MAXD 6
#endif
constexpr int kCheckMinBlocks = BPDEC_CHECK_MINB;  // k_check blocks per SM (register budget)
// k_check kernels (by maximum check degree) with a separate steady-state
// copy of every typed chunk loop, which also uses the phi-domain degree-1
// edge (kPhiD in check_batch_compute); wider kernels keep one copy
// (instruction cache; splitting k_check<8> measured -2% on a (3,1) code,
// splitting k_check<6> +6.7% on the rate-0.1 QC lift of scripts/qc_probe.py)
constexpr int kSplitMaxD = BPDEC_SPLIT_MAXD;
constexpr int kCheckGrab = 1;     // k_check chunks per scheduler atomic (2: -9% on cfg2, the two
                                  // chunks of a grab run back to back on one warp instead of side by side)
constexpr int kTermBlocks = 16;   // k_decide q-reduction blocks per group (q partial tree: fixed by the code)

// L2 residency hints (measured on cfg2, 384-slot stream, A/B of builds on
// one box): the posterior rows are written once by k_var and gathered ~deg
// times by the next k_check, between 5 GB of streamed messages per step.
// evict_last on the gathers (1) and also on k_var's posterior stores (2):
// +2.3 % / +3.5 % edge-updates/s (the variable pass -10 %: fewer DRAM writes
// between its gathers); evict_last on the per-edge hard-decision words
// (ebits, read by k_decide): +0.5 %.  0 = plain accesses (A/B builds).
#ifndef BPDEC_POST_EVICT_LAST
#define BPDEC_POST_EVICT_LAST 2
#endif

#ifndef BPDEC_EBITS_EVL
#define BPDEC_EBITS_EVL 1  // the per-edge hard-decision words of k_var are stored with an evict_last hint
#endif
// ------------------------------------------------------------ arguments --
struct Args {
  // code
  int32_t N, M, NH, NV, N1, n_tiles;
  int64_t EH;
  const int4* cdesc;        // [M] {hi_begin, hi_end, d1_begin, d1_end}
  const int32_t* chk_hi_h;  // [EH] H index of each degree>=2 edge, check-major
  const int32_t* vptr;      // [NV+1]
  const int32_t* vedge;     // [EH] c2v row of each edge of variable h, ascending check
  const int32_t* vmap;      // [N] original var -> h (>=0) or -1-d (degree 1)
  const int32_t* cdev;      // [M] original check -> device check
  const int4* ctype;        // [ceil(M/32)] {type NH*8+ND (homogeneous full chunk) or -1,
                            //  first hi edge, first degree-1 row, hi edge end}
  const int2* vtile;        // [n_tiles] {tile degree D (typed path) or -1 (generic), first slot in vedge_t}
  const int32_t* vedge_t;   // tile-padded CSC: per typed tile 64 x D edge ids, -1 = padding
  int32_t ve_stride;        // k_var edge-id buffer size (32 x largest typed tile degree)
  const int32_t* vsched;    // [n_tiles] k_var hand-out order: generic tiles first, then by degree
  const int32_t* csched;    // [ceil(M/32)] k_check hand-out order: generic chunks first
  // state
  int32_t G;
  float* llr_h;             // [G][NH][32]
  float* llr_d;             // [G][N1][32]
  float* post;              // [G][NV][32]
  float* c2v;               // [G][EH][32]
  float* d1post;            // [G][N1][32] (only when posteriors are requested)
  uint32_t* hbits;          // [G][NV]
  uint32_t* ebits;          // [G][EH] hard-decision word of each degree>=2 edge's variable (check-major)
  uint32_t* d1bits;         // [G][N1]
  uint32_t* synp;           // [G][M]  target syndrome ^ degree-1 parity
  uint32_t* syn_target;     // [G][M]
  double* q_part;           // [G][n_tiles][32]
  double* q_mid;            // [G][kTermBlocks][32]
  int32_t* stop_frame;      // [S] frame that stopped in the slot this step (read by k_turnover)
  double* qprev;            // [S]
  int32_t* slot_iter;       // [S] iteration the slot runs next (1-based)
  int32_t* slot_frame;      // [S]
  int32_t* pending_frame;   // [S]
  uint32_t* group_active;   // [G]
  uint32_t* fail;           // [G]
  uint32_t* stopped;        // [G]
  uint32_t* load_mask;      // [G]
  int32_t* counters;        // [0] next frame, [1] frames done, [2] error flags, [3] active slots,
                            // [4] active slots at the last compaction, [5] k_compact blocks done,
                            // [6] k_var tiles handed out, [7] k_check chunks handed out,
                            // [8] k_decide blocks done, [9] frames available (uploaded),
                            // [10] k_decide syndrome passes handed out, [11] lane width of
                            // the live groups' layout (32, or 16 / 8 for a narrow tail group),
                            // [12] slots were moved (k_compact) since the last k_check
  unsigned long long* frame_iters;
  // host polling: k_decide's deciding block copies counters[0..3] into slot
  // poll_slot of this pinned, mapped host ring at the end of every step
  // (no D2H copy between the step kernels)
  int32_t* h_poll;
  int32_t poll_slot;
  // decode parameters
  int32_t batch, d_max, use_pce, use_vnr, q_mode;
  float clamp;
  int32_t narrow_ok;          // the tail group may be re-laid out narrow (check degree <= 4, G >= 2)
  int32_t compact_hyst;       // k_compact re-packs only after this many more frames finished (32)
  int32_t group_refill;       // stream mode: refill only groups that are entirely free (dense loads)
                              // and compact while frames are queued, so no step refills single lanes
  // inputs / outputs (device)
  const float* in_llr;        // [batch][N]
  const uint32_t* in_syn;     // [batch][MW] or null
  int32_t MW, NW;
  uint8_t* out_bits_u8;       // [batch][N] or null
  uint32_t* out_bits_pk;      // [batch][NW] or null
  int32_t* out_iters;
  uint8_t* out_reasons;
  float* out_post;
  double* out_qtrace;
  uint8_t* out_syntrace;      // [batch][d_max] syndrome_ok per iteration, or null
  float* out_ptrace;          // [batch][d_max][N] posteriors per iteration, or null
  // stream mode (bpdec_stream_*): frame f's input and output rows live at
  // ring position f % ring_cap of device rings; 0 = rows indexed by f
  int32_t ring_cap;
  const int32_t* fbatch;      // [ring_cap] batch slot of the frame at each ring position
  int32_t* bdone;             // [kMaxStreamBatches] frames of each batch slot that stopped
  uint8_t* ferr;              // [ring_cap] frame had a non-finite input LLR
};

constexpr int kAvailPieces = 8;        // a submitted batch's LLR upload is cut into at most this many pieces
constexpr int kMaxStreamBatches = 32;  // batches in flight in stream mode (poll ring reports them)
constexpr int kPollWords = 4 + kMaxStreamBatches;

// Row of frame f in the input / output buffers.
__device__ __forceinline__ size_t frow(const Args& a, int f) {
  return static_cast<size_t>(a.ring_cap ? f % a.ring_cap : f);
}

__device__ __forceinline__ float clampf(float x, float c) { return fminf(fmaxf(x, -c), c); }
__device__ __forceinline__ uint32_t signbit_u(float x) { return __float_as_uint(x) >> 31; }
__device__ __forceinline__ float with_sign(float mag, uint32_t s) {
  return __uint_as_float(__float_as_uint(mag) | (s << 31));
}

// Per-slot arrays are [group][row][32 lanes].  A group that is the only
// live one in the decoder's tail can be re-laid out "narrow": its <= lw
// (16 or 8) live frames in lanes 0..lw-1 and rows of lw floats
// ([group][row][lw] inside the group's block), so a row is one or two
// sectors instead of a 128-byte line (see k_compact).  `lw` is 32 otherwise.
__device__ __forceinline__ size_t rix(int g, int64_t rows, int64_t row, int lw) {
  return static_cast<size_t>(g) * static_cast<size_t>(rows) * kLanes + static_cast<size_t>(row) * lw;
}

// Streaming loads/stores for the once-per-iteration message traffic; the
// posterior gathers use the default policy so the [G][NV][32] array stays in
// L2 between the variable pass that writes it and the check pass that
// re-reads it ~deg times.
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }

// Predicated loads/stores as single instructions (no branch), so a warp can
// keep all of a chunk's gathers in flight: a C++ `cond ? load : 0` compiles to
// a branch region per load with its consumer inside, which serialises them.
[[maybe_unused]] __device__ __forceinline__ float ld_pred(const float* p, bool pred) {
  float v = 0.0f;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.f32 %0, [%1];\n\t}"
               : "+f"(v)
               : "l"(p), "r"(static_cast<int>(pred)));
  return v;
}
[[maybe_unused]] __device__ __forceinline__ float ldcs_pred(const float* p, bool pred) {
  float v = 0.0f;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.cs.f32 %0, [%1];\n\t}"
               : "+f"(v)
               : "l"(p), "r"(static_cast<int>(pred)));
  return v;
}
__device__ __forceinline__ void stcs_pred(float* p, float v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.f32 [%0], %1;\n\t}"
               :
               : "l"(p), "f"(v), "r"(static_cast<int>(pred))
               : "memory");
}
__device__ __forceinline__ void st_pred(float* p, float v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f32 [%0], %1;\n\t}"
               :
               : "l"(p), "f"(v), "r"(static_cast<int>(pred))
               : "memory");
}

[[maybe_unused]] __device__ __forceinline__ void st_pred_pol(float* p, float v, bool pred, uint64_t pol) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.L2::cache_hint.f32 [%0], %1, %3;\n\t}"
               :
               : "l"(p), "f"(v), "r"(static_cast<int>(pred)), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void st_pred_u32(uint32_t* p, uint32_t v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.u32 [%0], %1;\n\t}"
               :
               : "l"(p), "r"(v), "r"(static_cast<int>(pred))
               : "memory");
}

[[maybe_unused]] __device__ __forceinline__ uint64_t policy_evict_last_nv() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
[[maybe_unused]] __device__ __forceinline__ void st_pred_u32_pol(uint32_t* p, uint32_t v, bool pred, uint64_t pol) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.L2::cache_hint.u32 [%0], %1, %3;\n\t}"
               :
               : "l"(p), "r"(v), "r"(static_cast<int>(pred)), "l"(pol)
               : "memory");
}

// Programmatic dependent launch: the step kernels are launched with
// programmatic stream serialisation, so a kernel's blocks can be scheduled
// while its predecessor drains; every kernel waits for the predecessor's
// completion (and memory) before its first global access, then lets its own
// successor launch.  No-ops when launched without the attribute.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// ------------------------------------------------------- work schedulers --
// k_check and k_var hand out work dynamically: a warp grabs the next index k
// from counters[ctr] (k_check resets k_var's counter and vice versa) and k
// maps to item sched[k % per_group] of the (k / per_group)-th group that
// has active slots.  The schedules put latency-bound generic items first so
// they overlap the streamed bulk instead of forming the tail.  The grab is
// split so the atomic can be issued one item ahead of its use.
__device__ __forceinline__ int sched_issue(const Args& a, int ctr, int lane) {
  int k = 0;
  if (lane == 0) k = atomicAdd(&a.counters[ctr], 1);
  return k;  // valid in lane 0 only
}

__device__ __forceinline__ int sched_issue_n(const Args& a, int ctr, int lane, int n) {
  int k = 0;
  if (lane == 0) k = atomicAdd(&a.counters[ctr], n);
  return k;  // valid in lane 0 only
}

// k uniform across the warp
__device__ __forceinline__ long long sched_map(const Args& a, int k, int lane, int per_group,
                                               const int32_t* __restrict__ sched) {
  const long long total = static_cast<long long>(a.G) * per_group;
  int gi = k / per_group;
  if (gi >= a.G) return total;
  const int t = __ldg(&sched[k - gi * per_group]);
  for (int g0 = 0; g0 < a.G; g0 += 32) {
    const int g = g0 + lane;
    const uint32_t live = __ballot_sync(0xffffffffu, g < a.G && a.group_active[g] != 0u);
    const int n = __popc(live);
    if (gi < n) {
      uint32_t m = live;
      for (int i = 0; i < gi; ++i) m &= m - 1;
      return static_cast<long long>(g0 + __ffs(m) - 1) * per_group + t;
    }
    gi -= n;
  }
  return total;
}

__device__ __forceinline__ long long sched_resolve(const Args& a, int k, int lane, int per_group,
                                                   const int32_t* __restrict__ sched) {
  return sched_map(a, __shfl_sync(0xffffffffu, k, 0), lane, per_group, sched);
}

// ------------------------------------------------------------- k_check --
// One warp = one chunk of 32 consecutive (device-order) checks x 32 slots of
// one group.  Checks are sorted by type (NH edges to degree>=2 variables, ND
// degree-1 edges) when the device layout is built, so almost every chunk is
// homogeneous: its c2v rows are hb + i*NH + j and its degree-1 rows db + i,
// only the H indices of the gathers come from (staged) memory, and the
// typed path below processes K checks at once with straight-line code so
// K*(NH+ND) message loads are in flight per warp.  Mixed chunks (at most one
// per type boundary) and unsupported types take the generic path.
//
// Iteration 1 (decoder.cpp:69-73): post was initialised to the channel LLR
// at load, and the c2v load is skipped, so v2c = llr - 0 = llr, unclamped.
// Later iterations: v2c = clamp(post - c2v) (decoder.cpp:104); degree-1
// edges: clamp(llr) (the reference's clamp((llr + c2v) - c2v)).
template <int MAXD>
struct CheckState {
  float m[MAXD];
  float l1[MAXD];
  int4 d;
  int deg, nh;
  uint32_t sbit, par;
};

template <int MAXD>
__device__ __forceinline__ void check_load(const Args& a, CheckState<MAXD>& s, int g, const int4 d, uint32_t sword,
                                           const int32_t* hh, int lane, bool act, bool first, int lw) {
  constexpr int kUnroll = MAXD <= 16 ? MAXD : 1;
  s.d = d;
  s.nh = d.y - d.x;
  s.deg = s.nh + (d.w - d.z);
  s.sbit = (sword >> lane) & 1u;
  s.par = s.sbit;
  const int lim = MAXD <= 16 ? MAXD : s.deg;
#pragma unroll kUnroll
  for (int j = 0; j < lim; ++j) {
    if (j < s.deg) {
      float v = 0.0f;
      if (j < s.nh) {
        const int h = hh[j];
        if (act) {
          const float p = a.post[rix(g, a.NV, h, lw) + lane];
          const float co = first ? 0.0f : ld_stream(&a.c2v[rix(g, a.EH, d.x + j, lw) + lane]);
          v = first ? p : clampf(p - co, a.clamp);
        }
        s.l1[j] = 0.0f;
      } else {
        const int dd = d.z + (j - s.nh);
        float l = 0.0f;
        if (act) l = ld_stream(&a.llr_d[rix(g, a.N1, dd, lw) + lane]);
        s.l1[j] = l;
        v = first ? l : clampf(l, a.clamp);
      }
      s.m[j] = v;
    }
  }
}

#ifndef BPDEC_PHI_DOMAIN
#define BPDEC_PHI_DOMAIN 0  // 0: t domain (phi.cuh, the shipped form); 1: phi domain (A/B builds)
#endif

// Magnitudes of the outgoing messages from the incoming ones; deg 1: empty
// product -> clamp; deg 2: phi(phi(x)) = x, passed through.
// `m` are magnitudes (already clamped to <= msg_clamp except in iteration 1).
//
// t domain (phi.cuh): t_i = e^-m_i, prefix / suffix (+)-sums, out_j =
// -ln(pre_j (+) suf_j+1).  Raw operands stay raw where the structure allows
// (pre_1, suf_D-1), so a degree-3 or degree-4 check needs no fraction (+)
// fraction.  phi domain: prefix / suffix sums of phi without the additions
// of 0 (phi >= 0, so bit-identical to starting both sums at 0).
//
// DSum: the hi-edge sum a degree-1 decision reads (check_magnitudes_d1):
// a float phi sum or a t-domain fraction.
#if BPDEC_PHI_DOMAIN
using DSum = float;
__device__ __forceinline__ float d1_stat(float x) { return dev::phi(x); }
__device__ __forceinline__ float d1_out(float s, float clamp) { return fminf(dev::phi(s), clamp); }
#else
using DSum = dev::TF;
__device__ __forceinline__ float d1_stat(float x) { return dev::tdom(x); }
__device__ __forceinline__ float d1_out(dev::TF s, float clamp) { return dev::tmag(s, clamp); }

// t-domain outputs of a check of degree D (>= 3) whose inputs are t[0..D-1];
// out[j] for j < NOUT (NOUT = D: all; D - 1: all but the last edge).
// Returns the prefix sum over t[0..D-2] (the hi sum of a d1 check).
template <int D, int NOUT>
__device__ __forceinline__ dev::TF t_outputs(const float (&t)[D], float (&out)[D], float clamp) {
  using dev::TF;
  TF pre[D];  // pre[j] = t[0] (+) ... (+) t[j-1], j >= 2 (pre[1] = t[0], raw)
  pre[2] = dev::tf_pair(t[0], t[1]);
#pragma unroll
  for (int j = 3; j < D; ++j) pre[j] = dev::tf_add(pre[j - 1], t[j - 1]);
  if (NOUT == D) out[D - 1] = dev::tmag(pre[D - 1], clamp);
  // suffix: suf = t[j+1] (+) ... (+) t[D-1], raw while it holds one term
  TF suf = dev::tf_pair(t[D - 2], t[D - 1]);  // j = D - 3
#pragma unroll
  for (int j = D - 2; j >= 0; --j) {
    TF o;
    if (j == D - 2) {
      o = j == 0 ? TF{t[D - 1], 1.0f} : (j == 1 ? dev::tf_pair(t[0], t[D - 1]) : dev::tf_add(pre[j], t[D - 1]));
    } else {
      if (j < D - 3) suf = dev::tf_add(suf, t[j + 1]);
      o = j == 0 ? suf : (j == 1 ? dev::tf_add(suf, t[0]) : dev::tf_join(pre[j], suf));
    }
    out[j] = dev::tmag(o, clamp);
  }
  return pre[D - 1];
}
#endif

template <int D>
__device__ __forceinline__ void check_magnitudes(const float (&m)[D], float (&out)[D], float clamp) {
  if (D == 1) {
    out[0] = clamp;
  } else if (D == 2) {
    out[0] = fminf(m[1], clamp);
    out[1] = fminf(m[D > 1 ? 0 : 0], clamp);
  } else {
#if BPDEC_PHI_DOMAIN
    float ph[D];
    float pre[D];
#pragma unroll
    for (int j = 0; j < D; ++j) ph[j] = dev::phi(m[j]);
    pre[1] = ph[0];
#pragma unroll
    for (int j = 2; j < D; ++j) pre[j] = pre[j - 1] + ph[j - 1];
    out[D - 1] = fminf(dev::phi(pre[D - 1]), clamp);
    float suf = ph[D - 1];
#pragma unroll
    for (int j = D - 2; j >= 1; --j) {
      out[j] = fminf(dev::phi(pre[j] + suf), clamp);
      suf += ph[j];
    }
    out[0] = fminf(dev::phi(suf), clamp);
#else
    float t[D];
#pragma unroll
    for (int j = 0; j < D; ++j) t[j] = dev::tdom(m[j]);
    t_outputs<D, D>(t, out, clamp);
#endif
  }
}

// Check with NH edges to degree>=2 variables and one degree-1 edge whose
// domain value phd (phi or t of its clamped magnitude, d1_stat) is given:
// outputs of the NH hi edges (same prefix / suffix order as
// check_magnitudes<NH+1>, so bit-identical to it when phd =
// d1_stat(m[NH])) and s_hi = the hi edges' sum (the degree-1 edge's output
// is d1_out(s_hi), not formed here).
template <int NH>
__device__ __forceinline__ void check_magnitudes_d1(const float (&m)[NH + 1], float phd, float (&out)[NH + 1],
                                                    float clamp, DSum& s_hi) {
  constexpr int D = NH + 1;
#if BPDEC_PHI_DOMAIN
  float ph[D];
  float pre[D];
#pragma unroll
  for (int j = 0; j < NH; ++j) ph[j] = dev::phi(m[j]);
  ph[NH] = phd;
  pre[1] = ph[0];
#pragma unroll
  for (int j = 2; j < D; ++j) pre[j] = pre[j - 1] + ph[j - 1];
  s_hi = pre[D - 1];
  float suf = ph[D - 1];
#pragma unroll
  for (int j = D - 2; j >= 1; --j) {
    out[j] = fminf(dev::phi(pre[j] + suf), clamp);
    suf += ph[j];
  }
  out[0] = fminf(dev::phi(suf), clamp);
#else
  float t[D];
#pragma unroll
  for (int j = 0; j < NH; ++j) t[j] = dev::tdom(m[j]);
  t[NH] = phd;
  s_hi = t_outputs<D, D - 1>(t, out, clamp);
#endif
}

// Hard decision of a degree-1 variable, post = l + o (o its check's output
// to it), decided without forming o: |o| = min(-ln T_hi, clamp) (t domain;
// phi domain: min(phi(s_hi), clamp)) against |l| through phd = d1_stat(
// min(|l|, clamp)) (both maps decreasing; phd <= phc = d1_stat(clamp) means
// |l| >= clamp).  sl / so: sign bits of l and o.  Same decision as (l + o <
// 0) except where |o| and |l| agree to float rounding (a posterior at zero:
// a tie).
__device__ __forceinline__ uint32_t d1_bit_phi(uint32_t sl, uint32_t so, DSum s_hi, float phd, float phc) {
  // branch-free (selects only: the branchy form compiled to divergent
  // branches and a convergence check before every ballot)
#if BPDEC_PHI_DOMAIN
  const float kInf = __int_as_float(0x7f800000);
  const bool zero = (phd == kInf) & (s_hi == kInf);  // l = 0 and o = 0: +0 or -0, not < 0
  const bool o_lt = s_hi < phd;                      // phi(|o|) < phi(|l|)
  const bool o_gt = s_hi > phd;
#else
  // l = 0 (t = 1) and o = 0 (T_hi = 1, n == d exactly)
  const bool zero = (phd == 1.0f) & (s_hi.n == s_hi.d);
  const float r = phd * s_hi.d;  // T_hi = n / d against t(|l|): n against t*d
  const bool o_lt = s_hi.n < r;
  const bool o_gt = s_hi.n > r;
#endif
  const bool l_small = phd > phc;       // |l| < clamp
  const bool o_big = l_small & o_lt;    // |o| > |l|
  const bool l_big = !l_small | o_gt;   // |l| > |o|  (neither: equal, post = +0)
  const uint32_t diff = o_big ? so : (l_big ? sl : 0u);
  const uint32_t same = zero ? 0u : sl;
  return sl == so ? same : diff;
}

template <int MAXD, bool WANT_POST>
__device__ __forceinline__ uint32_t check_finish(const Args& a, CheckState<MAXD>& s, int g, int lane, bool act, int lw) {
  constexpr int kUnroll = MAXD <= 16 ? MAXD : 1;
  const int deg = s.deg;
  const int lim = MAXD <= 16 ? MAXD : deg;
  uint32_t par = s.par;
#pragma unroll kUnroll
  for (int j = 0; j < lim; ++j)
    if (j < deg) par ^= signbit_u(s.m[j]);
  float out[MAXD];
  if (deg == 1) {
    out[0] = a.clamp;
  } else if (deg == 2) {
    out[0] = fminf(fabsf(s.m[1]), a.clamp);
    out[1] = fminf(fabsf(s.m[0]), a.clamp);
  } else if (deg > 2) {
    float ph[MAXD];
    float pre[MAXD];
    float run = 0.0f;
#pragma unroll kUnroll
    for (int j = 0; j < lim; ++j) {
      if (j < deg) {
        ph[j] = dev::phi(fabsf(s.m[j]));
        pre[j] = run;
        run += ph[j];
      }
    }
    float suf = 0.0f;
#pragma unroll kUnroll
    for (int j = lim - 1; j >= 0; --j) {
      if (j < deg) {
        out[j] = fminf(dev::phi(pre[j] + suf), a.clamp);
        suf += ph[j];
      }
    }
  }
  uint32_t dpar = 0u;
#pragma unroll kUnroll
  for (int j = 0; j < lim; ++j) {
    if (j < deg) {
      const float o = with_sign(out[j], par ^ signbit_u(s.m[j]));
      if (j < s.nh) {
        if (act) st_stream(&a.c2v[rix(g, a.EH, s.d.x + j, lw) + lane], o);
      } else {
        const int dd = s.d.z + (j - s.nh);
        const float pd = s.l1[j] + o;  // posterior of the degree-1 variable
        const uint32_t bit = (act && pd < 0.0f) ? 1u : 0u;
        dpar ^= bit;
        const uint32_t word = __ballot_sync(0xffffffffu, bit);
        if (lane == 0) a.d1bits[static_cast<size_t>(g) * a.N1 + dd] = word;
        if (WANT_POST && act) a.d1post[rix(g, a.N1, dd, lw) + lane] = pd;
      }
    }
  }
  return __ballot_sync(0xffffffffu, (s.sbit ^ dpar) & 1u);
}

// Typed chunk: 32 checks, each with NH edges to degree>=2 variables (c2v rows
// hb + 32-check-local i*NH + j) and ND <= 1 degree-1 edge (row db + i).
// K checks form a batch of R = K*(2*NH+ND) message rows.  Batches are
// copied asynchronously (16-byte cp.async: a warp instruction moves four
// 128-byte rows) into a per-warp shared-memory ring of NS stages: NS-1
// batches are in flight while one is computed from shared memory, and no
// registers are held for data in flight.  Lanes read rows other lanes
// copied, so a __syncwarp follows each cp.async.wait_group.
constexpr int kStageRows = 20;  // rows per batch stage (check shapes)
constexpr int kStages = 3;      // minimum ring depth (stages of kStageRows rows)
constexpr int kRingRows = kStages * kStageRows;

// NOC2V: the batch stages no previous-c2v rows (steady-state (1,1) checks,
// whose c2v is a constant of the frame), so twice as many checks fit a stage.
// Narrow groups (LW < 32): rows are LW floats, so a stage and the ring
// hold 32/LW times the rows (bigger batches, fewer per chunk).
template <int NH, int ND, int RING = kRingRows, bool NOC2V = false, int LW = 32>
struct CheckShape {
  static constexpr int CR = NOC2V ? 0 : NH;  // previous-c2v rows per check
  static constexpr int RPC = NH + CR + ND;   // rows per check
  static constexpr int SR = kStageRows * (32 / LW);  // stage rows
  static constexpr int RR = RING * (32 / LW);        // ring rows
  static constexpr int K = RPC == 0 ? 8 : (SR / RPC >= 8 ? 8 : (SR / RPC >= 4 ? 4 : (SR / RPC >= 2 ? 2 : 1)));
  static_assert(K * RPC <= SR, "stage too small");
  // the per-warp ring (kRingRows) is cut into as many stages of this shape's
  // batch size as fit (light shapes keep more batches in flight)
  static constexpr int ROWS = RPC == 0 ? 1 : K * RPC;
  static constexpr int NS = RR / ROWS >= 6 ? 6 : RR / ROWS;
  static_assert(NS >= kStages, "at least the default ring depth");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte copy: lane l moves floats [4(l%8), 4(l%8)+4) of row (l/8) of a
// 4-row group, so one warp instruction moves four 128-byte rows.
__device__ __forceinline__ void cp_async16(float* sdst, const float* gsrc, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
               "r"(pred ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async16_ef(float* sdst, const float* gsrc, bool pred, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(smem_u32(sdst)),
               "l"(gsrc), "r"(pred ? 16 : 0), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}

// Stage layout for a batch of K checks: [K*NH posterior rows][K*NH c2v rows]
// [K*ND llr rows], rows of LW floats.  `lrow`/`lcol` = this lane's 16-byte
// piece: a warp instruction moves 128/LW rows (LW = 32: four 128-byte
// rows); `qact` = any of the 4 frames covered by that piece is active.
// C2V = false: the previous c2v rows are not needed (steady-state (1,1)
// checks, whose c2v is a constant of the frame, see check_batch_compute).
template <int NH, int ND, int LW, bool C2V = true>
__device__ __forceinline__ void check_batch_issue(float* stage, const float* post0, const float* c2v0,
                                                  const float* llr0, const int32_t* hh, int i0, int lrow, int lcol,
                                                  bool qact, bool qc2v, uint64_t pol) {
  using SH = CheckShape<NH, ND, kRingRows, !C2V, LW>;
  constexpr int K = SH::K;
  constexpr int NPH = K * NH;       // posterior rows
  constexpr int NPC = K * SH::CR;   // previous-c2v rows (0 without C2V)
  constexpr int NPD = K * ND;       // degree-1 rows
  constexpr int RPI = 128 / LW;  // rows per warp instruction
#if BPDEC_POST_EVICT_LAST
  const uint64_t polp = policy_evict_last();
#endif
#pragma unroll
  for (int r0 = 0; r0 < NPH; r0 += RPI) {
    const int r = r0 + lrow;
    if (r < NPH) {
      const int h = hh[i0 * NH + r];
#if BPDEC_POST_EVICT_LAST
      cp_async16_ef(stage + r * LW + lcol, post0 + static_cast<size_t>(h) * LW + lcol, qact, polp);
#else
      cp_async16(stage + r * LW + lcol, post0 + static_cast<size_t>(h) * LW + lcol, qact);
#endif
      if (C2V)
        cp_async16_ef(stage + (NPH + r) * LW + lcol, c2v0 + static_cast<size_t>(i0 * NH + r) * LW + lcol, qc2v, pol);
    }
  }
#pragma unroll
  for (int r0 = 0; r0 < NPD; r0 += RPI) {
    const int r = r0 + lrow;
    if (r < NPD)
      cp_async16_ef(stage + (NPH + NPC + r) * LW + lcol, llr0 + static_cast<size_t>(i0 + r) * LW + lcol, qact, pol);
  }
  cp_async_commit();
}

// FM: some lane of the warp is in its first iteration (v2c = channel LLR,
// unclamped, no previous c2v).  The steady state runs the FM = false copy.
//
// LW < 32 (narrow group, steady state only): the warp is folded — lane
// (q = lane / LW, f = lane % LW) computes check kb + q of each sub-batch of
// FE = min(32/LW, K) checks for the frame in lane f — so a narrow group
// costs ~LW/32 of the instructions as well as of the bytes.  The arithmetic
// of every (check, frame) is that of LW = 32; the 32-bit words (degree-1
// hard bits, syndrome part) of check kb + qq are bits qq*LW .. of one ballot.
//
// kPhiD (one degree-1 edge and >= 2 hi edges, no posterior output): the
// degree-1 LLR row holds, after the frame's first iteration, phi(min(|l|,
// clamp)) with l's sign (written back by the first iteration), so the steady
// state reads the degree-1 edge's phi instead of computing it and decides
// the degree-1 hard bit in the phi domain (d1_bit_phi) instead of forming
// its output: two phi evaluations less per check.  The messages to the hi
// edges are bit-identical to the plain path.
template <int NH, int ND, bool WANT_POST, bool FM, int LW, bool PHID>
__device__ __forceinline__ void check_batch_compute(const float* stage, float* c2vg, float* d1p, float* llrg,
                                                    const uint32_t* ssyn, int i0, int lane, bool act, bool first,
                                                    float cl, float clamp, float phc, uint32_t* synw,
                                                    uint32_t* d1w) {
  constexpr int D = NH + ND;
  constexpr bool kPhiD = PHID && ND == 1 && NH >= 2 && !WANT_POST;
  // steady-state (1,1) check: the c2v to its degree>=2 variable is
  // (1-2s)*sign(l)*min(|l|, clamp) in every iteration (the degree-1 edge's
  // v2c is clamp(l)), so it is formed from l instead of being re-read (the
  // stage has no c2v rows), and the stored copy (written in the frame's
  // first iteration, moved with the frame) is not rewritten: 8 bytes per
  // check and frame less per pass
  constexpr bool kConstC = NH == 1 && ND == 1 && !FM;
  using SH = CheckShape<NH, ND, kRingRows, kConstC, LW>;
  constexpr int K = SH::K;
  constexpr int NPH = K * NH;
  constexpr int NPC = K * SH::CR;
  constexpr int F = 32 / LW;
  constexpr int FE = F < K ? F : K;  // checks per folded step
  constexpr uint32_t kSign = 0x80000000u;
  const int q = LW == 32 ? 0 : lane / LW;
  const int f = LW == 32 ? lane : lane % LW;
  const bool qok = q < FE;
  const bool on = act && qok;
  // this lane's rows: check kb + q of sub-batch kb
  const float* sp = stage + f + q * NH * LW;                // posterior rows
  const float* sc = stage + f + (NPH + q * SH::CR) * LW;   // previous c2v rows (none with kConstC)
  const float* sl = stage + f + (NPH + NPC + q) * LW;      // degree-1 llr rows
  float* cq = c2vg + q * NH * LW;
  float* dq = WANT_POST ? d1p + q * LW : nullptr;
#pragma unroll
  for (int kb = 0; kb < K; kb += FE) {
    float m[D > 0 ? D : 1];      // |v2c|, clamped (cl = inf in the first iteration)
    uint32_t sm[D > 0 ? D : 1];  // sign masks of v2c (the clamp keeps the sign)
    float l = 0.0f;
    if (ND) l = sl[kb * LW];
    const int ci = i0 + kb + (qok ? q : 0);  // this lane's check (chunk-local)
    const uint32_t sbit = (ssyn[ci] >> f) & 1u;
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      const float c = kConstC ? __uint_as_float(__float_as_uint(fminf(fabsf(l), clamp)) |
                                                ((sbit << 31) ^ (__float_as_uint(l) & kSign)))
                              : sc[(kb * NH + j) * LW];
      const float v = sp[(kb * NH + j) * LW] - (FM && first ? 0.0f : c);
      m[j] = fminf(fabsf(v), FM ? cl : clamp);
      sm[j] = __float_as_uint(v) & kSign;
    }
    if (ND) {
      m[NH] = fminf(fabsf(l), FM ? cl : clamp);
      sm[NH] = __float_as_uint(l) & kSign;
    }
    uint32_t par = sbit << 31;  // sign of the product times (1 - 2 s_c)
#pragma unroll
    for (int j = 0; j < D; ++j) par ^= sm[j];
    float out[D > 0 ? D : 1];
    uint32_t dbit = 0u;
    if constexpr (kPhiD) {
      // steady lanes: l is the stored phi (sign = l's); first-iteration
      // lanes (FM copy only): l is the LLR, phi formed here and stored
      float phd = fabsf(l);
      float phf = 0.0f;
      if (FM) {
        phf = d1_stat(m[NH]);  // unclamped in the first iteration (cl = inf)
        if (first) phd = phf;
      }
      DSum s_hi;
      check_magnitudes_d1<NH>(m, phd, out, clamp, s_hi);
      const uint32_t so = (par ^ sm[NH]) >> 31, sl = sm[NH] >> 31;
      if (FM) {
        // first lanes: the plain decision on the LLR, and the phi of the
        // clamped magnitude written back for the steady state
        const float o = __uint_as_float(__float_as_uint(d1_out(s_hi, clamp)) | (par ^ sm[NH]));
        const uint32_t fb = (l + o < 0.0f) ? 1u : 0u;
        dbit = first ? fb : d1_bit_phi(sl, so, s_hi, phd, phc);
        const float stored = __uint_as_float(__float_as_uint(fabsf(l) > clamp ? phc : phf) | sm[NH]);
        st_pred(llrg + static_cast<size_t>(i0 + kb) * LW, stored, on && first);
      } else {
        dbit = d1_bit_phi(sl, so, s_hi, phd, phc);
      }
      dbit = on ? dbit : 0u;
    } else {
      check_magnitudes<D>(m, out, clamp);
    }
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      const float o = __uint_as_float(__float_as_uint(out[j]) | (par ^ sm[j]));
      if (!kConstC) stcs_pred(cq + static_cast<size_t>((i0 + kb) * NH + j) * LW, o, on);
    }
    if (ND && !kPhiD) {
      const float o = __uint_as_float(__float_as_uint(out[NH]) | (par ^ sm[NH]));
      const float pd = l + o;  // posterior of the degree-1 variable
      dbit = (on && pd < 0.0f) ? 1u : 0u;
      if (WANT_POST) st_pred(dq + static_cast<size_t>(i0 + kb) * LW, pd, on);
    }
    if constexpr (LW == 32) {
      // the syndrome word is the target word xor the degree-1 word (a
      // ballot is linear over xor): one ballot per check, not two
      uint32_t dw = 0u;
      if (ND) {
        dw = __ballot_sync(0xffffffffu, dbit);
        if (lane == ci) *d1w = dw;
      }
      if (lane == ci) *synw = ssyn[ci] ^ dw;
    } else {
      constexpr uint32_t kMask = (1u << LW) - 1u;
      const uint32_t bd = ND ? __ballot_sync(0xffffffffu, dbit) : 0u;
      const uint32_t bs = __ballot_sync(0xffffffffu, qok && ((sbit ^ dbit) & 1u));
#pragma unroll
      for (int qq = 0; qq < FE; ++qq) {
        if (lane == i0 + kb + qq) {
          if (ND) *d1w = (bd >> (qq * LW)) & kMask;
          *synw = (bs >> (qq * LW)) & kMask;
        }
      }
    }
  }
}

template <int NH, int ND, bool WANT_POST, bool FM, int RING, int LW = 32, bool PHID = false>
__device__ __forceinline__ void check_chunk_loop(const Args& a, int g, int hb, int db, const int32_t* hh,
                                                 const uint32_t* ssyn, float* ring, int lane, bool act, bool first,
                                                 uint32_t amask, uint32_t fmask, uint32_t* synw, uint32_t* d1w) {
  constexpr bool kNoC = NH == 1 && ND == 1 && !FM;  // steady-state (1,1): no c2v rows staged
  using SH = CheckShape<NH, ND, RING, kNoC, LW>;
  constexpr int K = SH::K;
  constexpr int NB = 32 / K;
  const int f = LW == 32 ? lane : lane % LW;  // this lane's frame (slot lane)
  if (LW < 32) act = (amask >> f) & 1u;
  const float* post0 = a.post + rix(g, a.NV, 0, LW);
  const float* c2v0 = a.c2v + rix(g, a.EH, hb, LW);
  const float* llr0 = a.llr_d + rix(g, a.N1, db, LW);
  float* c2vg = a.c2v + rix(g, a.EH, hb, LW) + f;
  float* d1p = WANT_POST ? a.d1post + rix(g, a.N1, db, LW) + f : nullptr;
  float* llrg = a.llr_d + rix(g, a.N1, db, LW) + f;
  const float clamp = a.clamp;
  const float cl = first ? __int_as_float(0x7f800000) : clamp;
  const float phc = d1_stat(clamp);
  // this lane's 16-byte piece: frames lcol .. lcol+3 of row lrow of a row group
  constexpr int QPR = LW / 4;  // 16-byte pieces per row
  const int lrow = lane / QPR;
  const int lcol = (lane % QPR) * 4;
  const uint32_t qbits = (amask >> lcol) & 0xFu;
  const bool qact = qbits != 0u;
  const bool qc2v = (qbits & ~(fmask >> lcol)) != 0u;  // some active frame past its first iteration
  const uint64_t pol = policy_evict_first();
  constexpr int NS = SH::NS;
  constexpr int RS = SH::ROWS * LW;  // stage stride (floats)
  // one commit group per step (empty past the last batch), so the wait
  // count is a constant
#pragma unroll
  for (int p = 0; p < NS - 1; ++p) {
    if (p < NB)
      check_batch_issue<NH, ND, LW, !kNoC>(ring + p * RS, post0, c2v0, llr0, hh, p * K, lrow, lcol, qact, qc2v, pol);
    else
      cp_async_commit();
  }
  int slot_i = NS - 1, slot_c = 0;  // ring stages of the next batch to issue / compute
#pragma unroll 1
  for (int b = 0; b < NB; ++b) {
    if (b + NS - 1 < NB)
      check_batch_issue<NH, ND, LW, !kNoC>(ring + slot_i * RS, post0, c2v0, llr0, hh, (b + NS - 1) * K, lrow, lcol, qact,
                                    qc2v, pol);
    else
      cp_async_commit();
    if (++slot_i == NS) slot_i = 0;
    cp_async_wait<NS - 1>();
    __syncwarp();  // rows were copied by other lanes
    check_batch_compute<NH, ND, WANT_POST, FM, LW, PHID>(ring + slot_c * RS, c2vg, d1p, llrg, ssyn, b * K, lane, act, first,
                                                   cl, clamp, phc, synw, d1w);
    if (++slot_c == NS) slot_c = 0;
    __syncwarp();  // stage is refilled in the next round
  }
}

// SPLIT_FM: a separate steady-state copy (no first-iteration lanes) of the
// chunk loop.  Kernels for codes with heavy check types (MAXD >= 6) keep the
// general copy only: twice the typed code would thrash the instruction cache.
// Narrow groups (LW < 32) never have first-iteration lanes (the frame queue
// is drained before a group is narrowed).
template <int NH, int ND, bool WANT_POST, bool SPLIT_FM, int RING, int LW>
__device__ __forceinline__ void check_chunk_typed(const Args& a, int g, int hb, int db, const int32_t* hh,
                                                  const uint32_t* ssyn, float* ring, int lane, bool act, bool first,
                                                  uint32_t amask, uint32_t fmask, uint32_t* synw, uint32_t* d1w) {
  // the phi-domain degree-1 edge needs the steady-state copy (the general
  // copy would evaluate both forms: measured slower)
  if constexpr (LW < 32)
    check_chunk_loop<NH, ND, WANT_POST, false, RING, LW, SPLIT_FM>(a, g, hb, db, hh, ssyn, ring, lane, act, first,
                                                                   amask, 0u, synw, d1w);
  else if (!SPLIT_FM || fmask)
    check_chunk_loop<NH, ND, WANT_POST, true, RING, 32, SPLIT_FM>(a, g, hb, db, hh, ssyn, ring, lane, act, first,
                                                                  amask, fmask, synw, d1w);
  else
    check_chunk_loop<NH, ND, WANT_POST, false, RING, 32, SPLIT_FM>(a, g, hb, db, hh, ssyn, ring, lane, act, first,
                                                                   amask, fmask, synw, d1w);
}

template <int MAXD>
struct CheckSmem {
  static constexpr bool kStage = MAXD <= 16;
  static constexpr int kHH = kStage ? 32 * MAXD : 1;
  // ring rows per warp: 80 (four stages of the heaviest typed batch) where
  // the static shared memory allows it, else 60
  static constexpr int kRing = MAXD <= 4 ? 80 : kRingRows;
  int4 desc[kCheckThreads / 32][32];
  uint32_t syn[kCheckThreads / 32][32];
  int32_t hh[kCheckThreads / 32][kHH];
  __align__(16) float ring[kCheckThreads / 32][kRing * kLanes];
};

// The chunk loop of k_check for groups laid out with lane width LW.
template <int MAXD, bool WANT_POST, int LW>
__device__ __forceinline__ void check_body(const Args& a, CheckSmem<MAXD>& sm) {
  constexpr bool kStage = CheckSmem<MAXD>::kStage;
  constexpr int kRing = CheckSmem<MAXD>::kRing;
  auto& s_desc = sm.desc;
  auto& s_syn = sm.syn;
  auto& s_hh = sm.hh;
  auto& s_ring = sm.ring;
  const int lane = threadIdx.x & 31;
  const int wi = threadIdx.x >> 5;
  const bool moved = __ldcg(&a.counters[12]) != 0;
  const int chunks = (a.M + 31) / 32;
  const long long total = static_cast<long long>(a.G) * chunks;
  // dynamic chunk schedule (counters[7], generic chunks first): a grab is
  // kCheckGrab consecutive chunks per atomic (1: two consecutive chunks on
  // one warp measured 9 % slower than side by side on two warps; a static
  // warp-strided assignment 23 % slower: chunk costs differ by type), the
  // next grab in flight while the current one is processed
  int kbase = __shfl_sync(0xffffffffu, sched_issue_n(a, 7, lane, kCheckGrab), 0);
  int kpend = sched_issue_n(a, 7, lane, kCheckGrab);
  int sub = 0;
  auto next_chunk = [&]() {
    if (++sub == kCheckGrab) {
      sub = 0;
      kbase = __shfl_sync(0xffffffffu, kpend, 0);
      kpend = sched_issue_n(a, 7, lane, kCheckGrab);
    }
    return sched_map(a, kbase + sub, lane, chunks, a.csched);
  };
  long long w = sched_map(a, kbase, lane, chunks, a.csched);
  while (w < total) {
    const int g = static_cast<int>(w / chunks);
    const int ch = static_cast<int>(w - static_cast<long long>(g) * chunks);
    const int c0 = ch * 32;
    const int nc = min(32, a.M - c0);
    // the chunk's independent setup loads first (one round trip instead of
    // a chain: the slot iteration is loaded for every lane and masked, the
    // target syndrome word before the skip test)
    const int4 cdk = __ldg(&a.ctype[ch]);
    const uint32_t amask = a.group_active[g];
    const int it_raw = a.slot_iter[g * kLanes + lane];
    const uint32_t sy = lane < nc ? a.syn_target[static_cast<size_t>(g) * a.M + c0 + lane] : 0u;
    const bool act = (amask >> lane) & 1u;
    const int it = act ? it_raw : 0;
    const bool first = (it == 1);
    const uint32_t fmask = __ballot_sync(0xffffffffu, act && first);
    const int type = kStage ? cdk.x : -1;
    // degree-1 checks only change in a frame's first iteration (and their
    // bit words must follow frames that k_compact moved)
    if ((type == 1 || type == 8) && fmask == 0u && !moved) {
      w = next_chunk();
      continue;
    }
    __syncwarp();
    if (lane < nc) s_syn[wi][lane] = sy;
    int hb0 = cdk.y;  // = the first check's descriptor .x for generic chunks too
    if (type < 0) {  // generic chunk: per-check descriptors
      if (lane < nc) s_desc[wi][lane] = __ldg(&a.cdesc[c0 + lane]);
      __syncwarp();
      hb0 = s_desc[wi][0].x;
    }
    if (kStage) {
      const int nhh = cdk.w - hb0;
      for (int i = lane; i < nhh; i += 32) s_hh[wi][i] = __ldg(&a.chk_hi_h[hb0 + i]);
    }
    __syncwarp();
    uint32_t synw = 0u, d1w = 0u;
    const int db0 = cdk.z;
    bool typed = true;
    switch (type) {
#define BPDEC_TYPED(NH_, ND_)                                                                       \
  case NH_ * 8 + ND_:                                                                               \
    if (NH_ + ND_ <= MAXD)                                                                          \
      check_chunk_typed<NH_, ND_, WANT_POST, (MAXD <= kSplitMaxD), kRing, LW>(a, g, hb0, db0, s_hh[wi], s_syn[wi], s_ring[wi], \
                                             lane, act, first, amask, fmask, &synw, &d1w);          \
    else                                                                                            \
      typed = false;                                                                                \
    break;
      BPDEC_TYPED(0, 1)
      BPDEC_TYPED(1, 0)
      BPDEC_TYPED(1, 1)
      BPDEC_TYPED(2, 0)
      BPDEC_TYPED(2, 1)
      BPDEC_TYPED(3, 0)
      BPDEC_TYPED(3, 1)
      BPDEC_TYPED(4, 0)
      BPDEC_TYPED(4, 1)
      BPDEC_TYPED(5, 0)
      BPDEC_TYPED(5, 1)
      BPDEC_TYPED(6, 0)
#undef BPDEC_TYPED
      default:
        typed = false;
    }
    if (typed) {
      if ((type & 7) != 0) a.d1bits[static_cast<size_t>(g) * a.N1 + db0 + lane] = d1w;
    } else {
      // two checks in flight per step in k_check<3>; one in the wider
      // kernels (two states of MAXD >= 4 messages spill)
      constexpr int kGenPair = MAXD <= 3 ? 2 : 1;
      for (int j = 0; j < nc; j += kGenPair) {
        CheckState<MAXD> A, B;
        const int4 dA = s_desc[wi][j];
        check_load<MAXD>(a, A, g, dA, s_syn[wi][j], kStage ? &s_hh[wi][dA.x - hb0] : &a.chk_hi_h[dA.x], lane, act,
                         first, LW);
        const bool hasB = kGenPair == 2 && j + 1 < nc;
        if (hasB) {
          const int4 dB = s_desc[wi][j + 1];
          check_load<MAXD>(a, B, g, dB, s_syn[wi][j + 1], kStage ? &s_hh[wi][dB.x - hb0] : &a.chk_hi_h[dB.x], lane,
                           act, first, LW);
        }
        const uint32_t wa = check_finish<MAXD, WANT_POST>(a, A, g, lane, act, LW);
        if (lane == j) synw = wa;
        if (hasB) {
          const uint32_t wb = check_finish<MAXD, WANT_POST>(a, B, g, lane, act, LW);
          if (lane == j + 1) synw = wb;
        }
      }
    }
    if (lane < nc) a.synp[static_cast<size_t>(g) * a.M + c0 + lane] = synw;
    w = next_chunk();
  }
}

template <int MAXD, bool WANT_POST>
__global__ void __launch_bounds__(kCheckThreads, MAXD >= 16 ? kCheckMinBlocks - 1 : kCheckMinBlocks)
    k_check(const Args a) {  // the degree-16 / generic kernels: 4 blocks (128 registers, no spills)  // 5 blocks/SM, 96 regs: measured best
  pdl_begin();
  __shared__ CheckSmem<MAXD> sm;
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < a.G; t += blockDim.x) a.fail[t] = 0u;
    if (threadIdx.x == 0) a.counters[6] = 0;  // k_var tile scheduler (this step)
  }
  // lane width of the live groups' layout (narrow tail, k_compact); only
  // codes with check degree <= 4 are ever narrowed
  const int lw = MAXD <= 4 ? __ldcg(&a.counters[11]) : 32;
  if constexpr (MAXD <= 4) {
    if (lw == 8) {
      check_body<MAXD, WANT_POST, 8>(a, sm);
      return;
    }
    if (lw == 16) {
      check_body<MAXD, WANT_POST, 16>(a, sm);
      return;
    }
  }
  check_body<MAXD, WANT_POST, 32>(a, sm);
}

// --------------------------------------------------------------- k_var --
// A warp owns tiles of kQTile = 64 consecutive (device-order) degree>=2
// variables x 32 slots (tiles w, w + warps, ...).  Variables are sorted by
// degree, so almost every tile is homogeneous (degree D): the warp then runs
// ONE continuous cp.async pipeline over the batches of all its consecutive
// degree-D tiles — the CSC slice (edge ids) of the next tile is prefetched
// into the second half of a double buffer while the current tile is summed,
// and the first batches of the next tile are issued while the current one
// drains, so the random c2v row gathers stay in flight across tile
// boundaries.  Per variable: post = llr + sum of c2v in ascending original
// check order (decoder.cpp:99-105), the hard-decision word (ballot over the
// 32 slots) to hbits and to every edge of the variable (ebits, the
// check-major copy the syndrome kernel streams).  The tile's q partial is
// chunk0 + chunk1, each summed in variable order — an order fixed by the code
// (not by slots, batch size or GPU count).
constexpr int kVarRingRows = 40;   // per-warp ring of the variable kernel (rows of 128 B; 48/56 measured slower)
constexpr int kVarStageRows = 13;  // target rows per batch of the variable kernel (degree 12 unsplit)
constexpr int kVarMaxTyped = 32;   // largest tile degree on the typed (streamed) path

// Batch shape of degree-D tiles.  D + 1 <= kVarStageRows: K whole variables
// per batch (R = K(D+1) rows: K llr rows, then K*D c2v rows).  Larger D: one
// variable spans SB batches of R rows (its llr row, then its c2v rows in
// ascending check order); the posterior sum is carried across them in
// order.
template <int D, int LW = 32>
struct VarShape {
  // narrow groups (LW < 32): rows are LW floats, so the same ring bytes hold
  // 32/LW times the rows and a batch holds up to 4 variables (the fold)
  static constexpr int kStage = kVarStageRows * (32 / LW);
  static constexpr int kRing = kVarRingRows * (32 / LW);
  static constexpr int RV = D + 1;  // rows per variable
  static constexpr bool kSplit = RV > kStage;
  static constexpr int K0 = kSplit ? 1
                            : (kStage / RV >= 8 ? 8 : (kStage / RV >= 4 ? 4 : (kStage / RV >= 2 ? 2 : 1)));
  static constexpr int K = LW < 32 && K0 > 4 ? 4 : K0;
  static constexpr int SB = kSplit ? (RV + kStage - 1) / kStage : 1;  // batches per variable
  static constexpr int ROWS = kSplit ? (RV + SB - 1) / SB : K * RV;    // rows per batch
  static constexpr int NB = 32 / K * SB;                              // batches per chunk
  static constexpr int NS0 = kRing / ROWS >= 6 ? 6 : kRing / ROWS;      // ring stages
  static constexpr int NS = LW < 32 && NS0 > (NB + 1) / 2 ? (NB + 1) / 2 : NS0;
  static_assert(NS >= 2, "variable batch too large for the ring");
  static_assert(D <= kVarMaxTyped, "typed variable path limited to degree 32");
};

// Batch b of a chunk (variables i0 .. of the chunk).  Edge id -1 pads a
// variable of lower degree to the tile degree D, and variables at or beyond
// `nval` pad the last tile: their copies are predicated off, which
// zero-fills the stage rows (+0.0 leaves the ordered sum unchanged).  Rows
// of LW floats (narrow groups: LW = 16 / 8, see rix).
template <int D, int LW>
__device__ __forceinline__ void var_batch_issue(float* stage, const float* llr0, const float* c2vg, const int32_t* ve,
                                                int b, int nval, int lrow, int lcol, bool qact, uint64_t pol) {
  using S = VarShape<D, LW>;
  constexpr int K = S::K;
  constexpr int RPI = 128 / LW;  // rows per warp instruction
  if constexpr (!S::kSplit) {
    const int i0 = b * K;
#pragma unroll
    for (int r0 = 0; r0 < K; r0 += RPI) {
      const int r = r0 + lrow;
      if (r < K)
        cp_async16_ef(stage + r * LW + lcol, llr0 + static_cast<size_t>(i0 + r) * LW + lcol, qact && i0 + r < nval,
                      pol);
    }
#pragma unroll
    for (int r0 = 0; r0 < K * D; r0 += RPI) {
      const int r = r0 + lrow;
      if (r < K * D) {
        const int e = ve[i0 * D + r];
        cp_async16_ef(stage + (K + r) * LW + lcol,
                      c2vg + static_cast<size_t>(static_cast<uint32_t>(max(e, 0))) * LW + lcol, qact && e >= 0, pol);
      }
    }
  } else {
    const int i = b / S::SB;
    const int g0 = (b - i * S::SB) * S::ROWS;  // first variable row of this batch
#pragma unroll
    for (int r0 = 0; r0 < S::ROWS; r0 += RPI) {
      const int r = r0 + lrow;
      const int gr = g0 + r;
      if (r < S::ROWS && gr < S::RV) {
        const int e = gr > 0 ? ve[i * D + gr - 1] : 0;
        const float* src = gr == 0 ? llr0 + static_cast<size_t>(i) * LW
                                   : c2vg + static_cast<size_t>(static_cast<uint32_t>(max(e, 0))) * LW;
        cp_async16_ef(stage + r * LW + lcol, src + lcol, qact && (gr == 0 ? i < nval : e >= 0), pol);
      }
    }
  }
}

// Outputs of variables i0 .. i0+FE-1 (posterior p of this lane's frame f and
// variable i0 + q; `act` = that frame is live and the lane not idle):
// posterior row, q partial, hard-decision word (hbits via hw, and every
// edge's ebits).  Folded (FE > 1): `p` of variable i0 + qq is fetched from
// lane qq*LW + f, so the q partial is summed in variable order exactly as
// with LW = 32.
template <int D, int QMODE, int LW, int FE>
__device__ __forceinline__ void var_finish(float p, float* postg, uint32_t* ebg, const int32_t* ve, int i0, int nval,
                                           int lane, int q, int f, bool act, double& acc, uint32_t& hw) {
  const bool on = act && i0 + q < nval;
#if BPDEC_POST_EVICT_LAST >= 2
  uint64_t polp;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(polp));
  st_pred_pol(postg + static_cast<size_t>(i0 + q) * LW, p, on, polp);
#else
  st_pred(postg + static_cast<size_t>(i0 + q) * LW, p, on);
#endif
  if constexpr (FE == 1) {
    if (on) acc += QMODE == 0 ? static_cast<double>(p) : static_cast<double>(fabsf(p));
  } else {
#pragma unroll
    for (int qq = 0; qq < FE; ++qq) {  // this frame's posteriors in variable order
      const float pv = __shfl_sync(0xffffffffu, p, qq * LW + f);
      if (act && i0 + qq < nval) acc += QMODE == 0 ? static_cast<double>(pv) : static_cast<double>(fabsf(pv));
    }
  }
  const uint32_t bal = __ballot_sync(0xffffffffu, on && p < 0.0f);
#pragma unroll
  for (int qq = 0; qq < FE; ++qq) {
    const int i = i0 + qq;
    const uint32_t word = LW == 32 ? bal : (bal >> (qq * LW)) & ((1u << (LW & 31)) - 1u);
    if (lane == (i & 31)) hw = word;
#pragma unroll
    for (int j0 = 0; j0 < D; j0 += 32) {
      const int j = j0 + lane;
      const int e = ve[i * D + (j < D ? j : 0)];
#if BPDEC_EBITS_EVL
      st_pred_u32_pol(ebg + static_cast<uint32_t>(max(e, 0)), word, j < D && e >= 0, policy_evict_last_nv());
#else
      st_pred_u32(ebg + static_cast<uint32_t>(max(e, 0)), word, j < D && e >= 0);
#endif
    }
  }
}

template <int D, int QMODE, int LW>
__device__ __forceinline__ void var_batch_compute(const float* stage, float* postg, uint32_t* ebg, const int32_t* ve,
                                                  int b, int nval, int lane, bool act, double& acc, uint32_t& hw,
                                                  float& carry) {
  using S = VarShape<D, LW>;
  constexpr int K = S::K;
  constexpr int F = S::kSplit ? 1 : 32 / LW;
  constexpr int FE = F < K ? F : K;  // variables per folded step
  const int qr = LW == 32 ? 0 : lane / LW;  // lanes with qr >= FE idle (q = 0 keeps their reads in range)
  const int q = qr < FE ? qr : 0;
  const int f = LW == 32 ? lane : lane % LW;
  if constexpr (!S::kSplit) {
    const int i0 = b * K;
    const bool on = act && qr < FE;
    const float* st = stage + f + q * LW;
    const float* sc = stage + f + (K + q * D) * LW;
#pragma unroll
    for (int kb = 0; kb < K; kb += FE) {
      float p = st[kb * LW];
#pragma unroll
      for (int j = 0; j < D; ++j) p += sc[(kb * D + j) * LW];  // ascending check order (decoder.cpp:101)
      var_finish<D, QMODE, LW, FE>(p, postg, ebg, ve, i0 + kb, nval, lane, q, f, on, acc, hw);
    }
  } else {
    const int i = b / S::SB;
    const int sub = b - i * S::SB;
    const int n = min(S::ROWS, S::RV - sub * S::ROWS);  // rows of this batch
    const float* st = stage + f;
    float p = sub == 0 ? st[0] : carry + st[0];
#pragma unroll
    for (int j = 1; j < S::ROWS; ++j)
      if (j < n) p += st[j * LW];  // ascending check order (decoder.cpp:101)
    if (sub == S::SB - 1)
      var_finish<D, QMODE, LW, 1>(p, postg, ebg, ve, i, nval, lane, 0, f, act && lane < LW, acc, hw);
    else
      carry = p;
  }
}

struct VarTile {
  int g, tile, h0, kb;
};

__device__ __forceinline__ VarTile var_tile(const Args& a, long long w, int kb) {
  VarTile t;
  t.g = static_cast<int>(w / a.n_tiles);
  t.tile = static_cast<int>(w - static_cast<long long>(t.g) * a.n_tiles);
  t.h0 = t.tile * kQTile;
  t.kb = kb;
  return t;
}
__device__ __forceinline__ VarTile var_tile(const Args& a, long long w) {
  return var_tile(a, w, __ldg(&a.vtile[static_cast<int>(w % a.n_tiles)]).y);
}

// k_var tiles: counters[6], schedule vsched (generic tiles first).
__device__ __forceinline__ int var_grab_issue(const Args& a, int lane) { return sched_issue(a, 6, lane); }
__device__ __forceinline__ long long var_grab_resolve(const Args& a, int k, int lane) {
  return sched_resolve(a, k, lane, a.n_tiles, a.vsched);
}
__device__ __forceinline__ long long var_grab(const Args& a, int lane) {
  return var_grab_resolve(a, var_grab_issue(a, lane), lane);
}

// Stages one chunk's edge ids (32*D contiguous ints from kb) with 16-byte
// cp.async (4-byte copies when kb is not 16-byte aligned).
template <int D>
__device__ __forceinline__ void var_stage_ve(int32_t* dst, const int32_t* vedge, int kb, int lane) {
  constexpr int n = 32 * D;
  if ((kb & 3) == 0) {
#pragma unroll
    for (int i = lane * 4; i < n; i += 128)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + i)), "l"(vedge + kb + i)
                   : "memory");
  } else {
    for (int i = lane; i < n; i += 32)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst + i)), "l"(vedge + kb + i)
                   : "memory");
  }
}

// One 32-variable chunk of a homogeneous degree-D tile, with its base pointers.
struct VarChunk {
  int g, tile, half, kb, nval;
  uint32_t am;
  const float* llr0;  // llr_h row of the chunk's first variable
  const float* c2v0;  // c2v of the group
};

template <int D, int LW>
__device__ __forceinline__ VarChunk var_chunk(const Args& a, const VarTile& t, int half) {
  VarChunk c;
  c.g = t.g;
  c.tile = t.tile;
  c.half = half;
  c.kb = t.kb + half * 32 * D;
  c.nval = max(0, min(32, a.NV - (t.h0 + half * 32)));
  c.am = a.group_active[t.g];
  c.llr0 = a.llr_h + rix(t.g, a.NH, t.h0 + half * 32, LW);
  c.c2v0 = a.c2v + rix(t.g, a.EH, 0, LW);
  return c;
}

// Runs this warp's degree-D tiles (starting with grabbed tile w) as one
// pipeline over their chunks; returns the next grabbed tile it did not take.
template <int D, int QMODE, int LW>
__device__ long long var_stream(const Args& a, long long w, long long total, int32_t* sve0, int32_t* sve1,
                                float* ring, int lane) {
  constexpr int NS = VarShape<D, LW>::NS;
  constexpr int NB = VarShape<D, LW>::NB;          // batches per chunk
  constexpr int RS = VarShape<D, LW>::ROWS * LW;   // stage stride (floats)
  int32_t* ve_c = sve0;  // edge ids of cur
  int32_t* ve_n = sve1;  // edge ids of nxt
  static_assert(NB >= 2 * NS - 1, "the next chunk's edge ids must land before its first batch is issued");
  constexpr int QPR = LW / 4;  // 16-byte pieces per row
  const int lrow = lane / QPR;
  const int lcol = (lane % QPR) * 4;
  const int f = LW == 32 ? lane : lane % LW;  // this lane's frame (slot lane)
  const uint64_t pol = policy_evict_first();

  VarTile tile = var_tile(a, w);
  VarChunk cur = var_chunk<D, LW>(a, tile, 0), nxt = cur;
  bool has_nxt = false;
  long long w_after = total;  // the tile grabbed after the current one
  int2 desc_after = make_int2(-1, 0);
  int kpend = var_grab_issue(a, lane);  // grabbed one chunk ahead of its use
  var_stage_ve<D>(ve_c, a.vedge_t, cur.kb, lane);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  int slot_issue = 0, slot_comp = 0;  // ring slots of the next batch to issue / compute
  // issue contexts of cur and nxt as scalars (no struct selected at run time)
  const float* llr_c = cur.llr0;
  const float* c2v_c = cur.c2v0;
  int nval_c = cur.nval;
  bool qact_c = ((cur.am >> lcol) & 0xFu) != 0u;
  const float* llr_n = llr_c;
  const float* c2v_n = c2v_c;
  int nval_n = 0;
  bool qact_n = false;
  // one commit group per pipeline step (possibly empty); pos counts batches from cur's batch 0
  auto issue_at = [&](int pos) {
    const bool in_cur = pos < NB;
    if (in_cur || has_nxt) {
      var_batch_issue<D, LW>(ring + slot_issue * RS, in_cur ? llr_c : llr_n, in_cur ? c2v_c : c2v_n,
                         in_cur ? ve_c : ve_n, in_cur ? pos : pos - NB, in_cur ? nval_c : nval_n, lrow,
                         lcol, in_cur ? qact_c : qact_n, pol);
    }
    cp_async_commit();
    if (++slot_issue == NS) slot_issue = 0;
  };
#pragma unroll 1
  for (int p = 0; p < NS - 1; ++p) issue_at(p);
  double acc0 = 0.0;
  for (;;) {
    // the chunk after cur: the second half of the tile, or the grabbed tile
    // if it has the same degree.  The grab was issued a chunk earlier and its
    // descriptor loaded during the first half, so neither latency is exposed.
    if (cur.half == 0) {
      nxt = var_chunk<D, LW>(a, tile, 1);
      has_nxt = true;
      w_after = var_grab_resolve(a, kpend, lane);
      if (w_after < total) desc_after = __ldg(&a.vtile[static_cast<int>(w_after % a.n_tiles)]);
    } else {
      has_nxt = w_after < total && desc_after.x == D;
      if (has_nxt) {
        tile = var_tile(a, w_after, desc_after.y);
        nxt = var_chunk<D, LW>(a, tile, 0);
        kpend = var_grab_issue(a, lane);
      }
    }
    if (has_nxt) {
      var_stage_ve<D>(ve_n, a.vedge_t, nxt.kb, lane);  // travels with this step's group
      llr_n = nxt.llr0;
      c2v_n = nxt.c2v0;
      nval_n = nxt.nval;
      qact_n = ((nxt.am >> lcol) & 0xFu) != 0u;
    }
    const bool act = (cur.am >> f) & 1u;
    const size_t hv = static_cast<size_t>(cur.g) * a.NV + static_cast<size_t>(cur.tile) * kQTile + cur.half * 32;
    float* postg = a.post + rix(cur.g, a.NV, static_cast<int64_t>(cur.tile) * kQTile + cur.half * 32, LW) + f;
    uint32_t* ebg = a.ebits + static_cast<size_t>(cur.g) * a.EH;
    double acc = 0.0;
    uint32_t hw = 0u;
    float carry = 0.0f;  // posterior partial of a variable split over batches
#pragma unroll 1
    for (int b = 0; b < NB; ++b) {
      issue_at(b + NS - 1);
      cp_async_wait<NS - 1>();
      __syncwarp();  // rows (and the next chunk's edge ids) were copied by other lanes
      var_batch_compute<D, QMODE, LW>(ring + slot_comp * RS, postg, ebg, ve_c, b, cur.nval, lane, act, acc, hw,
                                      carry);
      if (++slot_comp == NS) slot_comp = 0;
      __syncwarp();  // stage is refilled in the next round
    }
    if (lane < cur.nval) a.hbits[hv + lane] = hw;
    if (cur.half == 0) {
      acc0 = acc;
    } else {
      a.q_part[(static_cast<size_t>(cur.g) * a.n_tiles + cur.tile) * kLanes + lane] = acc0 + acc;
    }
    if (!has_nxt) break;
    cur = nxt;
    llr_c = llr_n;
    c2v_c = c2v_n;
    nval_c = nval_n;
    qact_c = qact_n;
    int32_t* t = ve_c;
    ve_c = ve_n;
    ve_n = t;
  }
  cp_async_wait<0>();
  __syncwarp();
  return w_after;
}

// ve points at the edge ids of CSC slot `kb` (staged copy or global array).
__device__ __forceinline__ float var_sum(const Args& a, int g, int h, int k0, int k1, const int32_t* ve, int kb,
                                         int lane, int lw) {
  float p = ld_stream(&a.llr_h[rix(g, a.NH, h, lw) + lane]);
  for (int k = k0; k < k1; k += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = (k + u < k1) ? ld_stream(&a.c2v[rix(g, a.EH, ve[k + u - kb], lw) + lane]) : 0.0f;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k + u < k1) p += v[u];  // ascending check order (decoder.cpp:101)
  }
  return p;
}

// Generic tile (mixed degrees, partial, or degree > 12): per variable,
// register gathers.
template <int QMODE>
__device__ void var_tile_generic(const Args& a, long long w, int32_t* sptr, int lane, int lw) {
  const VarTile t = var_tile(a, w);
  const uint32_t amask = a.group_active[t.g];
  const bool act = lane < lw && ((amask >> lane) & 1u);
  const size_t gv = static_cast<size_t>(t.g) * a.NV;
  const size_t ge = static_cast<size_t>(t.g) * a.EH;
  double acc = 0.0, acc0 = 0.0;
  for (int cc = 0; cc < kQTile / 32; ++cc) {
    const int h0 = t.h0 + cc * 32;
    const int nv = max(0, min(kLanes, a.NV - h0));
    if (cc == 1) {
      acc0 = acc;
      acc = 0.0;
    }
    if (nv == 0) continue;
    __syncwarp();
    if (lane < nv) sptr[lane] = __ldg(&a.vptr[h0 + lane]);
    if (lane == 0) sptr[nv] = __ldg(&a.vptr[h0 + nv]);
    __syncwarp();
    uint32_t hw = 0u;
    for (int i = 0; i < nv; ++i) {
      const int h = h0 + i;
      const int k0 = sptr[i], k1 = sptr[i + 1];
      float p = 0.0f;
      if (act) {
        p = var_sum(a, t.g, h, k0, k1, a.vedge + k0, k0, lane, lw);
        a.post[rix(t.g, a.NV, h, lw) + lane] = p;
        acc += QMODE == 0 ? static_cast<double>(p) : static_cast<double>(fabsf(p));
      }
      const uint32_t word = __ballot_sync(0xffffffffu, act && p < 0.0f);
      if (lane == i) hw = word;
      for (int k = k0 + lane; k < k1; k += 32) a.ebits[ge + __ldg(&a.vedge[k])] = word;
    }
    if (lane < nv) a.hbits[gv + h0 + lane] = hw;
  }
  a.q_part[(static_cast<size_t>(t.g) * a.n_tiles + t.tile) * kLanes + lane] = acc0 + acc;
}

// Dynamic shared memory per warp: ring (kVarRingRows rows), two edge-id
// buffers of a.ve_stride ints (32 x the largest typed tile degree), vptr
// staging for generic tiles.
__host__ __device__ constexpr size_t var_smem_per_warp(int ve_stride) {
  return static_cast<size_t>(kVarRingRows) * kLanes * 4 + 2 * static_cast<size_t>(ve_stride) * 4 + 36 * 4;
}

// The tile loop of k_var for groups laid out with lane width LW (narrow
// groups: typed streams for tile degrees <= 16, the generic path otherwise).
template <int QMODE, int LW>
__device__ __forceinline__ void var_body(const Args& a, float* ring, int32_t* sve0, int32_t* sve1, int32_t* sptr,
                                         int lane) {
  const long long total = static_cast<long long>(a.G) * a.n_tiles;
  long long w = var_grab(a, lane);
  while (w < total) {
    const int d = __ldg(&a.vtile[static_cast<int>(w % a.n_tiles)]).x;
    switch (d) {
#define BPDEC_VSTREAM(D_)                                                     \
  case D_:                                                                    \
    w = var_stream<D_, QMODE, LW>(a, w, total, sve0, sve1, ring, lane);       \
    continue;
#define BPDEC_VSTREAM_WIDE(D_)                                                \
  case D_:                                                                    \
    if constexpr (LW == 32) {                                                 \
      w = var_stream<D_, QMODE, LW>(a, w, total, sve0, sve1, ring, lane);     \
      continue;                                                               \
    }                                                                         \
    break;
      BPDEC_VSTREAM(2)
      BPDEC_VSTREAM(3)
      BPDEC_VSTREAM(4)
      BPDEC_VSTREAM(6)
      BPDEC_VSTREAM(8)
      BPDEC_VSTREAM(12)
      BPDEC_VSTREAM(16)
      BPDEC_VSTREAM_WIDE(20)
      BPDEC_VSTREAM_WIDE(24)
      BPDEC_VSTREAM_WIDE(32)
#undef BPDEC_VSTREAM
#undef BPDEC_VSTREAM_WIDE
      default:
        break;
    }
    var_tile_generic<QMODE>(a, w, sptr, lane, LW);
    w = var_grab(a, lane);
  }
}

template <int QMODE>
__global__ void __launch_bounds__(kVarWarps * 32, 5) k_var(const Args a) {
  pdl_begin();  // 5 blocks/SM: measured best
  extern __shared__ __align__(16) unsigned char var_smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* base = var_smem + var_smem_per_warp(a.ve_stride) * warp;
  float* ring = reinterpret_cast<float*>(base);
  int32_t* sve0 = reinterpret_cast<int32_t*>(base + kVarRingRows * kLanes * 4);
  int32_t* sve1 = sve0 + a.ve_stride;
  int32_t* sptr = sve1 + a.ve_stride;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.counters[7] = 0;   // k_check chunk scheduler (next step)
    a.counters[10] = 0;  // k_decide syndrome passes (this step)
    a.counters[12] = 0;  // moved slots: k_check of this step has rewritten their degree-1-check words
  }
  const int lw = __ldcg(&a.counters[11]);  // lane width of the live groups (narrow tail)
  if (lw == 8)
    var_body<QMODE, 8>(a, ring, sve0, sve1, sptr, lane);
  else if (lw == 16)
    var_body<QMODE, 16>(a, ring, sve0, sve1, sptr, lane);
  else
    var_body<QMODE, 32>(a, ring, sve0, sve1, sptr, lane);
}

// ------------------------------------------------- k_decide: syndrome part --
// Warp = 32 consecutive (device-order) checks, lane = check, all groups.
// Parity of a check = target syndrome ^ degree-1 part (synp, from k_check)
// ^ the hard-decision words of its degree>=2 edges, which k_var stored per
// edge in check-major order (ebits): the check's words are contiguous, so
// the pass streams instead of gathering.  A group is skipped as soon as
// every active frame in it is known to fail (global fail masks, re-read per
// pass); new failing frames are published at once.
__device__ __forceinline__ uint32_t ldu32_pred(const uint32_t* p, bool pred) {
  uint32_t v = 0u;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.u32 %0, [%1];\n\t}"
               : "+r"(v)
               : "l"(p), "r"(static_cast<int>(pred)));
  return v;
}

constexpr int kSynChunks = 4;  // chunks per warp pass (their loads are in flight together)

// Syndrome part of k_decide.  Warps grab passes (kSynChunks chunks) from
// counters[10] (reset by k_var) and, before each, re-read the published
// failing frames: once every active frame is known to fail — in the high-FER
// regime after the first round of passes — the warps stop, so the pass costs
// about one round of loads instead of a sweep over all checks.
__device__ __forceinline__ void syndrome_block(const Args& a, int b, int nb, uint32_t* s_act) {
  for (int t = threadIdx.x; t < a.G; t += blockDim.x) s_act[t] = a.group_active[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int chunks = (a.M + 31) / 32;
  const int passes = (chunks + kSynChunks - 1) / kSynChunks;
  // first pass by warp index (no atomic round trip), then from counters[10]
  // (which k_var reset; handed-out passes start after the first round)
  const int nw = nb * static_cast<int>(blockDim.x >> 5);
  int q = b * static_cast<int>(blockDim.x >> 5) + static_cast<int>(threadIdx.x >> 5);
  for (bool first_pass = true;; first_pass = false) {
    if (!first_pass) {
      int k = 0;
      if (lane == 0) k = atomicAdd(&a.counters[10], 1);
      q = nw + __shfl_sync(0xffffffffu, k, 0);
    }
    if (q >= passes) break;
    bool live = first_pass;  // any group with an active frame not yet known to fail (k_check reset fail)
    for (int g0 = 0; g0 < a.G && !live; g0 += 32) {
      const int g = g0 + lane;
      const uint32_t am = g < a.G ? s_act[g] : 0u;
      const uint32_t fl = g < a.G ? __ldcg(&a.fail[g]) : 0u;
      live = __any_sync(0xffffffffu, am != 0u && (fl & am) != am);
    }
    if (!live) break;  // warp-uniform: nothing left to prove this step
    int e0[kSynChunks], nh[kSynChunks];
    bool valid[kSynChunks];
#pragma unroll
    for (int u = 0; u < kSynChunks; ++u) {
      const int ch = q * kSynChunks + u;
      const int c = ch * 32 + lane;
      valid[u] = ch < chunks && c < a.M;
      const int4 cdk = ch < chunks ? __ldg(&a.ctype[ch]) : make_int4(0, 0, 0, 0);
      if (cdk.x >= 0) {  // homogeneous chunk: NH hi edges per check, contiguous
        nh[u] = cdk.x >> 3;
        e0[u] = cdk.y + lane * nh[u];
      } else {
        const int4 d = valid[u] ? __ldg(&a.cdesc[c]) : make_int4(0, 0, 0, 0);
        e0[u] = d.x;
        nh[u] = d.y - d.x;
      }
      if (!valid[u]) nh[u] = 0;
    }
    for (int g0 = 0; g0 < a.G; g0 += 32) {
      const int gl = g0 + lane;
      const uint32_t aml = gl < a.G ? s_act[gl] : 0u;
      const uint32_t fll = gl < a.G ? __ldcg(&a.fail[gl]) : 0u;
      uint32_t need = __ballot_sync(0xffffffffu, aml != 0u && (fll & aml) != aml);
      while (need) {  // warp-uniform
        const int k = __ffs(need) - 1;
        need &= need - 1;
        const int g = g0 + k;
        const uint32_t amask = __shfl_sync(0xffffffffu, aml, k);
        const uint32_t fl = __shfl_sync(0xffffffffu, fll, k);
        const uint32_t* eb = a.ebits + static_cast<size_t>(g) * a.EH;
        const uint32_t* sp = a.synp + static_cast<size_t>(g) * a.M;
        uint32_t word[kSynChunks];
#pragma unroll
        for (int u = 0; u < kSynChunks; ++u) {
          const int c = (q * kSynChunks + u) * 32 + lane;
          word[u] = ldu32_pred(sp + (valid[u] ? c : 0), valid[u]);
#pragma unroll
          for (int j = 0; j < 4; ++j) word[u] ^= ldu32_pred(eb + e0[u] + (j < nh[u] ? j : 0), j < nh[u]);
        }
        uint32_t any = 0u;
#pragma unroll
        for (int u = 0; u < kSynChunks; ++u) {
          for (int j = 4; j < nh[u]; ++j) word[u] ^= eb[e0[u] + j];  // checks with more than 4 such edges
          any |= word[u];
        }
        any = __reduce_or_sync(0xffffffffu, any & amask);
        if (lane == 0 && (any & ~fl) != 0u) atomicOr(&a.fail[g], any);  // published at once
      }
    }
  }
}

// q part of k_decide: block p of group g sums its range of the k_var tile
// partials (warps interleaved, then the warp sums in order) into q_mid.
__device__ __forceinline__ void q_block(const Args& a, int g, int p, double (*red)[kLanes]) {
  constexpr int kW = kThreads / 32;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (a.group_active[g] == 0u) return;  // block-uniform
  const int t_lo = static_cast<int>(static_cast<long long>(a.n_tiles) * p / kTermBlocks);
  const int t_hi = static_cast<int>(static_cast<long long>(a.n_tiles) * (p + 1) / kTermBlocks);
  const double* qp = a.q_part + static_cast<size_t>(g) * a.n_tiles * kLanes + lane;
  double q = 0.0;
  for (int t0 = t_lo + warp; t0 < t_hi; t0 += kW * 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = t0 + kW * k;
      v[k] = t < t_hi ? qp[static_cast<size_t>(t) * kLanes] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (t0 + kW * k < t_hi) q += v[k];
    }
  }
  red[warp][lane] = q;
  __syncthreads();
  if (warp == 0) {
    q = red[0][lane];
#pragma unroll
    for (int k = 1; k < kW; ++k) q += red[k][lane];
    a.q_mid[(static_cast<size_t>(g) * kTermBlocks + p) * kLanes + lane] = q;
  }
}

// Decision for every slot of group g (one warp): q^(k) = the block sums in
// order; PCE, then VNR (k >= 2, strict), then d_max (decoder.cpp:114-123);
// stopping slots take the next queued frames.  Rewrites stopped[g] /
// load_mask[g] for k_turnover.
// Hands the free lanes of group g (lane order) the next available frames:
// at most counters[9] (frames uploaded) and batch; returns the load mask.
__device__ __forceinline__ uint32_t refill_lanes(const Args& a, int g, uint32_t free, int lane) {
  int take = 0, base = 0;
  if (lane == 0 && free != 0u) {
    const int want = __popc(free);
    const int limit = min(a.batch, *reinterpret_cast<volatile int32_t*>(&a.counters[9]));  // stream: batch = INT_MAX
    int old = *reinterpret_cast<volatile int32_t*>(&a.counters[0]);
    for (;;) {  // bounded grab: frames beyond the limit stay queued
      take = max(0, min(want, limit - old));
      if (take == 0) break;
      const int prev = atomicCAS(&a.counters[0], old, old + take);
      if (prev == old) break;
      old = prev;
    }
    base = old;
  }
  take = __shfl_sync(0xffffffffu, take, 0);
  base = __shfl_sync(0xffffffffu, base, 0);
  const int rank = __popc(free & ((1u << lane) - 1u));
  const bool refill = ((free >> lane) & 1u) && rank < take;
  if (refill) a.pending_frame[g * kLanes + lane] = base + rank;
  return __ballot_sync(0xffffffffu, refill);
}

__device__ __forceinline__ void decide_group(const Args& a, int g, int lane) {
  const uint32_t amask = a.group_active[g];
  if (amask == 0u) {  // idle group: frames may have become available since
    const uint32_t load = refill_lanes(a, g, 0xffffffffu, lane);
    if (lane == 0) {
      a.stopped[g] = 0u;
      a.load_mask[g] = load;
    }
    return;
  }
  double v[kTermBlocks];
#pragma unroll
  for (int k = 0; k < kTermBlocks; ++k) v[k] = __ldcg(&a.q_mid[(static_cast<size_t>(g) * kTermBlocks + k) * kLanes + lane]);
  double q = v[0];
#pragma unroll
  for (int k = 1; k < kTermBlocks; ++k) q += v[k];
  if (lane == 0) atomicAdd(a.frame_iters, static_cast<unsigned long long>(__popc(amask)));
  const uint32_t bit = 1u << lane;
  const bool act = (amask & bit) != 0u;
  const int s = g * kLanes + lane;
  int reason = -1, it = 0, f = 0;
  if (act) {
    it = a.slot_iter[s];
    f = a.slot_frame[s];
    const size_t fr = frow(a, f);
    if (a.out_qtrace) a.out_qtrace[fr * a.d_max + (it - 1)] = q;
    const bool syn_ok = !(__ldcg(&a.fail[g]) & bit);
    // the observer's syndrome_ok is computed every iteration, PCE or not
    // (decoder.cpp:110-112)
    if (a.out_syntrace) a.out_syntrace[fr * a.d_max + (it - 1)] = syn_ok ? 1 : 0;
    if (a.use_pce && syn_ok) {
      reason = 0;
    } else if (a.use_vnr && it >= 2 && q < a.qprev[s]) {
      reason = 1;
    } else if (it >= a.d_max) {
      reason = 2;
    }
    if (reason < 0) {
      a.slot_iter[s] = it + 1;
      a.qprev[s] = q;
    } else {
      a.out_iters[fr] = it;
      a.out_reasons[fr] = static_cast<uint8_t>(reason);
      a.stop_frame[s] = f;
      if (a.bdone) atomicAdd(&a.bdone[a.fbatch[fr]], 1);
    }
  }
  const uint32_t stop = __ballot_sync(0xffffffffu, reason >= 0);
  const int nstop = __popc(stop);
  if (lane == 0 && nstop > 0) {
    a.group_active[g] = amask & ~stop;
    atomicAdd(&a.counters[1], nstop);
    atomicSub(&a.counters[3], nstop);
  }
  // refill: every lane that is not active (this step's stops and lanes left
  // free earlier) takes the next available queued frame, in lane order --
  // or, with group_refill, only a group whose every lane is free (a refill
  // rewrites every row of the group: one dense load of up to 32 frames
  // instead of a partial-line pass per few frames; k_compact frees groups)
  const uint32_t left = amask & ~stop;
  const uint32_t load = refill_lanes(a, g, (a.group_refill && left != 0u) ? 0u : ~left, lane);
  if (lane == 0) {
    a.stopped[g] = stop;
    a.load_mask[g] = load;
  }
}

// ------------------------------------------------------------ k_decide --
// Syndrome, q^(k) and the stop decision of a step in one launch.  Blocks
// [0, syn_blocks): bit-sliced parity of every check vs its target
// (decoder.cpp:19-30), streaming synp and the check's contiguous ebits,
// OR-reduced fail masks, dynamically handed-out passes; the warps stop once
// every active frame is known to fail.  Blocks [syn_blocks, syn_blocks + G*kTermBlocks): the fixed
// -order q partial tree.  The last block to finish (counters[8]) takes the
// decisions for all groups, one warp per group.
__global__ void __launch_bounds__(kThreads) k_decide(const Args a, int syn_blocks) {
  pdl_begin();
  extern __shared__ uint32_t s_grp[];  // [G] active masks (syndrome blocks)
  __shared__ double red[kThreads / 32][kLanes];
  __shared__ int s_last;
  const int b = blockIdx.x;
  if (b < syn_blocks) {
    syndrome_block(a, b, syn_blocks, s_grp);
  } else {
    const int qb = b - syn_blocks;
    q_block(a, qb / kTermBlocks, qb - (qb / kTermBlocks) * kTermBlocks, red);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&a.counters[8], 1) == static_cast<int>(gridDim.x) - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int lane = threadIdx.x & 31;
  for (int g = static_cast<int>(threadIdx.x >> 5); g < a.G; g += kThreads / 32) decide_group(a, g, lane);
  __syncthreads();
  if (threadIdx.x == 0) {
    a.counters[8] = 0;
    if (a.h_poll) {  // frames done / error flags of this step for the host loop
      volatile int32_t* hp = a.h_poll + kPollWords * a.poll_slot;
#pragma unroll
      for (int k = 0; k < 4; ++k) hp[k] = __ldcg(&a.counters[k]);
      if (a.bdone)
        for (int k = 0; k < kMaxStreamBatches; ++k) hp[4 + k] = __ldcg(&a.bdone[k]);
      __threadfence_system();
    }
  }
}

// Posteriors of every active frame after this step's variable pass (the
// observer's per-iteration posteriors, decoder.cpp:111-112), in the original
// variable order: warp = (group, 32 variables), lane = variable.
__global__ void __launch_bounds__(kThreads) k_trace_post(const Args a) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int lw = __ldcg(&a.counters[11]);
  const long long items = static_cast<long long>(a.G) * a.NW;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < items; w += nwarps) {
    const int g = static_cast<int>(w / a.NW);
    const int ch = static_cast<int>(w - static_cast<long long>(g) * a.NW);
    uint32_t am = a.group_active[g];
    if (am == 0u) continue;
    const int i = ch * 32 + lane;
    const bool valid = i < a.N;
    const float* prow = nullptr;
    if (valid) {
      const int vm = __ldg(&a.vmap[i]);
      prow = vm >= 0 ? (vm < a.NV ? a.post + rix(g, a.NV, vm, lw) : a.llr_h + rix(g, a.NH, vm, lw))
                     : a.d1post + rix(g, a.N1, -1 - vm, lw);
    }
    while (am) {
      const int l = __ffs(am) - 1;
      am &= am - 1;
      const int s = g * kLanes + l;
      const int f = a.slot_frame[s];
      const int it = a.slot_iter[s];
      if (valid) a.out_ptrace[(frow(a, f) * a.d_max + (it - 1)) * a.N + i] = prow[l];
    }
  }
}

// Snapshot of out_iters (frames whose outputs are final) into mapped host
// memory, in stream order after a step's k_turnover: a frame with a non-zero
// entry has been extracted by then (eager output copies).
__global__ void k_snapshot(const int32_t* __restrict__ iters, int32_t n, int32_t* h_out) {
  pdl_begin();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) h_out[i] = iters[i];
  __threadfence_system();
}

// ---------------------------------------------------------- k_turnover --
// Frame turnover after the decision of a step, one launch:
//  * extract — outputs (hard bits, posteriors) of the frames that stopped
//    (decoder.cpp:126-128), in the original variable order;
//  * load — the next queued frames into the freed slots.
// Work items are (group with turnover, quad of 4 x 32 original variables),
// so groups are handled in parallel.  Per item: its warps extract the
// group's stopped lanes of the 4 chunks (warp = chunk, lane = variable; the
// bit-sliced hard-decision word serves every stopped lane; packed words come
// from one ballot); barrier; the same rows are overwritten with the new
// frames' LLRs — up to 32 frames x 128 variables read row-coalesced,
// transposed in shared memory, written as one [item][32 lanes] row per
// variable at its device position (vmap); a slot is recycled in the step it
// frees.  Check blocks: the target syndrome, one 32-check input word per warp
// bit-transposed with 32 ballots into the device-order words (cdev).  One
// block: slot state.
constexpr int kTurnChunks = 4;
constexpr int kMaxGroups = 1024;  // worklist capacity (slots <= 32768)
constexpr int kSparseLoad = 8;    // at most this many entering frames per group: direct scatter path

template <bool WANT_POST>
__device__ __forceinline__ void extract_chunk(const Args& a, int g, uint32_t sm, int ch, int lane, int lw) {
  const int i = ch * 32 + lane;
  const bool valid = i < a.N;
  const int vm = valid ? __ldg(&a.vmap[i]) : 0;
  uint32_t word = 0u;
  const float* prow = nullptr;  // row of 32 lanes holding this variable's posterior
  const bool deg0 = valid && vm >= a.NV;
  if (valid) {
    if (vm >= 0) {
      if (vm < a.NV) {
        word = a.hbits[static_cast<size_t>(g) * a.NV + vm];
        prow = a.post + rix(g, a.NV, vm, lw);
      } else {  // degree-0 variable: posterior = channel LLR
        prow = a.llr_h + rix(g, a.NH, vm, lw);
      }
    } else {
      const int dd = -1 - vm;
      word = a.d1bits[static_cast<size_t>(g) * a.N1 + dd];
      if (WANT_POST) prow = a.d1post + rix(g, a.N1, dd, lw);
    }
  }
  // frame of every stopped lane in a register (one load, not one per lane)
  const int fr = ((sm >> lane) & 1u) ? __ldcg(&a.stop_frame[g * kLanes + lane]) : 0;
  if (!WANT_POST && a.out_bits_u8 == nullptr && a.out_bits_pk != nullptr && !__any_sync(0xffffffffu, deg0)) {
    // packed bits only: a 32 x 32 bit transpose (lane i: bit f = frame f's
    // bit of variable i  ->  lane f: bit i) gives every stopped frame's
    // word of this chunk at once, the same word a ballot per frame gives
    uint32_t x = word;
#pragma unroll
    for (int k = 16; k >= 1; k >>= 1) {
      const uint32_t mk = k == 16 ? 0x0000ffffu : k == 8 ? 0x00ff00ffu : k == 4 ? 0x0f0f0f0fu : k == 2 ? 0x33333333u
                                                                                                    : 0x55555555u;
      const uint32_t y = __shfl_xor_sync(0xffffffffu, x, k);
      x = (lane & k) ? ((x & ~mk) | ((y & ~mk) >> k)) : ((x & mk) | ((y & mk) << k));
    }
    if ((sm >> lane) & 1u) a.out_bits_pk[frow(a, fr) * a.NW + ch] = x;
    return;
  }
  while (sm) {
    const int l = __ffs(sm) - 1;
    sm &= sm - 1;
    const size_t f = frow(a, __shfl_sync(0xffffffffu, fr, l));
    uint32_t bit = (word >> l) & 1u;
    float pv = 0.0f;
    if (deg0) {
      pv = prow[l];
      bit = pv < 0.0f ? 1u : 0u;
    } else if (WANT_POST && valid) {
      pv = prow[l];
    }
    if (valid) {
      if (a.out_bits_u8) a.out_bits_u8[f * a.N + i] = static_cast<uint8_t>(bit);
      if (WANT_POST) a.out_post[f * a.N + i] = pv;
    }
    if (a.out_bits_pk) {
      const uint32_t pw = __ballot_sync(0xffffffffu, bit);
      if (lane == 0) a.out_bits_pk[f * a.NW + ch] = pw;
    }
  }
}

// Dense refill of one quad (4 x 32 original variables) of group g: up to 32
// entering frames read row-coalesced, transposed in shared memory, written as
// one [item][32 lanes] row per variable at its device position (vmap).
// Block-level (two barriers).
__device__ __forceinline__ void load_quad_tile(const Args& a, int g, uint32_t lm, int ch0,
                                               float (*tile)[32][33], int lane, int warp) {
  constexpr int kW = kThreads / 32;
  // read: warp = slot lanes r = warp + 8m, lanes = consecutive original
  // variables; all 4 x 4 loads in flight before any use
  constexpr int kRpw = 32 / kW;
  float v[kTurnChunks][kRpw];
  size_t frs[kRpw];
#pragma unroll
  for (int m = 0; m < kRpw; ++m) {
    const int r = warp + kW * m;
    const bool on = (lm >> r) & 1u;
    frs[m] = frow(a, on ? a.pending_frame[g * kLanes + r] : 0);
    const float* src = a.in_llr + frs[m] * a.N;
#pragma unroll
    for (int c = 0; c < kTurnChunks; ++c) {
      const int i = (ch0 + c) * 32 + lane;
      v[c][m] = (on && i < a.N) ? src[i] : 0.0f;
    }
  }
  bool bad = false;
#pragma unroll
  for (int m = 0; m < kRpw; ++m) {
    bool bm = false;
#pragma unroll
    for (int c = 0; c < kTurnChunks; ++c) {
      bm |= !isfinite(v[c][m]);
      tile[c][warp + kW * m][lane] = v[c][m];
    }
    if (bm && a.ferr) a.ferr[frs[m]] = 1;  // stream mode: the batch of this frame fails
    bad |= bm;
  }
  if (bad) atomicOr(&a.counters[2], 1);
  __syncthreads();
  // write: warp = variable j, lanes = slots (one row); the device rows of
  // all this warp's variables are looked up first (loads in flight together)
  constexpr int kJ = 32 * kTurnChunks / kW;
  int vjs[kJ];
#pragma unroll
  for (int m = 0; m < kJ; ++m) {
    const int i = ch0 * 32 + warp + kW * m;
    vjs[m] = __ldg(&a.vmap[i < a.N ? i : 0]);
  }
#pragma unroll
  for (int m = 0; m < kJ; ++m) {
    const int jj = warp + kW * m;
    const int i = ch0 * 32 + jj;
    if (i < a.N && ((lm >> lane) & 1u)) {
      const float x = tile[jj >> 5][lane][jj & 31];
      const int vj = vjs[m];
      if (vj >= 0) {
        a.llr_h[(static_cast<size_t>(g) * a.NH + vj) * kLanes + lane] = x;
        // posterior state starts at the channel LLR (v2c of iteration 1)
        if (vj < a.NV) a.post[(static_cast<size_t>(g) * a.NV + vj) * kLanes + lane] = x;
      } else {
        a.llr_d[(static_cast<size_t>(g) * a.N1 + (-1 - vj)) * kLanes + lane] = x;
      }
    }
  }
  __syncthreads();  // the tile is reused
}

// Sparse refill of one chunk (32 original variables) of group g: few frames
// enter, so lane = variable, one coalesced LLR read per entering frame and a
// direct write into its slot lane (no transpose, no barrier).  Warp-level.
__device__ __forceinline__ void load_chunk_sparse(const Args& a, int g, uint32_t lm, int ch, int lane) {
  const int i = ch * 32 + lane;
  const bool in = i < a.N;
  const int vj = in ? __ldg(&a.vmap[i]) : 0;
  // all entering frames' values in flight at once (lm has <= kSparseLoad bits)
  int r[kSparseLoad];
  float v[kSparseLoad];
#pragma unroll
  for (int k = 0; k < kSparseLoad; ++k) {
    r[k] = lm ? __ffs(lm) - 1 : -1;
    lm &= lm - 1;
  }
  int f[kSparseLoad];
#pragma unroll
  for (int k = 0; k < kSparseLoad; ++k) f[k] = a.pending_frame[g * kLanes + max(r[k], 0)];  // safe index
#pragma unroll
  for (int k = 0; k < kSparseLoad; ++k)  // predicated loads: no branch per load
    v[k] = ld_pred(a.in_llr + frow(a, f[k]) * a.N + (in ? i : 0), r[k] >= 0 && in);
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kSparseLoad; ++k) {
    if (r[k] < 0 || !in) continue;
    if (!isfinite(v[k])) {
      bad = true;
      if (a.ferr) a.ferr[frow(a, f[k])] = 1;
    }
    if (vj >= 0) {
      a.llr_h[(static_cast<size_t>(g) * a.NH + vj) * kLanes + r[k]] = v[k];
      if (vj < a.NV) a.post[(static_cast<size_t>(g) * a.NV + vj) * kLanes + r[k]] = v[k];
    } else {
      a.llr_d[(static_cast<size_t>(g) * a.N1 + (-1 - vj)) * kLanes + r[k]] = v[k];
    }
  }
  if (bad) atomicOr(&a.counters[2], 1);
}

template <bool WANT_POST>
__global__ void __launch_bounds__(kThreads) k_turnover(const Args a, int item_blocks, int check_blocks) {
  pdl_begin();
  __shared__ float tile[kTurnChunks][32][33];
  __shared__ int16_t s_wg[kMaxGroups];  // groups with turnover (stops or loads), ascending
  __shared__ int16_t s_lg[kMaxGroups];  // groups with loads
  __shared__ int16_t s_sg[kMaxGroups];  // groups with stops
  __shared__ int16_t s_dg[kMaxGroups];  // groups with more than kSparseLoad entering frames
  __shared__ int16_t s_pg[kMaxGroups];  // groups with 1..kSparseLoad entering frames
  __shared__ int s_n[5];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int kW = kThreads / 32;
  // worklists (every block builds the same ones; warp 0, in group order)
  if (warp == 0) {
    int n[5] = {0, 0, 0, 0, 0};
    for (int g0 = 0; g0 < a.G; g0 += 32) {
      const int g = g0 + lane;
      const uint32_t st = g < a.G ? a.stopped[g] : 0u;
      const uint32_t lm = g < a.G ? a.load_mask[g] : 0u;
      const bool c[5] = {(st | lm) != 0u, lm != 0u, st != 0u, __popc(lm) > kSparseLoad,
                         lm != 0u && __popc(lm) <= kSparseLoad};
      int16_t* lists[5] = {s_wg, s_lg, s_sg, s_dg, s_pg};
      const uint32_t below = (1u << lane) - 1u;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const uint32_t bw = __ballot_sync(0xffffffffu, c[k]);
        if (c[k]) lists[k][n[k] + __popc(bw & below)] = static_cast<int16_t>(g);
        n[k] += __popc(bw);
      }
    }
    if (lane == 0)
      for (int k = 0; k < 5; ++k) s_n[k] = n[k];
  }
  __syncthreads();
  const int nw = s_n[0], nl = s_n[1];
  if (nw == 0) return;  // nothing to hand over this step
  // lane width of the live groups (a narrow tail group never refills: the
  // queue is drained before a group is narrowed)
  const int lw = __ldcg(&a.counters[11]);
  const int b = blockIdx.x;
  const int quads = (a.NW + kTurnChunks - 1) / kTurnChunks;
  if (b < item_blocks && (WANT_POST || a.NH != a.NV)) {
    // outputs read rows a refill overwrites (posteriors, degree-0 LLRs):
    // items (group, quad), extraction before the refill of the same rows
    const long long items = static_cast<long long>(nw) * quads;
    for (long long it = b; it < items; it += item_blocks) {
      const int wi = static_cast<int>(it / quads);
      const int qd = static_cast<int>(it - static_cast<long long>(wi) * quads);
      const int g = s_wg[wi];
      const uint32_t sm = a.stopped[g];
      const uint32_t lm = a.load_mask[g];
      const int ch0 = qd * kTurnChunks;
      if (sm) {
        if (warp < kTurnChunks && ch0 + warp < a.NW) extract_chunk<WANT_POST>(a, g, sm, ch0 + warp, lane, lw);
        __syncthreads();  // outputs read before the rows are refilled
      }
      if (lm) load_quad_tile(a, g, lm, ch0, tile, lane, warp);
    }
  } else if (b < item_blocks) {
    // packed/u8 bits only and no degree-0 variables: extraction reads only the
    // hard-decision words, which a refill does not touch, so the phases are
    // independent.  Dense refills: block-level (group, quad) items.
    const int nd = s_n[3], ns = s_n[2], np = s_n[4];
    const long long dense = static_cast<long long>(nd) * quads;
    for (long long it = b; it < dense; it += item_blocks) {
      const int di = static_cast<int>(it / quads);
      const int qd = static_cast<int>(it - static_cast<long long>(di) * quads);
      const int g = s_dg[di];
      load_quad_tile(a, g, a.load_mask[g], qd * kTurnChunks, tile, lane, warp);
    }
    // extraction and sparse refills: warp-level (group, chunk) items
    const long long ext = static_cast<long long>(ns) * a.NW;
    const long long total = ext + static_cast<long long>(np) * a.NW;
    const long long nwarps = static_cast<long long>(item_blocks) * kW;
    for (long long e = static_cast<long long>(b) * kW + warp; e < total; e += nwarps) {
      if (e < ext) {
        const int si = static_cast<int>(e / a.NW);
        const int g = s_sg[si];
        extract_chunk<WANT_POST>(a, g, a.stopped[g], static_cast<int>(e - static_cast<long long>(si) * a.NW), lane,
                                 lw);
      } else {
        const long long e2 = e - ext;
        const int pi = static_cast<int>(e2 / a.NW);
        const int g = s_pg[pi];
        load_chunk_sparse(a, g, a.load_mask[g], static_cast<int>(e2 - static_cast<long long>(pi) * a.NW), lane);
      }
    }
  } else if (b < item_blocks + check_blocks) {
    if (nl == 0) return;
    if (a.in_syn) {
      const int nwarp = check_blocks * kW;
      const long long items = static_cast<long long>(nl) * a.MW;
      for (long long w = static_cast<long long>(b - item_blocks) * kW + warp; w < items; w += nwarp) {
        const int li = static_cast<int>(w / a.MW);
        const int wi = static_cast<int>(w - static_cast<long long>(li) * a.MW);
        const int g = s_lg[li];
        const uint32_t lm = a.load_mask[g];
        uint32_t mine = 0u;  // lane r: input word wi of the frame entering slot r
        if ((lm >> lane) & 1u) {
          const int f = a.pending_frame[g * kLanes + lane];
          mine = __ldg(&a.in_syn[frow(a, f) * a.MW + wi]);
        }
        uint32_t col = 0u;  // lane k: check wi*32+k over the 32 slots
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const uint32_t t = __ballot_sync(0xffffffffu, (mine >> k) & 1u);
          if (lane == k) col = t;
        }
        const int c = wi * 32 + lane;
        if (c < a.M) {
          const size_t idx = static_cast<size_t>(g) * a.M + __ldg(&a.cdev[c]);
          a.syn_target[idx] = (a.syn_target[idx] & ~lm) | (col & lm);
        }
      }
    } else {
      const long long items = static_cast<long long>(nl) * a.M;
      const long long stride = static_cast<long long>(check_blocks) * blockDim.x;
      for (long long w = static_cast<long long>(b - item_blocks) * blockDim.x + threadIdx.x; w < items; w += stride) {
        const int li = static_cast<int>(w / a.M);
        const int g = s_lg[li];
        a.syn_target[static_cast<size_t>(g) * a.M + (w - static_cast<long long>(li) * a.M)] &= ~a.load_mask[g];
      }
    }
  } else {
    if (nl == 0) return;
    for (int s = threadIdx.x; s < a.G * kLanes; s += blockDim.x) {
      const int g = s >> 5;
      const uint32_t bit = 1u << (s & 31);
      if (a.load_mask[g] & bit) {
        a.slot_frame[s] = a.pending_frame[s];
        a.slot_iter[s] = 1;
        a.qprev[s] = 0.0;
        atomicOr(&a.group_active[g], bit);
        atomicAdd(&a.counters[3], 1);
      }
    }
    // frames entered: the compaction hysteresis starts over (stream mode
    // can refill after a compaction)
    if (threadIdx.x == 0) a.counters[4] = a.G * kLanes + 32;
  }
}

// ---------------------------------------------------------- compaction --
// When no frames are left to stream in, frames that are still iterating are
// packed into as few 32-slot groups as possible, so the tail of a batch (a
// few slow frames spread over many groups) stops paying full-warp compute in
// every group.  The plan is a pure function of group_active, computed
// redundantly by every block; k_compact copies the per-slot rows and its
// last block moves the slot state and rewrites group_active.
constexpr int kMaxCompactGroups = 256;
constexpr int kMaxMoves = 1024;

struct CompactPlan {
  int n;
  int narrow;          // 1: re-lay out the only live group narrow (moves = its live lanes, in order)
  int lw_old, lw_new;  // lane widths before / after (narrow plans)
  int16_t src[kMaxMoves];  // slot indices
  int16_t dst[kMaxMoves];
};

__device__ void compact_plan(const Args& a, CompactPlan& pl, int* cnt) {
  // single thread
  pl.n = 0;
  pl.narrow = 0;
  const int G = a.G;
  if (G > kMaxCompactGroups || G < 2) return;
  // frames still queued: freed slots get refilled instead (stream mode: the
  // frames submitted so far) -- except with group_refill, where compaction
  // is what frees whole groups for the queued frames
  if (!a.group_refill &&
      a.counters[0] < (a.ring_cap ? *reinterpret_cast<volatile int32_t*>(&a.counters[9]) : a.batch))
    return;
  int total = 0, alive = 0;
  for (int g = 0; g < G; ++g) {
    cnt[g] = __popc(a.group_active[g]);
    total += cnt[g];
    alive += cnt[g] > 0;
  }
  const int need = (total + 31) / 32;
  if (alive == 1 && a.narrow_ok) {
    // tail: the only live group holds <= 16 (<= 8) frames -> move them into
    // another (free) group laid out with 16 (8) lanes per row, so every
    // later pass moves 64 (32) bytes per row instead of a 128-byte line and
    // runs lane-folded (k_check / k_var)
    int gs = 0;
    while (cnt[gs] == 0) ++gs;
    const int n = cnt[gs];
    const int lw_old = a.counters[11];
    const int lw_new = n <= 8 ? 8 : (n <= 16 ? 16 : 32);
    if (lw_new >= lw_old) return;
    const int gd = gs == 0 ? 1 : 0;
    uint32_t m = a.group_active[gs];
    for (int f = 0; f < n; ++f) {
      const int ls = __ffs(m) - 1;
      m &= m - 1;
      pl.src[f] = static_cast<int16_t>(gs * kLanes + ls);
      pl.dst[f] = static_cast<int16_t>(gd * kLanes + f);
    }
    pl.n = n;
    pl.narrow = 1;
    pl.lw_old = lw_old;
    pl.lw_new = lw_new;
    return;
  }
  if (alive <= need) return;
  if (total > a.counters[4] - a.compact_hyst) return;  // hysteresis: re-pack only after more frames finished
  // targets: the `need` fullest groups (ties -> lower index); the rest are sources
  bool is_target[kMaxCompactGroups];
  for (int g = 0; g < G; ++g) is_target[g] = false;
  for (int t = 0; t < need; ++t) {
    int best = -1;
    for (int g = 0; g < G; ++g)
      if (!is_target[g] && (best < 0 || cnt[g] > cnt[best])) best = g;
    is_target[best] = true;
  }
  int tg = 0;
  uint32_t tfree = 0u;
  auto next_target = [&]() {
    while (tg < G && (!is_target[tg] || (tfree = ~a.group_active[tg]) == 0u)) ++tg;
  };
  next_target();
  for (int g = 0; g < G && pl.n < kMaxMoves; ++g) {
    if (is_target[g] || cnt[g] == 0) continue;
    uint32_t m = a.group_active[g];
    while (m && pl.n < kMaxMoves) {
      if (tg >= G) return;
      const int ls = __ffs(m) - 1;
      m &= m - 1;
      const int ld = __ffs(tfree) - 1;
      tfree &= tfree - 1;
      pl.src[pl.n] = static_cast<int16_t>(g * kLanes + ls);
      pl.dst[pl.n] = static_cast<int16_t>(tg * kLanes + ld);
      ++pl.n;
      if (tfree == 0u) {
        ++tg;
        next_target();
      }
    }
  }
}

// Narrowing move (plan.narrow): element (row r, lane f) of the target group
// = (row r, lane src_f) of the source group, every per-slot array, rows of
// lw_new floats in the target; then the target syndrome words (bit f = bit
// src_f), and the last block moves the slot state and sets counters[11].
__device__ void compact_narrow(const Args& a, const CompactPlan& pl, int& s_last) {
  const int n = pl.n, lwo = pl.lw_old, lwn = pl.lw_new;
  const int gs = pl.src[0] >> 5, gd = pl.dst[0] >> 5;
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long nth = static_cast<long long>(gridDim.x) * blockDim.x;
  const int f = static_cast<int>(tid % lwn);  // constant per thread (nth is a multiple of lwn)
  const int ls = f < n ? (pl.src[f] & 31) : 0;
  float* arrs[5] = {a.c2v, a.post, a.llr_h, a.llr_d, a.d1post};
  const long long rows[5] = {a.EH, a.NV, a.NH, a.N1, a.d1post != nullptr ? a.N1 : 0};
  for (int k = 0; k < 5; ++k) {
    const long long R = rows[k];
    if (R == 0) continue;
    const float* src = arrs[k] + rix(gs, R, 0, lwo) + ls;
    float* dst = arrs[k] + rix(gd, R, 0, lwn) + f;
    // thread = (row, lane f): 8 rows in flight per thread
    constexpr int kU = 8;
    const long long step = nth / lwn;
    for (long long r0 = tid / lwn; r0 < R; r0 += step * kU) {
      float v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const long long r = r0 + u * step;
        v[u] = (f < n && r < R) ? src[r * lwo] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const long long r = r0 + u * step;
        if (r < R) dst[r * lwn] = v[u];  // lanes f >= n: zero (idle)
      }
    }
  }
  for (long long c = tid; c < a.M; c += nth) {
    const uint32_t w = a.syn_target[static_cast<size_t>(gs) * a.M + c];
    uint32_t nw = 0u;
    for (int k = 0; k < n; ++k) nw |= ((w >> (pl.src[k] & 31)) & 1u) << k;
    a.syn_target[static_cast<size_t>(gd) * a.M + c] = nw;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&a.counters[5], 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  a.counters[5] = 0;
  for (int k = 0; k < n; ++k) {
    const int s = pl.src[k], d = pl.dst[k];
    a.slot_iter[d] = a.slot_iter[s];
    a.slot_frame[d] = a.slot_frame[s];
    a.qprev[d] = a.qprev[s];
  }
  a.group_active[gs] = 0u;
  a.group_active[gd] = (1u << n) - 1u;
  a.counters[11] = lwn;
  a.counters[12] = 1;
}

// One launch: every block computes the (identical) plan, moves its share of
// rows — warp = one row, lane = one move, so a row moves as one 128-byte
// read and write — and the last block to finish commits the slot state
// (counters[5] counts finished blocks).
__global__ void __launch_bounds__(kThreads) k_compact(const Args a) {
  pdl_begin();
  __shared__ CompactPlan pl;
  __shared__ int cnt[kMaxCompactGroups];
  __shared__ int s_last;
  if (threadIdx.x == 0) compact_plan(a, pl, cnt);
  __syncthreads();
  const int n = pl.n;
  if (n == 0) return;  // same decision in every block
  if (pl.narrow) {
    compact_narrow(a, pl, s_last);
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long rows_e = a.EH, rows_v = a.NV, rows_h = a.NH, rows_d = a.N1;
  const bool post_d = a.d1post != nullptr;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  // per array: warp = 8 rows per pass, lane = one move; sources and
  // targets are disjoint groups, so all 8 reads are issued before the writes
  constexpr int kRowsPer = 8;
  const long long warp0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  float* arrs[5] = {a.c2v, a.post, a.llr_h, a.llr_d, a.d1post};
  const long long rows[5] = {rows_e, rows_v, rows_h, rows_d, post_d ? rows_d : 0};
  for (int k0 = 0; k0 < n; k0 += 32) {
    const int k = k0 + lane;
    const bool mv = k < n;
    const int gs = mv ? pl.src[k] >> 5 : 0, ls = mv ? pl.src[k] & 31 : 0;
    const int gd = mv ? pl.dst[k] >> 5 : 0, ld = mv ? pl.dst[k] & 31 : 0;
    for (int q = 0; q < 5; ++q) {
      const long long R = rows[q];
      if (R == 0) continue;
      const float* src = arrs[q] + static_cast<size_t>(gs) * R * kLanes + ls;
      float* dst = arrs[q] + static_cast<size_t>(gd) * R * kLanes + ld;
      for (long long base = warp0 * kRowsPer; base < R; base += nwarps * kRowsPer) {
        float v[kRowsPer];
#pragma unroll
        for (int j = 0; j < kRowsPer; ++j) v[j] = (mv && base + j < R) ? src[(base + j) * kLanes] : 0.0f;
#pragma unroll
        for (int j = 0; j < kRowsPer; ++j)
          if (mv && base + j < R) dst[(base + j) * kLanes] = v[j];
      }
    }
  }
  // syndrome target bits: thread = one check; moves are ordered by source
  // and by target group, so each source word is read once and each target
  // word is read and written once
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long cc = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; cc < a.M; cc += stride) {
    int cur_s = -1, cur_d = -1;
    uint32_t ws = 0u, wd = 0u;
    for (int k = 0; k < n; ++k) {
      const int gs = pl.src[k] >> 5, ls = pl.src[k] & 31, gd = pl.dst[k] >> 5, ld = pl.dst[k] & 31;
      if (gs != cur_s) {
        cur_s = gs;
        ws = a.syn_target[static_cast<size_t>(gs) * a.M + cc];
      }
      if (gd != cur_d) {
        if (cur_d >= 0) a.syn_target[static_cast<size_t>(cur_d) * a.M + cc] = wd;
        cur_d = gd;
        wd = a.syn_target[static_cast<size_t>(gd) * a.M + cc];
      }
      wd = (wd & ~(1u << ld)) | (((ws >> ls) & 1u) << ld);
    }
    if (cur_d >= 0) a.syn_target[static_cast<size_t>(cur_d) * a.M + cc] = wd;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&a.counters[5], 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  a.counters[5] = 0;
  int total = 0;
  for (int g = 0; g < a.G; ++g) total += cnt[g];
  a.counters[4] = total;
  for (int k = 0; k < n; ++k) {
    const int s = pl.src[k], d = pl.dst[k];
    a.slot_iter[d] = a.slot_iter[s];
    a.slot_frame[d] = a.slot_frame[s];
    a.qprev[d] = a.qprev[s];
    a.group_active[s >> 5] &= ~(1u << (s & 31));
    a.group_active[d >> 5] |= 1u << (d & 31);
  }
  a.counters[12] = 1;  // degree-1-only checks are recomputed for the moved frames
}

// Start of a decode: frames 0..first-1 go to slots 0..first-1, per-decode
// counters and masks are reset (counters[4] = compaction hysteresis start).
__global__ void k_decode_init(const Args a, int first, int avail) {
  for (int s = threadIdx.x; s < a.G * kLanes; s += blockDim.x) a.pending_frame[s] = s < first ? s : 0;
  for (int g = threadIdx.x; g < a.G; g += blockDim.x) {
    const int lo = g * kLanes;
    const int n = min(max(first - lo, 0), kLanes);
    a.load_mask[g] = n == kLanes ? 0xffffffffu : ((1u << n) - 1u);
    a.group_active[g] = 0u;
    a.stopped[g] = 0u;
  }
  if (threadIdx.x < 16)
    a.counters[threadIdx.x] = threadIdx.x == 0 ? first
                              : threadIdx.x == 4 ? a.G * kLanes + 32
                              : threadIdx.x == 9 ? avail
                              : threadIdx.x == 11 ? kLanes
                                                 : 0;
  if (threadIdx.x == 0) *a.frame_iters = 0ull;
}

// ---------------------------------------------------------- generators --
// Syndrome-mode frames on device; same draws as bpdec_sample_frames
// (channel.cpp:44-61 with the message bit x and s = Hx on top).
// snr <= 0 selects per-frame efficiencies beta_f ~ U[beta_lo, beta_hi]
// (config 5), snr = 2^(2R/beta_f) - 1.
__global__ void k_gen_llr(int32_t N, int32_t NW, double snr_fixed, double beta_lo, double beta_hi, double rate,
                          uint64_t seed, int64_t first_frame, int32_t n_frames, int32_t all_zero, float* llr,
                          uint32_t* xpk) {
  const long long npad = (static_cast<long long>(N) + 31) / 32 * 32;
  const long long total = npad * n_frames;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int b = static_cast<int>(t / npad);
    const long long i = t - static_cast<long long>(b) * npad;
    const uint64_t f = static_cast<uint64_t>(first_frame + b);
    const double snr =
        snr_fixed > 0.0 ? snr_fixed : exp2(2.0 * rate / frame_beta(seed, f, beta_lo, beta_hi)) - 1.0;
    const double sigma2 = 1.0 / snr;
    const double sigma = sqrt(sigma2);
    const double scale = 2.0 / sigma2;
    unsigned x = 0;
    if (i < N) {
      const uint64_t nkey = stream_key(kNoiseDomain, seed, f);
      double u1, u2;
      noise_uniforms(nkey, static_cast<uint64_t>(i), &u1, &u2);
      const double gval = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
      x = all_zero ? 0u : message_bit(stream_key(kBitDomain, seed, f), static_cast<uint64_t>(i));
      const double y = (x ? -1.0 : 1.0) + sigma * gval;
      llr[static_cast<size_t>(b) * N + i] = static_cast<float>(scale * y);
    }
    const uint32_t word = __ballot_sync(0xffffffffu, x);
    if (xpk && (threadIdx.x & 31) == 0) xpk[static_cast<size_t>(b) * NW + (i >> 5)] = word;
  }
}

// s = H x from packed x (thread = 32 checks of one frame -> one word).
__global__ void k_gen_syndrome(const Args a, int32_t n_frames, const uint32_t* xpk, uint32_t* syn,
                               const int32_t* check_ptr, const int32_t* check_vars) {
  const long long total = static_cast<long long>(n_frames) * a.MW;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int b = static_cast<int>(t / a.MW);
    const int wd = static_cast<int>(t - static_cast<long long>(b) * a.MW);
    uint32_t word = 0u;
    for (int c = wd * 32; c < min(a.M, wd * 32 + 32); ++c) {
      uint32_t p = 0u;
      for (int e = check_ptr[c]; e < check_ptr[c + 1]; ++e) {
        const int v = check_vars[e];
        p ^= (xpk[static_cast<size_t>(b) * a.NW + (v >> 5)] >> (v & 31)) & 1u;
      }
      word |= p << (c & 31);
    }
    syn[static_cast<size_t>(b) * a.MW + wd] = word;
  }
}

template <typename T>
T* dalloc(size_t count, int64_t* bytes) {
  T* p = nullptr;
  if (count == 0) count = 1;
  CUDA_OK(dev_malloc(reinterpret_cast<void**>(&p), count * sizeof(T)));
  *bytes += static_cast<int64_t>(count * sizeof(T));
  return p;
}

bool is_device_ptr(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// Kernel launch with programmatic stream serialisation (see pdl_begin).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
#ifdef BPDEC_NO_PDL
  cfg.numAttrs = 0;
#else
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#endif
  CUDA_OK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// Device scratch that grows on demand.
struct Scratch {
  void* ptr = nullptr;
  size_t size = 0;
  void* get(size_t n) {
    if (n <= size) return ptr;
    if (ptr) CUDA_OK(dev_free(ptr));
    ptr = nullptr;
    size = 0;
    CUDA_OK(dev_malloc(&ptr, n));
    size = n;
    return ptr;
  }
  ~Scratch() {
    if (ptr) dev_free(ptr);
  }
};

}  // namespace

// -------------------------------------------------------- GpuDecoder --
class GpuDecoder {
 public:
  GpuDecoder(const Code& code, int device, int max_slots);
  ~GpuDecoder();
  void decode(const DecodeParams& p, const DecodeBuffers& b, cudaStream_t stream);
  void stage_inputs(int32_t batch, const float* llr_host, const uint32_t* syn_host);
  void sample_device(double snr, double beta_lo, double beta_hi, double rate, uint64_t seed, int64_t first_frame,
                     int32_t n_frames, bool all_zero,
                     float* d_llr, uint32_t* d_syn, uint32_t* d_x, cudaStream_t stream);
  // stream mode (bpdec_stream_*)
  void stream_open(const DecodeParams& p, bool packed, bool want_bits, bool want_post, bool want_q, int32_t ring_frames);
  int64_t stream_submit(int32_t n, const float* llr, const uint32_t* syn, const StreamOutputs& o);
  bool stream_query(int64_t ticket);
  void stream_wait(int64_t ticket);
  void stream_close();
  void stream_timer_reset();
  double stream_device_ms();

  int S = 0;
  int G = 0;
  int device = 0;
  int64_t dev_bytes = 0;
  bool profiling = false;
  bool no_narrow = false;  // BPDEC_NO_NARROW set at construction
  bool no_eager = false;   // BPDEC_NO_EAGER: host outputs copied after the decode only (A/B knob)

  double prof_ms[kNumKernels] = {};
  int64_t prof_launches[kNumKernels] = {};
  double prof_frame_iters = 0.0;
  std::atomic<int64_t> launches{0};
  int64_t compactions = 0;

 private:
  struct Stream;
  void stream_worker();
  void stream_release() noexcept;
  std::unique_ptr<Stream> stream_;
  template <typename F>
  void launch(int kid, cudaStream_t st, F&& f);
  void run_step(const Args& a, cudaStream_t st, bool want_post);
  void launch_turnover(const Args& a, cudaStream_t st, bool want_post);
  cudaError_t harvest_profile(const unsigned long long* d_frame_iters) noexcept;
  void init(const Code& code, int max_slots);
  void release() noexcept;

  Args base{};
  int32_t max_check_deg = 0;
  int32_t* d_check_ptr = nullptr;
  int32_t* d_check_vars = nullptr;
  std::vector<void*> owned;
  cudaStream_t own_stream = nullptr;
  int32_t* h_counters = nullptr;  // pinned, mapped poll ring [kRing][kPollWords] (k_decide)
  static constexpr int kRing = 8;
  cudaEvent_t ring_ev[kRing] = {};
  std::vector<cudaEvent_t> prof_ev;
  std::vector<int> prof_kid;
  Scratch s_llr, s_syn, s_bits, s_iters, s_reasons, s_post, s_qtrace, s_syntrace, s_ptrace;
  // host-input staging (bpdec_decoder_stage_inputs): the H2D copy of a later
  // batch runs on copy_stream while the current batch decodes
  struct Staged {
    const float* llr_host = nullptr;
    const uint32_t* syn_host = nullptr;
    int32_t batch = 0;
    Scratch llr, syn;
    cudaEvent_t done = nullptr;
    bool valid = false;
    int64_t seq = 0;
  };
  Staged staged[2];
  int64_t stage_seq = 0;
  cudaStream_t copy_stream = nullptr;
  // chunked upload of unstaged host inputs (frames available -> counters[9])
  int32_t* h_avail = nullptr;
  size_t h_avail_n = 0;
  cudaEvent_t up_start = nullptr, up_first = nullptr, up_done = nullptr;
  // eager D2H of finished frames' outputs (host output buffers): while the
  // tail decodes, rows of frames that already stopped are copied on
  // out_stream (k_decide writes out_iters at the stop; a snapshot of it,
  // taken after a polled step, says which rows are final)
  cudaStream_t out_stream = nullptr;
  int32_t* h_done = nullptr;  // pinned, mapped snapshot of out_iters (k_snapshot)
  int32_t* h_done_dev = nullptr;
  size_t h_done_cap = 0;
  cudaEvent_t done_ev = nullptr;
  int grid_check = 0, grid_var = 0, grid_syn = 0, sms_ = 148;
  int turn_item_blocks = 0, turn_check_blocks = 0;
  size_t var_smem = 0;
};

GpuDecoder::GpuDecoder(const Code& code, int dev, int max_slots) : device(dev) {
  // a failed construction (bad device, out of memory) releases what it got
  try {
    init(code, max_slots);
  } catch (...) {
    release();
    throw;
  }
}

void GpuDecoder::init(const Code& code, int max_slots) {
  const int dev = device;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    (void)cudaGetLastError();
    throw CudaError("no CUDA device available (the decoder has no CPU fallback)");
  }
  if (dev < 0 || dev >= count) throw ConfigError("device index out of range");
  CUDA_OK(cudaSetDevice(dev));
  cudaDeviceProp prop{};
  CUDA_OK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major < 10) {
    throw CudaError(std::string("device ") + prop.name + " is not sm_100-class; this build targets sm_100a only");
  }
  if (const char* e = std::getenv("BPDEC_NO_NARROW")) no_narrow = e[0] != '\0' && e[0] != '0';
  if (const char* e = std::getenv("BPDEC_NO_EAGER")) no_eager = e[0] != '\0' && e[0] != '0';
  if (max_slots < 1) throw ValidationError("decoder: max_slots must be positive");
  if (max_slots > 32 * kMaxGroups) throw ValidationError("decoder: max_slots above 32768 is not supported");
  S = (max_slots + 31) / 32 * 32;
  G = S / 32;

  // ---- device code layout
  // variables: degree>=2 sorted by (degree, index) -> h in [0, NV); then
  // degree 0 -> [NV, NH); degree-1 variables -> D1 rows in device check order.
  // checks: sorted by type (NH edges to degree>=2 vars, ND degree-1 edges).
  const int32_t N = code.n_vars, M = code.n_checks;
  std::vector<int32_t> deg(N);
  for (int32_t v = 0; v < N; ++v) deg[v] = code.var_degree(v);
  std::vector<int32_t> horig;
  for (int32_t v = 0; v < N; ++v)
    if (deg[v] >= 2) horig.push_back(v);
  std::stable_sort(horig.begin(), horig.end(), [&](int32_t x, int32_t y) { return deg[x] < deg[y]; });
  const int32_t NV = static_cast<int32_t>(horig.size());
  for (int32_t v = 0; v < N; ++v)
    if (deg[v] == 0) horig.push_back(v);
  const int32_t NH = static_cast<int32_t>(horig.size());
  std::vector<int32_t> vmap(N, 0);
  for (int32_t h = 0; h < NH; ++h) vmap[horig[h]] = h;
  std::vector<int32_t> cnh(M, 0), cnd(M, 0);
  for (int32_t c = 0; c < M; ++c) {
    for (int32_t e = code.check_ptr[c]; e < code.check_ptr[c + 1]; ++e) {
      const int32_t d = deg[code.check_vars[e]];
      if (d >= 2) ++cnh[c];
      else ++cnd[c];
    }
  }
  // within a type, checks follow their first (lowest device index)
  // degree>=2 variable: the c2v rows a tile of consecutive variables gathers
  // in the variable pass — every row of a (1,1) check, about half of the
  // others — and the posterior rows the check pass gathers then lie close
  // together instead of anywhere in the array (sums still follow the
  // original check order, so results do not change)
  std::vector<int32_t> minh(M, INT32_MAX);
  for (int32_t c = 0; c < M; ++c)
    for (int32_t e = code.check_ptr[c]; e < code.check_ptr[c + 1]; ++e) {
      const int32_t v = code.check_vars[e];
      if (deg[v] >= 2) minh[c] = std::min(minh[c], vmap[v]);
    }
  std::vector<int32_t> corig(M);
  for (int32_t c = 0; c < M; ++c) corig[c] = c;
  std::stable_sort(corig.begin(), corig.end(), [&](int32_t x, int32_t y) {
    if (cnh[x] != cnh[y]) return cnh[x] < cnh[y];
    if (cnd[x] != cnd[y]) return cnd[x] < cnd[y];
    return minh[x] < minh[y];
  });
  std::vector<int4> cdesc(M);
  std::vector<int32_t> chk_hi_h, dorig(horig), hi_of_edge(code.n_edges(), -1);
  int32_t n1 = 0;
  for (int32_t cd = 0; cd < M; ++cd) {
    const int32_t c = corig[cd];
    max_check_deg = std::max(max_check_deg, code.check_degree(c));
    int4 d;
    d.x = static_cast<int32_t>(chk_hi_h.size());
    for (int32_t e = code.check_ptr[c]; e < code.check_ptr[c + 1]; ++e) {
      const int32_t v = code.check_vars[e];
      if (deg[v] >= 2) {
        hi_of_edge[e] = static_cast<int32_t>(chk_hi_h.size());
        chk_hi_h.push_back(vmap[v]);
      }
    }
    d.y = static_cast<int32_t>(chk_hi_h.size());
    d.z = n1;
    for (int32_t e = code.check_ptr[c]; e < code.check_ptr[c + 1]; ++e) {
      const int32_t v = code.check_vars[e];
      if (deg[v] == 1) {
        vmap[v] = -1 - n1;
        dorig.push_back(v);
        ++n1;
      }
    }
    d.w = n1;
    cdesc[cd] = d;
  }
  if (max_check_deg > 256) throw ValidationError("decoder: check degree above 256 is not supported");
  // chunk descriptors: {NH*8+ND for a homogeneous full chunk of 32 checks of a
  // typed-path shape else -1, first hi edge, first degree-1 row, hi edge end}
  std::vector<int4> ctype((M + 31) / 32);
  for (size_t k = 0; k < ctype.size(); ++k) {
    const int32_t c0 = static_cast<int32_t>(k * 32);
    const int32_t c1 = std::min<int32_t>(M, c0 + 32);
    int4 t;
    t.x = -1;
    t.y = cdesc[c0].x;
    t.z = cdesc[c0].z;
    t.w = cdesc[c1 - 1].y;
    if (c1 - c0 == 32) {
      const int32_t t0 = cnh[corig[c0]] * 8 + cnd[corig[c0]];
      bool same = true;
      for (int32_t i = 1; i < 32 && same; ++i) same = cnh[corig[c0 + i]] * 8 + cnd[corig[c0 + i]] == t0;
      const bool shape_ok = t0 == 1 || t0 == 8 || t0 == 9 || t0 == 16 || t0 == 17 || t0 == 24 || t0 == 25 ||
                            t0 == 32 || t0 == 33 || t0 == 40 || t0 == 41 || t0 == 48;
      if (same && shape_ok) t.x = t0;
    }
    ctype[k] = t;
  }
  // k_check hand-out order: generic chunks (register path, latency-bound)
  // first, degree-1-only chunks (skipped after a frame's first iteration) last
  std::vector<int32_t> csched;
  csched.reserve(ctype.size());
  for (int pass = 0; pass < 3; ++pass)
    for (size_t k = 0; k < ctype.size(); ++k) {
      const int x = ctype[k].x;
      const int cls = x < 0 ? 0 : ((x == 1 || x == 8) ? 2 : 1);
      if (cls == pass) csched.push_back(static_cast<int32_t>(k));
    }
  const int64_t EH = static_cast<int64_t>(chk_hi_h.size());
  std::vector<int32_t> vptr(NV + 1, 0), vedge;
  vedge.reserve(EH);
  for (int32_t h = 0; h < NV; ++h) {
    const int32_t v = horig[h];
    // ascending ORIGINAL check order: the reference's summation order
    for (int32_t k = code.var_ptr[v]; k < code.var_ptr[v + 1]; ++k) vedge.push_back(hi_of_edge[code.var_edges[k]]);
    vptr[h + 1] = static_cast<int32_t>(vedge.size());
  }
  const int32_t n_tiles = std::max(1, (NV + kQTile - 1) / kQTile);
  // k_var tiles: a tile of max degree <= 16 runs the typed path at the next
  // supported degree D, its variables' CSC slices padded with -1 to D (and
  // missing variables of the last tile padded entirely)
  std::vector<int2> vtile(n_tiles);
  std::vector<int32_t> vedge_t;
  for (int32_t t = 0; t < n_tiles; ++t) {
    const int32_t h0 = t * kQTile, h1 = std::min(NV, h0 + kQTile);
    int32_t dmax = 0;
    for (int32_t h = h0; h < h1; ++h) dmax = std::max(dmax, vptr[h + 1] - vptr[h]);
    int32_t D = -1;
    for (int32_t d : {2, 3, 4, 6, 8, 12, 16, 20, 24, 32})
      if (D < 0 && dmax <= d) D = d;
    vtile[t] = make_int2(D, D < 0 ? vptr[std::min(h0, NV)] : static_cast<int32_t>(vedge_t.size()));
    if (D < 0) continue;
    for (int32_t i = 0; i < kQTile; ++i) {
      const int32_t h = h0 + i;
      int32_t k = 0;
      if (h < NV)
        for (; k < vptr[h + 1] - vptr[h]; ++k) vedge_t.push_back(vedge[vptr[h] + k]);
      for (; k < D; ++k) vedge_t.push_back(-1);
    }
  }
  int32_t dmax_typed = 2;
  for (int32_t t = 0; t < n_tiles; ++t) dmax_typed = std::max(dmax_typed, vtile[t].x);
  // keep 16-byte alignment of every tile slice (cp.async 16)
  for (int32_t t = 0; t < n_tiles; ++t)
    if (vtile[t].x >= 0 && (vtile[t].y & 3) != 0) throw CudaError("decoder: internal layout error (vedge_t alignment)");
  std::vector<int32_t> vsched;
  vsched.reserve(n_tiles);
  for (int32_t t = 0; t < n_tiles; ++t)
    if (vtile[t].x < 0) vsched.push_back(t);
  for (int32_t t = 0; t < n_tiles; ++t)
    if (vtile[t].x >= 0) vsched.push_back(t);

  Args& a = base;
  a.compact_hyst = 32;
  a.N = N;
  a.M = M;
  a.NH = NH;
  a.NV = NV;
  a.N1 = n1;
  a.EH = EH;
  a.n_tiles = n_tiles;
  a.G = G;
  a.MW = (M + 31) / 32;
  a.NW = (N + 31) / 32;
  auto up = [&](const auto& vec, auto* dptr) {
    using T = std::remove_pointer_t<decltype(dptr)>;
    T* p = dalloc<T>(vec.size(), &dev_bytes);
    owned.push_back(p);
    if (!vec.empty()) CUDA_OK(cudaMemcpy(p, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice));
    return p;
  };
  a.cdesc = up(cdesc, static_cast<int4*>(nullptr));
  a.chk_hi_h = up(chk_hi_h, static_cast<int32_t*>(nullptr));
  a.vptr = up(vptr, static_cast<int32_t*>(nullptr));
  a.vedge = up(vedge, static_cast<int32_t*>(nullptr));
  a.vmap = up(vmap, static_cast<int32_t*>(nullptr));
  std::vector<int32_t> cdev(M);
  for (int32_t cd = 0; cd < M; ++cd) cdev[corig[cd]] = cd;
  a.cdev = up(cdev, static_cast<int32_t*>(nullptr));
  a.ctype = up(ctype, static_cast<int4*>(nullptr));
  a.csched = up(csched, static_cast<int32_t*>(nullptr));
  a.vtile = up(vtile, static_cast<int2*>(nullptr));
  a.vsched = up(vsched, static_cast<int32_t*>(nullptr));
  a.vedge_t = up(vedge_t, static_cast<int32_t*>(nullptr));
  a.ve_stride = 32 * dmax_typed;
  var_smem = kVarWarps * var_smem_per_warp(a.ve_stride);
  d_check_ptr = up(code.check_ptr, static_cast<int32_t*>(nullptr));
  d_check_vars = up(code.check_vars, static_cast<int32_t*>(nullptr));

  auto own = [&](auto* p) {
    owned.push_back(p);
    return p;
  };
  const size_t L = kLanes;
  a.llr_h = own(dalloc<float>(static_cast<size_t>(G) * NH * L, &dev_bytes));
  a.llr_d = own(dalloc<float>(static_cast<size_t>(G) * n1 * L, &dev_bytes));
  a.post = own(dalloc<float>(static_cast<size_t>(G) * NV * L, &dev_bytes));
  a.c2v = own(dalloc<float>(static_cast<size_t>(G) * EH * L, &dev_bytes));
  a.d1post = nullptr;  // allocated on first request
  a.hbits = own(dalloc<uint32_t>(static_cast<size_t>(G) * NV, &dev_bytes));
  a.ebits = own(dalloc<uint32_t>(static_cast<size_t>(G) * EH, &dev_bytes));
  a.d1bits = own(dalloc<uint32_t>(static_cast<size_t>(G) * n1, &dev_bytes));
  a.synp = own(dalloc<uint32_t>(static_cast<size_t>(G) * M, &dev_bytes));
  a.syn_target = own(dalloc<uint32_t>(static_cast<size_t>(G) * M, &dev_bytes));
  a.q_part = own(dalloc<double>(static_cast<size_t>(G) * a.n_tiles * L, &dev_bytes));
  a.q_mid = own(dalloc<double>(static_cast<size_t>(G) * kTermBlocks * L, &dev_bytes));
  a.stop_frame = own(dalloc<int32_t>(S, &dev_bytes));
  a.qprev = own(dalloc<double>(S, &dev_bytes));
  a.slot_iter = own(dalloc<int32_t>(S, &dev_bytes));
  a.slot_frame = own(dalloc<int32_t>(S, &dev_bytes));
  a.pending_frame = own(dalloc<int32_t>(S, &dev_bytes));
  a.group_active = own(dalloc<uint32_t>(G, &dev_bytes));
  a.fail = own(dalloc<uint32_t>(G, &dev_bytes));
  a.stopped = own(dalloc<uint32_t>(G, &dev_bytes));
  a.load_mask = own(dalloc<uint32_t>(G, &dev_bytes));
  a.counters = own(dalloc<int32_t>(16, &dev_bytes));
  a.frame_iters = own(dalloc<unsigned long long>(1, &dev_bytes));
  CUDA_OK(cudaMemset(a.group_active, 0, G * sizeof(uint32_t)));
  CUDA_OK(cudaMemset(a.stopped, 0, G * sizeof(uint32_t)));
  CUDA_OK(cudaMemset(a.load_mask, 0, G * sizeof(uint32_t)));
  CUDA_OK(cudaMemset(a.syn_target, 0, static_cast<size_t>(G) * M * sizeof(uint32_t)));

  CUDA_OK(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
  CUDA_OK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
  CUDA_OK(cudaStreamCreateWithFlags(&out_stream, cudaStreamNonBlocking));
  CUDA_OK(cudaEventCreateWithFlags(&done_ev, cudaEventDisableTiming));
  for (auto& sg : staged) CUDA_OK(cudaEventCreateWithFlags(&sg.done, cudaEventDisableTiming));
  for (cudaEvent_t* e : {&up_start, &up_first, &up_done}) CUDA_OK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  CUDA_OK(cudaHostAlloc(&h_counters, kRing * kPollWords * sizeof(int32_t), cudaHostAllocMapped));
  std::memset(h_counters, 0, kRing * kPollWords * sizeof(int32_t));
  CUDA_OK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&base.h_poll), h_counters, 0));
  for (auto& e : ring_ev) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));

  const int sms = prop.multiProcessorCount;
  sms_ = sms;
  {
    // k_check warps run dynamically scheduled chunk loops: one wave
    int per_sm = 0, per_sm2 = 0;
    auto occ = [&](auto kern) {
      int n = 0;
      CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kCheckThreads, 0));
      return n;
    };
#define BPDEC_OCC(D)                                              \
  if (per_sm == 0 && max_check_deg <= D) {                        \
    per_sm = occ(k_check<D, false>);                              \
    per_sm2 = occ(k_check<D, true>);                              \
  }
    BPDEC_OCC(3)
    BPDEC_OCC(4)
    BPDEC_OCC(6)
    BPDEC_OCC(8)
    BPDEC_OCC(16)
    BPDEC_OCC(256)
#undef BPDEC_OCC
    grid_check = sms * std::max(1, std::min(per_sm, per_sm2));
  }
  {
    // k_var warps run persistent, dynamically scheduled tile streams: one wave
    int per_sm = 0;
    CUDA_OK(cudaFuncSetAttribute(k_var<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(var_smem)));
    CUDA_OK(cudaFuncSetAttribute(k_var<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(var_smem)));
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_var<1>, kVarWarps * 32, var_smem));
    grid_var = sms * std::max(1, per_sm);
  }
  grid_syn = sms * 2;  // syndrome warps grab passes dynamically (k_decide)
  // load / extract are no-ops on most steps: keep their grids small
  turn_item_blocks = sms * 8;
  turn_check_blocks = sms * 2;
}

GpuDecoder::~GpuDecoder() {
  stream_release();
  release();
}

void GpuDecoder::release() noexcept {
  cudaSetDevice(device);
  for (void* p : owned) dev_free(p);
  if (base.d1post) dev_free(base.d1post);
  for (auto& e : ring_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : prof_ev) cudaEventDestroy(e);
  prof_ev.clear();
  for (auto& e : ring_ev) e = nullptr;
  if (h_counters) cudaFreeHost(h_counters);
  for (auto& sg : staged)
    if (sg.done) cudaEventDestroy(sg.done);
  for (cudaEvent_t e : {up_start, up_first, up_done})
    if (e) cudaEventDestroy(e);
  if (h_avail) cudaFreeHost(h_avail);
  h_avail = nullptr;
  if (h_done) cudaFreeHost(h_done);
  h_done = nullptr;
  h_done_cap = 0;
  if (done_ev) cudaEventDestroy(done_ev);
  done_ev = nullptr;
  if (out_stream) cudaStreamDestroy(out_stream);
  out_stream = nullptr;
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (own_stream) cudaStreamDestroy(own_stream);
  owned.clear();
  base.d1post = nullptr;
  h_counters = nullptr;
  copy_stream = own_stream = nullptr;
}

template <typename F>
void GpuDecoder::launch(int kid, cudaStream_t st, F&& f) {
  // events come from a pool reused across decodes (creation is not free);
  // in stream mode the worker thread records them and stream_release
  // harvests them once the stream is closed
  const size_t k = prof_kid.size();
  const bool profiling = this->profiling;
  if (profiling) {
    while (prof_ev.size() < 2 * (k + 1)) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreate(&e));
      prof_ev.push_back(e);
    }
    CUDA_OK(cudaEventRecord(prof_ev[2 * k], st));
  }
  f();
  CUDA_OK(cudaGetLastError());
  ++launches;
  if (profiling) {
    CUDA_OK(cudaEventRecord(prof_ev[2 * k + 1], st));
    prof_kid.push_back(kid);
  }
}

// per-launch event times (and the frame-iterations counter) of the launches
// recorded since the last harvest; the launching stream is idle
cudaError_t GpuDecoder::harvest_profile(const unsigned long long* d_frame_iters) noexcept {
  unsigned long long fi = 0;
  cudaError_t e = cudaMemcpy(&fi, d_frame_iters, sizeof(fi), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return e;
  prof_frame_iters += static_cast<double>(fi);
  for (size_t k = 0; k < prof_kid.size(); ++k) {
    float ms = 0.0f;
    e = cudaEventElapsedTime(&ms, prof_ev[2 * k], prof_ev[2 * k + 1]);
    if (e != cudaSuccess) break;
    prof_ms[prof_kid[k]] += ms;
    prof_launches[prof_kid[k]] += 1;
  }
  prof_kid.clear();
  return e;
}

void GpuDecoder::launch_turnover(const Args& a, cudaStream_t st, bool want_post) {
  const int grid = turn_item_blocks + turn_check_blocks + 1;
  if (want_post)
    launch_pdl(k_turnover<true>, grid, kThreads, 0, st, a, turn_item_blocks, turn_check_blocks);
  else
    launch_pdl(k_turnover<false>, grid, kThreads, 0, st, a, turn_item_blocks, turn_check_blocks);
}

void GpuDecoder::run_step(const Args& a, cudaStream_t st, bool want_post) {
  const int md = max_check_deg;
  launch(kCheck, st, [&] {
#define BPDEC_CHECK_CASE(D)                                                                 \
  if (md <= D) {                                                                            \
    if (want_post)                                                                          \
      launch_pdl(k_check<D, true>, grid_check, kCheckThreads, 0, st, a);                         \
    else                                                                                    \
      launch_pdl(k_check<D, false>, grid_check, kCheckThreads, 0, st, a);                        \
    return;                                                                                 \
  }
    BPDEC_CHECK_CASE(3)
    BPDEC_CHECK_CASE(4)
    BPDEC_CHECK_CASE(6)
    BPDEC_CHECK_CASE(8)
    BPDEC_CHECK_CASE(16)
    BPDEC_CHECK_CASE(256)
#undef BPDEC_CHECK_CASE
  });
  launch(kVar, st, [&] {
    if (a.q_mode == 0)
      launch_pdl(k_var<0>, grid_var, kVarWarps * 32, var_smem, st, a);
    else
      launch_pdl(k_var<1>, grid_var, kVarWarps * 32, var_smem, st, a);
  });
  if (a.out_ptrace) launch(kTrace, st, [&] { launch_pdl(k_trace_post, sms_ * 4, kThreads, 0, st, a); });
  {
    const int syn_blocks = (a.use_pce || a.out_syntrace) ? grid_syn : 0;
    launch(kSyn, st, [&] {
      launch_pdl(k_decide, syn_blocks + G * kTermBlocks, kThreads, G * sizeof(uint32_t), st, a, syn_blocks);
    });
  }
  launch(kTurnover, st, [&] { launch_turnover(a, st, want_post); });
  // tail compaction (no-op unless the queue is drained and live frames fit
  // in fewer groups; decided on the device, no host round trip)
  if (G > 1 && G <= kMaxCompactGroups) launch(kCompact, st, [&] { launch_pdl(k_compact, sms_ * 4, kThreads, 0, st, a); });
}

void GpuDecoder::decode(const DecodeParams& p, const DecodeBuffers& b, cudaStream_t st_in) {
  DeviceGuard dg(device);
  CUDA_OK(dg.status());
  if (stream_) throw ConfigError("decode: a stream is open on this decoder (bpdec_stream_close first)");
  const cudaStream_t st = st_in ? st_in : own_stream;
  if (p.d_max <= 0) throw ValidationError("decode: d_max must be positive");
  if (!(p.msg_clamp > 0.0f)) throw ValidationError("decode: msg_clamp must be positive");
  if (b.batch < 0) throw ValidationError("decode: batch must be non-negative");
  if (b.batch == 0) return;
  if (b.llr == nullptr) throw ValidationError("decode: null LLR pointer");
  if (b.iterations == nullptr || b.reasons == nullptr) throw ValidationError("decode: iterations/reason outputs are required");
  Args a = base;
  const size_t B = static_cast<size_t>(b.batch);
  const bool want_post = b.posteriors != nullptr || b.post_trace != nullptr;
  if (want_post && a.d1post == nullptr) {
    a.d1post = dalloc<float>(static_cast<size_t>(G) * a.N1 * kLanes, &dev_bytes);
    base.d1post = a.d1post;
  }
  a.batch = b.batch;
  a.d_max = p.d_max;
  a.use_pce = p.use_pce;
  a.use_vnr = p.use_vnr;
  a.q_mode = p.q_mode;
  a.clamp = p.msg_clamp;
  // narrow tail groups: the folded check paths exist for check degree <= 4
  // (k_check<3|4>); a free group to move into needs G >= 2.
  // BPDEC_NO_NARROW=1 keeps every group wide (tests compare both).
  a.narrow_ok = (max_check_deg <= 4 && G >= 2 && !no_narrow) ? 1 : 0;

  // inputs (a host batch staged earlier by stage_inputs is used in place:
  // its copy already ran on copy_stream)
  Staged* sg = nullptr;
  if (!is_device_ptr(b.llr)) {
    for (auto& c : staged)
      if (c.valid && c.llr_host == b.llr && c.syn_host == b.syndrome && c.batch == b.batch &&
          (sg == nullptr || c.seq < sg->seq))
        sg = &c;
  }
  if (sg != nullptr) {
    CUDA_OK(cudaStreamWaitEvent(st, sg->done, 0));
    a.in_llr = static_cast<const float*>(sg->llr.ptr);
    a.in_syn = b.syndrome ? static_cast<const uint32_t*>(sg->syn.ptr) : nullptr;
    sg->valid = false;  // consumed; its buffers are free once this (synchronous) decode returns
  } else if (is_device_ptr(b.llr)) {
    a.in_llr = b.llr;
  } else {
    a.in_llr = static_cast<float*>(s_llr.get(B * a.N * sizeof(float)));
  }
  if (sg == nullptr) a.in_syn = nullptr;
  if (sg == nullptr && b.syndrome) {
    a.in_syn = is_device_ptr(b.syndrome) ? b.syndrome
                                         : static_cast<uint32_t*>(s_syn.get(B * a.MW * sizeof(uint32_t)));
  }
  // Host inputs not staged: uploaded chunk by chunk (S frames) on the copy
  // stream; after each chunk, counters[9] (frames available) is advanced by
  // a 4-byte copy on the same stream, and refills only take available frames
  // (k_decide), so the upload of later frames overlaps the decode of earlier
  // ones.  The decode waits for the first chunk only.
  const bool up_llr = sg == nullptr && !is_device_ptr(b.llr);
  const bool up_syn = sg == nullptr && b.syndrome != nullptr && !is_device_ptr(b.syndrome);
  const size_t nchunks = (B + S - 1) / S;
  // outputs (device targets; staged when the caller passed host memory)
  auto dev_out = [&](void* user, size_t bytes, Scratch& s, bool* staged) -> void* {
    *staged = false;
    if (user == nullptr) return nullptr;
    if (is_device_ptr(user)) return user;
    *staged = true;
    return s.get(bytes);
  };
  const size_t bits_bytes = b.bits_packed ? B * a.NW * sizeof(uint32_t) : B * a.N;
  bool st_bits, st_it, st_rs, st_post, st_q;
  void* d_bits = dev_out(b.bits, bits_bytes, s_bits, &st_bits);
  a.out_bits_u8 = (!b.bits_packed && d_bits) ? static_cast<uint8_t*>(d_bits) : nullptr;
  a.out_bits_pk = (b.bits_packed && d_bits) ? static_cast<uint32_t*>(d_bits) : nullptr;
  a.out_iters = static_cast<int32_t*>(dev_out(b.iterations, B * sizeof(int32_t), s_iters, &st_it));
  a.out_reasons = static_cast<uint8_t*>(dev_out(b.reasons, B, s_reasons, &st_rs));
  a.out_post = static_cast<float*>(dev_out(b.posteriors, B * a.N * sizeof(float), s_post, &st_post));
  a.out_qtrace = static_cast<double*>(dev_out(b.q_trace, B * p.d_max * sizeof(double), s_qtrace, &st_q));
  if (a.out_qtrace) CUDA_OK(cudaMemsetAsync(a.out_qtrace, 0xff, B * p.d_max * sizeof(double), st));  // NaN
  if (want_post && a.out_post == nullptr) a.out_post = static_cast<float*>(s_post.get(B * a.N * sizeof(float)));
  bool st_syt, st_pt;
  const size_t ptrace_n = B * static_cast<size_t>(p.d_max) * a.N;
  a.out_syntrace = static_cast<uint8_t*>(dev_out(b.syn_trace, B * p.d_max, s_syntrace, &st_syt));
  a.out_ptrace = static_cast<float*>(dev_out(b.post_trace, ptrace_n * sizeof(float), s_ptrace, &st_pt));
  if (a.out_syntrace) CUDA_OK(cudaMemsetAsync(a.out_syntrace, 0xff, B * p.d_max, st));
  if (a.out_ptrace) CUDA_OK(cudaMemsetAsync(a.out_ptrace, 0xff, ptrace_n * sizeof(float), st));  // NaN past the stop
  // eager output copies: per-frame rows of the staged host outputs
  const size_t row_bits = b.bits_packed ? a.NW * sizeof(uint32_t) : static_cast<size_t>(a.N);
  const bool eager = (st_bits || st_post || st_q) && a.out_iters != nullptr && !no_eager && !st_syt && !st_pt;
  std::vector<char> copied;
  if (eager) {
    CUDA_OK(cudaMemsetAsync(a.out_iters, 0, B * sizeof(int32_t), st));  // 0 = still decoding
    if (h_done_cap < B) {
      if (h_done) cudaFreeHost(h_done);
      h_done = nullptr;
      h_done_cap = 0;
      CUDA_OK(cudaHostAlloc(&h_done, B * sizeof(int32_t), cudaHostAllocMapped));
      CUDA_OK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_done_dev), h_done, 0));
      h_done_cap = B;
    }
    copied.assign(B, 0);
  }
  // copies rows [f0, f1) of every staged per-frame output on stream `s`
  auto copy_rows = [&](size_t f0, size_t f1, cudaStream_t s) {
    const size_t n = f1 - f0;
    if (st_bits)
      CUDA_OK(cudaMemcpyAsync(static_cast<char*>(b.bits) + f0 * row_bits, static_cast<char*>(d_bits) + f0 * row_bits,
                              n * row_bits, cudaMemcpyDeviceToHost, s));
    if (st_post)
      CUDA_OK(cudaMemcpyAsync(b.posteriors + f0 * a.N, a.out_post + f0 * a.N, n * a.N * sizeof(float),
                              cudaMemcpyDeviceToHost, s));
    if (st_q)
      CUDA_OK(cudaMemcpyAsync(b.q_trace + f0 * p.d_max, a.out_qtrace + f0 * p.d_max, n * p.d_max * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
  };
  // frames whose snapshot says "stopped" and that are not copied yet, as ranges
  auto copy_finished = [&](const int32_t* snap, cudaStream_t s, bool all) {
    size_t f = 0;
    while (f < B) {
      if (copied[f] || (!all && snap[f] == 0)) {
        ++f;
        continue;
      }
      size_t e = f;
      while (e < B && !copied[e] && (all || snap[e] != 0)) copied[e++] = 1;
      copy_rows(f, e, s);
      f = e;
    }
  };
  int64_t last_done_seen = 0;  // frames-done count when the last snapshot was requested
  bool snap_pending = false, snap_request = false;

  // initial slot assignment (frames 0..min(B,S)-1 -> slots 0..) and state
  // reset on the device: no host copies, no host synchronisation
  const int first = static_cast<int>(std::min<size_t>(B, S));
  k_decode_init<<<1, 1024, 0, st>>>(a, first, (up_llr || up_syn) ? first : static_cast<int>(B));
  CUDA_OK(cudaGetLastError());
  // (the uploads start after the init kernel, so its reset of counters[9]
  // cannot overwrite a later availability update)
  if (up_llr || up_syn) {
    if (h_avail_n < nchunks) {
      if (h_avail) cudaFreeHost(h_avail);
      h_avail = nullptr;
      h_avail_n = 0;
      CUDA_OK(cudaHostAlloc(&h_avail, nchunks * sizeof(int32_t), cudaHostAllocDefault));
      h_avail_n = nchunks;
    }
    CUDA_OK(cudaEventRecord(up_start, st));  // uploads begin after earlier work on st
    CUDA_OK(cudaStreamWaitEvent(copy_stream, up_start, 0));
    for (size_t c = 0; c < nchunks; ++c) {
      const size_t f0 = c * S, nf = std::min<size_t>(S, B - f0);
      if (up_llr)
        CUDA_OK(cudaMemcpyAsync(const_cast<float*>(a.in_llr) + f0 * a.N, b.llr + f0 * a.N, nf * a.N * sizeof(float),
                                cudaMemcpyHostToDevice, copy_stream));
      if (up_syn)
        CUDA_OK(cudaMemcpyAsync(const_cast<uint32_t*>(a.in_syn) + f0 * a.MW, b.syndrome + f0 * a.MW,
                                nf * a.MW * sizeof(uint32_t), cudaMemcpyHostToDevice, copy_stream));
      h_avail[c] = static_cast<int32_t>(f0 + nf);
      if (c == 0) CUDA_OK(cudaEventRecord(up_first, copy_stream));
      if (c > 0)  // chunk 0 is available by construction (the decode waits for it)
        CUDA_OK(cudaMemcpyAsync(a.counters + 9, h_avail + c, sizeof(int32_t), cudaMemcpyHostToDevice, copy_stream));
    }
    CUDA_OK(cudaEventRecord(up_done, copy_stream));
  }
  if (up_llr || up_syn) CUDA_OK(cudaStreamWaitEvent(st, up_first, 0));
  launch(kTurnover, st, [&] { launch_turnover(a, st, false); });
  CUDA_OK(cudaMemsetAsync(a.load_mask, 0, G * sizeof(uint32_t), st));

  // step loop: poll the frames-done counter with a lag so the GPU never idles
  const int64_t waves = (static_cast<int64_t>(B) + S - 1) / S;
  int64_t max_steps = static_cast<int64_t>(p.d_max) * waves + 2;
  // lag 2: the GPU always has the next step queued, and at most two empty
  // steps run after the last frame stops (lag 1/2/4 measured: 2 keeps slack
  // for a busy host at no cost)
  constexpr int kLag = 2;
  int64_t step = 0;
  bool done = false;
  bool uploading = up_llr || up_syn;
  // safety bound on the step count (frames must terminate within d_max
  // steps per wave); while chunks are still uploading, steps spent waiting
  // for frames do not count
  for (; (uploading || step < max_steps + kLag) && !done; ++step) {
    if (uploading) {
      const cudaError_t q = cudaEventQuery(up_done);
      if (q == cudaSuccess) {
        uploading = false;
        max_steps = std::max(max_steps, step + static_cast<int64_t>(p.d_max) * waves + 2);
      } else if (q == cudaErrorNotReady) {
        (void)cudaGetLastError();  // not an error: keep it out of the launch checks
      } else {
        CUDA_OK(q);
      }
    }
    const int slot = static_cast<int>(step % kRing);
    a.poll_slot = slot;  // k_decide of this step reports into h_counters[slot]
    run_step(a, st, want_post);
    if (snap_request) {
      // snapshot of out_iters in stream order after this step's k_turnover:
      // every frame it marks stopped has had its outputs extracted
      snap_request = false;
      launch(kSnapshot, st, [&] {
        launch_pdl(k_snapshot, 4, 256, 0, st, static_cast<const int32_t*>(a.out_iters), b.batch, h_done_dev);
      });
      CUDA_OK(cudaEventRecord(done_ev, st));
      snap_pending = true;
    }
    CUDA_OK(cudaEventRecord(ring_ev[slot], st));
    if (step >= kLag) {
      const int old = static_cast<int>((step - kLag) % kRing);
      CUDA_OK(cudaEventSynchronize(ring_ev[old]));
      const volatile int32_t* hp = h_counters + kPollWords * old;
      if (hp[2] != 0) break;  // invalid input detected
      if (hp[1] >= b.batch) done = true;
      if (eager) {
        // a finished snapshot: copy the rows it marks final (out_stream is
        // ordered after the snapshot, and so after the extraction)
        if (snap_pending && cudaEventQuery(done_ev) == cudaSuccess) {
          snap_pending = false;
          CUDA_OK(cudaStreamWaitEvent(out_stream, done_ev, 0));
          copy_finished(h_done, out_stream, false);
        } else {
          (void)cudaGetLastError();  // cudaErrorNotReady is not an error here
        }
        // frames stopped since the last snapshot: request a snapshot after
        // the next launched step
        const int64_t nd = hp[1];
        if (!snap_pending && !done && nd >= last_done_seen + 8) {
          last_done_seen = nd;
          snap_request = true;
        }
      }
    }
  }
  CUDA_OK(cudaStreamSynchronize(st));
  if (up_llr || up_syn) CUDA_OK(cudaEventSynchronize(up_done));  // host buffers no longer read
  int32_t ctr[4];
  CUDA_OK(cudaMemcpy(ctr, a.counters, sizeof(ctr), cudaMemcpyDeviceToHost));
  if (ctr[2] != 0 || ctr[1] < b.batch) {
    if (eager) CUDA_OK(cudaStreamSynchronize(out_stream));  // no copy into the caller's buffers after the throw
    if (ctr[2] != 0) throw ValidationError("decode: non-finite input LLR");
    throw CudaError("decode: internal error, frames did not terminate");
  }
  if (profiling) CUDA_OK(harvest_profile(a.frame_iters));
  // copy staged outputs back (eager: only the rows not copied during the decode)
  if (eager) {
    if (snap_pending) {
      CUDA_OK(cudaEventSynchronize(done_ev));
      CUDA_OK(cudaStreamWaitEvent(out_stream, done_ev, 0));
      copy_finished(h_done, out_stream, false);
    }
    copy_finished(nullptr, st, true);
  } else {
    if (st_bits) CUDA_OK(cudaMemcpyAsync(b.bits, d_bits, bits_bytes, cudaMemcpyDeviceToHost, st));
    if (st_post)
      CUDA_OK(cudaMemcpyAsync(b.posteriors, a.out_post, B * a.N * sizeof(float), cudaMemcpyDeviceToHost, st));
    if (st_q)
      CUDA_OK(cudaMemcpyAsync(b.q_trace, a.out_qtrace, B * p.d_max * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  if (st_syt) CUDA_OK(cudaMemcpyAsync(b.syn_trace, a.out_syntrace, B * p.d_max, cudaMemcpyDeviceToHost, st));
  if (st_pt)
    CUDA_OK(cudaMemcpyAsync(b.post_trace, a.out_ptrace, ptrace_n * sizeof(float), cudaMemcpyDeviceToHost, st));
  if (st_it) CUDA_OK(cudaMemcpyAsync(b.iterations, a.out_iters, B * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (st_rs) CUDA_OK(cudaMemcpyAsync(b.reasons, a.out_reasons, B, cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaStreamSynchronize(st));
  if (eager) CUDA_OK(cudaStreamSynchronize(out_stream));
}

void GpuDecoder::stage_inputs(int32_t batch, const float* llr_host, const uint32_t* syn_host) {
  DeviceGuard dg(device);
  CUDA_OK(dg.status());
  if (stream_) throw ConfigError("stage_inputs: a stream is open on this decoder (submit to it instead)");
  if (batch <= 0) throw ValidationError("stage_inputs: batch must be positive");
  if (llr_host == nullptr) throw ValidationError("stage_inputs: null LLR pointer");
  if (is_device_ptr(llr_host) || (syn_host && is_device_ptr(syn_host)))
    throw ValidationError("stage_inputs: inputs must be host memory (device inputs need no staging)");
  // the free slot, else the older staged batch is replaced
  Staged* sg = !staged[0].valid ? &staged[0] : !staged[1].valid ? &staged[1]
             : (staged[0].seq < staged[1].seq ? &staged[0] : &staged[1]);
  const size_t B = static_cast<size_t>(batch);
  float* dl = static_cast<float*>(sg->llr.get(B * base.N * sizeof(float)));
  CUDA_OK(cudaMemcpyAsync(dl, llr_host, B * base.N * sizeof(float), cudaMemcpyHostToDevice, copy_stream));
  if (syn_host) {
    uint32_t* ds = static_cast<uint32_t*>(sg->syn.get(B * base.MW * sizeof(uint32_t)));
    CUDA_OK(cudaMemcpyAsync(ds, syn_host, B * base.MW * sizeof(uint32_t), cudaMemcpyHostToDevice, copy_stream));
  }
  CUDA_OK(cudaEventRecord(sg->done, copy_stream));
  sg->llr_host = llr_host;
  sg->syn_host = syn_host;
  sg->batch = batch;
  sg->valid = true;
  sg->seq = ++stage_seq;
}

void GpuDecoder::sample_device(double snr, double beta_lo, double beta_hi, double rate, uint64_t seed,
                               int64_t first_frame, int32_t n_frames, bool all_zero,
                               float* d_llr, uint32_t* d_syn, uint32_t* d_x, cudaStream_t st_in) {
  DeviceGuard dg(device);
  CUDA_OK(dg.status());
  const cudaStream_t st = st_in ? st_in : own_stream;
  if (snr > 0.0) {
    if (!std::isfinite(snr)) throw ValidationError("sample: snr must be positive and finite");
  } else if (!(beta_lo > 0.0) || beta_hi > 1.0 || beta_hi < beta_lo || !(rate > 0.0) || rate >= 1.0) {
    throw ValidationError("sample: need snr > 0 or 0 < beta_lo <= beta_hi <= 1 and 0 < rate < 1");
  }
  if (n_frames <= 0) return;
  uint32_t* x = d_x;
  Scratch tmp;
  if (x == nullptr && d_syn != nullptr) x = static_cast<uint32_t*>(tmp.get(static_cast<size_t>(n_frames) * base.NW * 4));
  k_gen_llr<<<1184, kThreads, 0, st>>>(base.N, base.NW, snr > 0.0 ? snr : 0.0, beta_lo, beta_hi, rate, seed,
                                       first_frame, n_frames, all_zero ? 1 : 0, d_llr, x);
  CUDA_OK(cudaGetLastError());
  ++launches;
  if (d_syn) {
    k_gen_syndrome<<<592, kThreads, 0, st>>>(base, n_frames, x, d_syn, d_check_ptr, d_check_vars);
    CUDA_OK(cudaGetLastError());
    ++launches;
  }
  CUDA_OK(cudaStreamSynchronize(st));
}


// ------------------------------------------------------------ stream mode --
// Batches submitted back to back decode as ONE frame stream: frame g (global
// index since the stream opened) has its input and output rows at ring
// position g % cap of device rings, becomes available to the refill when its
// batch's upload has landed (counters[9], advanced by a 4-byte copy on the
// copy stream after the batch's rows), and a worker thread keeps launching
// decoding steps while frames are in flight.  k_decide counts stopped frames
// per batch slot (bdone, via fbatch) and reports the counts with the step's
// poll words; a batch whose count reached its size has final outputs after
// that step, which are then copied to the caller's buffers on out_stream.
// So the lanes an earlier batch's tail frees are refilled with the next
// batch's frames in the same step, and batch k+1's upload overlaps batch k's
// decode.  Per-frame results do not depend on slot, order or neighbours, so
// every batch's outputs equal a blocking decode of that batch.
struct GpuDecoder::Stream {
  DecodeParams p;
  bool packed = false, want_bits = true, want_post = false, want_q = false;
  int32_t cap = 0;
  // device rings
  float* r_llr = nullptr;
  uint32_t* r_syn = nullptr;
  int32_t* r_fbatch = nullptr;
  uint8_t* r_ferr = nullptr;
  int32_t* r_bdone = nullptr;
  void* r_bits = nullptr;
  int32_t* r_iters = nullptr;
  uint8_t* r_reasons = nullptr;
  float* r_post = nullptr;
  double* r_q = nullptr;
  // pinned host staging
  int32_t* h_fbatch = nullptr;  // [cap]
  int32_t* h_avail = nullptr;   // [kMaxStreamBatches][kAvailPieces]
  uint8_t* h_ferr = nullptr;    // [cap]
  Args a{};
  struct Batch {
    int state = 0;  // 0 free, 1 decoding, 2 copying outputs
    int64_t ticket = -1, g0 = 0, target = 0;
    int32_t n = 0;
    StreamOutputs out;
    cudaEvent_t ev = nullptr;
  };
  Batch batches[kMaxStreamBatches];
  int64_t slot_total[kMaxStreamBatches] = {};  // cumulative frames per batch slot (bdone targets)
  std::deque<int64_t> order;    // tickets of live batches in submission order (ring frees in order)
  std::map<int64_t, std::string> finished;  // ticket -> error ("" = ok) until waited for
  std::mutex mu, submit_mu;
  std::condition_variable cv_work, cv_done;
  std::thread worker;
  bool closing = false;
  std::string fatal;            // worker error: every pending and later call fails with it
  int64_t next_ticket = 0, next_g = 0, free_g = 0;
  int64_t decoding = 0;         // batches in state 1
  int64_t copying = 0;          // batches in state 2
  // device timer (bpdec_stream_device_ms): t_first before the first step
  // launched after a reset, t_last after each batch's output copies
  cudaEvent_t t_first = nullptr, t_last = nullptr;
  bool timer_armed = true, t_first_set = false, t_last_set = false;
};

void GpuDecoder::stream_open(const DecodeParams& p, bool packed, bool want_bits, bool want_post, bool want_q,
                             int32_t ring_frames) {
  DeviceGuard dg(device);
  CUDA_OK(dg.status());
  if (stream_) throw ConfigError("stream: already open on this decoder");
  if (p.d_max <= 0) throw ValidationError("decode: d_max must be positive");
  if (!(p.msg_clamp > 0.0f)) throw ValidationError("decode: msg_clamp must be positive");
  if (ring_frames <= 0) ring_frames = 4 * S;
  if (ring_frames < S) ring_frames = S;
  auto sp = std::make_unique<Stream>();
  Stream& z = *sp;
  z.p = p;
  z.packed = packed;
  z.want_bits = want_bits;
  z.want_post = want_post;
  z.want_q = want_q;
  z.cap = ring_frames;
  const size_t C = static_cast<size_t>(z.cap);
  std::vector<void*> got;
  auto alloc = [&](size_t bytes) {
    void* q = nullptr;
    CUDA_OK(dev_malloc(&q, std::max<size_t>(bytes, 16)));
    got.push_back(q);
    return q;
  };
  try {
    z.r_llr = static_cast<float*>(alloc(C * base.N * sizeof(float)));
    z.r_syn = static_cast<uint32_t*>(alloc(C * base.MW * sizeof(uint32_t)));
    z.r_fbatch = static_cast<int32_t*>(alloc(C * sizeof(int32_t)));
    z.r_ferr = static_cast<uint8_t*>(alloc(C));
    z.r_bdone = static_cast<int32_t*>(alloc(kMaxStreamBatches * sizeof(int32_t)));
    if (want_bits) z.r_bits = alloc(packed ? C * base.NW * sizeof(uint32_t) : C * base.N);
    z.r_iters = static_cast<int32_t*>(alloc(C * sizeof(int32_t)));
    z.r_reasons = static_cast<uint8_t*>(alloc(C));
    if (want_post) z.r_post = static_cast<float*>(alloc(C * base.N * sizeof(float)));
    if (want_q) z.r_q = static_cast<double*>(alloc(C * p.d_max * sizeof(double)));
    if (want_post && base.d1post == nullptr)
      base.d1post = dalloc<float>(static_cast<size_t>(G) * base.N1 * kLanes, &dev_bytes);
    CUDA_OK(cudaMemset(z.r_bdone, 0, kMaxStreamBatches * sizeof(int32_t)));
    CUDA_OK(cudaMemset(z.r_ferr, 0, C));
    CUDA_OK(cudaHostAlloc(&z.h_fbatch, C * sizeof(int32_t), cudaHostAllocDefault));
    CUDA_OK(cudaHostAlloc(&z.h_avail, kMaxStreamBatches * kAvailPieces * sizeof(int32_t), cudaHostAllocDefault));
    CUDA_OK(cudaHostAlloc(&z.h_ferr, C, cudaHostAllocDefault));
    for (auto& bt : z.batches) CUDA_OK(cudaEventCreateWithFlags(&bt.ev, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreate(&z.t_first));
    CUDA_OK(cudaEventCreate(&z.t_last));
  } catch (...) {
    for (void* q : got) dev_free(q);
    if (z.h_fbatch) cudaFreeHost(z.h_fbatch);
    if (z.h_avail) cudaFreeHost(z.h_avail);
    if (z.h_ferr) cudaFreeHost(z.h_ferr);
    for (auto& bt : z.batches)
      if (bt.ev) cudaEventDestroy(bt.ev);
    if (z.t_first) cudaEventDestroy(z.t_first);
    if (z.t_last) cudaEventDestroy(z.t_last);
    throw;
  }
  Args& a = z.a;
  a = base;
  a.batch = INT32_MAX;  // the refill limit is counters[9] (frames uploaded)
  a.d_max = p.d_max;
  a.use_pce = p.use_pce;
  a.use_vnr = p.use_vnr;
  a.q_mode = p.q_mode;
  a.clamp = p.msg_clamp;
  a.narrow_ok = 0;  // a narrow tail group cannot take refills
  a.group_refill = (G >= 2 && std::getenv("BPDEC_LANE_REFILL") == nullptr) ? 1 : 0;
  // group refill: compaction is what frees groups for queued frames, so it
  // re-packs sooner (8 frames finished: +2.3 % on cfg2 over 32; 1-8 equal)
  a.compact_hyst = a.group_refill ? 8 : 32;
  if (const char* h = std::getenv("BPDEC_COMPACT_HYST")) a.compact_hyst = std::max(1, std::atoi(h));
  a.in_llr = z.r_llr;
  a.in_syn = z.r_syn;
  a.out_bits_u8 = (want_bits && !packed) ? static_cast<uint8_t*>(z.r_bits) : nullptr;
  a.out_bits_pk = (want_bits && packed) ? static_cast<uint32_t*>(z.r_bits) : nullptr;
  a.out_iters = z.r_iters;
  a.out_reasons = z.r_reasons;
  a.out_post = z.r_post;
  a.out_qtrace = z.r_q;
  a.out_syntrace = nullptr;
  a.out_ptrace = nullptr;
  a.ring_cap = z.cap;
  a.fbatch = z.r_fbatch;
  a.bdone = z.r_bdone;
  a.ferr = z.r_ferr;
  // empty decoder: no frames, none available; refills start as batches land
  k_decode_init<<<1, 1024, 0, own_stream>>>(a, 0, 0);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaStreamSynchronize(own_stream));
  stream_ = std::move(sp);
  stream_->worker = std::thread([this] { stream_worker(); });
}

int64_t GpuDecoder::stream_submit(int32_t n, const float* llr, const uint32_t* syn, const StreamOutputs& o) {
  if (!stream_) throw ConfigError("stream: not open");
  Stream& z = *stream_;
  if (n <= 0) throw ValidationError("stream: batch must be positive");
  if (n > z.cap) throw ValidationError("stream: batch larger than the stream's ring (" + std::to_string(z.cap) + " frames)");
  if (llr == nullptr) throw ValidationError("decode: null LLR pointer");
  if (o.iterations == nullptr || o.reasons == nullptr) throw ValidationError("decode: iterations/reason outputs are required");
  if ((o.bits && !z.want_bits) || (o.posteriors && !z.want_post) || (o.q_trace && !z.want_q))
    throw ValidationError("stream: an output was requested that the stream was not opened for");
  DeviceGuard dg(device);
  CUDA_OK(dg.status());
  std::lock_guard<std::mutex> order_lock(z.submit_mu);  // ring positions and counters[9] in submission order
  int64_t t, g0;
  int slot;
  {
    std::unique_lock<std::mutex> lk(z.mu);
    z.cv_done.wait(lk, [&] {
      return !z.fatal.empty() || (z.next_g + n - z.free_g <= z.cap &&
                                  z.batches[z.next_ticket % kMaxStreamBatches].state == 0);
    });
    if (!z.fatal.empty()) throw CudaError(z.fatal);
    if (z.next_g + n > (int64_t{1} << 30)) throw ConfigError("stream: frame index space exhausted; reopen the stream");
    t = z.next_ticket++;
    slot = static_cast<int>(t % kMaxStreamBatches);
    g0 = z.next_g;
  }
  const size_t C = static_cast<size_t>(z.cap);
  const size_t p0 = static_cast<size_t>(g0 % z.cap);
  const size_t n1 = std::min<size_t>(static_cast<size_t>(n), C - p0), n2 = static_cast<size_t>(n) - n1;
  const cudaStream_t cs = copy_stream;
  // rows [p0, p0+n1) and [0, n2) of a ring
  auto rows = [&](auto* ring, const auto* src, size_t w) {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(src)>>;
    CUDA_OK(cudaMemcpyAsync(ring + p0 * w, src, n1 * w * sizeof(T), cudaMemcpyDefault, cs));
    if (n2) CUDA_OK(cudaMemcpyAsync(ring, src + n1 * w, n2 * w * sizeof(T), cudaMemcpyDefault, cs));
  };
  auto fill = [&](void* ring, size_t w, int value) {
    CUDA_OK(cudaMemsetAsync(static_cast<char*>(ring) + p0 * w, value, n1 * w, cs));
    if (n2) CUDA_OK(cudaMemsetAsync(ring, value, n2 * w, cs));
  };
  for (size_t i = 0; i < static_cast<size_t>(n); ++i) z.h_fbatch[(p0 + i) % C] = slot;
  CUDA_OK(cudaMemcpyAsync(z.r_fbatch + p0, z.h_fbatch + p0, n1 * sizeof(int32_t), cudaMemcpyHostToDevice, cs));
  if (n2) CUDA_OK(cudaMemcpyAsync(z.r_fbatch, z.h_fbatch, n2 * sizeof(int32_t), cudaMemcpyHostToDevice, cs));
  fill(z.r_ferr, 1, 0);
  if (z.want_q) fill(z.r_q, z.p.d_max * sizeof(double), 0xff);  // NaN past the stop
  if (syn) rows(z.r_syn, syn, base.MW);
  else fill(z.r_syn, base.MW * sizeof(uint32_t), 0);
  {
    std::lock_guard<std::mutex> lk(z.mu);
    Stream::Batch& bt = z.batches[slot];
    // bdone[slot] is cumulative (never reset, so a poll taken before this
    // batch's frames count cannot look complete): the batch is done at
    // the slot's previous total + n
    z.slot_total[slot] += n;
    bt.target = z.slot_total[slot];
    bt.state = 1;
    bt.ticket = t;
    bt.g0 = g0;
    bt.n = n;
    bt.out = o;
    z.order.push_back(t);
    z.next_g = g0 + n;
    ++z.decoding;
  }
  // the LLR rows in up to kAvailPieces pieces (whole 32-frame groups), each
  // followed by the advance of the frames-available counter: the first
  // group of a batch starts decoding while the rest is still uploading
  // (the start-up of a stream: one 276 MB cfg2 batch is ~5 ms of PCIe time)
  const size_t wN = static_cast<size_t>(base.N);
  const int piece = std::max(32, ((n + kAvailPieces - 1) / kAvailPieces + 31) / 32 * 32);
  int pi = 0;
  try {
  for (int i0 = 0; i0 < n; i0 += piece, ++pi) {
    const size_t cnt = static_cast<size_t>(std::min(piece, n - i0));
    const size_t q0 = (p0 + static_cast<size_t>(i0)) % C;
    const size_t m1 = std::min(cnt, C - q0);
    CUDA_OK(cudaMemcpyAsync(z.r_llr + q0 * wN, llr + static_cast<size_t>(i0) * wN, m1 * wN * sizeof(float),
                            cudaMemcpyDefault, cs));
    if (cnt > m1)
      CUDA_OK(cudaMemcpyAsync(z.r_llr, llr + (static_cast<size_t>(i0) + m1) * wN, (cnt - m1) * wN * sizeof(float),
                              cudaMemcpyDefault, cs));
    int32_t* ha = z.h_avail + slot * kAvailPieces + pi;
    *ha = static_cast<int32_t>(g0 + i0 + static_cast<int64_t>(cnt));
    // the frames become available once their rows have landed
    CUDA_OK(cudaMemcpyAsync(base.counters + 9, ha, sizeof(int32_t), cudaMemcpyHostToDevice, cs));
  }
  } catch (const std::exception& e) {
    // the batch is registered but its frames can no longer all arrive: the
    // stream is unusable (waits and later submits fail instead of hanging)
    std::lock_guard<std::mutex> lk(z.mu);
    z.fatal = std::string("stream submit: ") + e.what();
    z.cv_done.notify_all();
    z.cv_work.notify_all();
    throw;
  }
  z.cv_work.notify_one();
  return t;
}

void GpuDecoder::stream_worker() {
  Stream& z = *stream_;
  cudaSetDevice(device);
  const cudaStream_t st = own_stream;
  constexpr int kLag = 2;
  int64_t step = 0, polled = 0;  // steps launched / polled
  Args a = z.a;
  // outputs of batch bt (ring rows -> caller buffers) on out_stream
  auto copy_out = [&](Stream::Batch& bt) {
    const size_t C = static_cast<size_t>(z.cap);
    const size_t p0 = static_cast<size_t>(bt.g0 % z.cap);
    const size_t n1 = std::min<size_t>(static_cast<size_t>(bt.n), C - p0), n2 = static_cast<size_t>(bt.n) - n1;
    auto rows = [&](void* dst, const void* ring, size_t rb) {
      if (dst == nullptr) return;
      CUDA_OK(cudaMemcpyAsync(dst, static_cast<const char*>(ring) + p0 * rb, n1 * rb, cudaMemcpyDefault, out_stream));
      if (n2)
        CUDA_OK(cudaMemcpyAsync(static_cast<char*>(dst) + n1 * rb, ring, n2 * rb, cudaMemcpyDefault, out_stream));
    };
    rows(bt.out.bits, z.r_bits, z.packed ? base.NW * sizeof(uint32_t) : static_cast<size_t>(base.N));
    rows(bt.out.iterations, z.r_iters, sizeof(int32_t));
    rows(bt.out.reasons, z.r_reasons, 1);
    rows(bt.out.posteriors, z.r_post, base.N * sizeof(float));
    rows(bt.out.q_trace, z.r_q, z.p.d_max * sizeof(double));
    // per-frame input error flags, to the same ring positions of h_ferr
    CUDA_OK(cudaMemcpyAsync(z.h_ferr + p0, z.r_ferr + p0, n1, cudaMemcpyDeviceToHost, out_stream));
    if (n2) CUDA_OK(cudaMemcpyAsync(z.h_ferr, z.r_ferr, n2, cudaMemcpyDeviceToHost, out_stream));
    CUDA_OK(cudaEventRecord(bt.ev, out_stream));
    {
      std::lock_guard<std::mutex> lk(z.mu);
      if (z.t_first_set) {
        CUDA_OK(cudaEventRecord(z.t_last, out_stream));
        z.t_last_set = true;
      }
    }
  };
  auto finish = [&](Stream::Batch& bt) {  // outputs copied: ticket done, ring rows free
    const size_t C = static_cast<size_t>(z.cap);
    const size_t p0 = static_cast<size_t>(bt.g0 % z.cap);
    bool bad = false;
    for (int32_t i = 0; i < bt.n; ++i) bad |= z.h_ferr[(p0 + i) % C] != 0;
    std::lock_guard<std::mutex> lk(z.mu);
    z.finished[bt.ticket] = bad ? "decode: non-finite input LLR" : "";
    bt.state = 0;
    --z.copying;
    while (!z.order.empty()) {
      Stream::Batch& f = z.batches[z.order.front() % kMaxStreamBatches];
      if (f.ticket == z.order.front() && f.state != 0) break;
      z.order.pop_front();
    }
    z.free_g = z.order.empty() ? z.next_g : z.batches[z.order.front() % kMaxStreamBatches].g0;
    z.cv_done.notify_all();
  };
  try {
    for (;;) {
      bool run = false;
      {
        std::unique_lock<std::mutex> lk(z.mu);
        z.cv_work.wait(lk, [&] { return z.closing || z.decoding > 0 || z.copying > 0 || polled < step; });
        if (z.closing && z.decoding == 0 && z.copying == 0 && polled >= step) break;
        run = z.decoding > 0;
      }
      if (run) {
        {
          std::lock_guard<std::mutex> lk(z.mu);
          if (z.timer_armed) {
            CUDA_OK(cudaEventRecord(z.t_first, st));
            z.timer_armed = false;
            z.t_first_set = true;
            z.t_last_set = false;
          }
        }
        const int slot = static_cast<int>(step % kRing);
        a.poll_slot = slot;
        run_step(a, st, z.want_post);
        CUDA_OK(cudaEventRecord(ring_ev[slot], st));
        ++step;
      }
      // poll the step launched kLag steps ago (or every outstanding one when idle)
      while (polled < step && (polled + kLag < step || !run)) {
        const int old = static_cast<int>(polled % kRing);
        CUDA_OK(cudaEventSynchronize(ring_ev[old]));
        const volatile int32_t* hp = h_counters + kPollWords * old;
        ++polled;
        std::vector<Stream::Batch*> done;
        {
          std::lock_guard<std::mutex> lk(z.mu);
          for (auto& bt : z.batches)
            if (bt.state == 1 && hp[4 + (&bt - z.batches)] >= bt.target) done.push_back(&bt);
          for (Stream::Batch* bt : done) {
            bt->state = 2;
            --z.decoding;
            ++z.copying;
          }
        }
        if (!done.empty()) {
          CUDA_OK(cudaStreamWaitEvent(out_stream, ring_ev[old], 0));
          for (Stream::Batch* bt : done) copy_out(*bt);
        }
      }
      // batches whose outputs have been copied
      for (auto& bt : z.batches) {
        if (bt.state != 2) continue;
        const cudaError_t q = run ? cudaEventQuery(bt.ev) : cudaEventSynchronize(bt.ev);
        if (q == cudaErrorNotReady) {
          (void)cudaGetLastError();
          continue;
        }
        CUDA_OK(q);
        finish(bt);
      }
    }
  } catch (const std::exception& e) {
    std::lock_guard<std::mutex> lk(z.mu);
    z.fatal = std::string("stream worker: ") + e.what();
    z.cv_done.notify_all();
  }
}

bool GpuDecoder::stream_query(int64_t ticket) {
  if (!stream_) throw ConfigError("stream: not open");
  Stream& z = *stream_;
  std::lock_guard<std::mutex> lk(z.mu);
  if (ticket < 0 || ticket >= z.next_ticket) throw ValidationError("stream: unknown ticket");
  if (!z.fatal.empty()) throw CudaError(z.fatal);
  for (const auto& bt : z.batches)
    if (bt.state != 0 && bt.ticket == ticket) return false;
  return true;
}

void GpuDecoder::stream_wait(int64_t ticket) {
  if (!stream_) throw ConfigError("stream: not open");
  Stream& z = *stream_;
  std::unique_lock<std::mutex> lk(z.mu);
  if (ticket < 0 || ticket >= z.next_ticket) throw ValidationError("stream: unknown ticket");
  auto live = [&] {
    for (const auto& bt : z.batches)
      if (bt.state != 0 && bt.ticket == ticket) return true;
    return false;
  };
  z.cv_done.wait(lk, [&] { return !z.fatal.empty() || !live(); });
  if (!z.fatal.empty()) throw CudaError(z.fatal);
  auto it = z.finished.find(ticket);
  if (it == z.finished.end()) return;  // already collected
  const std::string err = it->second;
  z.finished.erase(it);
  if (!err.empty()) throw ValidationError(err);
}

void GpuDecoder::stream_timer_reset() {
  if (!stream_) throw ConfigError("stream: not open");
  Stream& z = *stream_;
  std::lock_guard<std::mutex> lk(z.mu);
  if (z.decoding > 0 || z.copying > 0) throw ConfigError("stream: timer reset while batches are in flight");
  z.timer_armed = true;
  z.t_first_set = z.t_last_set = false;
}

double GpuDecoder::stream_device_ms() {
  if (!stream_) throw ConfigError("stream: not open");
  Stream& z = *stream_;
  cudaEvent_t a, b;
  {
    std::lock_guard<std::mutex> lk(z.mu);
    if (!z.fatal.empty()) throw CudaError(z.fatal);
    if (!z.t_first_set || !z.t_last_set) throw ConfigError("stream: no batch completed since the timer reset");
    a = z.t_first;
    b = z.t_last;
  }
  DeviceGuard dg(device);
  CUDA_OK(dg.status());
  CUDA_OK(cudaEventSynchronize(b));
  float ms = 0.0f;
  CUDA_OK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

void GpuDecoder::stream_close() {
  if (!stream_) return;
  std::string fatal;
  {
    std::lock_guard<std::mutex> lk(stream_->mu);
    fatal = stream_->fatal;
  }
  stream_release();
  if (!fatal.empty()) throw CudaError(fatal);
}

void GpuDecoder::stream_release() noexcept {
  if (!stream_) return;
  Stream& z = *stream_;
  {
    std::lock_guard<std::mutex> lk(z.mu);
    z.closing = true;
  }
  z.cv_work.notify_all();
  if (z.worker.joinable()) z.worker.join();
  cudaSetDevice(device);
  cudaStreamSynchronize(copy_stream);
  cudaStreamSynchronize(out_stream);
  cudaStreamSynchronize(own_stream);
  if (!prof_kid.empty()) (void)harvest_profile(base.frame_iters);
  (void)cudaGetLastError();
  for (void* q : {static_cast<void*>(z.r_llr), static_cast<void*>(z.r_syn), static_cast<void*>(z.r_fbatch),
                  static_cast<void*>(z.r_ferr), static_cast<void*>(z.r_bdone), z.r_bits,
                  static_cast<void*>(z.r_iters), static_cast<void*>(z.r_reasons), static_cast<void*>(z.r_post),
                  static_cast<void*>(z.r_q)})
    if (q) dev_free(q);
  if (z.h_fbatch) cudaFreeHost(z.h_fbatch);
  if (z.h_avail) cudaFreeHost(z.h_avail);
  if (z.h_ferr) cudaFreeHost(z.h_ferr);
  for (auto& bt : z.batches)
    if (bt.ev) cudaEventDestroy(bt.ev);
  if (z.t_first) cudaEventDestroy(z.t_first);
  if (z.t_last) cudaEventDestroy(z.t_last);
  // the decoder returns to batch mode: counters and slot state are reset by
  // the next decode's init kernel
  stream_.reset();
}

// ------------------------------------------------------------ wrappers --
GpuDecoder* gpu_decoder_create(const Code& code, int device, int max_slots) {
  return new GpuDecoder(code, device, max_slots);
}
void gpu_decoder_destroy(GpuDecoder* dec) { delete dec; }
int gpu_decoder_slots(const GpuDecoder* dec) { return dec->S; }
int gpu_decoder_device(const GpuDecoder* dec) { return dec->device; }
int64_t gpu_decoder_device_bytes(const GpuDecoder* dec) { return dec->dev_bytes; }
void gpu_decode_batch(GpuDecoder* dec, const DecodeParams& p, const DecodeBuffers& b, void* stream) {
  dec->decode(p, b, static_cast<cudaStream_t>(stream));
}
void gpu_sample_frames_device(GpuDecoder* dec, double snr, double beta_lo, double beta_hi, double rate, uint64_t seed,
                              int64_t first_frame, int32_t n_frames, bool all_zero, float* d_llr, uint32_t* d_syndrome,
                              uint32_t* d_x_packed, void* stream) {
  dec->sample_device(snr, beta_lo, beta_hi, rate, seed, first_frame, n_frames, all_zero, d_llr, d_syndrome, d_x_packed,
                     static_cast<cudaStream_t>(stream));
}
void gpu_stage_inputs(GpuDecoder* dec, int32_t batch, const float* llr_host, const uint32_t* syn_host) {
  dec->stage_inputs(batch, llr_host, syn_host);
}
void gpu_stream_open(GpuDecoder* dec, const DecodeParams& p, bool packed, bool want_bits, bool want_post,
                     bool want_q, int32_t ring_frames) {
  dec->stream_open(p, packed, want_bits, want_post, want_q, ring_frames);
}
int64_t gpu_stream_submit(GpuDecoder* dec, int32_t n, const float* llr, const uint32_t* syn, const StreamOutputs& o) {
  return dec->stream_submit(n, llr, syn, o);
}
bool gpu_stream_query(GpuDecoder* dec, int64_t ticket) { return dec->stream_query(ticket); }
void gpu_stream_wait(GpuDecoder* dec, int64_t ticket) { dec->stream_wait(ticket); }
void gpu_stream_close(GpuDecoder* dec) { dec->stream_close(); }
void gpu_stream_timer_reset(GpuDecoder* dec) { dec->stream_timer_reset(); }
double gpu_stream_device_ms(GpuDecoder* dec) { return dec->stream_device_ms(); }
void gpu_set_profiling(GpuDecoder* dec, bool enable) { dec->profiling = enable; }
void gpu_profile(const GpuDecoder* dec, int kernel, double* total_ms, int64_t* launches, double* frame_iterations) {
  if (kernel < 0 || kernel >= kNumKernels) throw ValidationError("profile: kernel id out of range");
  if (total_ms) *total_ms = dec->prof_ms[kernel];
  if (launches) *launches = dec->prof_launches[kernel];
  if (frame_iterations) *frame_iterations = dec->prof_frame_iters;
}
void gpu_reset_profile(GpuDecoder* dec) {
  std::fill(std::begin(dec->prof_ms), std::end(dec->prof_ms), 0.0);
  std::fill(std::begin(dec->prof_launches), std::end(dec->prof_launches), 0);
  dec->prof_frame_iters = 0.0;
  dec->launches = 0;
}
int64_t gpu_launch_count(const GpuDecoder* dec) { return dec->launches; }

}  // namespace bpdec

#ifdef BPDEC_GUARD
// Guard-build self-test (not in include/bpdec.h; tests/test_guard_build.py):
// 0 when (a) fresh allocations read as poison, (b) a one-element write past
// the end of an allocation is reported by dev_verify, and (c) an in-bounds
// write is not.
namespace {
__global__ void k_guard_probe(uint32_t* p, int n, int write_at, uint32_t* first) {
  if (threadIdx.x == 0) {
    *first = p[0];
    if (write_at >= 0) p[write_at] = 7u;
    (void)n;
  }
}
}  // namespace
extern "C" int bpdec_guard_selftest() {
  using namespace bpdec;
  void *a = nullptr, *r = nullptr;
  if (dev_malloc(&a, 1000 * sizeof(uint32_t)) != cudaSuccess) return 1;
  if (cudaMalloc(&r, sizeof(uint32_t)) != cudaSuccess) return 1;
  uint32_t first = 0;
  int rc = 0;
  k_guard_probe<<<1, 32>>>(static_cast<uint32_t*>(a), 1000, 999, static_cast<uint32_t*>(r));  // in bounds
  cudaMemcpy(&first, r, sizeof(first), cudaMemcpyDeviceToHost);
  if (first != 0xFFFFFFFFu) rc |= 2;  // poison
  if (dev_verify(nullptr) != cudaSuccess) rc |= 4;  // false positive
  k_guard_probe<<<1, 32>>>(static_cast<uint32_t*>(a), 1000, 1000, static_cast<uint32_t*>(r));  // one past the end
  if (dev_verify(nullptr) == cudaSuccess) rc |= 8;  // missed
  cudaFree(r);
  dev_free(a);
  return rc;
}
#endif
