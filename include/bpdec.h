/*
 * bpdec.h — C ABI of the B200-native batched LDPC belief-propagation decoder.
 *
 * This is the drop-in boundary for the reconciliation hot path of
 * arXiv 2507.03509 (reference: /root/reference/proj, library `etdec_core`).
 * Every entry point below names the reference interface it replaces
 * (file:line under proj/core/).  The reference exposes a C++ API only; a
 * C++ caller keeps that API through include/bpdec/etdec_compat.hpp, other
 * callers (ctypes, cgo, JNI) bind these symbols directly.
 *
 * Conventions
 *  - Plain pointers and sizes only; no exceptions cross the ABI.
 *  - Every function returning int returns a bpdec_status; on failure a
 *    thread-local message is available from bpdec_last_error().
 *  - Status codes 1/2/3 are the reference's exception classes
 *    (include/etdec/errors.hpp:8-24: ConfigError / IoError / ValidationError,
 *    CLI exit codes 1/2/3); 4+ are device errors the CPU reference cannot have.
 *  - There is no CPU fallback: decoder creation fails with BPDEC_ERR_CUDA when
 *    no sm_100 device is present.
 */
#ifndef BPDEC_H_
#define BPDEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BPDEC_ABI_VERSION 1

typedef enum {
  BPDEC_OK = 0,
  BPDEC_ERR_CONFIG = 1,     /* ≙ etdec::ConfigError     errors.hpp:9-12  */
  BPDEC_ERR_IO = 2,         /* ≙ etdec::IoError         errors.hpp:15-18 */
  BPDEC_ERR_VALIDATION = 3, /* ≙ etdec::ValidationError errors.hpp:21-24 */
  BPDEC_ERR_CUDA = 4,
  BPDEC_ERR_OOM = 5,
  BPDEC_ERR_INTERNAL = 6
} bpdec_status;

/* ≙ etdec::StopReason (decoder.hpp:13-17), same numeric order. */
typedef enum {
  BPDEC_STOP_SYNDROME = 0, /* kSyndromeSatisfied: PCE-ET fired          */
  BPDEC_STOP_VNR = 1,      /* kVnrDrop: q^(k) < q^(k-1), k >= 2 (VNR-ET) */
  BPDEC_STOP_MAX_ITER = 2  /* kMaxIterations: d_max reached             */
} bpdec_stop_reason;

/* VNR statistic over the degree>=2 variables (decoder.cpp:32-36).
 * RAW is the reference formula q = sum posterior (correct in the
 * all-zero-equivalent frame, i.e. syndrome == NULL / all zero).  ABS is the
 * x-free reliability q = sum |posterior| for true syndrome-mode decoding,
 * where the transmitted word is unknown to the decoder. */
typedef enum { BPDEC_Q_RAW = 0, BPDEC_Q_ABS = 1 } bpdec_q_mode;

/* ≙ etdec::DecodeConfig (decoder.hpp:21-26) plus the q-mode switch. */
typedef struct {
  int32_t d_max;     /* iteration budget, > 0                 (default 100)  */
  int32_t use_pce;   /* syndrome check every iteration        (default 1)    */
  int32_t use_vnr;   /* q-statistic drop check, from k = 2     (default 0)    */
  int32_t q_mode;    /* bpdec_q_mode                          (default RAW)  */
  double msg_clamp;  /* message magnitude bound, > 0          (default 30.0) */
} bpdec_config;

/* Output flags for bpdec_decode_batch. */
#define BPDEC_BITS_PACKED 0x1u /* bits_out is uint32 [batch][ceil(N/32)], LSB-first */

typedef struct bpdec_code bpdec_code;       /* immutable host Tanner graph      */
typedef struct bpdec_decoder bpdec_decoder; /* per-device workspace, one thread */

/* ----------------------------------------------------------------- misc -- */
int bpdec_abi_version(void);
const char* bpdec_last_error(void);
/* ≙ etdec::to_string(StopReason) decoder.cpp:10-17 */
const char* bpdec_stop_reason_name(int32_t reason);

/* ----------------------------------------------------------- code model -- */
/* ≙ ParityCheckMatrix::from_check_lists (parity_check_matrix.hpp:16-17,
 * parity_check_matrix.cpp:10-62): check-major CSR, check_ptr[n_checks+1],
 * check_vars[check_ptr[n_checks]]; same validation (range, duplicates,
 * 0 < n_checks < n_vars) and the same ValidationError status. */
int bpdec_code_from_csr(int32_t n_vars, int32_t n_checks, const int32_t* check_ptr,
                        const int32_t* check_vars, bpdec_code** out);
/* ≙ load_alist_file / save_alist_file (alist.hpp:21,24; alist.cpp:78-202). */
int bpdec_code_load_alist(const char* path, bpdec_code** out);
int bpdec_code_save_alist(const bpdec_code* code, const char* path);
/* ≙ lift_protograph (protograph.hpp:31, protograph.cpp:52-101); base is a
 * row-major [rows][cols] multiplicity matrix. */
int bpdec_code_lift_protograph(const int32_t* base, int32_t rows, int32_t cols, int32_t z,
                               uint64_t seed, bpdec_code** out);
/* BASELINE.json multi-edge-style construction (new; not in the reference):
 * N variables, M checks, the last round(f1*N) variables degree 1 on an
 * identity block over the last checks, the rest with degrees deg[i] in
 * proportions prob[i], sockets matched by a seeded permutation. */
int bpdec_code_generate_met(int32_t n_vars, int32_t n_checks, double frac_deg1,
                            int32_t n_classes, const int32_t* degrees, const double* probs,
                            uint64_t seed, bpdec_code** out);
/* Two-edge-type low-rate construction with a core code (new; SURVEY §8f#2
 * "a MET-style generator so FER < 1"): core variables 0..nc-1 (nc = N -
 * n_deg1) with type-1 degrees core_degrees[i] in proportions core_probs[i]
 * on the M - n_deg1 core checks; each of the n_deg1 extension checks holds
 * ext_degree type-2 edges to core variables (dealt evenly, seeded shuffle)
 * and one degree-1 variable (nc + j).  Rule in csrc/code.cpp. */
int bpdec_code_generate_met_core(int32_t n_vars, int32_t n_checks, int32_t n_deg1, int32_t n_classes,
                                 const int32_t* core_degrees, const double* core_probs, int32_t ext_degree,
                                 uint64_t seed, bpdec_code** out);
void bpdec_code_destroy(bpdec_code* code);
/* n_active = |{v : deg(v) >= 2}| (ActiveVarSet, parity_check_matrix.hpp:66-70) */
int bpdec_code_dims(const bpdec_code* code, int32_t* n_vars, int32_t* n_checks,
                    int64_t* n_edges, int32_t* n_active);
/* copies of the CSR (check_ptr[M+1], check_vars[E]); either may be NULL */
int bpdec_code_csr(const bpdec_code* code, int32_t* check_ptr, int32_t* check_vars);
/* ≙ active_var_set (parity_check_matrix.cpp:64-70): ascending, n_active entries */
int bpdec_code_active_vars(const bpdec_code* code, int32_t* members);
/* s = H x (packed LSB-first, ceil(M/32) words per frame) for n_frames frames */
int bpdec_code_syndrome(const bpdec_code* code, int32_t n_frames, const uint8_t* bits,
                        uint32_t* syndrome_out);
/* ≙ syndrome_check (decoder.hpp:39, decoder.cpp:19-30) generalised to a
 * target syndrome (NULL = all zero); *ok = 1 iff H bits == syndrome. */
int bpdec_syndrome_check(const bpdec_code* code, const uint8_t* bits,
                         const uint32_t* syndrome, int32_t* ok);

/* -------------------------------------------------------------- channel -- */
/* ≙ snr_for_beta (channel.hpp:24, channel.cpp:29-42): snr = 2^(2R/beta) - 1 */
int bpdec_snr_for_beta(double beta, double rate, double* snr);
/* Seeded syndrome-mode frames (BASELINE.json configs).  For global frame
 * index f = first_frame + b: x_i ~ Bern(1/2) from a counter hash keyed by
 * (seed, f, i); g_i = NoiseStream(seed, f).normal(i) (rng.hpp:85-99);
 * llr_i = float((2/sigma^2) * ((1 - 2 x_i) + sigma * g_i)), which at x = 0
 * is sample_block (channel.cpp:44-61) rounded to float; s = H x.
 * all_zero != 0 forces x = 0 (the reference's all-zero codeword).
 * Outputs: llr [n][N] float, x [n][N] u8 (may be NULL), syndrome
 * [n][ceil(M/32)] (may be NULL).  Host implementation, threaded. */
int bpdec_sample_frames(const bpdec_code* code, double snr, uint64_t seed, int64_t first_frame,
                        int32_t n_frames, int32_t all_zero, float* llr_out, uint8_t* x_out,
                        uint32_t* syndrome_out);

/* Same, with a per-frame efficiency beta_f ~ U[beta_lo, beta_hi] drawn from a
 * counter hash keyed by (seed, f) and snr_f = 2^(2R/beta_f) - 1 (BASELINE
 * config 5, mixed-SNR stream); snr_out [n] (may be NULL) receives snr_f. */
int bpdec_sample_frames_beta(const bpdec_code* code, double beta_lo, double beta_hi, uint64_t seed,
                             int64_t first_frame, int32_t n_frames, int32_t all_zero, float* llr_out,
                             uint8_t* x_out, uint32_t* syndrome_out, double* snr_out);

/* -------------------------------------------------------------- decoder -- */
/* ≙ BpDecoder::BpDecoder (decoder.hpp:57, decoder.cpp:38-48), batched: a
 * device replica of the code plus message state for max_slots frames in
 * flight (rounded up to a multiple of 32).  One decoder per host thread. */
int bpdec_decoder_create(const bpdec_code* code, int32_t device, int32_t max_slots,
                         bpdec_decoder** out);
void bpdec_decoder_destroy(bpdec_decoder* dec);
int bpdec_decoder_slots(const bpdec_decoder* dec, int32_t* slots);
/* Device bytes held by the decoder (code replica + message state). */
int bpdec_decoder_device_bytes(const bpdec_decoder* dec, int64_t* bytes);

/* ≙ BpDecoder::decode (decoder.hpp:64-65, decoder.cpp:50-129), batched over
 * `batch` independent frames and syndrome-aware.
 *   llr        [batch][N] float32 channel LLRs (host or device pointer)
 *   syndrome   [batch][ceil(M/32)] target syndrome, LSB-first; NULL = 0
 *   cfg        decode configuration (validated like decoder.cpp:56-64)
 *   flags      BPDEC_BITS_PACKED or 0
 *   bits_out   [batch][N] u8 hard decisions (1 iff posterior < 0), or
 *              packed words with BPDEC_BITS_PACKED; may be NULL
 *   iterations_out [batch] int32; reason_out [batch] u8 (bpdec_stop_reason)
 *   posteriors_out [batch][N] float (stop-iteration posteriors) or NULL
 *   q_trace_out    [batch][d_max] double, q^(1..k), rest NaN; or NULL
 *   stream     cudaStream_t to order the work on (NULL = decoder's own)
 * Pointers may be host or device memory (detected per pointer).  The call
 * returns when every frame has terminated and outputs are written.  Frames
 * beyond the slot count stream through the slots as earlier frames stop. */
int bpdec_decode_batch(bpdec_decoder* dec, int32_t batch, const float* llr,
                       const uint32_t* syndrome, const bpdec_config* cfg, uint32_t flags,
                       void* bits_out, int32_t* iterations_out, uint8_t* reason_out,
                       float* posteriors_out, double* q_trace_out, void* stream);

/* ≙ BpDecoder::decode with an IterationObserver (decoder.hpp:53-55,
 * decoder.cpp:107-112): bpdec_decode_batch plus per-iteration traces for
 * replaying the observer's (iteration, posteriors, syndrome_ok, q) calls.
 *   syndrome_ok_trace_out [batch][d_max] u8: 1 iff H bits == s after
 *       iteration k (computed every iteration, PCE on or off, like
 *       decoder.cpp:111); 0xff past the stop iteration; or NULL
 *   posterior_trace_out [batch][d_max][N] float: the posteriors after every
 *       iteration (NaN past the stop); or NULL.  Sized for small batches.
 * q is q_trace_out.  Other arguments as bpdec_decode_batch. */
int bpdec_decode_batch_traced(bpdec_decoder* dec, int32_t batch, const float* llr,
                              const uint32_t* syndrome, const bpdec_config* cfg, uint32_t flags,
                              void* bits_out, int32_t* iterations_out, uint8_t* reason_out,
                              float* posteriors_out, double* q_trace_out,
                              uint8_t* syndrome_ok_trace_out, float* posterior_trace_out,
                              void* stream);

/* Pipelined host input: starts the host->device copy of a batch (pinned host
 * memory for full overlap) on the decoder's copy stream and returns at once.
 * A later bpdec_decode_batch with the same llr / syndrome pointers and batch
 * decodes from the staged copy, so staging batch k+1 before decoding batch k
 * overlaps its upload with the decode.  Two staging slots; staging a third
 * batch replaces the older unconsumed one (whose decode then copies again).
 * The match is by pointer: the staged bytes are what the buffers held when
 * this call was made, so the host buffers must not be rewritten between this
 * call and the decode that consumes them (refill a buffer only after its
 * decode returns, e.g. alternate two buffer sets).  No
 * reference counterpart (the reference decodes host spans on the CPU). */
int bpdec_decoder_stage_inputs(bpdec_decoder* dec, int32_t batch, const float* llr_host,
                               const uint32_t* syndrome_host);

/* ---------------------------------------------------------- stream mode -- */
/* Batches submitted back to back decode as ONE continuous frame stream
 * through the decoder's slots: the lanes a batch's slow frames leave free
 * are refilled with the next batch's frames in the same step, and a batch's
 * upload overlaps the decode of the earlier ones.  A worker thread owned by
 * the decoder launches the steps; outputs of a batch are copied to the
 * caller's buffers as soon as its last frame stopped.  Per-frame results are
 * those of bpdec_decode_batch on the same frames (no dependence on slot,
 * order or neighbours).  No reference counterpart: this replaces the
 * per-block loop of run_trials (channel.cpp:90-148) for a caller that keeps
 * the GPU busy across batches.
 *   open:   cfg / flags (BPDEC_BITS_PACKED) / which outputs exist are fixed
 *           for the stream; ring_frames = frames whose inputs and outputs can
 *           be in flight (0 = 4 x slots; a batch must fit).  While open, the
 *           decoder accepts only stream calls.
 *   submit: inputs host (pinned for overlap) or device pointers, read until
 *           the batch completes; outputs host or device pointers (pinned host
 *           memory keeps the worker from blocking on the copy), written when
 *           the batch completes.  Blocks while the ring or the batch slots
 *           (32 in flight) are full.  *ticket_out identifies the batch.
 *   wait:   blocks until the batch's outputs are written; returns its status
 *           (BPDEC_ERR_VALIDATION for a non-finite LLR in that batch).
 *   query:  *done = 1 once wait would not block.
 *   close:  waits for every submitted batch, frees the rings. */
int bpdec_stream_open(bpdec_decoder* dec, const bpdec_config* cfg, uint32_t flags, int32_t ring_frames,
                      int32_t want_bits, int32_t want_posteriors, int32_t want_q_trace);
int bpdec_stream_submit(bpdec_decoder* dec, int32_t batch, const float* llr, const uint32_t* syndrome,
                        void* bits_out, int32_t* iterations_out, uint8_t* reason_out, float* posteriors_out,
                        double* q_trace_out, int64_t* ticket_out);
int bpdec_stream_wait(bpdec_decoder* dec, int64_t ticket);
int bpdec_stream_query(bpdec_decoder* dec, int64_t ticket, int32_t* done);
int bpdec_stream_close(bpdec_decoder* dec);
/* Device timer of the stream (for throughput measurement): reset (only
 * while no batch is in flight) arms it; the first step launched afterwards
 * records the start on the decoder's stream, every batch's output copy the
 * end.  device_ms = the time between them, CUDA events (waits for the last
 * copy). */
int bpdec_stream_timer_reset(bpdec_decoder* dec);
int bpdec_stream_device_ms(bpdec_decoder* dec, double* ms);

/* ------------------------------------------------------------ multi-GPU -- */
/* Frame-sharded decoding over several GPUs of one host (the
 * reference's strided worker pool, channel.cpp:98-122): one decoder per
 * entry of devices[] (an entry may repeat a device), each fed by its own
 * host thread from a shared queue of chunk_frames-frame chunks (dynamic, so
 * devices that finish early take more; 0 = auto), no collective, per-frame
 * outputs written into the caller's buffers at their frame index.  Results
 * are identical for any device list and chunk size (per-frame
 * independence; the reference's worker-count invariance, channel.hpp:66-71).
 * frames_per_decoder_out [n_devices] (may be NULL) receives how many frames
 * each decoder took in this call. */
typedef struct bpdec_multi bpdec_multi;
int bpdec_multi_create(const bpdec_code* code, const int32_t* devices, int32_t n_devices,
                       int32_t slots_per_decoder, bpdec_multi** out);
void bpdec_multi_destroy(bpdec_multi* multi);
int bpdec_multi_count(const bpdec_multi* multi, int32_t* n_decoders);
int bpdec_multi_decode_batch(bpdec_multi* multi, int32_t batch, const float* llr,
                             const uint32_t* syndrome, const bpdec_config* cfg, uint32_t flags,
                             void* bits_out, int32_t* iterations_out, uint8_t* reason_out,
                             float* posteriors_out, double* q_trace_out, int32_t chunk_frames,
                             int64_t* frames_per_decoder_out);

/* Device-side frame generator for resident-input benchmarks: same draws as
 * bpdec_sample_frames, written to DEVICE buffers (llr [n][N], syndrome
 * [n][ceil(M/32)], x packed [n][ceil(N/32)]; x/syndrome may be NULL). */
int bpdec_decoder_sample_frames_device(bpdec_decoder* dec, double snr, uint64_t seed,
                                       int64_t first_frame, int32_t n_frames, int32_t all_zero,
                                       float* d_llr, uint32_t* d_syndrome, uint32_t* d_x_packed,
                                       void* stream);

/* Device-side mixed-SNR generator (draws of bpdec_sample_frames_beta). */
int bpdec_decoder_sample_frames_beta_device(bpdec_decoder* dec, double beta_lo, double beta_hi, uint64_t seed,
                                            int64_t first_frame, int32_t n_frames, int32_t all_zero,
                                            float* d_llr, uint32_t* d_syndrome, uint32_t* d_x_packed,
                                            void* stream);

/* ------------------------------------------------- Monte-Carlo harness -- */
/* ≙ etdec::StopRule (channel.hpp:42-45) */
typedef struct {
  int64_t min_frame_errors; /* stop at this many frame errors (0 disables) */
  int64_t max_frames;       /* or at this many frames (0 = uncapped)       */
} bpdec_stop_rule;

/* ≙ etdec::TrialStats (channel.hpp:47-61); the iteration histogram is
 * returned separately ([d_max+1] counts). */
typedef struct {
  int64_t frames, frame_errors, undetected_errors;
  double fer, fer_ci_low, fer_ci_high, d_bar;
  int64_t iteration_sum;
  int64_t stops_syndrome, stops_vnr, stops_max_iter;
  int32_t hit_max_frames;
  int32_t _pad;
} bpdec_trial_stats;

/* ≙ apply_puncture (puncture.hpp:26, puncture.cpp:16-48): positions
 * [round(N - (N-M)/target)] ascending (caller buffer of N entries);
 * *count and *effective_rate returned. */
int bpdec_code_apply_puncture(const bpdec_code* code, double target_rate, uint64_t seed,
                              int32_t* punctured_out, int32_t* count, double* effective_rate);
/* ≙ wilson_interval (channel.hpp:64, channel.cpp:63-72) */
int bpdec_wilson_interval(int64_t k, int64_t n, double* lo, double* hi);
/* ≙ run_trials (channel.hpp:72-74, channel.cpp:74-156) on the GPU: trials
 * 0,1,2,... of the all-zero codeword at `snr` (sample_block draws, rounded to
 * float32), punctured positions at LLR 0, decoded `block` at a time; the stop
 * rule is applied to the exact trial-index prefix, so results do not depend
 * on `block` (the reference's worker-count invariance).  A frame error is
 * bits != 0 or reason != syndrome (channel.cpp:109-112). */
int bpdec_run_trials(bpdec_decoder* dec, double snr, const int32_t* punctured, int32_t n_punctured,
                     const bpdec_config* cfg, const bpdec_stop_rule* stop, uint64_t seed, int32_t block,
                     bpdec_trial_stats* stats_out, int64_t* histogram_out);

/* Per-kernel timing of the most recent bpdec_decode_batch calls (CUDA events
 * on the launching stream).  Enable before decoding; kernel ids:
 * 0 check-node, 1 variable-node, 2 decide (syndrome + q^(k) + stop decision),
 * 3 unused (termination is part of 2), 4 turnover (outputs of stopped frames +
 * loading of queued frames), 5 tail compaction, 6 output snapshot (eager host
 * copies), 7 posterior trace (bpdec_decode_batch_traced). */
int bpdec_decoder_set_profiling(bpdec_decoder* dec, int32_t enable);
int bpdec_decoder_profile(const bpdec_decoder* dec, int32_t kernel, double* total_ms,
                          int64_t* launches, double* frame_iterations);
int bpdec_decoder_reset_profile(bpdec_decoder* dec);
/* Number of kernels launched by this decoder since creation / last reset. */
int bpdec_decoder_launch_count(const bpdec_decoder* dec, int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* BPDEC_H_ */
