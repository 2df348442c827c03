/* TEST INFRASTRUCTURE — CPU oracle interface (see oracle.c). */
#ifndef BPDEC_ORACLE_H_
#define BPDEC_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_REF_DOUBLE = 0, ORC_PHI_FLOAT = 1, ORC_T_FLOAT = 2 };
enum { ORC_Q_RAW = 0, ORC_Q_ABS = 1 };

typedef struct {
  int32_t d_max;
  int32_t use_pce;
  int32_t use_vnr;
  int32_t q_mode;
  double msg_clamp;
} orc_config;

/* returns 0 ok, 3 validation error (decoder.cpp:56-64), 1 bad variant */
int orc_decode(int n_vars, int n_checks, const int* check_ptr, const int* check_vars, const double* llr,
               const uint32_t* syndrome, const orc_config* cfg, int variant, uint8_t* bits, int32_t* iterations,
               int32_t* reason, double* posteriors, double* q_trace);

double orc_snr_for_beta(double beta, double rate);
double orc_noise_normal(uint64_t seed, uint64_t stream, uint64_t i);
int orc_message_bit(uint64_t seed, uint64_t frame, uint64_t i);
void orc_sample_frame(int n, double snr, uint64_t seed, uint64_t frame, int all_zero, float* llr, uint8_t* x);

#ifdef __cplusplus
}
#endif

#endif
