/* TEST INFRASTRUCTURE ONLY — CPU checker for the MPS sampling sweep (see mpsamp_oracle.c). */
#ifndef MPSAMP_ORACLE_H
#define MPSAMP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_F64 = 0, ORC_F32 = 1, ORC_TF32 = 2, ORC_F16 = 3 };                /* precision.hpp:15 */
enum { ORC_SCALE_NONE = 0, ORC_SCALE_GLOBAL = 1, ORC_SCALE_PER_SAMPLE = 2 }; /* precision.hpp:17 */
enum { ORC_ERR_NUMERIC = 3 };
#define ORC_DEAD 0xFF                                 /* sampler.hpp:17 */
#define ORC_MEASURE_STREAM 0x6d656173ull              /* rng.hpp:19 */

uint64_t orc_mix64(uint64_t z);
uint64_t orc_key(uint64_t seed, uint64_t stream, uint64_t sample, uint64_t site);
double orc_to_unit(uint64_t bits);
double orc_uniform(uint64_t seed, uint64_t stream, uint64_t sample, uint64_t site);
double orc_round_to_grid(double x, int mant_bits, int emin_normal, int emax);
double orc_round_scalar(double x, int precision);
int orc_contract_site(const double* env, size_t count, size_t chil, const double* gamma,
                      size_t chir, size_t d, int compute, double* out);
void orc_measure(const double* temp, size_t count, size_t chi, size_t d, const double* lambda,
                 const double* draws, uint8_t* alive, uint8_t* outcomes, double* env_out,
                 double* weights_out);
void orc_scale_rows(double* env, size_t count, size_t row, int mode, uint8_t* alive);
int orc_sample_range(size_t m, size_t d, const size_t* bonds, const double* const* gamma,
                     const double* const* lambda, uint64_t first, size_t count, uint64_t seed,
                     int compute, int scaling, const uint8_t* forced, uint8_t* rows,
                     double* marg, uint64_t* contraction_macs);
int orc_sample_range_displaced(size_t m, size_t d, const size_t* bonds, const double* const* gamma,
                               const double* const* lambda, uint64_t first, size_t count, uint64_t seed,
                               int compute, int scaling, const uint8_t* forced, const double* mu,
                               uint8_t* rows, double* marg, uint64_t* contraction_macs);
void orc_displacement(double mu_re, double mu_im, size_t n, double* out);
void orc_capped_bond_dims(size_t m, size_t d, size_t chi_max, size_t* out);
uint64_t orc_fnv1a(const uint8_t* p, size_t n);
uint64_t orc_site_step(const double* gamma, size_t chil, size_t chir, size_t d, const double* lambda,
                       size_t count, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
