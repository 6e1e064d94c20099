/* qsim_oracle.h -- CPU restatement of the reference's state-vector hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the checker;
 * the product (libqsb.so) never links or calls it.
 *
 * Each function restates the reference algorithm it cites (paths relative to
 * /root/reference/proj/include/qforge/).  The restatement is pinned against
 * golden vectors emitted by the reference itself (oracle/_ref/ref_driver, see
 * tests/golden/README.md).
 *
 * The gate record layout is identical to qs_gate in include/qsb.h so tests can
 * hand the same arrays to both sides.
 */
#ifndef QSIM_ORACLE_H_
#define QSIM_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { QO_I = 0, QO_X, QO_Y, QO_Z, QO_H, QO_S, QO_T, QO_RX, QO_RY, QO_RZ, QO_U3,
       QO_CNOT, QO_CZ, QO_SWAP, QO_TOFFOLI, QO_CUSTOM };

typedef struct qo_gate {
  int32_t kind;
  int32_t dagger;
  uint32_t num_targets;
  uint32_t num_controls;
  uint32_t targets[8];
  uint32_t controls[40];
  double params[3];
  const double* matrix;
} qo_gate;

/* rng.hpp:9-46 */
uint64_t qo_splitmix64(uint64_t x);
typedef struct qo_rng { uint64_t mt[312]; int idx; } qo_rng;
void qo_rng_seed(qo_rng* r, uint64_t seed);
void qo_rng_derive(qo_rng* r, uint64_t seed, uint64_t index);
uint64_t qo_rng_next(qo_rng* r);
double qo_rng_uniform(qo_rng* r);
uint64_t qo_rng_below(qo_rng* r, uint64_t k);
/* fills out[0..count) with Rng(seed).uniform() draws */
void qo_uniforms(uint64_t seed, uint64_t count, double* out);

/* gates.hpp:15-97: matrix on the targets (no extra controls), dagger applied.
 * out: (2^nt)^2 complex row-major interleaved.  Returns dimension or <0. */
int qo_base_matrix(const qo_gate* g, double* out);

/* statevector.hpp kernels; amps is 2^n interleaved complex. */
void qo_init_zero(double* amps, uint32_t n);
void qo_apply_1q(double* amps, uint32_t n, uint32_t q, const double m[8], const uint32_t* ctrls, uint32_t nc);
void qo_apply_diag(double* amps, uint32_t n, uint32_t q, const double d[4], const uint32_t* ctrls, uint32_t nc);
void qo_apply_flip(double* amps, uint32_t n, uint32_t q, const uint32_t* ctrls, uint32_t nc);
void qo_apply_swap2(double* amps, uint32_t n, uint32_t a, uint32_t b, const uint32_t* ctrls, uint32_t nc);
int qo_apply_matrix(double* amps, uint32_t n, const uint32_t* targets, uint32_t k, const double* m,
                    const uint32_t* ctrls, uint32_t nc);
/* StateVector::apply_gate (statevector.hpp:469-538). 0 ok, -1 validation */
int qo_apply_gate(double* amps, uint32_t n, const qo_gate* g);
int qo_apply_gates(double* amps, uint32_t n, const qo_gate* g, uint64_t count);

/* reductions */
double qo_norm2(const double* amps, uint32_t n);                  /* :158-162 chunked_sum */
double qo_prob_one(const double* amps, uint32_t n, uint32_t q);   /* :181-186 */
void qo_probs(const double* amps, uint32_t n, const uint32_t* qubits, uint32_t m, double* out); /* :190-208 */
void qo_probs_full(const double* amps, uint32_t n, double* out);  /* :210-215 */
int qo_collapse(double* amps, uint32_t n, uint32_t q, int outcome, double prob); /* :228-247 */
int qo_measure_collapse(double* amps, uint32_t n, uint32_t q, double u);        /* :219-225 */
double qo_checksum(const double* amps, uint32_t n);               /* bench.hpp:141-148 */

/* BasisSampler (statevector.hpp:542-570): cum has 2^n doubles. returns total */
double qo_sampler_build(const double* amps, uint32_t n, double* cum);
uint64_t qo_sampler_draw(const double* cum, uint64_t size, double total, double u);
/* run() trailing-measure sampling (simulator.hpp:164-178): basis index per shot */
void qo_sample_seeded(const double* amps, uint32_t n, uint64_t seed, uint64_t shots, uint64_t* out);

/* expectation (variational.hpp:19-54): letters[t*n + q] in IXYZ, coeff real.
 * Returns sum_t coeff_t <psi|P_t|psi> (real part); imag in *imag_out. */
double qo_expectation(const double* amps, uint32_t n, const char* letters, const double* coeffs,
                      uint32_t nterms, double* imag_out);

/* Circuit generators (gate count returned; out may be NULL to query size).
 * gen_random_circuit: bench.hpp:72-94.  The others are defined in
 * oracle/circuits.hpp (not in the reference) and mirrored by the product. */
uint64_t qo_gen_random_circuit(uint32_t n, uint32_t d, uint64_t seed, qo_gate* out);
uint64_t qo_gen_ghz(uint32_t n, qo_gate* out);
uint64_t qo_gen_qft(uint32_t n, uint64_t input_basis, qo_gate* out);
uint64_t qo_gen_hea(uint32_t n, uint32_t layers, uint64_t seed, qo_gate* out);

#ifdef __cplusplus
}
#endif

#endif
