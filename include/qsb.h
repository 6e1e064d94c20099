/* qsb.h -- C ABI of the B200 state-vector backend (libqsb.so).
 *
 * This is the drop-in boundary for the reference's simulation hot path.  The
 * reference (qforge, header-only C++20 under /root/reference/proj/include)
 * has no plugin or FFI layer: its seam is the StateVector member API that
 * every executor calls.  Each entry point below replaces one member of that
 * seam; the file:line in brackets is the reference interface it replaces
 * (paths relative to /root/reference/proj/include/qforge/).  The C++ facade
 * under paper_2212_14201_b200/include/qforge/ re-exposes the reference's own
 * types (Program, Gate, StateVector, run, expectation, ...) on top of this
 * ABI, and INTEGRATION.md shows the bindings a maintainer would add.
 *
 * Conventions (identical to the reference):
 *   - amplitude index i has bit q = qubit q (qubit 0 is the least significant
 *     bit); amplitudes are complex128, interleaved (re, im)  [statevector.hpp:134-156]
 *   - operand lists are most-significant-first; for a gate, the full operand
 *     list is controls ++ targets and CNOT/CZ/TOFFOLI carry their defining
 *     control(s) inside targets                           [circuit.hpp:108-114]
 *   - matrices are row-major, interleaved (re, im), 2^k x 2^k, with local bit
 *     b of the row/column index living at targets[k-1-b]   [statevector.hpp:385-390]
 *
 * Errors: every function returns QS_OK (0) or a negative status; no C++
 * exception crosses the ABI.  qs_last_error() returns the message of the last
 * failure on the calling thread.  QS_ERR_VALIDATION maps to
 * qforge::ValidationError, QS_ERR_RUNTIME to qforge::Error   [error.hpp:10-20].
 *
 * Threading: a state handle is owned by one thread at a time;
 * each handle has one CUDA stream on its device.  Host buffers belong to the
 * caller and every call is synchronous with respect to them on return.
 */
#ifndef QSB_H_
#define QSB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSB_ABI_VERSION 1

/* status codes */
#define QS_OK 0
#define QS_ERR_VALIDATION -1 /* bad operands, sizes, non-unitary matrix   */
#define QS_ERR_RUNTIME -2    /* e.g. collapse onto a zero-probability outcome */
#define QS_ERR_CUDA -3       /* CUDA / NCCL failure                         */
#define QS_ERR_MEMORY -4     /* allocation failure                          */
#define QS_ERR_UNSUPPORTED -5

/* Gate kinds, numbered exactly as qforge::GateKind          [circuit.hpp:22-27] */
enum qs_gate_kind {
  QS_I = 0, QS_X, QS_Y, QS_Z, QS_H, QS_S, QS_T,
  QS_RX, QS_RY, QS_RZ, QS_U3,
  QS_CNOT, QS_CZ, QS_SWAP, QS_TOFFOLI,
  QS_CUSTOM
};

#define QS_MAX_TARGETS 8
#define QS_MAX_CONTROLS 40

/* One gate application, the flat equivalent of qforge::Gate [circuit.hpp:115-139]. */
typedef struct qs_gate {
  int32_t kind;          /* enum qs_gate_kind                                  */
  int32_t dagger;        /* Gate::dagger                                       */
  uint32_t num_targets;  /* Gate::targets.size()                               */
  uint32_t num_controls; /* Gate::controls.size() (extra controls only)        */
  uint32_t targets[QS_MAX_TARGETS];   /* most significant first              */
  uint32_t controls[QS_MAX_CONTROLS];
  double params[3];      /* RX/RY/RZ: params[0]; U3: theta, phi, lambda        */
  const double* matrix;  /* Custom only: 2^nt x 2^nt row-major interleaved    */
} qs_gate;

typedef struct qs_state* qs_state_t;

/* --- library -------------------------------------------------------------- */
const char* qs_last_error(void);
int qs_abi_version(void);
/* Number of this library's own kernel launches since load (bench evidence). */
uint64_t qs_kernel_launches(void);
/* Tile-kernel JIT counters since load: NVRTC builds, in-process cache hits,
 * cubins loaded from the on-disk cache ($QSB_JIT_CACHE, default
 * ~/.cache/qsb-jit).  Any pointer may be NULL. */
int qs_jit_stats(uint64_t* nvrtc_builds, uint64_t* memory_hits, uint64_t* disk_hits);

/* --- lifecycle ------------------------------------------------------------- */
/* StateVector(n): |0...0> on `device`.  max_qubits bounds n (the reference caps
 * at 30 [statevector.hpp:137-138]; pass 0 for that default).                   */
int qs_create(uint32_t num_qubits, int device, uint32_t max_qubits, qs_state_t* out);
int qs_destroy(qs_state_t s);
/* StateVector copy constructor (device-to-device)     [statevector.hpp:134] */
int qs_clone(qs_state_t src, qs_state_t* out);
uint32_t qs_num_qubits(qs_state_t s);
int qs_device(qs_state_t s);
/* Raw device pointer of the amplitudes (for zero-copy interop, e.g. torch).
 * Plans that end in a qubit permutation (relabelled SWAPs) write out of place
 * into a second buffer of the same size and swap: query the pointer again
 * after executing a plan.                                                     */
void* qs_device_ptr(qs_state_t s);
/* Resets to |0...0>. */
int qs_reset(qs_state_t s);
/* Resets to the basis state |index>. */
int qs_set_basis_state(qs_state_t s, uint64_t index);
int qs_sync(qs_state_t s);
/* The state's CUDA stream (cudaStream_t) for event timing / interop.         */
void* qs_stream(qs_state_t s);

/* --- amplitude I/O (logical index order) -----------------------------------
 * from_amplitudes / amplitudes()           [statevector.hpp:143-156]         */
int qs_set_amplitudes(qs_state_t s, const double* interleaved, uint64_t offset, uint64_t count);
int qs_get_amplitudes(qs_state_t s, double* interleaved, uint64_t offset, uint64_t count);

/* --- single gates: one HBM pass each (the reference's per-gate kernels) ----- */
/* StateVector::apply_gate: validation, dagger, named-matrix dispatch  [statevector.hpp:469-538] */
int qs_apply_gate(qs_state_t s, const qs_gate* g);
/* apply_1q: 2x2 matrix m (row-major interleaved) on target    [statevector.hpp:268-290] */
int qs_apply_1q(qs_state_t s, uint32_t target, const double m[8], const uint32_t* controls, uint32_t nc);
/* apply_diag_1q: diag(d0, d1)                                  [statevector.hpp:292-319] */
int qs_apply_diag(qs_state_t s, uint32_t target, const double d[4], const uint32_t* controls, uint32_t nc);
/* apply_flip: X / CNOT / TOFFOLI                               [statevector.hpp:321-339] */
int qs_apply_flip(qs_state_t s, uint32_t target, const uint32_t* controls, uint32_t nc);
/* apply_swap2                                                  [statevector.hpp:341-361] */
int qs_apply_swap(qs_state_t s, uint32_t a, uint32_t b, const uint32_t* controls, uint32_t nc);
/* apply_matrix: dense 2^k x 2^k on targets (msb first), need not be unitary
 *                                                              [statevector.hpp:363-467] */
int qs_apply_matrix(qs_state_t s, const uint32_t* targets, uint32_t k, const double* m,
                    const uint32_t* controls, uint32_t nc);

/* --- batched circuits: the fused hot path ------------------------------------
 * Applies gates[0..n) in order.  The planner groups them into shared-memory
 * tile passes (many gates per HBM pass); results equal sequential apply_gate
 * within rounding.  Replaces the run() gate loop + fuse_circuit
 *                               [simulator.hpp:147-159, fusion.hpp:108-133]  */
#define QS_PLAN_DEFAULT 0u
#define QS_PLAN_UNFUSED 1u    /* one kernel per gate (reference execution order) */
#define QS_PLAN_DENSE_FUSION 2u /* reference fuse_circuit blocks, dense k<=5 kernels */
#define QS_PLAN_TILED 3u      /* shared-memory tile passes (default)            */
int qs_apply_circuit(qs_state_t s, const qs_gate* gates, uint64_t n, uint32_t plan,
                     uint32_t max_fused_qubits);

/* run() semantics: reset to the basis state |basis> and apply gates[0..n)
 * (StateVector(n) + the gate loop, simulator.hpp:147-159).  The reset is
 * fused into the first tile pass, which then writes the state without reading
 * it.                                                                          */
int qs_run_circuit(qs_state_t s, uint64_t basis, const qs_gate* gates, uint64_t n, uint32_t plan,
                   uint32_t max_fused_qubits);
/* qs_run_circuit + probability_checksum of the result (bench.hpp:141-148,
 * run_bench's checksum): the last tile pass sums |a_i|^2 (i+1) over what it
 * stores (one partial per CTA, fixed order), so no extra read of the state.  */
int qs_run_circuit_checksum(qs_state_t s, uint64_t basis, const qs_gate* gates, uint64_t n, uint32_t plan,
                            uint32_t max_fused_qubits, double* checksum);

/* Compiled circuit handle: plan once, run many times (bench / parameter sweeps). */
typedef struct qs_plan* qs_plan_t;
int qs_plan_create(uint32_t num_qubits, const qs_gate* gates, uint64_t n, uint32_t plan,
                   uint32_t max_fused_qubits, qs_plan_t* out);
int qs_plan_destroy(qs_plan_t p);
int qs_plan_execute(qs_state_t s, qs_plan_t p);
/* Enqueue without waiting (the state's stream is returned by qs_stream).    */
int qs_plan_enqueue(qs_state_t s, qs_plan_t p);
/* Execute with a CUDA event around every step; step_ms[i] receives the device
 * time of step i (qs_plan_stats' launch count entries).                       */
int qs_plan_execute_timed(qs_state_t s, qs_plan_t p, float* step_ms);
/* Resets the state to the basis state |basis> and runs the plan (run() from
 * |0...0>, simulator.hpp:147-159): when the plan starts with a tile pass the
 * reset is fused into it -- that pass writes the state without reading it.
 * The enqueue form does not wait.                                              */
int qs_plan_execute_from_basis(qs_state_t s, qs_plan_t p, uint64_t basis);
int qs_plan_enqueue_from_basis(qs_state_t s, qs_plan_t p, uint64_t basis);
/* qs_plan_execute_from_basis + the checksum fused into the last pass (above). */
int qs_plan_execute_from_basis_checksum(qs_state_t s, qs_plan_t p, uint64_t basis, double* checksum);
/* Diagnostics (bench.py roofline): qs_plan_execute_from_basis_checksum with a
 * CUDA event between consecutive steps; step_ms[i] = device time of step i,
 * step_bytes[i] = its algorithmic bytes (reads of possibly non-zero amplitudes
 * + writes); both arrays hold qs_plan_stats' launches entries (may be NULL).
 * checksum may be NULL.  Synchronises. */
int qs_plan_execute_from_basis_profile(qs_state_t s, qs_plan_t p, uint64_t basis, double* checksum, float* step_ms,
                                       double* step_bytes);
/* Executes steps [first, first+count) only (diagnostics, per-pass profiling). */
int qs_plan_execute_range(qs_state_t s, qs_plan_t p, uint64_t first, uint64_t count);
/* Planner statistics: passes (HBM sweeps) and kernel launches per execute.   */
int qs_plan_stats(qs_plan_t p, uint64_t* passes, uint64_t* launches, uint64_t* gates);

/* --- reference-mode gate fusion ----------------------------------------------
 * fuse_gate_run / fuse_circuit (fusion.hpp:20-133) on one run of gates: greedy
 * dependency-graph fusion into Custom blocks of <= max_fused_qubits qubits.
 * The result owns its matrices; qs_fused_get fills a qs_gate whose matrix
 * pointer stays valid until qs_fused_free.                                     */
typedef struct qs_fused* qs_fused_t;
int qs_fuse(const qs_gate* gates, uint64_t n, uint32_t num_qubits, uint32_t max_fused_qubits, qs_fused_t* out);
uint64_t qs_fused_count(qs_fused_t f);
int qs_fused_get(qs_fused_t f, uint64_t i, qs_gate* out);
int qs_fused_free(qs_fused_t f);

/* --- reductions (fixed-order trees; run-to-run deterministic) -------------- */
int qs_norm2(qs_state_t s, double* out);                              /* [statevector.hpp:158-162] */
int qs_prob_one(qs_state_t s, uint32_t q, double* out);               /* [statevector.hpp:181-186] */
/* marginal over qubits[0..m): result bit b <-> qubits[b]           [statevector.hpp:190-208] */
int qs_probs(qs_state_t s, const uint32_t* qubits, uint32_t m, double* out);
/* |a_i|^2 for i in [offset, offset+count)                           [statevector.hpp:210-215] */
int qs_probs_full(qs_state_t s, double* out, uint64_t offset, uint64_t count);
/* sum_i |a_i|^2 (i+1), the bench digest                                  [bench.hpp:141-148] */
int qs_checksum(qs_state_t s, double* out);
/* The same digest rounded exactly as the reference's serial loop (t_i =
 * fl(|a_i|^2 (i+1)), sum += t_i in index order): bit-identical to it on the
 * same amplitudes (serial-equivalent scan, DESIGN 3.4).  qs_checksum's tree
 * sum is the more accurate value; this one is for parity with the reference's
 * own rounding error (2^n serial adds).                       [bench.hpp:141-148] */
int qs_checksum_serial(qs_state_t s, double* out);

/* --- measurement ------------------------------------------------------------ */
/* collapse onto outcome with known probability                 [statevector.hpp:228-247] */
int qs_collapse(qs_state_t s, uint32_t q, int outcome, double prob);
/* measure_collapse: outcome = (u < P(0)) ? 0 : 1                [statevector.hpp:219-225] */
int qs_measure_collapse(qs_state_t s, uint32_t q, double u, int* outcome);
int qs_scale(qs_state_t s, double re, double im);                     /* [statevector.hpp:164-166] */

/* BasisSampler: cumulative |a|^2 in index order, upper-bound search of u*total
 * [statevector.hpp:542-570].  With exact != 0 the cumulative array reproduces
 * the reference's serial left-to-right double accumulation bit for bit (so
 * counts equal the reference's for the same amplitudes and draws); otherwise a
 * parallel scan is used.  out_index[i] is the basis state drawn for u[i].   */
int qs_sample(qs_state_t s, const double* uniforms, uint64_t shots, int exact, uint64_t* out_index);
/* Draws `shots` uniforms from the reference stream Rng(seed) (mt19937_64,
 * (next()>>11)*2^-53 [rng.hpp:33-35]) and samples them; out_index as above. */
int qs_sample_seeded(qs_state_t s, uint64_t seed, uint64_t shots, int exact, uint64_t* out_index);

/* --- expectation values -------------------------------------------------------
 * <psi| P_t |psi> for Pauli strings, one read pass per batch of terms
 * (replaces the per-term state copy + serial dot of       [variational.hpp:33-47]).
 * Term t has letters[t*n .. t*n+n) in {'I','X','Y','Z'} indexed by qubit.
 * out[2t], out[2t+1] = real and imaginary part of <psi|P_t|psi>.            */
int qs_expect_pauli(qs_state_t s, const char* letters, uint32_t nterms, double* out);

/* Reduced density matrix of 1..3 qubits (most significant first):
 * out[r][c] = sum over the other qubits of a[.. r ..] conj(a[.. c ..]),
 * 2^k x 2^k complex row-major interleaved.  One read pass.  The trajectory
 * noise step takes every Kraus weight ||K_i psi||^2 = Tr(K_i rho K_i^dag)
 * from it instead of one state copy per operator  [noise.hpp:259-311]. */
int qs_reduced_density(qs_state_t s, const uint32_t* qubits, uint32_t k, double* out);

/* --- shot batches (per-shot paths of run() / run_noisy for small states) ----
 * A state of n_total qubits holds B = 2^(n_total - shot_qubits) independent
 * shot_qubits-qubit states; shot s owns [s * 2^shot_qubits, (s+1) * 2^...).
 * Gates go through qs_apply_circuit (they never touch the shot bits); the
 * per-shot steps below take one uniform per shot (the caller draws them from
 * Rng::derive(seed, s) in program order, simulator.hpp:121-194):
 *   qs_batch_reset:   every shot to |0...0>
 *   qs_batch_measure: outcome_s = (u_s < 1 - P_s(1)) ? 0 : 1, collapse and
 *                     renormalise each shot       [statevector.hpp:219-247]
 *   qs_batch_kraus:   per shot, weights Tr(K_i rho_s K_i^dag) from the shot's
 *                     reduced density matrix, the reference's pick with u_s,
 *                     K_chosen / sqrt(w) applied  [noise.hpp:283-311]
 *                     (1- or 2-qubit channels, <= 16 operators, ops
 *                     nops x 2^k x 2^k complex row-major interleaved).       */
int qs_batch_reset(qs_state_t s, uint32_t shot_qubits);
int qs_batch_measure(qs_state_t s, uint32_t shot_qubits, uint32_t qubit, const double* uniforms, uint64_t shots,
                     signed char* outcomes);
int qs_batch_kraus(qs_state_t s, uint32_t shot_qubits, const uint32_t* qubits, uint32_t k, const double* ops,
                   uint32_t nops, const double* uniforms, uint64_t shots, int32_t* chosen);
/* Control flow in shot batches: a NEGATIVE uniform leaves that shot untouched
 * in qs_batch_measure (outcome -1) and qs_batch_kraus (chosen -1); and
 * qs_batch_apply applies one dense 2^k x 2^k matrix (k <= 3, qubits[0] most
 * significant, row-major interleaved) only to the shots with mask[s] != 0. */
int qs_batch_apply(qs_state_t s, uint32_t shot_qubits, const uint32_t* qubits, uint32_t k, const double* matrix,
                   const signed char* mask, uint64_t shots);

/* Gradient of <psi|H|psi>, psi = gates[0..count) applied to |0...0>, with
 * respect to the angle of each slot gate gates[slots[i]] (uncontrolled RX, RY
 * or RZ): out[i] = dE/dtheta_i -- the value the reference's parameter-shift
 * rule (E(t+pi/2) - E(t-pi/2)) / 2 yields for these gates
 * [variational.hpp:139-155].  Computed by adjoint differentiation: one
 * forward run, lambda = H psi, one backward sweep (2 state vectors resident).
 * H = sum_t coeffs[t] * P_t, coeffs complex interleaved, letters as in
 * qs_expect_pauli.  The state is used as workspace and is overwritten.       */
int qs_gradient(qs_state_t s, const qs_gate* gates, uint64_t count, const uint64_t* slots, uint64_t nslots,
                const char* letters, const double* coeffs, uint32_t nterms, double* out);

/* BasisSampler's cumulative array cum_i = sum_{j<=i} |a_j|^2 (host copy,
 * 2^n doubles) and its total, computed on the device with the serial-
 * equivalent exact scan: bit-identical to the reference's left-to-right
 * double accumulation                                  [statevector.hpp:544-552] */
int qs_cumulative(qs_state_t s, double* cum_out, double* total_out);

/* --- partial amplitudes (cut method) ------------------------------------------
 * partial_amplitude [pathsum.hpp:317-459]: the qubits split into block A
 * (block_a[0..na), ascending or not) and block B (the rest); every CZ / CNOT
 * across the cut is a branch variable.  Returns out[2t], out[2t+1] = the
 * amplitude <targets[t]|U|0...0> (targets as basis indices, qubit q = bit q),
 * summed over all 2^k branches.  The branches are batched as extra qubits of
 * two half-size states (2^batch_qubits amplitudes per block state at most;
 * 0 = 2^26), each block circuit runs as tile passes on `device`.  Gates: no
 * extra controls, 1 target or CNOT/CZ (QS_ERR_UNSUPPORTED otherwise, as the
 * reference's check_cuttable_gate).  The facade (qforge/pathsum.hpp,
 * qforge.plan_cut) chooses the cut and checks the CutPlan.                   */
int qs_partial_amplitude(uint32_t num_qubits, const qs_gate* gates, uint64_t n, const uint32_t* block_a, uint32_t na,
                         const uint64_t* targets, uint64_t ntargets, int device, uint32_t batch_qubits, double* out);

/* --- sharded state vectors (multi-GPU) -----------------------------------------
 * The reference keeps one 2^n vector in host memory [statevector.hpp:111-118]
 * and has no distributed mode; these entry points are the B200 extension the
 * survey's section 8(e) calls for.  An n-qubit state is split over 2^g shards:
 * the top g qubits are rank bits and shard r holds global indices
 * [r*2^(n-g), (r+1)*2^(n-g)).  A plan built by qs_plan_create_sharded runs tile
 * passes on every shard independently; a non-diagonal gate on a rank bit is
 * preceded by a pairwise half-shard exchange (rank bit <-> local qubit).
 *
 *   qs_shards_create_local: all 2^g shards in this process on one device
 *     (exchanges are device-local swaps; validates sharded plans on 1 GPU).
 *   qs_shards_create_dist: this rank's shard, exchanges via NCCL send/recv
 *     over NVLink.  libnccl.so.2 is loaded at run time (env QSB_NCCL_LIB
 *     overrides the name).  The 128-byte unique id from qs_dist_unique_id on
 *     one rank is broadcast by the caller (e.g. torch.distributed); world must
 *     be a power of two.  Destroy the shards before their communicator.
 *
 * Amplitude I/O takes global indices; a distributed handle only serves the
 * range of its own shard.  Reductions are summed in rank order on every rank
 * (bit-identical across ranks and runs).                                      */
typedef struct qs_dist* qs_dist_t;
typedef struct qs_shards* qs_shards_t;
int qs_dist_unique_id(unsigned char out[128]);
int qs_dist_create(const unsigned char id[128], int world, int rank, int device, qs_dist_t* out);
/* A communicator whose collectives are the caller's (no NCCL): allgather
 * gathers `bytes` from every rank into recv in rank order, barrier blocks
 * until every rank arrived; both return 0 on success.  The state's exchanges
 * then run only over CUDA-IPC peer memory (one kernel storing into the other
 * ranks' buffers, the stream drained, then the host barrier).  Used to run
 * the multi-process data path with torch.distributed over gloo -- e.g. ranks
 * as processes sharing one GPU, which NCCL refuses.                          */
typedef struct {
  void* ctx;
  int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes);
  int (*barrier)(void* ctx);
} qs_host_collectives;
int qs_dist_create_host(const qs_host_collectives* c, int world, int rank, int device, qs_dist_t* out);
int qs_dist_destroy(qs_dist_t d);
int qs_shards_create_local(uint32_t num_qubits, uint32_t global_qubits, int device, qs_shards_t* out);
int qs_shards_create_dist(uint32_t num_qubits, qs_dist_t d, qs_shards_t* out);
int qs_shards_destroy(qs_shards_t s);
/* global_qubits = g; first_rank = lowest shard index held by this handle;
 * local_count = shards held (2^g local, 1 distributed).                       */
int qs_shards_info(qs_shards_t s, uint32_t* num_qubits, uint32_t* global_qubits, uint32_t* first_rank,
                   uint32_t* local_count);
void* qs_shards_stream(qs_shards_t s);
int qs_shards_sync(qs_shards_t s);
int qs_shards_set_basis_state(qs_shards_t s, uint64_t index);
int qs_shards_set_amplitudes(qs_shards_t s, const double* data, uint64_t offset, uint64_t count);
int qs_shards_get_amplitudes(qs_shards_t s, double* data, uint64_t offset, uint64_t count);
/* Plans for a state with `global_qubits` rank bits (tile plans only).         */
int qs_plan_create_sharded(uint32_t num_qubits, uint32_t global_qubits, const qs_gate* gates, uint64_t n,
                           qs_plan_t* out);
/* Number of rank-bit exchanges one execution performs.                      */
int qs_plan_exchanges(qs_plan_t p, uint64_t* exchanges);
/* Step i of a plan: kind 0 = per-gate kernel, 1 = tile pass, 2 = rank-bit
 * exchange of rank bits gpos[b] (qubit n-g+gpos[b]) with local qubits
 * lpos[b], b < *nbits (arrays of QS_MAX_EXCHANGE_BITS; nbits = 0 otherwise). */
#define QS_MAX_EXCHANGE_BITS 16
int qs_plan_step_info(qs_plan_t p, uint64_t i, int* kind, uint32_t* nbits, uint32_t* gpos, uint32_t* lpos);
/* Tile pass i (diagnostics): tile qubits (*m of them, ascending, into
 * qubits[16]), register bits *r (2^r amplitudes per thread), shared-memory
 * exchanges *transposes, micro-ops *nops, source gates covered *gates.  *m = 0
 * when step i is not a tile pass. */
int qs_plan_tile_info(qs_plan_t p, uint64_t i, uint32_t* m, uint32_t* qubits, uint32_t* r, uint32_t* transposes,
                      uint32_t* nops, uint64_t* gates);
int qs_shards_plan_enqueue(qs_shards_t s, qs_plan_t p);
/* Reset to |basis> (global index) fused into the plan's first tile pass; no wait. */
int qs_shards_plan_enqueue_from_basis(qs_shards_t s, qs_plan_t p, uint64_t basis);
/* Executes with a CUDA event around every step (step_ms[i], one per step).   */
int qs_shards_plan_execute_timed(qs_shards_t s, qs_plan_t p, float* step_ms);
int qs_shards_plan_execute(qs_shards_t s, qs_plan_t p);
int qs_shards_apply_circuit(qs_shards_t s, const qs_gate* gates, uint64_t n);
/* run() on a sharded state: reset to |basis> fused into the first pass (runs
 * from a basis state skip provably zero tiles / shards), then the host gate
 * list; waits.                                                                 */
int qs_shards_run_circuit(qs_shards_t s, uint64_t basis, const qs_gate* gates, uint64_t n);
int qs_shards_norm2(qs_shards_t s, double* out);
/* Marginal probabilities over distinct qubits (result bit b <-> qubits[b]),
 * summed over shards in rank order                        [statevector.hpp:190-208] */
int qs_shards_probs(qs_shards_t s, const uint32_t* qubits, uint32_t m, double* out);
/* BasisSampler over the sharded state: the cumulative |a|^2 runs through the
 * shards in rank order (each shard continues the previous one's running sum,
 * so exact mode is bit-identical to the reference's serial loop); out_index
 * holds global basis indices, identical on every rank     [statevector.hpp:542-570] */
int qs_shards_sample(qs_shards_t s, const double* uniforms, uint64_t shots, int exact, uint64_t* out_index);
int qs_shards_sample_seeded(qs_shards_t s, uint64_t seed, uint64_t shots, int exact, uint64_t* out_index);
/* <psi|P_t|psi> (letters as in qs_expect_pauli); X on rank bits pairs shards. */
int qs_shards_expect_pauli(qs_shards_t s, const char* letters, uint32_t nterms, double* out);
int qs_shards_checksum(qs_shards_t s, double* out);

#ifdef __cplusplus
}
#endif

#endif /* QSB_H_ */
