// Launchers for the per-gate kernels, reductions, measurement and sampling
// (kernels.cu).  All run on the state's stream; host-visible results are
// synchronous on return.
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "common.hpp"
#include "gates.hpp"

namespace qsb {

// One HBM pass per op (the reference's per-gate kernels, statevector.hpp:268-467).
void launch_op(State& s, const Op& op);

// Out-of-place qubit permutation: bit q of every index moves to bit pos[q]
// (one HBM pass into the state's second buffer, then the buffers swap).
// red != null: also one checksum partial per block into red[0 .. return value)
unsigned permute_qubits(State& s, const std::vector<uint32_t>& pos, double* red = nullptr);

void fill_basis(State& s, uint64_t index);
void zero_outside(State& s, uint64_t mask, uint64_t val);
// sums per-CTA partials part[0..count) in a fixed order (part[count] is scratch); synchronises
double sum_partials(State& s, double* part, unsigned count);     // a[i] = 0 where (global i & mask) != val                      // |index> (local index; out of range = all 0)

// Rank-bit exchanges for sharded states (shard.cpp).
void swap_halves(State& a, State& b, uint32_t p);                // a: rank bit 0, b: rank bit 1, same device
// Peer-memory exchange of rank bits <-> local bits lpos[0..k): every amplitude
// is written to peers[d] (d = its bits at lpos) at its new local index (those
// bits replaced by aval).  peers[] are the owners' second buffers.
constexpr uint32_t kMaxExchangeBits = 4;
constexpr uint32_t kMaxPeers = 1u << kMaxExchangeBits;
void scatter_exchange(State& s, double2* const* peers, const uint32_t* lpos, uint32_t k, uint32_t aval);

// Block d of a k-bit exchange:local indices whose bits lpos[i] equal bit i of
// d, enumerated by the remaining bits ascending; [off, off+cnt) of it.
void pack_block(State& s, const uint32_t* lpos, uint32_t k, uint32_t d, uint64_t off, uint64_t cnt, double2* out);
void unpack_block(State& s, const uint32_t* lpos, uint32_t k, uint32_t d, uint64_t off, uint64_t cnt,
                  const double2* in);
double reduce_norm2(State& s);                                   // statevector.hpp:158-162
double reduce_prob_one(State& s, uint32_t q);                    // :181-186
double reduce_checksum(State& s);                                // bench.hpp:141-148
void marginal_probs(State& s, const uint32_t* q, uint32_t m, double* host_out);  // :190-208
void full_probs(State& s, double* host_out, uint64_t offset, uint64_t count);    // :210-215
void collapse(State& s, uint32_t q, int outcome, double inv_sqrt_p);             // :228-247
void scale(State& s, double re, double im);                                      // :164-166

// BasisSampler (statevector.hpp:542-570) + draws.  exact: reproduce the serial
// cumulative sum bit for bit (see kernels.cu, "serial-equivalent scan").
void sample(State& s, const double* uniforms_host, uint64_t shots, bool exact, uint64_t* out_host);
void sample_gen(State& s, uint64_t shots, bool exact, uint64_t* out_host,
                const std::function<void(double*, uint64_t)>& gen);

// <psi|P|psi> for Pauli strings given as (xmask, zmask, #Y) per term.
void expect_pauli(State& s, const std::vector<uint64_t>& xmask, const std::vector<uint64_t>& zmask,
                  const std::vector<int>& ny, double* out);

// Sharded sampling (shard.cpp): this shard's cumulative |a|^2 continuing from
// *carry_dev (the previous shard's total; null = 0), plus device room for
// `shots` uniforms and indices.
struct ShardCum {
  double* cum;
  double* total;  // device: this shard's final running sum
};
ShardCum shard_cumulative(State& s, bool exact, const double* carry_dev, uint64_t shots, double** u_dev,
                          unsigned long long** out_dev);
// Writes global indices for the shots this shard owns (targets in [*lo, total)).
void search_range(State& s, const ShardCum& c, const double* total_dev, const double* lo_dev, bool last,
                  const double* u_dev, uint64_t shots, unsigned long long* out_dev);
// sum_{j < size} conj(partner[j ^ xl]) a[j] (-1)^popc(j & smask) (host, synchronous; s
// supplies stream and scratch).
void pauli_cross(State& s, const double2* a, const double2* partner, uint64_t size, uint64_t xl, uint64_t smask_local,
                 double* out2);

// Reduced density matrix over 1..3 qubits (msb first): out = 2^k x 2^k
// complex, row-major interleaved (host, synchronous).
void reduced_density(State& s, const uint32_t* targets, uint32_t k, double* out);

// Shot batches: B n-qubit states as one vector (shot s at [s*2^n, (s+1)*2^n)).
void batch_reset(State& s, uint32_t n);
void batch_measure(State& s, uint32_t n, uint32_t q, const double* u_host, uint64_t shots, signed char* out_host);
// m (2^k x 2^k, row-major interleaved; qubits[0] = most significant) applied to the shots with mask[s] != 0
void batch_apply(State& s, uint32_t n, const uint32_t* qubits, uint32_t k, const double* m_host,
                 const signed char* mask_host, uint64_t shots);
void batch_kraus(State& s, uint32_t n, const uint32_t* qubits, uint32_t k, const double* ops_host, uint32_t nops,
                 const double* u_host, uint64_t shots, int* chosen_host);

// dst += f * P src (P = X^x Z^z, f complex incl. i^#Y), over s.size amplitudes.
void pauli_axpy(State& s, double2* dst, const double2* src, uint64_t xmask, uint64_t zmask, double fre, double fim);

// Exposed for tests of the exact scan (cum must hold s.size doubles on device).
double exact_cumulative(State& s, double* d_probs, double* d_cum);
// probability_checksum with the reference's serial rounding (bench.hpp:141-148):
// bitwise equal to the serial loop on the same amplitudes.
double serial_checksum(State& s);
// sum_b a[b 2^na + ta[t]] * b[b 2^nb + tb[t]] over b < 2^c, per target t (partial_amplitude).
void branch_dot(State& a, State& b, uint32_t na, uint32_t nb, uint32_t c, const std::vector<uint64_t>& ta,
                const std::vector<uint64_t>& tb, std::vector<cd>& out);

}  // namespace qsb
