// Execution plans: a circuit compiled once into a sequence of device steps.
//   - OpStep: one per-gate kernel (one HBM pass), kernels.cu
//   - TileStep: one shared-memory tile pass applying many gates, tile.cu
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "common.hpp"
#include "gates.hpp"

namespace qsb {

struct TileProgram;  // tile.hpp

struct Step {
  enum Kind { OpStep, TileStep, SwapStep, PermStep } kind = OpStep;
  Op op;                               // OpStep
  std::shared_ptr<TileProgram> tile;   // TileStep
  // SwapStep (sharded states): for every i, exchange physical qubit
  // n-g+gpos[i] (a rank bit) with local physical qubit lpos[i].  One bit is a
  // pairwise half-shard exchange; k bits are an all-to-all among the 2^k
  // ranks that differ in those rank bits (each sends 1 - 2^-k of its shard).
  std::vector<uint32_t> gpos, lpos;
  // PermStep: out-of-place qubit permutation, bit q of every index -> bit
  // perm[q] (restores the logical layout after relabeling SWAPs in one pass).
  std::vector<uint32_t> perm;
  // TileStep, runs started from a basis state |b> (qs_plan_execute_from_basis):
  // qubits that are still definite at the start of the pass, with their value
  // as an affine GF(2) form of b (parity(b & mask) ^ c).  A tile whose index
  // disagrees with the outside ones is all zero and stays zero: the pass skips
  // it (no HBM traffic in place; zeros written when out of place); inside a
  // tile, amplitudes that disagree with the inside ones are zero and not read.
  std::vector<uint32_t> def_pos;
  std::vector<uint64_t> def_mask;
  std::vector<uint8_t> def_const;
};

struct Plan {
  uint32_t n = 0;
  uint32_t g = 0;         // global (rank) qubits: the state is split over 2^g shards
  uint32_t mode = QS_PLAN_DEFAULT;
  uint64_t gates = 0;     // submitted gate count
  std::vector<Step> steps;
  uint64_t passes() const;
  uint64_t launches() const;
};

// Lowers and plans `count` gates for an n-qubit state.
// sharded: a plan for ShardSets (layout restored in place, no permutation steps).
std::unique_ptr<Plan> make_plan(uint32_t n, const qs_gate* gates, uint64_t count, uint32_t mode,
                                uint32_t max_fused_qubits, uint32_t global_qubits = 0, bool sharded = false);
// make_plan through a small LRU keyed by the exact submitted bytes (gates,
// custom matrices, options); QSB_PLAN_CACHE=0 disables it.
std::shared_ptr<const Plan> cached_plan(uint32_t n, const qs_gate* gates, uint64_t count, uint32_t mode,
                                        uint32_t max_fused_qubits, uint32_t global_qubits = 0, bool sharded = false);
void execute_plan(State& s, const Plan& p);
// Resets to |basis> and runs the plan; when the plan starts with a tile pass
// the reset is fused into it (no separate write pass, no read of the old state).
// checksum != null: also returns probability_checksum of the result, fused
// into the last tile pass when the plan ends with one (synchronises).
// prof != null (diagnostics, synchronises): per-step device time (CUDA events
// between the steps on the state's stream) and algorithmic bytes (reads of
// possibly non-zero amplitudes + writes of the amplitudes the step stores).
struct StepProfile {
  std::vector<float> ms;
  std::vector<double> bytes;
};
void execute_plan_from_basis(State& s, const Plan& p, uint64_t basis, double* checksum = nullptr,
                             StepProfile* prof = nullptr);
// The zero-tile mask of a tile step for a run started from |basis>.
struct TileSkip zero_tiles(const Step& st, uint64_t basis);
void execute_step(State& s, const Step& st);

}  // namespace qsb
