// Sharded state vectors: the top g qubits of an n-qubit state are
// rank bits; shard r holds the 2^(n-g) amplitudes whose global index has
// rank bits = r.  Tile passes run on every shard independently (rank bits are
// outside every tile: diagonal gates and controls on them are per-shard
// constants); a non-diagonal gate on a rank bit is preceded by a planner
// SwapStep: rank bits j_i <-> local qubits p_i (i < k).  For k = 1 it is a
// pairwise exchange of half a shard between ranks r and r ^ 2^j; for k > 1 an
// all-to-all among the 2^k ranks that differ in those bits, each rank keeping
// 1/2^k of its shard.
//
// Two transports:
//   * LocalTransport: all 2^g shards in one process on one device.  Used to
//     validate sharded plans on a single B200 with each distributed data path:
//     "swap" (one swap kernel per bit), "staged" (the NCCL fallback's
//     pack/unpack protocol) and "peer" (the peer-memory scatter kernel into
//     sibling shards' second buffers).
//   * NcclTransport: one shard per process/GPU.  Default ("peer"): every
//     rank maps every other rank's two shard buffers through CUDA IPC and an
//     exchange is ONE kernel storing each amplitude straight into its new
//     owner's free buffer over NVLink (no staging, no pack/unpack), followed
//     by a stream-ordered NCCL barrier; buffers then flip.  Fallback ("nccl"):
//     pack -> grouped ncclSend/ncclRecv in bounded chunks -> unpack.  libnccl
//     is loaded at run time; the unique id is exchanged by the caller (e.g.
//     torch.distributed).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "common.hpp"

namespace qsb {

struct Plan;

struct Transport {
  virtual ~Transport() = default;
  // Swaps rank bit gpos[i] with local qubit lpos[i] for every i (disjoint pairs).
  virtual void exchange(std::vector<State*>& shards, const std::vector<uint32_t>& gpos,
                        const std::vector<uint32_t>& lpos) = 0;
  // sum of one double per shard over all ranks, in rank order (deterministic)
  virtual double sum(const std::vector<double>& per_local_shard) = 0;
  virtual void barrier() {}
  // Releases transport resources that reference the shards (before they are freed).
  virtual void close() {}
  // Runs tile pass tp with the following exchange fused into its stores
  // (peer-memory transports); false = not supported, run them separately.
  virtual bool fused_exchange(std::vector<State*>& shards, const struct TileProgram& tp,
                              const std::vector<uint32_t>& gpos, const std::vector<uint32_t>& lpos) {
    return false;
  }
};

struct ShardSet {
  uint32_t n = 0, g = 0;
  int device = 0;
  std::vector<std::unique_ptr<State>> shards;  // the shards this process holds
  std::unique_ptr<Transport> tr;
  cudaStream_t stream = nullptr;               // shared by the local shards
  bool owns_stream = true;

  std::vector<State*> ptrs() {
    std::vector<State*> v;
    for (auto& s : shards) v.push_back(s.get());
    return v;
  }
  ~ShardSet();
};

// Single-process group of 2^g shards on `device`.
std::unique_ptr<ShardSet> make_local_shards(uint32_t n, uint32_t g, int device);

// NCCL communicator handle (dist API).
struct Dist;
void dist_unique_id(unsigned char out[128]);
Dist* dist_create(const unsigned char id[128], int world, int rank, int device);
// Communicator over the caller's host collectives (no NCCL; peer memory only).
Dist* dist_create_host(const qs_host_collectives& c, int world, int rank, int device);
void dist_destroy(Dist* d);
int dist_rank(const Dist* d);
int dist_world(const Dist* d);
// This process's shard of an n-qubit state over dist's world (a power of two).
std::unique_ptr<ShardSet> make_dist_shard(uint32_t n, Dist* d);

void shard_fill_basis(ShardSet& ss, uint64_t index);
// basis: the run started from |basis> (zero tiles skipped); unwritten: lazy
// zeros of that run (amplitudes outside (mask, val) not yet written; zeroed
// before any step that reads everything and at the end)
void shard_execute(ShardSet& ss, const Plan& p, uint64_t first = 0, uint64_t count = ~0ull,
                   const uint64_t* basis = nullptr, struct TileSkip* unwritten = nullptr);
// Resets to |basis> (global index) and runs the plan, the reset fused into a
// leading tile pass.  Enqueued on the shard stream.
void shard_execute_from_basis(ShardSet& ss, const Plan& p, uint64_t basis);
double shard_norm2(ShardSet& ss);
double shard_checksum(ShardSet& ss);
// Amplitude / probability I/O over [offset, offset+count) of the global index;
// in a distributed set the range must lie inside this rank's shard.
void shard_get(ShardSet& ss, double* out, uint64_t offset, uint64_t count);
void shard_set(ShardSet& ss, const double* in, uint64_t offset, uint64_t count);
void shard_sync(ShardSet& ss);
// Marginal over distinct qubits (result bit b <-> qubits[b]); every rank gets
// the full result, summed over shards in rank order.
void shard_probs(ShardSet& ss, const uint32_t* qubits, uint32_t m, double* out);
// BasisSampler over the whole sharded state: the cumulative sum runs serially
// through the shards in rank order (exact mode: bit-identical to the
// reference's serial loop); out[i] = global basis index for u[i], on every rank.
void shard_sample(ShardSet& ss, const double* u, uint64_t shots, bool exact, uint64_t* out);
// <psi|P_t|psi> for Pauli strings (xmask, zmask, #Y); X parts on rank bits pair
// each shard with its partner (peer memory, sibling shard, or streamed chunks).
void shard_expect_pauli(ShardSet& ss, const std::vector<uint64_t>& xm, const std::vector<uint64_t>& zm,
                        const std::vector<int>& ny, double* out);

}  // namespace qsb
