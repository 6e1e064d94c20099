// Shared-memory tile passes: many gates per HBM sweep.
//
// A pass picks a set S of m qubits (always containing the lowest L qubits, so
// global loads stay coalesced).  The state splits into 2^(n-m) tiles, each the
// 2^m amplitudes that share the values of the qubits outside S.  One CTA loads
// a tile into registers (16 amplitudes per thread), applies every gate of the
// pass whose non-diagonal targets lie in S, and writes the tile back: one HBM
// read + write for the whole gate run.
//
// Inside the CTA, 4 "register qubits" are held in registers; gates act on
// them with no data movement.  A TRANSPOSE micro-op permutes which tile qubits
// are register qubits through shared memory (XOR-swizzled, bank-conflict
// free).  Diagonal gates (RZ, Z, S, T, CZ, controlled phases) never need their
// qubits in S or in registers: their phase is known per register slot, per
// thread and per tile; runs of them merge into one PHASE micro-op.  Controls
// are predicates on the same three index levels.  Uncontrolled SWAPs are
// free relabels of the tile layout.
//
// Gate semantics follow StateVector::apply_gate (statevector.hpp:469-538);
// the reference has no multi-gate kernel -- this replaces its one-pass-per-
// gate loop (simulator.hpp:157-159) and its dense fusion (fusion.hpp:20-133).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <vector>

#include "common.hpp"
#include "gates.hpp"
#include "plan.hpp"

namespace qsb {

constexpr int kTileMinR = 4;    // register bits: 16 amplitudes per thread ...
constexpr int kTileMaxR = 5;    // ... or 32 (13-qubit tiles: fewer transposes)
constexpr int kTileMaxM = 13;   // tile qubits (2^13 x 16 B = 128 KiB of smem)
constexpr int kTileMaxT = kTileMaxM - kTileMinR;
constexpr int kTileMaxSlots = 1 << kTileMaxR;

enum TOpType : uint8_t {
  TO_MAT1 = 1,     // general 2x2 on register bit k
  TO_MAT1_REAL,    // real 2x2 (RY, H)
  TO_MAT1_RX,      // real diagonal, imaginary off-diagonal (RX)
  TO_FLIP,         // X / CNOT / TOFFOLI target on register bit k
  TO_PHASE,        // diagonal: c * prod_q w_q^{b_q} under a predicate
  TO_DENSE2,       // dense 4x4 on register bits 0..1
  TO_DENSE3,       // dense 8x8 on register bits 0..2
  TO_TRANSPOSE,    // register <-> thread qubit exchange through smem
  TO_RELABEL,      // SWAP as a relabel: thread-bit -> qubit map changes, no data moves
};

struct TOp {
  uint8_t type;
  uint8_t k;        // register bit (MAT1 / FLIP)
  uint16_t nlist;   // PHASE: number of non-register (qubit, w) factors
  uint16_t rmask;   // predicate on the register index p: (p & rmask) == rval
  uint16_t rval;
  unsigned long long gmask;  // predicate on the thread's global index bits
  unsigned long long gval;
  uint32_t coef;    // offset into the coefficient table (double2 units)
  uint32_t meta;    // offset into the metadata table (uint32 units)
};

// Per-config data for global addressing: thread bit k holds qubit tq[k];
// register bit k holds qubit with stride rs[k].
struct TileConfigAddr {
  uint32_t tq[kTileMaxT];
  unsigned long long rs[kTileMaxR];
};

struct TileHeader {
  uint32_t n, m, t, nops;
  uint32_t S[kTileMaxM];  // tile qubits, ascending
  TileConfigAddr load, store;
  uint32_t ops_off, meta_off, coef_off, bytes;
  unsigned long long ntiles;
  // Out-of-place pass (the plan's final qubit permutation folded in): stores
  // go to the second buffer; store addressing above is already permuted and
  // out_pos[i] is the output bit of tile-index bit i (non-tile qubits, ascending).
  uint32_t oop = 0;
  uint8_t out_pos[64] = {};
  uint32_t r = 4;  // register bits (2^r amplitudes per thread, t = m - r thread bits)
};

struct TileProgram {
  TileHeader h{};

  std::vector<TOp> ops;
  std::vector<uint32_t> meta;
  std::vector<double2> coef;
  uint64_t gates = 0;       // source ops covered
  uint32_t transposes = 0;
  std::vector<uint64_t> source;  // gate indices, for diagnostics
  std::shared_ptr<struct JitModule> jit;  // specialised kernel (jit.hpp)
  // lazily built variants (jit.cpp variant_module): from a basis state, sparse reads, fused checksum
  mutable std::map<unsigned, std::shared_ptr<struct JitModule>> variants;
  mutable std::map<uint64_t, std::shared_ptr<struct JitModule>> jit_xchg;  // exchange-fused variants, by local bits
  std::vector<double2> params;            // kernel parameter table (coef + generator constants)
};
// A pass that starts with a transpose out of the (coalesced) load layout: with
// prefetching, the cp.async writes land directly in the transpose's slots, so
// that transpose needs no shared-memory buffer or write phase of its own.
inline bool leading_transpose(const TileProgram& tp) { return !tp.ops.empty() && tp.ops[0].type == TO_TRANSPOSE; }
inline uint32_t buffered_transposes(const TileProgram& tp, bool prefetch) {
  return tp.transposes - ((prefetch && leading_transpose(tp)) ? 1u : 0u);
}


// The coefficient table travels as a __grid_constant__ kernel parameter
// (constant bank); the planner keeps every pass's tables below this size.
constexpr uint32_t kTileBlobBytes = 24 * 1024;
// Hard limit of the __grid_constant__ parameter (CUDA 12.1+: 32764 bytes).
constexpr uint32_t kParamLimitBytes = 32 * 1024 - 256;

// Bulk-copy (TMA) staging of the next tile instead of per-thread cp.async
// (jit_gen.hpp `tma`); QSB_TMA=1/0.
inline bool tma_enabled() {
  const char* e = std::getenv("QSB_TMA");
  return e && std::atoi(e) != 0;
}

// TMA tensor view of a tile: the tile qubits S split into <= 5 runs of
// consecutive positions (a[i], l[i]) -- a tensor map whose dimension i covers
// positions [a[i], a[i+1]) with a box of 2^l[i] (the tile's run) addresses one
// tile per coordinate set.  Boxes are at most 256 elements per dimension (8-B
// elements: the innermost run holds <= 128 amplitudes, the others <= 256), so
// long runs are split.  Returns the rank, or 0 when the tile needs more than 5
// dimensions or does not start with a 16-amplitude run.
inline uint32_t tma_segments(const TileHeader& h, uint32_t a[5], uint32_t l[5]) {
  uint32_t k = 0, b = 0;
  while (b < h.m) {
    uint32_t e = b + 1;
    while (e < h.m && h.S[e] == h.S[e - 1] + 1) ++e;
    uint32_t pos = h.S[b], len = e - b;
    while (len) {
      const uint32_t cap = k == 0 ? 7u : 8u;
      const uint32_t take = len < cap ? len : cap;
      if (k == 5) return 0;
      a[k] = pos;
      l[k] = take;
      ++k;
      pos += take;
      len -= take;
    }
    b = e;
  }
  if (a[0] != 0 || l[0] < 4) return 0;
  return k;
}

struct TileOptions {
  uint32_t m = 12;  // tile qubits
  uint32_t r = 4;   // register qubits per thread
  // 13-qubit passes: compile every pass with 4 and 5 register bits and keep
  // the cheaper by pass_cost (QSB_TILE_R fixes r instead)
  bool choose_r = true;
  uint32_t low = 4; // qubits 0..low-1 always in the tile: 256 B contiguous runs
                    // (measured: 128 B runs 70% of HBM per pass, 256 B 80%)
  bool remap = true;  // plan-level qubit relabelling (low slots hold the qubits needed next)
  // End a plan whose layout was relabeled with one out-of-place permutation
  // pass (needs a second state buffer) instead of in-place relabel passes.
  bool perm_step = true;
  // Drop X gates whose flip can be folded into later gates (absorb_pauli_x).
  bool absorb_x = true;
  // Fold that permutation into the last tile pass when possible (out of place).
  bool fold_perm = true;
  // The first register configuration is free: the prefetch writes the tile to
  // shared memory in the layout of the first transpose, so a pass may start
  // with the low qubits in registers at the cost of one barrier.
  bool free_load = true;
  uint32_t global_qubits = 0;  // sharded states: top qubits are rank bits, never in a tile
};
TileOptions tile_options_from_env();

void plan_tiles(uint32_t n, std::vector<Op>& ops, std::vector<Step>& steps, const TileOptions& opt);
// Estimated time of a plan in units of one HBM sweep (measured on B200, 30
// qubits, profiles/r1/random30_per_pass.txt: 12- and 13-qubit passes with <= 2
// shared-memory exchanges 5.8 ms, each further exchange +17%).
double plan_cost(const std::vector<Step>& steps);
// Estimated time of one tile pass in the same units (see plan_cost).
double pass_cost(const TileProgram& tp);
// Plans with and without qubit relabelling (unless fixed by QSB_TILE_REMAP),
// with 12- and, for large unsharded states, 13-qubit tiles (unless fixed by
// QSB_TILE_M), and keeps the cheapest plan.
// in_place_only: no out-of-place permutation pass (it needs a second state
// buffer): the layout is restored by in-place relabel passes instead.
void plan_tiles(uint32_t n, std::vector<Op>& ops, std::vector<Step>& steps, uint32_t global_qubits = 0,
                bool sharded = false, bool in_place_only = false);
// basis != null: the pass starts from |*basis> (global index) instead of
// reading the state -- a reset fused into the first pass.
// Exchange fused into a pass (sharded plans, peer memory): after the pass,
// rank bits gpos[i] trade places with local bits lpos[i].
struct TileXchg {
  uint32_t k = 0;
  uint32_t lpos[4] = {};
  double2* peers[16] = {};  // free buffer of the shard whose exchanged bits are d
  unsigned long long aval = 0;  // this shard's exchanged rank bits, placed at lpos
};
// Zero-tile skip (runs from a basis state): tiles with (index & mask) != val
// are zero and stay zero.
constexpr unsigned kMaxTileGrid = 8192;  // CTAs of a reducing tile pass (partials buffer size)

struct TileSkip {
  unsigned long long mask = 0, val = 0;    // definite qubits outside the tile: zero tiles
  unsigned long long imask = 0, ival = 0;  // definite tile qubits: only matching amplitudes are read
  // tile qubits still definite after the pass (the next step's definite qubits):
  // amplitudes that disagree are zero and are not stored (the next step does
  // not read them; in place, not the last step, only tile steps follow)
  unsigned long long omask = 0, oval = 0;
  // first pass of a run from a basis state: write only the tiles that can be
  // non-zero (the rest is zeroed later, only if some step would read it)
  bool lazy = false;
};
// red != null: also writes one checksum partial per CTA (sum |a_i|^2 (i+1) over
// the stored amplitudes) to red[0 .. return value)
unsigned launch_tile(State& s, const TileProgram& tp, const uint64_t* basis = nullptr, const TileXchg* x = nullptr,
                     const TileSkip* skip = nullptr, double* red = nullptr);

}  // namespace qsb
