// Gate fusion, reference mode: the greedy dependency-graph fusion of
// fuse_gate_run / fuse_circuit (fusion.hpp:20-133), producing dense Custom
// blocks of at most max_fused_qubits qubits.  Used by qs_fuse (the facade's
// fuse_circuit) and by the QS_PLAN_DENSE_FUSION execution mode.
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"

namespace qsb {

// An owned gate record (qs_gate plus storage for its matrix).
struct GateRec {
  qs_gate g{};
  std::vector<double> matrix;  // interleaved row-major, when Custom
  void bind() { g.matrix = matrix.empty() ? nullptr : matrix.data(); }
};

GateRec copy_gate(const qs_gate& g);

// Fuses one run of gates (no measurements inside) over an nq-qubit register.
std::vector<GateRec> fuse_gate_run(const qs_gate* gates, uint64_t count, uint32_t nq, uint32_t max_fused_qubits);

// Dense full matrix of a gate on its operand list controls ++ targets
// (controls in the high bits): gate_matrix, gates.hpp:101-103.
std::vector<cd> gate_matrix(const qs_gate& g, int* dim_out);

// embed_on_bits (gates.hpp:108-140): u acts on `bits` (local positions, most
// significant first) of a k-bit space.
std::vector<cd> embed_on_bits(const std::vector<cd>& u, int udim, const std::vector<uint32_t>& bits, uint32_t k);

}  // namespace qsb
