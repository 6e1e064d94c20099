// Host-side gate semantics: named matrices, dagger, validation, and lowering
// of a qs_gate to one kernel-level operation, following
//   standard_gate_matrix / base_matrix   gates.hpp:15-97
//   validate_gate                        circuit.hpp:429-469
//   StateVector::apply_gate dispatch     statevector.hpp:469-538
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"

namespace qsb {

enum class OpKind : uint8_t { Identity, Flip, Diag, Mat1, Swap, Dense };

// One kernel-level operation.  Controls hold every control qubit (the gate's
// extra controls plus the defining controls of CNOT/CZ/TOFFOLI).
struct Op {
  OpKind kind = OpKind::Identity;
  std::vector<uint32_t> targets;   // Flip/Diag/Mat1: 1, Swap: 2, Dense: k (msb first)
  std::vector<uint32_t> controls;
  std::vector<cd> m;               // Diag: {d0, d1}; Mat1: 2x2; Dense: 2^k x 2^k (row-major)
  uint64_t gate_index = 0;         // position in the submitted gate list
  uint64_t cneg = 0;               // controls that must be 0 (tile plans, diagonal ops only:
                                   // produced by Pauli-X absorption, tile_plan.cpp)
};

// Row-major matrix of a named gate on its targets (defining controls in the
// high bits), or the custom matrix; adjoint if dagger.  Returns the dimension.
int base_matrix(const qs_gate& g, std::vector<cd>& out);
bool is_unitary(const std::vector<cd>& m, int dim, double tol);

// Throws ValidationError with the reference's wording when the gate is not
// applicable to an n-qubit state.
void validate_gate(const qs_gate& g, uint32_t n);

// apply_gate lowering.  `validate` re-checks operands and custom unitarity.
Op lower_gate(const qs_gate& g, uint32_t n, bool validate = true);

// apply_matrix lowering (statevector.hpp:363-403): k == 1 becomes Mat1.
Op lower_matrix(const uint32_t* targets, uint32_t k, const double* m, const uint32_t* controls,
                uint32_t nc, uint32_t n);

// True when the op leaves the computational-basis bit of qubit q unchanged
// (diagonal action on q: controls, Diag targets, diagonal-in-q dense blocks).
bool op_preserves_bit(const Op& op, uint32_t q);

}  // namespace qsb
