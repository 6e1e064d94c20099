// Synthetic benchmark circuits that the reference does not ship (BASELINE.json
// configs 1, 3, 4, 5), written against the reference's own types so the
// reference CPU simulator can run them.  The product mirrors the same
// definitions (paper_2212_14201_b200/include/qforge/b200_circuits.hpp) and the
// C oracle restates them (qsim_oracle.c); tests/golden pins all three equal.
//
// TEST INFRASTRUCTURE ONLY (used by oracle/ref_driver.cpp).
#pragma once

#include <cstdint>
#include <numbers>

#include "qforge/circuit.hpp"
#include "qforge/pauli.hpp"
#include "qforge/rng.hpp"

namespace oraclegen {

using namespace qforge;

// GHZ(n): H(0), then CNOT(i, i+1) for i < n-1.
inline Program gen_ghz(std::uint32_t n) {
  Program p(n, 0);
  p.add(GateKind::H, {0});
  for (std::uint32_t i = 0; i + 1 < n; ++i) p.add(GateKind::CNOT, {i, i + 1});
  return p;
}

// QFT(n) applied to the basis state |input>: X on the set bits of input, then
// for j = n-1 .. 0: H(j) followed by the controlled phase U3(0, 0, pi/2^(j-k))
// (control k, target j) for k = j-1 .. 0; finally SWAP(i, n-1-i).  With qubit 0
// the least significant bit (gates.hpp:142-147) the output is
// sum_k exp(2 pi i input k / 2^n) |k> / sqrt(2^n).
inline Program gen_qft(std::uint32_t n, std::uint64_t input) {
  Program p(n, 0);
  for (std::uint32_t q = 0; q < n; ++q)
    if ((input >> q) & 1u) p.add(GateKind::X, {q});
  for (std::uint32_t j = n; j-- > 0;) {
    p.add(GateKind::H, {j});
    for (std::uint32_t k = j; k-- > 0;) {
      Gate g = make_gate(GateKind::U3, {j},
                         {0.0, 0.0, std::numbers::pi / static_cast<double>(1ull << (j - k))});
      g.controls = {k};
      p.add(std::move(g));
    }
  }
  for (std::uint32_t i = 0; i < n / 2; ++i) p.add(GateKind::SWAP, {i, n - 1 - i});
  return p;
}

// Hardware-efficient ansatz: per layer RY(theta), RZ(phi) on every qubit, then
// CNOT(q, q+1) for q < n-1; angles Rng(seed).uniform(2 pi) in program order.
inline Program gen_hea(std::uint32_t n, std::uint32_t layers, std::uint64_t seed) {
  Program p(n, 0);
  Rng rng(seed);
  for (std::uint32_t l = 0; l < layers; ++l) {
    for (std::uint32_t q = 0; q < n; ++q) {
      const double a = rng.uniform(2.0 * std::numbers::pi);
      p.add(GateKind::RY, {q}, {a});
      const double b = rng.uniform(2.0 * std::numbers::pi);
      p.add(GateKind::RZ, {q}, {b});
    }
    for (std::uint32_t q = 0; q + 1 < n; ++q) p.add(GateKind::CNOT, {q, q + 1});
  }
  return p;
}

// Config-5 observable: sum_{i<n-1} Z_i Z_{i+1} + 0.5 sum_i X_i.
inline PauliOperator hea_hamiltonian(std::uint32_t n) {
  PauliOperator h;
  for (std::uint32_t i = 0; i + 1 < n; ++i)
    h += PauliOperator::term("Z" + std::to_string(i) + " Z" + std::to_string(i + 1));
  for (std::uint32_t i = 0; i < n; ++i) h += PauliOperator::term("X" + std::to_string(i), 0.5);
  return h;
}

}  // namespace oraclegen
