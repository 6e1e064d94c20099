// qforge drop-in (B200 backend): amplitudes of selected basis states.
//
// Same names, signatures and error behaviour as the reference's
// pathsum.hpp:16-459 (single_amplitude, plan_cut, CutPlan, partial_amplitude,
// BudgetExceeded).  The values come from the GPU:
//   * single_amplitude: the program runs as tile passes on a device state
//     vector and one amplitude is read (the reference sums Feynman paths on
//     the host).  The path-count estimate and budget check are kept so callers
//     see the reference's exceptions.
//   * partial_amplitude: the cut method with every branch assignment batched as
//     extra qubits of two half-size device states (qs_partial_amplitude,
//     csrc/pathsum.cpp), one GPU reduction per target over the branches.
//   * plan_cut: host combinatorics (balanced bipartition, few crossing gates).
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <string_view>
#include <vector>

#include "qforge/circuit.hpp"
#include "qforge/error.hpp"
#include "qforge/statevector.hpp"

namespace qforge {

// error.hpp:43-48: a path-sum evaluation would branch beyond the caller's budget.
class BudgetExceeded : public Error {
 public:
  BudgetExceeded(const std::string& msg, std::uint64_t estimated_paths) : Error(msg), estimated_paths(estimated_paths) {}
  std::uint64_t estimated_paths;
};

inline constexpr std::uint64_t kDefaultPathBudget = 1ull << 22;

namespace detail {

// A gate as the path evaluator branches on it: one target, the controls it
// introduces path variables for (CNOT/CZ: one, TOFFOLI: two, SWAP: three
// CNOTs; extra controls carry over).
struct PathGate {
  std::uint32_t target = 0;
  std::vector<std::uint32_t> controls;
};

inline void require_gates_only(const Program& p, const char* what) {
  for (const auto& ins : p.body) {
    if (std::holds_alternative<GateOp>(ins)) continue;
    if (std::holds_alternative<MeasureOp>(ins))
      throw UnsupportedError(std::string(what) + " is defined for measurement-free programs");
    throw FlatCircuitRequired(std::string(what) + " requires a flat program");
  }
}

inline std::vector<PathGate> normalize_for_paths(const Program& p) {
  require_gates_only(p, "path-sum evaluation");
  std::vector<PathGate> out;
  for (const auto& ins : p.body) {
    const Gate& g = std::get<GateOp>(ins).gate;
    auto with = [&](std::initializer_list<std::uint32_t> more) {
      std::vector<std::uint32_t> c = g.controls;
      c.insert(c.end(), more);
      return c;
    };
    switch (g.kind) {
      case GateKind::I: break;
      case GateKind::CNOT:
      case GateKind::CZ: out.push_back({g.targets[1], with({g.targets[0]})}); break;
      case GateKind::TOFFOLI: out.push_back({g.targets[2], with({g.targets[0], g.targets[1]})}); break;
      case GateKind::SWAP:
        out.push_back({g.targets[1], with({g.targets[0]})});
        out.push_back({g.targets[0], with({g.targets[1]})});
        out.push_back({g.targets[1], with({g.targets[0]})});
        break;
      case GateKind::Custom:
        if (g.targets.size() != 1) throw UnsupportedError("path-sum evaluation supports custom gates on one target only");
        out.push_back({g.targets[0], g.controls});
        break;
      default: out.push_back({g.targets[0], g.controls}); break;
    }
  }
  return out;
}

inline std::uint64_t path_count_estimate(const std::vector<PathGate>& gates) {
  std::uint64_t bits = 0;
  for (const auto& g : gates) bits += g.controls.size();
  return bits > 62 ? UINT64_MAX : (std::uint64_t{1} << bits);
}

// Rightmost character is qubit 0 -> basis index (pathsum.hpp:165-178).
inline std::uint64_t parse_bitstring_index(std::string_view bits, std::uint32_t n) {
  if (bits.size() != n)
    throw ValidationError("target bitstring length " + std::to_string(bits.size()) + " does not match " +
                          std::to_string(n) + " qubits");
  std::uint64_t idx = 0;
  for (std::uint32_t q = 0; q < n; ++q) {
    const char c = bits[n - 1 - q];
    if (c != '0' && c != '1') throw ValidationError("target bitstring must contain only 0/1");
    if (c == '1') idx |= std::uint64_t{1} << q;
  }
  return idx;
}

inline void check_cuttable_gate(const Gate& g) {
  if (!g.controls.empty()) throw UnsupportedError("cut planning expects gates without extra controls");
  if (g.targets.size() == 1 || g.kind == GateKind::CNOT || g.kind == GateKind::CZ) return;
  throw UnsupportedError(std::string("cut planning cannot handle ") + gate_name(g.kind));
}

}  // namespace detail

inline cdouble single_amplitude(const Program& p, std::string_view target,
                                std::uint64_t path_budget = kDefaultPathBudget) {
  validate_or_throw(p);
  const auto gates = detail::normalize_for_paths(p);
  const std::uint64_t idx = detail::parse_bitstring_index(target, p.qubit_count);
  const std::uint64_t estimate = detail::path_count_estimate(gates);
  if (estimate > path_budget)
    throw BudgetExceeded("path count " + (estimate == UINT64_MAX ? std::string("overflows") : std::to_string(estimate)) +
                             " exceeds budget " + std::to_string(path_budget),
                         estimate);
  StateVector sv(p.qubit_count);
  std::vector<Gate> body;
  for (const auto& ins : p.body) body.push_back(std::get<GateOp>(ins).gate);
  if (!body.empty()) sv.apply_gates(body);
  return sv.amplitude(idx);
}

struct CutPlan {
  std::vector<std::uint32_t> block_a;       // sorted, ceil(n/2) qubits
  std::vector<std::uint32_t> block_b;       // sorted, floor(n/2)
  std::vector<std::size_t> crossing_gates;  // body indices, ascending
  std::uint64_t branch_count = 1;           // 2^|crossing_gates|
};

inline CutPlan plan_cut(const Program& p) {
  validate_or_throw(p);
  detail::require_gates_only(p, "cut planning");
  const std::uint32_t n = p.qubit_count;
  if (n < 2) throw ValidationError("cut planning needs at least 2 qubits");
  std::vector<std::pair<std::uint32_t, std::uint32_t>> pairs;
  for (const auto& ins : p.body) {
    const Gate& g = std::get<GateOp>(ins).gate;
    detail::check_cuttable_gate(g);
    if (g.targets.size() == 2) pairs.push_back({g.targets[0], g.targets[1]});
  }
  auto crossings = [&](std::uint64_t mask) {
    std::size_t c = 0;
    for (const auto& [a, b] : pairs) c += ((mask >> a) ^ (mask >> b)) & 1;
    return c;
  };
  const std::uint32_t size_a = (n + 1) / 2;
  std::uint64_t mask = (std::uint64_t{1} << size_a) - 1;
  if (n <= 12) {  // exhaustive: first subset with the fewest crossings
    std::size_t best = SIZE_MAX;
    for (std::uint64_t m = 0; m < (std::uint64_t{1} << n); ++m)
      if (static_cast<std::uint32_t>(__builtin_popcountll(m)) == size_a && crossings(m) < best) {
        best = crossings(m);
        mask = m;
      }
  } else {  // first-improving swaps of one qubit across the cut
    std::size_t cur = crossings(mask);
    for (bool moved = true; moved;) {
      moved = false;
      for (std::uint32_t a = 0; a < n && !moved; ++a) {
        if (!((mask >> a) & 1)) continue;
        for (std::uint32_t b = 0; b < n && !moved; ++b) {
          if ((mask >> b) & 1) continue;
          const std::uint64_t m2 = (mask & ~(std::uint64_t{1} << a)) | (std::uint64_t{1} << b);
          const std::size_t c = crossings(m2);
          if (c < cur) {
            cur = c;
            mask = m2;
            moved = true;
          }
        }
      }
    }
  }
  CutPlan plan;
  for (std::uint32_t q = 0; q < n; ++q) ((mask >> q) & 1 ? plan.block_a : plan.block_b).push_back(q);
  std::size_t i = 0;
  for (const auto& ins : p.body) {
    const Gate& g = std::get<GateOp>(ins).gate;
    if (g.targets.size() == 2 && (((mask >> g.targets[0]) ^ (mask >> g.targets[1])) & 1)) plan.crossing_gates.push_back(i);
    ++i;
  }
  plan.branch_count = plan.crossing_gates.size() >= 63 ? UINT64_MAX : (std::uint64_t{1} << plan.crossing_gates.size());
  return plan;
}

inline std::map<std::string, cdouble> partial_amplitude(const Program& p, const CutPlan& plan,
                                                        const std::vector<std::string>& targets,
                                                        std::uint64_t branch_budget = kDefaultPathBudget) {
  validate_or_throw(p);
  const std::uint32_t n = p.qubit_count;
  std::vector<int> side(n, -1);
  for (auto q : plan.block_a) {
    if (q >= n) throw ValidationError("cut plan qubit out of range");
    side[q] = 0;
  }
  for (auto q : plan.block_b) {
    if (q >= n || side[q] != -1) throw ValidationError("cut plan blocks must partition the qubits");
    side[q] = 1;
  }
  for (std::uint32_t q = 0; q < n; ++q)
    if (side[q] == -1) throw ValidationError("cut plan blocks must partition the qubits");
  if (plan.branch_count > branch_budget)
    throw BudgetExceeded("branch count " + std::to_string(plan.branch_count) + " exceeds budget " +
                             std::to_string(branch_budget),
                         plan.branch_count);
  std::vector<std::size_t> crossing;
  std::vector<Gate> body;
  for (const auto& ins : p.body) {
    const GateOp* op = std::get_if<GateOp>(&ins);
    if (!op) throw UnsupportedError("partial amplitude expects a gates-only program");
    detail::check_cuttable_gate(op->gate);
    if (op->gate.targets.size() == 2 && side[op->gate.targets[0]] != side[op->gate.targets[1]])
      crossing.push_back(body.size());
    body.push_back(op->gate);
  }
  if (crossing != plan.crossing_gates) throw ValidationError("cut plan does not match the program's gates");
  std::map<std::string, cdouble> out;
  std::vector<std::string> keys;
  std::vector<std::uint64_t> idx;
  std::set<std::string_view> seen;
  for (const auto& t : targets) {
    out[t] = cdouble(0);
    const std::uint64_t b = detail::parse_bitstring_index(t, n);
    if (seen.insert(t).second) {
      keys.push_back(t);
      idx.push_back(b);
    }
  }
  if (keys.empty()) return out;
  detail::GateBatch batch;
  for (const auto& g : body) batch.push(g);
  batch.rebind();
  std::vector<double> res(2 * keys.size());
  detail::qs_check(qs_partial_amplitude(n, batch.gates.data(), batch.gates.size(), plan.block_a.data(),
                                        static_cast<std::uint32_t>(plan.block_a.size()), idx.data(), idx.size(), 0, 0,
                                        res.data()));
  for (std::size_t j = 0; j < keys.size(); ++j) out[keys[j]] = cdouble(res[2 * j], res[2 * j + 1]);
  return out;
}

}  // namespace qforge
