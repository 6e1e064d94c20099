// qforge drop-in (B200 backend): gate fusion.
// fuse_circuit keeps the reference's semantics exactly (fusion.hpp:108-133):
// greedy dependency-graph fusion into Custom blocks of <= max_fused_qubits
// qubits, measurements pass through.  The fusion itself runs in libqsb
// (csrc/fusion.cpp, pinned block-for-block against the reference by the CPU
// tests).  run() does not need it: by default the GPU planner fuses into
// shared-memory tile passes, which is both more aggressive and cheaper.
#pragma once

#include <cstdint>
#include <vector>

#include "qforge/circuit.hpp"
#include "qforge/error.hpp"
#include "qforge/statevector.hpp"

namespace qforge {

namespace detail {
inline std::vector<Gate> fuse_run(const std::vector<Gate>& run, std::uint32_t nq, std::uint32_t k) {
  GateBatch b;
  for (const auto& g : run) b.push(g);
  b.rebind();
  qs_fused_t f = nullptr;
  qs_check(qs_fuse(b.gates.data(), b.gates.size(), nq, k, &f));
  std::vector<Gate> out;
  const uint64_t count = qs_fused_count(f);
  for (uint64_t i = 0; i < count; ++i) {
    qs_gate r{};
    qs_fused_get(f, i, &r);
    Gate g;
    g.kind = static_cast<GateKind>(r.kind);
    g.dagger = r.dagger != 0;
    g.targets.assign(r.targets, r.targets + r.num_targets);
    g.controls.assign(r.controls, r.controls + r.num_controls);
    if (g.kind == GateKind::Custom) {
      const Eigen::Index dim = Eigen::Index(1) << r.num_targets;
      CMatrix m(dim, dim);
      for (Eigen::Index a = 0; a < dim; ++a)
        for (Eigen::Index c = 0; c < dim; ++c)
          m(a, c) = cdouble(r.matrix[2 * (a * dim + c)], r.matrix[2 * (a * dim + c) + 1]);
      g.custom = std::make_shared<const CMatrix>(std::move(m));
    } else {
      g.params.assign(r.params, r.params + gate_param_arity(g.kind));
    }
    out.push_back(std::move(g));
  }
  qs_fused_free(f);
  return out;
}
}  // namespace detail

inline Program fuse_circuit(const Program& p, std::uint32_t max_fused_qubits = 3) {
  if (!p.is_flat()) throw FlatCircuitRequired("gate fusion requires a flat program");
  if (max_fused_qubits < 1) throw ValidationError("max_fused_qubits must be at least 1");
  Program out(p.qubit_count, p.cbit_count);
  std::vector<Gate> run;
  auto flush = [&] {
    if (run.empty()) return;
    for (auto& g : detail::fuse_run(run, p.qubit_count, max_fused_qubits)) out.add(std::move(g));
    run.clear();
  };
  for (const auto& ins : p.body) {
    if (const auto* g = std::get_if<GateOp>(&ins)) {
      run.push_back(g->gate);
    } else {
      flush();
      out.body.push_back(ins);
    }
  }
  flush();
  return out;
}

}  // namespace qforge
