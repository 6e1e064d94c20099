// qforge drop-in (B200 backend): run().
// Semantics of the reference's simulator.hpp:18-194: option validation, the
// trailing-measure fast path (evolve once, sample `shots` times from Rng(seed)
// with the c[0]-rightmost key), and the general per-shot path for mid-circuit
// measurement and classical control flow (Rng::derive(seed, shot)).
// Gate runs go to the GPU planner as single batched calls.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "qforge/circuit.hpp"
#include "qforge/error.hpp"
#include "qforge/fusion.hpp"
#include "qforge/rng.hpp"
#include "qforge/statevector.hpp"

namespace qforge {

struct SimOptions {
  std::uint64_t parallel_threshold = 1ull << 14;  // accepted; no effect on the GPU
  bool fusion_enabled = false;                    // see `plan`
  std::uint32_t max_fused_qubits = 3;
  std::uint64_t seed = 0;
  int workers = 0;                                // accepted; no effect on the GPU
  std::uint64_t max_while_iterations = 1'000'000;
  // B200 planner: QS_PLAN_DEFAULT = shared-memory tile passes; set
  // QS_PLAN_DENSE_FUSION to execute the reference's fuse_circuit blocks.
  std::uint32_t plan = QS_PLAN_DEFAULT;

  KernelOptions kernel_options() const { return KernelOptions{parallel_threshold, workers}; }
  void validate() const {
    if (parallel_threshold < 1) throw ValidationError("parallel_threshold must be at least 1");
    if (max_fused_qubits < 1 || max_fused_qubits > 5) throw ValidationError("max_fused_qubits must be in [1, 5]");
    if (workers < 0) throw ValidationError("workers must be non-negative");
  }
};

struct RunResult {
  std::map<std::string, std::uint64_t> counts;  // c[0] rightmost
  std::optional<StateVector> final_state;
};

namespace detail {

inline std::string cbit_key(const std::vector<std::int64_t>& cbits) {
  std::string key(cbits.size(), '0');
  for (std::size_t i = 0; i < cbits.size(); ++i)
    if (cbits[i]) key[cbits.size() - 1 - i] = '1';
  return key;
}

inline bool trailing_measure_form(const Program& p) {
  bool measuring = false;
  for (const auto& ins : p.body) {
    if (std::holds_alternative<GateOp>(ins)) {
      if (measuring) return false;
    } else if (std::holds_alternative<MeasureOp>(ins)) {
      measuring = true;
    } else {
      return false;
    }
  }
  return true;
}

// Per-shot executor for programs with mid-circuit measurement / control flow.
// Optional hooks (noise.hpp): gates for which `noisy` holds run one at a time
// followed by `after_gate`; the others keep batching into planned runs;
// `readout` maps each collapsed outcome to the recorded bit.
class ShotExecutor {
 public:
  using GateHook = std::function<void(const Gate&, StateVector&, Rng&)>;
  using ReadoutHook = std::function<std::int64_t(std::uint32_t, std::int64_t, Rng&)>;

  // `sv` is reused across shots (reset to |0...0> here): no allocation per shot.
  ShotExecutor(const Program& p, const SimOptions& o, Rng rng, StateVector& sv)
      : opts_(o), rng_(std::move(rng)), sv_(sv), cbits_(p.cbit_count, 0) {
    sv_.reset_to_zero();
  }

  void set_gate_hook(std::function<bool(const Gate&)> noisy, GateHook after) {
    noisy_ = std::move(noisy);
    after_ = std::move(after);
  }
  void set_readout(ReadoutHook r) { readout_ = std::move(r); }

  void exec(const Program& p) {
    std::vector<Gate> pending;
    auto drain = [&] {
      if (pending.empty()) return;
      sv_.apply_gates(pending, opts_.plan, opts_.max_fused_qubits);
      pending.clear();
    };
    for (const auto& ins : p.body) {
      if (const auto* g = std::get_if<GateOp>(&ins)) {
        if (noisy_ && noisy_(g->gate)) {
          drain();
          sv_.apply_gate(g->gate);
          after_(g->gate, sv_, rng_);
        } else {
          pending.push_back(g->gate);
        }
        continue;
      }
      drain();
      if (const auto* m = std::get_if<MeasureOp>(&ins)) {
        const std::int64_t o = sv_.measure_collapse(m->qubit, rng_.uniform());
        cbits_[m->cbit] = readout_ ? readout_(m->qubit, o, rng_) : o;
      } else if (const auto* f = std::get_if<IfOp>(&ins)) {
        if (f->condition.evaluate(cbits_) != 0) exec(*f->then_body);
        else if (f->else_body) exec(*f->else_body);
      } else if (const auto* w = std::get_if<WhileOp>(&ins)) {
        std::uint64_t iters = 0;
        while (w->condition.evaluate(cbits_) != 0) {
          if (++iters > opts_.max_while_iterations)
            throw NonTerminationGuard("QWhile exceeded " + std::to_string(opts_.max_while_iterations) + " iterations");
          exec(*w->body);
        }
      } else if (const auto* a = std::get_if<AssignOp>(&ins)) {
        cbits_[a->cbit] = a->expr.evaluate(cbits_);
      }
    }
    drain();
  }
  StateVector& state() { return sv_; }
  const std::vector<std::int64_t>& cbits() const { return cbits_; }

 private:
  const SimOptions& opts_;
  Rng rng_;
  StateVector& sv_;
  std::vector<std::int64_t> cbits_;
  std::function<bool(const Gate&)> noisy_;
  GateHook after_;
  ReadoutHook readout_;
};

}  // namespace detail

inline RunResult run(const Program& p, const SimOptions& opts = {}, std::uint64_t shots = 0) {
  opts.validate();
  validate_or_throw(p);
  RunResult result;
  if (detail::trailing_measure_form(p)) {
    StateVector sv(p.qubit_count);
    std::vector<Gate> gates;
    std::vector<MeasureOp> measures;
    for (const auto& ins : p.body) {
      if (const auto* g = std::get_if<GateOp>(&ins)) gates.push_back(g->gate);
      else measures.push_back(std::get<MeasureOp>(ins));
    }
    const std::uint32_t plan = (opts.fusion_enabled && opts.plan == QS_PLAN_DENSE_FUSION) ? QS_PLAN_DENSE_FUSION
                                                                                           : opts.plan;
    if (!gates.empty()) sv.apply_gates(gates, plan, opts.max_fused_qubits);
    if (shots > 0) {
      if (measures.empty()) {
        result.counts[std::string(p.cbit_count, '0')] += shots;
      } else {
        // Rng(seed) draws + exact serial-equivalent sampler, on the device
        std::vector<std::uint64_t> idx(shots);
        detail::qs_check(qs_sample_seeded(sv.handle(), opts.seed, shots, 1, idx.data()));
        std::map<std::uint64_t, std::uint64_t> per_key;
        for (auto b : idx) {
          std::uint64_t key = 0;
          for (const auto& m : measures)
            if ((b >> m.qubit) & 1) key |= std::uint64_t(1) << m.cbit;
          ++per_key[key];
        }
        for (const auto& [k, c] : per_key) {
          std::string s(p.cbit_count, '0');
          for (std::uint32_t b = 0; b < p.cbit_count; ++b)
            if ((k >> b) & 1) s[p.cbit_count - 1 - b] = '1';
          result.counts[s] += c;
        }
      }
    }
    result.final_state = std::move(sv);
    return result;
  }
  const std::uint64_t runs = shots > 0 ? shots : 1;
  StateVector sv(p.qubit_count);
  for (std::uint64_t s = 0; s < runs; ++s) {
    detail::ShotExecutor ex(p, opts, Rng::derive(opts.seed, s), sv);
    ex.exec(p);
    if (shots > 0) ++result.counts[detail::cbit_key(ex.cbits())];
  }
  result.final_state = std::move(sv);
  return result;
}

}  // namespace qforge
