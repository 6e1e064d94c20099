// qforge drop-in (B200 backend): run().
// Semantics of the reference's simulator.hpp:18-194: option validation, the
// trailing-measure fast path (evolve once, sample `shots` times from Rng(seed)
// with the c[0]-rightmost key), and the general per-shot path for mid-circuit
// measurement and classical control flow (Rng::derive(seed, shot)).
// Gate runs go to the GPU planner as single batched calls.
#pragma once

#include <cstdint>
#include <cstdlib>
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

// --- shot batches -------------------------------------------------------------
// Flat programs (no QIf / QWhile) consume a data-independent sequence of
// uniforms per shot, so many shots run together: B shots are one
// (n + log2 B)-qubit state, gates go through the planner once for all shots,
// measurements / Kraus choices are per-shot kernels (qs_batch_*), and the
// draws of shot s come from Rng::derive(seed, s) in program order -- counts
// equal the per-shot executor's (and the reference's).
struct NoiseApplication {
  const std::vector<CMatrix>* ops;
  std::vector<std::uint32_t> qubits;
};
using NoiseOf = std::function<std::vector<NoiseApplication>(const Gate&)>;
using ReadoutOf = std::function<const std::pair<double, double>*(std::uint32_t)>;  // (p01, p10) or null

// Programs with QIf / QWhile batch too: every instruction runs on the shots
// whose path reaches it (a mask); gates on a strict subset go through
// qs_batch_apply (<= 3 qubits incl. controls), measurements and Kraus steps
// skip inactive shots (negative uniform), and each shot draws from its own
// Rng::derive(seed, s) stream in its own program order.
inline bool batchable(const Program& p, std::uint64_t shots, const NoiseOf* noise) {
  if (std::getenv("QSB_NO_SHOT_BATCH")) return false;  // per-shot executor (cross-checks)
  if (shots < 2 || p.qubit_count > 22 || p.qubit_count < 1) return false;
  if (!p.is_flat() && std::getenv("QSB_NO_CF_BATCH")) return false;
  std::function<bool(const Program&, bool)> ok = [&](const Program& b, bool nested) {
    for (const auto& ins : b.body) {
      if (const auto* g = std::get_if<GateOp>(&ins)) {
        if (nested && g->gate.qubits().size() > 3) return false;
        if (noise)
          for (const auto& a : (*noise)(g->gate))
            if (a.qubits.size() > 2 || a.ops->size() > 16) return false;
      } else if (const auto* f = std::get_if<IfOp>(&ins)) {
        if (!ok(*f->then_body, true) || (f->else_body && !ok(*f->else_body, true))) return false;
      } else if (const auto* w = std::get_if<WhileOp>(&ins)) {
        if (!ok(*w->body, true)) return false;
      }
    }
    return true;
  };
  return ok(p, false);
}

// Runs shots [first, first + count) of a flat program; returns their cbits.
inline std::vector<std::vector<std::int64_t>> run_shot_batch(const Program& p, const SimOptions& opts,
                                                             std::uint64_t first, std::uint64_t count,
                                                             const NoiseOf* noise, const ReadoutOf* readout,
                                                             StateVector* last) {
  const std::uint32_t n = p.qubit_count;
  std::uint32_t b = 0;
  while ((std::uint64_t(1) << b) < count) ++b;
  // draws per shot, in program order
  std::size_t draws = 0;
  for (const auto& ins : p.body) {
    if (const auto* g = std::get_if<GateOp>(&ins)) {
      if (noise) draws += (*noise)(g->gate).size();
    } else if (const auto* m = std::get_if<MeasureOp>(&ins)) {
      draws += 1 + ((readout && (*readout)(m->qubit)) ? 1 : 0);
    }
  }
  std::vector<std::vector<double>> u(draws, std::vector<double>(count));
  for (std::uint64_t s = 0; s < count; ++s) {
    Rng r = Rng::derive(opts.seed, first + s);
    for (std::size_t d = 0; d < draws; ++d) u[d][s] = r.uniform();
  }
  qs_state_t big = nullptr;
  detail::qs_check(qs_create(n + b, 0, 40, &big));
  struct Guard {
    qs_state_t h;
    ~Guard() { qs_destroy(h); }
  } guard{big};
  detail::qs_check(qs_batch_reset(big, n));
  std::vector<std::vector<std::int64_t>> cbits(count, std::vector<std::int64_t>(p.cbit_count, 0));
  detail::GateBatch pending;
  auto drain = [&] {
    if (pending.gates.empty()) return;
    pending.rebind();
    detail::qs_check(qs_apply_circuit(big, pending.gates.data(), pending.gates.size(), opts.plan, opts.max_fused_qubits));
    pending = detail::GateBatch{};
  };
  std::size_t d = 0;
  std::vector<signed char> outc(count);
  for (const auto& ins : p.body) {
    if (const auto* g = std::get_if<GateOp>(&ins)) {
      pending.push(g->gate);
      if (!noise) continue;
      const auto apps = (*noise)(g->gate);
      if (apps.empty()) continue;
      drain();
      for (const auto& a : apps) {
        const std::size_t dim = std::size_t(1) << a.qubits.size();
        std::vector<double> flat;
        for (const auto& k : *a.ops)
          for (std::size_t r = 0; r < dim; ++r)
            for (std::size_t c = 0; c < dim; ++c) {
              flat.push_back(k(static_cast<long>(r), static_cast<long>(c)).real());
              flat.push_back(k(static_cast<long>(r), static_cast<long>(c)).imag());
            }
        detail::qs_check(qs_batch_kraus(big, n, a.qubits.data(), static_cast<std::uint32_t>(a.qubits.size()),
                                        flat.data(), static_cast<std::uint32_t>(a.ops->size()), u[d++].data(), count,
                                        nullptr));
      }
    } else if (const auto* m = std::get_if<MeasureOp>(&ins)) {
      drain();
      detail::qs_check(qs_batch_measure(big, n, m->qubit, u[d++].data(), count, outc.data()));
      const std::pair<double, double>* ro = readout ? (*readout)(m->qubit) : nullptr;
      for (std::uint64_t s = 0; s < count; ++s) {
        std::int64_t o = outc[s];
        if (ro) {
          const double flip = o ? ro->second : ro->first;
          if (u[d][s] < flip) o = o ? 0 : 1;
        }
        cbits[s][m->cbit] = o;
      }
      if (ro) ++d;
    } else if (const auto* a = std::get_if<AssignOp>(&ins)) {
      for (auto& c : cbits) c[a->cbit] = a->expr.evaluate(c);
    }
  }
  drain();
  if (last) {
    std::vector<cdouble> amps(std::size_t(1) << n);
    detail::qs_check(qs_get_amplitudes(big, reinterpret_cast<double*>(amps.data()), (count - 1) << n, amps.size()));
    *last = StateVector::from_amplitudes(n, amps);
  }
  return cbits;
}

// Shots [first, first + count) of a program with control flow (see batchable).
class ControlFlowBatch {
 public:
  ControlFlowBatch(const Program& p, const SimOptions& opts, std::uint64_t first, std::uint64_t count,
                   const NoiseOf* noise, const ReadoutOf* readout)
      : opts_(opts), noise_(noise), readout_(readout), n_(p.qubit_count), count_(count),
        cbits_(count, std::vector<std::int64_t>(p.cbit_count, 0)), outc_(count) {
    while ((std::uint64_t(1) << b_) < count) ++b_;
    rngs_.reserve(count);
    for (std::uint64_t s = 0; s < count; ++s) rngs_.push_back(Rng::derive(opts.seed, first + s));
    qs_check(qs_create(n_ + b_, 0, 40, &big_));
    qs_check(qs_batch_reset(big_, n_));
  }
  ~ControlFlowBatch() { qs_destroy(big_); }
  ControlFlowBatch(const ControlFlowBatch&) = delete;
  ControlFlowBatch& operator=(const ControlFlowBatch&) = delete;

  std::vector<std::vector<std::int64_t>> run(const Program& p, StateVector* last) {
    exec(p, std::vector<signed char>(count_, 1));
    drain();
    if (last) {
      std::vector<cdouble> amps(std::size_t(1) << n_);
      qs_check(qs_get_amplitudes(big_, reinterpret_cast<double*>(amps.data()), (count_ - 1) << n_, amps.size()));
      *last = StateVector::from_amplitudes(n_, amps);
    }
    return std::move(cbits_);
  }

 private:
  const SimOptions& opts_;
  const NoiseOf* noise_;
  const ReadoutOf* readout_;
  std::uint32_t n_, b_ = 0;
  std::uint64_t count_;
  qs_state_t big_ = nullptr;
  std::vector<Rng> rngs_;
  std::vector<std::vector<std::int64_t>> cbits_;
  std::vector<signed char> outc_;
  GateBatch pending_;

  static bool any(const std::vector<signed char>& m) {
    for (signed char x : m)
      if (x) return true;
    return false;
  }
  void drain() {
    if (pending_.gates.empty()) return;
    pending_.rebind();
    qs_check(qs_apply_circuit(big_, pending_.gates.data(), pending_.gates.size(), opts_.plan, opts_.max_fused_qubits));
    pending_ = GateBatch{};
  }
  std::vector<double> draws(const std::vector<signed char>& mask) {
    std::vector<double> u(count_, -1.0);  // negative: shot not on this path
    for (std::uint64_t s = 0; s < count_; ++s)
      if (mask[s]) u[s] = rngs_[s].uniform();
    return u;
  }
  void gate(const Gate& g, const std::vector<signed char>& mask, bool full) {
    if (full) {
      pending_.push(g);
    } else {  // a strict subset of the shots: one dense matrix on its operands
      drain();
      const CMatrix m = gate_matrix(g);
      std::vector<double> flat;
      for (long r = 0; r < m.rows(); ++r)
        for (long c = 0; c < m.cols(); ++c) {
          flat.push_back(m(r, c).real());
          flat.push_back(m(r, c).imag());
        }
      const std::vector<std::uint32_t> qs = g.qubits();
      qs_check(qs_batch_apply(big_, n_, qs.data(), static_cast<std::uint32_t>(qs.size()), flat.data(), mask.data(),
                              count_));
    }
    if (!noise_) return;
    const auto apps = (*noise_)(g);
    if (apps.empty()) return;
    drain();
    for (const auto& a : apps) {
      const std::size_t dim = std::size_t(1) << a.qubits.size();
      std::vector<double> flat;
      for (const auto& k : *a.ops)
        for (std::size_t r = 0; r < dim; ++r)
          for (std::size_t c = 0; c < dim; ++c) {
            flat.push_back(k(static_cast<long>(r), static_cast<long>(c)).real());
            flat.push_back(k(static_cast<long>(r), static_cast<long>(c)).imag());
          }
      const std::vector<double> u = draws(mask);
      qs_check(qs_batch_kraus(big_, n_, a.qubits.data(), static_cast<std::uint32_t>(a.qubits.size()), flat.data(),
                              static_cast<std::uint32_t>(a.ops->size()), u.data(), count_, nullptr));
    }
  }
  void measure(const MeasureOp& m, const std::vector<signed char>& mask) {
    drain();
    const std::vector<double> u = draws(mask);
    qs_check(qs_batch_measure(big_, n_, m.qubit, u.data(), count_, outc_.data()));
    const std::pair<double, double>* ro = readout_ ? (*readout_)(m.qubit) : nullptr;
    for (std::uint64_t s = 0; s < count_; ++s) {
      if (!mask[s]) continue;
      std::int64_t o = outc_[s];
      if (ro) {
        const double flip = o ? ro->second : ro->first;
        if (rngs_[s].uniform() < flip) o = o ? 0 : 1;
      }
      cbits_[s][m.cbit] = o;
    }
  }
  void exec(const Program& b, const std::vector<signed char>& mask) {
    bool full = true;
    for (signed char x : mask) full = full && x;
    for (const auto& ins : b.body) {
      if (const auto* g = std::get_if<GateOp>(&ins)) {
        gate(g->gate, mask, full);
      } else if (const auto* m = std::get_if<MeasureOp>(&ins)) {
        measure(*m, mask);
      } else if (const auto* f = std::get_if<IfOp>(&ins)) {
        drain();
        std::vector<signed char> yes(count_, 0), no(count_, 0);
        for (std::uint64_t s = 0; s < count_; ++s)
          if (mask[s]) (f->condition.evaluate(cbits_[s]) != 0 ? yes : no)[s] = 1;
        if (any(yes)) exec(*f->then_body, yes);
        if (f->else_body && any(no)) exec(*f->else_body, no);
      } else if (const auto* w = std::get_if<WhileOp>(&ins)) {
        drain();
        std::vector<signed char> cur = mask;
        for (std::uint64_t iters = 0;;) {
          for (std::uint64_t s = 0; s < count_; ++s)
            if (cur[s] && w->condition.evaluate(cbits_[s]) == 0) cur[s] = 0;  // this shot leaves the loop
          if (!any(cur)) break;
          if (++iters > opts_.max_while_iterations)
            throw NonTerminationGuard("QWhile exceeded " + std::to_string(opts_.max_while_iterations) + " iterations");
          exec(*w->body, cur);
          drain();
        }
      } else if (const auto* a = std::get_if<AssignOp>(&ins)) {
        for (std::uint64_t s = 0; s < count_; ++s)
          if (mask[s]) cbits_[s][a->cbit] = a->expr.evaluate(cbits_[s]);
      }
    }
  }
  static void qs_check(int rc) { detail::qs_check(rc); }
};

// Shots in batches sized to ~2 GiB of device memory.
inline std::vector<std::string> run_batched_keys(const Program& p, const SimOptions& opts, std::uint64_t shots,
                                                 const NoiseOf* noise, const ReadoutOf* readout, StateVector* last) {
  const std::uint32_t n = p.qubit_count;
  const std::uint64_t cap = std::max<std::uint64_t>(2, (std::uint64_t(1) << 27) >> n);  // 2^27 amplitudes
  std::vector<std::string> keys;
  keys.reserve(shots);
  for (std::uint64_t first = 0; first < shots; first += cap) {
    const std::uint64_t count = std::min(cap, shots - first);
    const bool tail = first + count == shots;
    std::vector<std::vector<std::int64_t>> cb;
    if (p.is_flat()) cb = run_shot_batch(p, opts, first, count, noise, readout, tail ? last : nullptr);
    else cb = ControlFlowBatch(p, opts, first, count, noise, readout).run(p, tail ? last : nullptr);
    for (auto& c : cb) keys.push_back(cbit_key(c));
  }
  return keys;
}

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
  if (detail::batchable(p, shots, nullptr)) {
    StateVector last(p.qubit_count);
    for (auto& k : detail::run_batched_keys(p, opts, shots, nullptr, nullptr, &last)) ++result.counts[k];
    result.final_state = std::move(last);
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
