// qforge drop-in (B200 backend): StateVector with its amplitudes in HBM.
//
// Same interface as the reference's StateVector (statevector.hpp:134-264):
// value semantics (copies are device-to-device clones), the 30-qubit cap,
// apply_gate / apply_matrix / reductions / measurement, and host spans via
// amplitudes().  Every amplitude-touching call runs in libqsb.so (C ABI,
// include/qsb.h); the host holds only a lazily synchronised mirror for the
// span accessors.  KernelOptions is accepted for source compatibility; its
// OpenMP knobs have no meaning on the GPU.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <vector>

#include "qforge/circuit.hpp"
#include "qforge/error.hpp"
#include "qforge/gates.hpp"
#include "qforge/linalg.hpp"
#include "qsb.h"

namespace qforge {

struct KernelOptions {
  std::uint64_t parallel_threshold = 1ull << 14;
  int workers = 0;
};

namespace detail {

// Source-compatibility helpers for code that used the reference's internals
// (statevector.hpp:42-64, 110-130).  Host-side only: the GPU kernels use the
// same zero-insertion indexing (csrc/kernels.cu `deposit`) and their own
// fixed-order reductions.
struct GroupIndexer {
  std::vector<std::uint32_t> slots;
  std::size_t force_mask = 0;
  void add_target(std::uint32_t q) { slots.push_back(q); }
  void add_control(std::uint32_t q) {
    slots.push_back(q);
    force_mask |= std::size_t(1) << q;
  }
  void finish() { std::sort(slots.begin(), slots.end()); }
  std::size_t groups(std::uint32_t n) const { return std::size_t(1) << (n - slots.size()); }
  std::size_t base(std::size_t g) const {
    for (auto p : slots) g = ((g >> p) << (p + 1)) | (g & ((std::size_t(1) << p) - 1));
    return g | force_mask;
  }
};

template <class F>
double chunked_sum(std::size_t size, const KernelOptions&, F&& f) {
  constexpr std::size_t kChunk = 4096;
  double total = 0.0;
  for (std::size_t lo = 0; lo < size; lo += kChunk) {
    double s = 0.0;
    for (std::size_t i = lo; i < std::min(size, lo + kChunk); ++i) s += f(i);
    total += s;
  }
  return total;
}

// Gate -> flat C ABI record.  `storage` keeps a custom matrix alive.
inline qs_gate to_qs(const Gate& g, std::vector<double>& storage) {
  qs_gate r{};
  r.kind = static_cast<int32_t>(g.kind);
  r.dagger = g.dagger ? 1 : 0;
  if (g.targets.size() > QS_MAX_TARGETS || g.controls.size() > QS_MAX_CONTROLS)
    throw ValidationError("gate has more operands than the backend supports");
  r.num_targets = static_cast<uint32_t>(g.targets.size());
  r.num_controls = static_cast<uint32_t>(g.controls.size());
  std::copy(g.targets.begin(), g.targets.end(), r.targets);
  std::copy(g.controls.begin(), g.controls.end(), r.controls);
  for (std::size_t k = 0; k < g.params.size() && k < 3; ++k) r.params[k] = g.params[k];
  if (g.kind == GateKind::Custom && g.custom) {
    const CMatrix& m = *g.custom;
    storage.resize(static_cast<std::size_t>(2 * m.rows() * m.cols()));
    std::size_t k = 0;
    for (Eigen::Index i = 0; i < m.rows(); ++i)
      for (Eigen::Index j = 0; j < m.cols(); ++j) {
        storage[k++] = m(i, j).real();
        storage[k++] = m(i, j).imag();
      }
    r.matrix = storage.data();
  }
  return r;
}

// A batch of gates in C ABI form (matrices owned by the batch).
struct GateBatch {
  std::vector<qs_gate> gates;
  std::vector<std::vector<double>> mats;
  void push(const Gate& g) {
    mats.emplace_back();
    gates.push_back(to_qs(g, mats.back()));
  }
  void rebind() {
    for (std::size_t i = 0; i < gates.size(); ++i)
      if (gates[i].kind == QS_CUSTOM) gates[i].matrix = mats[i].data();
  }
};

struct Handle {
  qs_state_t h = nullptr;
  ~Handle() {
    if (h) qs_destroy(h);
  }
};

inline int default_device() { return 0; }

}  // namespace detail

class StateVector {
 public:
  explicit StateVector(std::uint32_t num_qubits) : n_(num_qubits) {
    if (num_qubits > 30) throw ValidationError("state vector limited to 30 qubits");
    h_ = std::make_shared<detail::Handle>();
    detail::qs_check(qs_create(num_qubits, detail::default_device(), 30, &h_->h));
  }

  StateVector(const StateVector& o) : n_(o.n_) {
    o.flush();
    h_ = std::make_shared<detail::Handle>();
    detail::qs_check(qs_clone(o.h_->h, &h_->h));
  }
  StateVector& operator=(const StateVector& o) {
    if (this != &o) {
      StateVector tmp(o);
      *this = std::move(tmp);
    }
    return *this;
  }
  StateVector(StateVector&&) noexcept = default;
  StateVector& operator=(StateVector&&) noexcept = default;

  static StateVector from_amplitudes(std::uint32_t n, std::vector<cdouble> amps) {
    StateVector sv(n);
    if (amps.size() != sv.dimension()) throw ValidationError("amplitude count does not match qubit count");
    detail::qs_check(qs_set_amplitudes(sv.h_->h, reinterpret_cast<const double*>(amps.data()), 0, amps.size()));
    return sv;
  }

  std::uint32_t num_qubits() const { return n_; }
  std::size_t dimension() const { return std::size_t(1) << n_; }

  std::span<const cdouble> amplitudes() const {
    pull();
    return host_;
  }
  std::span<cdouble> mutable_amplitudes() {
    pull();
    dirty_ = true;
    return host_;
  }
  cdouble amplitude(std::size_t i) const {
    if (mirror_valid_ || dirty_) return host_[i];
    cdouble a;
    detail::qs_check(qs_get_amplitudes(h_->h, reinterpret_cast<double*>(&a), i, 1));
    return a;
  }

  double norm_squared(const KernelOptions& = {}) const {
    flush();
    double v = 0;
    detail::qs_check(qs_norm2(h_->h, &v));
    return v;
  }
  // Back to |0...0> on the device (extension: per-shot executors reuse one state).
  void reset_to_zero() {
    device_op();
    detail::qs_check(qs_reset(h_->h));
  }
  void scale(cdouble f) {
    device_op();
    detail::qs_check(qs_scale(h_->h, f.real(), f.imag()));
  }

  void apply_gate(const Gate& g, const KernelOptions& = {}) {
    device_op();
    std::vector<double> m;
    const qs_gate r = detail::to_qs(g, m);
    detail::qs_check(qs_apply_gate(h_->h, &r));
  }

  // A run of gates as one planned call (shared-memory tile passes).
  void apply_gates(std::span<const Gate> gates, std::uint32_t plan = QS_PLAN_DEFAULT, std::uint32_t max_fused = 3) {
    device_op();
    detail::GateBatch b;
    for (const auto& g : gates) b.push(g);
    b.rebind();
    detail::qs_check(qs_apply_circuit(h_->h, b.gates.data(), b.gates.size(), plan, max_fused));
  }

  void apply_matrix(std::span<const std::uint32_t> targets, const CMatrix& m,
                    std::span<const std::uint32_t> controls = {}, const KernelOptions& = {}) {
    const std::size_t k = targets.size();
    if (k + controls.size() > n_) throw ValidationError("apply_matrix: too many operands");
    if (m.rows() != (Eigen::Index(1) << k) || m.cols() != (Eigen::Index(1) << k))
      throw ValidationError("apply_matrix: matrix does not match target count");
    device_op();
    std::vector<double> flat(static_cast<std::size_t>(2 * m.rows() * m.cols()));
    std::size_t q = 0;
    for (Eigen::Index i = 0; i < m.rows(); ++i)
      for (Eigen::Index j = 0; j < m.cols(); ++j) {
        flat[q++] = m(i, j).real();
        flat[q++] = m(i, j).imag();
      }
    detail::qs_check(qs_apply_matrix(h_->h, targets.data(), static_cast<uint32_t>(k), flat.data(), controls.data(),
                                     static_cast<uint32_t>(controls.size())));
  }

  double probability_of_one(std::uint32_t q, const KernelOptions& = {}) const {
    flush();
    double v = 0;
    detail::qs_check(qs_prob_one(h_->h, q, &v));
    return v;
  }

  std::vector<double> probabilities(std::span<const std::uint32_t> qubits, const KernelOptions& = {}) const {
    if (qubits.empty()) throw ValidationError("probabilities: empty qubit subset");
    for (auto q : qubits)
      if (q >= n_) throw ValidationError("probabilities: qubit out of range");
    flush();
    std::vector<double> out(std::size_t(1) << qubits.size());
    detail::qs_check(qs_probs(h_->h, qubits.data(), static_cast<uint32_t>(qubits.size()), out.data()));
    return out;
  }
  std::vector<double> probabilities(const KernelOptions& = {}) const {
    flush();
    std::vector<double> out(dimension());
    detail::qs_check(qs_probs_full(h_->h, out.data(), 0, out.size()));
    return out;
  }

  int measure_collapse(std::uint32_t q, double u, const KernelOptions& = {}) {
    device_op();
    int outcome = 0;
    detail::qs_check(qs_measure_collapse(h_->h, q, u, &outcome));
    return outcome;
  }
  void collapse(std::uint32_t q, int outcome, double prob, const KernelOptions& = {}) {
    if (prob <= 0.0) throw Error("collapse onto a zero-probability outcome");
    device_op();
    detail::qs_check(qs_collapse(h_->h, q, outcome, prob));
  }

  // Backend access (sampling, expectation).
  qs_state_t handle() const {
    flush();
    return h_->h;
  }
  void invalidate_mirror() { mirror_valid_ = false; }

 private:
  void flush() const {  // host edits -> device
    if (!dirty_) return;
    detail::qs_check(qs_set_amplitudes(h_->h, reinterpret_cast<const double*>(host_.data()), 0, host_.size()));
    dirty_ = false;
  }
  void pull() const {  // device -> host mirror
    if (mirror_valid_ || dirty_) return;
    host_.resize(dimension());
    detail::qs_check(qs_get_amplitudes(h_->h, reinterpret_cast<double*>(host_.data()), 0, host_.size()));
    mirror_valid_ = true;
  }
  void device_op() {
    flush();
    mirror_valid_ = false;
  }

  std::uint32_t n_;
  std::shared_ptr<detail::Handle> h_;
  mutable std::vector<cdouble> host_;
  mutable bool mirror_valid_ = false;
  mutable bool dirty_ = false;
};

// Cumulative |a|^2 sampler (statevector.hpp:542-570).  The cumulative array is
// produced on the GPU by the serial-equivalent exact scan (bit-identical to
// the reference's serial loop); draws are upper-bound searches on u * total.
class BasisSampler {
 public:
  explicit BasisSampler(const StateVector& sv) : cum_(sv.dimension()) {
    detail::qs_check(qs_cumulative(sv.handle(), cum_.data(), &total_));
  }
  std::size_t sample(double u) const {
    const double target = u * total_;
    std::size_t lo = 0, hi = cum_.size() - 1;
    while (lo < hi) {
      const std::size_t mid = (lo + hi) / 2;
      if (cum_[mid] > target) hi = mid;
      else lo = mid + 1;
    }
    return lo;
  }

 private:
  std::vector<double> cum_;
  double total_ = 0;
};

}  // namespace qforge
