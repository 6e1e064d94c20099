#include "gates.hpp"

#include <algorithm>
#include <cmath>
#include <string>

namespace qsb {

namespace {

const double kPi = 3.14159265358979323846;

uint32_t target_arity(int kind) {
  switch (kind) {
    case QS_CNOT:
    case QS_CZ:
    case QS_SWAP: return 2;
    case QS_TOFFOLI: return 3;
    case QS_CUSTOM: return 0;
    default: return 1;
  }
}

const char* gate_name(int k) {
  static const char* names[] = {"I",  "X",  "Y",  "Z",  "H",    "S",    "T",    "RX",
                                "RY", "RZ", "U3", "CNOT", "CZ", "SWAP", "TOFFOLI", "CUSTOM"};
  return (k >= 0 && k <= QS_CUSTOM) ? names[k] : "?";
}

}  // namespace

int base_matrix(const qs_gate& g, std::vector<cd>& m) {
  const cd i1(0, 1);
  int dim;
  if (g.kind == QS_CUSTOM) {
    dim = 1 << g.num_targets;
    m.assign(static_cast<size_t>(dim) * dim, cd(0));
    for (int k = 0; k < dim * dim; ++k) m[k] = cd(g.matrix[2 * k], g.matrix[2 * k + 1]);
  } else {
    dim = 1 << target_arity(g.kind);
    m.assign(static_cast<size_t>(dim) * dim, cd(0));
    const double* p = g.params;
    auto set2 = [&](cd a, cd b, cd c, cd d) {
      m[0] = a;
      m[1] = b;
      m[2] = c;
      m[3] = d;
    };
    switch (g.kind) {
      case QS_I: set2(1, 0, 0, 1); break;
      case QS_X: set2(0, 1, 1, 0); break;
      case QS_Y: set2(0, -i1, i1, 0); break;
      case QS_Z: set2(1, 0, 0, -1); break;
      case QS_H: {
        const double s = 1.0 / std::sqrt(2.0);
        set2(s, s, s, -s);
        break;
      }
      case QS_S: set2(1, 0, 0, i1); break;
      case QS_T: set2(1, 0, 0, std::exp(i1 * (kPi / 4))); break;
      case QS_RX: {
        const double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
        set2(c, -i1 * s, -i1 * s, c);
        break;
      }
      case QS_RY: {
        const double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
        set2(c, -s, s, c);
        break;
      }
      case QS_RZ: set2(std::exp(-i1 * (p[0] / 2)), 0, 0, std::exp(i1 * (p[0] / 2))); break;
      case QS_U3: {
        const double th = p[0], ph = p[1], la = p[2];
        const double c = std::cos(th / 2), s = std::sin(th / 2);
        set2(c, -std::exp(i1 * la) * s, std::exp(i1 * ph) * s, std::exp(i1 * (la + ph)) * c);
        break;
      }
      case QS_CNOT:
        for (int k = 0; k < 4; ++k) m[k * 4 + k] = 1;
        m[2 * 4 + 2] = 0;
        m[3 * 4 + 3] = 0;
        m[2 * 4 + 3] = 1;
        m[3 * 4 + 2] = 1;
        break;
      case QS_CZ:
        for (int k = 0; k < 4; ++k) m[k * 4 + k] = 1;
        m[15] = -1;
        break;
      case QS_SWAP:
        for (int k = 0; k < 4; ++k) m[k * 4 + k] = 1;
        m[1 * 4 + 1] = 0;
        m[2 * 4 + 2] = 0;
        m[1 * 4 + 2] = 1;
        m[2 * 4 + 1] = 1;
        break;
      case QS_TOFFOLI:
        for (int k = 0; k < 8; ++k) m[k * 8 + k] = 1;
        m[6 * 8 + 6] = 0;
        m[7 * 8 + 7] = 0;
        m[6 * 8 + 7] = 1;
        m[7 * 8 + 6] = 1;
        break;
      default: throw ValidationError("unknown gate kind");
    }
  }
  if (g.dagger) {
    for (int r = 0; r < dim; ++r)
      for (int c = r; c < dim; ++c) {
        const cd a = m[r * dim + c], b = m[c * dim + r];
        m[r * dim + c] = std::conj(b);
        m[c * dim + r] = std::conj(a);
      }
  }
  return dim;
}

bool is_unitary(const std::vector<cd>& m, int dim, double tol) {  // linalg.hpp:28-32
  double worst = 0;
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j < dim; ++j) {
      cd s = 0;
      for (int k = 0; k < dim; ++k) s += std::conj(m[k * dim + i]) * m[k * dim + j];
      if (i == j) s -= 1.0;
      worst = std::max(worst, std::abs(s));
    }
  return worst <= tol;
}

void validate_gate(const qs_gate& g, uint32_t n) {  // circuit.hpp:429-469
  std::vector<std::string> bad;
  if (g.kind < QS_I || g.kind > QS_CUSTOM) throw ValidationError("unknown gate kind");
  if (g.num_targets > QS_MAX_TARGETS) throw ValidationError("too many targets");
  if (g.num_controls > QS_MAX_CONTROLS) throw ValidationError("too many controls");
  if (g.kind == QS_CUSTOM) {
    if (!g.matrix) throw ValidationError("custom gate has no matrix");
    if (g.num_targets == 0) throw ValidationError("custom gate has no targets");
    std::vector<cd> m;
    base_matrix(g, m);
    if (!is_unitary(m, 1 << g.num_targets, 1e-10))
      throw ValidationError("custom matrix is not unitary within 1e-10");
  } else if (g.num_targets != target_arity(g.kind)) {
    throw ValidationError(std::string(gate_name(g.kind)) + " expects " + std::to_string(target_arity(g.kind)) +
                          " target(s), got " + std::to_string(g.num_targets));
  }
  std::vector<uint32_t> all(g.controls, g.controls + g.num_controls);
  all.insert(all.end(), g.targets, g.targets + g.num_targets);
  for (auto q : all)
    if (q >= n)
      throw ValidationError("qubit q[" + std::to_string(q) + "] out of range (program has " + std::to_string(n) + ")");
  std::sort(all.begin(), all.end());
  if (std::adjacent_find(all.begin(), all.end()) != all.end()) throw ValidationError("duplicate qubit operand");
}

Op lower_gate(const qs_gate& g, uint32_t n, bool validate) {  // statevector.hpp:469-538
  if (validate) validate_gate(g, n);
  const cd i1(0, 1);
  Op op;
  op.controls.assign(g.controls, g.controls + g.num_controls);
  const uint32_t* t = g.targets;
  switch (g.kind) {
    case QS_I: op.kind = OpKind::Identity; return op;
    case QS_X: op.kind = OpKind::Flip; op.targets = {t[0]}; return op;
    case QS_CNOT:
      op.kind = OpKind::Flip;
      op.controls.push_back(t[0]);
      op.targets = {t[1]};
      return op;
    case QS_TOFFOLI:
      op.kind = OpKind::Flip;
      op.controls.push_back(t[0]);
      op.controls.push_back(t[1]);
      op.targets = {t[2]};
      return op;
    case QS_Z:
      op.kind = OpKind::Diag;
      op.targets = {t[0]};
      op.m = {1.0, -1.0};
      return op;
    case QS_CZ:
      op.kind = OpKind::Diag;
      op.controls.push_back(t[0]);
      op.targets = {t[1]};
      op.m = {1.0, -1.0};
      return op;
    case QS_S:
      op.kind = OpKind::Diag;
      op.targets = {t[0]};
      op.m = {1.0, g.dagger ? -i1 : i1};
      return op;
    case QS_T: {
      cd d = std::exp(i1 * (kPi / 4));
      op.kind = OpKind::Diag;
      op.targets = {t[0]};
      op.m = {1.0, g.dagger ? std::conj(d) : d};
      return op;
    }
    case QS_RZ: {
      const double th = g.dagger ? -g.params[0] : g.params[0];
      op.kind = OpKind::Diag;
      op.targets = {t[0]};
      op.m = {std::exp(-i1 * (th / 2)), std::exp(i1 * (th / 2))};
      return op;
    }
    case QS_SWAP: op.kind = OpKind::Swap; op.targets = {t[0], t[1]}; return op;
    case QS_Y:
    case QS_H:
    case QS_RX:
    case QS_RY:
    case QS_U3:
      op.kind = OpKind::Mat1;
      op.targets = {t[0]};
      base_matrix(g, op.m);
      return op;
    case QS_CUSTOM: {
      if (!g.matrix) throw ValidationError("custom gate has no matrix");
      const int dim = base_matrix(g, op.m);
      if (!validate && !is_unitary(op.m, dim, 1e-10))
        throw ValidationError("custom matrix is not unitary within 1e-10");
      if (g.num_targets + op.controls.size() > n) throw ValidationError("apply_matrix: too many operands");
      op.targets.assign(t, t + g.num_targets);
      op.kind = g.num_targets == 1 ? OpKind::Mat1 : OpKind::Dense;
      return op;
    }
  }
  throw RuntimeError("unknown gate kind");
}

Op lower_matrix(const uint32_t* targets, uint32_t k, const double* m, const uint32_t* controls, uint32_t nc,
                uint32_t n) {  // statevector.hpp:363-403
  if (k == 0 || k > QS_MAX_TARGETS) throw ValidationError("apply_matrix: bad target count");
  if (k + nc > n) throw ValidationError("apply_matrix: too many operands");
  std::vector<uint32_t> all(controls, controls + nc);
  all.insert(all.end(), targets, targets + k);
  for (auto q : all)
    if (q >= n) throw ValidationError("apply_matrix: qubit out of range");
  std::sort(all.begin(), all.end());
  if (std::adjacent_find(all.begin(), all.end()) != all.end()) throw ValidationError("duplicate qubit operand");
  Op op;
  op.kind = k == 1 ? OpKind::Mat1 : OpKind::Dense;
  op.targets.assign(targets, targets + k);
  op.controls.assign(controls, controls + nc);
  const size_t dim = size_t(1) << k;
  op.m.resize(dim * dim);
  for (size_t i = 0; i < dim * dim; ++i) op.m[i] = cd(m[2 * i], m[2 * i + 1]);
  return op;
}

bool op_preserves_bit(const Op& op, uint32_t q) {
  for (auto c : op.controls)
    if (c == q) return true;
  switch (op.kind) {
    case OpKind::Identity: return true;
    case OpKind::Diag: return true;
    case OpKind::Flip:
    case OpKind::Swap: return std::find(op.targets.begin(), op.targets.end(), q) == op.targets.end();
    case OpKind::Mat1:
      if (op.targets[0] != q) return true;
      return op.m[1] == cd(0) && op.m[2] == cd(0);
    case OpKind::Dense: {
      const auto it = std::find(op.targets.begin(), op.targets.end(), q);
      if (it == op.targets.end()) return true;
      const size_t k = op.targets.size(), dim = size_t(1) << k;
      const size_t b = k - 1 - static_cast<size_t>(it - op.targets.begin());  // local bit of q
      for (size_t r = 0; r < dim; ++r)
        for (size_t c = 0; c < dim; ++c)
          if (((r ^ c) >> b) & 1)
            if (op.m[r * dim + c] != cd(0)) return false;
      return true;
    }
  }
  return false;
}

}  // namespace qsb
