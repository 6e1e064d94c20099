#include "fusion.hpp"

#include <algorithm>
#include <set>

#include "gates.hpp"

namespace qsb {

GateRec copy_gate(const qs_gate& g) {
  GateRec r;
  r.g = g;
  if (g.kind == QS_CUSTOM && g.matrix) {
    const size_t dim = size_t(1) << g.num_targets;
    r.matrix.assign(g.matrix, g.matrix + 2 * dim * dim);
  }
  r.bind();
  return r;
}

std::vector<cd> gate_matrix(const qs_gate& g, int* dim_out) {
  std::vector<cd> base;
  int dim = base_matrix(g, base);
  // controlled_expand (gates.hpp:80-88): identity with u in the all-ones corner
  for (uint32_t c = 0; c < g.num_controls; ++c) {
    const int nd = dim * 2;
    std::vector<cd> next(static_cast<size_t>(nd) * nd, cd(0));
    for (int i = 0; i < dim; ++i) next[static_cast<size_t>(i) * nd + i] = 1.0;
    for (int r = 0; r < dim; ++r)
      for (int col = 0; col < dim; ++col) next[static_cast<size_t>(dim + r) * nd + dim + col] = base[static_cast<size_t>(r) * dim + col];
    base.swap(next);
    dim = nd;
  }
  *dim_out = dim;
  return base;
}

std::vector<cd> embed_on_bits(const std::vector<cd>& u, int udim, const std::vector<uint32_t>& bits, uint32_t k) {
  const size_t dim = size_t(1) << k;
  const size_t nb = bits.size();
  std::vector<cd> out(dim * dim, cd(0));
  std::vector<size_t> masks(nb);
  for (size_t b = 0; b < nb; ++b) masks[b] = size_t(1) << bits[nb - 1 - b];
  size_t op_mask = 0;
  for (auto m : masks) op_mask |= m;
  for (size_t col = 0; col < dim; ++col) {
    const size_t rest = col & ~op_mask;
    size_t lc = 0;
    for (size_t b = 0; b < nb; ++b)
      if (col & masks[b]) lc |= size_t(1) << b;
    for (size_t lr = 0; lr < static_cast<size_t>(udim); ++lr) {
      const cd v = u[lr * udim + lc];
      if (v == cd(0)) continue;
      size_t row = rest;
      for (size_t b = 0; b < nb; ++b)
        if (lr & (size_t(1) << b)) row |= masks[b];
      out[row * dim + col] += v;
    }
  }
  return out;
}

namespace {
std::vector<uint32_t> qubits_of(const qs_gate& g) {  // Gate::qubits(), controls first
  std::vector<uint32_t> q(g.controls, g.controls + g.num_controls);
  q.insert(q.end(), g.targets, g.targets + g.num_targets);
  return q;
}

std::vector<cd> matmul(const std::vector<cd>& a, const std::vector<cd>& b, size_t dim) {
  std::vector<cd> c(dim * dim, cd(0));
  for (size_t i = 0; i < dim; ++i)
    for (size_t k = 0; k < dim; ++k) {
      const cd aik = a[i * dim + k];
      if (aik == cd(0)) continue;
      for (size_t j = 0; j < dim; ++j) c[i * dim + j] += aik * b[k * dim + j];
    }
  return c;
}
}  // namespace

std::vector<GateRec> fuse_gate_run(const qs_gate* gates, uint64_t count, uint32_t nq, uint32_t max_fused_qubits) {
  // build_dag (dag.hpp:37-82) over the run
  const size_t n = count;
  std::vector<std::vector<uint32_t>> nq_of(n);
  std::vector<std::vector<size_t>> succ(n), pred(n);
  std::vector<int64_t> last(nq, -1);
  for (size_t i = 0; i < n; ++i) {
    nq_of[i] = qubits_of(gates[i]);
    for (auto q : nq_of[i]) {
      const int64_t from = last[q];
      if (from >= 0) {
        auto& s = succ[static_cast<size_t>(from)];
        if (std::find(s.begin(), s.end(), i) == s.end()) {
          s.push_back(i);
          pred[i].push_back(static_cast<size_t>(from));
        }
      }
      last[q] = static_cast<int64_t>(i);
    }
  }
  std::vector<size_t> indeg(n);
  for (size_t i = 0; i < n; ++i) indeg[i] = pred[i].size();
  auto key = [&](size_t v) {
    return std::pair<uint32_t, size_t>(*std::min_element(nq_of[v].begin(), nq_of[v].end()), v);
  };
  std::set<std::pair<uint32_t, size_t>> ready;
  for (size_t i = 0; i < n; ++i)
    if (indeg[i] == 0) ready.insert(key(i));

  std::set<uint32_t> block_qubits;
  std::vector<size_t> block_nodes;
  std::vector<GateRec> out;

  auto flush = [&]() {  // fusion.hpp:43-67
    if (block_nodes.empty()) return;
    if (block_nodes.size() == 1) {
      out.push_back(copy_gate(gates[block_nodes[0]]));
    } else {
      std::vector<uint32_t> qs(block_qubits.begin(), block_qubits.end());
      const uint32_t k = static_cast<uint32_t>(qs.size());
      const size_t dim = size_t(1) << k;
      std::vector<cd> m(dim * dim, cd(0));
      for (size_t i = 0; i < dim; ++i) m[i * dim + i] = 1.0;
      for (auto v : block_nodes) {
        std::vector<uint32_t> bits;
        for (auto q : nq_of[v]) bits.push_back(static_cast<uint32_t>(std::lower_bound(qs.begin(), qs.end(), q) - qs.begin()));
        int gd = 0;
        const std::vector<cd> gm = gate_matrix(gates[v], &gd);
        m = matmul(embed_on_bits(gm, gd, bits, k), m, dim);
      }
      GateRec r;
      r.g.kind = QS_CUSTOM;
      r.g.num_targets = k;
      for (uint32_t i = 0; i < k; ++i) r.g.targets[i] = qs[k - 1 - i];
      r.matrix.resize(2 * dim * dim);
      for (size_t i = 0; i < dim * dim; ++i) {
        r.matrix[2 * i] = m[i].real();
        r.matrix[2 * i + 1] = m[i].imag();
      }
      r.bind();
      out.push_back(std::move(r));
    }
    block_nodes.clear();
    block_qubits.clear();
  };
  auto fits = [&](size_t v) {
    std::set<uint32_t> u = block_qubits;
    for (auto q : nq_of[v]) u.insert(q);
    return u.size() <= max_fused_qubits;
  };

  while (!ready.empty()) {  // fusion.hpp:75-99
    size_t chosen = static_cast<size_t>(-1);
    for (const auto& kv : ready)
      if (fits(kv.second)) {
        chosen = kv.second;
        break;
      }
    if (chosen == static_cast<size_t>(-1)) {
      flush();
      chosen = ready.begin()->second;
    }
    ready.erase(key(chosen));
    for (auto s : succ[chosen])
      if (--indeg[s] == 0) ready.insert(key(s));
    if (nq_of[chosen].size() > max_fused_qubits) {
      flush();
      out.push_back(copy_gate(gates[chosen]));
      continue;
    }
    for (auto q : nq_of[chosen]) block_qubits.insert(q);
    block_nodes.push_back(chosen);
  }
  flush();
  // re-bind matrix pointers after vector moves
  for (auto& r : out) r.bind();
  return out;
}

}  // namespace qsb
