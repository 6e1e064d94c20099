// partial_amplitude (reference: pathsum.hpp:317-459) on batched half-size
// state vectors.
//
// The reference cuts the qubits into blocks A and B; every crossing CZ
// (crossing CNOTs become H.CZ.H) splits into |0><0| (x) I + |1><1| (x) Z, so
// each of the 2^k branch assignments factors into two block-local circuits and
// amplitude(t) = sum_branches ampA(t_A) * ampB(t_B).  It simulates the 2^k
// branches one after the other, two StateVector runs each (pathsum.hpp:434-457).
//
// Here the branches are state qubits.  For block X (n_X qubits) and c of the k
// branch variables, ONE state of n_X + c qubits holds 2^c branches at once
// (branch b = the top c index bits): H on the c branch qubits starts every
// branch in |0...0> (scaled by 2^(-c/2), undone exactly at the end), the
// branch-dependent operators become ordinary diagonal gates on (local qubit,
// branch qubit) -- the projector [q == b_v] is diag(0,1) on the branch qubit
// controlled by q times diag(0,1) on q controlled by the branch qubit, the
// conditional Z is a CZ -- and the whole block circuit runs through the tile
// planner (every branch in the same HBM passes).  Variables beyond c are fixed
// per chunk of 2^c branches (the chunk loop is over the remaining k - c bits).
// The branch sum is one GPU reduction per target (k_branch_dot).
#include <algorithm>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "gates.hpp"
#include "kernels.hpp"
#include "plan.hpp"
#include "tile.hpp"
#include "jit.hpp"

namespace qsb {

namespace {

struct OwnedState {
  State s;
  OwnedState(uint32_t n, int device) {
    s.n = n;
    s.device = device;
    s.size = 1ull << n;
    DeviceGuard dg(device);
    QSB_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    if (cudaMalloc(&s.amps, s.size * sizeof(double2)) != cudaSuccess) {
      cudaGetLastError();
      cudaStreamDestroy(s.stream);
      throw MemoryError("cannot allocate a " + std::to_string(n) + "-qubit branch batch");
    }
  }
  ~OwnedState() {
    DeviceGuard dg(s.device);
    cudaStreamSynchronize(s.stream);
    if (s.amps) cudaFree(s.amps);
    if (s.alt) cudaFree(s.alt);
    if (s.scratch) cudaFree(s.scratch);
    if (s.host_pinned) cudaFreeHost(s.host_pinned);
    cudaStreamDestroy(s.stream);
  }
};

// One entry of a block's op sequence: a fixed (block-local) op, or a
// branch-dependent one on local qubit q for variable var.
struct BlockOp {
  Op op;
  int var = -1;
  uint32_t q = 0;
  bool projector = false;  // A side of a crossing: |b_v><b_v| on q; B side: Z^(b_v) on q
};

Op diag_op(uint32_t target, cd d0, cd d1, std::vector<uint32_t> controls = {}) {
  Op o;
  o.kind = OpKind::Diag;
  o.targets = {target};
  o.controls = std::move(controls);
  o.m = {d0, d1};
  return o;
}

Op hadamard(uint32_t q, uint32_t n) {
  qs_gate g{};
  g.kind = QS_H;
  g.num_targets = 1;
  g.targets[0] = q;
  return lower_gate(g, n, false);
}

std::unique_ptr<Plan> plan_ops(uint32_t n, std::vector<Op> ops) {
  auto plan = std::make_unique<Plan>();
  plan->n = n;
  plan->mode = QS_PLAN_TILED;
  plan->gates = ops.size();
  plan_tiles(n, ops, plan->steps, 0, false);
  compile_tile_steps(plan->steps);
  return plan;
}

}  // namespace

void partial_amplitude(uint32_t n, const qs_gate* gates, uint64_t count, const uint32_t* block_a, uint32_t na_in,
                       const uint64_t* targets, uint64_t ntargets, int device, uint32_t batch_qubits,
                       double* out) {
  if (n < 2) throw ValidationError("cut planning needs at least 2 qubits");
  for (uint64_t i = 0; i < count; ++i) validate_gate(gates[i], n);
  std::vector<int> side(n, 1);
  std::vector<uint32_t> qa, qb;
  {
    std::vector<char> seen(n, 0);
    for (uint32_t i = 0; i < na_in; ++i) {
      if (block_a[i] >= n || seen[block_a[i]]) throw ValidationError("cut plan blocks must partition the qubits");
      seen[block_a[i]] = 1;
      side[block_a[i]] = 0;
    }
    for (uint32_t q = 0; q < n; ++q) (side[q] == 0 ? qa : qb).push_back(q);  // ascending
  }
  if (qa.empty() || qb.empty()) throw ValidationError("cut plan blocks must both be non-empty");
  std::vector<uint32_t> local(n);
  for (size_t i = 0; i < qa.size(); ++i) local[qa[i]] = static_cast<uint32_t>(i);
  for (size_t i = 0; i < qb.size(); ++i) local[qb[i]] = static_cast<uint32_t>(i);
  const uint32_t nx[2] = {static_cast<uint32_t>(qa.size()), static_cast<uint32_t>(qb.size())};

  // block-local sequences (pathsum.hpp:354-404)
  std::vector<BlockOp> seq[2];
  int k = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const qs_gate& g = gates[i];
    if (g.num_controls) throw UnsupportedError("cut planning expects gates without extra controls");
    const bool two = g.num_targets == 2;
    if (g.num_targets > 2 || (two && g.kind != QS_CNOT && g.kind != QS_CZ))
      throw UnsupportedError("cut planning cannot handle a gate with more than one target other than CNOT / CZ");
    if (!two || side[g.targets[0]] == side[g.targets[1]]) {
      qs_gate lg = g;
      for (uint32_t t = 0; t < g.num_targets; ++t) lg.targets[t] = local[g.targets[t]];
      const int sd = side[g.targets[0]];
      seq[sd].push_back(BlockOp{lower_gate(lg, nx[sd], false)});
      continue;
    }
    const int var = k++;
    const uint32_t a = g.targets[0], b = g.targets[1];
    auto branched = [&](uint32_t q) {
      BlockOp o;
      o.var = var;
      o.q = local[q];
      o.projector = side[q] == 0;
      seq[side[q]].push_back(o);
    };
    if (g.kind == QS_CNOT) {  // CNOT = (I (x) H) CZ (I (x) H) on the target
      seq[side[b]].push_back(BlockOp{hadamard(local[b], nx[side[b]])});
      branched(a);
      branched(b);
      seq[side[b]].push_back(BlockOp{hadamard(local[b], nx[side[b]])});
    } else {
      branched(a);
      branched(b);
    }
  }
  if (k > 62) throw ValidationError("too many crossing gates");

  // targets -> block-local indices
  std::vector<uint64_t> ta(ntargets), tb(ntargets);
  for (uint64_t t = 0; t < ntargets; ++t) {
    if (n < 64 && (targets[t] >> n)) throw ValidationError("target index out of range");
    uint64_t x = 0, y = 0;
    for (size_t i = 0; i < qa.size(); ++i) x |= ((targets[t] >> qa[i]) & 1ull) << i;
    for (size_t i = 0; i < qb.size(); ++i) y |= ((targets[t] >> qb[i]) & 1ull) << i;
    ta[t] = x;
    tb[t] = y;
  }

  // branch qubits per batch: both blocks hold the same 2^c branches
  const uint32_t cap = batch_qubits ? batch_qubits : 26;
  const uint32_t big = std::max(nx[0], nx[1]);
  const uint32_t c = static_cast<uint32_t>(std::min<int64_t>(k, std::max<int64_t>(0, int64_t(cap) - big)));
  if (big > 30) throw ValidationError("each block is limited to 30 qubits");
  if (k - static_cast<int>(c) > 40)
    throw ValidationError("partial amplitude: " + std::to_string(k) + " crossing gates need 2^" +
                          std::to_string(k - static_cast<int>(c)) + " sequential branch batches");
  std::unique_ptr<OwnedState> st[2] = {std::make_unique<OwnedState>(nx[0] + c, device),
                                       std::make_unique<OwnedState>(nx[1] + c, device)};
  std::vector<cd> acc(ntargets, cd(0)), part;
  const double scale = std::ldexp(1.0, static_cast<int>(c));  // H^{(x)c} on both blocks: 2^-c on the product
  const uint64_t chunks = 1ull << (k - c);
  for (uint64_t j = 0; j < chunks; ++j) {
    for (int sd = 0; sd < 2; ++sd) {
      const uint32_t nb = nx[sd] + c;
      std::vector<Op> ops;
      for (uint32_t v = 0; v < c; ++v) ops.push_back(hadamard(nx[sd] + v, nb));
      for (const BlockOp& e : seq[sd]) {
        if (e.var < 0) {
          ops.push_back(e.op);
          continue;
        }
        if (static_cast<uint32_t>(e.var) < c) {  // a branch qubit of this batch
          const uint32_t bq = nx[sd] + static_cast<uint32_t>(e.var);
          if (e.projector) {  // keep q == b: zero (q=1, b=0) and (q=0, b=1)
            ops.push_back(diag_op(bq, cd(0), cd(1), {e.q}));
            ops.push_back(diag_op(e.q, cd(0), cd(1), {bq}));
          } else {
            ops.push_back(diag_op(e.q, cd(1), cd(-1), {bq}));  // CZ
          }
          continue;
        }
        const bool bit = (j >> (static_cast<uint32_t>(e.var) - c)) & 1ull;
        if (e.projector) ops.push_back(diag_op(e.q, bit ? cd(0) : cd(1), bit ? cd(1) : cd(0)));
        else if (bit) ops.push_back(diag_op(e.q, cd(1), cd(-1)));
      }
      auto plan = plan_ops(nb, std::move(ops));
      execute_plan_from_basis(st[sd]->s, *plan, 0);
    }
    branch_dot(st[0]->s, st[1]->s, nx[0], nx[1], c, ta, tb, part);
    for (uint64_t t = 0; t < ntargets; ++t) acc[t] += part[t] * scale;  // chunks in branch order
  }
  for (uint64_t t = 0; t < ntargets; ++t) {
    out[2 * t] = acc[t].real();
    out[2 * t + 1] = acc[t].imag();
  }
}

}  // namespace qsb
