#include "plan.hpp"

#include <cmath>
#include <list>
#include <mutex>
#include <string>

#include "fusion.hpp"
#include "jit.hpp"
#include "kernels.hpp"
#include "tile.hpp"

namespace qsb {

uint64_t Plan::passes() const {
  uint64_t p = 0;
  for (const auto& s : steps)
    if (s.kind != Step::OpStep || s.op.kind != OpKind::Identity) ++p;
  return p;
}

uint64_t Plan::launches() const {
  uint64_t l = 0;
  for (const auto& s : steps) {
    if (s.kind == Step::TileStep || s.kind == Step::PermStep) l += 1;
    else if (s.op.kind != OpKind::Identity) l += 1;
  }
  return l;
}

// An out-of-place permutation pass needs a second 2^n-amplitude buffer: plan
// it only when two states fit in the current device's memory (a 33-qubit
// state, 128 GiB, fits a B200 once, not twice).
bool second_buffer_fits(uint32_t n) {
  int dev = 0;
  size_t free_b = 0, total_b = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    return n <= 32;  // no device to ask (planning on a host without a GPU)
  }
  const double need = 2.0 * 16.0 * std::ldexp(1.0, static_cast<int>(n));
  return need <= 0.9 * static_cast<double>(total_b);
}

std::unique_ptr<Plan> make_plan(uint32_t n, const qs_gate* gates, uint64_t count, uint32_t mode,
                                uint32_t max_fused_qubits, uint32_t global_qubits, bool sharded) {
  auto plan = std::make_unique<Plan>();
  plan->n = n;
  plan->g = global_qubits;
  if (global_qubits) {
    if (mode != QS_PLAN_DEFAULT && mode != QS_PLAN_TILED)
      throw ValidationError("sharded states are planned with tile passes only");
    if (global_qubits >= n || n - global_qubits < 6) throw ValidationError("each shard needs at least 6 local qubits");
  }
  plan->mode = mode == QS_PLAN_DEFAULT ? QS_PLAN_TILED : mode;
  plan->gates = count;
  // validation first (validate_or_throw, circuit.hpp:523), in program order
  for (uint64_t i = 0; i < count; ++i) validate_gate(gates[i], n);

  std::vector<Op> ops;
  ops.reserve(count);
  if (plan->mode == QS_PLAN_DENSE_FUSION) {
    if (max_fused_qubits < 1 || max_fused_qubits > 5) throw ValidationError("max_fused_qubits must be in [1, 5]");
    std::vector<GateRec> fused = fuse_gate_run(gates, count, n, max_fused_qubits);
    for (auto& r : fused) {
      r.bind();
      ops.push_back(lower_gate(r.g, n, /*validate=*/false));
    }
  } else {
    for (uint64_t i = 0; i < count; ++i) {
      Op op = lower_gate(gates[i], n, /*validate=*/false);
      op.gate_index = i;
      ops.push_back(std::move(op));
    }
  }
  if (plan->mode == QS_PLAN_TILED) {
    plan_tiles(n, ops, plan->steps, global_qubits, sharded, !sharded && !second_buffer_fits(n));
    compile_tile_steps(plan->steps);
  } else {
    for (auto& op : ops) {
      if (op.kind == OpKind::Identity) continue;
      Step s;
      s.kind = Step::OpStep;
      s.op = std::move(op);
      plan->steps.push_back(std::move(s));
    }
  }
  return plan;
}

// ------------------------------------------------------------- plan cache
// qs_apply_circuit re-submits the same gate list in loops (benchmarks,
// repeated runs): plans are cached by the exact bytes of the submission.
namespace {
std::string plan_key(uint32_t n, const qs_gate* gates, uint64_t count, uint32_t mode, uint32_t maxk, uint32_t g) {
  std::string k;
  auto put = [&](const void* p, size_t b) { k.append(static_cast<const char*>(p), b); };
  put(&n, 4);
  put(&mode, 4);
  put(&maxk, 4);
  put(&g, 4);
  put(&count, 8);
  for (uint64_t i = 0; i < count; ++i) {
    const qs_gate& q = gates[i];
    put(&q.kind, 4);
    put(&q.dagger, 4);
    put(&q.num_targets, 4);
    put(&q.num_controls, 4);
    put(q.targets, 4 * std::min<uint32_t>(q.num_targets, QS_MAX_TARGETS));
    put(q.controls, 4 * std::min<uint32_t>(q.num_controls, QS_MAX_CONTROLS));
    put(q.params, sizeof(q.params));
    if (q.kind == QS_CUSTOM && q.matrix && q.num_targets <= QS_MAX_TARGETS) {
      const size_t dim = size_t(1) << q.num_targets;
      put(q.matrix, dim * dim * 2 * sizeof(double));
    }
  }
  return k;
}
struct PlanCache {
  std::mutex mu;
  std::list<std::pair<std::string, std::shared_ptr<const Plan>>> lru;  // front = most recent
};
PlanCache& plan_cache() {
  static PlanCache c;
  return c;
}
}  // namespace

std::shared_ptr<const Plan> cached_plan(uint32_t n, const qs_gate* gates, uint64_t count, uint32_t mode,
                                        uint32_t max_fused_qubits, uint32_t global_qubits, bool sharded) {
  static const bool enabled = [] {
    const char* e = std::getenv("QSB_PLAN_CACHE");
    return !e || std::atoi(e) != 0;
  }();
  if (!enabled) return make_plan(n, gates, count, mode, max_fused_qubits, global_qubits, sharded);
  // planning / code-generation knobs (DESIGN 6e) are read when a plan is made,
  // so they are part of the key: a plan made under other settings is not reused
  std::string knobs;
  for (const char* k : {"QSB_TILE_M", "QSB_TILE_R", "QSB_TILE_LOW", "QSB_TILE_REMAP", "QSB_PERM_STEP", "QSB_ABSORB_X",
                        "QSB_NO_ABSORB_X", "QSB_FOLD_PERM", "QSB_FREE_LOAD", "QSB_SHARD_BATCH", "QSB_TILE_PREFETCH",
                        "QSB_TILE_SINGLEBUF", "QSB_TILE_MINB", "QSB_BASIS_MINB", "QSB_TILE_EARLY",
                        "QSB_NO_WARP_TRANSPOSE", "QSB_TILE_VARIANTS", "QSB_TMA", "QSB_NO_FLIP_FRAME", "QSB_SPARSE_ZERO_STORE",
                        "QSB_NO_ZERO_WARPS"})
    if (const char* v = std::getenv(k)) knobs += std::string(k) + "=" + v + ";";
  const std::string key =
      plan_key(n, gates, count, mode, max_fused_qubits, global_qubits) + (sharded ? "S" : "") + knobs;
  PlanCache& c = plan_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    for (auto it = c.lru.begin(); it != c.lru.end(); ++it)
      if (it->first == key) {
        c.lru.splice(c.lru.begin(), c.lru, it);
        return c.lru.front().second;
      }
  }
  std::shared_ptr<const Plan> p = make_plan(n, gates, count, mode, max_fused_qubits, global_qubits, sharded);
  std::lock_guard<std::mutex> lk(c.mu);
  c.lru.emplace_front(key, p);
  while (c.lru.size() > 8) c.lru.pop_back();
  return p;
}

void execute_plan(State& s, const Plan& p) {
  if (p.n != s.n) throw ValidationError("plan was compiled for a different qubit count");
  if (p.g != s.g) throw ValidationError("plan was compiled for a sharded state (use the shard API)");
  for (const auto& st : p.steps) execute_step(s, st);
}

TileSkip zero_tiles(const Step& st, uint64_t basis) {
  TileSkip k;
  const bool off = std::getenv("QSB_NO_ZERO_SKIP") != nullptr;
  const bool no_sparse = std::getenv("QSB_NO_SPARSE_LOAD") != nullptr;
  if (off || st.kind != Step::TileStep) return k;
  unsigned long long tile_bits = 0;
  for (uint32_t b = 0; b < st.tile->h.m; ++b) tile_bits |= 1ull << st.tile->h.S[b];
  for (size_t i = 0; i < st.def_pos.size(); ++i) {
    const unsigned long long bit = 1ull << st.def_pos[i];
    const bool one = (__builtin_popcountll(basis & st.def_mask[i]) & 1) ^ st.def_const[i];
    if (bit & tile_bits) {
      if (no_sparse) continue;
      k.imask |= bit;
      if (one) k.ival |= bit;
    } else {
      k.mask |= bit;
      if (one) k.val |= bit;
    }
  }
  return k;
}

// Algorithmic bytes of one per-gate kernel (read + write of the amplitudes
// it touches; `amp` = the state's bytes): controls halve the set per control,
// a phase with d0 == 1 and a SWAP touch half of what remains.
double op_bytes(const Op& op, double amp) {
  double f = std::ldexp(1.0, -static_cast<int>(op.controls.size()));
  switch (op.kind) {
    case OpKind::Identity: return 0.0;
    case OpKind::Diag:
      if (op.m[0] == cd(1.0)) f *= 0.5;
      break;
    case OpKind::Swap: f *= 0.5; break;
    default: break;
  }
  return 2.0 * amp * f;
}

void execute_plan_from_basis(State& s, const Plan& p, uint64_t basis, double* checksum, StepProfile* prof) {
  if (p.n != s.n) throw ValidationError("plan was compiled for a different qubit count");
  if (p.g != s.g) throw ValidationError("plan was compiled for a sharded state (use the shard API)");
  if (basis >> s.n) throw ValidationError("basis index out of range");
  // Lazy zeros: the first pass writes only its possibly non-zero tiles; every
  // later pass reads only amplitudes that can be non-zero (compact tile
  // counter + sparse loads), and those lie inside what the previous pass
  // wrote (a qubit definite outside a pass's tile stays definite through it).
  // Before a step that reads everything, and at the end, the complement of
  // the last pass's tiles is zeroed -- usually empty (every tile active).
  const bool lazy = !std::getenv("QSB_NO_LAZY_ZERO") && !std::getenv("QSB_NO_SPARSE_LOAD") &&
                           !std::getenv("QSB_NO_ZERO_SKIP") && !std::getenv("QSB_NO_TILE_COMPACT");
  TileSkip unwritten;  // amplitudes outside (mask, val) may hold stale data
  auto settle = [&]() {
    if (unwritten.mask) zero_outside(s, unwritten.mask, unwritten.val);
    unwritten = TileSkip{};
  };
  // the checksum rides on the last pass when the plan ends with a tile pass
  const bool fuse_sum = !std::getenv("QSB_NO_FUSED_CHECKSUM");
  const bool fused = checksum && fuse_sum && !p.steps.empty() &&
                     (p.steps.back().kind == Step::TileStep || p.steps.back().kind == Step::PermStep);
  double* part = fused ? static_cast<double*>(s.get_scratch(kMaxTileGrid * sizeof(double) + sizeof(double))) : nullptr;
  unsigned parts = 0;
  const size_t last = p.steps.size() - 1;
  // per-step profile: events between steps, algorithmic bytes per step
  std::vector<cudaEvent_t> ev;
  const double amp = 16.0 * static_cast<double>(s.size);
  auto mark = [&](size_t i, double bytes) {
    if (!prof) return;
    QSB_CUDA(cudaEventRecord(ev[i + 1], s.stream));
    prof->bytes[i] = bytes;
  };
  auto frac = [](unsigned long long mask) { return std::ldexp(1.0, -__builtin_popcountll(mask)); };
  if (prof) {
    ev.resize(p.steps.size() + 1);
    for (auto& e : ev) QSB_CUDA(cudaEventCreate(&e));
    prof->ms.assign(p.steps.size(), 0.f);
    prof->bytes.assign(p.steps.size(), 0.0);
    QSB_CUDA(cudaEventRecord(ev[0], s.stream));
  }
  // Known-zero stores skipped (kVarZeroSkip): an in-place pass that is not the
  // last one does not store the amplitudes that disagree with the qubits still
  // definite at the next step -- that step never reads them (zero tiles /
  // sparse reads), and they join `unwritten`, zeroed by settle() only if a
  // later step would read everything or at the end.
  const bool zskip_on = !std::getenv("QSB_NO_ZERO_STORE_SKIP");
  auto set_zskip = [&](size_t i, TileSkip& k) {
    if (!zskip_on || i == last || p.steps[i].tile->h.oop) return false;
    const TileSkip kn = zero_tiles(p.steps[i + 1], basis);
    unsigned long long tb = 0;
    for (uint32_t b = 0; b < p.steps[i].tile->h.m; ++b) tb |= 1ull << p.steps[i].tile->h.S[b];
    k.omask = (kn.mask | kn.imask) & tb;
    k.oval = (kn.val | kn.ival) & tb;
    if (!k.omask) return false;
    unwritten = TileSkip{kn.mask | kn.imask, kn.val | kn.ival};  // every amplitude disagreeing may be stale
    return true;
  };
  size_t i = 0;
  if (!p.steps.empty() && p.steps[0].kind == Step::TileStep && !std::getenv("QSB_NO_FUSED_RESET")) {
    TileSkip k = zero_tiles(p.steps[0], basis);
    k.lazy = lazy && !p.steps[0].tile->h.oop;
    const bool zs = set_zskip(0, k);
    const unsigned g0 = launch_tile(s, *p.steps[0].tile, &basis, nullptr, &k, last == 0 ? part : nullptr);
    if (last == 0) parts = g0;
    if (k.lazy && !zs) unwritten = TileSkip{k.mask, k.val};
    mark(0, amp * (k.lazy ? frac(k.mask) : 1.0) * (zs ? frac(k.omask) : 1.0));  // writes only
    i = 1;
  } else {
    fill_basis(s, basis);
  }
  // tiles still provably zero (definite qubits outside the tile) are skipped
  for (; i < p.steps.size(); ++i) {
    double bytes = 2 * amp;
    if (p.steps[i].kind == Step::TileStep) {
      TileSkip k = zero_tiles(p.steps[i], basis);
      const TileSkip before = unwritten;
      const bool zs = set_zskip(i, k);
      const unsigned gi = launch_tile(s, *p.steps[i].tile, nullptr, nullptr, &k, i == last ? part : nullptr);
      if (i == last) parts = gi;
      if (p.steps[i].tile->h.oop) unwritten = TileSkip{};  // the new buffer is written everywhere
      else if (!zs && before.mask) unwritten = TileSkip{k.mask, k.val};
      // in place: only possibly non-zero tiles are visited, inside them only
      // amplitudes agreeing with the definite tile qubits are read
      if (!p.steps[i].tile->h.oop) bytes = amp * frac(k.mask) * (frac(k.imask) + (zs ? frac(k.omask) : 1.0));
    } else if (i == last && part && p.steps[i].kind == Step::PermStep) {
      settle();
      parts = permute_qubits(s, p.steps[i].perm, part);
    } else {
      settle();
      execute_step(s, p.steps[i]);
      if (p.steps[i].kind == Step::OpStep) bytes = op_bytes(p.steps[i].op, amp);
    }
    mark(i, bytes);
  }
  settle();  // zeros only: the fused checksum is unchanged
  if (checksum) *checksum = fused ? sum_partials(s, part, parts) : reduce_checksum(s);
  if (prof) {
    s.sync();
    for (size_t j = 0; j < p.steps.size(); ++j) QSB_CUDA(cudaEventElapsedTime(&prof->ms[j], ev[j], ev[j + 1]));
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

void execute_step(State& s, const Step& st) {
  switch (st.kind) {
    case Step::OpStep: launch_op(s, st.op); break;
    case Step::TileStep: launch_tile(s, *st.tile); break;
    case Step::SwapStep: throw ValidationError("rank-bit exchange outside a shard set");
    case Step::PermStep: permute_qubits(s, st.perm); break;
  }
}

}  // namespace qsb
