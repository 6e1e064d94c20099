// Tile-pass planner (host): partitions a gate list into shared-memory tile
// passes and compiles each pass into a micro-program for tile.cu.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "tile.hpp"

namespace qsb {

namespace {

inline uint64_t bit(uint32_t q) { return 1ull << q; }

enum class PK { Mat1, Flip, Diag, SwapRel, Dense, Opaque };

// A kernel-level op with its planning attributes.
struct POp {
  PK k;
  Op op;
  uint64_t qmask = 0;     // every operand
  uint64_t needmask = 0;  // qubits that must be tile qubits (non-diagonal targets)
};

std::vector<POp> preprocess(std::vector<Op>& ops) {
  std::vector<POp> out;
  out.reserve(ops.size());
  auto push = [&](PK k, Op op) {
    POp p;
    p.k = k;
    for (auto q : op.controls) p.qmask |= bit(q);
    for (auto q : op.targets) p.qmask |= bit(q);
    switch (k) {
      case PK::Mat1:
      case PK::Flip:
      case PK::SwapRel:
      case PK::Dense:
      case PK::Opaque:
        for (auto q : op.targets) p.needmask |= bit(q);
        break;
      default: break;
    }
    p.op = std::move(op);
    out.push_back(std::move(p));
  };
  for (auto& op : ops) {
    switch (op.kind) {
      case OpKind::Identity: break;
      case OpKind::Mat1:
        if (op.m[1] == cd(0) && op.m[2] == cd(0)) {  // diagonal 2x2 (e.g. U3(0,0,l))
          Op d = op;
          d.kind = OpKind::Diag;
          d.m = {op.m[0], op.m[3]};
          push(PK::Diag, std::move(d));
        } else {
          push(PK::Mat1, std::move(op));
        }
        break;
      case OpKind::Flip: push(PK::Flip, std::move(op)); break;
      case OpKind::Diag: push(PK::Diag, std::move(op)); break;
      case OpKind::Swap:
        if (op.controls.empty()) {
          push(PK::SwapRel, std::move(op));
        } else {
          // Fredkin: CNOT(b->a) . CCNOT(C + a -> b) . CNOT(b->a)
          const uint32_t a = op.targets[0], b = op.targets[1];
          Op f1;
          f1.kind = OpKind::Flip;
          f1.targets = {a};
          f1.controls = {b};
          f1.gate_index = op.gate_index;
          Op f2 = f1;
          f2.targets = {b};
          f2.controls = op.controls;
          f2.controls.push_back(a);
          push(PK::Flip, f1);
          push(PK::Flip, f2);
          push(PK::Flip, f1);
        }
        break;
      case OpKind::Dense:
        if (op.targets.size() <= 3) push(PK::Dense, std::move(op));
        else push(PK::Opaque, std::move(op));
        break;
    }
  }
  return out;
}

// Ops of `rem` executable in one pass with tile set S, in program order; an op
// not executable blocks its qubits for every later op.
size_t scan(const std::vector<POp>& pops, const std::vector<uint32_t>& rem, uint64_t S, std::vector<char>* taken) {
  uint64_t blocked = 0;
  size_t cnt = 0;
  for (size_t i = 0; i < rem.size(); ++i) {
    const POp& p = pops[rem[i]];
    if ((p.qmask & blocked) || p.k == PK::Opaque || (p.needmask & ~S)) {
      blocked |= p.qmask;
      continue;
    }
    ++cnt;
    if (taken) (*taken)[i] = 1;
  }
  return cnt;
}

struct Cfg {
  int reg[kTileMaxR];
  int thr[kTileMaxT];
};

// Abstract micro-op before finalisation.
struct AOp {
  uint8_t type = 0;
  int cfg = 0;              // config index at this op
  uint32_t target = 0;      // MAT1 / FLIP qubit
  std::vector<uint32_t> dense_targets;
  uint64_t pred = 0;        // control qubits
  uint64_t pred_val = ~0ull;  // their required values (bits of pred; default all 1)
  cd m[4];
  std::vector<cd> dense;    // row-major
  // PHASE
  cd c = 1.0;
  std::map<uint32_t, cd> w;
  // TRANSPOSE
  int from = 0, to = 0;
};

struct Compiler {
  uint32_t n, m, t, L;
  int R = 4;  // register bits
  std::vector<uint32_t> S;
  int tb[64];
  std::vector<Cfg> cfgs;
  std::vector<AOp> aops;

  bool has_reg(const Cfg& c, int x, int* pos = nullptr) const {
    for (int k = 0; k < R; ++k)
      if (c.reg[k] == x) {
        if (pos) *pos = k;
        return true;
      }
    return false;
  }

  // Tile bit that must sit in lane k (k < L) when the pass stores: its global
  // position is the k-th lowest of the written index (coalescing).  Identity
  // unless the pass stores out of place through a qubit permutation.
  int lane[kTileMaxT] = {0, 1, 2, 3, 4, 5, 6, 7, 8};

  // Fill thread bits: lanes 0..L-1 take the load lanes (tile bits 0..L-1, for
  // the first configuration) or the store lanes when those are not register
  // bits; the rest ascending.
  void fill_threads(Cfg& c, bool load = false) const {
    std::vector<char> used(m, 0);
    for (int k = 0; k < R; ++k) used[c.reg[k]] = 1;
    for (uint32_t k = 0; k < t; ++k) c.thr[k] = -1;
    for (uint32_t k = 0; k < L; ++k) {
      const int y = load ? static_cast<int>(k) : lane[k];
      if (!used[y]) {
        c.thr[k] = y;
        used[y] = 1;
      }
    }
    uint32_t next = 0;
    for (uint32_t k = 0; k < t; ++k) {
      if (c.thr[k] >= 0) continue;
      while (used[next]) ++next;
      c.thr[k] = static_cast<int>(next);
      used[next] = 1;
    }
  }

  bool store_ok(const Cfg& c) const {
    for (uint32_t k = 0; k < L; ++k)
      if (c.thr[k] != lane[k]) return false;
    return true;
  }

  // Register requirement of op i: exact positions for DENSE, else one tile bit.
  static bool needs_reg(const POp& p) { return p.k == PK::Mat1 || p.k == PK::Flip || p.k == PK::Dense; }

  void transpose_to(int& cur, const Cfg& next) {
    if (std::getenv("QSB_PLAN_DEBUG")) {
      int kept = 0;
      for (int a = 0; a < R; ++a)
        for (int b = 0; b < R; ++b) kept += cfgs[cur].reg[a] == next.reg[b];
      std::fprintf(stderr, "transpose: %d of %d register qubits change\n", R - kept, R);
    }
    cfgs.push_back(next);
    AOp a;
    a.type = TO_TRANSPOSE;
    a.from = cur;
    a.to = static_cast<int>(cfgs.size() - 1);
    a.cfg = a.to;
    aops.push_back(a);
    cur = a.to;
  }

  bool satisfied(const Cfg& c, const POp& p) const {
    if (p.k == PK::Dense) {
      const size_t kd = p.op.targets.size();
      for (size_t b = 0; b < kd; ++b)
        if (c.reg[b] != tb[p.op.targets[kd - 1 - b]]) return false;
      return true;
    }
    return has_reg(c, tb[p.op.targets[0]]);
  }

  // --- intra-pass scheduling ------------------------------------------------
  // The pass's ops form a DAG (shared qubits; diagonal ops commute with each
  // other).  We run every op whose targets are register qubits, and when none
  // is left choose the next register set greedily: fill the 4 slots one by one
  // with the tile bit that lets the most pending ops run (a topological sweep
  // in program order), so transposes are amortised over as many gates as
  // possible.
  std::vector<std::vector<int>> succ;
  std::vector<int> indeg;
  std::vector<int> scratch_;

  void build_dag(const std::vector<const POp*>& list) {
    const size_t N = list.size();
    succ.assign(N, {});
    indeg.assign(N, 0);
    for (size_t j = 0; j < N; ++j)
      for (size_t i = 0; i < j; ++i) {
        if (!(list[i]->qmask & list[j]->qmask)) continue;
        if (list[i]->k == PK::Diag && list[j]->k == PK::Diag) continue;
        succ[i].push_back(static_cast<int>(j));
        ++indeg[j];
      }
  }

  bool sat_partial(const Cfg& c, const POp& p) const {
    if (!needs_reg(p)) return true;
    if (p.k == PK::Dense) {
      const size_t kd = p.op.targets.size();
      for (size_t b = 0; b < kd; ++b)
        if (c.reg[b] != tb[p.op.targets[kd - 1 - b]]) return false;
      return true;
    }
    return has_reg(c, tb[p.op.targets[0]]);
  }

  // (ops runnable with register set c without a transpose, -first index of a
  // runnable register op) from the current done/indeg state.
  std::pair<int, int> simulate(const Cfg& c, const std::vector<const POp*>& list, const std::vector<char>& done,
                               std::vector<int>& scratch) const {
    const size_t N = list.size();
    scratch = indeg;
    int cnt = 0, first = -1;
    for (size_t j = 0; j < N; ++j) {
      if (done[j] || scratch[j] != 0) continue;
      if (!sat_partial(c, *list[j])) continue;
      ++cnt;
      if (first < 0 && needs_reg(*list[j])) first = static_cast<int>(j);
      for (int s2 : succ[j]) --scratch[s2];
    }
    return {cnt, first < 0 ? -1000000 : -first};
  }

  Cfg choose_greedy(const Cfg* cur, const std::vector<const POp*>& list, const std::vector<char>& done,
                    bool exclude_low) {
    Cfg c;
    for (int k = 0; k < R; ++k) c.reg[k] = -1;
    std::vector<char> placed(m, 0);
    // a blocked dense op at the front dictates exact slots
    for (size_t j = 0; j < list.size(); ++j) {
      if (done[j] || indeg[j] != 0 || !needs_reg(*list[j])) continue;
      if (cur && sat_partial(*cur, *list[j])) continue;
      if (list[j]->k == PK::Dense) {
        const size_t kd = list[j]->op.targets.size();
        for (size_t b = 0; b < kd; ++b) {
          const int x = tb[list[j]->op.targets[kd - 1 - b]];
          c.reg[b] = x;
          placed[x] = 1;
        }
      }
      break;
    }
    std::vector<int> scratch;
    for (int k = 0; k < R; ++k) {
      if (c.reg[k] >= 0) continue;
      int best = -1;
      std::pair<int, int> bs{-1, -2000000};
      for (uint32_t y = 0; y < m; ++y) {
        if (placed[y] || (exclude_low && y < L)) continue;
        c.reg[k] = static_cast<int>(y);
        std::pair<int, int> sc = simulate(c, list, done, scratch);
        // prefer non-lane bits on ties (keeps the store layout coalesced)
        const bool better = sc > bs || (sc == bs && y >= L && best >= 0 && best < static_cast<int>(L));
        if (better) {
          bs = sc;
          best = static_cast<int>(y);
        }
      }
      if (best < 0)
        for (uint32_t y = 0; y < m; ++y)
          if (!placed[y]) {
            best = static_cast<int>(y);
            break;
          }
      c.reg[k] = best;
      placed[best] = 1;
    }
    fill_threads(c, /*load=*/cur == nullptr);  // the first configuration is the (coalesced) load
    return c;
  }

  bool free_load = false;

  void compile(const std::vector<const POp*>& list) {
    build_dag(list);
    std::vector<char> done(list.size(), 0);
    cfgs.push_back(choose_greedy(nullptr, list, done, /*exclude_low=*/true));
    int cur = 0;
    if (free_load) {
      // The load layout must keep the low qubits on lanes (coalesced reads);
      // if the best first register set holds one of them, start with a
      // transpose out of the load layout -- the GPU fuses it into the
      // prefetch (the cp.async destinations are the transpose's write slots).
      Cfg c1 = choose_greedy(&cfgs[0], list, done, /*exclude_low=*/false);
      bool low_reg = false;
      for (int k = 0; k < R; ++k) low_reg |= c1.reg[k] < static_cast<int>(L);
      if (low_reg && simulate(c1, list, done, scratch_).first > simulate(cfgs[0], list, done, scratch_).first)
        transpose_to(cur, c1);
    }

    int open = -1;           // open PHASE aop
    uint64_t x_open = 0;     // non-diagonal targets since it opened
    auto emit = [&](const POp& p) {
      uint64_t ctrl = 0;
      for (auto q : p.op.controls) ctrl |= bit(q);
      switch (p.k) {
        case PK::Diag: {
          const uint32_t tq = p.op.targets[0];
          const cd d0 = p.op.m[0], d1 = p.op.m[1];
          const uint64_t qm = ctrl | bit(tq);
          struct Rep {
            uint64_t pred, val;
            cd c;
            uint32_t q;
            cd w;
          };
          // negated controls (Pauli-X absorption) must be 0
          const uint64_t cval = ctrl & ~p.op.cneg;
          std::vector<Rep> reps;
          if (d0 == cd(1.0) || d1 == cd(1.0)) {
            // one phase d on a conjunction of literals (b_q = v_q over the
            // controls and the target); any literal can be the weight and the
            // rest the predicate: d^[b=1] = d^b,  d^[b=0] = d * (1/d)^b
            const cd d = d0 == cd(1.0) ? d1 : d0;
            const uint64_t lits = ctrl | bit(tq);
            const uint64_t vals = cval | (d0 == cd(1.0) ? bit(tq) : 0);
            std::vector<uint32_t> order{tq};
            order.insert(order.end(), p.op.controls.begin(), p.op.controls.end());
            for (uint32_t q : order) {
              const bool one = (vals >> q) & 1;
              if (!one && d == cd(0)) continue;  // 1/d: a projector (partial_amplitude) has no weight form here
              reps.push_back({lits & ~bit(q), vals & ~bit(q), one ? cd(1.0) : d, q, one ? d : 1.0 / d});
            }
            // always valid: d under the full conjunction, no weight (1^b)
            if (reps.empty()) reps.push_back({lits, vals, d, tq, cd(1.0)});
          } else {
            if (d0 == cd(0)) throw RuntimeError("tile planner: diagonal (0, d) without a unit entry");
            reps.push_back({ctrl, cval, d0, tq, d1 / d0});
          }
          bool merged = false;
          if (open >= 0 && !(qm & x_open)) {
            for (auto& r : reps)
              if (r.pred == aops[open].pred && r.val == aops[open].pred_val) {
                aops[open].c *= r.c;
                auto it = aops[open].w.find(r.q);
                if (it == aops[open].w.end()) aops[open].w[r.q] = r.w;
                else it->second *= r.w;
                merged = true;
                break;
              }
          }
          if (!merged) {
            const Rep& r = reps.back();  // prefer the predicate holding the target
            AOp a;
            a.type = TO_PHASE;
            a.cfg = cur;
            a.pred = r.pred;
            a.pred_val = r.val;
            a.c = r.c;
            a.w[r.q] = r.w;
            aops.push_back(a);
            open = static_cast<int>(aops.size() - 1);
            x_open = 0;
          }
          break;
        }
        case PK::SwapRel: {
          const int a = tb[p.op.targets[0]], b = tb[p.op.targets[1]];
          Cfg c = cfgs[cur];
          for (int k = 0; k < R; ++k) c.reg[k] = c.reg[k] == a ? b : (c.reg[k] == b ? a : c.reg[k]);
          for (uint32_t k = 0; k < t; ++k) c.thr[k] = c.thr[k] == a ? b : (c.thr[k] == b ? a : c.thr[k]);
          cfgs.push_back(c);
          cur = static_cast<int>(cfgs.size() - 1);
          x_open |= p.needmask;
          // thread bits now name different qubits: refresh the per-thread index
          bool thread_moved = false;
          for (uint32_t k = 0; k < t; ++k)
            if (c.thr[k] == a || c.thr[k] == b) thread_moved = true;
          if (thread_moved) {
            AOp r;
            r.type = TO_RELABEL;
            r.cfg = cur;
            aops.push_back(r);
          }
          break;
        }
        case PK::Mat1:
        case PK::Flip:
        case PK::Dense: {
          AOp a;
          a.cfg = cur;
          a.pred = ctrl;
          if (p.k == PK::Flip) {
            a.type = TO_FLIP;
            a.target = p.op.targets[0];
          } else if (p.k == PK::Mat1) {
            a.type = TO_MAT1;
            a.target = p.op.targets[0];
            for (int k = 0; k < 4; ++k) a.m[k] = p.op.m[k];
          } else {
            a.type = p.op.targets.size() == 2 ? TO_DENSE2 : TO_DENSE3;
            a.dense_targets = p.op.targets;
            a.dense = p.op.m;
          }
          aops.push_back(a);
          x_open |= p.needmask;
          break;
        }
        case PK::Opaque: throw RuntimeError("tile compiler: opaque op inside a pass");
      }
    };
    size_t remaining = list.size();
    while (remaining) {
      for (size_t j = 0; j < list.size(); ++j) {  // one sweep = closure (index order is topological)
        if (done[j] || indeg[j] != 0) continue;
        if (!sat_partial(cfgs[cur], *list[j])) continue;
        emit(*list[j]);
        done[j] = 1;
        --remaining;
        for (int s2 : succ[j]) --indeg[s2];
      }
      if (!remaining) break;
      transpose_to(cur, choose_greedy(&cfgs[cur], list, done, /*exclude_low=*/false));
    }
    if (!store_ok(cfgs[cur])) {
      Cfg c = cfgs[cur];
      bool lane_in_reg = false;
      for (int k = 0; k < R; ++k)
        if (is_store_lane(c.reg[k])) lane_in_reg = true;
      if (lane_in_reg) c = default_cfg();
      else fill_threads(c);
      transpose_to(cur, c);
      if (std::getenv("QSB_PLAN_DEBUG")) std::fprintf(stderr, "store-fix transpose (lanes %s)\n", lane_in_reg ? "in registers" : "on other thread bits");
    }
    final_cfg = cur;
  }
  int final_cfg = 0;

  bool is_store_lane(int y) const {
    for (uint32_t k = 0; k < L; ++k)
      if (lane[k] == y) return true;
    return false;
  }

  Cfg default_cfg() const {
    Cfg c;
    // registers: the highest tile bits not reserved for the store lanes
    int k = 0;
    for (int y = static_cast<int>(m) - 1; y >= 0 && k < R; --y)
      if (!is_store_lane(y) || m - L < static_cast<uint32_t>(R)) c.reg[k++] = y;
    fill_threads(c);
    return c;
  }
};

// 3 x (m-3) GF(2) swizzle: phys(j) = j ^ (parities of j & a[i]) in the low 3 bits.
struct Swizzle {
  uint32_t a[3] = {0, 0, 0};
  uint32_t phys(uint32_t j) const {
    uint32_t low = 0;
    for (int i = 0; i < 3; ++i) low |= static_cast<uint32_t>(__builtin_popcount(j & a[i]) & 1) << i;
    return j ^ low;
  }
};

bool conflict_free(const Swizzle& s, const Cfg& c, uint32_t t) {
  if (t < 3) return true;
  uint32_t v[3];
  for (int i = 0; i < 3; ++i) v[i] = s.phys(1u << c.thr[i]) & 7u;
  // rank 3 over GF(2)
  const uint32_t x = v[0], y = v[1], z = v[2];
  return x && y && z && (x ^ y) && (x ^ z) && (y ^ z) && (x ^ y ^ z);
}

Swizzle pick_swizzle(const Cfg& a, const Cfg& b, uint32_t m, uint32_t t) {
  Swizzle s;
  if (conflict_free(s, a, t) && conflict_free(s, b, t)) return s;
  std::mt19937 rng(12345u + static_cast<uint32_t>(a.thr[0] * 131 + b.thr[0]));
  const uint32_t himask = m > 3 ? ((1u << m) - 1) & ~7u : 0;
  for (int iter = 0; iter < 20000 && himask; ++iter) {
    for (int i = 0; i < 3; ++i) s.a[i] = rng() & himask;
    if (conflict_free(s, a, t) && conflict_free(s, b, t)) return s;
  }
  return Swizzle{};  // correct, possibly conflicted
}

// sigma (optional): the pass stores out of place, bit p of every written index
// moved to bit sigma[p] (the plan's final layout restore folded into its last
// pass); the compiler's store lanes must be sigma^-1 of the low positions.
std::shared_ptr<TileProgram> finalize(Compiler& C, uint64_t gates, const std::vector<uint64_t>& srcs,
                                      const std::vector<uint32_t>* sigma = nullptr) {
  auto tp = std::make_shared<TileProgram>();
  TileHeader& h = tp->h;
  h.n = C.n;
  h.m = C.m;
  h.t = C.t;
  h.r = static_cast<uint32_t>(C.R);
  for (uint32_t b = 0; b < C.m; ++b) h.S[b] = C.S[b];
  h.ntiles = 1ull << (C.n - C.m);
  auto sg = [&](uint32_t q) { return sigma ? (*sigma)[q] : q; };
  auto addr_of = [&](const Cfg& c, TileConfigAddr& a, bool out) {
    for (uint32_t k = 0; k < C.t; ++k) a.tq[k] = out ? sg(C.S[c.thr[k]]) : C.S[c.thr[k]];
    for (int k = 0; k < C.R; ++k) a.rs[k] = 1ull << (out ? sg(C.S[c.reg[k]]) : C.S[c.reg[k]]);
  };
  addr_of(C.cfgs[0], h.load, false);
  addr_of(C.cfgs[C.final_cfg], h.store, true);
  if (sigma) {
    h.oop = 1;
    uint32_t i = 0;
    for (uint32_t q = 0; q < C.n; ++q)
      if (C.tb[q] < 0) h.out_pos[i++] = static_cast<uint8_t>(sg(q));
  }

  auto split_pred = [&](const Cfg& c, uint64_t pred, TOp& o, uint64_t val = ~0ull) {
    o.rmask = 0;
    o.rval = 0;
    o.gmask = 0;
    o.gval = 0;
    for (uint32_t q = 0; q < 64; ++q) {
      if (!((pred >> q) & 1)) continue;
      const bool one = (val >> q) & 1;
      int pos;
      if (C.tb[q] >= 0 && C.has_reg(c, C.tb[q], &pos)) {
        o.rmask |= static_cast<uint16_t>(1u << pos);
        if (one) o.rval |= static_cast<uint16_t>(1u << pos);
      } else {
        o.gmask |= bit(q);
        if (one) o.gval |= bit(q);
      }
    }
  };

  for (const AOp& a : C.aops) {
    TOp o{};
    o.type = a.type;
    const Cfg& c = C.cfgs[a.cfg];
    switch (a.type) {
      case TO_MAT1: {
        int pos = 0;
        C.has_reg(c, C.tb[a.target], &pos);
        o.k = static_cast<uint8_t>(pos);
        split_pred(c, a.pred, o);
        bool real = true, rx = true;
        for (int k = 0; k < 4; ++k)
          if (a.m[k].imag() != 0) real = false;
        if (a.m[0].imag() != 0 || a.m[3].imag() != 0 || a.m[1].real() != 0 || a.m[2].real() != 0) rx = false;
        o.type = real ? TO_MAT1_REAL : (rx ? TO_MAT1_RX : TO_MAT1);
        o.coef = static_cast<uint32_t>(tp->coef.size());
        for (int k = 0; k < 4; ++k) tp->coef.push_back(make_double2(a.m[k].real(), a.m[k].imag()));
        break;
      }
      case TO_FLIP: {
        int pos = 0;
        C.has_reg(c, C.tb[a.target], &pos);
        o.k = static_cast<uint8_t>(pos);
        split_pred(c, a.pred, o);
        break;
      }
      case TO_DENSE2:
      case TO_DENSE3: {
        split_pred(c, a.pred, o);
        o.coef = static_cast<uint32_t>(tp->coef.size());
        for (const auto& e : a.dense) tp->coef.push_back(make_double2(e.real(), e.imag()));
        break;
      }
      case TO_PHASE: {
        split_pred(c, a.pred, o, a.pred_val);
        const int NS = 1 << C.R;
        cd G[kTileMaxSlots];
        for (int p = 0; p < NS; ++p) G[p] = 1.0;
        std::vector<std::pair<uint32_t, cd>> list;
        for (const auto& [q, w] : a.w) {
          if (w == cd(1.0)) continue;
          int pos;
          if (C.tb[q] >= 0 && C.has_reg(c, C.tb[q], &pos)) {
            for (int p = 0; p < NS; ++p)
              if ((p >> pos) & 1) G[p] *= w;
          } else {
            list.push_back({q, w});
          }
        }
        o.coef = static_cast<uint32_t>(tp->coef.size());
        o.meta = static_cast<uint32_t>(tp->meta.size());
        o.nlist = static_cast<uint16_t>(list.size());
        for (int p = 0; p < NS; ++p) tp->coef.push_back(make_double2(G[p].real(), G[p].imag()));
        tp->coef.push_back(make_double2(a.c.real(), a.c.imag()));
        for (auto& [q, w] : list) {
          tp->coef.push_back(make_double2(w.real(), w.imag()));
          tp->meta.push_back(q);
        }
        break;
      }
      case TO_TRANSPOSE: {
        const Cfg& fa = C.cfgs[a.from];
        const Cfg& fb = C.cfgs[a.to];
        const Swizzle sw = pick_swizzle(fa, fb, C.m, C.t);
        o.meta = static_cast<uint32_t>(tp->meta.size());
        for (uint32_t k = 0; k < C.t; ++k) tp->meta.push_back(sw.phys(1u << fa.thr[k]));
        for (int k = 0; k < C.R; ++k) tp->meta.push_back(sw.phys(1u << fa.reg[k]));
        for (uint32_t k = 0; k < C.t; ++k) tp->meta.push_back(sw.phys(1u << fb.thr[k]));
        for (int k = 0; k < C.R; ++k) tp->meta.push_back(sw.phys(1u << fb.reg[k]));
        for (uint32_t k = 0; k < C.t; ++k) tp->meta.push_back(C.S[fb.thr[k]]);
        for (int k = 0; k < C.R; ++k) tp->meta.push_back(C.S[fb.reg[k]]);
        ++tp->transposes;
        break;
      }
      case TO_RELABEL: {
        o.meta = static_cast<uint32_t>(tp->meta.size());
        for (uint32_t k = 0; k < C.t; ++k) tp->meta.push_back(C.S[c.thr[k]]);
        break;
      }
    }
    tp->ops.push_back(o);
  }
  h.nops = static_cast<uint32_t>(tp->ops.size());
  auto al = [](size_t x) { return static_cast<uint32_t>((x + 15) & ~size_t(15)); };
  h.ops_off = al(sizeof(TileHeader));
  h.meta_off = al(h.ops_off + tp->ops.size() * sizeof(TOp));
  h.coef_off = al(h.meta_off + tp->meta.size() * sizeof(uint32_t));
  h.bytes = al(h.coef_off + tp->coef.size() * sizeof(double2));
  tp->gates = gates;
  tp->source = srcs;
  return tp;
}

std::vector<uint32_t> C_S_debug(uint64_t S, uint32_t n) {
  std::vector<uint32_t> v;
  for (uint32_t q = 0; q < n; ++q)
    if ((S >> q) & 1) v.push_back(q);
  return v;
}

}  // namespace

TileOptions tile_options_from_env() {
  TileOptions o;
  if (const char* e = std::getenv("QSB_TILE_M")) o.m = static_cast<uint32_t>(std::atoi(e));
  if (const char* e = std::getenv("QSB_TILE_R"); e && std::atoi(e) > 0) {
    o.r = static_cast<uint32_t>(std::atoi(e));
    o.choose_r = false;
  }
  if (const char* e = std::getenv("QSB_TILE_LOW")) o.low = static_cast<uint32_t>(std::atoi(e));
  if (const char* e = std::getenv("QSB_TILE_REMAP")) o.remap = std::atoi(e) != 0;
  if (const char* e = std::getenv("QSB_PERM_STEP")) o.perm_step = std::atoi(e) != 0;
  if (const char* e = std::getenv("QSB_ABSORB_X")) o.absorb_x = std::atoi(e) != 0;
  if (const char* e = std::getenv("QSB_FOLD_PERM")) o.fold_perm = std::atoi(e) != 0;
  o.free_load = !tma_enabled();  // a bulk-copied tile starts in the load layout
  if (const char* e = std::getenv("QSB_FREE_LOAD")) o.free_load = std::atoi(e) != 0;
  o.m = std::max<uint32_t>(8, std::min<uint32_t>(kTileMaxM, o.m));
  o.r = std::max<uint32_t>(kTileMinR, std::min<uint32_t>(kTileMaxR, o.r));
  o.low = std::min<uint32_t>(5, o.low);
  return o;
}

namespace {

// A POp with its qubits renamed through the logical -> physical map.
POp to_physical(const POp& p, const std::vector<uint32_t>& perm) {
  POp q = p;
  for (auto& t : q.op.targets) t = perm[t];
  for (auto& c : q.op.controls) c = perm[c];
  q.op.cneg = 0;
  for (uint64_t m = p.op.cneg; m; m &= m - 1) q.op.cneg |= bit(perm[__builtin_ctzll(m)]);
  q.qmask = 0;
  q.needmask = 0;
  for (auto c : q.op.controls) q.qmask |= bit(c);
  for (auto t : q.op.targets) q.qmask |= bit(t);
  if (p.needmask)
    for (auto t : q.op.targets) q.needmask |= bit(t);
  return q;
}

POp swap_rel(uint32_t a, uint32_t b) {
  POp p;
  p.k = PK::SwapRel;
  p.op.kind = OpKind::Swap;
  p.op.targets = {a, b};
  p.qmask = p.needmask = bit(a) | bit(b);
  return p;
}

// Chooses the tile set S (physical qubits) for the next pass: starting from the
// always-resident low qubits, add the qubit that lets the most pending ops run.
uint64_t choose_tile_set(const std::vector<POp>& phys, const std::vector<uint32_t>& rem, uint64_t S0, uint32_t m,
                         uint64_t allowed) {
  uint64_t S = S0;
  size_t cur = scan(phys, rem, S, nullptr);
  while (static_cast<uint32_t>(__builtin_popcountll(S)) < m) {
    std::vector<uint32_t> cand;
    uint64_t seen = S;
    {
      std::vector<char> tk(rem.size(), 0);
      scan(phys, rem, S, &tk);
      size_t looked = 0;
      for (size_t i = 0; i < rem.size() && looked < 256; ++i) {
        if (tk[i]) continue;
        ++looked;
        uint64_t nm = phys[rem[i]].needmask & ~seen & allowed;
        while (nm) {
          const uint32_t q = static_cast<uint32_t>(__builtin_ctzll(nm));
          nm &= nm - 1;
          cand.push_back(q);
          seen |= bit(q);
        }
      }
    }
    if (cand.empty()) break;
    size_t best_cnt = cur;
    int best = -1;
    for (auto q : cand) {
      const size_t c = scan(phys, rem, S | bit(q), nullptr);
      if (c > best_cnt) {
        best_cnt = c;
        best = static_cast<int>(q);
      }
    }
    if (best < 0) {
      // no single qubit helps: add the need set of the first blocked op
      std::vector<char> tk(rem.size(), 0);
      scan(phys, rem, S, &tk);
      bool added = false;
      for (size_t i = 0; i < rem.size(); ++i) {
        if (tk[i] || phys[rem[i]].k == PK::Opaque) continue;
        const uint64_t ns = S | phys[rem[i]].needmask;
        if (!(ns & ~allowed) && static_cast<uint32_t>(__builtin_popcountll(ns)) <= m &&
            scan(phys, rem, ns, nullptr) > cur) {
          S = ns;
          cur = scan(phys, rem, S, nullptr);
          added = true;
        }
        break;
      }
      if (!added) break;
      continue;
    }
    S |= bit(static_cast<uint32_t>(best));
    cur = best_cnt;
  }
  return S;
}

}  // namespace

namespace {
bool is_diag(const Op& o) {
  return o.kind == OpKind::Diag || (o.kind == OpKind::Mat1 && o.m[1] == cd(0) && o.m[2] == cd(0));
}
bool touches(const Op& o, uint32_t q) {
  return std::find(o.targets.begin(), o.targets.end(), q) != o.targets.end() ||
         std::find(o.controls.begin(), o.controls.end(), q) != o.controls.end();
}
}  // namespace

// Pauli-X absorption (exact circuit identity).  An uncontrolled X on q is
// dropped when the next non-diagonal use of q is an uncontrolled 1-qubit (or
// dense) gate M on q: M becomes M.X, and the ops in between see q flipped --
// a diagonal with target q swaps d0/d1, a diagonal controlled by q gets a
// negated control (a tile predicate on q = 0); an X on q commutes.  Anything
// else touching q in between keeps the X.  (QFT of a basis state: the preparation X's no longer
// block the controlled phases, which then schedule like QFT|0>.)
void absorb_pauli_x(std::vector<Op>& ops) {
  for (size_t i = 0; i < ops.size(); ++i) {
    const Op& x = ops[i];
    if (x.kind != OpKind::Flip || !x.controls.empty()) continue;
    const uint32_t q = x.targets[0];
    size_t consumer = SIZE_MAX;
    bool ok = true;
    for (size_t j = i + 1; j < ops.size() && ok; ++j) {
      const Op& o = ops[j];
      if (!touches(o, q)) continue;
      if (is_diag(o)) continue;  // target q: d0 <-> d1; control q: negated control
      if (o.kind == OpKind::Flip && o.targets[0] == q &&
          std::find(o.controls.begin(), o.controls.end(), q) == o.controls.end())
        continue;  // X commutes with X (and controls elsewhere are unaffected)
      if (o.controls.empty() && (o.kind == OpKind::Mat1 || o.kind == OpKind::Dense) &&
          std::find(o.targets.begin(), o.targets.end(), q) != o.targets.end()) {
        consumer = j;
        break;
      }
      ok = false;
    }
    if (!ok || consumer == SIZE_MAX) continue;
    for (size_t j = i + 1; j < consumer; ++j) {
      Op& o = ops[j];
      if (!touches(o, q) || !is_diag(o)) continue;
      if (o.kind == OpKind::Mat1) {  // normalise to Diag
        o.kind = OpKind::Diag;
        o.m = {o.m[0], o.m[3]};
      }
      if (o.targets[0] == q) std::swap(o.m[0], o.m[1]);  // target q is flipped
      else o.cneg ^= bit(q);                              // control q now selects 0
    }
    Op& c = ops[consumer];
    if (c.kind == OpKind::Mat1) {
      std::swap(c.m[0], c.m[1]);
      std::swap(c.m[2], c.m[3]);
    } else {  // dense: columns permuted by the flip of q's local bit
      const size_t k = c.targets.size(), dim = size_t(1) << k;
      const size_t b = k - 1 - static_cast<size_t>(std::find(c.targets.begin(), c.targets.end(), q) - c.targets.begin());
      std::vector<cd> mm(c.m.size());
      for (size_t r = 0; r < dim; ++r)
        for (size_t cc = 0; cc < dim; ++cc) mm[r * dim + cc] = c.m[r * dim + (cc ^ (size_t(1) << b))];
      c.m = std::move(mm);
    }
    ops[i].kind = OpKind::Identity;
    ops[i].targets.clear();
  }
}

void plan_tiles(uint32_t n, std::vector<Op>& ops, std::vector<Step>& steps, const TileOptions& opt) {
  if (opt.absorb_x && n >= 6 && !std::getenv("QSB_NO_ABSORB_X")) absorb_pauli_x(ops);
  std::vector<POp> pops = preprocess(ops);
  // Tiny registers cannot host a 16-amplitude-per-thread tile: per-gate kernels.
  if (n < 6) {
    for (auto& p : pops) {
      Step s;
      s.kind = Step::OpStep;
      s.op = p.op;
      steps.push_back(std::move(s));
    }
    return;
  }
  // Sharded states: physical qubits [nl, n) are rank bits.  Tiles only hold
  // local qubits; a non-diagonal gate on a rank bit is preceded by a SwapStep
  // (pairwise half-shard exchange) that brings that qubit into the shard.
  const uint32_t nl = n - opt.global_qubits;
  const uint32_t m = std::min<uint32_t>(nl, opt.m);
  const uint32_t R = m >= opt.r + 4 ? opt.r : static_cast<uint32_t>(kTileMinR);  // register bits
  const uint32_t L = std::min<uint32_t>(opt.low, m - R);
  const uint64_t lowmask = (1ull << L) - 1;
  const uint64_t allmask = nl >= 64 ? ~0ull : (1ull << nl) - 1;  // every local position
  const uint64_t gmask = (n >= 64 ? ~0ull : (1ull << n) - 1) & ~allmask;
  const bool remap = opt.remap && nl > m;

  // Logical -> physical qubit map.  The low L physical qubits are in every
  // tile (coalescing); relabel SWAPs at pass ends move the qubits needed next
  // into them for free.  Every plan ends in the identity layout.
  std::vector<uint32_t> perm(n), inv(n);
  for (uint32_t q = 0; q < n; ++q) perm[q] = inv[q] = q;
  std::vector<POp> phys(pops.size());
  std::vector<POp> extra;  // relabel swaps appended to passes
  extra.reserve(4096);

  std::vector<uint32_t> rem(pops.size());
  for (size_t i = 0; i < pops.size(); ++i) rem[i] = static_cast<uint32_t>(i);

  auto refresh = [&]() {
    for (auto idx : rem) phys[idx] = to_physical(pops[idx], perm);
  };
  // --- definite qubits of a run started from a basis state |b>: value of
  // logical qubit q = parity(b & dmask[q]) ^ dconst[q] while ddef[q].
  std::vector<char> ddef(n, 1), dconst(n, 0);
  std::vector<uint64_t> dmask(n);
  for (uint32_t q = 0; q < n; ++q) dmask[q] = 1ull << q;
  auto undef = [&](uint32_t q) { ddef[q] = 0; };
  auto apply_def = [&](const Op& op) {
    // controls: all definite with a constant literal value 0 => the op is the identity
    bool all_def = true, never = false;
    for (auto c : op.controls) {
      if (!ddef[c]) {
        all_def = false;
        continue;
      }
      const bool want_one = !((op.cneg >> c) & 1);
      if (dmask[c] == 0 && dconst[c] != (want_one ? 1 : 0)) never = true;
    }
    if (never) return;
    switch (op.kind) {
      case OpKind::Identity:
      case OpKind::Diag: return;
      case OpKind::Flip: {
        const uint32_t t = op.targets[0];
        if (!ddef[t]) return;
        if (!all_def) return undef(t);
        if (op.controls.empty()) {
          dconst[t] ^= 1;
        } else if (op.controls.size() == 1) {  // t ^= (c == want)
          const uint32_t c = op.controls[0];
          dmask[t] ^= dmask[c];
          dconst[t] ^= dconst[c] ^ (((op.cneg >> c) & 1) ? 1 : 0);
        } else {
          undef(t);  // AND of two forms is not affine
        }
        return;
      }
      case OpKind::Mat1: {
        const uint32_t t = op.targets[0];
        if (op.m[1] == cd(0) && op.m[2] == cd(0)) return;           // diagonal
        if (op.m[0] == cd(0) && op.m[3] == cd(0) && op.controls.empty() && ddef[t]) {  // X up to phases
          dconst[t] ^= 1;
          return;
        }
        return undef(t);
      }
      case OpKind::Swap:
        if (op.controls.empty()) {
          const uint32_t a = op.targets[0], b2 = op.targets[1];
          std::swap(ddef[a], ddef[b2]);
          std::swap(dmask[a], dmask[b2]);
          std::swap(dconst[a], dconst[b2]);
        } else {
          undef(op.targets[0]);
          undef(op.targets[1]);
        }
        return;
      case OpKind::Dense:
        for (auto t : op.targets) undef(t);
        return;
    }
  };
  auto emit_ready_opaque = [&]() {
    uint64_t blocked = 0;
    std::vector<uint32_t> keep;
    keep.reserve(rem.size());
    for (auto idx : rem) {
      const POp& p = phys[idx];
      if (p.k == PK::Opaque && !(p.qmask & blocked) && !(p.needmask & gmask)) {
        apply_def(pops[idx].op);
        Step s;
        s.kind = Step::OpStep;
        s.op = p.op;
        steps.push_back(std::move(s));
        continue;
      }
      blocked |= p.qmask;
      keep.push_back(idx);
    }
    rem.swap(keep);
  };
  auto swap_phys = [&](uint32_t a, uint32_t b) {
    const uint32_t la = inv[a], lb = inv[b];
    std::swap(perm[la], perm[lb]);
    std::swap(inv[a], inv[b]);
  };
  auto identity = [&]() {
    for (uint32_t q = 0; q < n; ++q)
      if (perm[q] != q) return false;
    return true;
  };
  // One exchange step for a set of disjoint (rank position j, local position p) pairs.
  auto emit_swaps = [&](const std::vector<std::pair<uint32_t, uint32_t>>& pairs) {
    if (pairs.empty()) return;
    Step s;
    s.kind = Step::SwapStep;
    for (auto [j, p] : pairs) {
      s.gpos.push_back(j - nl);
      s.lpos.push_back(p);
    }
    steps.push_back(std::move(s));
    for (auto [j, p] : pairs) swap_phys(j, p);
  };
  const bool batch_exchanges = [] {
    const char* e = std::getenv("QSB_SHARD_BATCH");
    return !e || std::atoi(e) != 0;
  }();
  // Brings every rank bit the op needs into the shard, evicting the local
  // qubits needed furthest in the future (Belady); ties prefer the highest
  // position (the exchanged block is then contiguous).  Other rank bits whose
  // qubit is needed before the evicted one's next use join the same exchange:
  // a k-bit all-to-all moves 1 - 2^-k of a shard, so one more bit costs
  // 2^-(k+1) of a shard instead of a later half-shard exchange.
  auto global_swaps_for = [&](const POp& op) {
    std::vector<size_t> next(n, SIZE_MAX);
    for (size_t k = 0; k < rem.size(); ++k) {
      uint64_t nm = pops[rem[k]].needmask;  // logical
      while (nm) {
        const uint32_t l = static_cast<uint32_t>(__builtin_ctzll(nm));
        nm &= nm - 1;
        if (next[l] == SIZE_MAX) next[l] = k;
      }
    }
    std::vector<uint32_t> order;  // required rank positions, then optional by urgency
    std::vector<uint32_t> optional;
    for (uint32_t j = nl; j < n; ++j) {
      if ((op.needmask >> j) & 1) order.push_back(j);
      else if (batch_exchanges && next[inv[j]] != SIZE_MAX) optional.push_back(j);
    }
    const size_t required = order.size();
    std::stable_sort(optional.begin(), optional.end(),
                     [&](uint32_t a, uint32_t b) { return next[inv[a]] < next[inv[b]]; });
    order.insert(order.end(), optional.begin(), optional.end());
    uint64_t taken = op.qmask;
    std::vector<std::pair<uint32_t, uint32_t>> pairs;
    for (size_t i = 0; i < order.size(); ++i) {
      const uint32_t j = order[i];
      int best = -1;
      for (int p = static_cast<int>(nl) - 1; p >= 0; --p) {
        if ((taken >> p) & 1) continue;
        if (best < 0 || next[inv[p]] > next[inv[best]]) best = p;
      }
      if (best < 0) {
        if (i < required) throw RuntimeError("no local qubit available for a rank-bit exchange");
        break;
      }
      if (i >= required && !(next[inv[j]] < next[inv[best]])) break;
      pairs.push_back({j, static_cast<uint32_t>(best)});
      taken |= bit(static_cast<uint32_t>(best));
    }
    emit_swaps(pairs);
  };

  auto compile_pass_r = [&](uint64_t S, const std::vector<const POp*>& list, const std::vector<uint64_t>& srcs,
                            const std::vector<uint32_t>* sigma, uint32_t Rp) {
    Compiler C;
    C.n = n;
    C.m = m;
    C.R = static_cast<int>(Rp);
    C.t = m - Rp;
    C.L = std::min<uint32_t>(opt.low, m - Rp);
    C.free_load = opt.free_load;
    for (int q = 0; q < 64; ++q) C.tb[q] = -1;
    for (uint32_t q = 0; q < n; ++q)
      if ((S >> q) & 1) {
        C.tb[q] = static_cast<int>(C.S.size());
        C.S.push_back(q);
      }
    if (sigma)  // store lane k holds the tile bit whose output position is k
      for (uint32_t k = 0; k < L; ++k)
        for (uint32_t q = 0; q < n; ++q)
          if ((*sigma)[q] == k) C.lane[k] = C.tb[q];
    C.compile(list);
    return finalize(C, list.size(), srcs, sigma);
  };
  // 13-qubit tiles: 4 register bits (512 threads) or 5 (256 threads x 32
  // amplitudes: fewer shared-memory exchanges, fewer resident warps) -- per
  // pass, whichever pass_cost (measured on B200) says is faster.
  const bool try_r5 = opt.choose_r && m >= 13 && R == 4 && m >= 5 + 4;
  auto compile_pass = [&](uint64_t S, const std::vector<const POp*>& list, const std::vector<uint64_t>& srcs,
                          const std::vector<uint32_t>* sigma = nullptr) {
    auto a = compile_pass_r(S, list, srcs, sigma, R);
    if (!try_r5) return a;
    auto b = compile_pass_r(S, list, srcs, sigma, 5);
    return pass_cost(*b) < pass_cost(*a) - 1e-9 && b->h.bytes <= kTileBlobBytes ? b : a;
  };
  // inputs of the most recent tile pass (to recompile it storing out of place)
  uint64_t last_S = 0;
  std::vector<POp> last_ops;
  std::vector<uint64_t> last_srcs;
  std::shared_ptr<TileProgram> last_prog;
  auto push_step = [&](std::shared_ptr<TileProgram> prog, uint64_t S, size_t gates) {
    if (std::getenv("QSB_PLAN_DEBUG")) {
      int counts[16] = {0};
      for (const auto& o : prog->ops) counts[o.type & 15]++;
      std::fprintf(stderr, "pass %zu: ops=%zu gates=%zu lead=%d transposes=%u mat1=%d flip=%d phase=%d dense=%d relabel=%d S=",
                   steps.size(), prog->ops.size(), gates, int(leading_transpose(*prog)), prog->transposes,
                   counts[TO_MAT1] + counts[TO_MAT1_REAL] + counts[TO_MAT1_RX], counts[TO_FLIP], counts[TO_PHASE],
                   counts[TO_DENSE2] + counts[TO_DENSE3], counts[TO_RELABEL]);
      for (auto q : C_S_debug(S, n)) std::fprintf(stderr, "%u,", q);
      std::fprintf(stderr, "\n");
    }
    Step s;
    s.kind = Step::TileStep;
    s.tile = std::move(prog);
    steps.push_back(std::move(s));
  };

  // With an out-of-place restore at the end, an uncontrolled SWAP whose qubits
  // have no earlier pending op is absorbed into the logical->physical map (no
  // data movement); the accumulated permutation costs one pass at the end
  // (QFT's final bit reversal: 15 swaps -> 1 pass instead of 3-4).
  const bool absorb_swaps = opt.perm_step && opt.global_qubits == 0 && n >= 10;
  auto absorb_ready_swaps = [&]() {
    if (!absorb_swaps) return;
    uint64_t blocked = 0;
    std::vector<uint32_t> keep;
    keep.reserve(rem.size());
    for (auto idx : rem) {
      const POp& p = pops[idx];  // logical
      if (p.k == PK::SwapRel && !(p.qmask & blocked)) {
        swap_phys(perm[p.op.targets[0]], perm[p.op.targets[1]]);
        apply_def(p.op);  // the logical SWAP exchanges the two qubits' states
        continue;
      }
      blocked |= p.qmask;
      keep.push_back(idx);
    }
    rem.swap(keep);
  };
  absorb_ready_swaps();
  refresh();
  emit_ready_opaque();
  while (!rem.empty()) {
    for (size_t before = SIZE_MAX; before != rem.size() && !rem.empty();) {  // absorbing can free opaque ops
      before = rem.size();
      absorb_ready_swaps();
      refresh();
      emit_ready_opaque();
    }
    if (rem.empty()) break;
    refresh();
    // a non-diagonal gate on a rank bit at the head of the program: exchange first
    if (gmask && (phys[rem[0]].needmask & gmask)) {
      global_swaps_for(phys[rem[0]]);
      refresh();
      emit_ready_opaque();
      continue;
    }
    uint64_t S = choose_tile_set(phys, rem, nl <= m ? allmask : lowmask, m, allmask);
    std::vector<char> tk(rem.size(), 0);
    size_t cnt = scan(phys, rem, S, &tk);
    if (cnt == 0) throw RuntimeError("tile planner made no progress");
    const bool last = cnt == rem.size();
    // pad S to exactly m qubits: on the last pass prefer displaced positions
    // (so the layout can be restored for free), else the lowest unused
    if (last && remap)
      for (uint32_t q = 0; q < nl && static_cast<uint32_t>(__builtin_popcountll(S)) < m; ++q)
        if (inv[q] != q) S |= bit(q);
    for (uint32_t q = 0; q < nl && static_cast<uint32_t>(__builtin_popcountll(S)) < m; ++q) S |= bit(q);

    std::vector<size_t> taken_pos;  // positions in rem, program order
    for (size_t i = 0; i < rem.size(); ++i)
      if (tk[i]) taken_pos.push_back(i);

    // Any program-order prefix of the taken ops is dependency-closed, so a
    // program too large for the parameter blob is cut to a fitting prefix.
    size_t take = taken_pos.size();
    std::shared_ptr<TileProgram> prog;
    std::vector<std::pair<uint32_t, uint32_t>> swaps;
    while (true) {
      std::vector<const POp*> list;
      std::vector<uint64_t> srcs;
      for (size_t j = 0; j < take; ++j) {
        list.push_back(&phys[rem[taken_pos[j]]]);
        srcs.push_back(phys[rem[taken_pos[j]]].op.gate_index);
      }
      // layout change at the end of the pass (computed on copies of the map)
      swaps.clear();
      if (remap) {
        std::vector<uint32_t> pm = perm, iv = inv;
        auto sw = [&](uint32_t a, uint32_t b) {
          std::swap(pm[iv[a]], pm[iv[b]]);
          std::swap(iv[a], iv[b]);
          swaps.push_back({a, b});
        };
        const bool all_taken = take == rem.size();
        if (all_taken) {
          // restore the identity on every position inside S
          for (uint32_t p = 0; p < n; ++p) {
            if (!((S >> p) & 1) || iv[p] == p) continue;
            const uint32_t where = pm[p];  // physical position of logical p
            if ((S >> where) & 1) sw(p, where);
          }
        } else {
          // Belady: bring the logical qubits needed soonest into the low slots
          std::vector<size_t> urg(n, SIZE_MAX);
          std::vector<char> in_pass(rem.size(), 0);
          for (size_t j = 0; j < take; ++j) in_pass[taken_pos[j]] = 1;
          size_t k = 0;
          for (size_t i = 0; i < rem.size(); ++i) {
            if (in_pass[i]) continue;
            uint64_t nm = pops[rem[i]].needmask;  // logical
            while (nm) {
              const uint32_t l = static_cast<uint32_t>(__builtin_ctzll(nm));
              nm &= nm - 1;
              if (urg[l] == SIZE_MAX) urg[l] = k;
            }
            ++k;
          }
          std::vector<uint32_t> cands;
          for (uint32_t l = 0; l < n; ++l)
            if (((S >> pm[l]) & 1) && urg[l] != SIZE_MAX) cands.push_back(l);
          std::stable_sort(cands.begin(), cands.end(), [&](uint32_t a, uint32_t b) {
            if (urg[a] != urg[b]) return urg[a] < urg[b];
            return (pm[a] < L) > (pm[b] < L);
          });
          if (cands.size() > L) cands.resize(L);
          std::vector<char> want(n, 0);
          for (auto l : cands) want[l] = 1;
          for (uint32_t p = 0; p < L; ++p) {
            if (want[iv[p]]) continue;
            for (auto l : cands)
              if (pm[l] >= L) {
                sw(p, pm[l]);
                break;
              }
          }
        }
        extra.resize(0);
        for (auto& [a, b] : swaps) extra.push_back(swap_rel(a, b));
        for (const auto& e : extra) list.push_back(&e);
      }
      prog = compile_pass(S, list, srcs);
      if (prog->h.bytes <= kTileBlobBytes || take == 1) {
        last_S = S;
        last_ops.clear();
        for (auto* op : list) last_ops.push_back(*op);
        last_srcs = srcs;
        last_prog = prog;
        break;
      }
      take = std::max<size_t>(1, take * 3 / 4);
    }
    if (prog->h.bytes > kTileBlobBytes) throw RuntimeError("tile program for one op exceeds the parameter blob");
    const std::vector<uint32_t> perm_at_start = perm;
    for (auto& [a, b] : swaps) swap_phys(a, b);
    std::vector<char> used(rem.size(), 0);
    for (size_t j = 0; j < take; ++j) used[taken_pos[j]] = 1;
    std::vector<uint32_t> keep;
    for (size_t i = 0; i < rem.size(); ++i)
      if (!used[i]) keep.push_back(rem[i]);
    // definite qubits at the start of this pass (outside the tile: zero tiles;
    // inside: zero amplitudes that need not be read), then the pass's effect
    std::vector<uint32_t> dpos;
    std::vector<uint64_t> dm;
    std::vector<uint8_t> dc;
    for (uint32_t q = 0; q < n; ++q)
      if (ddef[q]) {
        dpos.push_back(perm_at_start[q]);
        dm.push_back(dmask[q]);
        dc.push_back(static_cast<uint8_t>(dconst[q]));
      }
    for (size_t j = 0; j < take; ++j) apply_def(pops[rem[taken_pos[j]]].op);
    push_step(std::move(prog), S, take);
    steps.back().def_pos = std::move(dpos);
    steps.back().def_mask = std::move(dm);
    steps.back().def_const = std::move(dc);
    rem.swap(keep);
    refresh();
    emit_ready_opaque();
  }
  // Restore the logical layout: rank bits by exchanges, then relabel-only
  // passes over the displaced local positions.
  while (true) {
    std::vector<std::pair<uint32_t, uint32_t>> pairs;  // one all-to-all for every directly fixable bit
    int misplaced = -1;
    for (uint32_t j = nl; j < n; ++j) {
      if (inv[j] == j) continue;
      misplaced = static_cast<int>(j);
      if (perm[j] < nl) pairs.push_back({j, perm[j]});  // logical j lives on local position perm[j]
    }
    if (misplaced < 0) break;
    if (pairs.empty()) pairs.push_back({perm[misplaced], nl - 1});  // on another rank bit: route via a local one
    emit_swaps(pairs);
  }
  if (opt.perm_step && opt.global_qubits == 0 && n >= 10 && !identity()) {
    const std::vector<uint32_t> sigma(inv.begin(), inv.end());  // data at bit p belongs to logical inv[p]
    // Fold into the last tile pass (out-of-place store through sigma) when it
    // ends the plan and holds the qubits that land on the low output bits.
    bool folded = false;
    if (opt.fold_perm && !steps.empty() && steps.back().kind == Step::TileStep && steps.back().tile == last_prog) {
      bool lanes_in = true;
      for (uint32_t k = 0; k < L; ++k) lanes_in = lanes_in && ((last_S >> perm[k]) & 1);
      if (lanes_in) {
        std::vector<const POp*> list;
        for (const auto& o : last_ops) list.push_back(&o);
        auto prog = compile_pass(last_S, list, last_srcs, &sigma);
        if (prog->h.bytes <= kTileBlobBytes) {
          steps.back().tile = std::move(prog);
          folded = true;
        }
      }
    }
    if (!folded) {
      Step s;
      s.kind = Step::PermStep;
      s.perm = sigma;
      steps.push_back(std::move(s));
    }
    for (uint32_t q = 0; q < n; ++q) perm[q] = inv[q] = q;
  }
  while (!identity()) {
    uint64_t S = lowmask;
    for (uint32_t p = 0; p < nl && static_cast<uint32_t>(__builtin_popcountll(S)) < m; ++p)
      if (inv[p] != p) {
        S |= bit(p);
        if (static_cast<uint32_t>(__builtin_popcountll(S)) < m) S |= bit(perm[p]);
      }
    for (uint32_t q = 0; q < nl && static_cast<uint32_t>(__builtin_popcountll(S)) < m; ++q) S |= bit(q);
    std::vector<std::pair<uint32_t, uint32_t>> swaps;
    for (uint32_t p = 0; p < nl; ++p) {
      if (!((S >> p) & 1) || inv[p] == p) continue;
      const uint32_t where = perm[p];
      if ((S >> where) & 1) {
        swaps.push_back({p, where});
        swap_phys(p, where);
      }
    }
    if (swaps.empty()) throw RuntimeError("layout restore made no progress");
    extra.clear();
    for (auto& [a, b] : swaps) extra.push_back(swap_rel(a, b));
    std::vector<const POp*> list;
    for (const auto& e : extra) list.push_back(&e);
    push_step(compile_pass(S, list, {}), S, 0);
  }
}

// Per-pass times measured on B200 (30 qubits, random30 plan, both register
// widths on the same passes; profiles/r2/random30_r4_vs_r5.txt), in units of
// a light 13-qubit pass (5.65 ms): with 4 register bits <= 2 buffered
// exchanges 1.0, 3: 1.28, 4: 1.5; with 5 register bits <= 1: 1.05, 2: 1.13,
// 3: 1.26, 4: 1.37.  12-qubit passes (two CTAs per SM): 1.0 up to two
// exchanges, +17% per further one.
double pass_cost(const TileProgram& tp) {
  const uint32_t tr = buffered_transposes(tp, true);
  if (tp.h.m >= 13) {
    if (tp.h.r >= 5) {
      static const double c5[] = {1.05, 1.05, 1.13, 1.26};
      return tr < 4 ? c5[tr] : 1.26 + 0.11 * (tr - 3);
    }
    static const double c4[] = {1.0, 1.0, 1.0, 1.28};
    return tr < 4 ? c4[tr] : 1.28 + 0.22 * (tr - 3);
  }
  return 1.0 + 0.17 * (tr > 2 ? tr - 2 : 0);
}

double plan_cost(const std::vector<Step>& steps) {
  double c = 0;
  for (const Step& st : steps) c += st.kind == Step::TileStep ? pass_cost(*st.tile) : 1.0;
  return c;
}

void plan_tiles(uint32_t n, std::vector<Op>& ops, std::vector<Step>& steps, uint32_t global_qubits, bool sharded,
                bool in_place_only) {
  TileOptions o = tile_options_from_env();
  o.global_qubits = global_qubits;
  if (sharded || in_place_only) o.perm_step = false;  // restore the layout in place
  std::vector<uint32_t> ms{o.m};
  // 13-qubit tiles when every shard has 2^13 tiles and more (enough CTAs)
  if (!std::getenv("QSB_TILE_M") && n - global_qubits >= 26) ms.push_back(13);
  std::vector<int> remaps{0, 1};
  if (const char* e = std::getenv("QSB_TILE_REMAP")) remaps = {std::atoi(e) != 0 ? 1 : 0};
  // The candidates are planned concurrently (independent; the planner has no
  // shared mutable state) and the cheapest is kept (ties: the first).
  struct Cand {
    TileOptions o;
    std::vector<Op> ops;
    std::vector<Step> steps;
    double cost = 0;
    std::string err;
  };
  std::vector<Cand> cands;
  for (uint32_t m : ms)
    for (int r : remaps) {
      Cand c;
      c.o = o;
      c.o.m = m;
      c.o.remap = r != 0;
      c.ops = ops;
      cands.push_back(std::move(c));
    }
  auto work = [](Cand& c, uint32_t nq) {
    try {
      plan_tiles(nq, c.ops, c.steps, c.o);
      c.cost = plan_cost(c.steps);
    } catch (const std::exception& e) {
      c.err = e.what();
    }
  };
  std::vector<std::thread> pool;
  for (size_t i = 1; i < cands.size(); ++i) pool.emplace_back(work, std::ref(cands[i]), n);
  work(cands[0], n);
  for (auto& t : pool) t.join();
  size_t best = 0;
  for (size_t i = 0; i < cands.size(); ++i) {
    if (!cands[i].err.empty()) throw RuntimeError(cands[i].err);
    if (cands[i].cost < cands[best].cost - 1e-9) best = i;
  }
  steps = std::move(cands[best].steps);
  ops = std::move(cands[best].ops);
}

}  // namespace qsb
