// Host emulator of libqsb execution plans -- TEST INFRASTRUCTURE ONLY.
//
// Links the product's planner sources (gates.cpp, fusion.cpp, tile_plan.cpp)
// and replays the planned steps on a host array exactly as the CUDA kernels
// would (k_tile's micro-program semantics, thread by thread in lockstep), so
// planner and micro-program bugs are caught by the CPU suite against the
// oracle.  Never part of the product path.
#include <array>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "../paper_2212_14201_b200/csrc/fusion.hpp"
#include "../paper_2212_14201_b200/csrc/gates.hpp"
#include "../paper_2212_14201_b200/csrc/plan.hpp"
#include "../paper_2212_14201_b200/csrc/tile.hpp"

using qsb::cd;

namespace {

cd c2(const double2& d) { return cd(d.x, d.y); }

void emu_op(std::vector<cd>& a, uint32_t n, const qsb::Op& op) {
  uint64_t cmask = 0;
  for (auto c : op.controls) cmask |= 1ull << c;
  const uint64_t N = 1ull << n;
  switch (op.kind) {
    case qsb::OpKind::Identity: return;
    case qsb::OpKind::Mat1: {
      const uint64_t b = 1ull << op.targets[0];
      for (uint64_t i = 0; i < N; ++i)
        if (!(i & b) && (i & cmask) == cmask) {
          const cd x = a[i], y = a[i | b];
          a[i] = op.m[0] * x + op.m[1] * y;
          a[i | b] = op.m[2] * x + op.m[3] * y;
        }
      return;
    }
    case qsb::OpKind::Diag: {
      const uint64_t b = 1ull << op.targets[0];
      for (uint64_t i = 0; i < N; ++i)
        if ((i & cmask) == cmask) a[i] *= (i & b) ? op.m[1] : op.m[0];
      return;
    }
    case qsb::OpKind::Flip: {
      const uint64_t b = 1ull << op.targets[0];
      for (uint64_t i = 0; i < N; ++i)
        if (!(i & b) && (i & cmask) == cmask) std::swap(a[i], a[i | b]);
      return;
    }
    case qsb::OpKind::Swap: {
      const uint64_t ba = 1ull << op.targets[0], bb = 1ull << op.targets[1];
      for (uint64_t i = 0; i < N; ++i)
        if ((i & ba) && !(i & bb) && (i & cmask) == cmask) std::swap(a[i], a[(i & ~ba) | bb]);
      return;
    }
    case qsb::OpKind::Dense: {
      const size_t k = op.targets.size(), dim = size_t(1) << k;
      uint64_t tmask = 0;
      for (auto t : op.targets) tmask |= 1ull << t;
      std::vector<cd> in(dim);
      for (uint64_t i = 0; i < N; ++i) {
        if ((i & tmask) || (i & cmask) != cmask) continue;
        auto idx = [&](size_t r) {
          uint64_t x = i;
          for (size_t bb = 0; bb < k; ++bb)
            if ((r >> bb) & 1) x |= 1ull << op.targets[k - 1 - bb];
          return x;
        };
        for (size_t c = 0; c < dim; ++c) in[c] = a[idx(c)];
        for (size_t r = 0; r < dim; ++r) {
          cd s = 0;
          for (size_t c = 0; c < dim; ++c) s += op.m[r * dim + c] * in[c];
          a[idx(r)] = s;
        }
      }
      return;
    }
  }
}

uint64_t regoff(int p, const unsigned long long (&rs)[qsb::kTileMaxR], int R) {
  uint64_t o = 0;
  for (int k = 0; k < R; ++k)
    if ((p >> k) & 1) o |= rs[k];
  return o;
}

void emu_tile(std::vector<cd>& a, const qsb::TileProgram& tp) {
  const qsb::TileHeader& h = tp.h;
  const int T = 1 << h.t;
  const int R = static_cast<int>(h.r), NS = 1 << R;
  std::vector<cd> sm(size_t(1) << h.m);
  std::vector<std::array<cd, qsb::kTileMaxSlots>> v(T);
  std::vector<uint64_t> G(T);
  std::vector<cd> outbuf;  // out-of-place pass: written through the final permutation
  if (h.oop) outbuf.assign(a.size(), cd(0));
  for (uint64_t tile = 0; tile < h.ntiles; ++tile) {
    uint64_t base = tile;
    for (uint32_t b = 0; b < h.m; ++b) {
      const uint32_t p = h.S[b];
      base = ((base >> p) << (p + 1)) | (base & ((1ull << p) - 1));
    }
    unsigned long long rs[qsb::kTileMaxR] = {};
    for (int k = 0; k < R; ++k) rs[k] = h.load.rs[k];
    for (int tid = 0; tid < T; ++tid) {
      G[tid] = base;
      for (uint32_t k = 0; k < h.t; ++k)
        if ((tid >> k) & 1) G[tid] |= 1ull << h.load.tq[k];
      for (int p = 0; p < NS; ++p) v[tid][p] = a[G[tid] | regoff(p, rs, R)];
    }
    for (const qsb::TOp& o : tp.ops) {
      if (o.type == qsb::TO_TRANSPOSE) {
        const uint32_t* mt = tp.meta.data() + o.meta;
        const uint32_t TB = h.t;
        for (int tid = 0; tid < T; ++tid) {
          uint32_t Tw = 0;
          for (uint32_t k = 0; k < TB; ++k)
            if ((tid >> k) & 1) Tw ^= mt[k];
          for (int p = 0; p < NS; ++p) {
            uint32_t ad = Tw;
            for (int k = 0; k < R; ++k)
              if ((p >> k) & 1) ad ^= mt[TB + k];
            sm.at(ad) = v[tid][p];
          }
        }
        for (int tid = 0; tid < T; ++tid) {
          uint32_t Tr = 0;
          for (uint32_t k = 0; k < TB; ++k)
            if ((tid >> k) & 1) Tr ^= mt[TB + R + k];
          for (int p = 0; p < NS; ++p) {
            uint32_t ad = Tr;
            for (int k = 0; k < R; ++k)
              if ((p >> k) & 1) ad ^= mt[2 * TB + R + k];
            v[tid][p] = sm.at(ad);
          }
          G[tid] = base;
          for (uint32_t k = 0; k < TB; ++k)
            if ((tid >> k) & 1) G[tid] |= 1ull << mt[2 * TB + 2 * R + k];
        }
        continue;
      }
      if (o.type == qsb::TO_RELABEL) {
        for (int tid = 0; tid < T; ++tid) {
          G[tid] = base;
          for (uint32_t k = 0; k < h.t; ++k)
            if ((tid >> k) & 1) G[tid] |= 1ull << tp.meta[o.meta + k];
        }
        continue;
      }
      for (int tid = 0; tid < T; ++tid) {
        if ((G[tid] & o.gmask) != o.gval) continue;
        auto& r = v[tid];
        const double2* c = tp.coef.data() + o.coef;
        switch (o.type) {
          case qsb::TO_MAT1:
          case qsb::TO_MAT1_REAL:
          case qsb::TO_MAT1_RX: {
            const int K = o.k;
            for (int p = 0; p < NS; ++p) {
              if (p & (1 << K)) continue;
              if ((p & o.rmask) != o.rval) continue;
              const int p1 = p | (1 << K);
              const cd x = r[p], y = r[p1];
              r[p] = c2(c[0]) * x + c2(c[1]) * y;
              r[p1] = c2(c[2]) * x + c2(c[3]) * y;
            }
            break;
          }
          case qsb::TO_FLIP: {
            const int K = o.k;
            for (int p = 0; p < NS; ++p) {
              if (p & (1 << K)) continue;
              if ((p & o.rmask) != o.rval) continue;
              std::swap(r[p], r[p | (1 << K)]);
            }
            break;
          }
          case qsb::TO_PHASE: {
            cd F = c2(c[NS]);
            for (uint32_t j = 0; j < o.nlist; ++j)
              if ((G[tid] >> tp.meta[o.meta + j]) & 1) F *= c2(c[NS + 1 + j]);
            for (int p = 0; p < NS; ++p)
              if ((p & o.rmask) == o.rval) r[p] *= F * c2(c[p]);
            break;
          }
          case qsb::TO_DENSE2:
          case qsb::TO_DENSE3: {
            const int KD = o.type == qsb::TO_DENSE2 ? 2 : 3, Gd = 1 << KD;
            for (int hi = 0; hi < (NS >> KD); ++hi) {
              const int p0 = hi << KD;
              if ((p0 & o.rmask) != o.rval) continue;
              cd in[8];
              for (int q = 0; q < Gd; ++q) in[q] = r[p0 + q];
              for (int rr = 0; rr < Gd; ++rr) {
                cd s = 0;
                for (int q = 0; q < Gd; ++q) s += c2(c[rr * Gd + q]) * in[q];
                r[p0 + rr] = s;
              }
            }
            break;
          }
          default: break;
        }
      }
    }
    for (int k = 0; k < R; ++k) rs[k] = h.store.rs[k];
    if (h.oop) {
      uint64_t bo = 0;
      for (uint32_t i = 0; i + h.m < h.n; ++i)
        if ((tile >> i) & 1) bo |= 1ull << h.out_pos[i];
      for (int tid = 0; tid < T; ++tid) {
        uint64_t go = bo;
        for (uint32_t k = 0; k < h.t; ++k)
          if ((tid >> k) & 1) go |= 1ull << h.store.tq[k];
        for (int p = 0; p < NS; ++p) outbuf[go | regoff(p, rs, R)] = v[tid][p];
      }
      continue;
    }
    for (int tid = 0; tid < T; ++tid)
      for (int p = 0; p < NS; ++p) a[G[tid] | regoff(p, rs, R)] = v[tid][p];
  }
  if (h.oop) a.swap(outbuf);
}

}  // namespace

extern "C" {

// Plans `gates` exactly as libqsb does and replays the plan on amps (2^n
// complex, interleaved, in/out).  Returns 0, or -1 with the message in err.
int te_run(uint32_t n, const qs_gate* gates, uint64_t count, uint32_t mode, uint32_t maxk, uint32_t tile_m,
           uint32_t low, double* amps, char* err, uint64_t* passes, uint32_t global_qubits, int remap) {
  try {
    std::vector<qsb::Op> ops;
    for (uint64_t i = 0; i < count; ++i) qsb::validate_gate(gates[i], n);
    std::vector<qsb::Step> steps;
    if (mode == QS_PLAN_DENSE_FUSION) {
      auto fused = qsb::fuse_gate_run(gates, count, n, maxk);
      for (auto& r : fused) {
        r.bind();
        ops.push_back(qsb::lower_gate(r.g, n, false));
      }
    } else {
      for (uint64_t i = 0; i < count; ++i) ops.push_back(qsb::lower_gate(gates[i], n, false));
    }
    if (mode == QS_PLAN_DENSE_FUSION || mode == QS_PLAN_UNFUSED) {
      for (auto& op : ops) {
        qsb::Step s;
        s.op = op;
        steps.push_back(s);
      }
    } else {
      qsb::TileOptions opt;
      opt.m = tile_m;
      opt.low = low;
      if (const char* e = std::getenv("QSB_TILE_R")) opt.r = static_cast<uint32_t>(std::atoi(e));
      opt.global_qubits = global_qubits;
      if (remap >= 0) {
        opt.remap = remap != 0;
        qsb::plan_tiles(n, ops, steps, opt);
      } else {  // as the library does: keep the plan with fewer steps
        std::vector<qsb::Op> copy = ops;
        std::vector<qsb::Step> a1, a2;
        opt.remap = false;
        qsb::plan_tiles(n, copy, a1, opt);
        opt.remap = true;
        qsb::plan_tiles(n, ops, a2, opt);
        steps = a2.size() < a1.size() ? std::move(a2) : std::move(a1);
      }
    }
    std::vector<cd> a(size_t(1) << n);
    std::memcpy(a.data(), amps, a.size() * sizeof(cd));
    const char* lim = std::getenv("TE_MAX_STEPS");
    const size_t max_steps = lim ? static_cast<size_t>(std::atoll(lim)) : steps.size();
    for (size_t i = 0; i < steps.size() && i < max_steps; ++i) {
      const auto& s = steps[i];
      if (s.kind == qsb::Step::OpStep) {
        emu_op(a, n, s.op);
      } else if (s.kind == qsb::Step::SwapStep) {  // exchange = physical bit swaps
        for (size_t b = 0; b < s.gpos.size(); ++b) {
          qsb::Op sw;
          sw.kind = qsb::OpKind::Swap;
          sw.targets = {n - global_qubits + s.gpos[b], s.lpos[b]};
          emu_op(a, n, sw);
        }
      } else if (s.kind == qsb::Step::PermStep) {  // bit q of every index -> bit perm[q]
        std::vector<cd> b(a.size());
        for (uint64_t i = 0; i < a.size(); ++i) {
          uint64_t o = 0;
          for (uint32_t q = 0; q < n; ++q)
            if ((i >> q) & 1) o |= 1ull << s.perm[q];
          b[o] = a[i];
        }
        a.swap(b);
      } else {
        emu_tile(a, *s.tile);
      }
    }
    std::memcpy(amps, a.data(), a.size() * sizeof(cd));
    if (passes) *passes = steps.size();
    return 0;
  } catch (const std::exception& e) {
    std::strncpy(err, e.what(), 255);
    err[255] = 0;
    return -1;
  }
}

// Step-wise access to a sharded plan, for the multi-process (gloo) tests: each
// rank replays the non-exchange steps on its own shard and performs the
// exchanges itself.
struct te_plan {
  std::unique_ptr<qsb::Plan> p;
};

int te_plan_create(uint32_t n, uint32_t g, const qs_gate* gates, uint64_t count, te_plan** out, char* err) {
  try {
    auto h = std::make_unique<te_plan>();
    h->p = std::make_unique<qsb::Plan>();
    h->p->n = n;
    h->p->g = g;
    std::vector<qsb::Op> ops;
    for (uint64_t i = 0; i < count; ++i) qsb::validate_gate(gates[i], n);
    for (uint64_t i = 0; i < count; ++i) ops.push_back(qsb::lower_gate(gates[i], n, false));
    qsb::plan_tiles(n, ops, h->p->steps, g, /*sharded=*/g > 0);  // as qs_plan_create_sharded
    *out = h.release();
    return 0;
  } catch (const std::exception& e) {
    std::strncpy(err, e.what(), 255);
    err[255] = 0;
    return -1;
  }
}

void te_plan_free(te_plan* h) { delete h; }
uint64_t te_plan_steps(te_plan* h) { return h->p->steps.size(); }
int te_plan_step(te_plan* h, uint64_t i, uint32_t* nbits, uint32_t* gpos, uint32_t* lpos) {
  const auto& s = h->p->steps[i];
  *nbits = static_cast<uint32_t>(s.gpos.size());
  for (size_t b = 0; b < s.gpos.size(); ++b) {
    gpos[b] = s.gpos[b];
    lpos[b] = s.lpos[b];
  }
  return static_cast<int>(s.kind);
}

// Runs non-exchange step i on a local shard: `shard` holds the 2^(n-g)
// amplitudes of rank `rank`.  The shard is embedded in a 2^n vector that is
// zero elsewhere; a correct sharded plan never moves amplitude across rank
// bits between exchanges, which the caller's comparison checks.
int te_exec_step(te_plan* h, uint64_t i, uint32_t rank, double* shard) {
  const auto& s = h->p->steps[i];
  const uint32_t n = h->p->n, nl = n - h->p->g;
  std::vector<cd> a(size_t(1) << n);
  const size_t base = static_cast<size_t>(rank) << nl;
  std::memcpy(a.data() + base, shard, (size_t(1) << nl) * sizeof(cd));
  if (s.kind == qsb::Step::OpStep) emu_op(a, n, s.op);
  else if (s.kind == qsb::Step::TileStep) emu_tile(a, *s.tile);
  else return -1;
  double leak = 0;
  for (size_t k = 0; k < a.size(); ++k)
    if ((k >> nl) != rank) leak += std::norm(a[k]);
  std::memcpy(shard, a.data() + base, (size_t(1) << nl) * sizeof(cd));
  return leak == 0 ? 0 : -2;
}

}  // extern "C"

