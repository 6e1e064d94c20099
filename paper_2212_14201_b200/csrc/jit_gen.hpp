// CUDA source generator for one tile pass (included by jit.cpp only).
//
// Emits straight-line code over 2^r (16 or 32) SSA amplitude values per thread:
//   * FLIPs on register bits (and register-controlled CNOTs) are renamings;
//   * diagonal phases are deferred: a per-thread scalar (thread / tile-
//     dependent factors) that commutes with every register-local gate, and
//     per-slot constants (register-qubit factors) that commute with a 2x2 on a
//     pair whenever both slots carry the same constant; both are applied only
//     when data leaves the thread (transpose, store) or a gate mixes slots with
//     different constants;
//   * factors that depend only on thread bits are computed once per thread
//     before the tile loop.
#pragma once

#include <complex>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "tile.hpp"

namespace qsb {
namespace jitgen {

inline std::string hexll(unsigned long long v) {
  char b[32];
  std::snprintf(b, sizeof b, "0x%llxull", v);
  return b;
}

struct Gen {
  const TileProgram& tp;
  std::ostringstream pro;   // before the tile loop (per-thread constants)
  std::ostringstream s;     // tile-loop body
  const int R;              // register bits
  const int NS;             // register slots (2^R)
  std::string name[kTileMaxSlots];
  cd K[kTileMaxSlots];                 // pending per-slot constant factors
  std::string Fp;           // pending per-thread scalar factor (empty = 1)
  std::string Fg;           // pending per-tile scalar (phases of qubits outside the tile; empty = 1)
  cd Kg = 1.0;              // pending tile-wide constant scalar
  std::vector<double2> extra;  // coefficients appended after tp.coef
  uint32_t cur_tq[kTileMaxT] = {};
  int counter = 0;
  bool prefetch = true;
  // from_basis: the pass starts from the basis state |basis> (kernel
  // parameter) instead of reading HBM -- the reset fused into the first pass.
  bool from_basis = false;
  // exchange-fused variant (sharded plans): the pass's stores go straight to
  // the owners' free buffers after the rank-bit exchange that follows it --
  // destination shard = bits of the local index at xlpos, local index with
  // those bits replaced by this rank's bits (xaval, a kernel parameter).
  uint32_t xk = 0;
  uint32_t xlpos[4] = {};
  // single_buf: the prefetch buffer doubles as the transpose buffer (64 KiB
  // per CTA, two resident CTAs per SM); the next tile's copies are issued
  // after the last transpose has read the buffer.
  bool single_buf = false;
  // early (single_buf only): the first `early` register slots of the next
  // tile are staged in a second region PE and issued as soon as the current
  // tile has read them (the rest follow the last transpose), so most of the
  // next tile's HBM reads overlap this tile's transposes.
  uint32_t early = 0;
  // sparse: amplitudes whose definite tile qubits (imask / ival, kernel
  // parameters) disagree are zero -- they are set, not read (runs from a
  // basis state: the first passes touch only a sliver of each tile)
  bool sparse = false;
  bool sparse_zero_store = false;  // QSB_SPARSE_ZERO_STORE=1: stage the zeros too (A/B)
  // zskip: amplitudes whose qubits in omask disagree with oval (kernel
  // parameters: qubits still definite when the pass ends) are zero after the
  // pass and never read before they are written again -- not stored
  bool zskip = false;
  // zwarp_qubits (zskip passes): tile qubits definite from the start to the
  // end of the pass.  If they sit on the same thread bits in every register
  // layout of the pass (never gated, never exchanged), the thread index is
  // permuted so that they land on the warp bits: a warp whose bits disagree
  // with ival holds only zeros for the whole pass and just keeps the block
  // barriers in step (no loads, arithmetic or stores).
  unsigned long long zwarp_qubits = 0;
  int zw_pos[kTileMaxT] = {};  // thread bit -> physical tid bit (identity unless zero warps apply)
  std::string zw_cond;        // per-thread: this warp holds only zeros
  // reduce: the pass also sums |a_i|^2 (i + 1) over what it stores (the
  // bench checksum, bench.hpp:141-148) -- one partial per CTA into red[]
  bool reduce = false;
  int transposes_total = 0;
  // tma: the next tile is staged by bulk copies (cp.async.bulk, one per run of
  // the always-resident low qubits, issued by warp 0 and completing on one
  // mbarrier) into a run-major buffer, instead of 16 per-thread LDGSTS; the
  // first register layout is the coalesced load layout (no fused transpose)
  bool tma = false;
  bool use_tma = false;
  uint32_t trank = 0, ta[5] = {}, tl[5] = {};  // tensor-map segments (tma_segments)
  // Warp-local transposes: when the qubits on thread bits >= 5 stay put, every
  // warp exchanges only its own amplitudes (under one exchange's swizzle each
  // has its own smem slot), so the barrier between the writes and the reads
  // is a __syncwarp; the barrier before the writes stays block-wide.
  bool tile_barrier_done = false;
  bool warp_local_ok = true;

  // Per-thread flip frame: a CNOT whose control is a thread bit and whose
  // target is register bit k is not applied with selects; it is recorded as
  // "register slot p holds logical slot p ^ (t ? 2^k : 0)" (t: the thread's
  // predicate).  Ops that commute with it (gates on other register bits,
  // frame-invariant phases) run unchanged; the next exchange or the store
  // absorbs it into its addresses (the smem swizzle and the register strides
  // are XOR-linear in the slot index), and anything else materialises the
  // selects first.  QSB_NO_FLIP_FRAME=1 applies every such flip at once.
  bool flip_frame = true;
  std::vector<std::pair<int, std::string>> frame;  // (register bit, predicate)
  // applies the pending flips on the register bits in `bits` (selects)
  const char* mat_reason = "";
  void materialize(uint32_t bits) {
    for (size_t i = 0; i < frame.size();) {
      const int Kb = frame[i].first;
      if (!((bits >> Kb) & 1u)) {
        ++i;
        continue;
      }
      const std::string t = frame[i].second;
      if (std::getenv("QSB_FRAME_DEBUG")) s << "    // materialize: " << mat_reason << "\n";
      frame.erase(frame.begin() + static_cast<long>(i));
      for (int p = 0; p < NS; ++p) {
        if ((p >> Kb) & 1) continue;
        const int p1 = p | (1 << Kb);
        flush_pair(p, p1);
        const std::string a = name[p], b = name[p1];
        const std::string na = fresh(), nb = fresh();
        s << "    const double2 " << na << " = " << t << " ? " << b << " : " << a << ";\n";
        s << "    const double2 " << nb << " = " << t << " ? " << a << " : " << b << ";\n";
        name[p] = na;
        name[p1] = nb;
      }
    }
  }
  // per-thread XOR of the frame's slot offsets (cols[k]: register bit k's
  // smem swizzle column or HBM stride)
  std::string frame_xor(const uint32_t* cols) const {
    std::ostringstream e;
    e << "0u";
    for (auto& f : frame) e << " ^ (" << f.second << " ? " << cols[f.first] << "u : 0u)";
    return e.str();
  }
  std::string frame_xor(const unsigned long long* cols) const {
    std::ostringstream e;
    e << "0ull";
    for (auto& f : frame) e << " ^ (" << f.second << " ? " << hexll(cols[f.first]) << " : 0ull)";
    return e.str();
  }

  // Tile-wide phase factors from qubits outside the tile: a product over up
  // to n-m bits of the tile's global index.  Bits are grouped in chunks of 6
  // of the compact tile index tix (tile | rank_base >> m); a chunk holding >= 2
  // factors becomes a 64-entry table in shared memory, built once per CTA, so
  // the per-tile cost is one lookup + one complex multiply per chunk.
  struct Table {
    uint32_t chunk, off;
    std::vector<std::pair<uint32_t, uint32_t>> bits;  // (bit within chunk, coefficient index)
  };
  std::vector<Table> tables;
  uint32_t table_entries = 0;
  static constexpr uint32_t kChunk = 6, kMaxTableEntries = 32 * 64;
  uint32_t tix_bit(uint32_t q) const {  // compact tile-index bit of an outside qubit
    uint32_t below = 0;
    for (uint32_t b = 0; b < tp.h.m; ++b) below += tp.h.S[b] < q;
    return q - below;
  }

  explicit Gen(const TileProgram& p) : tp(p), R(static_cast<int>(p.h.r)), NS(1 << p.h.r) {
    for (auto& k : K) k = 1.0;
  }

  std::string fresh(const char* pfx = "v") { return pfx + std::to_string(counter++); }
  // tile-local bit (position in S) of global qubit q
  uint32_t tile_bit(uint32_t q) const {
    for (uint32_t b = 0; b < tp.h.m; ++b)
      if (tp.h.S[b] == q) return b;
    throw RuntimeError("jit: qubit outside the tile");
  }
  // tile-local index offset of register slot p in the load layout
  uint32_t tile_off(int p) const {
    uint32_t o = 0;
    for (int k = 0; k < R; ++k)
      if ((p >> k) & 1) o |= 1u << tile_bit(static_cast<uint32_t>(__builtin_ctzll(tp.h.load.rs[k])));
    return o;
  }
  // leading tile bits that are the global qubits 0, 1, ...: one contiguous run
  uint32_t run_bits() const {
    uint32_t b = 0;
    while (b < tp.h.m && tp.h.S[b] == b) ++b;
    return b;
  }
  std::string coef(uint32_t i) { return "P.c[" + std::to_string(i) + "]"; }
  cd coefv(uint32_t i) const { return cd(tp.coef[i].x, tp.coef[i].y); }
  // compile-time constants, one coefficient slot per distinct value (equal
  // expressions such as cmul(F, P.c[i]) are then common subexpressions)
  std::map<std::pair<double, double>, uint32_t> kidx;
  std::string kconst(cd v) {
    auto it = kidx.find({v.real(), v.imag()});
    if (it != kidx.end()) return coef(it->second);
    extra.push_back(make_double2(v.real(), v.imag()));
    const uint32_t i = static_cast<uint32_t>(tp.coef.size() + extra.size() - 1);
    kidx[{v.real(), v.imag()}] = i;
    return coef(i);
  }
  static bool one(cd v) { return v == cd(1.0); }

  void emit_G(const uint32_t* tq, bool decl) {
    s << "    " << (decl ? "unsigned long long " : "") << "G = base";
    for (uint32_t k = 0; k < tp.h.t; ++k) s << " | ((unsigned long long)((tid >> " << k << ") & 1u) << " << tq[k] << ")";
    s << ";\n";
    for (uint32_t k = 0; k < tp.h.t; ++k) cur_tq[k] = tq[k];
  }

  std::string pred(const TOp& o) {
    if (!o.gmask) return "";
    const std::string t = fresh("t");
    s << "    const bool " << t << " = (G & " << hexll(o.gmask) << ") == " << hexll(o.gval) << ";\n";
    return t;
  }

  void set(int p, const std::string& expr, const std::string& t) {
    const std::string nv = fresh();
    if (t.empty()) s << "    const double2 " << nv << " = " << expr << ";\n";
    else s << "    const double2 " << nv << " = " << t << " ? " << expr << " : " << name[p] << ";\n";
    name[p] = nv;
  }

  // --- deferred phases ----------------------------------------------------
  void flush_const(int p) {
    if (one(K[p])) return;
    set(p, "cmul(" + name[p] + ", " + kconst(K[p]) + ")", "");
    K[p] = 1.0;
  }
  void flush_pair(int p, int p1) {
    if (K[p] != K[p1]) {
      flush_const(p);
      flush_const(p1);
    }
  }
  // Applies the pending per-thread scalar and per-slot constants (and, at the
  // store, the tile-wide scalar Kg).
  void flush_all(bool with_global) {
    const cd g = with_global ? Kg : cd(1.0);
    if (with_global && !Fg.empty()) {  // tile-wide factors wait for the store
      if (Fp.empty()) {
        Fp = Fg;
      } else {
        const std::string nf = fresh("FP");
        s << "    const double2 " << nf << " = cmul(" << Fp << ", " << Fg << ");\n";
        Fp = nf;
      }
      Fg.clear();
    }
    for (int p = 0; p < NS; ++p) {
      const cd kp = K[p] * g;
      const bool k1 = one(kp);
      if (k1 && Fp.empty()) continue;
      std::string f;
      if (k1) f = Fp;
      else if (Fp.empty()) f = kconst(kp);
      else f = "cmul(" + Fp + ", " + kconst(kp) + ")";
      if (Fp.empty() && kp.imag() == 0.0)  // real scale: two multiplies
        set(p, "make_double2(" + name[p] + ".x * " + f + ".x, " + name[p] + ".y * " + f + ".x)", "");
      else
        set(p, "cmul(" + name[p] + ", " + f + ")", "");
      K[p] = 1.0;
    }
    Fp.clear();
    if (with_global) Kg = 1.0;
  }

  // Unpredicated 2x2 whose rows share a pivot f (|m00| = |m11|, |m01| = |m10|:
  // rotations, H): M = f * N with one entry of each row of N exactly +-1, so
  // every output is a single fused multiply-add per real component; f joins
  // the tile-wide scalar Kg (commutes with every linear op, applied at store).
  // tf: a pending frame flip on the target bit (predicate): threads with tf
  // apply X M X instead -- accepted when it factors with the same pivots and
  // signs, so only the per-thread x coefficients differ (one select per row).
  bool mat1_factored(const TOp& o, const std::string& tf = "") {
    if (o.rmask != 0 || o.gmask != 0) return false;
    const cd m[4] = {coefv(o.coef), coefv(o.coef + 1), coefv(o.coef + 2), coefv(o.coef + 3)};
    // Pivot on the diagonal unless it is tiny: the generated code then does not
    // depend on the rotation angle (parameter sweeps reuse compiled passes);
    // the pending scale Kg is applied at the end of each pass, so the bounded
    // growth (< 2^10 per gate) cannot overflow.
    const cd f = std::abs(m[0]) >= 0x1p-10 * std::abs(m[1]) ? m[0] : m[1];
    if (f == cd(0)) return false;
    const cd n[4] = {m[0] / f, m[1] / f, m[2] / f, m[3] / f};
    auto unit = [](cd v) { return v.imag() == 0.0 && (v.real() == 1.0 || v.real() == -1.0); };
    struct Row {
      int piv;  // column holding +-1
      double sign;
      cd x;     // the other coefficient
    } rows[2];
    for (int r = 0; r < 2; ++r) {
      const cd u = n[2 * r], w = n[2 * r + 1];
      if (unit(u)) rows[r] = {0, u.real(), w};
      else if (unit(w)) rows[r] = {1, w.real(), u};
      else return false;
    }
    const int Kb = o.k;
    std::string xc[2];
    if (!tf.empty()) {
      const cd nx[4] = {n[3], n[2], n[1], n[0]};  // X M X / f
      for (int r = 0; r < 2; ++r) {
        const cd u = nx[2 * r], w = nx[2 * r + 1];
        Row c;
        if (unit(u)) c = {0, u.real(), w};
        else if (unit(w)) c = {1, w.real(), u};
        else return false;
        const bool same_kind = (rows[r].x.imag() == 0.0) == (c.x.imag() == 0.0) &&
                               (rows[r].x.real() == 0.0) == (c.x.real() == 0.0);
        if (c.piv != rows[r].piv || c.sign != rows[r].sign || !same_kind) return false;
        xc[r] = fresh("XS");
        s << "    const double2 " << xc[r] << " = " << tf << " ? " << kconst(c.x) << " : " << kconst(rows[r].x) << ";\n";
      }
    } else {
      for (int r = 0; r < 2; ++r) xc[r] = kconst(rows[r].x);
    }
    for (int p = 0; p < NS; ++p) {
      if ((p >> Kb) & 1) continue;
      const int p1 = p | (1 << Kb);
      flush_pair(p, p1);
      const std::string in[2] = {name[p], name[p1]};
      std::string out[2];
      for (int r = 0; r < 2; ++r) {
        const Row& R = rows[r];
        const std::string& pv = in[R.piv];
        const std::string& ot = in[1 - R.piv];
        const std::string sg = R.sign < 0 ? "-" : "";
        if (R.x.imag() == 0.0) {  // x real: (x*ot + s*pv)
          out[r] = "make_double2(fma(" + xc[r] + ".x, " + ot + ".x, " + sg + pv + ".x), fma(" + xc[r] + ".x, " + ot +
                   ".y, " + sg + pv + ".y))";
        } else if (R.x.real() == 0.0) {  // x = i*y: (i*y*ot + s*pv)
          out[r] = "make_double2(fma(-" + xc[r] + ".y, " + ot + ".y, " + sg + pv + ".x), fma(" + xc[r] + ".y, " + ot +
                   ".x, " + sg + pv + ".y))";
        } else {
          out[r] = "caxpy(" + xc[r] + ", " + ot + ", " + (R.sign < 0 ? "cneg(" + pv + ")" : pv) + ")";
        }
      }
      set(p, out[0], "");
      set(p1, out[1], "");
    }
    Kg *= f;
    return true;
  }

  // --- micro-ops ------------------------------------------------------------
  void mat1(const TOp& o) {
    mat_reason = o.rmask ? "mat1 rmask" : (o.type == TO_MAT1_RX ? "mat1 rx" : (o.type == TO_MAT1_REAL ? "mat1 real" : "mat1"));
    // a pending frame flip on the target: M itself when X M X == M, else X M X
    // through per-thread coefficients (factored rows, or the four entries)
    std::string tf;
    if (!o.rmask)
      for (auto& f : frame)
        if (f.first == static_cast<int>(o.k)) tf = f.second;
    const bool symmetric = coefv(o.coef) == coefv(o.coef + 3) && coefv(o.coef + 1) == coefv(o.coef + 2);
    std::string m0 = coef(o.coef), m1 = coef(o.coef + 1), m2 = coef(o.coef + 2), m3 = coef(o.coef + 3);
    if (!tf.empty() && symmetric) {
      materialize(static_cast<uint32_t>(o.rmask));
      if (mat1_factored(o)) return;
    } else if (!tf.empty()) {
      materialize(static_cast<uint32_t>(o.rmask));
      if (mat1_factored(o, tf)) return;
      if (o.type == TO_MAT1_RX) {
        materialize(1u << o.k);
      } else {  // per-thread entries of X M X: (m3, m2; m1, m0)
        const std::string e[4] = {fresh("ME"), fresh("ME"), fresh("ME"), fresh("ME")};
        const std::string orig[4] = {m0, m1, m2, m3};
        for (int i = 0; i < 4; ++i)
          s << "    const double2 " << e[i] << " = " << tf << " ? " << orig[3 - i] << " : " << orig[i] << ";\n";
        m0 = e[0], m1 = e[1], m2 = e[2], m3 = e[3];
      }
    } else {
      materialize((1u << o.k) | static_cast<uint32_t>(o.rmask));
      if (mat1_factored(o)) return;
    }
    const std::string t = pred(o);
    const int Kb = o.k;
    for (int p = 0; p < NS; ++p) {
      if ((p >> Kb) & 1) continue;
      if ((p & o.rmask) != o.rval) continue;
      const int p1 = p | (1 << Kb);
      flush_pair(p, p1);
      const std::string a = name[p], b = name[p1];
      std::string e0, e1;
      if (o.type == TO_MAT1) {
        e0 = "cmv2(" + m0 + ", " + a + ", " + m1 + ", " + b + ")";
        e1 = "cmv2(" + m2 + ", " + a + ", " + m3 + ", " + b + ")";
      } else if (o.type == TO_MAT1_REAL) {
        e0 = "rmv2(" + m0 + ".x, " + a + ", " + m1 + ".x, " + b + ")";
        e1 = "rmv2(" + m2 + ".x, " + a + ", " + m3 + ".x, " + b + ")";
      } else {
        e0 = "xmv2(" + m0 + ".x, " + a + ", " + m1 + ".y, " + b + ")";
        e1 = "xmv2(" + m3 + ".x, " + b + ", " + m2 + ".y, " + a + ")";
      }
      set(p, e0, t);
      set(p1, e1, t);
    }
  }

  void flip(const TOp& o) {
    const int Kb = o.k;
    mat_reason = "flip rmask";
    materialize(static_cast<uint32_t>(o.rmask));  // register controls select slots by logical bits
    if (o.gmask && !o.rmask && flip_frame) {
      const std::string t = pred(o);
      for (auto& f : frame)
        if (f.first == Kb) {  // two pending flips of one bit: XOR of the predicates
          const std::string tc = fresh("t");
          s << "    const bool " << tc << " = " << f.second << " != " << t << ";\n";
          f.second = tc;
          return;
        }
      frame.push_back({Kb, t});
      return;
    }
    const std::string t = o.gmask ? pred(o) : "";
    for (int p = 0; p < NS; ++p) {
      if ((p >> Kb) & 1) continue;
      if ((p & o.rmask) != o.rval) continue;
      const int p1 = p | (1 << Kb);
      if (t.empty()) {
        std::swap(name[p], name[p1]);  // pure renaming; pending constants travel along
        std::swap(K[p], K[p1]);
      } else {
        flush_pair(p, p1);
        const std::string a = name[p], b = name[p1];
        const std::string na = fresh(), nb = fresh();
        s << "    const double2 " << na << " = " << t << " ? " << b << " : " << a << ";\n";
        s << "    const double2 " << nb << " = " << t << " ? " << a << " : " << b << ";\n";
        name[p] = na;
        name[p1] = nb;
      }
    }
  }

  void phase(const TOp& o) {
    {  // register predicates and per-slot factors that differ across a pending flip
      uint32_t dep = static_cast<uint32_t>(o.rmask);
      for (auto& f : frame)
        for (int p = 0; p < NS; ++p)
          if (coefv(o.coef + p) != coefv(o.coef + (p ^ (1 << f.first)))) dep |= 1u << f.first;
      mat_reason = o.rmask ? "phase rmask" : "phase factors";
      materialize(dep);
    }
    const std::string t = pred(o);
    // split the non-register factors into thread-bit and tile (outside) ones
    std::vector<std::pair<uint32_t, uint32_t>> thr;  // (tid bit, coef index)
    std::vector<std::pair<uint32_t, uint32_t>> out;  // (qubit, coef index)
    for (uint32_t j = 0; j < o.nlist; ++j) {
      const uint32_t q = tp.meta[o.meta + j];
      int tb = -1;
      for (uint32_t k = 0; k < tp.h.t; ++k)
        if (cur_tq[k] == q) tb = static_cast<int>(k);
      if (tb >= 0) thr.push_back({static_cast<uint32_t>(tb), o.coef + NS + 1 + j});
      else out.push_back({q, o.coef + NS + 1 + j});
    }
    std::string F;
    if (!thr.empty()) {  // per-thread constant, hoisted out of the tile loop
      F = fresh("FT");
      pro << "  double2 " << F << " = make_double2(1.0, 0.0);\n";
      for (auto& [b, ci] : thr) pro << "  if ((tid >> " << b << ") & 1u) " << F << " = cmul(" << F << ", " << coef(ci) << ");\n";
    }
    const bool c1 = one(coefv(o.coef + NS));
    // Unpredicated whole-thread phase: the constant and the factors of qubits
    // outside the tile form a per-tile scalar that commutes with everything up
    // to the store (transposes included), so it joins Fg instead of Fp.
    const bool tile_scalar = t.empty() && o.rmask == 0;
    if (tile_scalar && out.empty()) {  // a constant: joins the compile-time tile scalar
      Kg *= coefv(o.coef + NS);
    } else if (!c1 || !out.empty()) {
      const std::string Fo = fresh("F");
      if (tile_scalar)
        s << "    double2 " << Fo << " = " << (c1 ? std::string("make_double2(1.0, 0.0)") : coef(o.coef + NS)) << ";\n";
      else
        s << "    double2 " << Fo << " = " << (F.empty() ? (c1 ? std::string("make_double2(1.0, 0.0)") : coef(o.coef + NS))
                                                          : (c1 ? F : "cmul(" + F + ", " + coef(o.coef + NS) + ")"))
          << ";\n";
      std::map<uint32_t, std::vector<std::pair<uint32_t, uint32_t>>> by_chunk;
      for (auto& [q, ci] : out) by_chunk[tix_bit(q) / kChunk].push_back({tix_bit(q) % kChunk, ci});
      for (auto& [c, bits] : by_chunk) {
        if (bits.size() >= 2 && table_entries + 64 <= kMaxTableEntries) {
          tables.push_back({c, table_entries, bits});
          s << "    " << Fo << " = cmul(" << Fo << ", TAB[" << table_entries << " + ((tix >> " << c * kChunk
            << ") & 63u)]);\n";
          table_entries += 64;
        } else {
          for (auto& [b, ci] : bits)
            s << "    if ((tix >> " << c * kChunk + b << ") & 1ull) " << Fo << " = cmul(" << Fo << ", " << coef(ci)
              << ");\n";
        }
      }
      if (tile_scalar) {
        if (Fg.empty()) {
          Fg = Fo;
        } else {
          const std::string nf = fresh("FG");
          s << "    const double2 " << nf << " = cmul(" << Fg << ", " << Fo << ");\n";
          Fg = nf;
        }
      } else {
        F = Fo;
      }
    }
    if (!t.empty() && !F.empty()) {
      const std::string Ft = fresh("F");
      s << "    const double2 " << Ft << " = " << t << " ? " << F << " : make_double2(1.0, 0.0);\n";
      F = Ft;
    }
    if (o.rmask == 0) {
      // whole-thread factor: defer; register-qubit factors: pending constants
      if (!F.empty()) {
        if (Fp.empty()) {
          Fp = F;
        } else {
          const std::string nf = fresh("FP");
          s << "    const double2 " << nf << " = cmul(" << Fp << ", " << F << ");\n";
          Fp = nf;
        }
      }
      if (t.empty()) {
        for (int p = 0; p < NS; ++p) K[p] *= coefv(o.coef + p);
      } else {
        // thread-predicated register factors cannot be folded into constants
        for (int p = 0; p < NS; ++p) {
          const cd g = coefv(o.coef + p);
          if (!one(g)) set(p, "cmul(" + name[p] + ", " + coef(o.coef + p) + ")", t);
        }
      }
      return;
    }
    // register-predicated phase: the per-slot constants join the pending K
    // (compile time); only the thread/tile factor F is applied now, to the
    // selected slots (one complex multiply each)
    if (t.empty()) {
      for (int p = 0; p < NS; ++p) {
        if ((p & o.rmask) != o.rval) continue;
        K[p] *= coefv(o.coef + p);
        if (!F.empty()) set(p, "cmul(" + name[p] + ", " + F + ")", "");
      }
      return;
    }
    for (int p = 0; p < NS; ++p) {
      if ((p & o.rmask) != o.rval) continue;
      const cd g = coefv(o.coef + p);
      std::string f;
      if (F.empty() && one(g)) continue;
      if (F.empty()) f = coef(o.coef + p);
      else if (one(g)) f = F;
      else f = "cmul(" + F + ", " + coef(o.coef + p) + ")";
      set(p, "cmul(" + name[p] + ", " + f + ")", t);
    }
  }

  void dense(const TOp& o) {
    mat_reason = "dense";
    materialize(~0u);
    const std::string t = pred(o);
    const int KD = o.type == TO_DENSE2 ? 2 : 3, Gd = 1 << KD;
    for (int hi = 0; hi < (NS >> KD); ++hi) {
      const int p0 = hi << KD;
      if ((p0 & o.rmask) != o.rval) continue;
      bool same = true;
      for (int c = 1; c < Gd; ++c) same = same && K[p0 + c] == K[p0];
      if (!same)
        for (int c = 0; c < Gd; ++c) flush_const(p0 + c);
      std::string in[8];
      for (int c = 0; c < Gd; ++c) in[c] = name[p0 + c];
      for (int r = 0; r < Gd; ++r) {
        std::ostringstream x;
        x << "dotrow" << Gd << "(P.c + " << (o.coef + r * Gd);
        for (int c = 0; c < Gd; ++c) x << ", " << in[c];
        x << ")";
        set(p0 + r, x.str(), t);
      }
    }
  }

  void transpose(const TOp& o, int idx) {
    flush_all(false);  // Kg (tile-wide) commutes with the exchange
    const uint32_t TB = tp.h.t;
    const uint32_t* mt = tp.meta.data() + o.meta;
    const std::string Tw = "Tw" + std::to_string(idx), Tr = "Tr" + std::to_string(idx);
    auto xorexpr = [&](const uint32_t* cols) {
      std::ostringstream e;
      e << "0u";
      for (uint32_t k = 0; k < TB; ++k)
        if (cols[k]) e << " ^ (((tid >> " << k << ") & 1u) * " << cols[k] << "u)";
      return e.str();
    };
    bool warp_local = warp_local_ok && TB > 5;
    for (uint32_t k = 5; warp_local && k < TB; ++k) warp_local = cur_tq[k] == mt[2 * TB + 2 * R + k];
    // the leading barrier stays block-wide: each exchange picks its own
    // swizzle, so this exchange's writes may hit slots other warps are still
    // reading from the previous one
    s << "    __syncthreads();\n";
    tile_barrier_done = true;
    s << "    const unsigned " << Tw << " = " << xorexpr(mt);
    if (!frame.empty()) s << " ^ " << frame_xor(mt + TB);  // slot p holds logical p ^ f
    s << ";\n";
    frame.clear();
    for (int p = 0; p < NS; ++p) {
      uint32_t a = 0;
      for (int k = 0; k < R; ++k)
        if ((p >> k) & 1) a ^= mt[TB + k];
      s << "    sm[" << Tw << " ^ " << a << "u] = " << name[p] << ";\n";
    }
    s << (warp_local ? "    __syncwarp();\n" : "    __syncthreads();\n");
    s << "    const unsigned " << Tr << " = " << xorexpr(mt + TB + R) << ";\n";
    for (int p = 0; p < NS; ++p) {
      uint32_t a = 0;
      for (int k = 0; k < R; ++k)
        if ((p >> k) & 1) a ^= mt[2 * TB + R + k];
      const std::string nv = fresh();
      s << "    const double2 " << nv << " = sm[" << Tr << " ^ " << a << "u];\n";
      name[p] = nv;
    }
    emit_G(mt + 2 * TB + 2 * R, false);
  }

  static constexpr const char* kIssueNext =
      "    { const unsigned long long nt = kk + gridDim.x; if (nt < ntiles) prefetch(expand(nt)); }\n";
  static constexpr const char* kIssueEarly =
      "    { const unsigned long long nt = kk + gridDim.x; if (nt < ntiles) prefetch_e(expand(nt)); }\n";
  static constexpr const char* kIssueLate =
      "    { const unsigned long long nt = kk + gridDim.x; if (nt < ntiles) prefetch_l(expand(nt)); }\n";

  std::string run(const std::string& kname, uint32_t threads, uint32_t minb) {
    const TileHeader& h = tp.h;
    transposes_total = 0;
    for (const TOp& o : tp.ops) transposes_total += o.type == TO_TRANSPOSE;
    const uint32_t T = 1u << h.t;
    const uint32_t TB = h.t;
    // leading transpose out of the load layout: fused into the prefetch (the
    // cp.async destinations are its write slots) or, from a basis state, into
    // the register initialisation
    const bool lead = leading_transpose(tp) && (from_basis || (prefetch && early == 0));
    // zero warps (see zwarp_qubits): every register layout must keep those
    // qubits on the same thread bits; up to TB - 5 of them go to the warp bits
    for (uint32_t b = 0; b < TB; ++b) zw_pos[b] = static_cast<int>(b);
    zw_cond.clear();
    if (zwarp_qubits && zskip && sparse && prefetch && early == 0 && !tma && !xk && !h.oop && !reduce && TB > 5) {
      std::vector<const uint32_t*> layouts{h.load.tq, h.store.tq};
      for (const TOp& o : tp.ops) {
        if (o.type == TO_TRANSPOSE) layouts.push_back(tp.meta.data() + o.meta + 2 * TB + 2 * R);
        if (o.type == TO_RELABEL) layouts.push_back(tp.meta.data() + o.meta);
      }
      std::vector<uint32_t> bits;  // thread bits holding zero-warp qubits, in every layout
      for (uint32_t b = 0; b < TB; ++b) {
        if (!((zwarp_qubits >> h.load.tq[b]) & 1)) continue;
        bool same = true;
        for (const uint32_t* tq : layouts) same = same && tq[b] == h.load.tq[b];
        if (same) bits.push_back(b);
      }
      const uint32_t W = TB - 5;  // warp bits of the block
      if (bits.size() > W) bits.resize(W);
      if (!bits.empty()) {
        std::vector<char> moved(TB, 0);
        std::ostringstream c;
        c << "(0u";
        for (size_t i = 0; i < bits.size(); ++i) {  // zero-warp bits -> the top physical bits
          zw_pos[bits[i]] = static_cast<int>(TB - 1 - i);
          moved[bits[i]] = 1;
          c << " | ((tid >> " << bits[i] << ") ^ (unsigned)(ival >> " << h.load.tq[bits[i]] << "))";
        }
        c << ") & 1u";
        int next = 0;  // the other logical bits keep their order on the remaining physical bits
        for (uint32_t b = 0; b < TB; ++b)
          if (!moved[b]) zw_pos[b] = next++;
        zw_cond = c.str();
        warp_local_ok = false;  // logical lanes no longer form the physical warps
      }
    }
    const uint32_t* mt0 = lead ? tp.meta.data() + tp.ops[0].meta : nullptr;
    auto xorexpr = [&](const uint32_t* cols) {
      std::ostringstream e;
      e << "0u";
      for (uint32_t k = 0; k < TB; ++k)
        if (cols[k]) e << " ^ (((tid >> " << k << ") & 1u) * " << cols[k] << "u)";
      return e.str();
    };
    auto slot_xor = [&](const uint32_t* cols, int p) {
      uint32_t a = 0;
      for (int k = 0; k < R; ++k)
        if ((p >> k) & 1) a ^= cols[k];
      return a;
    };
    unsigned long long loff[kTileMaxSlots];
    for (int p = 0; p < NS; ++p) {
      loff[p] = 0;
      for (int k = 0; k < R; ++k)
        if ((p >> k) & 1) loff[p] |= h.load.rs[k];
    }
    // ---- tile-loop body
    // Zero tiles of a run started from a basis state: a tile whose index
    // disagrees with the still-definite outside qubits (dmask / dval, kernel
    // parameters; dmask = 0 otherwise) is zero before and after the pass.  In
    // place it is skipped outright; a pass that writes elsewhere (the reset
    // fused into the first pass, an out-of-place pass) writes its zeros.
    use_tma = tma && prefetch && !lead && early == 0 && !sparse && !from_basis && tma_segments(h, ta, tl) > 0;
    trank = use_tma ? tma_segments(h, ta, tl) : 0;
    if (use_tma) s << "    mbar_wait(&QMB, QPH); QPH ^= 1u;  // this tile's bulk copies (or the zero-tile arrive)\n";
    if (!xk) {
      s << "    if ((base & dmask) != dval) {\n";
      if (from_basis || h.oop) {
        if (h.oop) {
        s << "      unsigned long long GZ = TLO;\n";
        for (uint32_t i = 0; i + h.m < h.n; ++i)
          s << "      if ((tix >> " << i << ") & 1ull) GZ |= " << hexll(1ull << h.out_pos[i]) << ";\n";
        for (int p = 0; p < NS; ++p) {
          unsigned long long off = 0;
          for (int k = 0; k < R; ++k)
            if ((p >> k) & 1) off |= h.store.rs[k];
          s << "      __stcs(out + (GZ | " << hexll(off) << "), make_double2(0.0, 0.0));\n";
        }
      } else {
        for (int p = 0; p < NS; ++p) {
          unsigned long long off = 0;
          for (int k = 0; k < R; ++k)
            if ((p >> k) & 1) off |= h.store.rs[k];
          s << "      __stcs(amps + ((base | TLS | " << hexll(off) << ") & lmask), make_double2(0.0, 0.0));\n";
        }
        }
      }
      if (prefetch) s << "  " << kIssueNext;
      s << "      continue;\n    }\n";
    }
    const size_t zw_at = s.str().size();  // the zero-warp path goes here (see below)
    int ti = 0;
    tile_barrier_done = lead && !from_basis;  // the fused leading exchange has its own block barrier
    if (from_basis) {
      unsigned long long off[kTileMaxSlots];
      for (int p = 0; p < NS; ++p) {
        off[p] = loff[p];
        if (lead) {  // registers start in the layout after the leading transpose
          off[p] = 0;
          for (int k = 0; k < R; ++k)
            if ((p >> k) & 1) off[p] |= 1ull << mt0[3 * TB + 2 * R + k];
        }
      }
      if (lead) {
        emit_G(mt0 + 2 * TB + 2 * R, false);
        ti = 1;
      }
      for (int p = 0; p < NS; ++p) {
        name[p] = fresh();
        s << "    const double2 " << name[p] << " = make_double2(((G | " << hexll(off[p])
          << ") == basis) ? 1.0 : 0.0, 0.0);\n";
      }
    } else if (use_tma) {
      // run-major buffer: amplitude (thread t, slot p) of the load layout sits
      // at its tile-local index; lanes 0-2 hold tile bits 0-2 (conflict-free)
      for (int p = 0; p < NS; ++p) {
        name[p] = fresh();
        s << "    const double2 " << name[p] << " = PB[TQ + " << tile_off(p) << "u];\n";
      }
      if (!single_buf || transposes_total == 0) s << "    __syncthreads();\n" << kIssueNext;
    } else if (prefetch) {
      s << "    cp_async_wait_all();\n";
      if (lead) {
        s << "    __syncthreads();\n";
        const bool zsel = sparse && !sparse_zero_store;  // zeros were not staged: select them here
        if (zsel) emit_G(mt0 + 2 * TB + 2 * R, false);  // the global index of each slot after the transpose
        for (int p = 0; p < NS; ++p) {
          name[p] = fresh();
          const std::string rd = "PB[R0 ^ " + std::to_string(slot_xor(mt0 + 2 * TB + R, p)) + "u]";
          if (zsel) {
            unsigned long long off = 0;  // register qubits of the first layout (transpose meta)
            for (int k = 0; k < R; ++k)
              if ((p >> k) & 1) off |= 1ull << mt0[3 * TB + 2 * R + k];
            s << "    const double2 " << name[p] << " = (((G | " << hexll(off) << ") & imask) == ival) ? " << rd
              << " : make_double2(0.0, 0.0);\n";
          } else {
            s << "    const double2 " << name[p] << " = " << rd << ";\n";
          }
        }
        if (!zsel) emit_G(mt0 + 2 * TB + 2 * R, false);
        ti = 1;
        if (!single_buf || transposes_total == 1) s << "    __syncthreads();\n" << kIssueNext;
      } else {
        for (int p = 0; p < NS; ++p) {
          name[p] = fresh();
          const std::string slot = static_cast<uint32_t>(p) < early
                                       ? "PE[" + std::to_string(p * T) + " + tid]"
                                       : "PB[" + std::to_string((p - static_cast<int>(early)) * T) + " + tid]";
          if (sparse && !sparse_zero_store)  // slots of amplitudes that disagree with the definite qubits were not staged
            s << "    const double2 " << name[p] << " = (((G | " << hexll(loff[p]) << ") & imask) == ival) ? " << slot
              << " : make_double2(0.0, 0.0);\n";
          else
            s << "    const double2 " << name[p] << " = " << slot << ";\n";
        }
        if (early) {  // own slots only: no barrier before re-filling them
          s << kIssueEarly;
          if (transposes_total == 0) s << kIssueLate;
        } else if (!single_buf || transposes_total == 0) {
          s << kIssueNext;
        }
      }
    } else {
      for (int p = 0; p < NS; ++p) {
        name[p] = fresh();
        if (sparse)
          s << "    const double2 " << name[p] << " = (((G | " << hexll(loff[p]) << ") & imask) == ival) ? __ldcs(amps + ((G | "
            << hexll(loff[p]) << ") & lmask)) : make_double2(0.0, 0.0);\n";
        else
          s << "    const double2 " << name[p] << " = __ldcs(amps + ((G | " << hexll(loff[p]) << ") & lmask));\n";
      }
    }
    if (ti == 0)
      for (uint32_t k = 0; k < h.t; ++k) cur_tq[k] = h.load.tq[k];
    for (size_t oi = static_cast<size_t>(ti); oi < tp.ops.size(); ++oi) {
      const TOp& o = tp.ops[oi];
      switch (o.type) {
        case TO_MAT1:
        case TO_MAT1_REAL:
        case TO_MAT1_RX: mat1(o); break;
        case TO_FLIP: flip(o); break;
        case TO_PHASE: phase(o); break;
        case TO_DENSE2:
        case TO_DENSE3: dense(o); break;
        case TO_TRANSPOSE:
          transpose(o, ti++);
          if (prefetch && single_buf && ti == transposes_total)
            s << "    __syncthreads();\n" << (early ? kIssueLate : kIssueNext);
          break;
        case TO_RELABEL: emit_G(tp.meta.data() + o.meta, false); break;
        default: throw RuntimeError("jit: unknown micro-op");
      }
    }
    flush_all(true);
    mat_reason = "store";
    if (xk || h.oop) materialize(~0u);  // these stores compute each slot's index separately
    // Relabels (free SWAPs) make threads store where other threads loaded; with
    // no transpose barrier in the pass, every load must retire before any store.
    if (xk) {
      unsigned long long pmask = 0;
      for (uint32_t i = 0; i < xk; ++i) pmask |= 1ull << xlpos[i];
      for (int p = 0; p < NS; ++p) {
        unsigned long long off = 0;
        for (int k = 0; k < R; ++k)
          if ((p >> k) & 1) off |= h.store.rs[k];
        s << "    { const unsigned long long L = (G | " << hexll(off) << ") & lmask; const unsigned d = 0u";
        for (uint32_t i = 0; i < xk; ++i) s << " | ((unsigned)((L >> " << xlpos[i] << ") & 1ull) << " << i << ")";
        s << "; __stcs(PEERS.p[d] + ((L & " << hexll(~pmask) << ") | xaval), " << name[p] << "); }\n";
      }
    } else if (h.oop) {
      // out of place through the final qubit permutation: the written index is
      // sigma(base) | sigma(thread bits) | sigma(register bits)
      s << "    unsigned long long GO = TLO;\n";
      for (uint32_t i = 0; i + h.m < h.n; ++i)
        s << "    if ((tix >> " << i << ") & 1ull) GO |= " << hexll(1ull << h.out_pos[i]) << ";\n";
      for (int p = 0; p < NS; ++p) {
        unsigned long long off = 0;
        for (int k = 0; k < R; ++k)
          if ((p >> k) & 1) off |= h.store.rs[k];
        s << "    __stcs(out + (GO | " << hexll(off) << "), " << name[p] << ");\n";
        if (reduce)
          s << "    ACC += __fma_rn(" << name[p] << ".x, " << name[p] << ".x, __dmul_rn(" << name[p] << ".y, " << name[p]
            << ".y)) * (double)((GO | " << hexll(off) << ") + 1ull);\n";
      }
    } else {
      if (ti == 0 && std::memcmp(&h.load, &h.store, sizeof(TileConfigAddr)) != 0) s << "    __syncthreads();\n";
      // (G | off) & lmask == (G & lmask) + off: the register strides are local
      // bits that G does not have -- one base pointer, constant offsets
      s << "    double2* const SP = amps + (G & lmask);\n";
      // pending flip frame: slot p goes to logical p ^ f, offset off(p) ^ off(f)
      // (register strides are disjoint bits: still no carry into G)
      std::string FO;
      if (!frame.empty()) {
        FO = fresh("FO");
        s << "    const unsigned long long " << FO << " = " << frame_xor(h.store.rs) << ";\n";
      }
      for (int p = 0; p < NS; ++p) {
        unsigned long long off = 0;
        for (int k = 0; k < R; ++k)
          if ((p >> k) & 1) off |= h.store.rs[k];
        const std::string offs = FO.empty() ? hexll(off) : "(" + hexll(off) + " ^ " + FO + ")";
        if (zskip)  // known-zero amplitudes (omask / oval) stay unwritten
          s << "    if (((G | " << offs << ") & omask) == oval) ";
        else
          s << "    ";
        s << "__stcs(SP + " << offs << ", " << name[p] << ");\n";
        if (reduce)
          s << "    ACC += __fma_rn(" << name[p] << ".x, " << name[p] << ".x, __dmul_rn(" << name[p] << ".y, " << name[p]
            << ".y)) * (double)((G | " << offs << ") + 1ull);\n";
      }
      frame.clear();
    }

    // ---- assemble
    std::ostringstream k;
    k << "struct __align__(16) QsbCoef { double2 c[" << std::max<size_t>(1, tp.coef.size() + extra.size()) << "]; };\n";
    k << "struct QsbPeers { double2* p[16]; };\n";
    k << "struct __align__(64) QsbTmap { unsigned long long v[16]; };\n";
    k << "extern \"C\" __global__ void __launch_bounds__(" << threads << ", " << minb << ") " << kname
      << "(double2* __restrict__ amps, double2* __restrict__ out, const unsigned long long rank_base,\n"
      << "    const unsigned long long lmask,\n"
      << "    const unsigned long long ntiles, const unsigned long long basis, const QsbPeers PEERS,\n"
    << "    const unsigned long long xaval, const unsigned long long dmask, const unsigned long long dval,\n"
    << "    const unsigned long long imask, const unsigned long long ival,\n"
    << "    const unsigned long long tmask, const unsigned long long tval,\n"
    << "    const unsigned long long omask, const unsigned long long oval, double* __restrict__ red,\n"
    << "    const __grid_constant__ QsbCoef P, const __grid_constant__ QsbTmap TMAP) {\n";
    k << "  extern __shared__ __align__(1024) double2 sm[];\n";
    if (reduce) k << "  double ACC = 0.0;\n";
    if (zw_cond.empty()) {
      k << "  const unsigned tid = threadIdx.x;\n";
    } else {  // logical thread bit b = physical bit zw_pos[b]
      k << "  const unsigned tid = 0u";
      for (uint32_t b = 0; b < h.t; ++b) k << " | (((threadIdx.x >> " << zw_pos[b] << ") & 1u) << " << b << ")";
      k << ";\n";
      k << "  const bool ZW = " << zw_cond << ";\n";
    }
    k << "  const unsigned long long TL = 0ull";
    for (uint32_t b = 0; b < h.t; ++b) k << " | ((unsigned long long)((tid >> " << b << ") & 1u) << " << h.load.tq[b] << ")";
    k << ";\n";
    if (!h.oop) {
      k << "  const unsigned long long TLS = 0ull";
      for (uint32_t b = 0; b < h.t; ++b) k << " | ((unsigned long long)((tid >> " << b << ") & 1u) << " << h.store.tq[b] << ")";
      k << ";\n  (void)TLS;\n";
    }
    if (h.oop) {
      k << "  const unsigned long long TLO = 0ull";
      for (uint32_t b = 0; b < h.t; ++b) k << " | ((unsigned long long)((tid >> " << b << ") & 1u) << " << h.store.tq[b] << ")";
      k << ";\n  (void)TLO;\n";
    }
    // Runs from a basis state, in place: only the tiles that can be non-zero
    // are visited -- the compact counter kk is spread over the tile-index bits
    // outside tmask, whose values are tval (load balance: every CTA gets work)
    k << "  auto expand = [&](unsigned long long c) {\n"
         "    if (!tmask) return c;\n"
         "    unsigned long long r = tval;\n"
         "    for (unsigned long long m = ~tmask; c && m; m &= m - 1, c >>= 1)\n"
         "      if (c & 1ull) r |= m & (0ull - m);\n"
         "    return r;\n  };\n";
    // tile index -> index with zeros at the tile qubits: the non-tile positions
    // form a few contiguous runs, each a shift-and-mask of the tile index
    k << "  auto base_of = [&](unsigned long long b) {\n    return 0ull";
    {
      bool in_tile[64] = {};
      for (uint32_t b = 0; b < h.m; ++b) in_tile[h.S[b]] = true;
      uint32_t c = 0;  // compact bit of the next run
      for (uint32_t q = 0; q < 64;) {
        if (in_tile[q]) {
          ++q;
          continue;
        }
        uint32_t e = q;
        while (e < 64 && !in_tile[e]) ++e;
        const uint32_t len = e - q;
        if (e >= 64 || len >= 64 - c) {  // last run: everything above
          k << " | ((b >> " << c << ") << " << q << ")";
          break;
        }
        k << " | (((b >> " << c << ") & " << hexll((1ull << len) - 1) << ") << " << q << ")";
        c += len;
        q = e;
      }
    }
    k << ";\n  };\n";
    k << pro.str();
    const uint32_t tbuf = tp.transposes - (lead ? 1u : 0u);
    const uint32_t tile_bufs = single_buf ? 1u : (tbuf ? 1u : 0u) + (prefetch ? 1u : 0u);
    const uint32_t early_amps = prefetch ? early * T : 0u;
    if (!tables.empty()) {
      k << "  double2* const TAB = sm + " << tile_bufs * (1u << h.m) + early_amps << ";\n";
      for (const Table& tb : tables) {
        k << "  for (unsigned e = tid; e < 64u; e += " << threads << "u) {\n    double2 f = make_double2(1.0, 0.0);\n";
        for (auto& [b, ci] : tb.bits) k << "    if ((e >> " << b << ") & 1u) f = cmul(f, " << coef(ci) << ");\n";
        k << "    TAB[" << tb.off << " + e] = f;\n  }\n";
      }
      k << "  __syncthreads();\n";
    }
    if (use_tma) {
      // one tensor copy per tile: dimension i of the map (built per launch by
      // launch_tile from the same segments) spans positions [a_i, a_(i+1));
      // the coordinates are the tile index bits between the runs
      k << "  double2* const PB = sm + " << (tbuf && !single_buf ? (1u << h.m) : 0u) << ";\n";
      k << "  __shared__ unsigned long long QMB;\n  unsigned QPH = 0;\n";
      k << "  if (tid == 0) { mbar_init(&QMB, 1u); fence_mbar_init(); }\n  __syncthreads();\n";
      k << "  const unsigned TQ = 0u";
      for (uint32_t b = 0; b < h.t; ++b) k << " | (((tid >> " << b << ") & 1u) << " << tile_bit(h.load.tq[b]) << ")";
      k << ";\n";
      k << "  auto prefetch = [&](unsigned long long t) {\n"
           "    if (tid != 0u) return;\n"
           "    const unsigned long long tb = base_of(t) | rank_base;\n"
           "    if ((tb & dmask) != dval) { mbar_arrive(&QMB); return; }  // zero tile: nothing to read\n"
           "    const unsigned long long lb = tb & lmask;\n"
           "    fence_proxy_async();  // the buffer's previous reads (ordered by the barrier) before these writes\n"
           "    mbar_expect_tx(&QMB, " << ((1u << h.m) * 16u) << "u);\n";
      for (uint32_t i = 0; i < trank; ++i) {
        const uint32_t hi = i + 1 < trank ? ta[i + 1] : 64u;
        const uint32_t span = hi - ta[i];
        const std::string mask = span >= 32 ? "0xffffffffull" : hexll((1ull << span) - 1);
        k << "    const int c" << i << " = (int)(((lb >> " << ta[i] << ") & " << mask << ")" << (i == 0 ? " << 1" : "")
          << ");\n";
      }
      k << "    tma_load_" << trank << "d(PB, &TMAP, &QMB";
      for (uint32_t i = 0; i < trank; ++i) k << ", c" << i;
      k << ");\n  };\n";
      k << "  unsigned long long kk = blockIdx.x;\n";
      k << "  if (kk < ntiles) prefetch(expand(kk));\n";
      k << "  for (; kk < ntiles; kk += gridDim.x) {\n";
    } else if (prefetch) {
      // Each thread stages its own 16 amplitudes of the next tile in its own
      // shared-memory slots (slot p*T + tid: conflict-free) with cp.async, so
      // HBM reads of tile i+1 overlap the arithmetic of tile i.
      k << "  double2* const PB = sm + " << (tbuf && !single_buf ? (1u << h.m) : 0u) << ";\n";
      if (lead) {  // per-thread write / read offsets of the fused leading transpose
        k << "  const unsigned W0 = " << xorexpr(mt0) << ";\n";
        k << "  const unsigned R0 = " << xorexpr(mt0 + TB + R) << ";\n";
      }
      auto lambda = [&](const char* fname, int p0, int p1) {
        k << "  auto " << fname << " = [&](unsigned long long t) {\n";
        k << "    const unsigned long long tb = base_of(t) | rank_base;\n";
        k << "    if ((tb & dmask) != dval) { cp_async_commit(); return; }  // zero tile: nothing to read\n";
        k << "    const unsigned long long g = tb | TL;\n";
        k << "    const double2* const gp = amps + (g & lmask);  // + loff[p] == (g | loff[p]) & lmask\n";
        for (int p = p0; p < p1; ++p) {
          if (sparse) {  // zero amplitudes: store the zero, skip the copy
            std::string dst;
            if (lead) dst = "PB + (W0 ^ " + std::to_string(slot_xor(mt0 + TB, p)) + "u)";
            else if (static_cast<uint32_t>(p) < early) dst = "PE + " + std::to_string(p * T) + " + tid";
            else dst = "PB + " + std::to_string((p - static_cast<int>(early)) * T) + " + tid";
            // the zero is selected where the slot is read (by the reading
            // thread, from its own global index) instead of stored here
            k << "    { const unsigned long long a = g | " << hexll(loff[p]) << "; if ((a & imask) == ival) cp_async16("
              << dst << ", amps + (a & lmask));";
            if (sparse_zero_store) k << " else *(" << dst << ") = make_double2(0.0, 0.0);";
            k << " }\n";
            continue;
          }
          if (lead)
            k << "    cp_async16(PB + (W0 ^ " << slot_xor(mt0 + TB, p) << "u), gp + " << hexll(loff[p]) << ");\n";
          else if (static_cast<uint32_t>(p) < early)
            k << "    cp_async16(PE + " << p * T << " + tid, gp + " << hexll(loff[p]) << ");\n";
          else
            k << "    cp_async16(PB + " << (p - static_cast<int>(early)) * T << " + tid, gp + " << hexll(loff[p])
              << ");\n";
        }
        k << "    cp_async_commit();\n  };\n";
      };
      if (early) {
        k << "  double2* const PE = sm + " << tile_bufs * (1u << h.m) << ";\n";
        lambda("prefetch_e", 0, static_cast<int>(early));
        lambda("prefetch_l", static_cast<int>(early), NS);
        k << "  auto prefetch = [&](unsigned long long t) { prefetch_e(t); prefetch_l(t); };\n";
      } else {
        lambda("prefetch", 0, NS);
      }
      k << "  unsigned long long kk = blockIdx.x;\n";
      k << "  if (kk < ntiles) prefetch(expand(kk));\n";
      k << "  for (; kk < ntiles; kk += gridDim.x) {\n";
    } else {
      k << "  for (unsigned long long kk = blockIdx.x; kk < ntiles; kk += gridDim.x) {\n";
    }
    k << "    const unsigned long long tile = expand(kk);\n";
    k << "    const unsigned long long base = base_of(tile) | rank_base;\n";
    k << "    const unsigned long long tix = tile | (rank_base >> " << h.m << ");\n    (void)tix;\n";
    k << "    unsigned long long G = base | TL;\n    (void)G;\n";
    std::string body = s.str();
    if (!zw_cond.empty()) {  // zero warps: only the block barriers of the pass, in the same order
      const std::string tail = body.substr(zw_at);
      size_t nb = 0;
      for (size_t at = tail.find("__syncthreads();"); at != std::string::npos; at = tail.find("__syncthreads();", at + 1))
        ++nb;
      std::string zb = "    if (ZW) {\n      cp_async_wait_all();\n";
      for (size_t i = 0; i < nb; ++i) zb += "      __syncthreads();\n";
      zb += "      continue;\n    }\n";
      body = body.substr(0, zw_at) + zb + tail;
    }
    k << body;
    k << "  }\n";
    // peer stores must be visible system-wide before the stream barrier that follows
    if (xk) k << "  __threadfence_system();\n";
    if (reduce) {  // fixed-order block sum of the per-thread checksums -> red[blockIdx.x]
      k << "  {\n    __shared__ double RS[" << (threads / 32) << "];\n"
           "    double v = ACC;\n"
           "    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);\n"
           "    if ((tid & 31u) == 0) RS[tid >> 5] = v;\n"
           "    __syncthreads();\n"
           "    if (tid == 0) {\n      double t = 0.0;\n"
           "      for (unsigned w = 0; w < " << (threads / 32) << "u; ++w) t += RS[w];\n"
           "      red[blockIdx.x] = t;\n    }\n  }\n";
    }
    k << "}\n";
    return k.str();
  }
};

}  // namespace jitgen
}  // namespace qsb
