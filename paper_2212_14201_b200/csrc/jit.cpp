// Per-pass CUDA code generation + NVRTC compilation (see jit.hpp).
#include "jit.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>
#include <thread>
#include <unordered_map>

#include "plan.hpp"
#include "tile.hpp"

namespace qsb {

namespace {

std::atomic<uint64_t> g_compiles{0}, g_hits{0};

// ------------------------------------------------------------ driver API
// libcuda is resolved through the runtime (cudaGetDriverEntryPoint), so the
// library still loads on machines without a driver (CPU-side planning/tests).
struct Driver {
  CUresult (*moduleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           CUstream, void**, void**) = nullptr;
  CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
  CUresult (*getErrorString)(CUresult, const char**) = nullptr;
};

template <class F>
void resolve(const char* sym, F*& fp) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  QSB_CUDA(cudaGetDriverEntryPoint(sym, &p, cudaEnableDefault, &q));
  if (!p || q != cudaDriverEntryPointSuccess) throw CudaError(std::string("driver entry point missing: ") + sym);
  fp = reinterpret_cast<F*>(p);
}

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    resolve("cuModuleLoadData", d.moduleLoadData);
    resolve("cuModuleGetFunction", d.moduleGetFunction);
    resolve("cuLaunchKernel", d.launchKernel);
    resolve("cuFuncSetAttribute", d.funcSetAttribute);
    resolve("cuOccupancyMaxActiveBlocksPerMultiprocessor", d.occupancy);
    resolve("cuGetErrorString", d.getErrorString);
  });
  return d;
}

void cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = "unknown";
  if (driver().getErrorString) driver().getErrorString(r, &s);
  throw CudaError(std::string(what) + ": " + s);
}

// ------------------------------------------------------------ generator

std::string hexll(unsigned long long v) {
  char b[32];
  std::snprintf(b, sizeof b, "0x%llxull", v);
  return b;
}

struct Gen {
  const TileProgram& tp;
  std::ostringstream s;
  std::string name[16];
  int counter = 0;
  explicit Gen(const TileProgram& p) : tp(p) {}

  std::string fresh() { return "v" + std::to_string(counter++); }
  std::string coef(uint32_t i) { return "P.c[" + std::to_string(i) + "]"; }
  bool is_one(uint32_t i) const {
    const double2 c = tp.coef[i];
    return c.x == 1.0 && c.y == 0.0;
  }

  // G = base | (thread bit k -> qubit tq[k])
  void emit_G(const uint32_t* tq, bool decl) {
    s << "    " << (decl ? "unsigned long long " : "") << "G = base";
    for (uint32_t k = 0; k < tp.h.t; ++k)
      s << " | ((unsigned long long)((tid >> " << k << ") & 1u) << " << tq[k] << ")";
    s << ";\n";
  }

  std::string pred(const TOp& o) {
    if (!o.gmask) return "";
    const std::string t = "t" + std::to_string(counter++);
    s << "    const bool " << t << " = (G & " << hexll(o.gmask) << ") == " << hexll(o.gval) << ";\n";
    return t;
  }

  void set(int p, const std::string& expr, const std::string& t) {
    const std::string nv = fresh();
    if (t.empty()) s << "    const double2 " << nv << " = " << expr << ";\n";
    else s << "    const double2 " << nv << " = " << t << " ? " << expr << " : " << name[p] << ";\n";
    name[p] = nv;
  }

  void mat1(const TOp& o) {
    const std::string t = pred(o);
    const int K = o.k;
    const std::string m0 = coef(o.coef), m1 = coef(o.coef + 1), m2 = coef(o.coef + 2), m3 = coef(o.coef + 3);
    for (int p = 0; p < 16; ++p) {
      if ((p >> K) & 1) continue;
      if ((p & o.rmask) != o.rval) continue;
      const int p1 = p | (1 << K);
      const std::string a = name[p], b = name[p1];
      std::string e0, e1;
      if (o.type == TO_MAT1) {
        e0 = "cmv2(" + m0 + ", " + a + ", " + m1 + ", " + b + ")";
        e1 = "cmv2(" + m2 + ", " + a + ", " + m3 + ", " + b + ")";
      } else if (o.type == TO_MAT1_REAL) {
        e0 = "rmv2(" + m0 + ".x, " + a + ", " + m1 + ".x, " + b + ")";
        e1 = "rmv2(" + m2 + ".x, " + a + ", " + m3 + ".x, " + b + ")";
      } else {  // RX-type: real diagonal, imaginary off-diagonal
        e0 = "xmv2(" + m0 + ".x, " + a + ", " + m1 + ".y, " + b + ")";
        e1 = "xmv2(" + m3 + ".x, " + b + ", " + m2 + ".y, " + a + ")";
      }
      set(p, e0, t);
      set(p1, e1, t);
    }
  }

  void flip(const TOp& o) {
    const int K = o.k;
    const std::string t = o.gmask ? pred(o) : "";
    for (int p = 0; p < 16; ++p) {
      if ((p >> K) & 1) continue;
      if ((p & o.rmask) != o.rval) continue;
      const int p1 = p | (1 << K);
      if (t.empty()) {
        std::swap(name[p], name[p1]);  // pure renaming
      } else {
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
    const std::string t = pred(o);
    const std::string F = "F" + std::to_string(counter++);
    const bool const_one = is_one(o.coef + 16) && o.nlist == 0;
    if (!const_one) {
      s << "    double2 " << F << " = " << coef(o.coef + 16) << ";\n";
      for (uint32_t j = 0; j < o.nlist; ++j)
        s << "    if ((G >> " << tp.meta[o.meta + j] << ") & 1ull) " << F << " = cmul(" << F << ", "
          << coef(o.coef + 17 + j) << ");\n";
    }
    for (int p = 0; p < 16; ++p) {
      if ((p & o.rmask) != o.rval) continue;
      const bool g1 = is_one(o.coef + p);
      std::string f;
      if (const_one && g1) continue;  // identity on this slot
      if (const_one) f = coef(o.coef + p);
      else if (g1) f = F;
      else f = "cmul(" + F + ", " + coef(o.coef + p) + ")";
      set(p, "cmul(" + name[p] + ", " + f + ")", t);
    }
  }

  void dense(const TOp& o) {
    const std::string t = pred(o);
    const int KD = o.type == TO_DENSE2 ? 2 : 3, Gd = 1 << KD;
    for (int hi = 0; hi < (16 >> KD); ++hi) {
      const int p0 = hi << KD;
      if ((p0 & o.rmask) != o.rval) continue;
      std::string in[8];
      for (int c = 0; c < Gd; ++c) in[c] = name[p0 + c];
      for (int r = 0; r < Gd; ++r) {
        std::string e = "make_double2(0.0, 0.0)";
        // acc = sum_c M[r][c] in[c] as an fma chain
        std::ostringstream x;
        x << "dotrow" << Gd << "(P.c + " << (o.coef + r * Gd);
        for (int c = 0; c < Gd; ++c) x << ", " << in[c];
        x << ")";
        set(p0 + r, x.str(), t);
      }
    }
  }

  void transpose(const TOp& o, int idx) {
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
    s << "    __syncthreads();\n";
    s << "    const unsigned " << Tw << " = " << xorexpr(mt) << ";\n";
    for (int p = 0; p < 16; ++p) {
      uint32_t K = 0;
      for (int k = 0; k < 4; ++k)
        if ((p >> k) & 1) K ^= mt[TB + k];
      s << "    sm[" << Tw << " ^ " << K << "u] = " << name[p] << ";\n";
    }
    s << "    __syncthreads();\n";
    s << "    const unsigned " << Tr << " = " << xorexpr(mt + TB + 4) << ";\n";
    for (int p = 0; p < 16; ++p) {
      uint32_t K = 0;
      for (int k = 0; k < 4; ++k)
        if ((p >> k) & 1) K ^= mt[2 * TB + 4 + k];
      const std::string nv = fresh();
      s << "    const double2 " << nv << " = sm[" << Tr << " ^ " << K << "u];\n";
      name[p] = nv;
    }
    emit_G(mt + 2 * TB + 8, false);
  }

  bool prefetch = true;

  std::string run(const std::string& kname, uint32_t threads, uint32_t minb) {
    const TileHeader& h = tp.h;
    s << "struct __align__(16) QsbCoef { double2 c[" << std::max<size_t>(1, tp.coef.size()) << "]; };\n";
    s << "extern \"C\" __global__ void __launch_bounds__(" << threads << ", " << minb << ") " << kname
      << "(double2* __restrict__ amps, const __grid_constant__ QsbCoef P) {\n";
    const uint32_t T = 1u << h.t;
    s << "  extern __shared__ double2 sm[];\n";
    s << "  const unsigned tid = threadIdx.x;\n";
    // thread contribution to the global index under the load layout
    s << "  const unsigned long long TL = 0ull";
    for (uint32_t k = 0; k < h.t; ++k) s << " | ((unsigned long long)((tid >> " << k << ") & 1u) << " << h.load.tq[k] << ")";
    s << ";\n";
    s << "  auto base_of = [&](unsigned long long b) {\n";
    for (uint32_t b = 0; b < h.m && h.ntiles > 1; ++b) {
      const uint32_t q = h.S[b];
      s << "    b = ((b >> " << q << ") << " << (q + 1) << ") | (b & " << hexll((1ull << q) - 1) << ");\n";
    }
    s << "    return b;\n  };\n";
    unsigned long long loff[16];
    for (int p = 0; p < 16; ++p) {
      loff[p] = 0;
      for (int k = 0; k < 4; ++k)
        if ((p >> k) & 1) loff[p] |= h.load.rs[k];
    }
    if (prefetch) {
      // Each thread stages its own 16 amplitudes of the next tile in its own
      // shared-memory slots (slot p*T + tid: conflict-free) with cp.async, so
      // HBM reads of tile i+1 overlap the arithmetic of tile i.
      s << "  double2* const PB = sm + " << (tp.transposes ? (1u << h.m) : 0u) << ";\n";
      s << "  auto prefetch = [&](unsigned long long t) {\n";
      s << "    const unsigned long long g = base_of(t) | TL;\n";
      for (int p = 0; p < 16; ++p)
        s << "    cp_async16(PB + " << p * T << " + tid, amps + (g | " << hexll(loff[p]) << "));\n";
      s << "    cp_async_commit();\n  };\n";
      s << "  unsigned long long tile = blockIdx.x;\n";
      s << "  if (tile < " << h.ntiles << "ull) prefetch(tile);\n";
      s << "  for (; tile < " << h.ntiles << "ull; tile += gridDim.x) {\n";
      s << "    const unsigned long long base = base_of(tile);\n";
      s << "    unsigned long long G = base | TL;\n";
      s << "    cp_async_wait_all();\n";
      for (int p = 0; p < 16; ++p) {
        name[p] = fresh();
        s << "    const double2 " << name[p] << " = PB[" << p * T << " + tid];\n";
      }
      s << "    { const unsigned long long nt = tile + gridDim.x; if (nt < " << h.ntiles << "ull) prefetch(nt); }\n";
    } else {
      s << "  for (unsigned long long tile = blockIdx.x; tile < " << h.ntiles << "ull; tile += gridDim.x) {\n";
      s << "    const unsigned long long base = base_of(tile);\n";
      s << "    unsigned long long G = base | TL;\n";
      for (int p = 0; p < 16; ++p) {
        name[p] = fresh();
        s << "    const double2 " << name[p] << " = __ldcs(amps + (G | " << hexll(loff[p]) << "));\n";
      }
    }
    int ti = 0;
    for (const TOp& o : tp.ops) {
      switch (o.type) {
        case TO_MAT1:
        case TO_MAT1_REAL:
        case TO_MAT1_RX: mat1(o); break;
        case TO_FLIP: flip(o); break;
        case TO_PHASE: phase(o); break;
        case TO_DENSE2:
        case TO_DENSE3: dense(o); break;
        case TO_TRANSPOSE: transpose(o, ti++); break;
        case TO_RELABEL: emit_G(tp.meta.data() + o.meta, false); break;
        default: throw RuntimeError("jit: unknown micro-op");
      }
    }
    // Relabels (free SWAPs) make threads store where other threads loaded; with
    // no transpose barrier in the pass, every load must retire before any store.
    if (ti == 0 && std::memcmp(&h.load, &h.store, sizeof(TileConfigAddr)) != 0) s << "    __syncthreads();\n";
    for (int p = 0; p < 16; ++p) {
      unsigned long long off = 0;
      for (int k = 0; k < 4; ++k)
        if ((p >> k) & 1) off |= h.store.rs[k];
      s << "    __stcs(amps + (G | " << hexll(off) << "), " << name[p] << ");\n";
    }
    s << "  }\n}\n";
    return s.str();
  }
};

const char* kPreamble = R"(
// Generated by libqsb (csrc/jit.cpp) for one shared-memory tile pass.
__device__ __forceinline__ void cp_async16(double2* smem, const double2* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// m0*a + m1*b (complex)
__device__ __forceinline__ double2 cmv2(double2 m0, double2 a, double2 m1, double2 b) {
  double re = m0.x * a.x; re = fma(-m0.y, a.y, re); re = fma(m1.x, b.x, re); re = fma(-m1.y, b.y, re);
  double im = m0.x * a.y; im = fma(m0.y, a.x, im); im = fma(m1.x, b.y, im); im = fma(m1.y, b.x, im);
  return make_double2(re, im);
}
// r0*a + r1*b, real coefficients
__device__ __forceinline__ double2 rmv2(double r0, double2 a, double r1, double2 b) {
  return make_double2(fma(r0, a.x, r1 * b.x), fma(r0, a.y, r1 * b.y));
}
// r*a + i*s*b (real r, imaginary i*s)
__device__ __forceinline__ double2 xmv2(double r, double2 a, double s, double2 b) {
  return make_double2(fma(r, a.x, -s * b.y), fma(r, a.y, s * b.x));
}
__device__ __forceinline__ double2 dotrow4(const double2* m, double2 a0, double2 a1, double2 a2, double2 a3) {
  const double2 in[4] = {a0, a1, a2, a3};
  double re = 0.0, im = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) { re = fma(m[c].x, in[c].x, re); re = fma(-m[c].y, in[c].y, re);
                                im = fma(m[c].x, in[c].y, im); im = fma(m[c].y, in[c].x, im); }
  return make_double2(re, im);
}
__device__ __forceinline__ double2 dotrow8(const double2* m, double2 a0, double2 a1, double2 a2, double2 a3,
                                           double2 a4, double2 a5, double2 a6, double2 a7) {
  const double2 in[8] = {a0, a1, a2, a3, a4, a5, a6, a7};
  double re = 0.0, im = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) { re = fma(m[c].x, in[c].x, re); re = fma(-m[c].y, in[c].y, re);
                                im = fma(m[c].x, in[c].y, im); im = fma(m[c].y, in[c].x, im); }
  return make_double2(re, im);
}
)";

std::mutex g_cache_mu;
std::unordered_map<std::string, std::shared_ptr<JitModule>>& cache() {
  static std::unordered_map<std::string, std::shared_ptr<JitModule>> c;
  return c;
}

void nvrtc_compile(JitModule& jm) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, jm.source.c_str(), (jm.name + ".cu").c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS)
    throw RuntimeError("nvrtcCreateProgram failed");
  const char* opts[] = {"-arch=sm_100a", "--std=c++17", "-default-device", "-lineinfo"};
  const nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
  if (r != NVRTC_SUCCESS) {
    size_t ls = 0;
    nvrtcGetProgramLogSize(prog, &ls);
    std::string log(ls, '\0');
    nvrtcGetProgramLog(prog, log.data());
    nvrtcDestroyProgram(&prog);
    throw RuntimeError("NVRTC failed for " + jm.name + ": " + log.substr(0, 2000));
  }
  size_t cs = 0;
  nvrtcGetCUBINSize(prog, &cs);
  jm.cubin.resize(cs);
  nvrtcGetCUBIN(prog, jm.cubin.data());
  nvrtcDestroyProgram(&prog);
  g_compiles.fetch_add(1);
}

uint64_t fnv(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace

uint64_t jit_compiles() { return g_compiles.load(); }
uint64_t jit_cache_hits() { return g_hits.load(); }

namespace {
bool prefetch_enabled() {
  const char* e = std::getenv("QSB_TILE_PREFETCH");
  return !e || std::atoi(e) != 0;
}
uint32_t min_blocks_for(const TileProgram& tp) {
  if (const char* e = std::getenv("QSB_TILE_MINB")) return static_cast<uint32_t>(std::max(1, std::atoi(e)));
  return prefetch_enabled() ? 1 : (tp.h.m >= 13 ? 1 : 2);
}
size_t smem_for(const TileProgram& tp) {
  const size_t tile_bytes = (size_t(1) << tp.h.m) * sizeof(double2);
  return (tp.transposes ? tile_bytes : 0) + (prefetch_enabled() ? tile_bytes : 0);
}
}  // namespace

std::string tile_source(const TileProgram& tp, const std::string& name) {
  Gen g(tp);
  g.prefetch = prefetch_enabled();
  const uint32_t threads = 1u << tp.h.t;
  return std::string(kPreamble) + g.run(name, threads, min_blocks_for(tp));
}

void compile_tile_steps(std::vector<Step>& steps) {
  std::vector<TileProgram*> todo;
  std::vector<std::shared_ptr<JitModule>> fresh;
  for (auto& st : steps) {
    if (st.kind != Step::TileStep) continue;
    TileProgram& tp = *st.tile;
    // name from the body (structure); the source embeds it, so hash twice
    const std::string body = tile_source(tp, "qsb_tile");
    const std::string name = "qsb_tile_" + std::to_string(fnv(body));
    std::string src = tile_source(tp, name);
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = cache().find(src);
    if (it != cache().end()) {
      tp.jit = it->second;
      g_hits.fetch_add(1);
      continue;
    }
    if (const char* dir = std::getenv("QSB_JIT_DUMP")) {  // diagnostics: keep the generated source
      const std::string fn = std::string(dir) + "/step" + std::to_string(&st - steps.data()) + "_" + name + ".cu";
      if (FILE* f = std::fopen(fn.c_str(), "w")) {
        std::fputs(src.c_str(), f);
        std::fclose(f);
      }
    }
    auto jm = std::make_shared<JitModule>();
    jm->name = name;
    jm->source = std::move(src);
    jm->threads = 1u << tp.h.t;
    jm->min_blocks = min_blocks_for(tp);
    jm->smem = smem_for(tp);
    cache()[jm->source] = jm;
    tp.jit = jm;
    fresh.push_back(jm);
  }
  if (fresh.empty()) return;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nthreads = std::min<size_t>(fresh.size(), hw);
  std::atomic<size_t> next{0};
  std::vector<std::string> errors(nthreads);
  auto worker = [&](size_t w) {
    try {
      for (size_t i = next++; i < fresh.size(); i = next++) nvrtc_compile(*fresh[i]);
    } catch (const std::exception& e) {
      errors[w] = e.what();
    }
  };
  std::vector<std::thread> pool;
  for (size_t w = 1; w < nthreads; ++w) pool.emplace_back(worker, w);
  worker(0);
  for (auto& t : pool) t.join();
  for (auto& e : errors)
    if (!e.empty()) {
      std::lock_guard<std::mutex> lk(g_cache_mu);
      for (auto& jm : fresh) cache().erase(jm->source);
      throw RuntimeError(e);
    }
}

void launch_tile(State& s, const TileProgram& tp) {
  if (!tp.jit || tp.jit->cubin.empty()) throw RuntimeError("tile program was not compiled");
  DeviceGuard dg(s.device);
  JitModule& jm = *tp.jit;
  const Driver& d = driver();
  const int dev = s.device & 63;
  const size_t smem = jm.smem;
  CUfunction fn;
  int per_sm;
  {
    std::lock_guard<std::mutex> lk(jm.mu);
    if (!jm.fn[dev]) {
      CUmodule mod;
      cu_check(d.moduleLoadData(&mod, jm.cubin.data()), "cuModuleLoadData");
      CUfunction f;
      cu_check(d.moduleGetFunction(&f, mod, jm.name.c_str()), "cuModuleGetFunction");
      cu_check(d.funcSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                  static_cast<int>(std::max<size_t>(smem, 1))),
               "cuFuncSetAttribute");
      int occ = 0;
      cu_check(d.occupancy(&occ, f, static_cast<int>(jm.threads), smem), "cuOccupancyMaxActiveBlocksPerMultiprocessor");
      jm.mod[dev] = mod;
      jm.fn[dev] = f;
      jm.per_sm[dev] = std::max(occ, 1);
    }
    fn = static_cast<CUfunction>(jm.fn[dev]);
    per_sm = jm.per_sm[dev];
  }
  const unsigned long long cap = static_cast<unsigned long long>(per_sm) * num_sms(s.device);
  const unsigned grid = static_cast<unsigned>(std::min<unsigned long long>(tp.h.ntiles, cap));
  const size_t pbytes = std::max<size_t>(1, tp.coef.size()) * sizeof(double2);
  if (pbytes > kTileBlobBytes) throw RuntimeError("tile coefficient table exceeds the parameter limit");
  alignas(16) static thread_local unsigned char params[kTileBlobBytes];
  std::memset(params, 0, pbytes);
  if (!tp.coef.empty()) std::memcpy(params, tp.coef.data(), tp.coef.size() * sizeof(double2));
  double2* amps = s.amps;
  void* args[] = {&amps, params};
  cu_check(d.launchKernel(fn, grid, 1, 1, jm.threads, 1, 1, static_cast<unsigned>(smem),
                          reinterpret_cast<CUstream>(s.stream), args, nullptr),
           "cuLaunchKernel");
  QSB_LAUNCHED();
}

}  // namespace qsb
