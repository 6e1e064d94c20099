// Per-gate kernels, reductions, measurement and sampling for complex128 state
// vectors on sm_100a.  Every kernel here is one streaming pass over HBM (or
// less); the multi-gate shared-memory passes live in tile.cu.
//
// Reference correspondences (proj/include/qforge/):
//   k_mat1 / k_diag / k_flip / k_swap   statevector.hpp:268-361
//   k_dense<K>                          statevector.hpp:69-106, 363-467
//   reductions                          statevector.hpp:110-130, 158-215; bench.hpp:141-148
//   k_collapse                          statevector.hpp:228-247
//   sampler (serial-equivalent scan)    statevector.hpp:542-570
//   k_pauli                             variational.hpp:33-47
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>

#include "kernels.hpp"

namespace qsb {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxSlots = QS_MAX_TARGETS + QS_MAX_CONTROLS;

// Reserved bit positions (targets and controls) sorted ascending, and the
// forced-one control mask: the GroupIndexer of statevector.hpp:42-64.
struct Slots {
  uint32_t count;
  uint32_t pos[kMaxSlots];
  unsigned long long force;
};

Slots make_slots(const std::vector<uint32_t>& targets, const std::vector<uint32_t>& controls) {
  Slots s{};
  std::vector<uint32_t> all(targets);
  all.insert(all.end(), controls.begin(), controls.end());
  std::sort(all.begin(), all.end());
  s.count = static_cast<uint32_t>(all.size());
  for (size_t i = 0; i < all.size(); ++i) s.pos[i] = all[i];
  s.force = 0;
  for (auto c : controls) s.force |= 1ull << c;
  return s;
}

__device__ __forceinline__ uint64_t deposit(uint64_t g, const Slots& s) {
  for (uint32_t k = 0; k < s.count; ++k) {
    const uint32_t p = s.pos[k];
    const uint64_t low = g & ((1ull << p) - 1);
    g = ((g >> p) << (p + 1)) | low;
  }
  return g | s.force;
}

// deposit specialised for at most MS slots (fully unrolled, early exit); MS =
// 0 is the general loop.  Per-gate kernels with <= 3 slots (1 target + 2
// controls) use MS = 3: no loop control per amplitude group.
template <int MS>
__device__ __forceinline__ uint64_t deposit_n(uint64_t g, const Slots& s) {
  if constexpr (MS == 0) {
    return deposit(g, s);
  } else {
#pragma unroll
    for (int k = 0; k < MS; ++k) {
      if (k >= static_cast<int>(s.count)) break;
      const uint32_t p = s.pos[k];
      const uint64_t low = g & ((1ull << p) - 1);
      g = ((g >> p) << (p + 1)) | low;
    }
    return g | s.force;
  }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// m0*a + m1*b
__device__ __forceinline__ double2 cmv2(double2 m0, double2 a, double2 m1, double2 b) {
  double re = m0.x * a.x;
  re = fma(-m0.y, a.y, re);
  re = fma(m1.x, b.x, re);
  re = fma(-m1.y, b.y, re);
  double im = m0.x * a.y;
  im = fma(m0.y, a.x, im);
  im = fma(m1.x, b.y, im);
  im = fma(m1.y, b.x, im);
  return make_double2(re, im);
}
// |a|^2 exactly as g++ contracts std::norm: fma(re, re, im*im).
__device__ __forceinline__ double norm_ref(double2 a) { return __fma_rn(a.x, a.x, __dmul_rn(a.y, a.y)); }

// 32 B (two adjacent amplitudes) per instruction: sm_100's 256-bit global
// accesses (SASS LDG.E.ENL2.256 / STG.E.ENL2.256).  Used where an amplitude
// pair differs in qubit 0, so one thread's accesses fill whole sectors.
__device__ __forceinline__ void ld_pair(const double2* p, double2& x, double2& y) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(x.x), "=d"(x.y), "=d"(y.x), "=d"(y.y)
               : "l"(p));
}
__device__ __forceinline__ void st_pair(double2* p, double2 x, double2 y) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(x.x), "d"(x.y), "d"(y.x), "d"(y.y)
               : "memory");
}

uint32_t grid_for(uint64_t work, int device, int per_sm = 8) {
  const uint64_t blocks = (work + kThreads - 1) / kThreads;
  const uint64_t cap = static_cast<uint64_t>(num_sms(device)) * per_sm;
  return static_cast<uint32_t>(std::max<uint64_t>(1, std::min(blocks, cap)));
}

// ------------------------------------------------------------------ gates

template <int MS>
__global__ void __launch_bounds__(kThreads) k_mat1(double2* __restrict__ a, uint64_t groups, Slots sl,
                                                   uint64_t bit, double2 m0, double2 m1, double2 m2,
                                                   double2 m3) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = deposit_n<MS>(g, sl), i1 = i0 ^ bit;  // bit: the target (or a SWAP's two bits)
    const double2 x = a[i0], y = a[i1];
    a[i0] = cmv2(m0, x, m1, y);
    a[i1] = cmv2(m2, x, m3, y);
  }
}

// Target qubit 0: each pair is 32 contiguous bytes, one 256-bit load / store.
template <int MS>
__global__ void __launch_bounds__(kThreads) k_mat1_q0(double2* __restrict__ a, uint64_t groups, Slots sl, double2 m0,
                                                      double2 m1, double2 m2, double2 m3) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = deposit_n<MS>(g, sl);
    double2 x, y;
    ld_pair(a + i0, x, y);
    st_pair(a + i0, cmv2(m0, x, m1, y), cmv2(m2, x, m3, y));
  }
}

// skip_zero: only the bit-set half is multiplied by d1 (the target is then a
// forced-one slot); otherwise pairs get (d0, d1).
template <int MS>
__global__ void __launch_bounds__(kThreads) k_diag(double2* __restrict__ a, uint64_t groups, Slots sl,
                                                   uint64_t bit, double2 d0, double2 d1, int skip_zero) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = deposit_n<MS>(g, sl);
    if (skip_zero) {
      a[i0] = cmul(a[i0], d1);
    } else {
      a[i0] = cmul(a[i0], d0);
      a[i0 | bit] = cmul(a[i0 | bit], d1);
    }
  }
}

// Diagonal on qubit 0 (both entries applied): one 256-bit access per pair.
template <int MS>
__global__ void __launch_bounds__(kThreads) k_diag_q0(double2* __restrict__ a, uint64_t groups, Slots sl, double2 d0,
                                                      double2 d1) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = deposit_n<MS>(g, sl);
    double2 x, y;
    ld_pair(a + i0, x, y);
    st_pair(a + i0, cmul(x, d0), cmul(y, d1));
  }
}

template <int MS>
__global__ void __launch_bounds__(kThreads) k_flip(double2* __restrict__ a, uint64_t groups, Slots sl,
                                                   uint64_t bit) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = deposit_n<MS>(g, sl);
    const double2 x = __ldcs(a + i0), y = __ldcs(a + (i0 | bit));
    __stcs(a + i0, y);
    __stcs(a + (i0 | bit), x);
  }
}

template <int MS>
__global__ void __launch_bounds__(kThreads) k_swap(double2* __restrict__ a, uint64_t groups, Slots sl,
                                                   uint64_t ba, uint64_t bb) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t base = deposit_n<MS>(g, sl);
    const double2 x = __ldcs(a + (base | ba)), y = __ldcs(a + (base | bb));
    __stcs(a + (base | ba), y);
    __stcs(a + (base | bb), x);
  }
}

// Dense 2^K x 2^K block (K <= 5): a group of 2^K consecutive lanes handles one
// amplitude group; lane r owns output row r with its matrix row in registers;
// inputs are exchanged through shared memory (broadcast reads).
struct TargetMasks {
  unsigned long long m[QS_MAX_TARGETS];  // m[b] = 1 << targets[K-1-b]
};

// The block's matrix travels as a __grid_constant__ kernel parameter
// (constant bank: uniform operands of the FMAs; no upload, no host sync).
template <int K>
struct DenseM {
  double2 m[1 << (2 * K)];
};
template <int K>
constexpr int dense_k(const DenseM<K>*) { return K; }

// Dense 2^K x 2^K block, K <= 4: one thread per amplitude group.  Consecutive
// lanes take consecutive groups, so every load / store instruction of a warp
// covers contiguous runs (2^lowest-target amplitudes); the 2^K inputs stay in
// registers and each output row is an FMA chain with constant-bank
// coefficients (same summation order as the reference's row dot product,
// statevector.hpp:69-106).
// P >= 0: the block's bit P is qubit 0 (tm.m[P] == 1), so x[c] and
// x[c | 1 << P] are adjacent and travel as one 256-bit access.
template <int K, int P = -1>
__global__ void __launch_bounds__(kThreads) k_dense_g(double2* __restrict__ a, uint64_t groups, Slots sl,
                                                      TargetMasks tm, const __grid_constant__ DenseM<K> M) {
  constexpr int G = 1 << K;
  auto offset = [&](int c) {
    uint64_t off = 0;
#pragma unroll
    for (int b = 0; b < K; ++b)
      if ((c >> b) & 1) off |= tm.m[b];
    return off;
  };
  auto row = [&](int r, const double2* x) {
    double re = 0, im = 0;
#pragma unroll
    for (int c = 0; c < G; ++c) {
      const double2 m = M.m[r * G + c];
      re = fma(m.x, x[c].x, re);
      re = fma(-m.y, x[c].y, re);
      im = fma(m.x, x[c].y, im);
      im = fma(m.y, x[c].x, im);
    }
    return make_double2(re, im);
  };
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t base = deposit(g, sl);
    double2 x[G];
#pragma unroll
    for (int c = 0; c < G; ++c) {
      if constexpr (P < 0) {
        x[c] = __ldcs(a + (base | offset(c)));
      } else if (!((c >> P) & 1)) {
        ld_pair(a + (base | offset(c)), x[c], x[c | (1 << P)]);
      }
    }
#pragma unroll
    for (int r = 0; r < G; ++r) {
      if constexpr (P < 0) {
        __stcs(a + (base | offset(r)), row(r, x));
      } else if (!((r >> P) & 1)) {
        st_pair(a + (base | offset(r)), row(r, x), row(r | (1 << P), x));
      }
    }
  }
}

// Dense block on the low qubits (every target < 12, no controls): a block
// owns a contiguous 4096-amplitude chunk -- read and written back with
// coalesced 512 B warp accesses through shared memory (XOR-swizzled 16 B
// slots: conflict-free for the strided per-group reads of targets {0..K-1})
// -- and each thread applies the block to the complete groups it is given.
constexpr int kStageLog = 12;
__device__ __forceinline__ uint32_t stage_slot(uint32_t i) { return i ^ ((i >> 3) & 7u); }

template <int K>
__global__ void __launch_bounds__(kThreads) k_dense_s(double2* __restrict__ a, uint64_t chunks, Slots sl,
                                                      TargetMasks tm, const __grid_constant__ DenseM<K> M) {
  constexpr int G = 1 << K;
  constexpr uint32_t C = 1u << kStageLog, NG = C >> K;
  extern __shared__ double2 st[];
  for (uint64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    double2* base = a + (ch << kStageLog);
    for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) st[stage_slot(i)] = __ldcs(base + i);
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < NG; g += blockDim.x) {
      const uint32_t b0 = static_cast<uint32_t>(deposit(g, sl));
      double2 x[G];
      uint32_t off[G];
#pragma unroll
      for (int c = 0; c < G; ++c) {
        uint32_t o = 0;
#pragma unroll
        for (int b = 0; b < K; ++b)
          if ((c >> b) & 1) o |= static_cast<uint32_t>(tm.m[b]);
        off[c] = b0 | o;
        x[c] = st[stage_slot(off[c])];
      }
#pragma unroll
      for (int r = 0; r < G; ++r) {
        double re = 0, im = 0;
#pragma unroll
        for (int c = 0; c < G; ++c) {
          const double2 m = M.m[r * G + c];
          re = fma(m.x, x[c].x, re);
          re = fma(-m.y, x[c].y, re);
          im = fma(m.x, x[c].y, im);
          im = fma(m.y, x[c].x, im);
        }
        st[stage_slot(off[r])] = make_double2(re, im);  // this thread's own group: no other reader
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) __stcs(base + i, st[stage_slot(i)]);
    __syncthreads();
  }
}

// Lane-cooperative form (K = 5, which is FP64-bound at 8 * 32 flop per
// amplitude, and blocks on the lowest qubits, whose 2^K amplitudes are
// contiguous): a group of 2^K consecutive lanes handles one amplitude group;
// lane r owns output row r; inputs are exchanged through shared memory
// (broadcast reads).  The matrix is staged transposed in shared memory first
// (a per-lane row read straight from the parameter bank would serialise).
template <int K>
__global__ void __launch_bounds__(kThreads) k_dense(double2* __restrict__ a, uint64_t groups, Slots sl,
                                                    TargetMasks tm, const __grid_constant__ DenseM<K> M) {
  constexpr int G = 1 << K;
  constexpr int GPB = kThreads / G;  // groups per block iteration
  __shared__ double2 v[kThreads];
  __shared__ double2 mt[G * G];  // mt[c * G + r] = M[r][c]
  for (int i = threadIdx.x; i < G * G; i += blockDim.x) mt[(i % G) * G + i / G] = M.m[i];
  __syncthreads();
  const int tid = threadIdx.x, r = tid & (G - 1), gl = tid >> K;
  double2 row[G];
#pragma unroll
  for (int c = 0; c < G; ++c) row[c] = mt[c * G + r];
  uint64_t offr = 0;
#pragma unroll
  for (int b = 0; b < K; ++b)
    if ((r >> b) & 1) offr |= tm.m[b];
  for (uint64_t gb = (uint64_t)blockIdx.x * GPB; gb < groups; gb += (uint64_t)gridDim.x * GPB) {
    const uint64_t g = gb + gl;
    const bool valid = g < groups;
    const uint64_t idx = valid ? (deposit(g, sl) | offr) : 0;
    v[tid] = valid ? __ldcs(a + idx) : make_double2(0, 0);
    __syncwarp();
    double re = 0, im = 0;
#pragma unroll
    for (int c = 0; c < G; ++c) {
      const double2 x = v[(gl << K) + c];
      re = fma(row[c].x, x.x, re);
      re = fma(-row[c].y, x.y, re);
      im = fma(row[c].x, x.y, im);
      im = fma(row[c].y, x.x, im);
    }
    __syncwarp();
    if (valid) __stcs(a + idx, make_double2(re, im));
  }
}

bool pair256_enabled() { return !std::getenv("QSB_NO_PAIR256"); }

// k_dense_g with the pair bit P = pbit (qubit 0 at block bit P), or unpaired.
template <int K, int P>
void launch_dense_g(const State& s, uint64_t groups, const Slots& sl, const TargetMasks& tm, const DenseM<K>& M,
                    int pbit) {
  if constexpr (P < 0) {
    k_dense_g<K><<<grid_for(groups, s.device), kThreads, 0, s.stream>>>(s.amps, groups, sl, tm, M);
  } else {
    if (pbit == P) k_dense_g<K, P><<<grid_for(groups, s.device), kThreads, 0, s.stream>>>(s.amps, groups, sl, tm, M);
    else launch_dense_g<K, P - 1>(s, groups, sl, tm, M, pbit);
  }
}

void launch_mat1(const State& s, uint64_t groups, const Slots& sl, uint64_t bit, double2 m0, double2 m1, double2 m2,
                 double2 m3) {
  const uint32_t grid = grid_for(groups, s.device);
  if (bit == 1 && pair256_enabled())
    (sl.count <= 3 ? k_mat1_q0<3> : k_mat1_q0<0>)<<<grid, kThreads, 0, s.stream>>>(s.amps, groups, sl, m0, m1, m2, m3);
  else
    (sl.count <= 3 ? k_mat1<3> : k_mat1<0>)<<<grid, kThreads, 0, s.stream>>>(s.amps, groups, sl, bit, m0, m1, m2, m3);
}

// Dense block with K > 5: one group per 2^K threads spread over the block,
// matrix rows read through the cache.  Rare (custom gates wider than the
// fusion cap); correctness path.
__global__ void __launch_bounds__(kThreads) k_dense_wide(double2* __restrict__ a, uint64_t groups, Slots sl,
                                                         TargetMasks tm, int K, const double2* __restrict__ M) {
  extern __shared__ double2 vbuf[];
  const int G = 1 << K;
  for (uint64_t g = blockIdx.x; g < groups; g += gridDim.x) {
    const uint64_t base = deposit(g, sl);
    for (int r = threadIdx.x; r < G; r += blockDim.x) {
      uint64_t off = 0;
      for (int b = 0; b < K; ++b)
        if ((r >> b) & 1) off |= tm.m[b];
      vbuf[r] = a[base | off];
    }
    __syncthreads();
    for (int r = threadIdx.x; r < G; r += blockDim.x) {
      uint64_t off = 0;
      for (int b = 0; b < K; ++b)
        if ((r >> b) & 1) off |= tm.m[b];
      double re = 0, im = 0;
      for (int c = 0; c < G; ++c) {
        const double2 mm = M[(uint64_t)r * G + c], x = vbuf[c];
        re = fma(mm.x, x.x, re);
        re = fma(-mm.y, x.y, re);
        im = fma(mm.x, x.y, im);
        im = fma(mm.y, x.x, im);
      }
      a[base | off] = make_double2(re, im);
    }
    __syncthreads();
  }
}

// Dense 64 x 64 block (K = 6, wider than the fusion cap): one warp per
// amplitude group, the matrix transposed in shared memory (lane r reads row r
// of column c: consecutive 16 B, conflict-free), the group's 64 inputs in a
// per-warp slice (broadcast reads); lane l owns rows l and l + 32.
__global__ void __launch_bounds__(kThreads) k_dense6(double2* __restrict__ a, uint64_t groups, Slots sl, TargetMasks tm,
                                                     const double2* __restrict__ Mg) {
  extern __shared__ double2 s6[];
  double2* Mt = s6;                 // Mt[c * 64 + r] = M[r][c]
  double2* xin = s6 + 64 * 64;      // 64 inputs per warp
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) Mt[(i & 63) * 64 + (i >> 6)] = Mg[i];
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  double2* xw = xin + w * 64;
  uint64_t off0 = 0, off1 = 0;
#pragma unroll
  for (int b = 0; b < 6; ++b) {
    if ((l >> b) & 1) off0 |= tm.m[b];
    if (((l + 32) >> b) & 1) off1 |= tm.m[b];
  }
  for (uint64_t g = (uint64_t)blockIdx.x * nw + w; g < groups; g += (uint64_t)gridDim.x * nw) {
    const uint64_t base = deposit(g, sl);
    xw[l] = a[base | off0];
    xw[l + 32] = a[base | off1];
    __syncwarp();
    double r0 = 0, i0 = 0, r1 = 0, i1 = 0;
    for (int c = 0; c < 64; ++c) {
      const double2 x = xw[c], m0 = Mt[c * 64 + l], m1 = Mt[c * 64 + l + 32];
      r0 = fma(m0.x, x.x, r0);
      r0 = fma(-m0.y, x.y, r0);
      i0 = fma(m0.x, x.y, i0);
      i0 = fma(m0.y, x.x, i0);
      r1 = fma(m1.x, x.x, r1);
      r1 = fma(-m1.y, x.y, r1);
      i1 = fma(m1.x, x.y, i1);
      i1 = fma(m1.y, x.x, i1);
    }
    __syncwarp();
    a[base | off0] = make_double2(r0, i0);
    a[base | off1] = make_double2(r1, i1);
  }
}

// ------------------------------------------------------------- reductions
// Fixed grid and fixed per-block ranges: run-to-run deterministic (no atomics).
constexpr uint32_t kRedBlocks = 1184;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
  __syncthreads();
  return t;  // valid in thread 0
}

// mode 0: sum |a|^2 ; 1: sum over i with bit q set ; 2: sum |a_i|^2 (i+1)
__global__ void __launch_bounds__(kThreads) k_reduce(const double2* __restrict__ a, uint64_t n_items, int mode,
                                                     uint64_t bit, uint64_t index_base, double* __restrict__ partial) {
  __shared__ double sh[kThreads / 32];
  const uint64_t chunk = (n_items + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * chunk, hi = min(n_items, lo + chunk);
  double s = 0;
  for (uint64_t g = lo + threadIdx.x; g < hi; g += blockDim.x) {
    if (mode == 1) {
      const uint64_t low = g & (bit - 1);
      const uint64_t i = ((g & ~(bit - 1)) << 1) | bit | low;
      s += norm_ref(a[i]);
    } else if (mode == 2) {
      s += norm_ref(a[g]) * (double)(index_base + g + 1);
    } else {
      s += norm_ref(a[g]);
    }
  }
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void k_finalize(const double* __restrict__ partial, int count, double* __restrict__ out) {
  __shared__ double sh[kThreads / 32];
  double s = 0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) s += partial[i];
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) *out = t;
}

// Marginal over m <= 12 qubits: block (x, b) reduces a fixed range of group
// indices of bin b.
__global__ void __launch_bounds__(kThreads) k_marginal(const double2* __restrict__ a, uint64_t per_bin, Slots sl,
                                                       const uint32_t* __restrict__ qubits, uint32_t m,
                                                       double* __restrict__ partial) {
  __shared__ double sh[kThreads / 32];
  const uint32_t bin = blockIdx.y;
  uint64_t fixed = 0;
  for (uint32_t b = 0; b < m; ++b)
    if ((bin >> b) & 1) fixed |= 1ull << qubits[b];
  const uint64_t chunk = (per_bin + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * chunk, hi = min(per_bin, lo + chunk);
  double s = 0;
  for (uint64_t g = lo + threadIdx.x; g < hi; g += blockDim.x) s += norm_ref(a[deposit(g, sl) | fixed]);
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) partial[(uint64_t)bin * gridDim.x + blockIdx.x] = t;
}

// Marginal with coalesced reads (m <= 12, >= 5 local qubits): lane l of every
// warp reads amplitude (.. | l) of a 32-amplitude aligned run, so the marginal
// qubits below 5 are lane bits (each lane's bin part is fixed) and those
// above are fixed per block (blockIdx.y enumerates them).  A lane sums its
// amplitudes; lanes that differ only in non-marginal bits are combined by a
// fixed xor butterfly, warps in index order: deterministic, no atomics, and
// every byte of the state is read once (the strided per-bin form re-read the
// 32 B sectors of bins that fix low qubits).
struct MarginalMap {
  uint32_t kh;            // marginal qubits >= 5
  uint32_t qh[12];        // ... ascending
  uint32_t rh[12];        // their result bits
  int rl[5];              // result bit of lane bit b, -1 if b is not a marginal qubit
  uint32_t lane_free;     // lane bits that are not marginal qubits
};

__global__ void __launch_bounds__(kThreads) k_marginal_lanes(const double2* __restrict__ a, uint64_t per_hi, Slots slh,
                                                             MarginalMap mm, double* __restrict__ partial) {
  __shared__ double sh[kThreads / 32][32];
  const uint32_t bh = blockIdx.y, lane = threadIdx.x & 31u, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t fixed = 0;
  uint32_t bin = 0;
#pragma unroll
  for (uint32_t j = 0; j < 12; ++j)  // static indices: no local copy of the map
    if (j < mm.kh && ((bh >> j) & 1u)) {
      fixed |= 1ull << mm.qh[j];
      bin |= 1u << mm.rh[j];
    }
  for (int b = 0; b < 5; ++b)
    if (mm.rl[b] >= 0 && ((lane >> b) & 1u)) bin |= 1u << mm.rl[b];
  const uint64_t chunk = (per_hi + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * chunk, hi = min(per_hi, lo + chunk);
  double s = 0;
  uint64_t g = lo + w;
  for (; g + 3 * nw < hi; g += 4 * nw) {  // four runs in flight per lane, summed in order
    const double2 v0 = __ldcs(a + ((deposit(g, slh) << 5) | fixed | lane));
    const double2 v1 = __ldcs(a + ((deposit(g + nw, slh) << 5) | fixed | lane));
    const double2 v2 = __ldcs(a + ((deposit(g + 2 * nw, slh) << 5) | fixed | lane));
    const double2 v3 = __ldcs(a + ((deposit(g + 3 * nw, slh) << 5) | fixed | lane));
    s += norm_ref(v0);
    s += norm_ref(v1);
    s += norm_ref(v2);
    s += norm_ref(v3);
  }
  for (; g < hi; g += nw) s += norm_ref(__ldcs(a + ((deposit(g, slh) << 5) | fixed | lane)));
  for (int b = 0; b < 5; ++b)
    if ((mm.lane_free >> b) & 1u) s += __shfl_xor_sync(0xffffffffu, s, 1 << b);
  sh[w][lane] = s;
  __syncthreads();
  if (w == 0 && (lane & mm.lane_free) == 0) {
    double t = 0;
    for (uint32_t i = 0; i < nw; ++i) t += sh[i][lane];
    partial[(uint64_t)bin * gridDim.x + blockIdx.x] = t;
  }
}

// Marginal over states of >= 8 + kh qubits: a warp reads whole 256-amplitude
// runs (qubits 0..7: lane = qubits 0..4, j = qubits 5..7; eight 512 B loads in
// flight per warp), so every block streams contiguous 4 KiB pieces whatever
// low marginal qubits there are; per-lane accumulators per j, combined per
// result bin in fixed order (deterministic).  blockIdx.y = the marginal
// qubits >= 8.
struct MarginalRuns {
  uint32_t kh;         // marginal qubits >= 8
  uint32_t qh[12];     // ... ascending
  uint32_t rh[12];     // their result bits
  int rl[5];           // result bit of lane bit b (qubit b), -1 if not marginal
  int rm[3];           // result bit of j bit b (qubit 5 + b), -1 if not marginal
  uint32_t lane_free;  // lane bits that are not marginal qubits
  uint32_t mid_free;   // j bits that are not marginal qubits
};

__global__ void __launch_bounds__(kThreads) k_marginal_runs(const double2* __restrict__ a, uint64_t per_hi, Slots slh,
                                                            MarginalRuns mm, double* __restrict__ partial) {
  __shared__ double sh[kThreads / 32][8][32];
  const uint32_t bh = blockIdx.y, lane = threadIdx.x & 31u, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t fixed = 0;
  uint32_t bin_hi = 0;
#pragma unroll
  for (uint32_t j = 0; j < 12; ++j)
    if (j < mm.kh && ((bh >> j) & 1u)) {
      fixed |= 1ull << mm.qh[j];
      bin_hi |= 1u << mm.rh[j];
    }
  const uint64_t chunk = (per_hi + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * chunk, hi = min(per_hi, lo + chunk);
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (uint64_t g = lo + w; g < hi; g += nw) {
    const double2* r = a + ((deposit(g, slh) << 8) | fixed | lane);
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcs(r + 32 * j);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += norm_ref(v[j]);
  }
  // j values that differ only in non-marginal bits share a bin: fold them
  // into the representative (free bits zero), in ascending j
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j & mm.mid_free) continue;
    double t = 0;
#pragma unroll
    for (int j2 = 0; j2 < 8; ++j2)
      if ((j2 & ~mm.mid_free) == static_cast<uint32_t>(j)) t += acc[j2];
    for (int b = 0; b < 5; ++b)
      if ((mm.lane_free >> b) & 1u) t += __shfl_xor_sync(0xffffffffu, t, 1 << b);
    sh[w][j][lane] = t;
  }
  __syncthreads();
  const uint32_t j = threadIdx.x >> 5, l = threadIdx.x & 31u;  // one (j, lane) entry per thread
  if ((j & mm.mid_free) == 0 && (l & mm.lane_free) == 0) {
    double t = 0;
    for (uint32_t i = 0; i < nw; ++i) t += sh[i][j][l];
    uint32_t bin = bin_hi;
    for (int b = 0; b < 5; ++b)
      if (mm.rl[b] >= 0 && ((l >> b) & 1u)) bin |= 1u << mm.rl[b];
    for (int b = 0; b < 3; ++b)
      if (mm.rm[b] >= 0 && ((j >> b) & 1u)) bin |= 1u << mm.rm[b];
    partial[(uint64_t)bin * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void k_marginal_finalize(const double* __restrict__ partial, uint32_t per, uint32_t bins,
                                    double* __restrict__ out) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= bins) return;
  double s = 0;
  for (uint32_t i = 0; i < per; ++i) s += partial[(uint64_t)b * per + i];
  out[b] = s;
}

// Marginal over many qubits: one thread per bin, serial over its members.
__global__ void k_marginal_wide(const double2* __restrict__ a, uint64_t per_bin, Slots sl,
                                const uint32_t* __restrict__ qubits, uint32_t m, double* __restrict__ out) {
  const uint64_t bins = 1ull << m;
  for (uint64_t bin = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; bin < bins;
       bin += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t fixed = 0;
    for (uint32_t b = 0; b < m; ++b)
      if ((bin >> b) & 1) fixed |= 1ull << qubits[b];
    double s = 0;
    for (uint64_t g = 0; g < per_bin; ++g) s += norm_ref(a[deposit(g, sl) | fixed]);
    out[bin] = s;
  }
}

__global__ void __launch_bounds__(kThreads) k_probs(const double2* __restrict__ a, uint64_t off, uint64_t count,
                                                    double* __restrict__ p) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = norm_ref(a[off + i]);
}

__global__ void __launch_bounds__(kThreads) k_collapse(double2* __restrict__ a, uint64_t size, uint64_t bit,
                                                       int outcome, double inv) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < size; i += (uint64_t)gridDim.x * blockDim.x) {
    const bool one = (i & bit) != 0;
    if (one == (outcome == 1)) {
      const double2 x = a[i];
      a[i] = make_double2(x.x * inv, x.y * inv);
    } else {
      a[i] = make_double2(0, 0);
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_scale(double2* __restrict__ a, uint64_t size, double2 f) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < size; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = cmul(a[i], f);
}

__global__ void __launch_bounds__(kThreads) k_basis(double2* __restrict__ a, uint64_t size, uint64_t index) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < size; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = make_double2(i == index ? 1.0 : 0.0, 0.0);
}

// zeros every amplitude whose global index disagrees with (mask, val): the
// part of a run from a basis state that no tile pass has written yet
__global__ void __launch_bounds__(kThreads) k_zero_outside(double2* __restrict__ a, uint64_t size, uint64_t rank_base,
                                                           uint64_t mask, uint64_t val) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < size; i += (uint64_t)gridDim.x * blockDim.x)
    if (((i | rank_base) & mask) != val) a[i] = make_double2(0.0, 0.0);
}

// ------------------------------------------------- rank-bit exchanges
// Swapping rank bit j with local bit p: the shard whose bit j is x keeps the
// half with local bit p == x and trades the other half with its partner.

// Both shards on this device (single-process shard groups): a holds x = 0
// (sends its p == 1 half), b holds x = 1 (sends its p == 0 half).
__global__ void __launch_bounds__(kThreads) k_swap_halves(double2* __restrict__ a, double2* __restrict__ b,
                                                          uint64_t count, uint32_t p) {
  const uint64_t bit = 1ull << p;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t l = ((i >> p) << (p + 1)) | (i & (bit - 1));
    const double2 x = a[l | bit], y = b[l];
    a[l | bit] = y;
    b[l] = x;
  }
}

struct ExchangeBits {
  uint32_t lpos[kMaxExchangeBits];
  unsigned long long pmask, aval;
};

// Multi-bit exchanges (all-to-all among 2^k ranks): block d of a shard is the
// set of local indices whose bits at positions lpos[0..k) equal d's bits,
// enumerated by the remaining bits in ascending order (both ends agree).
struct BlockSpec {
  uint32_t k;
  uint32_t sorted[16];      // lpos ascending (zero-bit insertion order)
  unsigned long long val;   // sum of d_i << lpos[i]
};

__device__ __forceinline__ uint64_t block_index(const BlockSpec& b, uint64_t i) {
  for (uint32_t s = 0; s < b.k; ++s) {
    const uint32_t p = b.sorted[s];
    i = ((i >> p) << (p + 1)) | (i & ((1ull << p) - 1));
  }
  return i | b.val;
}

// Gathers elements [off, off + cnt) of block `b` into out.
__global__ void __launch_bounds__(kThreads) k_pack_block(const double2* __restrict__ a, const BlockSpec b,
                                                         uint64_t off, uint64_t cnt, double2* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = a[block_index(b, off + i)];
}

__global__ void __launch_bounds__(kThreads) k_unpack_block(double2* __restrict__ a, const BlockSpec b, uint64_t off,
                                                           uint64_t cnt, const double2* __restrict__ in) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x)
    a[block_index(b, off + i)] = in[i];
}

// Peer-memory exchange (one kernel, no staging): every amplitude of this
// shard is stored straight into its owner's second buffer after the swap of
// rank bits gpos[i] <-> local bits lpos[i].  Local index l goes to the rank
// whose exchanged bits equal l's bits at lpos (table slot d) at local index
// l with those bits replaced by this rank's exchanged bits (aval).  Remote
// slots are NVLink peer pointers (CUDA IPC) or sibling shards on this device.
struct PeerTable {
  double2* p[kMaxPeers];
};

__global__ void __launch_bounds__(kThreads) k_scatter_exchange(const double2* __restrict__ src, const PeerTable t,
                                                               uint64_t size, uint32_t k, ExchangeBits eb) {
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < size; l += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t d = 0;
    for (uint32_t i = 0; i < k; ++i) d |= static_cast<uint32_t>((l >> eb.lpos[i]) & 1ull) << i;
    t.p[d][(l & ~eb.pmask) | eb.aval] = src[l];
  }
  __threadfence_system();
}

// ------------------------------------------------- qubit permutation
// Out-of-place bit permutation of the index (the layout restore that ends a
// plan whose SWAPs were absorbed as relabels): out[sigma(i)] = in[i], where
// sigma moves index bit q to bit pos[q].  One HBM pass, coalesced on both
// sides: a tile covers the 10 input bits A = {0..4} + sigma^-1({0..4}) (+ the
// lowest others), staged in shared memory; reads run over input bits 0..4 and
// writes over output bits 0..4.  Offsets come from 32-entry tables.
constexpr uint32_t kPermTileBits = 10, kPermTile = 1u << kPermTileBits;

struct PermSpec {
  uint32_t nb;                              // base (tile-index) bits
  uint8_t bin[64], bout[64];                // their input / output positions
  unsigned long long in_lo[32], in_hi[32];  // input offset of local e (bits 0-4 / 5-9)
  unsigned long long out_lo[32], out_hi[32];// output offset of local f
  uint16_t e_lo[32], e_hi[32];              // local e feeding output local f
};

__global__ void __launch_bounds__(kThreads) k_permute(const double2* __restrict__ in, double2* __restrict__ out,
                                                      const PermSpec ps, uint64_t ntiles, double* __restrict__ red) {
  __shared__ double2 tile[kPermTile];
  __shared__ double sh[kThreads / 32];
  double acc = 0.0;  // red != null: checksum of what this block stores (bench.hpp:141-148)
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint64_t bi = 0, bo = 0;
    for (uint32_t k = 0; k < ps.nb; ++k)
      if ((t >> k) & 1ull) {
        bi |= 1ull << ps.bin[k];
        bo |= 1ull << ps.bout[k];
      }
    for (uint32_t e = threadIdx.x; e < kPermTile; e += kThreads)
      tile[e ^ ((e >> 5) & 7u)] = __ldcs(in + (bi | ps.in_lo[e & 31u] | ps.in_hi[e >> 5]));
    __syncthreads();
    for (uint32_t f = threadIdx.x; f < kPermTile; f += kThreads) {
      const uint32_t e = ps.e_lo[f & 31u] | ps.e_hi[f >> 5];
      const uint64_t o = bo | ps.out_lo[f & 31u] | ps.out_hi[f >> 5];
      const double2 v = tile[e ^ ((e >> 5) & 7u)];
      __stcs(out + o, v);
      if (red) acc += norm_ref(v) * (double)(o + 1);
    }
    __syncthreads();
  }
  if (red) {
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) red[blockIdx.x] = t;
  }
}

// ------------------------------------------------- serial-equivalent scan
// The reference's BasisSampler accumulates acc += |a_i|^2 left to right in
// double (statevector.hpp:544-552); counts depend on those exact roundings.
// For non-negative addends the running sum is monotone, and while it stays in
// one binade [2^e, 2^(e+1)) every partial sum is a multiple of u = 2^(e-52),
// so fl(acc + p) = acc + u * rint(p / u) exactly unless p/u is a tie (then the
// result depends on acc's parity) or the sum leaves the binade.  We therefore
//   B) per chunk, guess the starting binade from a plain parallel estimate and
//      sum the integers rint(p/u) (flagging ties / oversize addends);
//   C) walk the chunks in order on one warp: a chunk whose guess matches the
//      exact running value and which cannot leave the binade advances by an
//      exact integer add; any other chunk is replayed 32 elements at a time
//      (same integer trick per 32, true serial double adds when it fails);
//   D) expand the clean chunks in parallel: cum_j = (A_c/u + prefix k) * u.
// Every cum_j equals the serial double accumulation bit for bit.

__global__ void __launch_bounds__(kThreads) k_chunk_sum(const double* __restrict__ p, uint64_t n, uint64_t C,
                                                        double* __restrict__ S) {
  __shared__ double sh[kThreads / 32];
  const uint64_t lo = blockIdx.x * C, hi = min(n, lo + C);
  double s = 0;
  for (uint64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) s += p[j];
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) S[blockIdx.x] = t;
}

// exclusive scan of chunk sums (estimates only: they pick each chunk's binade
// guess, any summation order will do), one warp
__global__ void k_scan_estimate(const double* __restrict__ S, uint32_t nc, double* __restrict__ E,
                                const double* __restrict__ carry) {
  const int lane = threadIdx.x & 31;
  double acc = carry ? *carry : 0.0;
  for (uint32_t c0 = 0; c0 < nc; c0 += 32) {
    const double x = c0 + lane < nc ? S[c0 + lane] : 0.0;
    double v = x;
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    if (c0 + lane < nc) E[c0 + lane] = acc + (v - x);
    acc += __shfl_sync(0xffffffffu, v, 31);
  }
}

struct ChunkInfo {
  long long K;  // sum of rint(p/u) over the chunk
  int e;        // assumed binade exponent at chunk start
  int clean;    // 1: no ties, no oversize addend, normal range; 2: every addend is
                //    exactly 0 (the chunk leaves any running sum unchanged)
};

// Exponent / power-of-two helpers by bit manipulation (exact; normal,
// positive arguments): no DDIV, no libm ilogb / ldexp in the scan loops.
__device__ __forceinline__ int exp_of(double x) { return (int)((__double_as_longlong(x) >> 52) & 0x7ff) - 1023; }
__device__ __forceinline__ double pow2(int k) { return __longlong_as_double((long long)(k + 1023) << 52); }

// returns false for a tie or an addend too large for the one-binade model;
// inv_u = 1/u = 2^(52-e), so p * inv_u is p/u exactly
__device__ __forceinline__ bool int_step(double p, double inv_u, long long& k) {
  const double x = p * inv_u;
  if (!(x < 4503599627370496.0)) return false;  // 2^52
  const double f = floor(x);
  const double frac = x - f;
  if (frac == 0.5) return false;
  k = (long long)(frac > 0.5 ? f + 1.0 : f);
  return true;
}

// Each chunk is also split into kSub sub-chunks with their own records: a
// chunk that cannot advance in one step (a tie, a binade exit) is walked
// sub-chunk by sub-chunk, and only the sub-chunks that fail are replayed
// element by element.
constexpr int kSub = 16;

__global__ void __launch_bounds__(kThreads) k_chunk_ints(const double* __restrict__ p, uint64_t n, uint64_t C,
                                                         const double* __restrict__ E, ChunkInfo* __restrict__ info,
                                                         ChunkInfo* __restrict__ sub) {
  __shared__ long long shk[kSub];
  __shared__ int shb[kSub];
  const uint64_t lo = blockIdx.x * C, hi = min(n, lo + C), Cs = C / kSub;
  const double est = E[blockIdx.x];
  const bool usable = est >= 2.2250738585072014e-308 * 4503599627370496.0;  // u stays normal
  const int e = usable ? exp_of(est) : 0;
  const double inv_u = usable ? pow2(52 - e) : 1.0;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int sc = w; sc < kSub; sc += (int)(blockDim.x >> 5)) {  // one warp per sub-chunk
    const uint64_t slo = min(hi, lo + sc * Cs), shi = min(hi, slo + Cs);
    long long K = 0;
    int bad = usable ? 0 : 1, nz = 0;
    for (uint64_t jj = slo + l; jj < shi; jj += 32) {
      const double pj = p[jj];
      nz |= pj != 0.0;
      long long k;
      if (usable && int_step(pj, inv_u, k)) K += k;
      else bad = 1;
    }
    for (int o = 16; o > 0; o >>= 1) {
      K += __shfl_down_sync(0xffffffffu, K, o);
      bad |= __shfl_down_sync(0xffffffffu, bad, o);
      nz |= __shfl_down_sync(0xffffffffu, nz, o);
    }
    if (l == 0) {
      const int cl = nz ? !bad : 2;
      shk[sc] = K;
      shb[sc] = cl;
      sub[(uint64_t)blockIdx.x * kSub + sc] = ChunkInfo{nz ? K : 0, e, cl};
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    int all_zero = 1, all_clean = 1;
    for (int i = 0; i < kSub; ++i) {
      t += shk[i];
      all_zero &= shb[i] == 2;
      all_clean &= shb[i] != 0;
    }
    info[blockIdx.x] = ChunkInfo{all_zero ? 0 : t, e, all_zero ? 2 : all_clean};
  }
}

__device__ __forceinline__ long long warp_incl_scan_ll(long long v) {
  const int l = threadIdx.x & 31;
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (l >= o) v += t;
  }
  return v;
}

// Phase C: one warp walks the chunks in order.  Chunk records are fetched 32
// at a time (lane j loads chunk c0 + j, then they are broadcast in order).  A
// chunk that cannot advance in one exact integer step is walked through its
// kSub sub-chunk records the same way; only a failing sub-chunk is replayed 32
// elements at a time (integer trick per 32, true serial adds when that fails).
// cum == nullptr: only the final sum is wanted (nothing is written per element).
__device__ __forceinline__ bool int_advance(double& A, long long K, int e, int clean) {
  const double kMinNormalScaled = 2.2250738585072014e-308 * 4503599627370496.0;
  if (clean == 2) return true;  // all addends zero: fl(A + 0) == A
  if (!clean || !(A >= kMinNormalScaled) || exp_of(A) != e) return false;
  const long long a = (long long)(A * pow2(52 - e));
  if (a + K >= 9007199254740991LL) return false;  // would leave the binade
  A = (double)(a + K) * pow2(e - 52);
  return true;
}

__device__ void replay_range(const double* __restrict__ p, uint64_t lo, uint64_t hi, double& A,
                             double* __restrict__ cum) {
  const int lane = threadIdx.x & 31;
  const double kMinNormalScaled = 2.2250738585072014e-308 * 4503599627370496.0;
  constexpr int kAhead = 8;  // 8 x 32 addends loaded per trip: one dependent load latency per 256
  for (uint64_t jb = lo; jb < hi; jb += 32 * kAhead) {
    double pv[kAhead];
#pragma unroll
    for (int q = 0; q < kAhead; ++q) {
      const uint64_t j = jb + 32 * q + lane;
      pv[q] = j < hi ? p[j] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kAhead; ++q) {
      const uint64_t j0 = jb + 32 * q;
      if (j0 >= hi) break;
      const uint64_t j = j0 + lane;
      const double pj = pv[q];
      bool done = false;
      if (A >= kMinNormalScaled) {
        const int eA = exp_of(A);
        const double u = pow2(eA - 52), inv_u = pow2(52 - eA);
        long long k = 0;
        const bool ok = int_step(pj, inv_u, k);
        if (__all_sync(0xffffffffu, ok)) {
          const long long incl = warp_incl_scan_ll(k);
          const long long Ksum = __shfl_sync(0xffffffffu, incl, 31);
          const long long a = (long long)(A * inv_u);
          if (a + Ksum < 9007199254740991LL) {
            if (cum && j < hi) cum[j] = (double)(a + incl) * u;
            A = (double)(a + Ksum) * u;
            done = true;
          }
        }
      }
      if (!done) {
        double acc = A;
        for (int t2 = 0; t2 < 32; ++t2) {
          const double pt = __shfl_sync(0xffffffffu, pj, t2);
          if (j0 + t2 < hi) {
            acc = __dadd_rn(acc, pt);
            if (cum && lane == t2) cum[j] = acc;
          }
        }
        A = acc;
      }
    }
  }
}

__global__ void k_sequential(const double* __restrict__ p, uint64_t n, uint64_t C, uint32_t nc,
                             const ChunkInfo* __restrict__ info, const ChunkInfo* __restrict__ sub,
                             double* __restrict__ start, unsigned char* __restrict__ fast,
                             double* __restrict__ sub_start, unsigned char* __restrict__ sub_fast,
                             double* __restrict__ cum, double* __restrict__ total, const double* __restrict__ carry) {
  const int lane = threadIdx.x & 31;
  const uint64_t Cs = C / kSub;
  double A = carry ? *carry : 0.0;  // sharded states: the previous shard's final running sum
  for (uint32_t c0 = 0; c0 < nc; c0 += 32) {
    ChunkInfo mine{0, 0, 0};
    if (c0 + lane < nc) mine = info[c0 + lane];
    double my_start = 0.0;
    unsigned char my_fast = 0;
    const uint32_t cn = min(32u, nc - c0);
    // All 32 chunks clean and guessed in the running value's binade: the
    // serial integer advances are one warp prefix sum (K >= 0, so the group
    // stays in the binade iff its total does) -- the same starts, exactly.
    // (All-zero chunks join any group: they leave the running value as is.)
    {
      const double kMinNormalScaled = 2.2250738585072014e-308 * 4503599627370496.0;
      const bool an = A >= kMinNormalScaled;
      const int eA = an ? exp_of(A) : 0;
      const bool zero = mine.clean == 2;
      const bool ok = (uint32_t)lane >= cn || zero || (mine.clean == 1 && an && mine.e == eA);
      if (__all_sync(0xffffffffu, ok)) {
        const long long k = ((uint32_t)lane < cn && !zero) ? mine.K : 0;
        const long long incl = warp_incl_scan_ll(k);
        const long long tot = __shfl_sync(0xffffffffu, incl, 31);
        if (!an) {  // only all-zero chunks (a clean one needs a normal running value)
          if (c0 + lane < nc) {
            start[c0 + lane] = A;
            fast[c0 + lane] = 1;
          }
          continue;
        }
        const long long a = (long long)(A * pow2(52 - eA));
        if (a + tot < 9007199254740991LL) {
          if (c0 + lane < nc) {
            start[c0 + lane] = (double)(a + incl - k) * pow2(eA - 52);
            fast[c0 + lane] = 1;
          }
          A = (double)(a + tot) * pow2(eA - 52);
          continue;
        }
      }
    }
    for (uint32_t t = 0; t < cn; ++t) {
      const uint32_t c = c0 + t;
      const long long ciK = __shfl_sync(0xffffffffu, mine.K, t);
      const int cie = __shfl_sync(0xffffffffu, mine.e, t);
      const int ciclean = __shfl_sync(0xffffffffu, mine.clean, t);
      const double A0 = A;
      if (int_advance(A, ciK, cie, ciclean)) {
        if (lane == (int)t) {
          my_start = A0;
          my_fast = 1;
        }
        continue;
      }
      // sub-chunk walk (records of this chunk: lanes 0..kSub-1)
      ChunkInfo sm{0, 0, 0};
      if (lane < kSub) sm = sub[(uint64_t)c * kSub + lane];
      double s_start = 0.0;
      unsigned char s_fast = 0;
      const uint64_t lo = (uint64_t)c * C, hi = min(n, lo + C);
      for (int sc = 0; sc < kSub; ++sc) {
        const long long sK = __shfl_sync(0xffffffffu, sm.K, sc);
        const int se = __shfl_sync(0xffffffffu, sm.e, sc);
        const int sclean = __shfl_sync(0xffffffffu, sm.clean, sc);
        const uint64_t slo = min(hi, lo + sc * Cs), shi = min(hi, slo + Cs);
        const double As = A;
        if (slo < shi && int_advance(A, sK, se, sclean)) {
          if (lane == sc) {
            s_start = As;
            s_fast = 1;
          }
          continue;
        }
        replay_range(p, slo, shi, A, cum);
      }
      if (cum && lane < kSub) {
        sub_start[(uint64_t)c * kSub + lane] = s_start;
        sub_fast[(uint64_t)c * kSub + lane] = s_fast;
      }
    }
    if (c0 + lane < nc) {
      start[c0 + lane] = my_start;
      fast[c0 + lane] = my_fast;
    }
  }
  if (lane == 0) *total = A;
}

// Phase D: expand the chunks (or the sub-chunks) the walk advanced in one
// integer step, in parallel (block per chunk): cum_j = (a + prefix_j) * u.
__device__ void expand_range(const double* __restrict__ p, uint64_t lo, uint64_t hi, int e, int clean, double start,
                             double* __restrict__ cum, long long* warp_tot) {
  if (clean == 2) {  // all addends zero: every partial sum is the start value
    for (uint64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) cum[j] = start;
    return;
  }
  const double u = pow2(e - 52), inv_u = pow2(52 - e);
  long long carry = (long long)(start * inv_u);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (uint64_t base = lo; base < hi; base += blockDim.x) {
    const uint64_t j = base + threadIdx.x;
    long long k = 0;
    if (j < hi) int_step(p[j], inv_u, k);
    const long long incl = warp_incl_scan_ll(k);
    if (l == 31) warp_tot[w] = incl;
    __syncthreads();
    long long before = 0, all = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      if (i < w) before += warp_tot[i];
      all += warp_tot[i];
    }
    if (j < hi) cum[j] = (double)(carry + before + incl) * u;
    carry += all;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) k_expand(const double* __restrict__ p, uint64_t n, uint64_t C,
                                                     const ChunkInfo* __restrict__ info,
                                                     const ChunkInfo* __restrict__ sub,
                                                     const double* __restrict__ start,
                                                     const unsigned char* __restrict__ fast,
                                                     const double* __restrict__ sub_start,
                                                     const unsigned char* __restrict__ sub_fast,
                                                     double* __restrict__ cum) {
  __shared__ long long warp_tot[kThreads / 32];
  const uint64_t lo = blockIdx.x * C, hi = min(n, lo + C);
  if (fast[blockIdx.x]) {
    expand_range(p, lo, hi, info[blockIdx.x].e, info[blockIdx.x].clean, start[blockIdx.x], cum, warp_tot);
    return;
  }
  const uint64_t Cs = C / kSub;
  for (int sc = 0; sc < kSub; ++sc) {
    const uint64_t k = (uint64_t)blockIdx.x * kSub + sc;
    if (!sub_fast[k]) continue;  // replayed by the walk (cum already written)
    const uint64_t slo = min(hi, lo + sc * Cs), shi = min(hi, slo + Cs);
    expand_range(p, slo, shi, sub[k].e, sub[k].clean, sub_start[k], cum, warp_tot);
  }
}

// Plain parallel scan for the fast (non-exact) mode: per-chunk serial sums in
// a block + the estimated chunk offsets.
__global__ void __launch_bounds__(kThreads) k_expand_approx(const double* __restrict__ p, uint64_t n, uint64_t C,
                                                            const double* __restrict__ E, double* __restrict__ cum) {
  __shared__ double warp_tot[kThreads / 32];
  double carry = E[blockIdx.x];
  const uint64_t lo = blockIdx.x * C, hi = min(n, lo + C);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (uint64_t base = lo; base < hi; base += blockDim.x) {
    const uint64_t j = base + threadIdx.x;
    double v = j < hi ? p[j] : 0.0;
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, v, o);
      if (l >= o) v += t;
    }
    if (l == 31) warp_tot[w] = v;
    __syncthreads();
    double before = 0, all = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      if (i < w) before += warp_tot[i];
      all += warp_tot[i];
    }
    if (j < hi) cum[j] = carry + before + v;
    carry += all;
    __syncthreads();
  }
}

// upper-bound binary search of u * total (statevector.hpp:554-565)
__global__ void __launch_bounds__(kThreads) k_search(const double* __restrict__ cum, uint64_t size,
                                                     const double* __restrict__ total_p, const double* __restrict__ u,
                                                     uint64_t shots, unsigned long long* __restrict__ out) {
  const double total = *total_p;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < shots; s += (uint64_t)gridDim.x * blockDim.x) {
    const double target = u[s] * total;
    uint64_t lo = 0, hi = size - 1;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (cum[mid] > target) hi = mid;
      else lo = mid + 1;
    }
    out[s] = lo;
  }
}

// Sharded sampling: this shard answers the shots whose target lies in
// [*lo, *hi) (lo = previous shards' total, null for the first shard; the last
// shard also takes targets >= *hi, the reference's size-1 fallback).  Global
// indices; other shots are left untouched.
__global__ void __launch_bounds__(kThreads) k_search_range(const double* __restrict__ cum, uint64_t size,
                                                           const double* __restrict__ total_p,
                                                           const double* __restrict__ lo_p,
                                                           const double* __restrict__ hi_p, int last,
                                                           const double* __restrict__ u, uint64_t shots,
                                                           uint64_t rank_base, unsigned long long* __restrict__ out) {
  const double total = *total_p, hi = *hi_p;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < shots; s += (uint64_t)gridDim.x * blockDim.x) {
    const double target = u[s] * total;
    if (lo_p && target < *lo_p) continue;
    if (!last && target >= hi) continue;
    uint64_t a = 0, b = size - 1;
    while (a < b) {
      const uint64_t mid = (a + b) / 2;
      if (cum[mid] > target) b = mid;
      else a = mid + 1;
    }
    out[s] = rank_base | a;
  }
}

// Reduced density matrix of qubits targets (msb first, local bit b <->
// targets[K-1-b]): rho[r][c] = sum_rest a[rest|r] conj(a[rest|c]).  One read
// pass; per-block partials (D*D complex) summed in block order afterwards.
// R = rows accumulated per launch (row0 .. row0+R-1): all D for K <= 2, one
// row at a time for K = 3 (keeps the accumulators in registers).
template <int K, int R>
__global__ void __launch_bounds__(kThreads) k_reduced_density(const double2* __restrict__ a, uint64_t groups, Slots sl,
                                                              TargetMasks tm, int row0, double2* __restrict__ partial) {
  constexpr int D = 1 << K;
  __shared__ double sh[kThreads / 32];
  double re[R * D], im[R * D];
#pragma unroll
  for (int i = 0; i < R * D; ++i) re[i] = im[i] = 0;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t base = deposit(g, sl);
    double2 v[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      uint64_t off = 0;
#pragma unroll
      for (int b = 0; b < K; ++b)
        if ((r >> b) & 1) off |= tm.m[b];
      v[r] = a[base | off];
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      double2 vr = v[rr];
      if constexpr (R < D) {  // rows picked at run time: select without dynamic indexing
#pragma unroll
        for (int c = 0; c < D; ++c)
          if (c == row0 + rr) vr = v[c];
      }
#pragma unroll
      for (int c = 0; c < D; ++c) {  // v_r * conj(v_c)
        re[rr * D + c] = fma(vr.x, v[c].x, fma(vr.y, v[c].y, re[rr * D + c]));
        im[rr * D + c] = fma(vr.y, v[c].x, fma(-vr.x, v[c].y, im[rr * D + c]));
      }
    }
  }
  for (int i = 0; i < R * D; ++i) {
    const double tr = block_sum(re[i], sh);
    const double ti = block_sum(im[i], sh);
    if (threadIdx.x == 0) partial[(uint64_t)blockIdx.x * D * D + row0 * D + i] = make_double2(tr, ti);
  }
}

__global__ void k_sum_partials(const double2* __restrict__ partial, int blocks, int width, double2* __restrict__ out) {
  const int i = threadIdx.x;
  if (i >= width) return;
  double re = 0, im = 0;
  for (int b = 0; b < blocks; ++b) {
    re += partial[(uint64_t)b * width + i].x;
    im += partial[(uint64_t)b * width + i].y;
  }
  out[i] = make_double2(re, im);
}

// ---------------------------------------------------------- shot batches
// B independent n-qubit states held as one (n + b)-qubit vector: shot s owns
// [s * 2^n, (s + 1) * 2^n).  Gates run through the ordinary planner (they
// never touch the shot bits); measurements and Kraus choices differ per shot.
__global__ void __launch_bounds__(kThreads) k_batch_basis(double2* __restrict__ a, uint64_t total, uint64_t lmask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = make_double2((i & lmask) == 0 ? 1.0 : 0.0, 0.0);
}

// p1[s] = sum over shot s of |a_i|^2 with bit set (one block per shot).
__global__ void __launch_bounds__(kThreads) k_batch_prob_one(const double2* __restrict__ a, uint32_t n, uint64_t bit,
                                                             uint64_t shots, double* __restrict__ p1) {
  __shared__ double sh[kThreads / 32];
  const uint64_t len = 1ull << n;
  for (uint64_t s = blockIdx.x; s < shots; s += gridDim.x) {
    const double2* b = a + s * len;
    double acc = 0;
    for (uint64_t i = threadIdx.x; i < len; i += blockDim.x)
      if (i & bit) acc += norm_ref(b[i]);
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) p1[s] = t;
  }
}

// Per shot: outcome = (u < 1 - p1) ? 0 : 1 (statevector.hpp:219-225); keep and
// rescale by 1/sqrt(prob) or zero.  A zero-probability pick raises *err.
__global__ void __launch_bounds__(kThreads) k_batch_collapse(double2* __restrict__ a, uint32_t n, uint64_t bit,
                                                             const double* __restrict__ p1, const double* __restrict__ u,
                                                             uint64_t total, signed char* __restrict__ out,
                                                             int* __restrict__ err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = i >> n;
    if (u[s] < 0.0) {  // shot not on this path (control flow): untouched
      if ((i & ((1ull << n) - 1)) == 0) out[s] = -1;
      continue;
    }
    const double q1 = p1[s], q0 = 1.0 - q1;
    const int o = (u[s] < q0) ? 0 : 1;
    const double prob = o ? q1 : q0;
    if ((i & ((1ull << n) - 1)) == 0) {
      out[s] = static_cast<signed char>(o);
      if (prob <= 0.0) *err = 1;
    }
    if (((i & bit) != 0) == (o == 1)) {
      const double inv = 1.0 / sqrt(prob);
      const double2 x = a[i];
      a[i] = make_double2(x.x * inv, x.y * inv);
    } else {
      a[i] = make_double2(0, 0);
    }
  }
}

// Reduced density matrix of K qubits per shot (one block per shot).
template <int K>
__global__ void __launch_bounds__(kThreads) k_batch_rdm(const double2* __restrict__ a, uint32_t n, Slots sl,
                                                        TargetMasks tm, uint64_t shots, double2* __restrict__ rdm) {
  constexpr int D = 1 << K;
  __shared__ double sh[kThreads / 32];
  const uint64_t groups = 1ull << (n - K);
  for (uint64_t s = blockIdx.x; s < shots; s += gridDim.x) {
    const double2* b = a + (s << n);
    double re[D * D], im[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) re[i] = im[i] = 0;
    for (uint64_t g = threadIdx.x; g < groups; g += blockDim.x) {
      const uint64_t base = deposit(g, sl);
      double2 v[D];
#pragma unroll
      for (int r = 0; r < D; ++r) {
        uint64_t off = 0;
#pragma unroll
        for (int t = 0; t < K; ++t)
          if ((r >> t) & 1) off |= tm.m[t];
        v[r] = b[base | off];
      }
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) {
          re[r * D + c] = fma(v[r].x, v[c].x, fma(v[r].y, v[c].y, re[r * D + c]));
          im[r * D + c] = fma(v[r].y, v[c].x, fma(-v[r].x, v[c].y, im[r * D + c]));
        }
    }
    for (int i = 0; i < D * D; ++i) {
      const double tr = block_sum(re[i], sh);
      const double ti = block_sum(im[i], sh);
      if (threadIdx.x == 0) rdm[s * D * D + i] = make_double2(tr, ti);
    }
  }
}

// Per shot: w_i = Tr(K_i rho K_i^dag), the reference's pick (u * total against
// the running sum, noise.hpp:290-305), scale = 1/sqrt(w_chosen).
template <int K>
__global__ void k_batch_choose(const double2* __restrict__ rdm, const double2* __restrict__ ops, int nops,
                               const double* __restrict__ u, uint64_t shots, int* __restrict__ chosen,
                               double* __restrict__ scale, int* __restrict__ err) {
  constexpr int D = 1 << K;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < shots; s += (uint64_t)gridDim.x * blockDim.x) {
    if (u[s] < 0.0) {  // shot not on this path (control flow)
      chosen[s] = -1;
      scale[s] = 1.0;
      continue;
    }
    const double2* rho = rdm + s * D * D;
    double w[16];
    double total = 0;
    for (int i = 0; i < nops; ++i) {
      const double2* k = ops + (uint64_t)i * D * D;
      double t = 0;
      for (int r = 0; r < D; ++r)
        for (int x = 0; x < D; ++x) {
          double cr = 0, ci = 0;  // (K rho)[r][x]
          for (int y = 0; y < D; ++y) {
            const double2 kk = k[r * D + y], rr = rho[y * D + x];
            cr = fma(kk.x, rr.x, fma(-kk.y, rr.y, cr));
            ci = fma(kk.x, rr.y, fma(kk.y, rr.x, ci));
          }
          const double2 kc = k[r * D + x];  // times conj(K[r][x])
          t = fma(cr, kc.x, fma(ci, kc.y, t));
        }
      w[i] = t > 0 ? t : 0.0;
      total += w[i];
    }
    const double target = u[s] * total;
    double acc = 0;
    int pick = nops - 1;
    for (int i = 0; i < nops; ++i) {
      acc += w[i];
      if (target < acc) {
        pick = i;
        break;
      }
    }
    chosen[s] = pick;
    if (w[pick] <= 0) {
      *err = 1;
      scale[s] = 0;
    } else {
      scale[s] = 1.0 / sqrt(w[pick]);
    }
  }
}

// a <- scale[s] * K_{chosen[s]} a on the K qubits, per shot.
template <int K>
__global__ void __launch_bounds__(kThreads) k_batch_apply(double2* __restrict__ a, uint32_t n, Slots sl, TargetMasks tm,
                                                          uint64_t shots, const double2* __restrict__ ops,
                                                          const int* __restrict__ chosen,
                                                          const double* __restrict__ scale) {
  constexpr int D = 1 << K;
  const uint64_t groups = 1ull << (n - K), work = groups * shots;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < work; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = w / groups, g = w % groups;
    if (chosen[s] < 0) continue;  // shot not on this path
    double2* b = a + (s << n);
    const uint64_t base = deposit(g, sl);
    const double2* k = ops + (uint64_t)chosen[s] * D * D;
    const double f = scale[s];
    uint64_t off[D];
    double2 v[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      off[r] = 0;
#pragma unroll
      for (int t = 0; t < K; ++t)
        if ((r >> t) & 1) off[r] |= tm.m[t];
      v[r] = b[base | off[r]];
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double re = 0, im = 0;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double2 kk = k[r * D + c];
        re = fma(kk.x, v[c].x, fma(-kk.y, v[c].y, re));
        im = fma(kk.x, v[c].y, fma(kk.y, v[c].x, im));
      }
      b[base | off[r]] = make_double2(re * f, im * f);
    }
  }
}

// dst[k] += f * (-1)^popc((k ^ x) & z) * src[k ^ x]: dst += f * P src for the
// Pauli string (X part x, Z part z; f carries the coefficient and i^#Y).
__global__ void __launch_bounds__(kThreads) k_pauli_axpy(double2* __restrict__ dst, const double2* __restrict__ src,
                                                         uint64_t size, uint64_t xmask, uint64_t zmask, double2 f) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < size; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = k ^ xmask;
    double2 v = src[j];
    if (__popcll(j & zmask) & 1) v = make_double2(-v.x, -v.y);
    const double2 d = dst[k];
    dst[k] = make_double2(fma(f.x, v.x, fma(-f.y, v.y, d.x)), fma(f.x, v.y, fma(f.y, v.x, d.y)));
  }
}

// ---------------------------------------------------------- expectation
// Pauli term whose X part crosses shards: sum_j conj(b[j ^ xl]) a[j] (-1)^popc(j & smask)
// with b the partner shard (rank ^ X's rank bits).
__global__ void __launch_bounds__(kThreads) k_pauli2(const double2* __restrict__ a, const double2* __restrict__ b,
                                                     uint64_t size, uint64_t xmask, uint64_t smask,
                                                     double2* __restrict__ partial) {
  __shared__ double sh[kThreads / 32];
  const uint64_t chunk = (size + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * chunk, hi = min(size, lo + chunk);
  double re = 0, im = 0;
  for (uint64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
    const double2 x = a[j];
    const double2 y = b[j ^ xmask];
    double pr = fma(y.x, x.x, y.y * x.y);
    double pi = fma(y.x, x.y, -y.y * x.x);
    if (__popcll(j & smask) & 1) {
      pr = -pr;
      pi = -pi;
    }
    re += pr;
    im += pi;
  }
  const double tr = block_sum(re, sh);
  const double ti = block_sum(im, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = make_double2(tr, ti);
}

// Pauli terms sharing one X mask in one read pass: v_j = conj(a[j^x]) a[j]
// once, accumulated under each term's Z sign.  partial[block][t].
constexpr int kPauliGroup = 8;
struct ZMasks {
  unsigned long long z[kPauliGroup];
};
__global__ void __launch_bounds__(kThreads) k_pauli_group(const double2* __restrict__ a, uint64_t size, uint64_t xmask,
                                                          ZMasks zm, int T, double2* __restrict__ partial) {
  __shared__ double sh[kThreads / 32];
  const uint64_t chunk = (size + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * chunk, hi = min(size, lo + chunk);
  double re[kPauliGroup], im[kPauliGroup];
#pragma unroll
  for (int t = 0; t < kPauliGroup; ++t) re[t] = im[t] = 0;
  auto add = [&](uint64_t j, double2 x, double2 y) {
    const double pr = fma(y.x, x.x, y.y * x.y);
    const double pi = fma(y.x, x.y, -y.y * x.x);
#pragma unroll
    for (int t = 0; t < kPauliGroup; ++t) {
      if (t >= T) break;
      const bool neg = __popcll(j & zm.z[t]) & 1;
      re[t] += neg ? -pr : pr;
      im[t] += neg ? -pi : pi;
    }
  };
  constexpr int U = 4;  // elements (pairs) in flight per thread
  if (!xmask) {
    uint64_t j = lo + threadIdx.x;
    for (; j + (U - 1) * blockDim.x < hi; j += U * blockDim.x) {
      double2 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = __ldcs(a + j + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < U; ++u) add(j + u * blockDim.x, x[u], x[u]);
    }
    for (; j < hi; j += blockDim.x) {
      const double2 x = __ldcs(a + j);
      add(j, x, x);
    }
  } else {
    // each pair (j, j ^ x) once, from the member whose top bit of x is clear:
    // c = conj(a[j ^ x]) a[j] contributes s_t(j) c + s_t(j ^ x) conj(c) --
    // every amplitude is read once
    const int hb = 63 - __clzll(xmask);
    const uint64_t half = size >> 1;
    const uint64_t pchunk = (half + gridDim.x - 1) / gridDim.x;
    const uint64_t plo = blockIdx.x * pchunk, phi = min(half, plo + pchunk);
    auto pair = [&](uint64_t j, double2 x, double2 y) {
      const double pr = fma(y.x, x.x, y.y * x.y);
      const double pi = fma(y.x, x.y, -y.y * x.x);
#pragma unroll
      for (int t = 0; t < kPauliGroup; ++t) {
        if (t >= T) break;
        const bool n1 = __popcll(j & zm.z[t]) & 1, n2 = __popcll((j ^ xmask) & zm.z[t]) & 1;
        re[t] += (n1 ? -pr : pr) + (n2 ? -pr : pr);
        im[t] += (n1 ? -pi : pi) - (n2 ? -pi : pi);
      }
    };
    auto jof = [&](uint64_t k) { return ((k >> hb) << (hb + 1)) | (k & ((1ull << hb) - 1)); };
    uint64_t k = plo + threadIdx.x;
    for (; k + (U - 1) * blockDim.x < phi; k += U * blockDim.x) {
      double2 x[U], y[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t j = jof(k + u * blockDim.x);
        x[u] = __ldcs(a + j);
        y[u] = __ldcs(a + (j ^ xmask));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) pair(jof(k + u * blockDim.x), x[u], y[u]);
    }
    for (; k < phi; k += blockDim.x) {
      const uint64_t j = jof(k);
      pair(j, __ldcs(a + j), __ldcs(a + (j ^ xmask)));
    }
  }
#pragma unroll
  for (int t = 0; t < kPauliGroup; ++t) {  // static indices: re/im stay in registers
    if (t >= T) break;
    const double tr = block_sum(re[t], sh);
    const double ti = block_sum(im[t], sh);
    if (threadIdx.x == 0) partial[(uint64_t)blockIdx.x * kPauliGroup + t] = make_double2(tr, ti);
  }
}

__global__ void k_finalize2_strided(const double2* __restrict__ partial, int count, int stride,
                                    double2* __restrict__ out) {
  __shared__ double sh[kThreads / 32];
  double re = 0, im = 0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    re += partial[(uint64_t)i * stride].x;
    im += partial[(uint64_t)i * stride].y;
  }
  const double tr = block_sum(re, sh);
  const double ti = block_sum(im, sh);
  if (threadIdx.x == 0) *out = make_double2(tr, ti);
}

__global__ void k_finalize2(const double2* __restrict__ partial, int count, double2* __restrict__ out) {
  __shared__ double sh[kThreads / 32];
  double re = 0, im = 0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    re += partial[i].x;
    im += partial[i].y;
  }
  const double tr = block_sum(re, sh);
  const double ti = block_sum(im, sh);
  if (threadIdx.x == 0) *out = make_double2(tr, ti);
}

inline double2 d2(cd c) { return make_double2(c.real(), c.imag()); }

}  // namespace

// ------------------------------------------------------------ launchers

void launch_op(State& s, const Op& op_in) {
  if (op_in.cneg) throw RuntimeError("negated control in a per-gate kernel (planner invariant)");
  DeviceGuard dg(s.device);
  const uint32_t n = s.local_qubits();
  Op local;
  const Op* opp = &op_in;
  if (s.g) {
    // Sharded: controls on rank bits are this shard's constants; targets are
    // local (the planner exchanges rank bits in first).
    local = op_in;
    local.controls.clear();
    for (auto c : op_in.controls) {
      if (c < n) local.controls.push_back(c);
      else if (!((s.rank >> (c - n)) & 1)) return;  // control is 0 on this shard
    }
    for (auto t : op_in.targets)
      if (t >= n) throw RuntimeError("per-gate kernel on a rank bit (planner invariant)");
    opp = &local;
  }
  const Op& op = *opp;
  switch (op.kind) {
    case OpKind::Identity: return;
    case OpKind::Mat1: {
      const Slots sl = make_slots(op.targets, op.controls);
      const uint64_t groups = 1ull << (n - sl.count);
      launch_mat1(s, groups, sl, 1ull << op.targets[0], d2(op.m[0]), d2(op.m[1]), d2(op.m[2]), d2(op.m[3]));
      QSB_LAUNCHED();
      return;
    }
    case OpKind::Diag: {
      const bool skip_zero = op.m[0] == cd(1.0);  // statevector.hpp:296
      std::vector<uint32_t> ctrls = op.controls;
      std::vector<uint32_t> targs;
      if (skip_zero) ctrls.push_back(op.targets[0]);
      else targs.push_back(op.targets[0]);
      const Slots sl = make_slots(targs, ctrls);
      const uint64_t groups = 1ull << (n - sl.count);
      if (!skip_zero && op.targets[0] == 0 && pair256_enabled())
        (sl.count <= 3 ? k_diag_q0<3> : k_diag_q0<0>)<<<grid_for(groups, s.device), kThreads, 0, s.stream>>>(
            s.amps, groups, sl, d2(op.m[0]), d2(op.m[1]));
      else
        (sl.count <= 3 ? k_diag<3> : k_diag<0>)<<<grid_for(groups, s.device), kThreads, 0, s.stream>>>(
            s.amps, groups, sl, 1ull << op.targets[0], d2(op.m[0]), d2(op.m[1]), skip_zero ? 1 : 0);
      QSB_LAUNCHED();
      return;
    }
    case OpKind::Flip: {
      const Slots sl = make_slots(op.targets, op.controls);
      const uint64_t groups = 1ull << (n - sl.count);
      // the 2x2 kernel with [[0,1],[1,0]] (exact: the products by 0 and 1 are
      // exact): measured 0.89 of HBM where the plain swap kernel reached 0.72
      const double2 z = make_double2(0, 0), o = make_double2(1, 0);
      launch_mat1(s, groups, sl, 1ull << op.targets[0], z, o, o, z);
      QSB_LAUNCHED();
      return;
    }
    case OpKind::Swap: {
      const Slots sl = make_slots(op.targets, op.controls);
      const uint64_t groups = 1ull << (n - sl.count);
      // as the 2x2 kernel on the pairs (.. a=1 b=0 ..) <-> (.. a=0 b=1 ..): i0
      // has bit a forced, i1 = i0 ^ (a | b); [[0,1],[1,0]] is exact (see Flip)
      Slots sw = sl;
      sw.force |= 1ull << op.targets[0];
      const double2 z = make_double2(0, 0), o = make_double2(1, 0);
      (sw.count <= 3 ? k_mat1<3> : k_mat1<0>)<<<grid_for(groups, s.device), kThreads, 0, s.stream>>>(
          s.amps, groups, sw, (1ull << op.targets[0]) | (1ull << op.targets[1]), z, o, o, z);
      QSB_LAUNCHED();
      return;
    }
    case OpKind::Dense: {
      const int K = static_cast<int>(op.targets.size());
      const Slots sl = make_slots(op.targets, op.controls);
      const uint64_t groups = 1ull << (n - sl.count);
      TargetMasks tm{};
      for (int b = 0; b < K; ++b) tm.m[b] = 1ull << op.targets[K - 1 - b];
      const size_t dim = size_t(1) << K;
      auto fill = [&](auto& M) {
        for (size_t i = 0; i < dim * dim; ++i) M.m[i] = d2(op.m[i]);
      };
      // thread per group (measured on B200, 28 qubits: 0.88-0.93 of HBM for
      // targets >= 3, 0.6-0.71 on the lowest qubits, where the lane-cooperative
      // form was slower still); QSB_DENSE_LANES=1 forces the lane-cooperative form
      const char* form_env = std::getenv("QSB_DENSE_FORM");  // g | lanes | s: force one form
      const std::string form = form_env ? form_env : "";
      bool per_group = !std::getenv("QSB_DENSE_LANES");
      // blocks wholly inside the low 12 qubits, without controls: staged chunks
      // (measured at 28 qubits: K = 3 on qubits 2,1,0: 0.85 of HBM staged vs 0.60
      // per group; K = 2 and 4 stay per group, 0.83 / 0.60 vs 0.78 / 0.51 staged)
      const bool staged = op.controls.empty() && n >= kStageLog && K == 3 &&
                          *std::max_element(op.targets.begin(), op.targets.end()) < static_cast<uint32_t>(kStageLog) &&
                          *std::min_element(op.targets.begin(), op.targets.end()) < 3 && !std::getenv("QSB_NO_DENSE_STAGE") &&
                          (form.empty() || form == "s");
      if (staged) {
        const uint64_t chunks = s.size >> kStageLog;
        const Slots sls = make_slots(op.targets, {});
        const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>(chunks, num_sms(s.device) * 3ull));
        const size_t smem = (size_t(1) << kStageLog) * sizeof(double2);
        auto launch = [&](auto kern, auto& M) {  // 64 KiB of dynamic smem needs the opt-in
          QSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
          kern<<<blocks, kThreads, smem, s.stream>>>(s.amps, chunks, sls, tm, M);
        };
        DenseM<3> M;
        fill(M);
        launch(k_dense_s<3>, M);
        QSB_LAUNCHED();
        return;
      }
      if (form == "g") per_group = true;
      if (form == "lanes") per_group = false;
      // qubit 0 among the targets: pairs as 256-bit accesses
      int pbit = -1;
      for (int b = 0; b < K; ++b)
        if (tm.m[b] == 1) pbit = b;
      if (!pair256_enabled()) pbit = -1;
      auto launch_g = [&](auto& M) {
        constexpr int KK = dense_k(static_cast<std::decay_t<decltype(M)>*>(nullptr));
        launch_dense_g<KK, KK - 1>(s, groups, sl, tm, M, pbit);
      };
      switch (K) {
        case 2: { DenseM<2> M; fill(M);
          if (per_group) launch_g(M);
          else k_dense<2><<<grid_for(groups << K, s.device), kThreads, 0, s.stream>>>(s.amps, groups, sl, tm, M);
          break; }
        case 3: { DenseM<3> M; fill(M);
          if (per_group) launch_g(M);
          else k_dense<3><<<grid_for(groups << K, s.device), kThreads, 0, s.stream>>>(s.amps, groups, sl, tm, M);
          break; }
        case 4: { static thread_local DenseM<4> M; fill(M);
          if (per_group) launch_g(M);
          else k_dense<4><<<grid_for(groups << K, s.device), kThreads, 0, s.stream>>>(s.amps, groups, sl, tm, M);
          break; }
        case 5: {
          static thread_local DenseM<5> M;  // 16 KiB: off the stack; the launch copies it
          fill(M);
          if (per_group) launch_g(M);
          else k_dense<5><<<grid_for(groups << K, s.device, 4), kThreads, 0, s.stream>>>(s.amps, groups, sl, tm, M);
          break;
        }
        default: {
          double2* dM = static_cast<double2*>(s.get_scratch(dim * dim * sizeof(double2)));
          std::vector<double2> hm(dim * dim);
          for (size_t i = 0; i < dim * dim; ++i) hm[i] = d2(op.m[i]);
          QSB_CUDA(cudaMemcpyAsync(dM, hm.data(), dim * dim * sizeof(double2), cudaMemcpyHostToDevice, s.stream));
          if (K == 6) {
            const size_t smem6 = (64 * 64 + 64 * (kThreads / 32)) * sizeof(double2);
            QSB_CUDA(cudaFuncSetAttribute(k_dense6, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem6)));
            const uint32_t b6 = static_cast<uint32_t>(
                std::min<uint64_t>((groups + kThreads / 32 - 1) / (kThreads / 32), num_sms(s.device) * 3ull));
            k_dense6<<<b6, kThreads, smem6, s.stream>>>(s.amps, groups, sl, tm, dM);
          } else {
            const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>(groups, num_sms(s.device) * 8ull));
            k_dense_wide<<<blocks, kThreads, dim * sizeof(double2), s.stream>>>(s.amps, groups, sl, tm, K, dM);
          }
          QSB_LAUNCHED();
          QSB_CUDA(cudaStreamSynchronize(s.stream));  // the host staging vector must outlive the copy
          return;
        }
      }
      QSB_LAUNCHED();
      return;
    }
  }
}

void swap_halves(State& a, State& b, uint32_t p) {
  DeviceGuard dg(a.device);
  const uint64_t count = a.size / 2;
  k_swap_halves<<<grid_for(count, a.device), kThreads, 0, a.stream>>>(a.amps, b.amps, count, p);
  QSB_LAUNCHED();
}

static BlockSpec block_spec(const uint32_t* lpos, uint32_t k, uint32_t d) {
  if (k > 16) throw ValidationError("too many exchange bits");
  BlockSpec b{};
  b.k = k;
  for (uint32_t i = 0; i < k; ++i) {
    b.sorted[i] = lpos[i];
    if ((d >> i) & 1) b.val |= 1ull << lpos[i];
  }
  std::sort(b.sorted, b.sorted + k);
  return b;
}

void pack_block(State& s, const uint32_t* lpos, uint32_t k, uint32_t d, uint64_t off, uint64_t cnt, double2* out) {
  DeviceGuard dg(s.device);
  k_pack_block<<<grid_for(cnt, s.device), kThreads, 0, s.stream>>>(s.amps, block_spec(lpos, k, d), off, cnt, out);
  QSB_LAUNCHED();
}

void scatter_exchange(State& s, double2* const* peers, const uint32_t* lpos, uint32_t k, uint32_t aval) {
  if (k > kMaxExchangeBits) throw ValidationError("peer exchange limited to 4 rank bits at once");
  PeerTable t{};
  for (uint32_t d = 0; d < (1u << k); ++d) t.p[d] = peers[d];
  ExchangeBits eb{};
  for (uint32_t i = 0; i < k; ++i) {
    eb.lpos[i] = lpos[i];
    eb.pmask |= 1ull << lpos[i];
    if ((aval >> i) & 1) eb.aval |= 1ull << lpos[i];
  }
  DeviceGuard dg(s.device);
  k_scatter_exchange<<<grid_for(s.size, s.device), kThreads, 0, s.stream>>>(s.amps, t, s.size, k, eb);
  QSB_LAUNCHED();
}

void unpack_block(State& s, const uint32_t* lpos, uint32_t k, uint32_t d, uint64_t off, uint64_t cnt,
                  const double2* in) {
  DeviceGuard dg(s.device);
  k_unpack_block<<<grid_for(cnt, s.device), kThreads, 0, s.stream>>>(s.amps, block_spec(lpos, k, d), off, cnt, in);
  QSB_LAUNCHED();
}

unsigned permute_qubits(State& s, const std::vector<uint32_t>& pos, double* red) {
  const uint32_t n = s.local_qubits();
  if (pos.size() != n) throw ValidationError("permutation size does not match the state");
  if (n < kPermTileBits) throw ValidationError("qubit permutation needs at least 10 qubits");
  std::vector<int> inv(n, -1);
  for (uint32_t q = 0; q < n; ++q) {
    if (pos[q] >= n || inv[pos[q]] >= 0) throw ValidationError("not a permutation");
    inv[pos[q]] = static_cast<int>(q);
  }
  // tile bits A: input 0..4, the inputs that land on output 0..4, then the lowest others
  std::vector<char> inA(n, 0);
  for (uint32_t q = 0; q < 5; ++q) inA[q] = inA[inv[q]] = 1;
  uint32_t cnt = 0;
  for (uint32_t q = 0; q < n; ++q) cnt += inA[q];
  for (uint32_t q = 0; q < n && cnt < kPermTileBits; ++q)
    if (!inA[q]) {
      inA[q] = 1;
      ++cnt;
    }
  std::vector<uint32_t> A, B;
  for (uint32_t q = 0; q < n; ++q) (inA[q] ? A : B).push_back(q);
  std::vector<uint32_t> C;  // output positions of the tile, ascending
  for (auto q : A) C.push_back(pos[q]);
  std::sort(C.begin(), C.end());
  PermSpec ps{};
  ps.nb = static_cast<uint32_t>(B.size());
  for (size_t k = 0; k < B.size(); ++k) {
    ps.bin[k] = static_cast<uint8_t>(B[k]);
    ps.bout[k] = static_cast<uint8_t>(pos[B[k]]);
  }
  for (uint32_t v = 0; v < 32; ++v) {
    for (uint32_t j = 0; j < 5; ++j) {
      if (!((v >> j) & 1)) continue;
      ps.in_lo[v] |= 1ull << A[j];
      ps.in_hi[v] |= 1ull << A[j + 5];
      ps.out_lo[v] |= 1ull << C[j];
      ps.out_hi[v] |= 1ull << C[j + 5];
      // output bit C[j] comes from input bit inv[C[j]] = A[k]
      const uint32_t klo = static_cast<uint32_t>(std::find(A.begin(), A.end(), static_cast<uint32_t>(inv[C[j]])) - A.begin());
      const uint32_t khi =
          static_cast<uint32_t>(std::find(A.begin(), A.end(), static_cast<uint32_t>(inv[C[j + 5]])) - A.begin());
      ps.e_lo[v] |= static_cast<uint16_t>(1u << klo);
      ps.e_hi[v] |= static_cast<uint16_t>(1u << khi);
    }
  }
  DeviceGuard dg(s.device);
  if (!s.alt && cudaMalloc(&s.alt, s.size * sizeof(double2)) != cudaSuccess) {
    cudaGetLastError();
    s.alt = nullptr;
    throw MemoryError("cannot allocate the second state buffer for a qubit permutation");
  }
  const uint64_t ntiles = s.size >> kPermTileBits;
  const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(ntiles, num_sms(s.device) * 8ull));
  k_permute<<<grid, kThreads, 0, s.stream>>>(s.amps, s.alt, ps, ntiles, red);
  QSB_LAUNCHED();
  std::swap(s.amps, s.alt);
  return grid;
}

void fill_basis(State& s, uint64_t index) {
  DeviceGuard dg(s.device);
  k_basis<<<grid_for(s.size, s.device), kThreads, 0, s.stream>>>(s.amps, s.size, index);
  QSB_LAUNCHED();
}

double sum_partials(State& s, double* part, unsigned count) {
  DeviceGuard dg(s.device);
  double* h = static_cast<double*>(s.get_pinned(sizeof(double)));
  if (count) {
    k_finalize<<<1, kThreads, 0, s.stream>>>(part, static_cast<int>(count), part + count);
    QSB_LAUNCHED();
    QSB_CUDA(cudaMemcpyAsync(h, part + count, sizeof(double), cudaMemcpyDeviceToHost, s.stream));
  } else {
    *h = 0.0;
  }
  QSB_CUDA(cudaStreamSynchronize(s.stream));
  return *h;
}

void zero_outside(State& s, uint64_t mask, uint64_t val) {
  DeviceGuard dg(s.device);
  k_zero_outside<<<grid_for(s.size, s.device), kThreads, 0, s.stream>>>(s.amps, s.size, s.rank_base, mask, val);
  QSB_LAUNCHED();
}

namespace {
double reduce_mode(State& s, int mode, uint32_t q) {
  DeviceGuard dg(s.device);
  double* part = static_cast<double*>(s.get_scratch((kRedBlocks + 1) * sizeof(double)));
  const uint64_t items = mode == 1 ? s.size / 2 : s.size;
  k_reduce<<<kRedBlocks, kThreads, 0, s.stream>>>(s.amps, items, mode, 1ull << q, s.rank_base, part);
  QSB_LAUNCHED();
  k_finalize<<<1, kThreads, 0, s.stream>>>(part, kRedBlocks, part + kRedBlocks);
  QSB_LAUNCHED();
  double* h = static_cast<double*>(s.get_pinned(sizeof(double)));
  QSB_CUDA(cudaMemcpyAsync(h, part + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaStreamSynchronize(s.stream));
  return *h;
}
}  // namespace

double reduce_norm2(State& s) { return reduce_mode(s, 0, 0); }
double reduce_prob_one(State& s, uint32_t q) { return reduce_mode(s, 1, q); }
double reduce_checksum(State& s) { return reduce_mode(s, 2, 0); }

void marginal_probs(State& s, const uint32_t* qubits, uint32_t m, double* host_out) {
  DeviceGuard dg(s.device);
  std::vector<uint32_t> qs(qubits, qubits + m);
  const Slots sl = make_slots(qs, {});
  const uint64_t per_bin = 1ull << (s.local_qubits() - m);
  const uint64_t bins = 1ull << m;
  const size_t out_bytes = bins * sizeof(double);
  uint32_t kh = 0, k8 = 0;
  for (uint32_t b = 0; b < m; ++b) {
    kh += qubits[b] >= 5;
    k8 += qubits[b] >= 8;
  }
  static_assert(kThreads == 8 * 32, "k_marginal_runs maps one (j, lane) entry per thread");
  if (m <= 12 && s.local_qubits() >= 8 + k8 && !std::getenv("QSB_MARGINAL_LANES")) {
    MarginalRuns mm{};
    std::vector<std::pair<uint32_t, uint32_t>> hq;  // (qubit, result bit)
    for (int b = 0; b < 5; ++b) mm.rl[b] = -1;
    for (int b = 0; b < 3; ++b) mm.rm[b] = -1;
    for (uint32_t b = 0; b < m; ++b) {
      if (qubits[b] >= 8) hq.push_back({qubits[b], b});
      else if (qubits[b] >= 5) mm.rm[qubits[b] - 5] = static_cast<int>(b);
      else mm.rl[qubits[b]] = static_cast<int>(b);
    }
    std::sort(hq.begin(), hq.end());
    mm.kh = k8;
    std::vector<uint32_t> rel;
    for (uint32_t j = 0; j < k8; ++j) {
      mm.qh[j] = hq[j].first;
      mm.rh[j] = hq[j].second;
      rel.push_back(hq[j].first - 8);
    }
    for (int b = 0; b < 5; ++b)
      if (mm.rl[b] < 0) mm.lane_free |= 1u << b;
    for (int b = 0; b < 3; ++b)
      if (mm.rm[b] < 0) mm.mid_free |= 1u << b;
    const Slots slh = make_slots(rel, {});
    const uint64_t per_hi = 1ull << (s.local_qubits() - 8 - k8);
    const uint64_t ybins = 1ull << k8;
    const uint32_t per = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(kRedBlocks / ybins + 1, per_hi)));
    char* scr = static_cast<char*>(s.get_scratch(bins * per * sizeof(double) + out_bytes));
    double* part = reinterpret_cast<double*>(scr);
    double* dout = part + bins * per;
    k_marginal_runs<<<dim3(per, static_cast<uint32_t>(ybins)), kThreads, 0, s.stream>>>(s.amps, per_hi, slh, mm, part);
    QSB_LAUNCHED();
    k_marginal_finalize<<<static_cast<uint32_t>((bins + 255) / 256), 256, 0, s.stream>>>(part, per,
                                                                                         static_cast<uint32_t>(bins), dout);
    QSB_LAUNCHED();
    QSB_CUDA(cudaMemcpyAsync(host_out, dout, out_bytes, cudaMemcpyDeviceToHost, s.stream));
  } else if (m <= 12 && s.local_qubits() >= 5 + kh) {
    MarginalMap mm{};
    std::vector<std::pair<uint32_t, uint32_t>> hq;  // (qubit, result bit)
    for (int b = 0; b < 5; ++b) mm.rl[b] = -1;
    for (uint32_t b = 0; b < m; ++b) {
      if (qubits[b] >= 5) hq.push_back({qubits[b], b});
      else mm.rl[qubits[b]] = static_cast<int>(b);
    }
    std::sort(hq.begin(), hq.end());
    mm.kh = kh;
    std::vector<uint32_t> rel;
    for (uint32_t j = 0; j < kh; ++j) {
      mm.qh[j] = hq[j].first;
      mm.rh[j] = hq[j].second;
      rel.push_back(hq[j].first - 5);
    }
    for (int b = 0; b < 5; ++b)
      if (mm.rl[b] < 0) mm.lane_free |= 1u << b;
    const Slots slh = make_slots(rel, {});
    const uint64_t per_hi = 1ull << (s.local_qubits() - 5 - kh);
    const uint64_t ybins = 1ull << kh;
    const uint32_t per = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(kRedBlocks / ybins + 1, per_hi)));
    char* scr = static_cast<char*>(s.get_scratch(bins * per * sizeof(double) + out_bytes));
    double* part = reinterpret_cast<double*>(scr);
    double* dout = part + bins * per;
    k_marginal_lanes<<<dim3(per, static_cast<uint32_t>(ybins)), kThreads, 0, s.stream>>>(s.amps, per_hi, slh, mm, part);
    QSB_LAUNCHED();
    k_marginal_finalize<<<static_cast<uint32_t>((bins + 255) / 256), 256, 0, s.stream>>>(part, per,
                                                                                         static_cast<uint32_t>(bins), dout);
    QSB_LAUNCHED();
    QSB_CUDA(cudaMemcpyAsync(host_out, dout, out_bytes, cudaMemcpyDeviceToHost, s.stream));
  } else if (m <= 12) {
    const uint32_t per = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(kRedBlocks / bins + 1, per_bin)));
    char* scr = static_cast<char*>(s.get_scratch(256 + m * 4 + bins * per * sizeof(double) + out_bytes));
    uint32_t* dq = reinterpret_cast<uint32_t*>(scr);
    double* part = reinterpret_cast<double*>(scr + 256);
    double* dout = part + bins * per;
    QSB_CUDA(cudaMemcpyAsync(dq, qubits, m * 4, cudaMemcpyHostToDevice, s.stream));
    k_marginal<<<dim3(per, static_cast<uint32_t>(bins)), kThreads, 0, s.stream>>>(s.amps, per_bin, sl, dq, m, part);
    QSB_LAUNCHED();
    k_marginal_finalize<<<static_cast<uint32_t>((bins + 255) / 256), 256, 0, s.stream>>>(part, per,
                                                                                         static_cast<uint32_t>(bins), dout);
    QSB_LAUNCHED();
    QSB_CUDA(cudaMemcpyAsync(host_out, dout, out_bytes, cudaMemcpyDeviceToHost, s.stream));
  } else {
    char* scr = static_cast<char*>(s.get_scratch(256 + out_bytes));
    uint32_t* dq = reinterpret_cast<uint32_t*>(scr);
    double* dout = reinterpret_cast<double*>(scr + 256);
    QSB_CUDA(cudaMemcpyAsync(dq, qubits, m * 4, cudaMemcpyHostToDevice, s.stream));
    k_marginal_wide<<<grid_for(bins, s.device), kThreads, 0, s.stream>>>(s.amps, per_bin, sl, dq, m, dout);
    QSB_LAUNCHED();
    QSB_CUDA(cudaMemcpyAsync(host_out, dout, out_bytes, cudaMemcpyDeviceToHost, s.stream));
  }
  QSB_CUDA(cudaStreamSynchronize(s.stream));
}

void full_probs(State& s, double* host_out, uint64_t offset, uint64_t count) {
  DeviceGuard dg(s.device);
  const uint64_t step = 1ull << 26;  // bounded scratch
  for (uint64_t done = 0; done < count; done += step) {
    const uint64_t c = std::min(step, count - done);
    double* dp = static_cast<double*>(s.get_scratch(c * sizeof(double)));
    k_probs<<<grid_for(c, s.device), kThreads, 0, s.stream>>>(s.amps, offset + done, c, dp);
    QSB_LAUNCHED();
    QSB_CUDA(cudaMemcpyAsync(host_out + done, dp, c * sizeof(double), cudaMemcpyDeviceToHost, s.stream));
    QSB_CUDA(cudaStreamSynchronize(s.stream));
  }
}

void collapse(State& s, uint32_t q, int outcome, double inv) {
  DeviceGuard dg(s.device);
  k_collapse<<<grid_for(s.size, s.device), kThreads, 0, s.stream>>>(s.amps, s.size, 1ull << q, outcome, inv);
  QSB_LAUNCHED();
}

void scale(State& s, double re, double im) {
  DeviceGuard dg(s.device);
  k_scale<<<grid_for(s.size, s.device), kThreads, 0, s.stream>>>(s.amps, s.size, make_double2(re, im));
  QSB_LAUNCHED();
}

namespace {
struct SamplerBuffers {
  double* p;
  double* cum;
  double* S;
  double* E;
  ChunkInfo* info;
  ChunkInfo* sub;          // kSub records per chunk
  double* start;
  unsigned char* fast;
  double* sub_start;
  unsigned char* sub_fast;
  double* total;
  uint64_t C;
  uint32_t nc;
};

SamplerBuffers sampler_buffers(State& s, uint64_t extra_bytes, char** extra) {
  SamplerBuffers b{};
  const uint64_t N = s.size;
  b.C = std::max<uint64_t>(1024, N / 16384);
  b.nc = static_cast<uint32_t>((N + b.C - 1) / b.C);
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  const uint64_t bytes = al(N * 8) * 2 + al(b.nc * 8) * 3 + al(b.nc * sizeof(ChunkInfo)) + al(b.nc) + 256 +
                         al(b.nc * kSub * sizeof(ChunkInfo)) + al(b.nc * kSub * 8) + al(b.nc * kSub) + al(extra_bytes);
  char* base = static_cast<char*>(s.get_scratch(bytes));
  char* q = base;
  auto take = [&](uint64_t sz) {
    char* r = q;
    q += al(sz);
    return r;
  };
  b.p = reinterpret_cast<double*>(take(N * 8));
  b.cum = reinterpret_cast<double*>(take(N * 8));
  b.S = reinterpret_cast<double*>(take(b.nc * 8));
  b.E = reinterpret_cast<double*>(take(b.nc * 8));
  b.start = reinterpret_cast<double*>(take(b.nc * 8));
  b.info = reinterpret_cast<ChunkInfo*>(take(b.nc * sizeof(ChunkInfo)));
  b.fast = reinterpret_cast<unsigned char*>(take(b.nc));
  b.sub = reinterpret_cast<ChunkInfo*>(take(b.nc * kSub * sizeof(ChunkInfo)));
  b.sub_start = reinterpret_cast<double*>(take(b.nc * kSub * 8));
  b.sub_fast = reinterpret_cast<unsigned char*>(take(b.nc * kSub));
  b.total = reinterpret_cast<double*>(take(256));
  *extra = take(extra_bytes);
  return b;
}

void build_cumulative(State& s, SamplerBuffers& b, bool exact, const double* carry = nullptr) {
  const uint64_t N = s.size;
  k_probs<<<grid_for(N, s.device), kThreads, 0, s.stream>>>(s.amps, 0, N, b.p);
  QSB_LAUNCHED();
  k_chunk_sum<<<b.nc, kThreads, 0, s.stream>>>(b.p, N, b.C, b.S);
  QSB_LAUNCHED();
  k_scan_estimate<<<1, 32, 0, s.stream>>>(b.S, b.nc, b.E, carry);
  QSB_LAUNCHED();
  if (exact) {
    k_chunk_ints<<<b.nc, kThreads, 0, s.stream>>>(b.p, N, b.C, b.E, b.info, b.sub);
    QSB_LAUNCHED();
    k_sequential<<<1, 32, 0, s.stream>>>(b.p, N, b.C, b.nc, b.info, b.sub, b.start, b.fast, b.sub_start, b.sub_fast,
                                         b.cum, b.total, carry);
    QSB_LAUNCHED();
    k_expand<<<b.nc, kThreads, 0, s.stream>>>(b.p, N, b.C, b.info, b.sub, b.start, b.fast, b.sub_start, b.sub_fast,
                                              b.cum);
    QSB_LAUNCHED();
  } else {
    k_expand_approx<<<b.nc, kThreads, 0, s.stream>>>(b.p, N, b.C, b.E, b.cum);
    QSB_LAUNCHED();
    QSB_CUDA(cudaMemcpyAsync(b.total, b.cum + (N - 1), sizeof(double), cudaMemcpyDeviceToDevice, s.stream));
  }
}
}  // namespace

ShardCum shard_cumulative(State& s, bool exact, const double* carry_dev, uint64_t shots, double** u_dev,
                          unsigned long long** out_dev) {
  DeviceGuard dg(s.device);
  char* extra;
  SamplerBuffers b = sampler_buffers(s, shots * 16, &extra);
  build_cumulative(s, b, exact, carry_dev);
  if (u_dev) *u_dev = reinterpret_cast<double*>(extra);
  if (out_dev) *out_dev = reinterpret_cast<unsigned long long*>(extra + shots * 8);
  return ShardCum{b.cum, b.total};
}

void search_range(State& s, const ShardCum& c, const double* total_dev, const double* lo_dev, bool last,
                  const double* u_dev, uint64_t shots, unsigned long long* out_dev) {
  DeviceGuard dg(s.device);
  if (!shots) return;
  k_search_range<<<grid_for(shots, s.device), kThreads, 0, s.stream>>>(c.cum, s.size, total_dev, lo_dev, c.total, last,
                                                                       u_dev, shots, s.rank_base, out_dev);
  QSB_LAUNCHED();
}

void pauli_cross(State& s, const double2* a, const double2* partner, uint64_t size, uint64_t xl, uint64_t smask_local,
                 double* out2) {
  DeviceGuard dg(s.device);
  double2* part = static_cast<double2*>(s.get_scratch((kRedBlocks + 1) * sizeof(double2)));
  k_pauli2<<<kRedBlocks, kThreads, 0, s.stream>>>(a, partner, size, xl, smask_local, part);
  QSB_LAUNCHED();
  k_finalize2<<<1, kThreads, 0, s.stream>>>(part, kRedBlocks, part + kRedBlocks);
  QSB_LAUNCHED();
  double2 h;
  QSB_CUDA(cudaMemcpyAsync(&h, part + kRedBlocks, sizeof(double2), cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaStreamSynchronize(s.stream));
  out2[0] = h.x;
  out2[1] = h.y;
}

// probability_checksum rounded exactly as the reference's serial loop rounds
// it (bench.hpp:141-148, as g++ -O3 compiles it: t_i = fl(fl(|a_i|^2) * (i+1)),
// then sum += t_i in index order): the serial-equivalent scan of the t_i.
__global__ void __launch_bounds__(kThreads) k_checksum_terms(const double2* __restrict__ a, uint64_t count,
                                                             uint64_t base, double* __restrict__ t) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    t[i] = __dmul_rn(norm_ref(a[i]), (double)(base + i + 1));
}

double serial_checksum(State& s) {
  DeviceGuard dg(s.device);
  char* extra;
  SamplerBuffers b = sampler_buffers(s, 0, &extra);
  const uint64_t N = s.size;
  k_checksum_terms<<<grid_for(N, s.device), kThreads, 0, s.stream>>>(s.amps, N, s.rank_base, b.p);
  QSB_LAUNCHED();
  k_chunk_sum<<<b.nc, kThreads, 0, s.stream>>>(b.p, N, b.C, b.S);
  QSB_LAUNCHED();
  k_scan_estimate<<<1, 32, 0, s.stream>>>(b.S, b.nc, b.E, nullptr);
  QSB_LAUNCHED();
  k_chunk_ints<<<b.nc, kThreads, 0, s.stream>>>(b.p, N, b.C, b.E, b.info, b.sub);
  QSB_LAUNCHED();
  k_sequential<<<1, 32, 0, s.stream>>>(b.p, N, b.C, b.nc, b.info, b.sub, b.start, b.fast, b.sub_start, b.sub_fast,
                                       nullptr, b.total, nullptr);
  QSB_LAUNCHED();
  double* h = static_cast<double*>(s.get_pinned(8));
  QSB_CUDA(cudaMemcpyAsync(h, b.total, 8, cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaStreamSynchronize(s.stream));
  return *h;
}

// partial_amplitude's branch sum (pathsum.hpp:453-456), one block per target:
// sum over b < 2^c of A[b 2^na + ta] * B[b 2^nb + tb] -- fixed per-thread
// ranges + fixed-order block tree (deterministic).
__global__ void __launch_bounds__(kThreads) k_branch_dot(const double2* __restrict__ A, const double2* __restrict__ B,
                                                         uint32_t na, uint32_t nb, uint64_t branches,
                                                         const unsigned long long* __restrict__ ta,
                                                         const unsigned long long* __restrict__ tb,
                                                         double2* __restrict__ out) {
  __shared__ double sh[kThreads / 32];
  const unsigned long long a0 = ta[blockIdx.x], b0 = tb[blockIdx.x];
  double re = 0, im = 0;
  for (uint64_t b = threadIdx.x; b < branches; b += blockDim.x) {
    const double2 x = A[(b << na) | a0], y = B[(b << nb) | b0];
    re += x.x * y.x - x.y * y.y;
    im += x.x * y.y + x.y * y.x;
  }
  const double tr = block_sum(re, sh);
  const double ti = block_sum(im, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = make_double2(tr, ti);
}

void branch_dot(State& a, State& b, uint32_t na, uint32_t nb, uint32_t c, const std::vector<uint64_t>& ta,
                const std::vector<uint64_t>& tb, std::vector<cd>& out) {
  DeviceGuard dg(a.device);
  const size_t T = ta.size();
  out.assign(T, cd(0));
  if (!T) return;
  QSB_CUDA(cudaStreamSynchronize(b.stream));
  char* scr = static_cast<char*>(a.get_scratch(T * (16 + 16)));
  unsigned long long* dta = reinterpret_cast<unsigned long long*>(scr);
  unsigned long long* dtb = dta + T;
  double2* dout = reinterpret_cast<double2*>(dtb + T);
  QSB_CUDA(cudaMemcpyAsync(dta, ta.data(), T * 8, cudaMemcpyHostToDevice, a.stream));
  QSB_CUDA(cudaMemcpyAsync(dtb, tb.data(), T * 8, cudaMemcpyHostToDevice, a.stream));
  for (size_t t0 = 0; t0 < T; t0 += 65535) {
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>(65535, T - t0));
    k_branch_dot<<<blocks, kThreads, 0, a.stream>>>(a.amps, b.amps, na, nb, 1ull << c, dta + t0, dtb + t0, dout + t0);
    QSB_LAUNCHED();
  }
  std::vector<double2> h(T);
  QSB_CUDA(cudaMemcpyAsync(h.data(), dout, T * 16, cudaMemcpyDeviceToHost, a.stream));
  QSB_CUDA(cudaStreamSynchronize(a.stream));
  for (size_t t = 0; t < T; ++t) out[t] = cd(h[t].x, h[t].y);
}

double exact_cumulative(State& s, double* d_probs, double* d_cum) {
  DeviceGuard dg(s.device);
  char* extra;
  SamplerBuffers b = sampler_buffers(s, 0, &extra);
  build_cumulative(s, b, true);
  QSB_CUDA(cudaMemcpyAsync(d_cum, b.cum, s.size * 8, cudaMemcpyDeviceToDevice, s.stream));
  if (d_probs) QSB_CUDA(cudaMemcpyAsync(d_probs, b.p, s.size * 8, cudaMemcpyDeviceToDevice, s.stream));
  double* h = static_cast<double*>(s.get_pinned(8));
  QSB_CUDA(cudaMemcpyAsync(h, b.total, 8, cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaStreamSynchronize(s.stream));
  return *h;
}

// The cumulative array is built asynchronously while the host fills the
// uniforms (gen(dst, count): the next `count` draws of the Rng stream, or of
// the caller's array) into pinned staging; then per batch of <= 2^24 shots one
// H2D copy, the search and one D2H copy (bounded pinned / device staging).
void sample_gen(State& s, uint64_t shots, bool exact, uint64_t* out_host,
                const std::function<void(double*, uint64_t)>& gen) {
  DeviceGuard dg(s.device);
  if (shots == 0) return;
  const uint64_t B = std::min<uint64_t>(shots, 1ull << 24);
  double* hu = static_cast<double*>(s.get_pinned(B * 16));  // before any async work (may reallocate)
  uint64_t* hout = reinterpret_cast<uint64_t*>(hu + B);
  char* extra;
  SamplerBuffers b = sampler_buffers(s, B * 16, &extra);
  double* du = reinterpret_cast<double*>(extra);
  unsigned long long* dout = reinterpret_cast<unsigned long long*>(extra + B * 8);
  build_cumulative(s, b, exact);
  for (uint64_t done = 0; done < shots; done += B) {
    const uint64_t cnt = std::min(B, shots - done);
    gen(hu, cnt);  // the first batch overlaps the cumulative build on the GPU
    QSB_CUDA(cudaMemcpyAsync(du, hu, cnt * 8, cudaMemcpyHostToDevice, s.stream));
    k_search<<<grid_for(cnt, s.device), kThreads, 0, s.stream>>>(b.cum, s.size, b.total, du, cnt, dout);
    QSB_LAUNCHED();
    QSB_CUDA(cudaMemcpyAsync(hout, dout, cnt * 8, cudaMemcpyDeviceToHost, s.stream));
    QSB_CUDA(cudaStreamSynchronize(s.stream));
    std::memcpy(out_host + done, hout, cnt * 8);
  }
}

void sample(State& s, const double* uniforms_host, uint64_t shots, bool exact, uint64_t* out_host) {
  uint64_t next = 0;
  sample_gen(s, shots, exact, out_host, [&](double* hu, uint64_t cnt) {
    std::memcpy(hu, uniforms_host + next, cnt * 8);
    next += cnt;
  });
}

void reduced_density(State& s, const uint32_t* targets, uint32_t k, double* out) {
  if (k < 1 || k > 3) throw ValidationError("reduced density matrix supports 1 to 3 qubits");
  std::vector<uint32_t> tg(targets, targets + k);
  for (auto q : tg)
    if (q >= s.local_qubits()) throw ValidationError("reduced density: qubit out of range");
  const Slots sl = make_slots(tg, {});
  if (sl.count != k) throw ValidationError("reduced density: repeated qubit");
  TargetMasks tm{};
  for (uint32_t b = 0; b < k; ++b) tm.m[b] = 1ull << tg[k - 1 - b];
  const uint64_t groups = 1ull << (s.local_qubits() - k);
  const int width = 1 << (2 * k);
  const int blocks = static_cast<int>(std::min<uint64_t>(kRedBlocks / 4, std::max<uint64_t>(1, groups / kThreads)));
  DeviceGuard dg(s.device);
  double2* part = static_cast<double2*>(s.get_scratch((static_cast<size_t>(blocks) + 1) * width * sizeof(double2)));
  double2* res = part + static_cast<size_t>(blocks) * width;
  switch (k) {
    case 1:
      k_reduced_density<1, 2><<<blocks, kThreads, 0, s.stream>>>(s.amps, groups, sl, tm, 0, part);
      QSB_LAUNCHED();
      break;
    case 2:
      k_reduced_density<2, 4><<<blocks, kThreads, 0, s.stream>>>(s.amps, groups, sl, tm, 0, part);
      QSB_LAUNCHED();
      break;
    default:
      for (int r = 0; r < 8; ++r) {
        k_reduced_density<3, 1><<<blocks, kThreads, 0, s.stream>>>(s.amps, groups, sl, tm, r, part);
        QSB_LAUNCHED();
      }
      break;
  }
  k_sum_partials<<<1, 64, 0, s.stream>>>(part, blocks, width, res);
  QSB_LAUNCHED();
  QSB_CUDA(cudaMemcpyAsync(out, res, width * sizeof(double2), cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaStreamSynchronize(s.stream));
}

void batch_reset(State& s, uint32_t n) {
  if (n > s.local_qubits()) throw ValidationError("batch: shot size exceeds the state");
  DeviceGuard dg(s.device);
  k_batch_basis<<<grid_for(s.size, s.device), kThreads, 0, s.stream>>>(s.amps, s.size, (1ull << n) - 1);
  QSB_LAUNCHED();
}

void batch_measure(State& s, uint32_t n, uint32_t q, const double* u_host, uint64_t shots, signed char* out_host) {
  if (n > s.local_qubits() || q >= n) throw ValidationError("batch measure: qubit out of range");
  if (shots > (s.size >> n)) throw ValidationError("batch measure: more shots than the batch holds");
  if (!shots) return;
  DeviceGuard dg(s.device);
  char* scr = static_cast<char*>(s.get_scratch(shots * 17 + 512));
  double* p1 = reinterpret_cast<double*>(scr);
  double* u = p1 + shots;
  int* err = reinterpret_cast<int*>(u + shots);
  signed char* out = reinterpret_cast<signed char*>(err + 4);
  QSB_CUDA(cudaMemcpyAsync(u, u_host, shots * 8, cudaMemcpyHostToDevice, s.stream));
  QSB_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s.stream));
  const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>(shots, num_sms(s.device) * 8ull));
  k_batch_prob_one<<<blocks, kThreads, 0, s.stream>>>(s.amps, n, 1ull << q, shots, p1);
  QSB_LAUNCHED();
  k_batch_collapse<<<grid_for(shots << n, s.device), kThreads, 0, s.stream>>>(s.amps, n, 1ull << q, p1, u, shots << n,
                                                                              out, err);
  QSB_LAUNCHED();
  int h_err = 0;
  QSB_CUDA(cudaMemcpyAsync(out_host, out, shots, cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaStreamSynchronize(s.stream));
  if (h_err) throw RuntimeError("collapse onto a zero-probability outcome");
}

void batch_apply(State& s, uint32_t n, const uint32_t* qubits, uint32_t k, const double* m_host,
                 const signed char* mask_host, uint64_t shots) {
  if (k < 1 || k > 3) throw ValidationError("batch apply: 1 to 3 qubits");
  if (n > s.local_qubits() || shots > (s.size >> n)) throw ValidationError("batch apply: bad batch shape");
  std::vector<uint32_t> tg(qubits, qubits + k);
  for (auto q : tg)
    if (q >= n) throw ValidationError("batch apply: qubit out of range");
  const Slots sl = make_slots(tg, {});
  if (sl.count != k) throw ValidationError("batch apply: repeated qubit");
  if (!shots) return;
  TargetMasks tm{};
  for (uint32_t b = 0; b < k; ++b) tm.m[b] = 1ull << tg[k - 1 - b];
  const int D = 1 << k;
  DeviceGuard dg(s.device);
  const size_t mbytes = static_cast<size_t>(D) * D * sizeof(double2);
  char* scr = static_cast<char*>(s.get_scratch(mbytes + shots * (4 + 8) + 256));
  double2* m = reinterpret_cast<double2*>(scr);
  double* scale = reinterpret_cast<double*>(scr + mbytes);
  int* chosen = reinterpret_cast<int*>(scale + shots);
  std::vector<int> ch(shots);
  std::vector<double> one(shots, 1.0);
  for (uint64_t i = 0; i < shots; ++i) ch[i] = mask_host[i] ? 0 : -1;
  QSB_CUDA(cudaMemcpyAsync(m, m_host, mbytes, cudaMemcpyHostToDevice, s.stream));
  QSB_CUDA(cudaMemcpyAsync(scale, one.data(), shots * 8, cudaMemcpyHostToDevice, s.stream));
  QSB_CUDA(cudaMemcpyAsync(chosen, ch.data(), shots * 4, cudaMemcpyHostToDevice, s.stream));
  switch (k) {
    case 1: k_batch_apply<1><<<grid_for(shots << (n - 1), s.device), kThreads, 0, s.stream>>>(s.amps, n, sl, tm, shots, m, chosen, scale); break;
    case 2: k_batch_apply<2><<<grid_for(shots << (n - 2), s.device), kThreads, 0, s.stream>>>(s.amps, n, sl, tm, shots, m, chosen, scale); break;
    default: k_batch_apply<3><<<grid_for(shots << (n - 3), s.device), kThreads, 0, s.stream>>>(s.amps, n, sl, tm, shots, m, chosen, scale); break;
  }
  QSB_LAUNCHED();
  QSB_CUDA(cudaStreamSynchronize(s.stream));  // host staging buffers go out of scope
}

void batch_kraus(State& s, uint32_t n, const uint32_t* qubits, uint32_t k, const double* ops_host, uint32_t nops,
                 const double* u_host, uint64_t shots, int* chosen_host) {
  if (k < 1 || k > 2) throw ValidationError("batch Kraus step supports 1- and 2-qubit channels");
  if (nops < 1 || nops > 16) throw ValidationError("batch Kraus step: 1 to 16 operators");
  if (n > s.local_qubits() || shots > (s.size >> n)) throw ValidationError("batch Kraus step: bad batch shape");
  std::vector<uint32_t> tg(qubits, qubits + k);
  for (auto q : tg)
    if (q >= n) throw ValidationError("batch Kraus step: qubit out of range");
  const Slots sl = make_slots(tg, {});
  if (sl.count != k) throw ValidationError("batch Kraus step: repeated qubit");
  if (!shots) return;
  TargetMasks tm{};
  for (uint32_t b = 0; b < k; ++b) tm.m[b] = 1ull << tg[k - 1 - b];
  const int D = 1 << k;
  DeviceGuard dg(s.device);
  const size_t ops_bytes = static_cast<size_t>(nops) * D * D * sizeof(double2);
  char* scr = static_cast<char*>(s.get_scratch(ops_bytes + shots * (D * D * 16 + 8 + 8 + 4) + 1024));
  double2* ops = reinterpret_cast<double2*>(scr);
  double2* rdm = ops + static_cast<size_t>(nops) * D * D;
  double* u = reinterpret_cast<double*>(rdm + shots * D * D);
  double* scale = u + shots;
  int* chosen = reinterpret_cast<int*>(scale + shots);
  int* err = chosen + shots + 1;
  QSB_CUDA(cudaMemcpyAsync(ops, ops_host, ops_bytes, cudaMemcpyHostToDevice, s.stream));
  QSB_CUDA(cudaMemcpyAsync(u, u_host, shots * 8, cudaMemcpyHostToDevice, s.stream));
  QSB_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s.stream));
  const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>(shots, num_sms(s.device) * 8ull));
  if (k == 1) {
    k_batch_rdm<1><<<blocks, kThreads, 0, s.stream>>>(s.amps, n, sl, tm, shots, rdm);
    QSB_LAUNCHED();
    k_batch_choose<1><<<grid_for(shots, s.device), kThreads, 0, s.stream>>>(rdm, ops, nops, u, shots, chosen, scale, err);
    QSB_LAUNCHED();
    k_batch_apply<1><<<grid_for(shots << (n - 1), s.device), kThreads, 0, s.stream>>>(s.amps, n, sl, tm, shots, ops,
                                                                                      chosen, scale);
    QSB_LAUNCHED();
  } else {
    k_batch_rdm<2><<<blocks, kThreads, 0, s.stream>>>(s.amps, n, sl, tm, shots, rdm);
    QSB_LAUNCHED();
    k_batch_choose<2><<<grid_for(shots, s.device), kThreads, 0, s.stream>>>(rdm, ops, nops, u, shots, chosen, scale, err);
    QSB_LAUNCHED();
    k_batch_apply<2><<<grid_for(shots << (n - 2), s.device), kThreads, 0, s.stream>>>(s.amps, n, sl, tm, shots, ops,
                                                                                      chosen, scale);
    QSB_LAUNCHED();
  }
  int h_err = 0;
  if (chosen_host) QSB_CUDA(cudaMemcpyAsync(chosen_host, chosen, shots * sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaStreamSynchronize(s.stream));
  if (h_err) throw RuntimeError("trajectory selected a zero-probability Kraus branch");
}

void pauli_axpy(State& s, double2* dst, const double2* src, uint64_t xmask, uint64_t zmask, double fre, double fim) {
  DeviceGuard dg(s.device);
  k_pauli_axpy<<<grid_for(s.size, s.device), kThreads, 0, s.stream>>>(dst, src, s.size, xmask, zmask,
                                                                      make_double2(fre, fim));
  QSB_LAUNCHED();
}

void expect_pauli(State& s, const std::vector<uint64_t>& xmask, const std::vector<uint64_t>& smask,
                  const std::vector<int>& ny, double* out) {
  DeviceGuard dg(s.device);
  const size_t T = xmask.size();
  // terms grouped by X mask (first-appearance order), up to kPauliGroup per pass
  std::vector<std::vector<size_t>> groups;
  {
    std::vector<uint64_t> keys;
    for (size_t t = 0; t < T; ++t) {
      size_t g = 0;
      while (g < keys.size() && (keys[g] != xmask[t] || groups[g].size() == kPauliGroup)) ++g;
      if (g == keys.size()) {
        keys.push_back(xmask[t]);
        groups.emplace_back();
      }
      groups[g].push_back(t);
    }
  }
  const uint32_t blocks = kRedBlocks / 2;
  double2* part = static_cast<double2*>(s.get_scratch((static_cast<size_t>(blocks) * kPauliGroup + T) * sizeof(double2)));
  double2* res = part + static_cast<size_t>(blocks) * kPauliGroup;
  for (const auto& g : groups) {
    ZMasks zm{};
    for (size_t i = 0; i < g.size(); ++i) zm.z[i] = smask[g[i]];
    k_pauli_group<<<blocks, kThreads, 0, s.stream>>>(s.amps, s.size, xmask[g[0]], zm, static_cast<int>(g.size()), part);
    QSB_LAUNCHED();
    for (size_t i = 0; i < g.size(); ++i) {
      k_finalize2_strided<<<1, kThreads, 0, s.stream>>>(part + i, static_cast<int>(blocks), kPauliGroup, res + g[i]);
      QSB_LAUNCHED();
    }
  }
  std::vector<double2> h(T);
  QSB_CUDA(cudaMemcpyAsync(h.data(), res, T * sizeof(double2), cudaMemcpyDeviceToHost, s.stream));
  QSB_CUDA(cudaStreamSynchronize(s.stream));
  for (size_t t = 0; t < T; ++t) {
    // multiply by i^ny
    double re = h[t].x, im = h[t].y;
    for (int k = 0; k < (ny[t] & 3); ++k) {
      const double r2 = -im, i2 = re;
      re = r2;
      im = i2;
    }
    out[2 * t] = re;
    out[2 * t + 1] = im;
  }
}

}  // namespace qsb
