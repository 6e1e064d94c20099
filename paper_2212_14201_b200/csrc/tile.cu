// Shared-memory tile pass kernel (see tile.hpp for the design).
//
// One CTA of 2^(M-4) threads owns one tile of 2^M amplitudes at a time
// (persistent loop over tiles); each thread holds 16 amplitudes in registers.
// The micro-program (header, TOp list, coefficient and metadata tables) is a
// __grid_constant__ kernel parameter: it lives in the constant bank, so every
// warp-uniform read is a constant-cache broadcast instead of an L1 load.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "tile.hpp"

namespace qsb {

namespace {

struct __align__(16) TileBlob {
  unsigned char b[kTileBlobBytes];
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
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

// 2x2 on register bit K.  CHECK: honour the register-index predicate.
template <int K, int VAR, bool CHECK>
__device__ __forceinline__ void mat1(double2 (&v)[16], const double2* c, int rmask, int rval) {
  const double2 m0 = c[0], m1 = c[1], m2 = c[2], m3 = c[3];
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    if (p & (1 << K)) continue;
    const int p1 = p | (1 << K);
    if (CHECK && (p & rmask) != rval) continue;
    const double2 a = v[p], b = v[p1];
    if (VAR == 0) {  // general complex
      v[p] = cmv2(m0, a, m1, b);
      v[p1] = cmv2(m2, a, m3, b);
    } else if (VAR == 1) {  // real matrix (RY, H)
      v[p] = make_double2(fma(m0.x, a.x, m1.x * b.x), fma(m0.x, a.y, m1.x * b.y));
      v[p1] = make_double2(fma(m2.x, a.x, m3.x * b.x), fma(m2.x, a.y, m3.x * b.y));
    } else {  // real diagonal, imaginary off-diagonal (RX)
      v[p] = make_double2(fma(m0.x, a.x, -m1.y * b.y), fma(m0.x, a.y, m1.y * b.x));
      v[p1] = make_double2(fma(m3.x, b.x, -m2.y * a.y), fma(m3.x, b.y, m2.y * a.x));
    }
  }
}

template <int K, bool CHECK>
__device__ __forceinline__ void flip(double2 (&v)[16], int rmask, int rval) {
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    if (p & (1 << K)) continue;
    const int p1 = p | (1 << K);
    if (CHECK && (p & rmask) != rval) continue;
    const double2 a = v[p];
    v[p] = v[p1];
    v[p1] = a;
  }
}

template <int KD>
__device__ __forceinline__ void dense(double2 (&v)[16], const double2* M, int rmask, int rval) {
  constexpr int G = 1 << KD;
#pragma unroll
  for (int hi = 0; hi < (16 >> KD); ++hi) {
    const int p0 = hi << KD;
    if ((p0 & rmask) != rval) continue;
    double2 in[G];
#pragma unroll
    for (int c = 0; c < G; ++c) in[c] = v[p0 + c];
#pragma unroll
    for (int r = 0; r < G; ++r) {
      double re = 0, im = 0;
#pragma unroll
      for (int c = 0; c < G; ++c) {
        const double2 m = M[r * G + c];
        re = fma(m.x, in[c].x, re);
        re = fma(-m.y, in[c].y, re);
        im = fma(m.x, in[c].y, im);
        im = fma(m.y, in[c].x, im);
      }
      v[p0 + r] = make_double2(re, im);
    }
  }
}

template <int VAR>
__device__ __forceinline__ void mat1_any(double2 (&v)[16], int k, const double2* c, int rmask, int rval) {
  if (rmask == 0) {
    switch (k) {
      case 0: mat1<0, VAR, false>(v, c, 0, 0); break;
      case 1: mat1<1, VAR, false>(v, c, 0, 0); break;
      case 2: mat1<2, VAR, false>(v, c, 0, 0); break;
      default: mat1<3, VAR, false>(v, c, 0, 0); break;
    }
  } else {
    switch (k) {
      case 0: mat1<0, VAR, true>(v, c, rmask, rval); break;
      case 1: mat1<1, VAR, true>(v, c, rmask, rval); break;
      case 2: mat1<2, VAR, true>(v, c, rmask, rval); break;
      default: mat1<3, VAR, true>(v, c, rmask, rval); break;
    }
  }
}

__device__ __forceinline__ void flip_any(double2 (&v)[16], int k, int rmask, int rval) {
  if (rmask == 0) {
    switch (k) {
      case 0: flip<0, false>(v, 0, 0); break;
      case 1: flip<1, false>(v, 0, 0); break;
      case 2: flip<2, false>(v, 0, 0); break;
      default: flip<3, false>(v, 0, 0); break;
    }
  } else {
    switch (k) {
      case 0: flip<0, true>(v, rmask, rval); break;
      case 1: flip<1, true>(v, rmask, rval); break;
      case 2: flip<2, true>(v, rmask, rval); break;
      default: flip<3, true>(v, rmask, rval); break;
    }
  }
}

__device__ __forceinline__ uint64_t reg_offset(int p, const unsigned long long (&rs)[4]) {
  uint64_t o = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if ((p >> k) & 1) o |= rs[k];
  return o;
}

template <int M>
__global__ void __launch_bounds__(1 << (M - 4), (M >= 13 ? 1 : 2))
    k_tile(double2* __restrict__ amps, const __grid_constant__ TileBlob blob) {
  constexpr int TB = M - 4;
  extern __shared__ double2 sm[];
  const TileHeader* H = reinterpret_cast<const TileHeader*>(blob.b);
  const TOp* ops = reinterpret_cast<const TOp*>(blob.b + H->ops_off);
  const uint32_t* meta = reinterpret_cast<const uint32_t*>(blob.b + H->meta_off);
  const double2* coef = reinterpret_cast<const double2*>(blob.b + H->coef_off);
  const int tid = threadIdx.x;
  const uint32_t nops = H->nops;
  const unsigned long long ntiles = H->ntiles;

  for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // tile base: the tile id deposited into the qubits outside S
    uint64_t base = tile;
#pragma unroll
    for (int b = 0; b < M; ++b) {
      const uint32_t p = H->S[b];
      base = ((base >> p) << (p + 1)) | (base & ((1ull << p) - 1));
    }
    uint64_t G = base;
#pragma unroll
    for (int k = 0; k < TB; ++k)
      if ((tid >> k) & 1) G |= 1ull << H->load.tq[k];
    unsigned long long rs[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) rs[k] = H->load.rs[k];
    double2 v[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) v[p] = __ldcs(amps + (G | reg_offset(p, rs)));

#pragma unroll 1
    for (uint32_t i = 0; i < nops; ++i) {
      const TOp& o = ops[i];
      const bool tp = (G & o.gmask) == o.gval;
      switch (o.type) {
        case TO_MAT1:
          if (tp) mat1_any<0>(v, o.k, coef + o.coef, o.rmask, o.rval);
          break;
        case TO_MAT1_REAL:
          if (tp) mat1_any<1>(v, o.k, coef + o.coef, o.rmask, o.rval);
          break;
        case TO_MAT1_RX:
          if (tp) mat1_any<2>(v, o.k, coef + o.coef, o.rmask, o.rval);
          break;
        case TO_FLIP:
          if (tp) flip_any(v, o.k, o.rmask, o.rval);
          break;
        case TO_PHASE:
          if (tp) {
            const double2* c = coef + o.coef;
            double2 F = c[16];
            const uint32_t nl = o.nlist;
            for (uint32_t j = 0; j < nl; ++j)
              if ((G >> meta[o.meta + j]) & 1) F = cmul(F, c[17 + j]);
            const int rm = o.rmask, rv = o.rval;
            if (rm == 0) {
#pragma unroll
              for (int p = 0; p < 16; ++p) v[p] = cmul(v[p], cmul(F, c[p]));
            } else {
#pragma unroll
              for (int p = 0; p < 16; ++p)
                if ((p & rm) == rv) v[p] = cmul(v[p], cmul(F, c[p]));
            }
          }
          break;
        case TO_DENSE2:
          if (tp) dense<2>(v, coef + o.coef, o.rmask, o.rval);
          break;
        case TO_DENSE3:
          if (tp) dense<3>(v, coef + o.coef, o.rmask, o.rval);
          break;
        case TO_TRANSPOSE: {
          const uint32_t* mt = meta + o.meta;
          uint32_t Tw = 0, Tr = 0;
#pragma unroll
          for (int k = 0; k < TB; ++k)
            if ((tid >> k) & 1) {
              Tw ^= mt[k];
              Tr ^= mt[TB + 4 + k];
            }
          uint32_t wR[4], rR[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            wR[k] = mt[TB + k];
            rR[k] = mt[2 * TB + 4 + k];
          }
          __syncthreads();  // previous transpose's reads are done
#pragma unroll
          for (int p = 0; p < 16; ++p) {
            uint32_t a = Tw;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if ((p >> k) & 1) a ^= wR[k];
            sm[a] = v[p];
          }
          __syncthreads();
#pragma unroll
          for (int p = 0; p < 16; ++p) {
            uint32_t a = Tr;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if ((p >> k) & 1) a ^= rR[k];
            v[p] = sm[a];
          }
          G = base;
#pragma unroll
          for (int k = 0; k < TB; ++k)
            if ((tid >> k) & 1) G |= 1ull << mt[2 * TB + 8 + k];
          break;
        }
        case TO_RELABEL: {
          const uint32_t* mt = meta + o.meta;
          G = base;
#pragma unroll
          for (int k = 0; k < TB; ++k)
            if ((tid >> k) & 1) G |= 1ull << mt[k];
          break;
        }
        default: break;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) rs[k] = H->store.rs[k];
#pragma unroll
    for (int p = 0; p < 16; ++p) __stcs(amps + (G | reg_offset(p, rs)), v[p]);
  }
}

template <int M>
void launch_m(State& s, const TileProgram& tp) {
  constexpr int T = 1 << (M - 4);
  const size_t smem = tp.transposes ? (size_t(1) << M) * sizeof(double2) : 0;
  static std::once_flag once[64];
  std::call_once(once[s.device & 63], [&] {
    QSB_CUDA(cudaFuncSetAttribute(k_tile<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>((size_t(1) << M) * sizeof(double2))));
  });
  int per_sm = 0;
  QSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile<M>, T, smem));
  per_sm = std::max(per_sm, 1);
  const unsigned long long ntiles = tp.h.ntiles;
  const unsigned long long cap = static_cast<unsigned long long>(per_sm) * num_sms(s.device);
  const unsigned grid = static_cast<unsigned>(std::min(ntiles, cap));
  if (tp.h.bytes > kTileBlobBytes) throw RuntimeError("tile program exceeds the parameter blob");
  static thread_local TileBlob blob;
  std::memcpy(blob.b, tp.blob.data(), tp.h.bytes);
  k_tile<M><<<grid, T, smem, s.stream>>>(s.amps, blob);
  QSB_LAUNCHED();
}

}  // namespace

void TileProgram::pack() {
  blob.assign(h.bytes, 0);
  std::memcpy(blob.data(), &h, sizeof(TileHeader));
  if (!ops.empty()) std::memcpy(blob.data() + h.ops_off, ops.data(), ops.size() * sizeof(TOp));
  if (!meta.empty()) std::memcpy(blob.data() + h.meta_off, meta.data(), meta.size() * sizeof(uint32_t));
  if (!coef.empty()) std::memcpy(blob.data() + h.coef_off, coef.data(), coef.size() * sizeof(double2));
}

void launch_tile(State& s, const TileProgram& tp) {
  DeviceGuard dg(s.device);
  switch (tp.h.m) {
    case 6: launch_m<6>(s, tp); break;
    case 7: launch_m<7>(s, tp); break;
    case 8: launch_m<8>(s, tp); break;
    case 9: launch_m<9>(s, tp); break;
    case 10: launch_m<10>(s, tp); break;
    case 11: launch_m<11>(s, tp); break;
    case 12: launch_m<12>(s, tp); break;
    case 13: launch_m<13>(s, tp); break;
    default: throw RuntimeError("unsupported tile size");
  }
}

}  // namespace qsb
