// Diagnostic: read+write bandwidth of an in-place streaming pass over a
// complex128 buffer as a function of its size (L2-resident vs HBM), and of a
// "blocked" schedule that sweeps each L2-sized block k times before moving on.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/l2_probe tools/l2_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void pass(double2* __restrict__ a, size_t n, double s) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = __ldcg(a + i);
    v.x *= s;
    v.y *= s;
    __stcg(a + i, v);
  }
}

// sweeps block b (blk amplitudes) `reps` times with a grid barrier-free
// schedule: every CTA handles a fixed slice of every block (same slice each
// sweep, so no cross-CTA dependency), the whole grid moves block to block.
__global__ void blocked(double2* __restrict__ a, size_t n, size_t blk, int reps, double s) {
  const size_t per = blk / gridDim.x;
  for (size_t b = 0; b < n; b += blk) {
    double2* p = a + b + size_t(blockIdx.x) * per;
    for (int r = 0; r < reps; ++r)
      for (size_t i = threadIdx.x; i < per; i += blockDim.x) {
        double2 v = __ldcg(p + i);
        v.x *= s;
        v.y *= s;
        __stcg(p + i, v);
      }
  }
}

int main(int argc, char** argv) {
  const int sms = 148;
  double2* a;
  const size_t maxn = size_t(1) << 30;
  if (cudaMalloc(&a, maxn * sizeof(double2)) != cudaSuccess) return 1;
  cudaMemset(a, 0, maxn * sizeof(double2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int lg = 18; lg <= 30; ++lg) {
    const size_t n = size_t(1) << lg;
    const int reps = lg <= 24 ? 200 : (lg <= 27 ? 20 : 5);
    for (int w = 0; w < 3; ++w) pass<<<sms * 4, 512>>>(a, n, 1.0);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) pass<<<sms * 4, 512>>>(a, n, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("{\"probe\":\"pass\",\"log2n\":%d,\"MiB\":%zu,\"GBps_rw\":%.1f,\"us_per_pass\":%.2f}\n", lg,
                n * 16 >> 20, 32.0 * n * reps / (ms * 1e6), ms * 1e3 / reps);
  }
  // blocked schedule over the full 16 GiB: each block swept k times
  for (int lgb = 20; lgb <= 24; ++lgb)
    for (int k = 1; k <= 4; k *= 2) {
      const size_t blk = size_t(1) << lgb;
      blocked<<<sms, 1024>>>(a, maxn, blk, k, 1.0);
      cudaEventRecord(e0);
      blocked<<<sms, 1024>>>(a, maxn, blk, k, 1.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::printf("{\"probe\":\"blocked\",\"log2blk\":%d,\"MiB\":%zu,\"sweeps\":%d,\"ms\":%.2f,\"ms_per_sweep\":%.3f,"
                  "\"GBps_rw_per_sweep\":%.1f}\n",
                  lgb, blk * 16 >> 20, k, ms, ms / k, 32.0 * maxn * k / (ms * 1e6));
    }
  cudaError_t err = cudaGetLastError();
  std::printf("{\"status\":\"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
