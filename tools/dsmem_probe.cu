// Diagnostic: distributed shared memory (DSMEM) exchange bandwidth on B200,
// the cost a 14-qubit tile split over a 2-CTA cluster would pay per
// cross-CTA exchange ("chain bound").  Each CTA of a 2-CTA
// cluster writes HALF of its 128 KiB tile buffer into its partner's buffer
// (st.shared::cluster via cooperative_groups map_shared_rank), cluster
// barrier, repeat; compared with the same volume exchanged inside one CTA's
// own shared memory (the local transpose).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dsmem_probe tools/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

constexpr int kThreads = 512;
constexpr int kAmps = 8192;  // 128 KiB of double2 per CTA

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) dsmem_exchange(int reps, double* sink) {
  extern __shared__ double2 buf[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank();
  double2* peer = cl.map_shared_rank(buf, me ^ 1u);
  for (int i = threadIdx.x; i < kAmps; i += blockDim.x) buf[i] = make_double2(i, me);
  cl.sync();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    // half of the tile (the amplitudes whose cluster bit changes) goes to the partner
    for (int i = threadIdx.x; i < kAmps / 2; i += blockDim.x) peer[kAmps / 2 + i] = buf[i];
    cl.sync();
    acc += buf[kAmps / 2 + (threadIdx.x + r) % (kAmps / 2)].x;
    cl.sync();
  }
  if (acc == -1.0) *sink = acc;
}

__global__ void __launch_bounds__(kThreads, 1) local_exchange(int reps, double* sink) {
  extern __shared__ double2 buf[];
  for (int i = threadIdx.x; i < kAmps; i += blockDim.x) buf[i] = make_double2(i, 0);
  __syncthreads();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < kAmps / 2; i += blockDim.x) buf[kAmps / 2 + (i ^ 32)] = buf[i];
    __syncthreads();
    acc += buf[kAmps / 2 + (threadIdx.x + r) % (kAmps / 2)].x;
    __syncthreads();
  }
  if (acc == -1.0) *sink = acc;
}

int main() {
  double* sink;
  cudaMalloc(&sink, 8);
  const size_t smem = kAmps * sizeof(double2);
  cudaFuncSetAttribute(dsmem_exchange, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(local_exchange, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 2000, grid = 148;
  for (int which = 0; which < 2; ++which) {
    for (int w = 0; w < 2; ++w) {
      if (which == 0) dsmem_exchange<<<grid, kThreads, smem>>>(10, sink);
      else local_exchange<<<grid, kThreads, smem>>>(10, sink);
    }
    cudaEventRecord(e0);
    if (which == 0) dsmem_exchange<<<grid, kThreads, smem>>>(reps, sink);
    else local_exchange<<<grid, kThreads, smem>>>(reps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(grid) * reps * (kAmps / 2) * sizeof(double2);  // written per CTA per rep
    const double per_cta_bps = bytes / grid / (ms * 1e-3);
    std::printf("{\"probe\":\"%s\",\"ms\":%.3f,\"GBps_total\":%.1f,\"per_cta_GBps\":%.2f,\"per_cta_B_per_clk\":%.2f,"
                "\"us_per_64KiB_exchange\":%.3f,\"clock_khz\":%d,\"status\":\"%s\"}\n",
                which == 0 ? "dsmem 2-CTA cluster, half tile to the partner" : "local smem, half tile",
                ms, bytes / (ms * 1e-3) / 1e9, per_cta_bps / 1e9, per_cta_bps / (clk * 1e3), ms * 1e3 / reps, clk,
                cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
