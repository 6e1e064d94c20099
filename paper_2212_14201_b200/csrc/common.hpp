// Shared host-side definitions of libqsb: error types, the state handle,
// CUDA checking.  Exceptions never cross the C ABI (abi.cpp converts them).
#pragma once

#include <cuda_runtime.h>

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/qsb.h"

namespace qsb {

using cd = std::complex<double>;

// Mirrors qforge::ValidationError / qforge::Error (error.hpp:10-20).
struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct MemoryError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Mirrors qforge::UnsupportedError (error.hpp): valid input the operation does not handle.
struct UnsupportedError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define QSB_CUDA(expr)                                                                     \
  do {                                                                                     \
    cudaError_t qsb_e_ = (expr);                                                           \
    if (qsb_e_ != cudaSuccess)                                                             \
      throw ::qsb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(qsb_e_) +       \
                             " (" __FILE__ ":" + std::to_string(__LINE__) + ")");          \
  } while (0)

// Kernel launch accounting (qs_kernel_launches) + error check.
void note_launch(int count = 1);
#define QSB_LAUNCHED()                   \
  do {                                   \
    ::qsb::note_launch();                \
    QSB_CUDA(cudaPeekAtLastError());     \
  } while (0)

// A state vector on one device: 2^n complex128 amplitudes, logical order.
struct State {
  uint32_t n = 0;             // qubits of the whole state
  int device = 0;
  uint64_t size = 0;          // amplitudes held here: 2^(n-g)
  // Sharded states: the top g qubits are rank bits; this object holds the
  // shard with rank `rank` (global index = rank_base | local index).
  uint32_t g = 0;
  uint32_t rank = 0;
  uint64_t rank_base = 0;
  uint32_t local_qubits() const { return n - g; }
  double2* amps = nullptr;    // device
  double2* alt = nullptr;     // second buffer of a shard exchanged through peer memory
  cudaStream_t stream = nullptr;
  // scratch (grown on demand)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* host_pinned = nullptr;
  size_t host_pinned_bytes = 0;

  void* get_scratch(size_t bytes);
  void* get_pinned(size_t bytes);
  void sync();
};

// RAII device guard.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    QSB_CUDA(cudaGetDevice(&prev));
    if (prev != dev) QSB_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

inline uint32_t num_sms(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cached[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cached[device] = v > 0 ? v : 148;
  }
  return static_cast<uint32_t>(cached[device]);
}

}  // namespace qsb
