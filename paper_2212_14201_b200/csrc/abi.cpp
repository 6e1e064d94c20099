// extern "C" boundary of libqsb.so (include/qsb.h).  Converts exceptions to
// status codes + a thread-local message; owns state / plan handles.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <random>
#include <string>

#include "common.hpp"
#include "fusion.hpp"
#include "gates.hpp"
#include "jit.hpp"
#include "kernels.hpp"
#include "plan.hpp"
#include "shard.hpp"

namespace qsb {
void partial_amplitude(uint32_t n, const qs_gate* gates, uint64_t count, const uint32_t* block_a, uint32_t na,
                       const uint64_t* targets, uint64_t ntargets, int device, uint32_t batch_qubits,
                       double* out);  // pathsum.cpp
void gradient_adjoint(State& s, const qs_gate* gates, uint64_t count, const uint64_t* slots, uint64_t nslots,
                      const std::vector<uint64_t>& xm, const std::vector<uint64_t>& zm, const std::vector<int>& ny,
                      const double* coeffs, double* out);  // gradient.cpp
}
#include "tile.hpp"

struct qs_state {
  qsb::State s;
};
struct qs_plan {
  std::unique_ptr<qsb::Plan> p;
};
struct qs_fused {
  std::vector<qsb::GateRec> gates;
};
struct qs_dist {
  qsb::Dist* d = nullptr;
};
struct qs_shards {
  std::unique_ptr<qsb::ShardSet> ss;
};

namespace qsb {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return QS_OK;
  } catch (const ValidationError& e) {
    g_last_error = e.what();
    return QS_ERR_VALIDATION;
  } catch (const RuntimeError& e) {
    g_last_error = e.what();
    return QS_ERR_RUNTIME;
  } catch (const MemoryError& e) {
    g_last_error = e.what();
    return QS_ERR_MEMORY;
  } catch (const UnsupportedError& e) {
    g_last_error = e.what();
    return QS_ERR_UNSUPPORTED;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return QS_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return QS_ERR_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return QS_ERR_RUNTIME;
  }
}

State& st(qs_state_t h) {
  if (!h) throw ValidationError("null state handle");
  return h->s;
}

void check_qubit(const State& s, uint32_t q) {
  if (q >= s.n) throw ValidationError("qubit q[" + std::to_string(q) + "] out of range");
}
}  // namespace

void note_launch(int count) { g_launches.fetch_add(static_cast<uint64_t>(count), std::memory_order_relaxed); }

void* State::get_scratch(size_t bytes) {
  if (bytes > scratch_bytes) {
    DeviceGuard dg(device);
    if (scratch) {
      QSB_CUDA(cudaStreamSynchronize(stream));
      cudaFree(scratch);
      scratch = nullptr;
      scratch_bytes = 0;
    }
    const size_t want = std::max<size_t>(bytes, 1 << 20);
    if (cudaMalloc(&scratch, want) != cudaSuccess) {
      cudaGetLastError();
      throw MemoryError("device scratch allocation of " + std::to_string(want) + " bytes failed");
    }
    scratch_bytes = want;
  }
  return scratch;
}

void* State::get_pinned(size_t bytes) {
  if (bytes > host_pinned_bytes) {
    if (host_pinned) cudaFreeHost(host_pinned);
    host_pinned = nullptr;
    QSB_CUDA(cudaMallocHost(&host_pinned, std::max<size_t>(bytes, 4096)));
    host_pinned_bytes = std::max<size_t>(bytes, 4096);
  }
  return host_pinned;
}

void State::sync() {
  DeviceGuard dg(device);
  QSB_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace qsb

using namespace qsb;

extern "C" {

const char* qs_last_error(void) { return qsb::g_last_error.c_str(); }
int qs_abi_version(void) { return QSB_ABI_VERSION; }
uint64_t qs_kernel_launches(void) { return qsb::g_launches.load(); }
int qs_jit_stats(uint64_t* nvrtc_builds, uint64_t* memory_hits, uint64_t* disk_hits) {
  if (nvrtc_builds) *nvrtc_builds = qsb::jit_compiles();
  if (memory_hits) *memory_hits = qsb::jit_cache_hits();
  if (disk_hits) *disk_hits = qsb::jit_disk_hits();
  return QS_OK;
}

int qs_create(uint32_t num_qubits, int device, uint32_t max_qubits, qs_state_t* out) {
  return guarded([&] {
    if (!out) throw ValidationError("null output handle");
    *out = nullptr;
    const uint32_t cap = max_qubits ? max_qubits : 30;
    if (num_qubits > cap)
      throw ValidationError("state vector limited to " + std::to_string(cap) + " qubits");
    if (num_qubits > 40) throw ValidationError("state vector limited to 40 qubits per device");
    int ndev = 0;
    QSB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ValidationError("CUDA device " + std::to_string(device) + " not present");
    auto* h = new qs_state();
    State& s = h->s;
    s.n = num_qubits;
    s.device = device;
    s.size = 1ull << num_qubits;
    try {
      DeviceGuard dg(device);
      QSB_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
      if (cudaMalloc(&s.amps, s.size * sizeof(double2)) != cudaSuccess) {
        cudaGetLastError();
        throw MemoryError("cannot allocate " + std::to_string(s.size * 16) + " bytes for a " +
                          std::to_string(num_qubits) + "-qubit state");
      }
      fill_basis(s, 0);
      s.sync();
    } catch (...) {
      if (s.amps) cudaFree(s.amps);
      if (s.stream) cudaStreamDestroy(s.stream);
      delete h;
      throw;
    }
    *out = h;
  });
}

int qs_destroy(qs_state_t h) {
  return guarded([&] {
    if (!h) return;
    State& s = h->s;
    {
      DeviceGuard dg(s.device);
      cudaStreamSynchronize(s.stream);
      if (s.amps) cudaFree(s.amps);
      if (s.alt) cudaFree(s.alt);
      if (s.scratch) cudaFree(s.scratch);
      if (s.host_pinned) cudaFreeHost(s.host_pinned);
      cudaStreamDestroy(s.stream);
    }
    delete h;
  });
}

int qs_clone(qs_state_t src, qs_state_t* out) {
  return guarded([&] {
    State& a = st(src);
    qs_state_t h = nullptr;
    const int rc = qs_create(a.n, a.device, 64, &h);
    if (rc != QS_OK) throw RuntimeError(qs_last_error());
    DeviceGuard dg(a.device);
    a.sync();
    QSB_CUDA(cudaMemcpyAsync(h->s.amps, a.amps, a.size * sizeof(double2), cudaMemcpyDeviceToDevice, h->s.stream));
    h->s.sync();
    *out = h;
  });
}

uint32_t qs_num_qubits(qs_state_t s) { return s ? s->s.n : 0; }
int qs_device(qs_state_t s) { return s ? s->s.device : -1; }
void* qs_device_ptr(qs_state_t s) { return s ? s->s.amps : nullptr; }

int qs_reset(qs_state_t h) {
  return guarded([&] {
    fill_basis(st(h), 0);
    st(h).sync();
  });
}

int qs_set_basis_state(qs_state_t h, uint64_t index) {
  return guarded([&] {
    State& s = st(h);
    if (index >= s.size) throw ValidationError("basis index out of range");
    fill_basis(s, index);
    s.sync();
  });
}

int qs_sync(qs_state_t h) {
  return guarded([&] { st(h).sync(); });
}

void* qs_stream(qs_state_t h) { return h ? static_cast<void*>(h->s.stream) : nullptr; }

int qs_set_amplitudes(qs_state_t h, const double* data, uint64_t offset, uint64_t count) {
  return guarded([&] {
    State& s = st(h);
    if (offset > s.size || count > s.size - offset) throw ValidationError("amplitude count does not match qubit count");
    DeviceGuard dg(s.device);
    QSB_CUDA(cudaMemcpyAsync(s.amps + offset, data, count * sizeof(double2), cudaMemcpyHostToDevice, s.stream));
    s.sync();
  });
}

int qs_get_amplitudes(qs_state_t h, double* data, uint64_t offset, uint64_t count) {
  return guarded([&] {
    State& s = st(h);
    if (offset > s.size || count > s.size - offset) throw ValidationError("amplitude range out of bounds");
    DeviceGuard dg(s.device);
    QSB_CUDA(cudaMemcpyAsync(data, s.amps + offset, count * sizeof(double2), cudaMemcpyDeviceToHost, s.stream));
    s.sync();
  });
}

int qs_apply_gate(qs_state_t h, const qs_gate* g) {
  return guarded([&] {
    State& s = st(h);
    if (!g) throw ValidationError("null gate");
    launch_op(s, lower_gate(*g, s.n, true));
    s.sync();
  });
}

static Op simple_op(State& s, OpKind k, std::vector<uint32_t> targets, const uint32_t* controls, uint32_t nc) {
  Op op;
  op.kind = k;
  op.targets = std::move(targets);
  op.controls.assign(controls, controls + nc);
  std::vector<uint32_t> all = op.controls;
  all.insert(all.end(), op.targets.begin(), op.targets.end());
  for (auto q : all) check_qubit(s, q);
  std::sort(all.begin(), all.end());
  if (std::adjacent_find(all.begin(), all.end()) != all.end()) throw ValidationError("duplicate qubit operand");
  return op;
}

int qs_apply_1q(qs_state_t h, uint32_t target, const double m[8], const uint32_t* controls, uint32_t nc) {
  return guarded([&] {
    State& s = st(h);
    Op op = simple_op(s, OpKind::Mat1, {target}, controls, nc);
    op.m = {cd(m[0], m[1]), cd(m[2], m[3]), cd(m[4], m[5]), cd(m[6], m[7])};
    launch_op(s, op);
    s.sync();
  });
}

int qs_apply_diag(qs_state_t h, uint32_t target, const double d[4], const uint32_t* controls, uint32_t nc) {
  return guarded([&] {
    State& s = st(h);
    Op op = simple_op(s, OpKind::Diag, {target}, controls, nc);
    op.m = {cd(d[0], d[1]), cd(d[2], d[3])};
    launch_op(s, op);
    s.sync();
  });
}

int qs_apply_flip(qs_state_t h, uint32_t target, const uint32_t* controls, uint32_t nc) {
  return guarded([&] {
    State& s = st(h);
    launch_op(s, simple_op(s, OpKind::Flip, {target}, controls, nc));
    s.sync();
  });
}

int qs_apply_swap(qs_state_t h, uint32_t a, uint32_t b, const uint32_t* controls, uint32_t nc) {
  return guarded([&] {
    State& s = st(h);
    launch_op(s, simple_op(s, OpKind::Swap, {a, b}, controls, nc));
    s.sync();
  });
}

int qs_apply_matrix(qs_state_t h, const uint32_t* targets, uint32_t k, const double* m, const uint32_t* controls,
                    uint32_t nc) {
  return guarded([&] {
    State& s = st(h);
    if (!targets || !m) throw ValidationError("null targets or matrix");
    launch_op(s, lower_matrix(targets, k, m, controls, nc, s.n));
    s.sync();
  });
}

int qs_apply_circuit(qs_state_t h, const qs_gate* gates, uint64_t n, uint32_t plan, uint32_t max_fused_qubits) {
  return guarded([&] {
    State& s = st(h);
    if (n && !gates) throw ValidationError("null gate array");
    auto p = cached_plan(s.n, gates, n, plan, max_fused_qubits);
    execute_plan(s, *p);
    s.sync();
  });
}

int qs_run_circuit(qs_state_t h, uint64_t basis, const qs_gate* gates, uint64_t n, uint32_t plan,
                   uint32_t max_fused_qubits) {
  return guarded([&] {
    State& s = st(h);
    if (n && !gates) throw ValidationError("null gate array");
    auto p = cached_plan(s.n, gates, n, plan, max_fused_qubits);
    execute_plan_from_basis(s, *p, basis);
    s.sync();
  });
}

int qs_plan_create(uint32_t num_qubits, const qs_gate* gates, uint64_t n, uint32_t plan, uint32_t max_fused_qubits,
                   qs_plan_t* out) {
  return guarded([&] {
    if (!out) throw ValidationError("null output handle");
    if (n && !gates) throw ValidationError("null gate array");
    auto* h = new qs_plan();
    try {
      h->p = make_plan(num_qubits, gates, n, plan, max_fused_qubits);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int qs_plan_destroy(qs_plan_t p) {
  return guarded([&] { delete p; });
}

int qs_plan_execute(qs_state_t h, qs_plan_t p) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    State& s = st(h);
    execute_plan(s, *p->p);
    s.sync();
  });
}

int qs_plan_enqueue(qs_state_t h, qs_plan_t p) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    execute_plan(st(h), *p->p);
  });
}

int qs_plan_enqueue_from_basis(qs_state_t h, qs_plan_t p, uint64_t basis) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    execute_plan_from_basis(st(h), *p->p, basis);
  });
}

int qs_plan_execute_from_basis_checksum(qs_state_t h, qs_plan_t p, uint64_t basis, double* checksum) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    if (!checksum) throw ValidationError("null checksum output");
    execute_plan_from_basis(st(h), *p->p, basis, checksum);
  });
}

int qs_run_circuit_checksum(qs_state_t h, uint64_t basis, const qs_gate* gates, uint64_t n, uint32_t plan,
                            uint32_t max_fused_qubits, double* checksum) {
  return guarded([&] {
    State& s = st(h);
    if (n && !gates) throw ValidationError("null gate array");
    if (!checksum) throw ValidationError("null checksum output");
    auto p = cached_plan(s.n, gates, n, plan, max_fused_qubits);
    execute_plan_from_basis(s, *p, basis, checksum);
  });
}

int qs_plan_execute_from_basis_profile(qs_state_t h, qs_plan_t p, uint64_t basis, double* checksum, float* step_ms,
                                       double* step_bytes) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    StepProfile prof;
    execute_plan_from_basis(st(h), *p->p, basis, checksum, &prof);
    const auto& steps = p->p->steps;
    for (size_t i = 0, o = 0; i < prof.ms.size(); ++i) {
      if (steps[i].kind == Step::OpStep && steps[i].op.kind == OpKind::Identity) continue;  // not a launch
      if (step_ms) step_ms[o] = prof.ms[i];
      if (step_bytes) step_bytes[o] = prof.bytes[i];
      ++o;
    }
  });
}

int qs_plan_execute_from_basis(qs_state_t h, qs_plan_t p, uint64_t basis) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    execute_plan_from_basis(st(h), *p->p, basis);
    st(h).sync();
  });
}

int qs_plan_execute_range(qs_state_t h, qs_plan_t p, uint64_t first, uint64_t count) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    State& s = st(h);
    const auto& steps = p->p->steps;
    if (first > steps.size()) throw ValidationError("step range out of bounds");
    const uint64_t last = std::min<uint64_t>(steps.size(), first + count);
    for (uint64_t i = first; i < last; ++i) execute_step(s, steps[i]);
    s.sync();
  });
}

int qs_plan_execute_timed(qs_state_t h, qs_plan_t p, float* step_ms) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    State& s = st(h);
    DeviceGuard dg(s.device);
    const size_t ns = p->p->steps.size();
    std::vector<cudaEvent_t> ev(ns + 1);
    for (auto& e : ev) QSB_CUDA(cudaEventCreate(&e));
    QSB_CUDA(cudaEventRecord(ev[0], s.stream));
    for (size_t i = 0; i < ns; ++i) {
      execute_step(s, p->p->steps[i]);
      QSB_CUDA(cudaEventRecord(ev[i + 1], s.stream));
    }
    s.sync();
    for (size_t i = 0; i < ns; ++i) QSB_CUDA(cudaEventElapsedTime(&step_ms[i], ev[i], ev[i + 1]));
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

int qs_plan_stats(qs_plan_t p, uint64_t* passes, uint64_t* launches, uint64_t* gates) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    if (passes) *passes = p->p->passes();
    if (launches) *launches = p->p->launches();
    if (gates) *gates = p->p->gates;
  });
}

int qs_fuse(const qs_gate* gates, uint64_t n, uint32_t num_qubits, uint32_t max_fused_qubits, qs_fused_t* out) {
  return guarded([&] {
    if (!out) throw ValidationError("null output handle");
    if (max_fused_qubits < 1) throw ValidationError("max_fused_qubits must be at least 1");
    for (uint64_t i = 0; i < n; ++i) validate_gate(gates[i], num_qubits);
    auto* f = new qs_fused();
    f->gates = fuse_gate_run(gates, n, num_qubits, max_fused_qubits);
    for (auto& g : f->gates) g.bind();
    *out = f;
  });
}

uint64_t qs_fused_count(qs_fused_t f) { return f ? f->gates.size() : 0; }

int qs_fused_get(qs_fused_t f, uint64_t i, qs_gate* out) {
  return guarded([&] {
    if (!f || i >= f->gates.size() || !out) throw ValidationError("bad fused gate index");
    f->gates[i].bind();
    *out = f->gates[i].g;
  });
}

int qs_fused_free(qs_fused_t f) {
  return guarded([&] { delete f; });
}

int qs_norm2(qs_state_t h, double* out) {
  return guarded([&] { *out = reduce_norm2(st(h)); });
}

int qs_prob_one(qs_state_t h, uint32_t q, double* out) {
  return guarded([&] {
    check_qubit(st(h), q);
    *out = reduce_prob_one(st(h), q);
  });
}

int qs_probs(qs_state_t h, const uint32_t* qubits, uint32_t m, double* out) {
  return guarded([&] {
    State& s = st(h);
    if (m == 0) throw ValidationError("probabilities: empty qubit subset");
    std::vector<uint32_t> qs(qubits, qubits + m);
    for (auto q : qs)
      if (q >= s.n) throw ValidationError("probabilities: qubit out of range");
    std::sort(qs.begin(), qs.end());
    if (std::adjacent_find(qs.begin(), qs.end()) != qs.end()) {
      // The reference tolerates repeated qubits (each bit reads the same
      // qubit); fold through the full distribution.
      std::vector<double> full(s.size);
      full_probs(s, full.data(), 0, s.size);
      std::fill(out, out + (1ull << m), 0.0);
      for (uint64_t i = 0; i < s.size; ++i) {
        uint64_t key = 0;
        for (uint32_t b = 0; b < m; ++b)
          if (i & (1ull << qubits[b])) key |= 1ull << b;
        out[key] += full[i];
      }
      return;
    }
    marginal_probs(s, qubits, m, out);
  });
}

int qs_probs_full(qs_state_t h, double* out, uint64_t offset, uint64_t count) {
  return guarded([&] {
    State& s = st(h);
    if (offset > s.size || count > s.size - offset) throw ValidationError("probability range out of bounds");
    full_probs(s, out, offset, count);
  });
}

int qs_checksum(qs_state_t h, double* out) {
  return guarded([&] { *out = reduce_checksum(st(h)); });
}

int qs_checksum_serial(qs_state_t h, double* out) {
  return guarded([&] { *out = serial_checksum(st(h)); });
}

int qs_collapse(qs_state_t h, uint32_t q, int outcome, double prob) {
  return guarded([&] {
    State& s = st(h);
    check_qubit(s, q);
    if (prob <= 0.0) throw RuntimeError("collapse onto a zero-probability outcome");
    collapse(s, q, outcome, 1.0 / std::sqrt(prob));
    s.sync();
  });
}

int qs_measure_collapse(qs_state_t h, uint32_t q, double u, int* outcome) {
  return guarded([&] {
    State& s = st(h);
    check_qubit(s, q);
    const double p1 = reduce_prob_one(s, q);
    const double p0 = 1.0 - p1;
    const int o = (u < p0) ? 0 : 1;
    const double prob = o ? p1 : p0;
    if (prob <= 0.0) throw RuntimeError("collapse onto a zero-probability outcome");
    collapse(s, q, o, 1.0 / std::sqrt(prob));
    s.sync();
    if (outcome) *outcome = o;
  });
}

int qs_scale(qs_state_t h, double re, double im) {
  return guarded([&] {
    scale(st(h), re, im);
    st(h).sync();
  });
}

int qs_sample(qs_state_t h, const double* uniforms, uint64_t shots, int exact, uint64_t* out_index) {
  return guarded([&] {
    if (shots && (!uniforms || !out_index)) throw ValidationError("null sample buffers");
    sample(st(h), uniforms, shots, exact != 0, out_index);
  });
}

int qs_sample_seeded(qs_state_t h, uint64_t seed, uint64_t shots, int exact, uint64_t* out_index) {
  return guarded([&] {
    if (shots && !out_index) throw ValidationError("null sample buffer");
    // Rng(seed).uniform() stream (rng.hpp:20-46): std::mt19937_64 raw draws
    // (generated while the GPU builds the cumulative array)
    std::mt19937_64 eng(seed);
    sample_gen(st(h), shots, exact != 0, out_index, [&](double* u, uint64_t cnt) {
      for (uint64_t i = 0; i < cnt; ++i) u[i] = static_cast<double>(eng() >> 11) * 0x1.0p-53;
    });
  });
}

static void parse_pauli(const char* letters, uint32_t nterms, uint32_t n, std::vector<uint64_t>& xm,
                        std::vector<uint64_t>& sm, std::vector<int>& ny) {
  if (nterms && !letters) throw ValidationError("null Pauli letters");
  xm.assign(nterms, 0);
  sm.assign(nterms, 0);
  ny.assign(nterms, 0);
  for (uint32_t t = 0; t < nterms; ++t) {
    uint64_t x = 0, z = 0;
    int y = 0;
    for (uint32_t q = 0; q < n; ++q) {
      const char c = letters[static_cast<uint64_t>(t) * n + q];
      switch (c) {
        case 'I': break;
        case 'X': x |= 1ull << q; break;
        case 'Y': x |= 1ull << q; z |= 1ull << q; ++y; break;
        case 'Z': z |= 1ull << q; break;
        default: throw ValidationError(std::string("unknown Pauli letter '") + c + "'");
      }
    }
    xm[t] = x;
    sm[t] = z;
    ny[t] = y;
  }
}

int qs_expect_pauli(qs_state_t h, const char* letters, uint32_t nterms, double* out) {
  return guarded([&] {
    State& s = st(h);
    std::vector<uint64_t> xm, sm;
    std::vector<int> ny;
    parse_pauli(letters, nterms, s.n, xm, sm, ny);
    expect_pauli(s, xm, sm, ny, out);
  });
}

int qs_batch_reset(qs_state_t h, uint32_t shot_qubits) {
  return guarded([&] {
    batch_reset(st(h), shot_qubits);
    st(h).sync();
  });
}

int qs_batch_measure(qs_state_t h, uint32_t shot_qubits, uint32_t qubit, const double* uniforms, uint64_t shots,
                     signed char* outcomes) {
  return guarded([&] {
    if (shots && (!uniforms || !outcomes)) throw ValidationError("null batch buffers");
    batch_measure(st(h), shot_qubits, qubit, uniforms, shots, outcomes);
  });
}

int qs_batch_kraus(qs_state_t h, uint32_t shot_qubits, const uint32_t* qubits, uint32_t k, const double* ops,
                   uint32_t nops, const double* uniforms, uint64_t shots, int32_t* chosen) {
  return guarded([&] {
    if (!qubits || !ops || (shots && !uniforms)) throw ValidationError("null batch buffers");
    batch_kraus(st(h), shot_qubits, qubits, k, ops, nops, uniforms, shots, chosen);
  });
}

int qs_batch_apply(qs_state_t h, uint32_t shot_qubits, const uint32_t* qubits, uint32_t k, const double* matrix,
                   const signed char* mask, uint64_t shots) {
  return guarded([&] {
    if (!qubits || !matrix || (shots && !mask)) throw ValidationError("null batch buffers");
    batch_apply(st(h), shot_qubits, qubits, k, matrix, mask, shots);
  });
}

int qs_reduced_density(qs_state_t h, const uint32_t* qubits, uint32_t k, double* out) {
  return guarded([&] {
    if (!qubits || !out) throw ValidationError("null buffer");
    reduced_density(st(h), qubits, k, out);
  });
}

int qs_gradient(qs_state_t h, const qs_gate* gates, uint64_t count, const uint64_t* slots, uint64_t nslots,
                const char* letters, const double* coeffs, uint32_t nterms, double* out) {
  return guarded([&] {
    State& s = st(h);
    if ((count && !gates) || (nslots && (!slots || !out)) || (nterms && !coeffs))
      throw ValidationError("null gradient buffers");
    for (uint64_t i = 0; i < count; ++i) validate_gate(gates[i], s.n);
    std::vector<uint64_t> xm, zm;
    std::vector<int> ny;
    parse_pauli(letters, nterms, s.n, xm, zm, ny);
    gradient_adjoint(s, gates, count, slots, nslots, xm, zm, ny, coeffs, out);
  });
}

int qs_cumulative(qs_state_t h, double* cum_out, double* total_out) {
  return guarded([&] {
    State& s = st(h);
    if (!cum_out) throw ValidationError("null cumulative buffer");
    DeviceGuard dg(s.device);
    double* d = nullptr;
    if (cudaMalloc(&d, s.size * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      throw MemoryError("cannot allocate the cumulative array");
    }
    double total = 0;
    try {
      total = exact_cumulative(s, nullptr, d);
      QSB_CUDA(cudaMemcpy(cum_out, d, s.size * sizeof(double), cudaMemcpyDeviceToHost));
    } catch (...) {
      cudaFree(d);
      throw;
    }
    cudaFree(d);
    if (total_out) *total_out = total;
  });
}

int qs_dist_unique_id(unsigned char out[128]) {
  return guarded([&] {
    if (!out) throw ValidationError("null id buffer");
    dist_unique_id(out);
  });
}

int qs_dist_create(const unsigned char id[128], int world, int rank, int device, qs_dist_t* out) {
  return guarded([&] {
    if (!id || !out) throw ValidationError("null id or output handle");
    *out = nullptr;
    int ndev = 0;
    QSB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ValidationError("CUDA device " + std::to_string(device) + " not present");
    auto* h = new qs_dist();
    try {
      h->d = dist_create(id, world, rank, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int qs_partial_amplitude(uint32_t num_qubits, const qs_gate* gates, uint64_t n, const uint32_t* block_a, uint32_t na,
                         const uint64_t* targets, uint64_t ntargets, int device, uint32_t batch_qubits, double* out) {
  return guarded([&] {
    if ((n && !gates) || (na && !block_a) || (ntargets && (!targets || !out))) throw ValidationError("null argument");
    if (num_qubits > 60) throw ValidationError("partial amplitude: at most 60 qubits");
    int ndev = 0;
    QSB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ValidationError("CUDA device " + std::to_string(device) + " not present");
    partial_amplitude(num_qubits, gates, n, block_a, na, targets, ntargets, device, batch_qubits, out);
  });
}

int qs_dist_create_host(const qs_host_collectives* c, int world, int rank, int device, qs_dist_t* out) {
  return guarded([&] {
    if (!c || !out) throw ValidationError("null collectives or output handle");
    *out = nullptr;
    int ndev = 0;
    QSB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ValidationError("CUDA device " + std::to_string(device) + " not present");
    auto* h = new qs_dist();
    try {
      h->d = dist_create_host(*c, world, rank, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int qs_dist_destroy(qs_dist_t d) {
  return guarded([&] {
    if (!d) return;
    dist_destroy(d->d);
    delete d;
  });
}

static ShardSet& sh(qs_shards_t h) {
  if (!h || !h->ss) throw ValidationError("null shard handle");
  return *h->ss;
}

int qs_shards_create_local(uint32_t num_qubits, uint32_t global_qubits, int device, qs_shards_t* out) {
  return guarded([&] {
    if (!out) throw ValidationError("null output handle");
    *out = nullptr;
    if (num_qubits > 40) throw ValidationError("sharded states limited to 40 qubits");
    int ndev = 0;
    QSB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ValidationError("CUDA device " + std::to_string(device) + " not present");
    auto h = std::make_unique<qs_shards>();
    h->ss = make_local_shards(num_qubits, global_qubits, device);
    *out = h.release();
  });
}

int qs_shards_create_dist(uint32_t num_qubits, qs_dist_t d, qs_shards_t* out) {
  return guarded([&] {
    if (!out || !d) throw ValidationError("null communicator or output handle");
    *out = nullptr;
    if (num_qubits > 44) throw ValidationError("sharded states limited to 44 qubits");
    auto h = std::make_unique<qs_shards>();
    h->ss = make_dist_shard(num_qubits, d->d);
    *out = h.release();
  });
}

int qs_shards_destroy(qs_shards_t s) {
  return guarded([&] { delete s; });
}

int qs_shards_info(qs_shards_t s, uint32_t* num_qubits, uint32_t* global_qubits, uint32_t* first_rank,
                   uint32_t* local_count) {
  return guarded([&] {
    ShardSet& ss = sh(s);
    if (num_qubits) *num_qubits = ss.n;
    if (global_qubits) *global_qubits = ss.g;
    if (first_rank) *first_rank = ss.shards.front()->rank;
    if (local_count) *local_count = static_cast<uint32_t>(ss.shards.size());
  });
}

void* qs_shards_stream(qs_shards_t s) { return (s && s->ss) ? static_cast<void*>(s->ss->stream) : nullptr; }

int qs_shards_sync(qs_shards_t s) {
  return guarded([&] { shard_sync(sh(s)); });
}

int qs_shards_set_basis_state(qs_shards_t s, uint64_t index) {
  return guarded([&] {
    ShardSet& ss = sh(s);
    if (index >= (1ull << ss.n)) throw ValidationError("basis index out of range");
    shard_fill_basis(ss, index);
  });
}

int qs_shards_set_amplitudes(qs_shards_t s, const double* data, uint64_t offset, uint64_t count) {
  return guarded([&] {
    if (count && !data) throw ValidationError("null amplitude buffer");
    shard_set(sh(s), data, offset, count);
  });
}

int qs_shards_get_amplitudes(qs_shards_t s, double* data, uint64_t offset, uint64_t count) {
  return guarded([&] {
    if (count && !data) throw ValidationError("null amplitude buffer");
    shard_get(sh(s), data, offset, count);
  });
}

int qs_plan_create_sharded(uint32_t num_qubits, uint32_t global_qubits, const qs_gate* gates, uint64_t n,
                           qs_plan_t* out) {
  return guarded([&] {
    if (!out) throw ValidationError("null output handle");
    if (n && !gates) throw ValidationError("null gate array");
    auto h = std::make_unique<qs_plan>();
    h->p = make_plan(num_qubits, gates, n, QS_PLAN_TILED, 0, global_qubits, /*sharded=*/true);
    *out = h.release();
  });
}

int qs_plan_exchanges(qs_plan_t p, uint64_t* exchanges) {
  return guarded([&] {
    if (!p || !exchanges) throw ValidationError("null plan or output");
    uint64_t c = 0;
    for (const auto& st : p->p->steps) c += st.kind == Step::SwapStep;
    *exchanges = c;
  });
}

int qs_plan_tile_info(qs_plan_t p, uint64_t i, uint32_t* m, uint32_t* qubits, uint32_t* r, uint32_t* transposes,
                      uint32_t* nops, uint64_t* gates) {
  return guarded([&] {
    if (!p || i >= p->p->steps.size()) throw ValidationError("bad plan step index");
    const Step& st = p->p->steps[i];
    const TileProgram* tp = st.kind == Step::TileStep ? st.tile.get() : nullptr;
    if (m) *m = tp ? tp->h.m : 0;
    if (!tp) return;
    for (uint32_t b = 0; b < tp->h.m && qubits; ++b) qubits[b] = tp->h.S[b];
    if (r) *r = tp->h.r;
    if (transposes) *transposes = tp->transposes;
    if (nops) *nops = static_cast<uint32_t>(tp->ops.size());
    if (gates) *gates = tp->gates;
  });
}

int qs_plan_step_info(qs_plan_t p, uint64_t i, int* kind, uint32_t* nbits, uint32_t* gpos, uint32_t* lpos) {
  return guarded([&] {
    if (!p || i >= p->p->steps.size()) throw ValidationError("bad plan step index");
    const Step& st = p->p->steps[i];
    if (kind) *kind = static_cast<int>(st.kind);
    if (nbits) *nbits = static_cast<uint32_t>(st.gpos.size());
    for (size_t b = 0; b < st.gpos.size() && b < QS_MAX_EXCHANGE_BITS; ++b) {
      if (gpos) gpos[b] = st.gpos[b];
      if (lpos) lpos[b] = st.lpos[b];
    }
  });
}

int qs_shards_plan_execute_timed(qs_shards_t s, qs_plan_t p, float* step_ms) {
  return guarded([&] {
    if (!p || !step_ms) throw ValidationError("null plan or output");
    ShardSet& ss = sh(s);
    DeviceGuard dg(ss.device);
    const size_t ns = p->p->steps.size();
    std::vector<cudaEvent_t> ev(ns + 1);
    for (auto& e : ev) QSB_CUDA(cudaEventCreate(&e));
    QSB_CUDA(cudaEventRecord(ev[0], ss.stream));
    for (size_t i = 0; i < ns; ++i) {
      shard_execute(ss, *p->p, i, 1);
      QSB_CUDA(cudaEventRecord(ev[i + 1], ss.stream));
    }
    shard_sync(ss);
    for (size_t i = 0; i < ns; ++i) QSB_CUDA(cudaEventElapsedTime(&step_ms[i], ev[i], ev[i + 1]));
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

int qs_shards_plan_enqueue(qs_shards_t s, qs_plan_t p) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    shard_execute(sh(s), *p->p);
  });
}

int qs_shards_plan_enqueue_from_basis(qs_shards_t s, qs_plan_t p, uint64_t basis) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    shard_execute_from_basis(sh(s), *p->p, basis);
  });
}

int qs_shards_plan_execute(qs_shards_t s, qs_plan_t p) {
  return guarded([&] {
    if (!p) throw ValidationError("null plan");
    shard_execute(sh(s), *p->p);
    shard_sync(sh(s));
  });
}

int qs_shards_apply_circuit(qs_shards_t s, const qs_gate* gates, uint64_t n) {
  return guarded([&] {
    ShardSet& ss = sh(s);
    if (n && !gates) throw ValidationError("null gate array");
    auto p = cached_plan(ss.n, gates, n, QS_PLAN_TILED, 0, ss.g, /*sharded=*/true);
    shard_execute(ss, *p);
    shard_sync(ss);
  });
}

int qs_shards_run_circuit(qs_shards_t s, uint64_t basis, const qs_gate* gates, uint64_t n) {
  return guarded([&] {
    ShardSet& ss = sh(s);
    if (n && !gates) throw ValidationError("null gate array");
    auto p = cached_plan(ss.n, gates, n, QS_PLAN_TILED, 0, ss.g, /*sharded=*/true);
    shard_execute_from_basis(ss, *p, basis);
    shard_sync(ss);
  });
}

int qs_shards_probs(qs_shards_t s, const uint32_t* qubits, uint32_t m, double* out) {
  return guarded([&] {
    if (!out || (m && !qubits)) throw ValidationError("null buffer");
    shard_probs(sh(s), qubits, m, out);
  });
}

int qs_shards_sample(qs_shards_t s, const double* uniforms, uint64_t shots, int exact, uint64_t* out_index) {
  return guarded([&] {
    if (shots && (!uniforms || !out_index)) throw ValidationError("null sample buffers");
    shard_sample(sh(s), uniforms, shots, exact != 0, out_index);
  });
}

int qs_shards_sample_seeded(qs_shards_t s, uint64_t seed, uint64_t shots, int exact, uint64_t* out_index) {
  return guarded([&] {
    if (shots && !out_index) throw ValidationError("null sample buffer");
    std::vector<double> u(shots);  // Rng(seed).uniform() stream (rng.hpp:20-46)
    std::mt19937_64 eng(seed);
    for (uint64_t i = 0; i < shots; ++i) u[i] = static_cast<double>(eng() >> 11) * 0x1.0p-53;
    shard_sample(sh(s), u.data(), shots, exact != 0, out_index);
  });
}

int qs_shards_expect_pauli(qs_shards_t s, const char* letters, uint32_t nterms, double* out) {
  return guarded([&] {
    ShardSet& ss = sh(s);
    std::vector<uint64_t> xm, sm;
    std::vector<int> ny;
    parse_pauli(letters, nterms, ss.n, xm, sm, ny);
    shard_expect_pauli(ss, xm, sm, ny, out);
  });
}

int qs_shards_norm2(qs_shards_t s, double* out) {
  return guarded([&] {
    if (!out) throw ValidationError("null output");
    *out = shard_norm2(sh(s));
  });
}

int qs_shards_checksum(qs_shards_t s, double* out) {
  return guarded([&] {
    if (!out) throw ValidationError("null output");
    *out = shard_checksum(sh(s));
  });
}

}  // extern "C"
