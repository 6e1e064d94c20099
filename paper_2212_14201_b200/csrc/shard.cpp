#include "shard.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "kernels.hpp"
#include "plan.hpp"
#include "tile.hpp"

namespace qsb {

namespace {

void alloc_shard(State& s, uint32_t n, uint32_t g, uint32_t rank, int device, cudaStream_t stream) {
  s.n = n;
  s.g = g;
  s.rank = rank;
  s.device = device;
  s.size = 1ull << (n - g);
  s.rank_base = static_cast<uint64_t>(rank) << (n - g);
  s.stream = stream;
  DeviceGuard dg(device);
  if (cudaMalloc(&s.amps, s.size * sizeof(double2)) != cudaSuccess) {
    cudaGetLastError();
    s.amps = nullptr;
    throw MemoryError("cannot allocate " + std::to_string(s.size * 16) + " bytes for a shard");
  }
}

void free_shard(State& s) {
  DeviceGuard dg(s.device);
  if (s.amps) cudaFree(s.amps);
  if (s.scratch) cudaFree(s.scratch);
  if (s.host_pinned) cudaFreeHost(s.host_pinned);
  s.amps = nullptr;
  s.scratch = nullptr;
  s.host_pinned = nullptr;
}

// Exchange chunk (amplitudes per direction); QSB_SHARD_CHUNK overrides (tests).
uint64_t exchange_chunk(uint64_t half) {
  uint64_t c = 1ull << 26;  // 1 GiB per direction
  if (const char* e = std::getenv("QSB_SHARD_CHUNK")) c = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  return std::min(half, c);
}

// Device staging buffer for pack/unpack exchanges (grown on demand).
struct Staging {
  double2* buf = nullptr;
  uint64_t elems = 0;  // per direction
  int device = 0;
  double2* get(uint64_t chunk, int dev) {
    if (elems < chunk) {
      release();
      device = dev;
      DeviceGuard dg(dev);
      if (cudaMalloc(&buf, 2 * chunk * sizeof(double2)) != cudaSuccess) {
        cudaGetLastError();
        buf = nullptr;
        throw MemoryError("cannot allocate exchange staging buffers");
      }
      elems = chunk;
    }
    return buf;
  }
  void release() {
    if (buf) {
      DeviceGuard dg(device);
      cudaFree(buf);
    }
    buf = nullptr;
    elems = 0;
  }
  ~Staging() { release(); }
};

struct LocalTransport : Transport {
  // staged: move halves through pack -> staging -> unpack like NcclTransport
  // (with a device copy in place of send/recv) instead of one swap kernel.
  bool staged = false;
  Staging stage;
  void exchange(std::vector<State*>& shards, uint32_t gpos, uint32_t lpos) override {
    const uint32_t bit = 1u << gpos;
    for (uint32_t r = 0; r < shards.size(); ++r) {
      if (r & bit) continue;
      State& a = *shards[r];
      State& b = *shards[r | bit];
      if (!staged) {
        swap_halves(a, b, lpos);
        continue;
      }
      // a (rank bit 0) sends its lpos=1 half, b sends its lpos=0 half
      const uint64_t half = a.size / 2;
      const uint64_t chunk = exchange_chunk(half);
      double2* ab = stage.get(chunk, a.device);
      double2* ba = ab + chunk;
      for (uint64_t off = 0; off < half; off += chunk) {
        const uint64_t c = std::min(chunk, half - off);
        pack_half(a, lpos, 1, off, c, ab);
        pack_half(b, lpos, 0, off, c, ba);
        unpack_half(a, lpos, 1, off, c, ba);
        unpack_half(b, lpos, 0, off, c, ab);
      }
    }
  }
  double sum(const std::vector<double>& v) override {
    double t = 0;
    for (double x : v) t += x;
    return t;
  }
};

// ------------------------------------------------------------------ NCCL
// Loaded at run time (the library must load on hosts without NCCL/GPUs).
using ncclComm_t = void*;
struct NcclId {
  char internal[128];
};
struct Nccl {
  void* h = nullptr;
  int (*getUniqueId)(NcclId*) = nullptr;
  int (*commInitRank)(ncclComm_t*, int, NcclId, int) = nullptr;
  int (*commDestroy)(ncclComm_t) = nullptr;
  int (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  int (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(int) = nullptr;
};
constexpr int kNcclDouble = 8;  // ncclFloat64

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    const char* env = std::getenv("QSB_NCCL_LIB");
    const char* names[] = {env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names)
      if ((n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!n.h) {
      err = "cannot load libnccl.so.2";
      return;
    }
    auto sym = [&](const char* s) { return dlsym(n.h, s); };
    n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(sym("ncclGetUniqueId"));
    n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(sym("ncclCommInitRank"));
    n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(sym("ncclCommDestroy"));
    n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
    n.groupStart = reinterpret_cast<decltype(n.groupStart)>(sym("ncclGroupStart"));
    n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(sym("ncclGroupEnd"));
    n.allGather = reinterpret_cast<decltype(n.allGather)>(sym("ncclAllGather"));
    n.errorString = reinterpret_cast<decltype(n.errorString)>(sym("ncclGetErrorString"));
  });
  if (!n.h || !n.send || !n.recv || !n.commInitRank) throw RuntimeError(err.empty() ? "incomplete libnccl" : err);
  return n;
}

void nccl_check(int r, const char* what) {
  if (r == 0) return;
  const char* s = nccl().errorString ? nccl().errorString(r) : "?";
  throw CudaError(std::string(what) + ": " + s);
}

}  // namespace

struct Dist {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
};

namespace {

struct NcclTransport : Transport {
  Dist* d;
  Staging stage;              // send + recv chunks
  double* red = nullptr;      // allgather buffer
  explicit NcclTransport(Dist* dd) : d(dd) {}
  ~NcclTransport() override {
    DeviceGuard dg(d->device);
    if (red) cudaFree(red);
  }
  void exchange(std::vector<State*>& shards, uint32_t gpos, uint32_t lpos) override {
    State& s = *shards.at(0);
    const Nccl& N = nccl();
    DeviceGuard dg(s.device);
    const int partner = static_cast<int>(s.rank ^ (1u << gpos));
    const uint32_t v = 1u - ((s.rank >> gpos) & 1u);  // half that changes hands
    const uint64_t half = s.size / 2;
    const uint64_t chunk = exchange_chunk(half);
    double2* sendb = stage.get(chunk, s.device);
    double2* recvb = sendb + chunk;
    for (uint64_t off = 0; off < half; off += chunk) {
      const uint64_t c = std::min(chunk, half - off);
      pack_half(s, lpos, v, off, c, sendb);
      nccl_check(N.groupStart(), "ncclGroupStart");
      nccl_check(N.send(sendb, 2 * c, kNcclDouble, partner, d->comm, s.stream), "ncclSend");
      nccl_check(N.recv(recvb, 2 * c, kNcclDouble, partner, d->comm, s.stream), "ncclRecv");
      nccl_check(N.groupEnd(), "ncclGroupEnd");
      unpack_half(s, lpos, v, off, c, recvb);
    }
  }
  double sum(const std::vector<double>& v) override {
    const Nccl& N = nccl();
    DeviceGuard dg(d->device);
    if (!red) QSB_CUDA(cudaMalloc(&red, (d->world + 1) * sizeof(double)));
    double mine = 0;
    for (double x : v) mine += x;
    cudaStream_t st = nullptr;
    QSB_CUDA(cudaMemcpy(red + d->world, &mine, sizeof(double), cudaMemcpyHostToDevice));
    nccl_check(N.allGather(red + d->world, red, 1, kNcclDouble, d->comm, st), "ncclAllGather");
    std::vector<double> all(d->world);
    QSB_CUDA(cudaMemcpy(all.data(), red, d->world * sizeof(double), cudaMemcpyDeviceToHost));
    double t = 0;
    for (double x : all) t += x;  // rank order
    return t;
  }
};

}  // namespace

ShardSet::~ShardSet() {
  for (auto& s : shards) {
    if (s->stream) {
      DeviceGuard dg(s->device);
      cudaStreamSynchronize(s->stream);
    }
    free_shard(*s);
  }
  tr.reset();
  if (stream && owns_stream) {
    DeviceGuard dg(device);
    cudaStreamDestroy(stream);
  }
}

std::unique_ptr<ShardSet> make_local_shards(uint32_t n, uint32_t g, int device) {
  if (g == 0 || g > 10) throw ValidationError("shard groups need 1..10 rank bits");
  if (n < g + 6) throw ValidationError("each shard needs at least 6 local qubits");
  auto ss = std::make_unique<ShardSet>();
  ss->n = n;
  ss->g = g;
  ss->device = device;
  DeviceGuard dg(device);
  QSB_CUDA(cudaStreamCreateWithFlags(&ss->stream, cudaStreamNonBlocking));
  for (uint32_t r = 0; r < (1u << g); ++r) {
    auto s = std::make_unique<State>();
    alloc_shard(*s, n, g, r, device, ss->stream);
    ss->shards.push_back(std::move(s));
  }
  auto tr = std::make_unique<LocalTransport>();
  const char* st = std::getenv("QSB_SHARD_STAGED");
  tr->staged = st && *st && *st != '0';
  ss->tr = std::move(tr);
  shard_fill_basis(*ss, 0);
  return ss;
}

void dist_unique_id(unsigned char out[128]) {
  NcclId id;
  nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

Dist* dist_create(const unsigned char id[128], int world, int rank, int device) {
  if (world < 1 || (world & (world - 1))) throw ValidationError("world size must be a power of two");
  if (rank < 0 || rank >= world) throw ValidationError("rank out of range");
  auto d = std::make_unique<Dist>();
  d->world = world;
  d->rank = rank;
  d->device = device;
  NcclId nid;
  std::memcpy(nid.internal, id, 128);
  DeviceGuard dg(device);
  nccl_check(nccl().commInitRank(&d->comm, world, nid, rank), "ncclCommInitRank");
  return d.release();
}

void dist_destroy(Dist* d) {
  if (!d) return;
  if (d->comm && nccl().commDestroy) nccl().commDestroy(d->comm);
  delete d;
}
int dist_rank(const Dist* d) { return d->rank; }
int dist_world(const Dist* d) { return d->world; }

std::unique_ptr<ShardSet> make_dist_shard(uint32_t n, Dist* d) {
  uint32_t g = 0;
  while ((1 << g) < d->world) ++g;
  if (n < g + 6) throw ValidationError("each shard needs at least 6 local qubits");
  auto ss = std::make_unique<ShardSet>();
  ss->n = n;
  ss->g = g;
  ss->device = d->device;
  DeviceGuard dg(d->device);
  QSB_CUDA(cudaStreamCreateWithFlags(&ss->stream, cudaStreamNonBlocking));
  auto s = std::make_unique<State>();
  alloc_shard(*s, n, g, static_cast<uint32_t>(d->rank), d->device, ss->stream);
  ss->shards.push_back(std::move(s));
  ss->tr = std::make_unique<NcclTransport>(d);
  shard_fill_basis(*ss, 0);
  return ss;
}

void shard_fill_basis(ShardSet& ss, uint64_t index) {
  for (auto& s : ss.shards) {
    const bool mine = (index >> s->local_qubits()) == s->rank;
    fill_basis(*s, mine ? (index & (s->size - 1)) : ~0ull);
  }
  shard_sync(ss);
}

void shard_execute(ShardSet& ss, const Plan& p, uint64_t first, uint64_t count) {
  if (p.n != ss.n || p.g != ss.g) throw ValidationError("plan was compiled for a different state shape");
  auto shards = ss.ptrs();
  const uint64_t last = std::min<uint64_t>(p.steps.size(), count == ~0ull ? p.steps.size() : first + count);
  for (uint64_t i = first; i < last; ++i) {
    const Step& st = p.steps[i];
    switch (st.kind) {
      case Step::TileStep:
        for (auto* s : shards) launch_tile(*s, *st.tile);
        break;
      case Step::OpStep:
        for (auto* s : shards) launch_op(*s, st.op);
        break;
      case Step::SwapStep: ss.tr->exchange(shards, st.gpos, st.lpos); break;
    }
  }
}

double shard_norm2(ShardSet& ss) {
  std::vector<double> v;
  for (auto& s : ss.shards) v.push_back(reduce_norm2(*s));
  return ss.tr->sum(v);
}

double shard_checksum(ShardSet& ss) {
  std::vector<double> v;
  for (auto& s : ss.shards) v.push_back(reduce_checksum(*s));
  return ss.tr->sum(v);
}

namespace {
template <class F>
void for_segments(ShardSet& ss, uint64_t offset, uint64_t count, F&& f) {
  const uint64_t total = 1ull << ss.n;
  if (offset > total || count > total - offset) throw ValidationError("amplitude range out of bounds");
  uint64_t done = 0;
  while (done < count) {
    const uint64_t gi = offset + done;
    const uint32_t r = static_cast<uint32_t>(gi >> (ss.n - ss.g));
    State* s = nullptr;
    for (auto& sh : ss.shards)
      if (sh->rank == r) s = sh.get();
    if (!s) throw ValidationError("amplitude range outside this rank's shard");
    const uint64_t li = gi & (s->size - 1);
    const uint64_t c = std::min(count - done, s->size - li);
    f(*s, li, c, done);
    done += c;
  }
}
}  // namespace

void shard_get(ShardSet& ss, double* out, uint64_t offset, uint64_t count) {
  for_segments(ss, offset, count, [&](State& s, uint64_t li, uint64_t c, uint64_t done) {
    DeviceGuard dg(s.device);
    QSB_CUDA(cudaMemcpyAsync(out + 2 * done, s.amps + li, c * sizeof(double2), cudaMemcpyDeviceToHost, s.stream));
  });
  shard_sync(ss);
}

void shard_set(ShardSet& ss, const double* in, uint64_t offset, uint64_t count) {
  for_segments(ss, offset, count, [&](State& s, uint64_t li, uint64_t c, uint64_t done) {
    DeviceGuard dg(s.device);
    QSB_CUDA(cudaMemcpyAsync(s.amps + li, in + 2 * done, c * sizeof(double2), cudaMemcpyHostToDevice, s.stream));
  });
  shard_sync(ss);
}

void shard_sync(ShardSet& ss) {
  DeviceGuard dg(ss.device);
  QSB_CUDA(cudaStreamSynchronize(ss.stream));
}

}  // namespace qsb
