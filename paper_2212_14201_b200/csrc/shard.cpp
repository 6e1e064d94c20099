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

bool alloc_alt(State& s) {
  DeviceGuard dg(s.device);
  if (cudaMalloc(&s.alt, s.size * sizeof(double2)) != cudaSuccess) {
    cudaGetLastError();
    s.alt = nullptr;
    return false;
  }
  return true;
}

void free_shard(State& s) {
  DeviceGuard dg(s.device);
  if (s.amps) cudaFree(s.amps);
  if (s.alt) cudaFree(s.alt);
  if (s.scratch) cudaFree(s.scratch);
  if (s.host_pinned) cudaFreeHost(s.host_pinned);
  s.amps = nullptr;
  s.alt = nullptr;
  s.scratch = nullptr;
  s.host_pinned = nullptr;
}

// QSB_SHARD_EXCHANGE: local sets "swap" (default) | "staged" | "peer";
// distributed sets "peer" (default, falls back to NCCL) | "nccl".
// QSB_SHARD_STAGED=1 is the older spelling of "staged".
std::string exchange_mode() {
  if (const char* e = std::getenv("QSB_SHARD_EXCHANGE")) return e;
  const char* st = std::getenv("QSB_SHARD_STAGED");
  if (st && *st && *st != '0') return "staged";
  return "";
}

// Exchange chunk (amplitudes per block and peer); QSB_SHARD_CHUNK overrides (tests).
uint64_t exchange_chunk(uint64_t block, uint32_t peers) {
  uint64_t c = (1ull << 27) / std::max<uint32_t>(1, peers);  // <= 2 GiB in flight per direction
  if (const char* e = std::getenv("QSB_SHARD_CHUNK")) c = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  return std::max<uint64_t>(1, std::min(block, c));
}

// Device staging buffer for pack/unpack exchanges (grown on demand).
struct Staging {
  double2* buf = nullptr;
  uint64_t elems = 0;
  int device = 0;
  double2* get(uint64_t want, int dev) {
    if (elems < want) {
      release();
      device = dev;
      DeviceGuard dg(dev);
      if (cudaMalloc(&buf, want * sizeof(double2)) != cudaSuccess) {
        cudaGetLastError();
        buf = nullptr;
        throw MemoryError("cannot allocate exchange staging buffers");
      }
      elems = want;
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

// Value of rank r's exchanged bits (bit i <- rank bit gpos[i]).
uint32_t rank_bits(uint32_t r, const std::vector<uint32_t>& gpos) {
  uint32_t a = 0;
  for (size_t i = 0; i < gpos.size(); ++i) a |= ((r >> gpos[i]) & 1u) << i;
  return a;
}
// r with its exchanged rank bits replaced by d.
uint32_t with_bits(uint32_t r, const std::vector<uint32_t>& gpos, uint32_t d) {
  for (size_t i = 0; i < gpos.size(); ++i) r = (r & ~(1u << gpos[i])) | (((d >> i) & 1u) << gpos[i]);
  return r;
}

struct LocalTransport : Transport {
  // swap: one swap kernel per exchanged bit and shard pair (no extra memory);
  // staged: the NCCL transport's protocol (pack block -> staging -> unpack at
  //   the peer) with device copies in place of send/recv;
  // peer: the peer-memory transport's scatter kernel into sibling shards'
  //   second buffers (needs 2x memory).
  enum Mode { Swap, Staged, Peer } mode = Swap;
  Staging stage;
  void exchange(std::vector<State*>& shards, const std::vector<uint32_t>& gpos,
                const std::vector<uint32_t>& lpos) override {
    const uint32_t k = static_cast<uint32_t>(gpos.size()), K = 1u << k;
    const uint32_t P = static_cast<uint32_t>(shards.size());
    if (mode == Peer && k <= kMaxExchangeBits) {
      for (uint32_t r = 0; r < P; ++r) {
        double2* peers[kMaxPeers];
        for (uint32_t d = 0; d < K; ++d) peers[d] = shards[with_bits(r, gpos, d)]->alt;
        scatter_exchange(*shards[r], peers, lpos.data(), k, rank_bits(r, gpos));
      }
      for (auto* s : shards) std::swap(s->amps, s->alt);
      return;
    }
    if (mode != Staged) {  // disjoint transpositions commute: one bit at a time
      for (size_t i = 0; i < gpos.size(); ++i) {
        const uint32_t bit = 1u << gpos[i];
        for (uint32_t r = 0; r < P; ++r)
          if (!(r & bit)) swap_halves(*shards[r], *shards[r | bit], lpos[i]);
      }
      return;
    }
    const uint64_t B = shards[0]->size >> k;
    const uint64_t chunk = exchange_chunk(B, K - 1);
    double2* buf = stage.get(static_cast<uint64_t>(P) * K * chunk, shards[0]->device);
    auto slot = [&](uint32_t r, uint32_t d) { return buf + (static_cast<uint64_t>(r) * K + d) * chunk; };
    for (uint64_t off = 0; off < B; off += chunk) {
      const uint64_t c = std::min(chunk, B - off);
      for (uint32_t r = 0; r < P; ++r) {
        const uint32_t a = rank_bits(r, gpos);
        for (uint32_t d = 0; d < K; ++d)
          if (d != a) pack_block(*shards[r], lpos.data(), k, d, off, c, slot(r, d));
      }
      for (uint32_t r = 0; r < P; ++r) {
        const uint32_t a = rank_bits(r, gpos);
        for (uint32_t d = 0; d < K; ++d)
          if (d != a) unpack_block(*shards[r], lpos.data(), k, d, off, c, slot(with_bits(r, gpos, d), a));
      }
    }
  }
  bool fused_exchange(std::vector<State*>& shards, const TileProgram& tp, const std::vector<uint32_t>& gpos,
                      const std::vector<uint32_t>& lpos) override {
    const uint32_t k = static_cast<uint32_t>(gpos.size());
    if (mode != Peer || k > kMaxExchangeBits) return false;
    for (uint32_t r = 0; r < shards.size(); ++r) {
      TileXchg x;
      x.k = k;
      const uint32_t a = rank_bits(r, gpos);
      for (uint32_t i = 0; i < k; ++i) {
        x.lpos[i] = lpos[i];
        if ((a >> i) & 1) x.aval |= 1ull << lpos[i];
      }
      for (uint32_t d = 0; d < (1u << k); ++d) x.peers[d] = shards[with_bits(r, gpos, d)]->alt;
      launch_tile(*shards[r], tp, nullptr, &x);
    }
    for (auto* s : shards) std::swap(s->amps, s->alt);
    return true;
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
  int (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(int) = nullptr;
};
constexpr int kNcclUint8 = 1;   // ncclUint8
constexpr int kNcclDouble = 8;  // ncclFloat64
constexpr int kNcclUint64 = 5;  // ncclUint64
constexpr int kNcclSum = 0, kNcclMax = 2, kNcclMin = 3;

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
    n.allReduce = reinterpret_cast<decltype(n.allReduce)>(sym("ncclAllReduce"));
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
  // Host collectives (qs_dist_create_host): the caller's all-gather and barrier
  // (e.g. torch.distributed over gloo) stand in for NCCL.  Needs peer memory:
  // every data movement between ranks goes through the CUDA-IPC mappings.
  qs_host_collectives host{};
  bool hosted() const { return host.allgather != nullptr; }
};

namespace {
void host_check(int rc, const char* what) {
  if (rc != 0) throw RuntimeError(std::string("host collective failed: ") + what);
}
// all-gather of `bytes` per rank (rank order) between device buffers, ordered on `st`
void coll_allgather(Dist* d, const void* dsend, void* drecv, size_t bytes, cudaStream_t st) {
  if (!d->hosted()) {
    nccl_check(nccl().allGather(dsend, drecv, bytes, kNcclUint8, d->comm, st), "ncclAllGather");
    return;
  }
  std::vector<unsigned char> hs(bytes), hr(bytes * d->world);
  QSB_CUDA(cudaMemcpyAsync(hs.data(), dsend, bytes, cudaMemcpyDeviceToHost, st));
  QSB_CUDA(cudaStreamSynchronize(st));
  host_check(d->host.allgather(d->host.ctx, hs.data(), hr.data(), bytes), "allgather");
  QSB_CUDA(cudaMemcpyAsync(drecv, hr.data(), hr.size(), cudaMemcpyHostToDevice, st));
  QSB_CUDA(cudaStreamSynchronize(st));
}
// element-wise all-reduce of `count` doubles / uint64 in place (device buffer)
template <class T, class F>
void coll_allreduce(Dist* d, T* dbuf, size_t count, int nccl_type, int nccl_op, F op, cudaStream_t st) {
  if (!d->hosted()) {
    nccl_check(nccl().allReduce(dbuf, dbuf, count, nccl_type, nccl_op, d->comm, st), "ncclAllReduce");
    return;
  }
  std::vector<T> mine(count), all(count * d->world);
  QSB_CUDA(cudaMemcpyAsync(mine.data(), dbuf, count * sizeof(T), cudaMemcpyDeviceToHost, st));
  QSB_CUDA(cudaStreamSynchronize(st));
  host_check(d->host.allgather(d->host.ctx, mine.data(), all.data(), count * sizeof(T)), "allgather");
  for (size_t i = 0; i < count; ++i) {
    T acc = all[i];
    for (int r = 1; r < d->world; ++r) acc = op(acc, all[static_cast<size_t>(r) * count + i]);  // rank order
    mine[i] = acc;
  }
  QSB_CUDA(cudaMemcpyAsync(dbuf, mine.data(), count * sizeof(T), cudaMemcpyHostToDevice, st));
  QSB_CUDA(cudaStreamSynchronize(st));
}
}  // namespace

namespace {

struct NcclTransport : Transport {
  Dist* d_;
  Staging stage;              // send + recv chunks (staged mode)
  double* red = nullptr;      // allgather / barrier buffer
  // Peer mode: every rank's two shard buffers, mapped into this process
  // (own: cudaMalloc; peers: CUDA IPC over NVLink).  cur = index of the
  // buffer holding the state (identical on all ranks: same plan).
  bool peer = false;
  std::vector<double2*> bufs[2];
  std::vector<char> opened;   // bufs[*][r] opened through IPC
  int cur = 0;
  explicit NcclTransport(Dist* dd) : d_(dd) {}
  ~NcclTransport() override { close(); }

  double* scratch() {
    DeviceGuard dg(d_->device);
    if (!red) QSB_CUDA(cudaMalloc(&red, (d_->world + 1) * sizeof(double)));
    return red;
  }
  // Stream-ordered barrier: completes on every rank only after every rank's
  // prior work on its stream (incl. remote stores) has finished.
  // Host collectives: the stream is drained first, so every store of this
  // rank (incl. remote ones over the IPC mappings) is complete before the
  // host barrier releases the other ranks.
  void stream_barrier(cudaStream_t st) {
    if (d_->hosted()) {
      QSB_CUDA(st ? cudaStreamSynchronize(st) : cudaDeviceSynchronize());
      host_check(d_->host.barrier(d_->host.ctx), "barrier");
      return;
    }
    double* r = scratch();
    nccl_check(nccl().allReduce(r, r, 1, kNcclDouble, kNcclSum, d_->comm, st), "ncclAllReduce");
  }
  void barrier() override {
    DeviceGuard dg(d_->device);
    stream_barrier(nullptr);
    QSB_CUDA(cudaDeviceSynchronize());
  }

  // Exports both buffers of this rank's shard and maps every peer's; all
  // ranks agree (allreduce-min) before peer mode is used.
  void setup_peer(State& s) {
    DeviceGuard dg(d_->device);
    const int W = d_->world;
    int ok = alloc_alt(s) ? 1 : 0;
    cudaIpcMemHandle_t h[2]{};
    if (ok && (cudaIpcGetMemHandle(&h[0], s.amps) != cudaSuccess || cudaIpcGetMemHandle(&h[1], s.alt) != cudaSuccess)) {
      cudaGetLastError();
      ok = 0;
    }
    unsigned char* dev = nullptr;
    const size_t hb = sizeof(h);
    QSB_CUDA(cudaMalloc(&dev, hb * (W + 1)));
    QSB_CUDA(cudaMemcpy(dev + hb * W, h, hb, cudaMemcpyHostToDevice));
    coll_allgather(d_, dev + hb * W, dev, hb, nullptr);
    std::vector<cudaIpcMemHandle_t> all(2 * W);
    QSB_CUDA(cudaMemcpy(all.data(), dev, hb * W, cudaMemcpyDeviceToHost));
    cudaFree(dev);
    bufs[0].assign(W, nullptr);
    bufs[1].assign(W, nullptr);
    opened.assign(W, 0);
    for (int r = 0; r < W && ok; ++r) {
      if (r == d_->rank) {
        bufs[0][r] = s.amps;
        bufs[1][r] = s.alt;
        continue;
      }
      void* p0 = nullptr;
      void* p1 = nullptr;
      if (cudaIpcOpenMemHandle(&p0, all[2 * r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        break;
      }
      if (cudaIpcOpenMemHandle(&p1, all[2 * r + 1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        cudaIpcCloseMemHandle(p0);
        ok = 0;
        break;
      }
      bufs[0][r] = static_cast<double2*>(p0);
      bufs[1][r] = static_cast<double2*>(p1);
      opened[r] = 1;
    }
    // agree on the mode
    double* r = scratch();
    double mine = ok;
    QSB_CUDA(cudaMemcpy(r, &mine, sizeof(double), cudaMemcpyHostToDevice));
    coll_allreduce(d_, r, 1, kNcclDouble, kNcclMin, [](double a, double b) { return std::min(a, b); }, nullptr);
    double all_ok = 0;
    QSB_CUDA(cudaMemcpy(&all_ok, r, sizeof(double), cudaMemcpyDeviceToHost));
    peer = all_ok > 0.5;
    if (!peer) close_peers(s);
    if (!peer && d_->hosted()) throw RuntimeError("host-collective communicator: CUDA IPC peer mapping failed");
  }
  void close_peers(State& s) {
    DeviceGuard dg(d_->device);
    for (size_t r = 0; r < opened.size(); ++r)
      if (opened[r]) {
        cudaIpcCloseMemHandle(bufs[0][r]);
        cudaIpcCloseMemHandle(bufs[1][r]);
        opened[r] = 0;
      }
    if (s.alt && !peer) {
      cudaFree(s.alt);
      s.alt = nullptr;
    }
  }
  State* owner = nullptr;
  void close() override {
    if (!d_) return;
    DeviceGuard dg(d_->device);
    if (peer && owner) {
      // no rank may free a buffer another rank still maps
      try {
        barrier();
      } catch (...) {
      }
      for (size_t r = 0; r < opened.size(); ++r)
        if (opened[r]) {
          cudaIpcCloseMemHandle(bufs[0][r]);
          cudaIpcCloseMemHandle(bufs[1][r]);
          opened[r] = 0;
        }
      try {
        barrier();
      } catch (...) {
      }
      peer = false;
    }
    if (red) cudaFree(red);
    red = nullptr;
  }

  bool fused_exchange(std::vector<State*>& shards, const TileProgram& tp, const std::vector<uint32_t>& gpos,
                      const std::vector<uint32_t>& lpos) override {
    const uint32_t k = static_cast<uint32_t>(gpos.size());
    if (!peer || k > kMaxExchangeBits) return false;
    State& s = *shards.at(0);
    DeviceGuard dg(s.device);
    TileXchg x;
    x.k = k;
    const uint32_t a = rank_bits(s.rank, gpos);
    for (uint32_t i = 0; i < k; ++i) {
      x.lpos[i] = lpos[i];
      if ((a >> i) & 1) x.aval |= 1ull << lpos[i];
    }
    for (uint32_t d = 0; d < (1u << k); ++d) x.peers[d] = bufs[cur ^ 1][with_bits(s.rank, gpos, d)];
    launch_tile(s, tp, nullptr, &x);  // stores land in the owners' free buffers over NVLink
    stream_barrier(s.stream);
    cur ^= 1;
    s.amps = bufs[cur][s.rank];
    s.alt = bufs[cur ^ 1][s.rank];
    return true;
  }

  void exchange(std::vector<State*>& shards, const std::vector<uint32_t>& gpos,
                const std::vector<uint32_t>& lpos) override {
    State& s = *shards.at(0);
    DeviceGuard dg(s.device);
    const uint32_t k = static_cast<uint32_t>(gpos.size()), K = 1u << k;
    const uint32_t a = rank_bits(s.rank, gpos);
    if (peer && k <= kMaxExchangeBits) {
      // one kernel: every amplitude straight into its owner's free buffer over NVLink
      double2* peers[kMaxPeers];
      for (uint32_t d = 0; d < K; ++d) peers[d] = bufs[cur ^ 1][with_bits(s.rank, gpos, d)];
      scatter_exchange(s, peers, lpos.data(), k, a);
      stream_barrier(s.stream);
      cur ^= 1;
      s.amps = bufs[cur][s.rank];
      s.alt = bufs[cur ^ 1][s.rank];
      return;
    }
    if (d_->hosted()) throw RuntimeError("host-collective communicators exchange over peer memory only");
    const Nccl& N = nccl();
    // All-to-all among the 2^k ranks that differ in the exchanged rank bits:
    // block d (local bits lpos = d) goes to the peer whose rank bits are d, and
    // that peer's block a (a = our rank bits) lands in our block d.
    const uint64_t B = s.size >> k;
    const uint64_t chunk = exchange_chunk(B, K - 1);
    double2* sendb = stage.get(2ull * K * chunk, s.device);
    double2* recvb = sendb + static_cast<uint64_t>(K) * chunk;
    for (uint64_t off = 0; off < B; off += chunk) {
      const uint64_t c = std::min(chunk, B - off);
      for (uint32_t d = 0; d < K; ++d)
        if (d != a) pack_block(s, lpos.data(), k, d, off, c, sendb + d * chunk);
      nccl_check(N.groupStart(), "ncclGroupStart");
      for (uint32_t d = 0; d < K; ++d) {
        if (d == a) continue;
        const int peer_rank = static_cast<int>(with_bits(s.rank, gpos, d));
        nccl_check(N.send(sendb + d * chunk, 2 * c, kNcclDouble, peer_rank, d_->comm, s.stream), "ncclSend");
        nccl_check(N.recv(recvb + d * chunk, 2 * c, kNcclDouble, peer_rank, d_->comm, s.stream), "ncclRecv");
      }
      nccl_check(N.groupEnd(), "ncclGroupEnd");
      for (uint32_t d = 0; d < K; ++d)
        if (d != a) unpack_block(s, lpos.data(), k, d, off, c, recvb + d * chunk);
    }
  }
  double sum(const std::vector<double>& v) override {
    DeviceGuard dg(d_->device);
    double* r = scratch();
    double mine = 0;
    for (double x : v) mine += x;
    QSB_CUDA(cudaMemcpy(r + d_->world, &mine, sizeof(double), cudaMemcpyHostToDevice));
    coll_allgather(d_, r + d_->world, r, sizeof(double), nullptr);
    std::vector<double> all(d_->world);
    QSB_CUDA(cudaMemcpy(all.data(), r, d_->world * sizeof(double), cudaMemcpyDeviceToHost));
    double t = 0;
    for (double x : all) t += x;  // rank order
    return t;
  }
};

}  // namespace

ShardSet::~ShardSet() {
  for (auto& s : shards)
    if (s->stream) {
      DeviceGuard dg(s->device);
      cudaStreamSynchronize(s->stream);
    }
  if (tr) tr->close();  // unmaps peer buffers (collective for distributed sets)
  for (auto& s : shards) free_shard(*s);
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
  const std::string mode = exchange_mode();
  if (mode == "staged") tr->mode = LocalTransport::Staged;
  if (mode == "peer") {
    bool ok = true;
    for (auto& s : ss->shards) ok = ok && alloc_alt(*s);
    tr->mode = ok ? LocalTransport::Peer : LocalTransport::Swap;
  }
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

Dist* dist_create_host(const qs_host_collectives& c, int world, int rank, int device) {
  if (world < 1 || (world & (world - 1))) throw ValidationError("world size must be a power of two");
  if (rank < 0 || rank >= world) throw ValidationError("rank out of range");
  if (!c.allgather || !c.barrier) throw ValidationError("host collectives need allgather and barrier callbacks");
  auto d = std::make_unique<Dist>();
  d->world = world;
  d->rank = rank;
  d->device = device;
  d->host = c;
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
  auto tr = std::make_unique<NcclTransport>(d);
  tr->owner = ss->shards[0].get();
  // peer memory (CUDA IPC over NVLink) unless disabled; collective on all ranks
  if (d->world > 1 && (exchange_mode() != "nccl" || d->hosted())) tr->setup_peer(*ss->shards[0]);
  ss->tr = std::move(tr);
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

void shard_execute(ShardSet& ss, const Plan& p, uint64_t first, uint64_t count, const uint64_t* basis,
                   TileSkip* unwritten) {
  if (p.n != ss.n || p.g != ss.g) throw ValidationError("plan was compiled for a different state shape");
  auto shards = ss.ptrs();
  auto settle = [&]() {
    if (!unwritten || !unwritten->mask) return;
    for (auto* s : shards) zero_outside(*s, unwritten->mask, unwritten->val);
    *unwritten = TileSkip{};
  };
  const uint64_t last = std::min<uint64_t>(p.steps.size(), count == ~0ull ? p.steps.size() : first + count);
  const bool fuse = [] {
    const char* e = std::getenv("QSB_FUSE_EXCHANGE");
    return !e || std::atoi(e) != 0;
  }();
  for (uint64_t i = first; i < last; ++i) {
    const Step& st = p.steps[i];
    switch (st.kind) {
      case Step::TileStep:
        // a tile pass followed by an exchange: one kernel writing over peer memory
        if (fuse && i + 1 < last && p.steps[i + 1].kind == Step::SwapStep) {
          settle();  // the fused kernel reads every tile
          if (ss.tr->fused_exchange(shards, *st.tile, p.steps[i + 1].gpos, p.steps[i + 1].lpos)) {
            ++i;
            break;
          }
        }
        if (basis) {  // a run from |basis>: skip tiles that are still provably zero
          const TileSkip k = zero_tiles(st, *basis);
          for (auto* s : shards) launch_tile(*s, *st.tile, nullptr, nullptr, &k);
          if (unwritten && unwritten->mask) *unwritten = TileSkip{k.mask, k.val};
        } else {
          for (auto* s : shards) launch_tile(*s, *st.tile);
        }
        break;
      case Step::OpStep:
        settle();
        for (auto* s : shards) launch_op(*s, st.op);
        break;
      case Step::SwapStep:
        settle();
        ss.tr->exchange(shards, st.gpos, st.lpos);
        break;
      case Step::PermStep: throw ValidationError("sharded plans restore their layout in place");
    }
  }
}

void shard_execute_from_basis(ShardSet& ss, const Plan& p, uint64_t basis) {
  if (p.n != ss.n || p.g != ss.g) throw ValidationError("plan was compiled for a different state shape");
  if (basis >> ss.n) throw ValidationError("basis index out of range");
  // Exchanges before the first pass move a basis state to another basis state:
  // start from that one instead (QFT: the qubits that receive H last start in
  // the rank slots, SURVEY 8e -- one all-to-all fewer).
  uint64_t b = basis, first = 0;
  const uint32_t nl = ss.n - ss.g;
  for (; first < p.steps.size() && p.steps[first].kind == Step::SwapStep; ++first) {
    const Step& st = p.steps[first];
    for (size_t i = 0; i < st.gpos.size(); ++i) {
      const uint32_t hi = nl + st.gpos[i], lo = st.lpos[i];
      if (((b >> hi) ^ (b >> lo)) & 1) b ^= (1ull << hi) | (1ull << lo);
    }
  }
  const bool lazy = !std::getenv("QSB_NO_LAZY_ZERO") && !std::getenv("QSB_NO_SPARSE_LOAD") &&
                           !std::getenv("QSB_NO_ZERO_SKIP") && !std::getenv("QSB_NO_TILE_COMPACT");
  TileSkip unwritten;
  if (first < p.steps.size() && p.steps[first].kind == Step::TileStep) {
    TileSkip k = zero_tiles(p.steps[first], basis);  // forms are in the submitted basis bits
    k.lazy = lazy;  // write only the tiles that can be non-zero (see execute_plan_from_basis)
    for (auto& s : ss.shards) launch_tile(*s, *p.steps[first].tile, &b, nullptr, &k);  // one shard holds |b>
    if (k.lazy) unwritten = TileSkip{k.mask, k.val};
    ++first;
  } else {
    for (auto& s : ss.shards) {
      const bool mine = (b >> s->local_qubits()) == s->rank;
      fill_basis(*s, mine ? (b & (s->size - 1)) : ~0ull);
    }
  }
  shard_execute(ss, p, first, ~0ull, &basis, &unwritten);
  if (unwritten.mask)
    for (auto& s : ss.shards) zero_outside(*s, unwritten.mask, unwritten.val);
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


// ------------------------------------------------------------ reductions
namespace {
NcclTransport* dist_of(ShardSet& ss) { return dynamic_cast<NcclTransport*>(ss.tr.get()); }

struct DevBuf {  // small device buffer freed on scope exit
  void* p = nullptr;
  int dev = 0;
  DevBuf(size_t bytes, int device) : dev(device) {
    DeviceGuard dg(device);
    if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw MemoryError("device allocation failed");
    }
  }
  ~DevBuf() {
    DeviceGuard dg(dev);
    cudaFree(p);
  }
  template <class T>
  T* as() {
    return static_cast<T*>(p);
  }
};
}  // namespace

void shard_probs(ShardSet& ss, const uint32_t* qubits, uint32_t m, double* out) {
  if (m == 0) throw ValidationError("probabilities: empty qubit subset");
  if (m > 26) throw ValidationError("probabilities: at most 26 qubits for a sharded state");
  uint64_t seen = 0;
  for (uint32_t b = 0; b < m; ++b) {
    if (qubits[b] >= ss.n) throw ValidationError("probabilities: qubit out of range");
    if ((seen >> qubits[b]) & 1) throw ValidationError("probabilities: repeated qubit");
    seen |= 1ull << qubits[b];
  }
  const uint32_t nl = ss.n - ss.g;
  std::vector<uint32_t> lq, lb;  // local qubits of the subset and their result bits
  for (uint32_t b = 0; b < m; ++b)
    if (qubits[b] < nl) {
      lq.push_back(qubits[b]);
      lb.push_back(b);
    }
  const uint64_t R = 1ull << m;
  // one full-size vector per held shard, summed in rank order
  std::vector<double> mine(R * ss.shards.size(), 0.0);
  for (size_t i = 0; i < ss.shards.size(); ++i) {
    State& s = *ss.shards[i];
    uint64_t fixed = 0;  // result bits set by this shard's rank bits
    for (uint32_t b = 0; b < m; ++b)
      if (qubits[b] >= nl && ((s.rank >> (qubits[b] - nl)) & 1)) fixed |= 1ull << b;
    double* dst = mine.data() + i * R;
    if (lq.empty()) {
      dst[fixed] = reduce_norm2(s);
      continue;
    }
    std::vector<double> loc(1ull << lq.size());
    marginal_probs(s, lq.data(), static_cast<uint32_t>(lq.size()), loc.data());
    for (uint64_t k = 0; k < loc.size(); ++k) {
      uint64_t idx = fixed;
      for (size_t j = 0; j < lq.size(); ++j)
        if ((k >> j) & 1) idx |= 1ull << lb[j];
      dst[idx] = loc[k];
    }
  }
  std::vector<double> all;
  if (NcclTransport* nt = dist_of(ss)) {
    const int W = nt->d_->world;
    DeviceGuard dg(ss.device);
    DevBuf buf(R * 8 * (W + 1), ss.device);
    double* d = buf.as<double>();
    QSB_CUDA(cudaMemcpy(d + R * W, mine.data(), R * 8, cudaMemcpyHostToDevice));
    coll_allgather(nt->d_, d + R * W, d, R * 8, nullptr);
    all.resize(R * W);
    QSB_CUDA(cudaMemcpy(all.data(), d, R * W * 8, cudaMemcpyDeviceToHost));
  } else {
    all = std::move(mine);
  }
  const size_t parts = all.size() / R;
  for (uint64_t k = 0; k < R; ++k) {
    double t = 0;
    for (size_t r = 0; r < parts; ++r) t += all[r * R + k];  // rank order
    out[k] = t;
  }
}

void shard_sample(ShardSet& ss, const double* u_host, uint64_t shots, bool exact, uint64_t* out_host) {
  if (!shots) return;
  DeviceGuard dg(ss.device);
  if (NcclTransport* nt = dist_of(ss)) {
    State& s = *ss.shards[0];
    const int W = nt->d_->world, r = nt->d_->rank;
    DevBuf small(32, ss.device);
    double* carry = small.as<double>();
    double* total = carry + 1;
    if (nt->d_->hosted()) {
      // the serial chain, one all-gather per rank: rank k scans its shard
      // continuing from rank k-1's final running sum, then publishes its own
      double* u = nullptr;
      unsigned long long* out = nullptr;
      ShardCum c{};
      double prev = 0.0, fin = 0.0;
      for (int k = 0; k < W; ++k) {
        double mine = 0.0;
        if (k == r) {
          if (r > 0) QSB_CUDA(cudaMemcpyAsync(carry, &prev, 8, cudaMemcpyHostToDevice, s.stream));
          c = shard_cumulative(s, exact, r > 0 ? carry : nullptr, shots, &u, &out);
          QSB_CUDA(cudaMemcpyAsync(&mine, c.total, 8, cudaMemcpyDeviceToHost, s.stream));
          QSB_CUDA(cudaStreamSynchronize(s.stream));
        }
        std::vector<double> all(W);
        host_check(nt->d_->host.allgather(nt->d_->host.ctx, &mine, all.data(), 8), "allgather");
        if (k + 1 == r) prev = all[k];
        if (k + 1 == W) fin = all[k];
      }
      QSB_CUDA(cudaMemcpyAsync(total, &fin, 8, cudaMemcpyHostToDevice, s.stream));
      QSB_CUDA(cudaMemcpyAsync(u, u_host, shots * 8, cudaMemcpyHostToDevice, s.stream));
      QSB_CUDA(cudaMemsetAsync(out, 0, shots * 8, s.stream));
      search_range(s, c, total, r > 0 ? carry : nullptr, r + 1 == W, u, shots, out);
      coll_allreduce(nt->d_, out, shots, kNcclUint64, kNcclMax,
                     [](unsigned long long a, unsigned long long b) { return std::max(a, b); }, s.stream);
      QSB_CUDA(cudaMemcpyAsync(out_host, out, shots * 8, cudaMemcpyDeviceToHost, s.stream));
      QSB_CUDA(cudaStreamSynchronize(s.stream));
      return;
    }
    // serial chain: rank r continues the running sum of ranks < r (bit-exact serial order)
    if (r > 0) nccl_check(nccl().recv(carry, 1, kNcclDouble, r - 1, nt->d_->comm, s.stream), "ncclRecv");
    double* u = nullptr;
    unsigned long long* out = nullptr;
    ShardCum c = shard_cumulative(s, exact, r > 0 ? carry : nullptr, shots, &u, &out);
    if (r + 1 < W) nccl_check(nccl().send(c.total, 1, kNcclDouble, r + 1, nt->d_->comm, s.stream), "ncclSend");
    nccl_check(nccl().allReduce(c.total, total, 1, kNcclDouble, kNcclMax, nt->d_->comm, s.stream), "ncclAllReduce");
    QSB_CUDA(cudaMemcpyAsync(u, u_host, shots * 8, cudaMemcpyHostToDevice, s.stream));
    QSB_CUDA(cudaMemsetAsync(out, 0, shots * 8, s.stream));
    search_range(s, c, total, r > 0 ? carry : nullptr, r + 1 == W, u, shots, out);
    nccl_check(nccl().allReduce(out, out, shots, kNcclUint64, kNcclMax, nt->d_->comm, s.stream), "ncclAllReduce");
    QSB_CUDA(cudaMemcpyAsync(out_host, out, shots * 8, cudaMemcpyDeviceToHost, s.stream));
    QSB_CUDA(cudaStreamSynchronize(s.stream));
    return;
  }
  const size_t P = ss.shards.size();
  std::vector<ShardCum> c(P);
  double* u = nullptr;
  unsigned long long* out = nullptr;
  for (size_t i = 0; i < P; ++i)
    c[i] = shard_cumulative(*ss.shards[i], exact, i ? c[i - 1].total : nullptr, i ? 0 : shots, i ? nullptr : &u,
                            i ? nullptr : &out);
  QSB_CUDA(cudaMemcpyAsync(u, u_host, shots * 8, cudaMemcpyHostToDevice, ss.stream));
  QSB_CUDA(cudaMemsetAsync(out, 0, shots * 8, ss.stream));
  for (size_t i = 0; i < P; ++i)
    search_range(*ss.shards[i], c[i], c[P - 1].total, i ? c[i - 1].total : nullptr, i + 1 == P, u, shots, out);
  QSB_CUDA(cudaMemcpyAsync(out_host, out, shots * 8, cudaMemcpyDeviceToHost, ss.stream));
  QSB_CUDA(cudaStreamSynchronize(ss.stream));
}

void shard_expect_pauli(ShardSet& ss, const std::vector<uint64_t>& xm, const std::vector<uint64_t>& zm,
                        const std::vector<int>& ny, double* out) {
  const uint32_t nl = ss.n - ss.g;
  const uint64_t lmask = (1ull << nl) - 1;
  NcclTransport* nt = dist_of(ss);
  for (size_t t = 0; t < xm.size(); ++t) {
    const uint64_t xl = xm[t] & lmask, xr = xm[t] >> nl, zl = zm[t] & lmask, zr = zm[t] >> nl;
    std::vector<double> re, im;
    for (auto& sp : ss.shards) {
      State& s = *sp;
      const double sg = (__builtin_popcountll(s.rank & zr) & 1) ? -1.0 : 1.0;
      double v[2] = {0, 0};
      if (!xr) {
        expect_pauli(s, {xl}, {zl}, {0}, v);
      } else if (!nt) {  // partner shard on this device
        const uint32_t pr = s.rank ^ static_cast<uint32_t>(xr);
        const State* partner = nullptr;
        for (auto& q : ss.shards)
          if (q->rank == pr) partner = q.get();
        pauli_cross(s, s.amps, partner->amps, s.size, xl, zl, v);
      } else if (nt->peer) {  // partner shard mapped over NVLink
        const uint32_t pr = s.rank ^ static_cast<uint32_t>(xr);
        pauli_cross(s, s.amps, nt->bufs[nt->cur][pr], s.size, xl, zl, v);
      } else {  // stream the partner's shard in aligned chunks (X maps each chunk onto itself)
        if (nt->d_->hosted()) throw RuntimeError("host-collective communicators need peer memory");
        const uint32_t pr = s.rank ^ static_cast<uint32_t>(xr);
        uint64_t C = exchange_chunk(s.size, 1);
        const uint64_t need = xl ? (1ull << (64 - __builtin_clzll(xl))) : 1;
        C = std::max(C, need);
        C = std::min<uint64_t>(C, s.size);
        double2* stg = nt->stage.get(2 * C, s.device);
        for (uint64_t off = 0; off < s.size; off += C) {
          nccl_check(nccl().groupStart(), "ncclGroupStart");
          nccl_check(nccl().send(s.amps + off, 2 * C, kNcclDouble, static_cast<int>(pr), nt->d_->comm, s.stream),
                     "ncclSend");
          nccl_check(nccl().recv(stg, 2 * C, kNcclDouble, static_cast<int>(pr), nt->d_->comm, s.stream), "ncclRecv");
          nccl_check(nccl().groupEnd(), "ncclGroupEnd");
          double w[2];
          pauli_cross(s, s.amps + off, stg, C, xl, zl, w);
          const double so = (__builtin_popcountll(off & zl) & 1) ? -1.0 : 1.0;
          v[0] += so * w[0];
          v[1] += so * w[1];
        }
      }
      re.push_back(sg * v[0]);
      im.push_back(sg * v[1]);
    }
    double r = ss.tr->sum(re), i = ss.tr->sum(im);
    for (int k = 0; k < (ny[t] & 3); ++k) {  // times i^ny
      const double r2 = -i, i2 = r;
      r = r2;
      i = i2;
    }
    out[2 * t] = r;
    out[2 * t + 1] = i;
  }
}

}  // namespace qsb
