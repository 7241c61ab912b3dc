// Communicator transports (comm.h): NCCL across processes, LocalHub for
// virtual ranks inside one process.
#include "comm.h"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ctx.h"

namespace s2d {

// ---- device / pinned buffers ------------------------------------------------

namespace {
std::atomic<int> g_local_ctxs{0};
std::mutex g_grave_mu;
std::vector<std::pair<void*, bool>> g_grave;  // (pointer, pinned host)

int hub_timeout_ms() {
  static const int ms = [] {
    const char* e = std::getenv("S2D_HUB_TIMEOUT_MS");
    return e ? std::max(1000, std::atoi(e)) : 120000;
  }();
  return ms;
}
}  // namespace

void dev_free(void* p) {
  if (!p) return;
  if (g_local_ctxs.load() > 0) {
    std::lock_guard<std::mutex> lk(g_grave_mu);
    g_grave.push_back({p, false});
    return;
  }
  cudaFree(p);
}

void host_free(void* p) {
  if (!p) return;
  if (g_local_ctxs.load() > 0) {
    std::lock_guard<std::mutex> lk(g_grave_mu);
    g_grave.push_back({p, true});
    return;
  }
  cudaFreeHost(p);
}

void local_ctx_enter() { g_local_ctxs.fetch_add(1); }

void local_ctx_leave() {
  if (g_local_ctxs.fetch_sub(1) != 1) return;
  std::vector<std::pair<void*, bool>> g;
  {
    std::lock_guard<std::mutex> lk(g_grave_mu);
    g.swap(g_grave);
  }
  for (auto& [p, host] : g) {
    if (host)
      cudaFreeHost(p);
    else
      cudaFree(p);
  }
}

void DevBuf::ensure(size_t bytes) {
  if (bytes <= cap && p) return;
  release();
  size_t want = std::max<size_t>(bytes + bytes / 8, 256);
  S2D_CUDA(cudaMalloc(&p, want));
  cap = want;
}

void DevBuf::release() {
  dev_free(p);
  p = nullptr;
  cap = 0;
}

void HostBuf::ensure(size_t bytes) {
  if (bytes <= cap && p) return;
  host_free(p);
  p = nullptr;
  S2D_CUDA(cudaMallocHost(&p, std::max<size_t>(bytes, 256)));
  cap = std::max<size_t>(bytes, 256);
}

HostBuf::~HostBuf() { host_free(p); }

void set_max_dynamic_smem_raw(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, size_t>> done;
  int dev = 0;
  S2D_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : done)
    if (e.first.first == kernel && e.first.second == dev && e.second >= bytes) return;
  S2D_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done.push_back({{kernel, dev}, bytes});
}

// ---- LocalHub ---------------------------------------------------------------

LocalHub::Slot& LocalHub::slot(uint64_t key) {
  std::lock_guard<std::mutex> lk(mu_);
  auto& s = slots_[key];
  if (!s) s = std::make_unique<Slot>();
  return *s;
}

void LocalHub::claim_rank(uint32_t rank) {
  std::lock_guard<std::mutex> lk(mu_);
  if (rank >= T) throw Error(S2D_EINVAL, "rank out of range for the hub");
  claimed_.resize(T, 0);
  if (claimed_[rank]) throw Error(S2D_EINVAL, "rank " + std::to_string(rank) + " already has a context on this hub");
  claimed_[rank] = 1;
}

void LocalHub::release_rank(uint32_t rank) {
  std::lock_guard<std::mutex> lk(mu_);
  if (rank < claimed_.size()) claimed_[rank] = 0;
}

// Generation rendezvous: the last arrival publishes the gathered bytes and
// bumps the generation; `out` of a generation is replaced only when every
// member has arrived for the next one, i.e. after every member read it.
void LocalHub::allgather(uint64_t key, uint32_t n, uint32_t me, const void* in, size_t bytes, void* out) {
  Slot& s = slot(key);
  std::unique_lock<std::mutex> lk(s.m);
  if (s.arrived == 0) s.in.assign((size_t)n * bytes, 0);
  if (s.in.size() != (size_t)n * bytes) throw Error(S2D_EINVAL, "local collective size mismatch between ranks");
  if (bytes) std::memcpy(s.in.data() + (size_t)me * bytes, in, bytes);
  const uint64_t gen = s.gen;
  if (++s.arrived == n) {
    s.out.swap(s.in);
    s.arrived = 0;
    ++s.gen;
    s.cv.notify_all();
  } else if (!s.cv.wait_for(lk, std::chrono::milliseconds(hub_timeout_ms()), [&] { return s.gen != gen; })) {
    --s.arrived;
    throw Error(S2D_ENCCL, "local mesh rendezvous timed out (a virtual rank stopped calling in)");
  }
  if (bytes) std::memcpy(out, s.out.data(), (size_t)n * bytes);
}

// ---- Comm ---------------------------------------------------------------------

void Comm::allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) {
  if (nccl) {
    S2D_NCCL(ncclAllGather(send, recv, bytes, ncclUint8, nccl, st));
    return;
  }
  if (!hub) throw Error(S2D_EINVAL, "communicator not initialised");
  std::vector<uint8_t> mine(bytes), all((size_t)n * bytes);
  S2D_CUDA(cudaMemcpyAsync(mine.data(), send, bytes, cudaMemcpyDeviceToHost, st));
  S2D_CUDA(cudaStreamSynchronize(st));
  hub->allgather(key, n, me, mine.data(), bytes, all.data());
  S2D_CUDA(cudaMemcpyAsync(recv, all.data(), all.size(), cudaMemcpyHostToDevice, st));
  S2D_CUDA(cudaStreamSynchronize(st));
}

void Comm::allreduce_i32(int32_t* buf, ncclRedOp_t op, cudaStream_t st) {
  if (nccl) {
    S2D_NCCL(ncclAllReduce(buf, buf, 1, ncclInt32, op, nccl, st));
    return;
  }
  if (!hub) throw Error(S2D_EINVAL, "communicator not initialised");
  int32_t mine = 0;
  std::vector<int32_t> all(n);
  S2D_CUDA(cudaMemcpyAsync(&mine, buf, 4, cudaMemcpyDeviceToHost, st));
  S2D_CUDA(cudaStreamSynchronize(st));
  hub->allgather(key, n, me, &mine, 4, all.data());
  int32_t r = all[0];
  for (uint32_t i = 1; i < n; ++i) {
    if (op == ncclSum) r += all[i];
    else if (op == ncclMin) r = std::min(r, all[i]);
    else if (op == ncclMax) r = std::max(r, all[i]);
    else throw Error(S2D_EINVAL, "unsupported local reduction");
  }
  S2D_CUDA(cudaMemcpyAsync(buf, &r, 4, cudaMemcpyHostToDevice, st));
  S2D_CUDA(cudaStreamSynchronize(st));
}

void Comm::host_allgather(const void* in, size_t bytes, void* out, cudaStream_t st, DevBuf& scratch) {
  S2D_CUDA(cudaStreamSynchronize(st));
  if (hub) {
    hub->allgather(key, n, me, in, bytes, out);
    return;
  }
  if (!nccl) throw Error(S2D_EINVAL, "communicator not initialised");
  scratch.ensure((size_t)(n + 1) * bytes + 64);
  uint8_t* d = scratch.as<uint8_t>();
  S2D_CUDA(cudaMemcpyAsync(d + (size_t)n * bytes, in, bytes, cudaMemcpyHostToDevice, st));
  S2D_NCCL(ncclAllGather(d + (size_t)n * bytes, d, bytes, ncclUint8, nccl, st));
  S2D_CUDA(cudaMemcpyAsync(out, d, (size_t)n * bytes, cudaMemcpyDeviceToHost, st));
  S2D_CUDA(cudaStreamSynchronize(st));
}

void Comm::barrier(cudaStream_t st, DevBuf& scratch) {
  uint8_t one = 1;
  std::vector<uint8_t> all(n);
  host_allgather(&one, 1, all.data(), st, scratch);
}

void Comm::destroy() {
  if (nccl) ncclCommDestroy(nccl);
  nccl = nullptr;
  hub.reset();
}

std::vector<void*> map_peer_buffers(Comm& c, void* mine, int device, cudaStream_t st, DevBuf& scratch,
                                    std::vector<void*>& opened) {
  std::vector<void*> ptr(c.n, nullptr);
  if (c.local()) {
    struct Rec {
      void* p;
      int64_t dev;
    } rec{mine, device};
    std::vector<Rec> all(c.n);
    c.host_allgather(&rec, sizeof(Rec), all.data(), st, scratch);
    for (uint32_t q = 0; q < c.n; ++q) {
      ptr[q] = all[q].p;
      if (all[q].dev != device) {  // virtual ranks on different GPUs of one process
        const cudaError_t e = cudaDeviceEnablePeerAccess((int)all[q].dev, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled)
          (void)cudaGetLastError();
        else
          S2D_CUDA(e);
      }
    }
    return ptr;
  }
  cudaIpcMemHandle_t h;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  S2D_CUDA(cudaIpcGetMemHandle(&h, mine));
  std::vector<cudaIpcMemHandle_t> all(c.n);
  c.host_allgather(&h, sizeof(h), all.data(), st, scratch);
  for (uint32_t q = 0; q < c.n; ++q) {
    if (q == c.me) {
      ptr[q] = mine;
      continue;
    }
    void* mapped = nullptr;
    S2D_CUDA(cudaIpcOpenMemHandle(&mapped, all[q], cudaIpcMemLazyEnablePeerAccess));
    ptr[q] = mapped;
    opened.push_back(mapped);
  }
  return ptr;
}

}  // namespace s2d
