// Communicators of one rank: the world, its MP group and its DP group.
//
// Two transports behind one interface:
//  * NCCL (one process per GPU, bootstrapped from a 128-byte unique id), the
//    production path; peer buffers are mapped through CUDA IPC.
//  * an in-process LocalHub (virtual ranks: several contexts in one process,
//    one host thread each, on one GPU or several), the single-process mesh
//    the reference Trainer itself runs (src/trainer.cpp:80-97, 164-257).
//    Collectives become host rendezvous; peer buffers are plain device
//    pointers (peer access enabled between distinct devices).  Every device
//    kernel -- bucketing, fused exchanges, barriers, replica sync -- is the
//    same code as on the NCCL path.
//
// The collectives here are control-plane only (buffer growth, dirty-list
// union, checkpoint agreement); the data exchanges of the step are fused
// into the producing kernels over peer memory (ctx.cu).
#pragma once

#include <nccl.h>

#include <atomic>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "common.h"

namespace s2d {

struct LocalHub {
  explicit LocalHub(uint32_t total) : T(total) {}
  const uint32_t T;
  struct Slot {
    std::mutex m;
    std::condition_variable cv;
    uint64_t gen = 0;
    uint32_t arrived = 0;
    std::vector<uint8_t> in, out;
  };
  // host all-gather of `bytes` per member among the n members of slot `key`
  // (every member passes the same n and bytes); out receives n * bytes.
  // Throws S2D_ENCCL after the rendezvous timeout.
  void allgather(uint64_t key, uint32_t n, uint32_t me, const void* in, size_t bytes, void* out);
  void claim_rank(uint32_t rank);
  void release_rank(uint32_t rank);

 private:
  Slot& slot(uint64_t key);
  std::mutex mu_;
  std::map<uint64_t, std::unique_ptr<Slot>> slots_;
  std::vector<uint8_t> claimed_;
};

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes);
  void release();
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
  ~DevBuf() { release(); }
};

struct HostBuf {  // pinned
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes);
  ~HostBuf();
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

struct Comm {
  ncclComm_t nccl = nullptr;
  std::shared_ptr<LocalHub> hub;
  uint64_t key = 0;
  uint32_t n = 1, me = 0;
  bool local() const { return hub != nullptr; }
  bool active() const { return nccl != nullptr || hub != nullptr; }
  // device-buffer collectives, stream-ordered on st (the local transport
  // drains st, exchanges on the host and copies back before returning)
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st);
  void allreduce_i32(int32_t* buf, ncclRedOp_t op, cudaStream_t st);
  // blocking host all-gather (drains st first); scratch: device bounce
  // buffer for the NCCL transport
  void host_allgather(const void* in, size_t bytes, void* out, cudaStream_t st, DevBuf& scratch);
  // blocking barrier over the members (drains st first)
  void barrier(cudaStream_t st, DevBuf& scratch);
  void destroy();
};

// Deferred frees while any in-process (LocalHub) context is alive: cudaFree /
// cudaFreeHost synchronise the whole device, which would stall behind
// another virtual rank's device barrier that waits on this host thread.  The
// memory is released once the last local context is gone.
void dev_free(void* p);
void host_free(void* p);
void local_ctx_enter();
void local_ctx_leave();

// Map every member's `mine` (collective over c): IPC handles on the NCCL
// transport (mappings appended to `opened`), raw pointers on the local one.
std::vector<void*> map_peer_buffers(Comm& c, void* mine, int device, cudaStream_t st, DevBuf& scratch,
                                    std::vector<void*>& opened);

}  // namespace s2d
