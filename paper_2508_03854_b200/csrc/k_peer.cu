// Cross-GPU primitives for the fused all-to-alls over NVLink peer memory
// (CUDA IPC mappings of the MP group's receive buffers).
//
// k_peer_barrier: one warp; lane p publishes `epoch` into slot [me] of peer
// p's flag array with a system-scope release store, then waits (acquire,
// system scope) until every peer has published `epoch` into our slot [p].
// Every write this GPU made to peer memory in earlier kernels of the stream
// is ordered before the release (kernel boundary + fence.sc.sys), so after
// the barrier each rank may read what its peers wrote into its buffers.  The
// spin is bounded (~20 s) and reports a fault instead of hanging.
#include "device.cuh"

namespace s2d {
namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_peer_barrier(PeerPtrs flags, uint64_t* my_flags, uint32_t me, uint32_t n, uint64_t epoch,
                               uint32_t* err) {
  pdl_wait();  // every prior kernel (its peer stores included) completed and flushed
  const uint32_t p = threadIdx.x;
  __threadfence_system();
  if (p < n) st_release_sys(reinterpret_cast<uint64_t*>(flags.p[p]) + me, epoch);
  if (p < n) {
    const long long t0 = clock64();
    while (ld_acquire_sys(my_flags + p) < epoch) {
      if (clock64() - t0 > 40000000000ll) {  // ~20 s at 2 GHz
        atomicOr(err, kErrPeerTimeout);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncwarp();
  __threadfence_system();
}

// row `me` of every peer's count matrix: per destination owner o, (ids to o,
// partial floats for o) from the exclusive scans' block boundaries.
__global__ void k_publish_counts(const uint32_t* send_off, const uint64_t* eoff, uint32_t N, uint64_t BF,
                                 uint64_t batch, PeerPtrs xcnt, uint32_t me) {
  pdl_wait();
  const uint32_t o = threadIdx.x;
  if (o >= N) return;
  const uint64_t ids = (uint64_t)send_off[(uint64_t)(o + 1) * BF] - send_off[(uint64_t)o * BF];
  const uint64_t efl = eoff[(uint64_t)(o + 1) * BF] - eoff[(uint64_t)o * BF];
  for (uint32_t p = 0; p < N; ++p) {
    uint64_t* row = reinterpret_cast<uint64_t*>(xcnt.p[p]) + ((uint64_t)me * N + o) * 3;
    row[0] = ids;
    row[1] = efl;
    row[2] = batch;
  }
}

}  // namespace

void launch_peer_barrier(const PeerPtrs& flags, uint64_t* my_flags, uint32_t me, uint32_t n, uint64_t epoch,
                         uint32_t* err, cudaStream_t st) {
  pdl_launch(k_peer_barrier, dim3(1), dim3(32), 0, st, flags, my_flags, me, n, epoch, err);
}

void launch_publish_counts(const uint32_t* send_off, const uint64_t* eoff, uint32_t N, uint64_t BF, uint64_t batch,
                           const PeerPtrs& xcnt, uint32_t me, cudaStream_t st) {
  pdl_launch(k_publish_counts, dim3(1), dim3(32), 0, st, send_off, eoff, N, BF, batch, xcnt, me);
}

}  // namespace s2d
