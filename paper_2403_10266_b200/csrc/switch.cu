// switch.cu — byte-movement kernels of the dynamic switch (§3.1) and of
// split / gather: a strided run copy (pack / unpack), the P2P direct-put over NVLink
// peer mappings, and a signal-pad barrier.  All moves are 16-B vectorised and
// coalesced: every run is Sn*C*elem contiguous bytes (SURVEY §8a "The switch as an
// exact index map"), so no shared-memory transpose is needed.
#include "dsp_internal.h"
#include "sm100.cuh"

namespace dsp {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// run index (((i0*n1 + i1)*n2 + i2)*n3 + i3) = blockIdx.y + k*gridDim.y; blockIdx.x strides over
// the run's 16-B vectors.
__global__ void __launch_bounds__(kThreads) run_copy_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                            RunCopy rc, PeerPtrs peers, int use_peers, int64_t peer_off) {
  griddep_wait();
  griddep_launch_dependents();
  const int64_t runs = rc.n[0] * rc.n[1] * rc.n[2] * rc.n[3];
  const int64_t nv = rc.run_bytes / 16;
  const int64_t step = (int64_t)gridDim.x * kThreads * kUnroll;
  for (int64_t run = blockIdx.y; run < runs; run += gridDim.y) {
    const int64_t i3 = run % rc.n[3];
    const int64_t i2 = (run / rc.n[3]) % rc.n[2];
    const int64_t i1 = (run / (rc.n[3] * rc.n[2])) % rc.n[1];
    const int64_t i0 = run / (rc.n[3] * rc.n[2] * rc.n[1]);
    const uint4* s = reinterpret_cast<const uint4*>(src + i0 * rc.ss[0] + i1 * rc.ss[1] + i2 * rc.ss[2] + i3 * rc.ss[3]);
    uint8_t* dbase = use_peers ? static_cast<uint8_t*>(peers.p[i0]) + peer_off : dst + i0 * rc.ds[0];
    uint4* d = reinterpret_cast<uint4*>(dbase + i1 * rc.ds[1] + i2 * rc.ds[2] + i3 * rc.ds[3]);
    for (int64_t v0 = (int64_t)blockIdx.x * kThreads * kUnroll + threadIdx.x; v0 < nv; v0 += step) {
      uint4 buf[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t v = v0 + u * kThreads;
        if (v < nv) buf[u] = ld_stream(s + v);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t v = v0 + u * kThreads;
        if (v < nv) st_stream(d + v, buf[u]);
      }
    }
  }
}

// Signal-pad barrier across `world` ranks (one block, one thread per peer):
// release-store `epoch` into slot [rank] of every peer's pad, then acquire-spin until
// every peer has written >= epoch into our own pad.  Bounded spin: a peer that never
// arrives (dead rank, mismatched collective sequence) traps the kernel -- a CUDA error on
// the stream instead of a hang or a switch that silently proceeds without the peer's data.
__global__ void p2p_barrier_kernel(PeerPtrs signals, int rank, int world, uint64_t epoch) {
  griddep_wait();
  const int i = threadIdx.x;
  if (i < world) {
    __threadfence_system();
    uint64_t* remote = static_cast<uint64_t*>(signals.p[i]) + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(remote), "l"(epoch) : "memory");
    const uint64_t* mine = static_cast<const uint64_t*>(signals.p[rank]) + i;
    uint64_t v = 0;
    for (long spin = 0; spin < (1L << 26); ++spin) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
      if (v >= epoch) break;
      __nanosleep(64);
    }
    if (v < epoch) __trap();
  }
  __syncthreads();
}

}  // namespace

static cudaError_t launch_copy(const void* src, void* dst, const RunCopy& rc, const PeerPtrs& peers, int use_peers,
                               int64_t peer_off, int num_sms, cudaStream_t st) {
  const int64_t runs = rc.n[0] * rc.n[1] * rc.n[2] * rc.n[3];
  if (runs == 0 || rc.run_bytes == 0) return cudaSuccess;
  if (rc.run_bytes % 16) return cudaErrorInvalidValue;
  const int64_t nv = rc.run_bytes / 16;
  int64_t bx = (nv + kThreads * kUnroll - 1) / (kThreads * kUnroll);
  const int64_t want = (int64_t)num_sms * 8;  // ~8 resident CTAs per SM in total
  int64_t cap = (want + runs - 1) / runs;
  if (cap < 1) cap = 1;
  if (bx > cap) bx = cap;
  const int64_t gy = runs < 65535 ? runs : 65535;  // runs beyond gridDim.y are strided over
  dim3 grid((unsigned)bx, (unsigned)gy);
  return launch_k(run_copy_kernel, grid, dim3(kThreads), 0, st, 1, static_cast<const uint8_t*>(src),
                  static_cast<uint8_t*>(dst), rc, peers, use_peers, peer_off);
}

cudaError_t launch_run_copy(const void* src, void* dst, const RunCopy& rc, int num_sms, cudaStream_t st) {
  PeerPtrs none{};
  return launch_copy(src, dst, rc, none, 0, 0, num_sms, st);
}

cudaError_t launch_p2p_put(const void* src, const PeerPtrs& peer_base, int64_t dst_off, const RunCopy& rc, int num_sms,
                           cudaStream_t st) {
  return launch_copy(src, nullptr, rc, peer_base, 1, dst_off, num_sms, st);
}

cudaError_t launch_p2p_barrier(const PeerPtrs& signals, int rank, int world, uint64_t epoch, cudaStream_t st) {
  return launch_k(p2p_barrier_kernel, dim3(1), dim3(32), 0, st, 1, signals, rank, world, epoch);
}

}  // namespace dsp
