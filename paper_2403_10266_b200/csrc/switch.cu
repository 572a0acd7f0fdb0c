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
    // use_peers 1: level 0 selects the DESTINATION peer (P2P put); 2: the SOURCE peer (pull, the
    // emulated all-to-all / all-gather of virtual ranks)
    const uint8_t* sbase = use_peers == 2 ? static_cast<const uint8_t*>(peers.p[i0]) + peer_off : src + i0 * rc.ss[0];
    const uint4* s = reinterpret_cast<const uint4*>(sbase + i1 * rc.ss[1] + i2 * rc.ss[2] + i3 * rc.ss[3]);
    uint8_t* dbase = use_peers == 1 ? static_cast<uint8_t*>(peers.p[i0]) + peer_off : dst + i0 * rc.ds[0];
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

// Short runs (< 4 KB, e.g. the head-group runs of the Ulysses exchange): one flat index space of
// 16-B vectors over all runs, so no thread idles on a run shorter than the CTA.
__global__ void __launch_bounds__(kThreads) run_copy_flat_kernel(const uint8_t* __restrict__ src,
                                                                 uint8_t* __restrict__ dst, RunCopy rc, PeerPtrs peers,
                                                                 int use_peers, int64_t peer_off) {
  griddep_wait();
  griddep_launch_dependents();
  const int64_t nv = rc.run_bytes / 16;
  const int64_t total = rc.n[0] * rc.n[1] * rc.n[2] * rc.n[3] * nv;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t b = (int64_t)blockIdx.x * kThreads + threadIdx.x; b < total; b += stride * kUnroll) {
    uint4 buf[kUnroll];
    uint4* dp[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t idx = b + u * stride;
      dp[u] = nullptr;
      if (idx < total) {
        const int64_t run = idx / nv, v = idx - run * nv;
        const int64_t i3 = run % rc.n[3];
        const int64_t i2 = (run / rc.n[3]) % rc.n[2];
        const int64_t i1 = (run / (rc.n[3] * rc.n[2])) % rc.n[1];
        const int64_t i0 = run / (rc.n[3] * rc.n[2] * rc.n[1]);
        const uint8_t* sb = use_peers == 2 ? static_cast<const uint8_t*>(peers.p[i0]) + peer_off : src + i0 * rc.ss[0];
        uint8_t* db = use_peers == 1 ? static_cast<uint8_t*>(peers.p[i0]) + peer_off : dst + i0 * rc.ds[0];
        buf[u] = ld_stream(reinterpret_cast<const uint4*>(sb + i1 * rc.ss[1] + i2 * rc.ss[2] + i3 * rc.ss[3]) + v);
        dp[u] = reinterpret_cast<uint4*>(db + i1 * rc.ds[1] + i2 * rc.ds[2] + i3 * rc.ds[3]) + v;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (dp[u]) st_stream(dp[u], buf[u]);
  }
}

// Signal-pad barrier across `world` ranks (one block, one thread per peer).  Pad layout
// (uint64 slots of every rank's pad): [0, kMaxPeers) = the epoch peer i last arrived at;
// kPadEpoch = this rank's own barrier counter; kPadError = first timeout record.  The epoch
// lives in DEVICE memory and is advanced by the kernel itself, so a captured CUDA graph
// replays a fresh epoch every time (a host-side counter would be frozen into the graph and
// every replayed barrier would pass at once).  Thread i release-stores the new epoch into
// slot [rank] of peer i's pad, then acquire-spins until peer i has written >= epoch into our
// slot [i].  Timeout (wall clock, %globaltimer; 0 = wait forever): the waiting thread records
// (epoch << 16 | 1 << 8 | peer) in kPadError and returns instead of trapping -- a trap would
// kill the whole CUDA context; dsp_ctx_check_errors() reports the record to the host.
__global__ void p2p_barrier_kernel(PeerPtrs signals, int rank, int world, uint64_t timeout_ns) {
  griddep_wait();
  __shared__ uint64_t s_epoch;
  uint64_t* pad = static_cast<uint64_t*>(signals.p[rank]);
  if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile uint64_t*>(pad + kPadEpoch) + 1;
  __syncthreads();
  const uint64_t epoch = s_epoch;
  const int i = threadIdx.x;
  if (i < world) {
    __threadfence_system();
    uint64_t* remote = static_cast<uint64_t*>(signals.p[i]) + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(remote), "l"(epoch) : "memory");
    const uint64_t* mine = pad + i;
    uint64_t v = 0, t0 = 0;
    if (timeout_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
      if (v >= epoch) break;
      if (timeout_ns) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) {
          atomicCAS(reinterpret_cast<unsigned long long*>(pad + kPadError), 0ull,
                    (unsigned long long)((epoch << 16) | (1u << 8) | (unsigned)i));
          break;
        }
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) pad[kPadEpoch] = epoch;  // read by the next barrier in stream order
}

}  // namespace

static cudaError_t launch_copy(const void* src, void* dst, const RunCopy& rc, const PeerPtrs& peers, int use_peers,
                               int64_t peer_off, int num_sms, cudaStream_t st) {
  const int64_t runs = rc.n[0] * rc.n[1] * rc.n[2] * rc.n[3];
  if (runs == 0 || rc.run_bytes == 0) return cudaSuccess;
  if (rc.run_bytes % 16) return cudaErrorInvalidValue;
  const int64_t nv = rc.run_bytes / 16;
  if (nv < 256) {  // short runs: flat vector index space, ~8 resident CTAs per SM
    const int64_t total = runs * nv;
    int64_t blocks = (total + kThreads * kUnroll - 1) / (kThreads * kUnroll);
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    return launch_k(run_copy_flat_kernel, dim3((unsigned)blocks), dim3(kThreads), 0, st, 1,
                    static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), rc, peers, use_peers, peer_off);
  }
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

cudaError_t launch_p2p_pull(const PeerPtrs& peer_base, int64_t src_off, void* dst, const RunCopy& rc, int num_sms,
                            cudaStream_t st) {
  return launch_copy(nullptr, dst, rc, peer_base, 2, src_off, num_sms, st);
}

cudaError_t launch_p2p_barrier(const PeerPtrs& signals, int rank, int world, uint64_t timeout_ns, cudaStream_t st) {
  return launch_k(p2p_barrier_kernel, dim3(1), dim3(32), 0, st, 1, signals, rank, world, timeout_ns);
}

}  // namespace dsp
