// Forward plane-sum reduction over peer memory: the per-rank
// plane-group partial spectra are summed and reduce-scattered straight into the
// owning rank's inbox by one kernel, then each rank reduces its slice and
// all-gathers it into every rank's result buffer by a second kernel -- in place
// of sum_groups + ncclAllReduce.  Deterministic: every element is summed in
// rank order.
//
// Symmetric buffers per rank (PeerSet holds every rank's device pointers; over
// NVLink they are CUDA IPC mappings, in the in-process rank group plain
// pointers of the other engines):
//   inbox  [nranks][L] complex64  slot r <- rank r's partial of this rank's slice
//   result [nranks * L] complex64 the reduced spectrum (slice j written by rank j)
//   flags  [2][kMaxPeers] u64     epoch counters: [0][r] rank r scattered into
//                                 this rank, [1][r] rank r gathered into this rank
// Completion: each kernel ends with a threadfence reduction; the last CTA
// publishes the epoch to every rank's flag with st.release.sys, and
// k_peer_wait (one thread, ld.acquire.sys) holds the stream until all ranks'
// flags reached the epoch.  Reuse is safe because a rank scatters epoch e+1
// only after its own wait for every rank's epoch-e gather (i.e. after every
// reader of its slots finished).
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace holo {
namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Last CTA of the grid (threadfence reduction) publishes `epoch` as flag
// [which][rank] on every rank.
__device__ void publish(const PeerSet& ps, int which, unsigned long long epoch, unsigned* counter) {
  __threadfence_system();  // this CTA's stores (local and remote) before its arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    if (t == gridDim.x - 1) {  // every CTA's stores are performed
      *counter = 0u;
      __threadfence_system();
      for (int j = 0; j < ps.nranks; ++j) st_release_sys(ps.flags[j] + which * kMaxPeers + ps.rank, epoch);
    }
  }
}

// sum over plane groups + reduce-scatter: element i goes to rank i / L, slot rank
__global__ void k_peer_scatter(const float2* __restrict__ Spart, int groups, long long P, const PeerSet ps,
                               unsigned long long epoch, unsigned* counter) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (long long)gridDim.x * blockDim.x) {
    float2 s = Spart[i];
    for (int g = 1; g < groups; ++g) s = cadd(s, Spart[(long long)g * P + i]);
    const int owner = (int)(i / ps.L);
    ps.inbox[owner][(long long)ps.rank * ps.L + (i - (long long)owner * ps.L)] = s;
  }
  publish(ps, 0, epoch, counter);
}

// wait for [which][j] >= epoch for every rank j (one thread); err = 1 on timeout
__global__ void k_peer_wait(const PeerSet ps, int which, unsigned long long epoch, long long max_polls, int* err) {
  const unsigned long long* f = ps.flags[ps.rank] + which * kMaxPeers;
  for (int j = 0; j < ps.nranks; ++j) {
    long long polls = 0;
    while (ld_acquire_sys(f + j) < epoch) {
      if (++polls > max_polls) {
        *err = 1;
        return;
      }
      __nanosleep(256);
    }
  }
}

// reduce this rank's slice (rank order) + all-gather it into every result buffer
__global__ void k_peer_gather(long long P, const PeerSet ps, unsigned long long epoch, unsigned* counter) {
  __shared__ int ok;
  if (threadIdx.x == 0) {  // acquire (already satisfied: k_peer_wait ran before)
    const unsigned long long* f = ps.flags[ps.rank];
    int good = 1;
    for (int j = 0; j < ps.nranks; ++j) good &= ld_acquire_sys(f + j) >= epoch;
    ok = good;
  }
  __syncthreads();
  if (ok) {
    const float2* in = ps.inbox[ps.rank];
    const long long base = (long long)ps.rank * ps.L;
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < ps.L && base + o < P;
         o += (long long)gridDim.x * blockDim.x) {
      float2 s = in[o];
      for (int j = 1; j < ps.nranks; ++j) s = cadd(s, in[(long long)j * ps.L + o]);
      for (int k = 0; k < ps.nranks; ++k) ps.result[k][base + o] = s;
    }
  }
  publish(ps, 1, epoch, counter);
}

}  // namespace

long long peer_slice(long long P, int nranks) {
  const long long L = (P + nranks - 1) / nranks;
  return (L + 63) / 64 * 64;  // 512-byte aligned slices
}

cudaError_t peer_scatter(const float2* Spart, int groups, long long P, const PeerSet& ps, unsigned long long epoch,
                         unsigned* counter, cudaStream_t s) {
  const int threads = 256;
  const int blocks = (int)std::min<long long>((P + threads - 1) / threads, 148LL * 8);
  k_peer_scatter<<<blocks, threads, 0, s>>>(Spart, groups, P, ps, epoch, counter);
  return cudaGetLastError();
}

cudaError_t peer_wait(const PeerSet& ps, int which, unsigned long long epoch, long long max_polls, int* err,
                      cudaStream_t s) {
  k_peer_wait<<<1, 1, 0, s>>>(ps, which, epoch, max_polls, err);
  return cudaGetLastError();
}

cudaError_t peer_gather(long long P, const PeerSet& ps, unsigned long long epoch, unsigned* counter,
                        cudaStream_t s) {
  const int threads = 256;
  const int blocks = (int)std::min<long long>((ps.L + threads - 1) / threads, 148LL * 4);
  k_peer_gather<<<blocks, threads, 0, s>>>(P, ps, epoch, counter);
  return cudaGetLastError();
}

}  // namespace holo
