// 26-connected component labelling of a sparse voxel set on the GPU
// (the connectivity step of segment.py:106-146, which the reference runs as
// a Python BFS over a dict).
//
// Input: n voxels (k, i, j) sorted lexicographically (the COO export order).
// A dense int32 index volume maps a voxel position to its id; union-find
// links every voxel to its 13 lexicographically-smaller neighbours, always
// hooking the larger root under the smaller one, so after flattening each
// voxel's root is the smallest voxel id of its component -- which is the
// component's smallest (k, i, j) voxel, the reference's emission order.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/holo_b200.h"

namespace holo {
namespace {

__global__ void k_scatter_ids(const int32_t* __restrict__ kij, long long n, int ny, int nx, int32_t* __restrict__ idx) {
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x) {
    const long long pos = ((long long)kij[3 * u] * ny + kij[3 * u + 1]) * nx + kij[3 * u + 2];
    idx[pos] = (int32_t)u;
  }
}

__device__ int32_t find_root(int32_t* parent, int32_t u) {
  while (true) {
    const int32_t p = parent[u];
    if (p == u) return u;
    const int32_t g = parent[p];
    if (g != p) atomicCAS(&parent[u], p, g);  // path halving
    u = p;
  }
}

__device__ void unite(int32_t* parent, int32_t a, int32_t b) {
  while (true) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    const int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    if (atomicCAS(&parent[hi], hi, lo) == hi) return;  // hi was still a root: hooked
    a = lo;
    b = hi;  // hi got a new parent concurrently: retry from its new root
  }
}

__global__ void k_init_parent(int32_t* __restrict__ parent, long long n) {
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x)
    parent[u] = (int32_t)u;
}

__global__ void k_link(const int32_t* __restrict__ kij, long long n, int nz, int ny, int nx,
                       const int32_t* __restrict__ idx, int32_t* __restrict__ parent) {
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x) {
    const int k = kij[3 * u], i = kij[3 * u + 1], j = kij[3 * u + 2];
    // the 13 neighbours that precede (k, i, j) lexicographically
    for (int dk = -1; dk <= 0; ++dk) {
      const int kk = k + dk;
      if (kk < 0) continue;
      for (int di = -1; di <= 1; ++di) {
        if (dk == 0 && di > 0) break;
        const int ii = i + di;
        if (ii < 0 || ii >= ny) continue;
        for (int dj = -1; dj <= 1; ++dj) {
          if (dk == 0 && di == 0 && dj >= 0) break;
          const int jj = j + dj;
          if (jj < 0 || jj >= nx) continue;
          const int32_t v = idx[((long long)kk * ny + ii) * nx + jj];
          if (v >= 0) unite(parent, (int32_t)u, v);
        }
      }
    }
  }
}

__global__ void k_flatten(int32_t* __restrict__ parent, long long n) {
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x)
    parent[u] = find_root(parent, (int32_t)u);
}

int grid_of(long long n) {
  long long g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

}  // namespace
}  // namespace holo

extern "C" int holo_label_components(const int32_t* kij, int64_t n, int32_t nz, int32_t ny, int32_t nx,
                                     int32_t* roots, void* stream) {
  if (n < 0 || nz < 1 || ny < 1 || nx < 1 || (n > 0 && (!kij || !roots))) return HOLO_ERR_INVALID;
  if (n == 0) return HOLO_OK;
  if (n > 0x7fffffffLL) return HOLO_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  const long long V = (long long)nz * ny * nx;
  int32_t* idx = nullptr;
  if (cudaMallocAsync(&idx, sizeof(int32_t) * V, s) != cudaSuccess) return HOLO_ERR_CUDA;
  cudaMemsetAsync(idx, 0xFF, sizeof(int32_t) * V, s);
  const int g = holo::grid_of(n);
  holo::k_scatter_ids<<<g, 256, 0, s>>>(kij, n, ny, nx, idx);
  holo::k_init_parent<<<g, 256, 0, s>>>(roots, n);
  holo::k_link<<<g, 256, 0, s>>>(kij, n, nz, ny, nx, idx, roots);
  holo::k_flatten<<<g, 256, 0, s>>>(roots, n);
  cudaFreeAsync(idx, s);
  return cudaGetLastError() == cudaSuccess ? HOLO_OK : HOLO_ERR_CUDA;
}
