// Does a 2D TMA tiled load with elementStrides {2, 1} deliver every other
// float of a row (the Re or Im part of complex64 data) and complete_tx the
// number of loaded bytes?  Prints the loaded box and whether the mbarrier
// completed with expect_tx = rows * (box_inner / 2) * 4 bytes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>

__global__ void k(const __grid_constant__ CUtensorMap m, float* out, int c0, unsigned bytes, int* ok) {
  __shared__ __align__(128) float box[4 * 128];
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 4 * 128; i += blockDim.x) box[i] = -1.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(box)),
        "l"(reinterpret_cast<uint64_t>(&m)), "r"(c0), "r"(1), "r"((unsigned)__cvta_generic_to_shared(&bar))
        : "memory");
  }
  unsigned done = 0;
  for (long it = 0; it < 20000000 && !done; ++it)
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(0)
        : "memory");
  if (threadIdx.x == 0) *ok = done;
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 128; i += blockDim.x) out[i] = box[i];
}

int main() {
  const int W = 512, H = 16;  // floats per row, rows
  float h[W * H];
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < W; ++c) h[r * W + c] = r * 1000 + c;
  float *d, *o;
  int* ok;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, 4 * 128 * 4);
  cudaMalloc(&ok, 4);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m;
  const cuuint64_t dims[2] = {W, H};
  const cuuint64_t strides[1] = {W * 4};
  const cuuint32_t box[2] = {128, 4};
  const cuuint32_t estr[2] = {2, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc %d\n", (int)r);
  for (int c0 : {64, 65}) {
    for (unsigned bytes : {4u * 64u * 4u, 4u * 128u * 4u}) {
      k<<<1, 128>>>(m, o, c0, bytes, ok);
      cudaError_t e = cudaDeviceSynchronize();
      float out[4 * 128];
      int okh = 0;
      cudaMemcpy(out, o, sizeof(out), cudaMemcpyDeviceToHost);
      cudaMemcpy(&okh, ok, 4, cudaMemcpyDeviceToHost);
      printf("c0 %d expect_tx %u: err %d completed %d\n  row0:", c0, bytes, (int)e, okh);
      for (int i = 0; i < 6; ++i) printf(" %g", out[i]);
      printf(" ... [62..66]:");
      for (int i = 62; i < 67; ++i) printf(" %g", out[i]);
      printf("\n  row1 (at 64):");
      for (int i = 64; i < 68; ++i) printf(" %g", out[i]);
      printf(" row1 (at 128):");
      for (int i = 128; i < 132; ++i) printf(" %g", out[i]);
      printf("\n");
    }
  }
  return 0;
}
