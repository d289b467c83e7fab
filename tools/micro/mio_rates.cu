// Throughput of the MIO-side operations a column FFT exchange can use on
// sm_100a: SHFL.BFLY (32-bit), LDS.64 / STS.64 (conflict-free, 256 B per warp),
// LDS.128 (512 B per warp).  One CTA per SM, 8 independent operations per
// thread per loop trip; prints cycles per warp-instruction per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  __shared__ __align__(16) float sm[1024 * 8];
  for (int i = threadIdx.x; i < 1024 * 8; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 7;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + (w * 32 + lane) * 8;
  const unsigned base16 = (unsigned)__cvta_generic_to_shared(sm) + (w * 32 + lane) * 16;
  float a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; b[i] = 0.f; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("shfl.sync.bfly.b32 %0, %0, 1, 0x1f, -1;" : "+f"(a[i]));
      const unsigned rot = (it & 7) << 8;  // the addresses move every trip
      if (MODE == 1) {
        float x, y;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"((base + i * 2048 + rot) & 0x7fff));
        a[i] += x; b[i] += y;
      }
      if (MODE == 2) asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"((base + i * 2048 + rot) & 0x7fff), "f"(a[i]), "f"(b[i]));
      if (MODE == 3) {
        float x, y, z, u;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(u) : "r"((base16 + i * 4096 + 2 * rot) & 0x7fff));
        a[i] += x + z; b[i] += y + u;
      }
      if (MODE == 5) {  // exchange: STS.64 then LDS.64 of another warp-slot
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"((base + i * 2048 + rot) & 0x7fff), "f"(a[i]), "f"(b[i]));
        float x, y;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"((base + i * 2048 + rot + 4096) & 0x7fff));
        a[i] += x; b[i] += y;
      }
      if (MODE == 6) asm volatile("st.shared.v4.f32 [%0], {%1, %2, %1, %2};" ::"r"((base16 + i * 4096 + 2 * rot) & 0x7fff), "f"(a[i]), "f"(b[i]));
      if (MODE == 4) {  // one float2 exchange by shuffle: two SHFL
        asm volatile("shfl.sync.bfly.b32 %0, %0, 1, 0x1f, -1;" : "+f"(a[i]));
        asm volatile("shfl.sync.bfly.b32 %0, %0, 1, 0x1f, -1;" : "+f"(b[i]));
      }
    }
  }
  __syncthreads();  // every warp's loop inside the timed span
  long long t1 = clock64();
  float acc = 0.f;
  for (int i = 0; i < 8; ++i) acc += a[i] + b[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, sizeof(float) * 148 * 1024); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  const char* names[7] = {"SHFL.BFLY b32", "LDS.64", "STS.64", "LDS.128", "2x SHFL (float2)", "STS.64+LDS.64", "STS.128"};
  for (int threads : {256, 512, 1024}) {
    for (int m = 0; m < 7; ++m) {
      auto run = [&]() {
        switch (m) { case 0: k<0><<<148, threads>>>(out, iters, cyc); break; case 1: k<1><<<148, threads>>>(out, iters, cyc); break;
          case 2: k<2><<<148, threads>>>(out, iters, cyc); break; case 3: k<3><<<148, threads>>>(out, iters, cyc); break;
          case 4: k<4><<<148, threads>>>(out, iters, cyc); break; case 5: k<5><<<148, threads>>>(out, iters, cyc); break;
          default: k<6><<<148, threads>>>(out, iters, cyc); }
      };
      run(); cudaDeviceSynchronize();
      run(); cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double winst = threads / 32.0 * iters * 8 * (m == 4 || m == 5 ? 2 : 1);  // per SM
      printf("%4d threads  %-18s  %.3f cycles per warp-instruction per SM  (%.1f B/clk/SM moved)\n", threads, names[m],
             c / winst, (m == 3 || m == 6 ? 512.0 : m == 0 ? 128.0 : m == 4 ? 128.0 : 256.0) / (c / winst));
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
