// Throughput of packed-FP32 forms on sm_100a: FFMA2 with 3 register pairs,
// with a broadcast scalar register, with an immediate; FADD2; FFMA (scalar).
// 8 independent chains per thread, 4 warps per SMSP... prints cycles per warp-instruction per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*(unsigned long long*)&d) : "l"(*(unsigned long long*)&a), "l"(*(unsigned long long*)&b), "l"(*(unsigned long long*)&c));
  return d;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(*(unsigned long long*)&d) : "l"(*(unsigned long long*)&a), "l"(*(unsigned long long*)&b));
  return d;
}
template <int MODE>
__global__ void k(float2* out, float s, int iters, long long* cyc) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  const float2 b = make_float2(s, s * 0.5f), c = make_float2(0.25f, 0.125f), bs = make_float2(s, s);
  const float2 br = make_float2(s + threadIdx.x * 1e-9f, s * 0.5f), cr = make_float2(0.25f + threadIdx.x * 1e-9f, 0.125f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fma2(a[i], b, c);                              // 3 register pairs
      if (MODE == 1) a[i] = fma2(a[i], bs, c);                             // splat (same value both halves)
      if (MODE == 2) a[i] = fma2(a[i], make_float2(0.5f, 0.5f), c);        // immediate candidate
      if (MODE == 3) a[i] = add2(a[i], c);                                 // FADD2
      if (MODE == 4) { a[i].x = fmaf(a[i].x, s, 0.25f); a[i].y = fmaf(a[i].y, s, 0.125f); }  // 2 scalar FFMA (imm)
      if (MODE == 5) { a[i].x = fmaf(a[i].x, br.x, cr.x); a[i].y = fmaf(a[i].y, br.y, cr.y); }   // 2 scalar FFMA (reg)
      if (MODE == 6) a[i] = fma2(a[i], br, cr);                            // FFMA2 all per-thread registers
      if (MODE == 7) a[i] = add2(a[i], cr);                                // FADD2 per-thread registers
    }
  }
  __syncthreads();  // every warp's loop inside the timed span
  long long t1 = clock64();
  float2 acc = make_float2(0, 0);
  for (int i = 0; i < 8; ++i) acc = add2(acc, a[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float2* out; long long* cyc; cudaMalloc(&out, sizeof(float2) * 148 * 512 * 4); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  const char* names[8] = {"FFMA2 R,R,UR", "FFMA2 R,UR.F32,R", "FFMA2 R,imm,R", "FADD2 R,UR", "2x FFMA imm", "2x FFMA R,R,R", "FFMA2 R,R,R", "FADD2 R,R"};
  for (int threads : {512, 1024}) {
    for (int m = 0; m < 8; ++m) {
      auto run = [&]() {
        switch (m) { case 0: k<0><<<148, threads>>>(out, 1.0001f, iters, cyc); break; case 1: k<1><<<148, threads>>>(out, 1.0001f, iters, cyc); break;
          case 2: k<2><<<148, threads>>>(out, 1.0001f, iters, cyc); break; case 3: k<3><<<148, threads>>>(out, 1.0001f, iters, cyc); break;
          case 4: k<4><<<148, threads>>>(out, 1.0001f, iters, cyc); break; case 5: k<5><<<148, threads>>>(out, 1.0001f, iters, cyc); break;
          case 6: k<6><<<148, threads>>>(out, 1.0001f, iters, cyc); break; default: k<7><<<148, threads>>>(out, 1.0001f, iters, cyc); }
      };
      run(); cudaDeviceSynchronize();
      run(); cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      // warp-instructions issued per SMSP in the loop: (threads/32/4) warps x iters x 8 (x2 for the scalar pairs)
      const double winst = threads / 32.0 / 4.0 * iters * 8 * (m == 4 || m == 5 ? 2 : 1);
      printf("%4d threads  %-12s  %.2f cycles per warp-instruction per SMSP\n", threads, names[m], c / winst);
    }
  }
  return 0;
}
