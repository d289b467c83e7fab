// Shared device helpers: complex float2 arithmetic, the fixed-point transfer
// phase, and deterministic fp64 block reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HD __device__ __forceinline__

// Checked build (make checked -> libholo_b200_checked.so, -DHOLO_CHECKS): the
// kernels test their global indices, tensor-copy boxes and region frames
// against the buffers' bounds and record violations as bits in a per-file
// device word (no trap: the run completes and holo_debug_checks reports);
// the prox poisons its shared memory with NaN before use and the engine fills
// fresh device buffers with 0xFF (NaN), so a value read from a never-written
// slot or allocation reaches the output as NaN.  compute-sanitizer is closed
// on the GPU pool this was built on; this is the substitute.  The normal build
// compiles all of it away.
enum HoloCheckBit : unsigned {
  CK_PROX_FRAME = 1u << 0,   // a strip-prox region frame outside its plane
  CK_PROX_STORE = 1u << 1,   // x_new / partial / multi-pass state index out of range
  CK_ROWS = 1u << 2,         // row-pass index out of range
  CK_COLS = 1u << 3,         // column-pass box / index out of range
  CK_GENERIC = 1u << 4,      // generic prox index out of range
  CK_COO = 1u << 5,          // COO compaction beyond its counted total
  CK_SENSOR = 1u << 6,       // sensor / group-sum index out of range
};
#ifdef HOLO_CHECKS
static __device__ unsigned int g_holo_check = 0u;
#define HOLO_DCHECK(cond, bit)                                \
  do {                                                        \
    if (!(cond)) atomicOr(&::g_holo_check, (unsigned)(bit)); \
  } while (0)
// host side: read and clear this translation unit's word
#define HOLO_CHECK_TU(fn)                                                              \
  unsigned fn() {                                                                      \
    unsigned v = 0, z = 0;                                                             \
    cudaMemcpyFromSymbol(&v, ::g_holo_check, sizeof(v));                               \
    cudaMemcpyToSymbol(::g_holo_check, &z, sizeof(z));                                 \
    return v;                                                                          \
  }
#else
#define HOLO_DCHECK(cond, bit) \
  do {                         \
  } while (0)
#define HOLO_CHECK_TU(fn) \
  unsigned fn() { return 0u; }
#endif

namespace holo {

// checked build: fill this block's dynamic shared memory with NaN (then a
// CTA barrier) so a read of a never-written slot shows up in the output
HD void poison_dyn_smem() {
#ifdef HOLO_CHECKS
  extern __shared__ __align__(16) float4 holo_poison_smem[];
  unsigned bytes;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(bytes));
  const float nan = __int_as_float(0x7fffffff);
  for (unsigned i = threadIdx.x; i < bytes / 16u; i += blockDim.x) holo_poison_smem[i] = make_float4(nan, nan, nan, nan);
  __syncthreads();
#endif
}


// Packed fp32x2 arithmetic (sm_100 FADD2/FMUL2/FFMA2): one instruction
// updates a (re, im) pair, used where both parts follow the same formula.
HD unsigned long long pk2(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
HD float2 upk2(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
HD float2 add2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
HD float2 sub2(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
HD float2 mul2(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
// a * b + c
HD float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
  return upk2(d);
}
HD float2 splat2(float a) { return make_float2(a, a); }

// complex helpers on packed pairs
HD float2 cadd(float2 a, float2 b) { return add2(a, b); }
HD float2 csub(float2 a, float2 b) { return sub2(a, b); }
// a * b = a.x (b) + a.y (-b.y, b.x)
HD float2 cmul(float2 a, float2 b) { return fma2(splat2(a.y), make_float2(-b.y, b.x), mul2(splat2(a.x), b)); }
// a * conj(b) = a.x (b.x, -b.y) + a.y (b.y, b.x)
HD float2 cmulc(float2 a, float2 b) { return fma2(splat2(a.y), make_float2(b.y, b.x), mul2(splat2(a.x), make_float2(b.x, -b.y))); }
HD float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
HD float2 cscale(float2 a, float s) { return mul2(a, splat2(s)); }
HD float2 czero() { return make_float2(0.f, 0.f); }

// single-instruction MUFU approximations (rel. error ~2^-22), no IEEE slow paths
HD float rsqrt_a(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
HD float sqrt_a(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// exp(2*pi*i * ph / 2^64).  ph is the transfer phase in cycles as a 64-bit
// binary fraction, so "mod 1" is free integer wrap-around.  The top 8 bits
// index a 256-entry unit-circle table (fp64-exact entries); the remaining
// < 2^-8 cycle is a short Taylor rotation (|theta| < 0.0246 rad, truncation
// error < 1e-10).  Max error vs exact ~2 ulp of fp32.
HD float2 cis_cycles(uint64_t ph, const float2* __restrict__ circle256) {
  const uint32_t c = (uint32_t)(ph >> 32);
  const float2 base = circle256[c >> 24];
  const float th = (float)(c & 0xFFFFFFu) * 1.4629180792671596e-09f;  // 2*pi / 2^32
  const float th2 = th * th;
  const float cs = fmaf(th2, fmaf(th2, 1.0f / 24.0f, -0.5f), 1.0f);
  const float sn = th * fmaf(th2, -1.0f / 6.0f, 1.0f);
  // base * (cs + i sn) = base cs + (base.y, base.x) (-sn, sn)
  return fma2(make_float2(base.y, base.x), make_float2(-sn, sn), mul2(base, splat2(cs)));
}

// Phase of plane k at one pixel in cycles as a 64-bit binary fraction:
// A + k*B (mod 2^64), A = frac(z0 q), B = frac(dz q), q = sqrt(1-(lam f)^2)/lam.
// Packed in one word: top 26 bits = A (error <= 2^-27 cycle), low 38 bits =
// B (error <= 2^-39 cycle per plane, <= 7.5e-9 cycle at k = 4096): the phase
// error is < 1e-7 rad, below the fp32 resolution of cis().
constexpr int kPhaseBBits = 38;
HD uint64_t plane_phase(uint64_t packed, int k) {
  const uint64_t A = packed & ~((1ull << kPhaseBBits) - 1ull);
  const uint64_t B = (packed & ((1ull << kPhaseBBits) - 1ull)) << (64 - kPhaseBBits);
  return A + (uint64_t)(uint32_t)k * B;
}

// Deterministic block reduction of NV doubles per thread; thread 0..NV-1 of
// warp 0 end up holding the block sums in out[] (written to global by caller).
template <int NV, int NT>
HD void block_sum(double (&v)[NV], double* __restrict__ dst) {
  static_assert(NT % 32 == 0, "block must be whole warps");
  constexpr int NW = NT / 32;
  __shared__ double red[NW][NV];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    v[i] = x;
  }
  __syncthreads();  // red[] may be reused by a previous call
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[w][i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < NW; ++k) s += red[k][threadIdx.x];
    dst[threadIdx.x] = s;
  }
}

}  // namespace holo
