// sm_100a kernels of the RIHVR fused-lasso FISTA hot path.
//
//   K1  plan tables      transfer phase (64-bit cycle fractions), band mask, twiddles
//   K2  adj_cols         column IFFT of H_k * R          (R L2-resident, H_k on the fly)
//   K3  fft_rows         row (I)FFT                        (adjoint row pass: scale 2/P)
//   K4  prox             y = (1+b)x - b x', v = y - step g, FGP-TV (re, im), guard
//                        sums, soft threshold, penalty / backtracking partial sums
//   K5  fwd_cols         column FFT * conj(H_k), deterministic z-accumulation
//   K6  sensor           R = m (S(f) + conj S(-f))/2 - FFT(b), ||r||^2 by Parseval
//   K7  coo_*            COO compaction of the final volume
//
// Reference operations replaced (see DESIGN.md for the full map):
//   optics.py:119-122, 146-169 (TransferLadder)  -> K1 + on-the-fly cis in K2/K5
//   solver.py:110-124 (forward_sparse)           -> K3 (fwd rows) + K5 + K6
//   solver.py:126-132 (gradient_chunks)          -> K6 + K2 + K3
//   solver.py:309-318, prox.py:83-148            -> K4
//   sparsevol.py:75-88 (from_dense)              -> K7
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace holo {

namespace {

constexpr int kRowThreads = 256;
// row-pass CTA size: 4 rows of 64-element threads (2 CTAs per SM by shared memory)
template <int E>
constexpr int row_threads() { return E == 64 ? 128 : kRowThreads; }

template <class F>
bool dispatch_n(int n, F&& f) {
  switch (n) {
    case 8: f(std::integral_constant<int, 8>{}); return true;
    case 16: f(std::integral_constant<int, 16>{}); return true;
    case 32: f(std::integral_constant<int, 32>{}); return true;
    case 64: f(std::integral_constant<int, 64>{}); return true;
    case 128: f(std::integral_constant<int, 128>{}); return true;
    case 256: f(std::integral_constant<int, 256>{}); return true;
    case 512: f(std::integral_constant<int, 512>{}); return true;
    case 1024: f(std::integral_constant<int, 1024>{}); return true;
    case 2048: f(std::integral_constant<int, 2048>{}); return true;
    case 4096: f(std::integral_constant<int, 4096>{}); return true;
    default: return false;
  }
}

inline int col_width(int ny) { return ny >= 4096 ? 4 : 8; }

#ifndef HOLO_ROW_E64_N
#define HOLO_ROW_E64_N 2048  // 2048-point rows: 64 x 32, one exchange instead of two
#endif
// elements per thread: 32 (one shared-memory exchange per 1024-point line)
// where registers allow; the accumulating forward column pass keeps 16
template <int N>
struct EBig {
  static constexpr int value = N == HOLO_ROW_E64_N ? 64 : N >= 512 ? 32 : DefaultE<N>::value;
};
template <int E>
constexpr int tw_slot() { return E >= 32 ? 1 : 0; }

// ------------------------------------------------------------ K1 tables ----

// per-pass twiddle tables (TwLayout): entry (r-1)*NS + kk of the pass with
// product-of-earlier-radices NS holds w = exp(-2 pi i kk r / (NS R)) as (w, conj w)
template <int N, int E>
__global__ void k_twiddles(float4* tw) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  using TL = TwLayout<N, E>;
  if (e >= TL::size()) return;
  int off = 0;
  for (int ns = E; ns < N; ns *= TL::radix(ns)) {
    const int R = TL::radix(ns), cols = TL::cols(ns), n = TL::rows(ns) * cols;
    if (e < off + n) {
      const int row = (e - off) / cols, kk = (e - off) % cols;
      const int r = TL::split(ns) ? (row < 3 ? row + 1 : 4 * (row - 2)) : row + 1;
      double sn, cs;
      sincospi(-2.0 * (double)kk * r / ((double)ns * R), &sn, &cs);
      tw[e] = make_float4((float)cs, (float)sn, (float)cs, (float)-sn);
      return;
    }
    off += n;
  }
}

__global__ void k_circle(float2* c256) {
  int m = threadIdx.x;
  double s, c;
  sincospi(2.0 * (double)m / 256.0, &s, &c);
  c256[m] = make_float2((float)c, (float)s);
}

// fftfreq(n, d)[i] = k * (1 / (n d)),  k = i for i <= (n-1)/2 else i - n   (numpy convention)
__device__ double fftfreq(int i, int n, double d) {
  const int k = (i <= (n - 1) / 2) ? i : i - n;
  return (double)k * (1.0 / ((double)n * d));
}

// frac(a) rounded to `bits` bits, as an integer in [0, 2^bits)
__device__ uint64_t frac_bits(double a, int bits) {
  double f = a - floor(a);
  uint64_t v = __double2ull_rn(f * (double)(1ull << bits));
  return v & ((1ull << bits) - 1ull);  // f rounding up to 1.0 wraps to 0 (same phase)
}

// Phase cycles of H(z) at a pixel: (z / lam) * sqrt(1 - (lam fx)^2 - (lam fy)^2)
// (optics.py:98-116).  Evanescent pixels (arg < 0) get mask 0 and phase 0.
__global__ void k_phase(uint64_t* tab, uint8_t* mask, int ny, int nx, double pitch, double lam, double z0,
                        double dz) {
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (long long)ny * nx) return;
  const int i = (int)(p / nx), j = (int)(p % nx);
  const double fy = fftfreq(i, ny, pitch), fx = fftfreq(j, nx, pitch);
  const double ax = lam * fx, ay = lam * fy;
  const double arg = 1.0 - ax * ax - ay * ay;
  const bool prop = arg >= 0.0;
  const double root = prop ? sqrt(arg) : 0.0;
  const uint64_t A = frac_bits((z0 / lam) * root, 64 - kPhaseBBits);
  const uint64_t B = frac_bits((dz / lam) * root, kPhaseBBits);
  tab[p] = (A << kPhaseBBits) | B;
  mask[p] = prop ? 1 : 0;
}

// ------------------------------------------------------------- K3 rows -----

// Shared twiddle slots of the row kernel: the compact table for 2048-point
// rows (C4 row passes 71.3 -> 65.6 ms per 5 iterations); 1024-point rows keep
// the full-size slot, i.e. 4 CTAs per SM -- at 5 (compact table) the C3 row
// passes slowed 14.45 -> 16.4 ms per 10 iterations, at 3 they are unchanged,
// at 2 they take 23.2 / 19.4.
template <int N, int E>
constexpr int row_tw_f2() {
  return N >= 2048 ? tw_f2<N, E>() : 2 * N;
}

#ifndef HOLO_ROW_PF_DIST
#define HOLO_ROW_PF_DIST 1  // row groups ahead (grid strides) prefetched into L2 (2: 14.0-15.0, 3: 15.0-15.8 ms)
#endif
template <int N, bool INV, int E_>
__global__ void __launch_bounds__(row_threads<E_>()) k_fft_rows(const float2* __restrict__ in, float2* __restrict__ out,
                                                          long long nrows, float scale, const float4* __restrict__ twg,
                                                          const uint8_t* __restrict__ live, int rpp) {
  using Sh = FftShape<N, E_>;
  constexpr int TPF = Sh::TPF, E = Sh::E;
  constexpr int RPC = row_threads<E_>() / TPF;
  extern __shared__ float2 smem[];
  poison_dyn_smem();
  float4* tw = reinterpret_cast<float4*>(smem);
  float2* buf = smem + row_tw_f2<N, E_>();
  for (int i = threadIdx.x; i < TwLayout<N, E_>::size(); i += blockDim.x) tw[i] = twg[i];
  __syncthreads();
  const int lr = threadIdx.x / TPF, j = threadIdx.x % TPF;
  for (long long row0 = (long long)blockIdx.x * RPC; row0 < nrows; row0 += (long long)gridDim.x * RPC) {
    const long long row = row0 + lr;
    bool active = row < nrows;
    if (live) {  // sparsity-aware forward (solver.py:115-119): rows of all-zero planes are skipped
      if (active && !live[(int)row / rpp]) active = false;
      if (!__syncthreads_or(active)) continue;  // the whole row group: no FFT either
    }
    float2 v[E];
    const float2* src = in + row * N + j;
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = active ? src[m * TPF] : czero();
    // the next row group (contiguous rows) into L2 while this one transforms:
    // the loads above only start once the previous group is written, and with
    // 2-4 CTAs per SM the HBM queue runs dry during the FFTs (C3 row passes
    // 14.48 -> 12.83 ms per 10 iterations, C4's 2048-point rows 26.4 -> 20.4)
    if (threadIdx.x == 0) {
      const long long nr0 = row0 + (long long)HOLO_ROW_PF_DIST * gridDim.x * RPC;
      const long long cnt = nrows - nr0 < RPC ? nrows - nr0 : RPC;
      if (nr0 < nrows && (!live || live[(int)nr0 / rpp] || live[(int)(nr0 + cnt - 1) / rpp])) {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(in + nr0 * N),
                     "r"((unsigned)(cnt * N * sizeof(float2)))
                     : "memory");
      }
    }
    fft_line<N, INV, E_>(v, j, buf + lr * Sh::PADN, 1, tw);
    if (active) {
      HOLO_DCHECK(row >= 0 && row < nrows && (!live || (int)row / rpp < (int)((nrows + rpp - 1) / rpp)), CK_ROWS);
      float2* dst = out + row * N + j;
      const float2 sc = splat2(scale);
#pragma unroll
      for (int m = 0; m < E; ++m) dst[m * TPF] = mul2(v[m], sc);
    }
  }
}

// ---------------------------------------------------------- column passes --
// Thread (j, c): column c of the CTA's C interleaved columns, FFT thread j.
// Element m of thread (j, c) is row j + m*TPF.  Lanes vary fastest in c, so a
// warp loads C-wide contiguous row segments.

template <int N, bool INV, int C, int E_>
__global__ void __launch_bounds__(C * FftShape<N, E_>::TPF) k_fft_cols(const float2* __restrict__ in,
                                                                    float2* __restrict__ out, int nx, long long P,
                                                                    float scale, const float4* __restrict__ twg) {
  using Sh = FftShape<N, E_>;
  constexpr int TPF = Sh::TPF, E = Sh::E;
  extern __shared__ float2 smem[];
  float4* tw = reinterpret_cast<float4*>(smem);
  float2* buf = smem + 2 * N;
  for (int i = threadIdx.x; i < TwLayout<N, E_>::size(); i += blockDim.x) tw[i] = twg[i];
  __syncthreads();
  const int c = threadIdx.x % C, j = threadIdx.x / C;
  const int col = blockIdx.x * C + c;
  const long long base = (long long)blockIdx.y * P + (long long)j * nx + col;
  const long long st = (long long)TPF * nx;
  float2 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = in[base + m * st];
  fft_line<N, INV, E_>(v, j, buf + c, C, tw);
#pragma unroll
  for (int m = 0; m < E; ++m) out[base + m * st] = cscale(v[m], scale);
}

template <int N, int C, int E>
constexpr bool adj_separate_stage() {
  return sizeof(float2) * (2 * N + 256 + (size_t)(N + N / E) * C + (size_t)N * C + 16) <= 227 * 1024;
}
// K2: out[k] = column-IFFT( H_{k0+k} * R ), one plane per blockIdx.y
#ifndef HOLO_ADJ_MINB
#define HOLO_ADJ_MINB 2  // 2 CTAs / 16 warps per SM at <= 128 registers (12.48 -> 12.32 ms per 10 C3 iterations)
#endif
// PK (packed real engine, see engine.cu): stack plane k holds real planes
// j = k0 + 2k (Re) and j + 1 (Im), and its weight is U_k = c_j + i c_{j+1},
// c = Re H = cos(phase), so that ifft2(U_k R) = ifft2(c_j R) + i ifft2(c_{j+1} R)
// packs the two real gradients (R Hermitian).  U_k R = rA + rB with
// rA = R H_j (1 + i G) / 2, rB = R conj(H_j) (1 + i conj G) / 2, carried from
// stack plane to stack plane by G^2 and conj(G^2).
template <int N, int C, int E_, bool PK = false>
__global__ void __launch_bounds__(C * FftShape<N, E_>::TPF, PK ? 1 : (C * FftShape<N, E_>::TPF <= 256 ? HOLO_ADJ_MINB : 1)) k_adj_cols(const float2* __restrict__ R,
                                                                    const __grid_constant__ CUtensorMap out_map,
                                                                    int nx, int ny, int k0, int nzl, int ppc,
                                                                    const uint64_t* __restrict__ tab,
                                                                    const float4* __restrict__ twg,
                                                                    const float2* __restrict__ circg) {
  using Sh = FftShape<N, E_>;
  constexpr int TPF = Sh::TPF, E = Sh::E;
  constexpr int BOX_ROWS = N < 256 ? N : 256;
  extern __shared__ __align__(128) float2 smem[];
  float4* tw = reinterpret_cast<float4*>(smem);
  float2* circ = smem + 2 * N;
  float2* buf = smem + 2 * N + 256;
  // output stage [N][C], separate from the FFT exchange buffer where it fits
  // (N <= 2048): plane k+1's transform runs while the bulk stores still read
  // plane k's stage; else the exchange buffer doubles as the stage
  constexpr bool kSep = adj_separate_stage<N, C, E_>();
  float2* stage = kSep ? buf + (((N + N / E_) * C + 15) & ~15) : buf;  // 128-byte aligned for the bulk stores
  poison_dyn_smem();
  for (int i = threadIdx.x; i < TwLayout<N, E_>::size(); i += blockDim.x) tw[i] = twg[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) circ[i] = circg[i];
  __syncthreads();
  const int c = threadIdx.x % C, j = threadIdx.x / C;
  const int col = blockIdx.x * C + c;
  const long long p0 = (long long)j * nx + col, st = (long long)TPF * nx;
  const bool leader = threadIdx.x == 0;
  // H_{k+1} = H_k * G with G = cis(2 pi dz q) per pixel: R H_k is carried from
  // plane to plane by one complex multiply (the reference's TransferLadder
  // recurrence, optics.py:146-169), exact cis() only at the CTA's first plane
  // (<= kMaxRecur steps: < 4e-6 relative drift worst case).
  const int kb = blockIdx.y * ppc, ke = min(nzl, kb + ppc);
  float2 r[E], g[E];
  float2 rb[PK ? E : 1];
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const uint64_t t = tab[p0 + m * st];
    if constexpr (PK) {
      const float2 G = cis_cycles(plane_phase(t, 1) - plane_phase(t, 0), circ);
      const float2 H = cis_cycles(plane_phase(t, k0 + 2 * kb), circ), Rv = R[p0 + m * st];
      r[m] = cmul(cmul(Rv, H), make_float2(0.5f - 0.5f * G.y, 0.5f * G.x));    // (1 + i G) / 2
      rb[m] = cmul(cmulc(Rv, H), make_float2(0.5f + 0.5f * G.y, 0.5f * G.x));  // (1 + i conj G) / 2
      g[m] = cmul(G, G);
    } else {
      r[m] = cmul(R[p0 + m * st], cis_cycles(plane_phase(t, k0 + kb), circ));
      g[m] = cis_cycles(plane_phase(t, 1) - plane_phase(t, 0), circ);
    }
  }
#ifndef HOLO_ADJ_UNROLL
#define HOLO_ADJ_UNROLL 2  // alternating register roles for r / v: 12.69 -> 12.48 ms per 10 C3 iterations
#endif
  constexpr int kUnroll = E_ >= 32 ? 1 : HOLO_ADJ_UNROLL;  // (radix-32 columns: 236 registers at 1, 254 at 2)
#pragma unroll kUnroll
  for (int k = kb; k < ke; ++k) {
    float2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) {
      if constexpr (PK) {
        v[m] = add2(r[m], rb[m]);
        rb[m] = cmulc(rb[m], g[m]);
      } else {
        v[m] = r[m];
      }
      r[m] = cmul(r[m], g[m]);
    }
    // (shared stage: the previous plane's stores must have read buf before
    // fft_line's first barrier lets anyone write it)
    if (!kSep && leader) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    fft_line<N, true, E_>(v, j, buf + c, C, tw);
    // dense [row][C] stage, then one bulk tensor store per 256 rows: the
    // column block leaves as full boxes instead of C x 8-byte row segments.
    // The previous plane's stores must have read the stage first.
    if (kSep && leader) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncthreads();  // (shared stage: the last FFT pass read buf)
#pragma unroll
    for (int m = 0; m < E; ++m) stage[(j + m * TPF) * C + c] = v[m];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (leader) {
      HOLO_DCHECK(k >= 0 && k < nzl && (blockIdx.x + 1) * C <= nx, CK_COLS);
#pragma unroll
      for (int r0 = 0; r0 < N; r0 += BOX_ROWS)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                         reinterpret_cast<uint64_t>(&out_map)),
                     "r"(2 * (int)blockIdx.x * C), "r"(k * ny + r0),
                     "r"((unsigned)__cvta_generic_to_shared(stage + r0 * C))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  if (leader) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // smem outlives the reads
}

// Horner ratio of the forward plane sum, held as z.x and the pair (-z.y, z.y)
// (acc z = swap(acc) (-z.y, z.y) + acc z.x, no sign shuffles): conj(G) for
// the complex engine; G^2 for the packed real engine (its second sum uses
// conj(G^2), i.e. the negated pair).
template <bool PK>
HD void fwd_ratio(uint64_t t, const float2* circ, float& zx, float2& zyy) {
  const float2 g = cis_cycles(plane_phase(t, 1) - plane_phase(t, 0), circ);
  if constexpr (PK) {
    const float2 g2 = cmul(g, g);
    zx = g2.x;
    zyy = make_float2(-g2.y, g2.y);
  } else {
    zx = g.x;
    zyy = make_float2(g.y, -g.y);
  }
}
// Close the forward sum of a CTA whose first stack plane is kb.  Complex:
// sum_k v_k conj(H_k) = conj(H_kb) acc.  Packed real (stack plane k = real
// planes j = k0 + 2k, j + 1; weight conj(U_k) = c_j - i c_{j+1}): with
// A = sum v G^(2(k-kb)) (acc) and B = sum v conj(G)^(2(k-kb)) (accb),
// sum_k v_k conj(U_k) = [(H_j0 - i H_j1) A + (conj H_j0 - i conj H_j1) B] / 2.
template <bool PK>
HD float2 fwd_close(float2 acc, float2 accb, uint64_t t, int k0, int kb, const float2* circ) {
  if constexpr (PK) {
    const float2 h0 = cis_cycles(plane_phase(t, k0 + 2 * kb), circ);
    const float2 h1 = cis_cycles(plane_phase(t, k0 + 2 * kb + 1), circ);
    const float2 ca = make_float2(h0.x + h1.y, h0.y - h1.x), cb = make_float2(h0.x - h1.y, -h0.y - h1.x);
    return mul2(add2(cmul(acc, ca), cmul(accb, cb)), splat2(0.5f));
  } else {
    (void)accb;
    return cmulc(acc, cis_cycles(plane_phase(t, k0 + kb), circ));
  }
}

// Horner step of an all-zero plane: acc <- acc z (+ 0), the same values as
// the full step with v = 0 (fma(a, b, 0) = a b), without loading the plane
template <bool PK, int E>
__device__ __forceinline__ void horner_zero(float2 (&acc)[E], float2 (&accb)[PK ? E : 1], const float (&zx)[E],
                                            const float2 (&zyy)[E]) {
#pragma unroll
  for (int m = 0; m < E; ++m) {
    acc[m] = fma2(swp(acc[m]), zyy[m], mul2(acc[m], splat2(zx[m])));
    if constexpr (PK)
      accb[m] = fma2(swp(accb[m]), make_float2(-zyy[m].x, -zyy[m].y), mul2(accb[m], splat2(zx[m])));
  }
}

// K5: Spart[g] = sum over planes k of group g of column-FFT(in[k]) * conj(H_{k0+k})
template <int N, int C, int E_, bool PK = false>
__global__ void __launch_bounds__(C * FftShape<N, E_>::TPF) k_fwd_cols(const float2* __restrict__ in,
                                                                    float2* __restrict__ Spart, int nx, long long P,
                                                                    int nzl, int ppg, int k0,
                                                                    const uint64_t* __restrict__ tab,
                                                                    const float4* __restrict__ twg,
                                                                    const float2* __restrict__ circg,
                                                                    const uint8_t* __restrict__ live) {
  using Sh = FftShape<N, E_>;
  constexpr int TPF = Sh::TPF, E = Sh::E;
  extern __shared__ float2 smem[];
  float4* tw = reinterpret_cast<float4*>(smem);
  float2* circ = smem + 2 * N;
  float2* buf = smem + 2 * N + 256;
  for (int i = threadIdx.x; i < TwLayout<N, E_>::size(); i += blockDim.x) tw[i] = twg[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) circ[i] = circg[i];
  __syncthreads();
  const int c = threadIdx.x % C, j = threadIdx.x / C;
  const int col = blockIdx.x * C + c;
  const int kb = blockIdx.y * ppg, ke = min(nzl, kb + ppg);
  float2 acc[E], accb[PK ? E : 1];
#pragma unroll
  for (int m = 0; m < E; ++m) acc[m] = czero();
#pragma unroll
  for (int m = 0; m < (PK ? E : 1); ++m) accb[m] = czero();
  const long long p0 = (long long)j * nx + col, st = (long long)TPF * nx;
  // Horner from the last plane, as in k_fwd_cols_staged
  float zx[E];
  float2 zyy[E];
#pragma unroll
  for (int m = 0; m < E; ++m) fwd_ratio<PK>(tab[p0 + m * st], circ, zx[m], zyy[m]);
  for (int k = ke - 1; k >= kb; --k) {
    if (live && !live[k]) {  // all-zero plane: v = 0
      horner_zero<PK, E>(acc, accb, zx, zyy);
      continue;
    }
    float2 v[E];
    const float2* src = in + (long long)k * P + p0;
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = src[m * st];
    fft_line<N, false, E_>(v, j, buf + c, C, tw);
#pragma unroll
    for (int m = 0; m < E; ++m) {
      acc[m] = fma2(swp(acc[m]), zyy[m], fma2(acc[m], splat2(zx[m]), v[m]));
      if constexpr (PK)
        accb[m] = fma2(swp(accb[m]), make_float2(-zyy[m].x, -zyy[m].y), fma2(accb[m], splat2(zx[m]), v[m]));
    }
  }
#pragma unroll
  for (int m = 0; m < E; ++m) acc[m] = fwd_close<PK>(acc[m], accb[PK ? m : 0], tab[p0 + m * st], k0, kb, circ);
  float2* dst = Spart + (long long)blockIdx.y * P + p0;
#pragma unroll
  for (int m = 0; m < E; ++m) dst[m * st] = acc[m];
}

// K5 with TMA staging (N <= 1024): one elected thread streams plane k+1's
// C-column block (N rows x C complex) into the other half of a double-buffered
// shared-memory stage with 2D tensor copies while the CTA transforms plane k,
// so the column loads leave the critical path (the plain kernel waited on HBM
// once per plane with only 16 warps per SM to hide it).
// 2 columns per CTA (128 threads) at <= 160 registers: 3 CTAs / 12 warps per
// SM (4 columns at 190 registers fit one CTA / 8 warps: 14.5 vs 12.3 ms per 10
// C3 iterations)
#ifndef HOLO_FWD_MINB
#define HOLO_FWD_MINB 3
#endif
template <int N, int C, int E_, bool PK = false>
__global__ void __launch_bounds__(C * FftShape<N, E_>::TPF, PK ? 2 : (C * FftShape<N, E_>::TPF <= 128 ? HOLO_FWD_MINB : 1)) k_fwd_cols_staged(
    const __grid_constant__ CUtensorMap in_map, float2* __restrict__ Spart, int nx, long long P, int ny, int nzl,
    int ppg, int k0, const uint64_t* __restrict__ tab, const float4* __restrict__ twg,
    const float2* __restrict__ circg, const uint8_t* __restrict__ live) {
  using Sh = FftShape<N, E_>;
  constexpr int TPF = Sh::TPF, E = Sh::E;
  constexpr int BOX_ROWS = N < 256 ? N : 256;
  extern __shared__ __align__(128) float2 smem[];
  float2* stage = smem;                             // [2][N][C]
  float4* tw = reinterpret_cast<float4*>(smem + 2 * N * C);
  float2* circ = smem + 2 * N * C + 2 * N;
  float2* buf = smem + 2 * N * C + 2 * N + 256;
  __shared__ uint64_t bars[2];
  const int kb = blockIdx.y * ppg, ke = min(nzl, kb + ppg);
  const bool leader = threadIdx.x == 0;
  poison_dyn_smem();
  auto issue = [&](int k, int b) {
    HOLO_DCHECK(k >= 0 && k < nzl && (blockIdx.x + 1) * C <= nx, CK_COLS);
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[b]);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                 "r"((unsigned)(N * C * sizeof(float2)))
                 : "memory");
#pragma unroll
    for (int r0 = 0; r0 < N; r0 += BOX_ROWS)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
              (unsigned)__cvta_generic_to_shared(stage + (size_t)b * N * C + (size_t)r0 * C)),
          "l"(reinterpret_cast<uint64_t>(&in_map)), "r"(2 * (int)blockIdx.x * C), "r"(k * ny + r0), "r"(bar)
          : "memory");
  };
  if (leader) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bars[b]))
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // sparsity-aware forward (solver.py:115-119): all-zero planes (live[k] == 0)
  // are neither loaded nor transformed; the stage ring advances per live plane
  auto next_live = [&](int k) {
    if (live)
      while (k >= kb && !live[k]) --k;
    return k;
  };
  {
    const int kf = next_live(ke - 1);
    if (leader && kf >= kb) issue(kf, 0);  // planes are walked last to first (Horner)
  }
  for (int i = threadIdx.x; i < TwLayout<N, E_>::size(); i += blockDim.x) tw[i] = twg[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) circ[i] = circg[i];
  __syncthreads();
  const int c = threadIdx.x % C, j = threadIdx.x / C;
  const int col = blockIdx.x * C + c;
  float2 acc[E], accb[PK ? E : 1];
#pragma unroll
  for (int m = 0; m < E; ++m) acc[m] = czero();
#pragma unroll
  for (int m = 0; m < (PK ? E : 1); ++m) accb[m] = czero();
  const long long p0 = (long long)j * nx + col, st = (long long)TPF * nx;
  // sum_k v_k conj(H_k) over the CTA's planes = conj(H_kb) sum_k v_k z^(k-kb),
  // z = conj(G) = cis(-2 pi dz q) (the reference's ladder step, optics.py:146-169):
  // Horner from the last plane, acc <- acc z + v_k, one complex FMA pair per
  // element and plane; z is held as z.x and the pair (-z.y, z.y) so that
  // acc z = swap(acc) (-z.y, z.y) + acc z.x needs no sign shuffles.
  float zx[E];
  float2 zyy[E];
#pragma unroll
  for (int m = 0; m < E; ++m) fwd_ratio<PK>(tab[p0 + m * st], circ, zx[m], zyy[m]);
  int i = 0;  // live planes consumed so far
  for (int k = ke - 1; k >= kb; --k) {
    if (live && !live[k]) {  // v = 0
      horner_zero<PK, E>(acc, accb, zx, zyy);
      continue;
    }
    const int b = i & 1;
    // the other stage was last read in the previous live plane, before fft_line's barriers
    if (leader) {
      const int kn = next_live(k - 1);
      if (kn >= kb) issue(kn, b ^ 1);
    }
    {
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[b]), par = (i >> 1) & 1;
      unsigned done = 0;
      do {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(par)
            : "memory");
      } while (!done);
    }
    float2 v[E];
    const float2* src = stage + (size_t)b * N * C + c;
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = src[(j + m * TPF) * C];
    fft_line<N, false, E_>(v, j, buf + c, C, tw);
#pragma unroll
    for (int m = 0; m < E; ++m) {
      acc[m] = fma2(swp(acc[m]), zyy[m], fma2(acc[m], splat2(zx[m]), v[m]));
      if constexpr (PK)
        accb[m] = fma2(swp(accb[m]), make_float2(-zyy[m].x, -zyy[m].y), fma2(accb[m], splat2(zx[m]), v[m]));
    }
    ++i;
  }
  // times conj(H_kb) (packed: the two-sum closure), exact (64-bit phase)
#pragma unroll
  for (int m = 0; m < E; ++m) acc[m] = fwd_close<PK>(acc[m], accb[PK ? m : 0], tab[p0 + m * st], k0, kb, circ);
  float2* dst = Spart + (long long)blockIdx.y * P + p0;
  HOLO_DCHECK(p0 + (long long)(E - 1) * st < P && col < nx, CK_COLS);
#pragma unroll
  for (int m = 0; m < E; ++m) dst[m * st] = acc[m];
}

__global__ void k_sum_groups(const float2* __restrict__ Spart, int groups, long long P, float2* __restrict__ S) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    float2 s = Spart[p];
    for (int g = 1; g < groups; ++g) s = cadd(s, Spart[(long long)g * P + p]);
    S[p] = s;
  }
}

// ---------------------------------------------------------------- K6 -------

constexpr int kSensorThreads = 256;

__global__ void __launch_bounds__(kSensorThreads) k_sensor(const float2* __restrict__ Sa, const float2* __restrict__ Sb,
                                                          float ca, float cb, const float2* __restrict__ B,
                                                          const uint8_t* __restrict__ mask, float2* __restrict__ Rout,
                                                          int ny, int nx, double* __restrict__ part) {
  const long long P = (long long)ny * nx;
  double acc[1] = {0.0};
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(p / nx), j = (int)(p - (long long)i * nx);
    const int im = (i == 0) ? 0 : ny - i, jm = (j == 0) ? 0 : nx - j;
    const long long q = (long long)im * nx + jm;
    float2 s1 = cscale(Sa[p], ca), s2 = cscale(Sa[q], ca);
    if (Sb) {
      s1 = cadd(s1, cscale(Sb[p], cb));
      s2 = cadd(s2, cscale(Sb[q], cb));
    }
    const bool m = mask[p] != 0;
    // Re-part projection of the masked spectrum: FFT(Re IFFT(mS)) = m (S(f) + conj S(-f)) / 2
    float2 r = m ? make_float2(0.5f * (s1.x + s2.x), 0.5f * (s1.y - s2.y)) : czero();
    if (B) r = csub(r, B[p]);
    acc[0] += (double)r.x * r.x + (double)r.y * r.y;
    if (Rout) Rout[p] = m ? r : czero();
  }
  block_sum<1, kSensorThreads>(acc, part + blockIdx.x);
}

template <int NT>
__global__ void __launch_bounds__(NT) k_final_sum(const double* __restrict__ part, int n, double scale,
                                                  double* __restrict__ out) {
  double acc[1] = {0.0};
  for (int i = threadIdx.x; i < n; i += NT) acc[0] += part[i];
  __shared__ double res[1];
  block_sum<1, NT>(acc, res);
  __syncthreads();
  if (threadIdx.x == 0) *out = res[0] * scale;
}

// ---------------------------------------------------------------- K4 -------
// Fused-lasso prox on 2D tiles with a (T+2)-deep halo recomputed per tile
// (temporal blocking).  Per owned pixel the thread keeps v, p, q (re and im)
// in registers; the extrapolated dual (rp, rq) and the primal u live in smem.
// Semantics follow prox.py:104-148 (FGP, step 1/(8 tau), replicated edges,
// per-plane guard) and prox.py:83-96 (strict |w| > tau soft threshold).

constexpr int kProxThreads = 512;
constexpr int kProxMaxPx = 12;

template <int NT, int MAXPX>
__global__ void __launch_bounds__(NT, 1) k_prox(const ProxArgs a) {
  const int plane = blockIdx.y, tile = blockIdx.x;
  uint32_t force = 0;
  if (a.force) {
    force = a.force[plane];
    if (!force) return;  // fix-up pass: only planes whose guard fired
  }
  const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
  const int i0 = ty * a.tile, j0 = tx * a.tile;
  const int i1 = min(a.ny, i0 + a.tile), j1 = min(a.nx, j0 + a.tile);
  const int H = a.halo;
  const int ri0 = max(0, i0 - H), rj0 = max(0, j0 - H);
  const int ri1 = min(a.ny, i1 + H), rj1 = min(a.nx, j1 + H);
  const int EW = rj1 - rj0, EH = ri1 - ri0, NPX = EW * EH;
  const int ei0 = i0 - ri0, ei1 = i1 - ri0, ej0 = j0 - rj0, ej1 = j1 - rj0;  // interior in region coords

  extern __shared__ float sm[];
  float* rpr = sm;
  float* rpi = sm + NPX;
  float* rqr = sm + 2 * NPX;
  float* rqi = sm + 3 * NPX;
  float* ur = sm + 4 * NPX;
  float* ui = sm + 5 * NPX;

  const long long pbase = (long long)plane * a.P;
  const int tid = threadIdx.x;
  float vr[MAXPX], vi[MAXPX], pr[MAXPX], pi[MAXPX], qr[MAXPX], qi[MAXPX];
  uint32_t geo[MAXPX];

#pragma unroll
  for (int m = 0; m < MAXPX; ++m) {
    const int idx = tid + m * NT;
    pr[m] = pi[m] = qr[m] = qi[m] = 0.f;
    vr[m] = vi[m] = 0.f;
    geo[m] = 0xFFFFFFFFu;
    if (idx < NPX) {
      const int er = idx / EW, ec = idx - er * EW;
      geo[m] = ((uint32_t)er << 16) | (uint32_t)ec;
      const long long g = pbase + (long long)(ri0 + er) * a.nx + (rj0 + ec);
      float2 y = a.x[g];
      if (a.beta != 0.f) {
        const float2 o = a.xp[g];
        y = make_float2(fmaf(1.f + a.beta, y.x, -a.beta * o.x), fmaf(1.f + a.beta, y.y, -a.beta * o.y));
      }
      if (a.grad) {
        const float2 gg = a.grad[g];
        y = make_float2(fmaf(-a.step, gg.x, y.x), fmaf(-a.step, gg.y, y.y));
      }
      vr[m] = y.x;
      vi[m] = y.y;
      ur[idx] = y.x;
      ui[idx] = y.y;
    }
  }
  __syncthreads();

  // partial sums (fp64): guard (tv(w), |w-v|^2, tv(v)) then ip, dx2, l1, tv(x)
  double acc[kProxParts];
#pragma unroll
  for (int i = 0; i < kProxParts; ++i) acc[i] = 0.0;

  const bool tv_on = a.tau_tv > 0.f;
  const float tau = a.tau_tv, lr = a.lr_tv;
  if (tv_on) {
    for (int t = 0; t < a.inner; ++t) {
      if (t > 0) {
        // u = v - tau * D^T(rp, rq)
#pragma unroll
        for (int m = 0; m < MAXPX; ++m) {
          if (geo[m] == 0xFFFFFFFFu) continue;
          const int er = geo[m] >> 16, ec = geo[m] & 0xFFFF;
          const int idx = er * EW + ec;
          const bool dn = er + 1 < EH, rt = ec + 1 < EW;
          float dr = rpr[idx] + rqr[idx], di = rpi[idx] + rqi[idx];
          if (dn) { dr -= rpr[idx + EW]; di -= rpi[idx + EW]; }
          if (rt) { dr -= rqr[idx + 1]; di -= rqi[idx + 1]; }
          ur[idx] = fmaf(-tau, dr, vr[m]);
          ui[idx] = fmaf(-tau, di, vi[m]);
        }
        __syncthreads();
      }
      const float bt = a.fgp_beta[t];
#pragma unroll
      for (int m = 0; m < MAXPX; ++m) {
        if (geo[m] == 0xFFFFFFFFu) continue;
        const int er = geo[m] >> 16, ec = geo[m] & 0xFFFF;
        const int idx = er * EW + ec;
        const float uor = ur[idx], uoi = ui[idx];
        float gyr = 0.f, gyi = 0.f, gxr = 0.f, gxi = 0.f;
        if (er > 0) { gyr = uor - ur[idx - EW]; gyi = uoi - ui[idx - EW]; }
        if (ec > 0) { gxr = uor - ur[idx - 1]; gxi = uoi - ui[idx - 1]; }
        if (t == 0 && er >= ei0 && er < ei1 && ec >= ej0 && ec < ej1) {
          acc[PT_G_R] -= (double)tau * sqrtf(gyr * gyr + gxr * gxr);
          acc[PT_G_I] -= (double)tau * sqrtf(gyi * gyi + gxi * gxi);
        }
        float opr = 0.f, opi = 0.f, oqr = 0.f, oqi = 0.f;
        if (t > 0) { opr = rpr[idx]; opi = rpi[idx]; oqr = rqr[idx]; oqi = rqi[idx]; }
        float npr = fmaf(lr, gyr, opr), nqr = fmaf(lr, gxr, oqr);
        float npi = fmaf(lr, gyi, opi), nqi = fmaf(lr, gxi, oqi);
        const float n2r = fmaf(npr, npr, nqr * nqr), n2i = fmaf(npi, npi, nqi * nqi);
        if (n2r > 1.f) { const float s = rsqrtf(n2r); npr *= s; nqr *= s; }
        if (n2i > 1.f) { const float s = rsqrtf(n2i); npi *= s; nqi *= s; }
        rpr[idx] = fmaf(bt, npr - pr[m], npr);
        rqr[idx] = fmaf(bt, nqr - qr[m], nqr);
        rpi[idx] = fmaf(bt, npi - pi[m], npi);
        rqi[idx] = fmaf(bt, nqi - qi[m], nqi);
        pr[m] = npr; qr[m] = nqr; pi[m] = npi; qi[m] = nqi;
      }
      __syncthreads();
    }
    // w = v - tau * D^T(p, q): publish p, q
#pragma unroll
    for (int m = 0; m < MAXPX; ++m) {
      if (geo[m] == 0xFFFFFFFFu) continue;
      const int idx = (geo[m] >> 16) * EW + (geo[m] & 0xFFFF);
      rpr[idx] = pr[m]; rpi[idx] = pi[m]; rqr[idx] = qr[m]; rqi[idx] = qi[m];
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MAXPX; ++m) {
      if (geo[m] == 0xFFFFFFFFu) continue;
      const int er = geo[m] >> 16, ec = geo[m] & 0xFFFF;
      const int idx = er * EW + ec;
      float dr = pr[m] + qr[m], di = pi[m] + qi[m];
      if (er + 1 < EH) { dr -= rpr[idx + EW]; di -= rpi[idx + EW]; }
      if (ec + 1 < EW) { dr -= rqr[idx + 1]; di -= rqi[idx + 1]; }
      // keep w in the p registers from here on
      pr[m] = fmaf(-tau, dr, vr[m]);
      pi[m] = fmaf(-tau, di, vi[m]);
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MAXPX; ++m) {
      if (geo[m] == 0xFFFFFFFFu) continue;
      const int idx = (geo[m] >> 16) * EW + (geo[m] & 0xFFFF);
      ur[idx] = pr[m];
      ui[idx] = pi[m];
    }
    __syncthreads();
  } else {
#pragma unroll
    for (int m = 0; m < MAXPX; ++m) { pr[m] = vr[m]; pi[m] = vi[m]; }
  }

  // guard statistics on the interior, then the speculative soft threshold
#pragma unroll
  for (int m = 0; m < MAXPX; ++m) {
    if (geo[m] == 0xFFFFFFFFu) continue;
    const int er = geo[m] >> 16, ec = geo[m] & 0xFFFF;
    const int idx = er * EW + ec;
    const bool interior = er >= ei0 && er < ei1 && ec >= ej0 && ec < ej1;
    float wr = pr[m], wi = pi[m];
    if (tv_on && interior) {
      float gyr = 0.f, gyi = 0.f, gxr = 0.f, gxi = 0.f;
      if (er > 0) { gyr = wr - ur[idx - EW]; gyi = wi - ui[idx - EW]; }
      if (ec > 0) { gxr = wr - ur[idx - 1]; gxi = wi - ui[idx - 1]; }
      const float dr = wr - vr[m], di = wi - vi[m];
      acc[PT_G_R] += (double)tau * sqrtf(gyr * gyr + gxr * gxr) + 0.5 * (double)(dr * dr);
      acc[PT_G_I] += (double)tau * sqrtf(gyi * gyi + gxi * gxi) + 0.5 * (double)(di * di);
    }
    if (force & 1u) wr = vr[m];
    if (force & 2u) wi = vi[m];
    if (a.real_mode) {  // solver.py:208-210: max(w - tau, 0), per packed real plane (Re, Im)
      wr = fmaxf(wr - a.tau_l1, 0.f);
      wi = fmaxf(wi - a.tau_l1, 0.f);
    } else if (a.tau_l1 > 0.f) {
      const float mag = hypotf(wr, wi);
      if (mag > a.tau_l1) {
        const float gscale = 1.f - a.tau_l1 / mag;
        wr *= gscale;
        wi *= gscale;
      } else {
        wr = 0.f;
        wi = 0.f;
      }
    }
    pr[m] = wr;
    pi[m] = wi;
  }
  if (tv_on) __syncthreads();  // guard reads of u done before x_new overwrites rp
#pragma unroll
  for (int m = 0; m < MAXPX; ++m) {
    if (geo[m] == 0xFFFFFFFFu) continue;
    const int idx = (geo[m] >> 16) * EW + (geo[m] & 0xFFFF);
    rpr[idx] = pr[m];
    rpi[idx] = pi[m];
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < MAXPX; ++m) {
    if (geo[m] == 0xFFFFFFFFu) continue;
    const int er = geo[m] >> 16, ec = geo[m] & 0xFFFF;
    if (!(er >= ei0 && er < ei1 && ec >= ej0 && ec < ej1)) continue;
    const int idx = er * EW + ec;
    const float xr = pr[m], xi = pi[m];
    float gyr = 0.f, gyi = 0.f, gxr = 0.f, gxi = 0.f;
    if (er > 0) { gyr = xr - rpr[idx - EW]; gyi = xi - rpi[idx - EW]; }
    if (ec > 0) { gxr = xr - rpr[idx - 1]; gxi = xi - rpi[idx - 1]; }
    acc[PT_TVX] += (double)sqrtf(gyr * gyr + gxr * gxr) + (double)sqrtf(gyi * gyi + gxi * gxi);
    acc[PT_L1] += a.real_mode ? (double)xr + (double)xi : (double)hypotf(xr, xi);
    const long long g = pbase + (long long)(ri0 + er) * a.nx + (rj0 + ec);
    float2 y = a.x[g];
    if (a.beta != 0.f) {
      const float2 o = a.xp[g];
      y = make_float2(fmaf(1.f + a.beta, y.x, -a.beta * o.x), fmaf(1.f + a.beta, y.y, -a.beta * o.y));
    }
    const float dxr = xr - y.x, dxi = xi - y.y;
    if (a.grad) {
      const float2 gg = a.grad[g];
      acc[PT_IP] += (double)gg.x * dxr + (double)gg.y * dxi;
    }
    acc[PT_DX2] += (double)dxr * dxr + (double)dxi * dxi;
    a.xnew[g] = make_float2(xr, xi);
  }
  block_sum<kProxParts, NT>(acc, a.part + ((long long)plane * a.tiles_per_plane + tile) * kProxParts);
}

constexpr int kReduceThreads = 128;

// part: per tile fp64 sums (generic kernel, nw == 0) or per (tile, warp) fp32
// sums (strip kernel, nw warps per tile), summed here in fp64
// Boundary-row statistics of the strip prox with tvfix (kernels.cuh): for
// every tile below the first tile row, the TV(w) (guard, per part) and
// TV(x_new) terms of its first row, whose row above lies in the tile above
// (prox.py:61-72 isotropic TV, backward differences, zero at the plane's left
// edge).  w of a tile's first / last row comes from the prox's side buffer,
// x_new from the output.  One CTA of 64 threads per tile, fp32 partials per
// tile -> bpart[plane][3][tile] (k_prox_reduce adds them in fp64).
__global__ void __launch_bounds__(64) k_prox_tvfix(const ProxArgs a) {
  const int tile = blockIdx.x, plane = blockIdx.y;
  const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
  float g_re = 0.f, g_im = 0.f, tvx = 0.f;
  if (ty > 0) {
    const int i0 = ty * a.tile_h, j0 = tx * a.tile, j1 = min(a.nx, j0 + a.tile);
    auto rj0_of = [&](int t) { return min(max(t * a.tile - a.halo, 0), a.nx - 64); };
    const int rj0 = rj0_of(tx), j = j0 + (int)threadIdx.x;
    if (j < j1) {
      const float2* X = a.xnew + (long long)plane * a.P;
      const float2 xa = X[(long long)i0 * a.nx + j], xu = X[(long long)(i0 - 1) * a.nx + j];
      const float2 xl = j > 0 ? X[(long long)i0 * a.nx + j - 1] : xa;
      const float2* W = reinterpret_cast<const float2*>(a.wside);  // [plane][tile][2][64]
      const long long base = (long long)plane * a.tiles_per_plane;
      auto wrow = [&](int t, int which) { return W + ((base + t) * 2 + which) * 64; };
      HOLO_DCHECK(j - rj0 >= 0 && j - rj0 < 64 && i0 - 1 >= 0 && i0 < a.ny, CK_PROX_STORE);
      const float2 wa = wrow(tile, 0)[j - rj0], wu = wrow(tile - a.tiles_x, 1)[j - rj0];
      float2 wl = wa;
      if (j > 0) wl = j - 1 >= j0 ? wrow(tile, 0)[j - 1 - rj0] : wrow(tile - 1, 0)[j - 1 - rj0_of(tx - 1)];
      auto nrm = [](float gy, float gx) { return sqrt_a(fmaf(gy, gy, gx * gx)); };
      g_re = nrm(wa.x - wu.x, wa.x - wl.x);
      g_im = nrm(wa.y - wu.y, wa.y - wl.y);
      tvx = nrm(xa.x - xu.x, xa.x - xl.x) + nrm(xa.y - xu.y, xa.y - xl.y);
    }
  }
  __shared__ float red[2][3];
  float v3[3] = {a.tau_tv * g_re, a.tau_tv * g_im, tvx};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v3[i] += __shfl_down_sync(0xffffffffu, v3[i], o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][i] = v3[i];
  }
  __syncthreads();
  if (threadIdx.x < 3)
    a.bpart[((long long)plane * 3 + threadIdx.x) * a.tiles_per_plane + tile] =
        red[0][threadIdx.x] + red[1][threadIdx.x];
}

__global__ void __launch_bounds__(kReduceThreads) k_prox_reduce(const double* __restrict__ part, int tpp, int nw,
                                                                double tau, int tv_on, uint8_t* __restrict__ force_acc,
                                                                double* __restrict__ plane_out,
                                                                int* __restrict__ new_fail,
                                                                uint8_t* __restrict__ live, int skip_ok,
                                                                const uint8_t* __restrict__ only,
                                                                const float* __restrict__ bpart) {
  const int plane = blockIdx.x;
  // guard fix-up pass (only = its force bits): planes it did not rerun keep
  // the main pass's sums
  if (only && !only[plane]) {
    if (threadIdx.x == 0) new_fail[plane] = 0;
    return;
  }
  double acc[kProxParts];
#pragma unroll
  for (int i = 0; i < kProxParts; ++i) acc[i] = 0.0;
  if (nw > 0) {  // [part][tile][warp]: coalesced float4 rows per part
    const long long n = (long long)tpp * nw;
    const float* src = reinterpret_cast<const float*>(part) + (long long)plane * kProxParts * n;
#pragma unroll
    for (int i = 0; i < kProxParts; ++i) {
      const float4* s4 = reinterpret_cast<const float4*>(src + i * n);
      for (long long t = threadIdx.x; t < n / 4; t += kReduceThreads) {
        const float4 f = s4[t];
        acc[i] += ((double)f.x + (double)f.y) + ((double)f.z + (double)f.w);
      }
    }
  } else {
    const double* src = part + (long long)plane * tpp * kProxParts;
    for (int t = threadIdx.x; t < tpp; t += kReduceThreads) {
#pragma unroll
      for (int i = 0; i < kProxParts; ++i) acc[i] += src[(long long)t * kProxParts + i];
    }
  }
  if (bpart) {  // boundary-row TV terms (k_prox_tvfix)
    const float* b = bpart + (long long)plane * 3 * tpp;
    for (int t = threadIdx.x; t < tpp; t += kReduceThreads) {
      acc[PT_G_R] += (double)b[t];
      acc[PT_G_I] += (double)b[tpp + t];
      acc[PT_TVX] += (double)b[2 * tpp + t];
    }
  }
  __shared__ double s[kProxParts];
  block_sum<kProxParts, kReduceThreads>(acc, s);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t bits = 0;
    if (tv_on) {
      // prox.py:138-147: reject the TV output when tau TV(w) + |w-v|^2/2 > tau TV(v)
      if (s[PT_G_R] > 0.0) bits |= 1u;
      if (s[PT_G_I] > 0.0) bits |= 2u;
    }
    const uint32_t old = force_acc[plane];
    force_acc[plane] = (uint8_t)(old | bits);
    new_fail[plane] = (bits & ~old) ? 1 : 0;
    double* o = plane_out + (long long)plane * 4;
    o[0] = s[PT_IP];
    o[1] = s[PT_DX2];
    o[2] = s[PT_L1];
    o[3] = s[PT_TVX];
    // all-zero plane: sum |x_new| == 0 exactly (NaN compares unequal: live)
    if (live) live[plane] = (skip_ok && s[PT_L1] == 0.0) ? 0 : 1;
  }
}

__global__ void __launch_bounds__(kReduceThreads) k_plane_total(const double* __restrict__ plane_out,
                                                                const int* __restrict__ new_fail, int nplanes,
                                                                double* __restrict__ scalars,
                                                                const uint8_t* __restrict__ live) {
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int k = threadIdx.x; k < nplanes; k += kReduceThreads) {
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] += plane_out[(long long)k * 4 + i];
    acc[4] += (double)new_fail[k];
    if (live) acc[5] += live[k] ? 0.0 : 1.0;
  }
  block_sum<6, kReduceThreads>(acc, scalars);
}

// ------------------------------------------------------------ misc ---------

constexpr int kEltThreads = 256;

__global__ void k_load_hologram(const double* __restrict__ b, float2* __restrict__ bc, long long P,
                                double* __restrict__ part) {
  double acc[1] = {0.0};
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    const double v = b[p];
    acc[0] += v * v;
    bc[p] = make_float2((float)v, 0.f);
  }
  block_sum<1, kEltThreads>(acc, part + blockIdx.x);
}

__global__ void k_real_part(const float2* __restrict__ in, float* __restrict__ out, long long n, float scale) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    out[p] = in[p].x * scale;
}

__global__ void k_real_to_complex(const float* __restrict__ in, float2* __restrict__ out, long long n) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    out[p] = make_float2(in[p], 0.f);
}

__global__ void k_apply_mask(float2* __restrict__ spec, const uint8_t* __restrict__ mask, long long P, long long n) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    if (!mask[p % P]) spec[p] = czero();
}

__global__ void k_transfer(const uint64_t* __restrict__ tab, const uint8_t* __restrict__ mask,
                           const float2* __restrict__ circ, long long P, int k0, int nk, int conj,
                           float2* __restrict__ out) {
  const long long n = P * nk;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long p = e % P;
    const int k = k0 + (int)(e / P);
    float2 h = mask[p] ? cis_cycles(plane_phase(tab[p], k), circ) : czero();
    out[e] = conj ? cconj(h) : h;
  }
}

__global__ void k_spec_combine(const float2* __restrict__ Sa, const float2* __restrict__ Sb, float ca, float cb,
                               float2* __restrict__ out, long long P) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    float2 s = cscale(Sa[p], ca);
    if (Sb) s = cadd(s, cscale(Sb[p], cb));
    out[p] = s;
  }
}

// per pixel: sum_k cos^2(2 pi (A + k B)) for the propagating band; block max
__global__ void __launch_bounds__(256) k_real_opnorm(const uint64_t* __restrict__ tab, const uint8_t* __restrict__ mask,
                                                     const float2* __restrict__ circg, long long P, int nz,
                                                     double* __restrict__ part) {
  __shared__ float2 circ[256];
  circ[threadIdx.x] = circg[threadIdx.x];
  __syncthreads();
  double best = 0.0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    if (!mask[p]) continue;
    double acc = 0.0;
    for (int k = 0; k < nz; ++k) {
      const float c = cis_cycles(plane_phase(tab[p], k), circ).x;
      acc += (double)c * c;
    }
    best = fmax(best, acc);
  }
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_down_sync(0xffffffffu, best, o));
  __shared__ double red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < 8; ++i) m = fmax(m, red[i]);
    part[blockIdx.x] = m;
  }
}

__global__ void k_max_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) m = fmax(m, part[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) *out = m;
}

__global__ void __launch_bounds__(256) k_vol_norm2(const float2* __restrict__ x, long long n, double* __restrict__ part) {
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float2 v = x[i];
    acc[0] += (double)v.x * v.x + (double)v.y * v.y;
  }
  block_sum<1, 256>(acc, part + blockIdx.x);
}

__global__ void k_vol_rescale(float2* __restrict__ x, long long n, const double* __restrict__ nrm2, int real) {
  const float sc = nrm2 ? (float)(1.0 / sqrt(*nrm2)) : 1.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float2 v = x[i];
    x[i] = make_float2(v.x * sc, real ? 0.f : v.y * sc);
  }
}

constexpr int kCooChunk = 1024;
constexpr int kCooThreads = 256;

__global__ void __launch_bounds__(kCooThreads) k_coo_count(const float2* __restrict__ x, long long P, int cpp,
                                                           int* __restrict__ counts) {
  const int plane = blockIdx.y, ch = blockIdx.x;
  const long long start = (long long)ch * kCooChunk;
  const float2* src = x + (long long)plane * P;
  int c = 0;
  for (int e = threadIdx.x; e < kCooChunk; e += kCooThreads) {
    const long long p = start + e;
    if (p < P) {
      const float2 v = src[p];
      c += (v.x != 0.f || v.y != 0.f) ? 1 : 0;
    }
  }
  double acc[1] = {(double)c};
  __shared__ double res[1];
  block_sum<1, kCooThreads>(acc, res);
  __syncthreads();
  if (threadIdx.x == 0) counts[(long long)plane * cpp + ch] = (int)res[0];
}

// row-major compaction: each thread owns 4 consecutive elements of the chunk;
// values are written as complex64 (vals) or widened to complex128 (vals64)
__global__ void __launch_bounds__(kCooThreads) k_coo_compact(const float2* __restrict__ x, long long P, int nx,
                                                             int cpp, const long long* __restrict__ offsets,
                                                             int* __restrict__ rows, int* __restrict__ cols,
                                                             float2* __restrict__ vals, double2* __restrict__ vals64) {
  constexpr int PER = kCooChunk / kCooThreads;
  const int plane = blockIdx.y, ch = blockIdx.x;
  const long long start = (long long)ch * kCooChunk + (long long)threadIdx.x * PER;
  const float2* src = x + (long long)plane * P;
  float2 v[PER];
  int flag[PER], mine = 0;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const long long p = start + e;
    v[e] = (p < P) ? src[p] : czero();
    flag[e] = (v[e].x != 0.f || v[e].y != 0.f) ? 1 : 0;
    mine += flag[e];
  }
  // exclusive block scan of `mine` (warp shuffles + smem)
  __shared__ int wsum[kCooThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  int before = 0;
  for (int k = 0; k < w; ++k) before += wsum[k];
  long long out = offsets[(long long)plane * cpp + ch] + before + incl - mine;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    if (flag[e]) {
      const long long p = start + e;
      rows[out] = (int)(p / nx);
      cols[out] = (int)(p % nx);
      if (vals64)
        vals64[out] = make_double2((double)v[e].x, (double)v[e].y);
      else
        vals[out] = v[e];
      ++out;
    }
  }
}

inline int grid_for(long long n, int threads, int cap = 148 * 16) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  return (int)std::min<long long>(g, cap);
}

}  // namespace

// =================================================================== host ==

static std::atomic<long long> g_launches{0};
long long launch_count() { return g_launches.load(); }
#define COUNT_LAUNCH(n) g_launches.fetch_add((n), std::memory_order_relaxed)
void add_launches(long long n) { COUNT_LAUNCH(n); }

bool plan_supported(int nx, int ny) {
  // powers of two: the fused production passes; other sides: gfft.cu (an odd
  // nx runs the generic tile prox: the strip prox's tensor maps need even rows)
  if (pow2_side(nx) && pow2_side(ny)) return true;
  return generic_side(nx) && generic_side(ny);
}

cudaError_t plan_build(Plan& p, int nx, int ny, int nz, double pitch, double dz, double z0, double lam,
                       cudaStream_t s) {
  p.nx = nx; p.ny = ny; p.nz = nz;
  p.P = (long long)nx * ny;
  p.pitch = pitch; p.dz = dz; p.z0 = z0; p.lam = lam;
  p.col_c = col_width(ny);
  // a power-of-two side keeps its fused passes when the other side is general
  // (1280x1024: fused TMA columns, mixed-radix rows)
  p.generic_x = pow2_side(nx) ? 0 : 1;
  p.generic_y = (pow2_side(ny) && nx % 8 == 0) ? 0 : 1;
  p.generic = p.generic_x | p.generic_y;
  cudaError_t e;
  for (int k = 0; k < 2; ++k) {
    if ((e = cudaMalloc(&p.tw_x[k], sizeof(float4) * std::max(nx, 32)))) return e;
    if ((e = cudaMalloc(&p.tw_y[k], sizeof(float4) * std::max(ny, 32)))) return e;
  }
  if ((e = cudaMalloc(&p.circle, sizeof(float2) * 256))) return e;
  if ((e = cudaMalloc(&p.phase, sizeof(uint64_t) * p.P))) return e;
  if ((e = cudaMalloc(&p.mask, p.P))) return e;
  // one table layout per element count: [0] E = 16 (or N), [1] E = 32 (or the E=16 one)
  auto tables = [&](int n, float4** tw) {
    dispatch_n(n, [&](auto nc) {
      constexpr int N = decltype(nc)::value;
      constexpr int E0 = DefaultE<N>::value, E1 = EBig<N>::value;
      k_twiddles<N, E0><<<(TwLayout<N, E0>::size() + 255) / 256, 256, 0, s>>>(tw[0]);
      k_twiddles<N, E1><<<(TwLayout<N, E1>::size() + 255) / 256, 256, 0, s>>>(tw[1]);
    });
  };
  tables(nx, p.tw_x);
  tables(ny, p.tw_y);
  COUNT_LAUNCH(2);
  k_circle<<<1, 256, 0, s>>>(p.circle);
  COUNT_LAUNCH(1);
  k_phase<<<(int)((p.P + 255) / 256), 256, 0, s>>>(p.phase, p.mask, ny, nx, pitch, lam, z0, dz);
  COUNT_LAUNCH(1);
  if (p.generic && (e = gplan_build(p, s))) return e;
  // the DC sample (fx = fy = 0, arg = 1) always propagates, so ||A||^2 = nz exactly
  p.any_propagating = 1;
  if ((e = cudaStreamSynchronize(s))) return e;
  return cudaGetLastError();
}

void plan_free(Plan& p) {
  cudaFree(p.groots_x);
  cudaFree(p.groots_y);
  p.groots_x = p.groots_y = nullptr;
  for (int k = 0; k < 2; ++k) {
    cudaFree(p.tw_x[k]);
    cudaFree(p.tw_y[k]);
    p.tw_x[k] = p.tw_y[k] = nullptr;
  }
  cudaFree(p.circle); cudaFree(p.phase); cudaFree(p.mask);
  p.circle = nullptr;
  p.phase = nullptr;
  p.mask = nullptr;
}

template <class K>
static cudaError_t set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

HOLO_CHECK_TU(check_bits_kernels)

cudaError_t fft_rows(const Plan& p, const float2* in, float2* out, long long nrows, bool inverse, float scale,
                     cudaStream_t s, const uint8_t* live, int rows_per_plane) {
  if (live && (rows_per_plane <= 0 || nrows >= (1LL << 31))) return cudaErrorInvalidValue;
  if (p.generic_x) return g_fft_rows(p, in, out, nrows, inverse, scale, s, live, rows_per_plane);
  cudaError_t err = cudaSuccess;
  const bool ok = dispatch_n(p.nx, [&](auto nc) {
    constexpr int N = decltype(nc)::value;
    constexpr int E = EBig<N>::value;
    using Sh = FftShape<N, E>;
    constexpr int NT = row_threads<E>();
    constexpr int RPC = NT / Sh::TPF;
    const size_t smem = sizeof(float2) * (row_tw_f2<N, E>() + (size_t)RPC * Sh::PADN);
    const int grid = grid_for((nrows + RPC - 1) / RPC, 1, 148 * 64);
    if (inverse) {
      err = set_smem(k_fft_rows<N, true, E>, smem);
      k_fft_rows<N, true, E><<<grid, NT, smem, s>>>(in, out, nrows, scale, p.tw_x[tw_slot<E>()], live,
                                                                  rows_per_plane);
  COUNT_LAUNCH(1);
    } else {
      err = set_smem(k_fft_rows<N, false, E>, smem);
      k_fft_rows<N, false, E><<<grid, NT, smem, s>>>(in, out, nrows, scale, p.tw_x[tw_slot<E>()], live,
                                                                  rows_per_plane);
  COUNT_LAUNCH(1);
    }
  });
  if (!ok) return cudaErrorInvalidValue;
  return err ? err : cudaGetLastError();
}

// 2D tiled tensor map over float32 rows (inner = floats per row, rows), box
// box_inner x box_rows; nonzero on failure.  The driver entry point is looked
// up at run time (no libcuda link dependency).
int encode_tiled_2d(CUtensorMap* m, const void* base, long long inner, long long rows, int box_inner, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return 1;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)inner * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS;
}

template <int N, int C, int E>
static size_t col_smem(int extra) {
  return sizeof(float2) * (2 * N + extra + (size_t)(N + N / E) * C);
}

cudaError_t fft_cols(const Plan& p, const float2* in, float2* out, int nplanes, bool inverse, float scale,
                     cudaStream_t s) {
  if (p.generic_y) return g_fft_cols(p, in, out, nplanes, inverse, scale, s);
  cudaError_t err = cudaSuccess;
  const bool ok = dispatch_n(p.ny, [&](auto nc) {
    constexpr int N = decltype(nc)::value;
    constexpr int E = DefaultE<N>::value;  // radix-32 columns measured slower (occupancy)
    constexpr int C = N >= 4096 ? 4 : 8;
    constexpr int NT = C * FftShape<N, E>::TPF;
    const size_t smem = col_smem<N, C, E>(0);
    dim3 grid(p.nx / C, nplanes);
    if (inverse) {
      err = set_smem(k_fft_cols<N, true, C, E>, smem);
      k_fft_cols<N, true, C, E><<<grid, NT, smem, s>>>(in, out, p.nx, p.P, scale, p.tw_y[tw_slot<E>()]);
    } else {
      err = set_smem(k_fft_cols<N, false, C, E>, smem);
      k_fft_cols<N, false, C, E><<<grid, NT, smem, s>>>(in, out, p.nx, p.P, scale, p.tw_y[tw_slot<E>()]);
    }
    COUNT_LAUNCH(1);
  });
  if (!ok) return cudaErrorInvalidValue;
  return err ? err : cudaGetLastError();
}

// planes per CTA in the column passes = H_k recurrence length (error bound)
constexpr int kMaxRecur = 32;
#define HOLO_ADJ_PPC kMaxRecur
// 4 columns (256 threads) per CTA: with R / phase held in registers across the
// CTA's planes (126 registers) two CTAs fit per SM (measured best at 1024^2)
#ifndef HOLO_ADJ_CC
#define HOLO_ADJ_CC 4
#endif
#define HOLO_ADJ_C(N) HOLO_ADJ_CC
// staged (N <= 1024): 2 columns per CTA, 3 CTAs per SM (see k_fwd_cols_staged);
// direct loads (N > 1024): 4 columns, 32-byte row segments per warp load
#ifndef HOLO_FWD_CC
#define HOLO_FWD_CC 2
#endif
#ifndef HOLO_FWD_STAGED_MAX
#define HOLO_FWD_STAGED_MAX 2048
#endif
#define HOLO_FWD_C(N) ((N) <= HOLO_FWD_STAGED_MAX ? HOLO_FWD_CC : 4)

cudaError_t adj_cols(const Plan& p, const float2* R, float2* out, int nzl, int k0, cudaStream_t s, bool packed) {
  if (p.generic_y) return g_adj_cols(p, R, out, nzl, k0, s, packed);
  cudaError_t err = cudaSuccess;
  const bool ok = dispatch_n(p.ny, [&](auto nc) {
    constexpr int N = decltype(nc)::value;
    // 512- and 1024-point columns of the complex engine: radix-32 (one shared-memory
    // exchange and one table-twiddle pass instead of two; 236 registers, 2 CTAs of
    // 128 threads per SM): C3 adjoint columns 10.97 -> 9.58 ms per 10 iterations.
    // The packed real engine carries a second recurrence (rb[]) and keeps radix 16.
    auto launch = [&](auto cc, auto ee) {
      constexpr int C = decltype(cc)::value;  // C x 8-byte row segments per warp load / store
      constexpr int E = decltype(ee)::value;
      constexpr int NT = C * FftShape<N, E>::TPF;
      const size_t smem =
          col_smem<N, C, E>(256) + (adj_separate_stage<N, C, E>() ? sizeof(float2) * ((size_t)N * C + 16) : 0);
      // planes per CTA: >= ~8 waves of CTAs in the grid
      const long long blocks = p.nx / C;
      const int ppc = (int)std::max(1LL, std::min<long long>(HOLO_ADJ_PPC, blocks * nzl / (148LL * 8)));
      dim3 grid(p.nx / C, (nzl + ppc - 1) / ppc);
      CUtensorMap map;
      if (encode_tiled_2d(&map, out, 2 * p.nx, (long long)nzl * p.ny, 2 * C, N < 256 ? N : 256)) {
        err = cudaErrorInvalidValue;
        return;
      }
      auto go = [&](auto kern) {
        if ((err = set_smem(kern, smem))) return;
        kern<<<grid, NT, smem, s>>>(R, map, p.nx, p.ny, k0, nzl, ppc, p.phase, p.tw_y[tw_slot<E>()], p.circle);
      };
      if constexpr (E == DefaultE<N>::value) {
        if (packed)
          go(k_adj_cols<N, C, E, true>);
        else
          go(k_adj_cols<N, C, E>);
      } else {
        go(k_adj_cols<N, C, E>);
      }
    };
    constexpr int E32 = (N == 512 || N == 1024) ? 32 : DefaultE<N>::value;
    if (!packed && E32 == 32 && !std::getenv("HOLO_ADJ_E16"))
      launch(std::integral_constant<int, HOLO_ADJ_C(N)>(), std::integral_constant<int, E32>());  // nx >= 8 always
    else
      launch(std::integral_constant<int, HOLO_ADJ_C(N)>(), std::integral_constant<int, DefaultE<N>::value>());
    COUNT_LAUNCH(1);
  });
  if (!ok) return cudaErrorInvalidValue;
  return err ? err : cudaGetLastError();
}

int fwd_groups(const Plan& p, int nzl) {
  const int tiles = std::max(1, p.nx / HOLO_FWD_C(p.ny));
  int g = (16 * 148 + tiles - 1) / tiles;  // ~8 waves of 2 CTAs/SM: small tail
  g = std::max(g, (nzl + kMaxRecur - 1) / kMaxRecur);  // H_k recurrence length <= kMaxRecur planes
  g = std::max(1, std::min(g, nzl));
  return std::min(g, 64);
}

cudaError_t fwd_cols(const Plan& p, const float2* in, float2* Spart, int nzl, int k0, int groups, cudaStream_t s,
                     bool packed, const uint8_t* live) {
  if (p.generic_y) return g_fwd_cols(p, in, Spart, nzl, k0, groups, s, packed, live);
  cudaError_t err = cudaSuccess;
  const int ppg = (nzl + groups - 1) / groups;
  const bool ok = dispatch_n(p.ny, [&](auto nc) {
    constexpr int N = decltype(nc)::value;
    constexpr int E = DefaultE<N>::value;  // acc[] + v[] per thread
    constexpr int C = HOLO_FWD_C(N);  // acc[] + v[] stay in registers at <= 128 per thread
    constexpr int NT = C * FftShape<N, E>::TPF;
    dim3 grid(p.nx / C, groups);
    if constexpr (N <= HOLO_FWD_STAGED_MAX) {
      CUtensorMap map;
      if (encode_tiled_2d(&map, in, 2 * p.nx, (long long)nzl * p.ny, 2 * C, N < 256 ? N : 256)) {
        err = cudaErrorInvalidValue;
        return;
      }
      const size_t smem = col_smem<N, C, E>(256) + sizeof(float2) * 2 * N * C;
      auto go = [&](auto kern) {
        if ((err = set_smem(kern, smem))) return;
        kern<<<grid, NT, smem, s>>>(map, Spart, p.nx, p.P, p.ny, nzl, ppg, k0, p.phase, p.tw_y[tw_slot<E>()],
                                    p.circle, live);
      };
      if (packed)
        go(k_fwd_cols_staged<N, C, E, true>);
      else
        go(k_fwd_cols_staged<N, C, E>);
    } else {
      const size_t smem = col_smem<N, C, E>(256);
      auto go = [&](auto kern) {
        if ((err = set_smem(kern, smem))) return;
        kern<<<grid, NT, smem, s>>>(in, Spart, p.nx, p.P, nzl, ppg, k0, p.phase, p.tw_y[tw_slot<E>()], p.circle,
                                    live);
      };
      if (packed)
        go(k_fwd_cols<N, C, E, true>);
      else
        go(k_fwd_cols<N, C, E>);
    }
  COUNT_LAUNCH(1);
  });
  if (!ok) return cudaErrorInvalidValue;
  return err ? err : cudaGetLastError();
}

cudaError_t sum_groups(const Plan& p, const float2* Spart, int groups, float2* S, cudaStream_t s) {
  k_sum_groups<<<grid_for(p.P, kEltThreads), kEltThreads, 0, s>>>(Spart, groups, p.P, S);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

int sensor_blocks(const Plan& p) { return grid_for(p.P, kSensorThreads, 148 * 4); }

cudaError_t sensor(const Plan& p, const float2* Sa, const float2* Sb, float ca, float cb, const float2* B,
                   float2* Rout, double* part, cudaStream_t s) {
  k_sensor<<<sensor_blocks(p), kSensorThreads, 0, s>>>(Sa, Sb, ca, cb, B, p.mask, Rout, p.ny, p.nx, part);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t final_sum(const double* part, int n, double scale, double* out, cudaStream_t s) {
  k_final_sum<256><<<1, 256, 0, s>>>(part, n, scale, out);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

size_t prox_setup(ProxArgs& a, int ny, int nx, int inner) {
  if (prox_strip_applicable(ny, nx, inner) && !getenv("HOLO_PROX_GENERIC")) {
    prox_strip_setup(a, ny, nx, inner);
    a.kind = 1;
    return 0;
  }
  a.kind = 0;
  a.ny = ny;
  a.nx = nx;
  a.P = (long long)ny * nx;
  a.inner = inner;
  a.halo = inner + 2;
  const int cap = kProxThreads * kProxMaxPx;
  int side = 1;
  while ((side + 1 + 2 * a.halo) * (side + 1 + 2 * a.halo) <= cap && side < 64) ++side;
  a.tile = side;
  a.tiles_x = (nx + side - 1) / side;
  const int tiles_y = (ny + side - 1) / side;
  a.tiles_per_plane = a.tiles_x * tiles_y;
  const int ew = std::min(nx, side + 2 * a.halo), eh = std::min(ny, side + 2 * a.halo);
  return sizeof(float) * 6 * (size_t)ew * eh;
}

bool prox_supported(int ny, int nx, int inner) {
  ProxArgs a;
  prox_setup(a, ny, nx, inner);
  if (a.kind == 1) return true;
  const int ew = std::min(nx, a.tile + 2 * a.halo), eh = std::min(ny, a.tile + 2 * a.halo);
  return ew * eh <= kProxThreads * kProxMaxPx;
}

cudaError_t prox(const ProxArgs& a, cudaStream_t s) {
  if (a.kind == 1) {
    if (!a.pass_len || !(a.tau_tv > 0.f)) {  // no TV: nothing to split into passes
      COUNT_LAUNCH(1);
      cudaError_t e = prox_strip(a, s);
      if (!e && prox_tvfix_launch(a)) {
        k_prox_tvfix<<<dim3(a.tiles_per_plane, a.nplanes), 64, 0, s>>>(a);
        COUNT_LAUNCH(1);
        e = cudaGetLastError();
      }
      return e;
    }
    if (!a.vbuf || !a.sbuf || !a.rbuf || !a.tvv) return cudaErrorInvalidValue;
    // guard fix-up (force): the state of every pass is still in HBM, rerun the last
    const int last0 = ((a.inner - 1) / a.pass_len) * a.pass_len;
    for (int t0 = a.force ? last0 : 0; t0 < a.inner; t0 += a.pass_len) {
      ProxArgs b = a;
      b.t0 = t0;
      b.t1 = std::min(a.inner, t0 + a.pass_len);
      COUNT_LAUNCH(1);
      cudaError_t e = prox_strip(b, s);
      if (e) return e;
    }
    return cudaSuccess;
  }
  const int ew = std::min(a.nx, a.tile + 2 * a.halo), eh = std::min(a.ny, a.tile + 2 * a.halo);
  if (ew * eh > kProxThreads * kProxMaxPx) return cudaErrorInvalidValue;
  const size_t smem = sizeof(float) * 6 * (size_t)ew * eh;
  cudaError_t err = set_smem(k_prox<kProxThreads, kProxMaxPx>, smem);
  if (err) return err;
  dim3 grid(a.tiles_per_plane, a.nplanes);
  k_prox<kProxThreads, kProxMaxPx><<<grid, kProxThreads, smem, s>>>(a);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t prox_reduce(const ProxArgs& a, double tau_tv, int tv_on, uint8_t* force_acc, double* plane_out,
                        int* new_fail, cudaStream_t s, uint8_t* live, int skip_ok) {
  k_prox_reduce<<<a.nplanes, kReduceThreads, 0, s>>>(a.part, a.tiles_per_plane, a.kind == 1 ? a.part_warps : 0,
                                                     tau_tv, tv_on, force_acc, plane_out, new_fail, live, skip_ok,
                                                     a.force, prox_tvfix_launch(a) ? a.bpart : nullptr);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t plane_total(const double* plane_out, const int* new_fail, int nplanes, double* scalars, cudaStream_t s,
                        const uint8_t* live) {
  k_plane_total<<<1, kReduceThreads, 0, s>>>(plane_out, new_fail, nplanes, scalars, live);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t load_hologram(const double* b, float2* bc, long long P, double* part, int* nblocks, cudaStream_t s) {
  const int g = grid_for(P, kEltThreads, 148 * 4);
  *nblocks = g;
  k_load_hologram<<<g, kEltThreads, 0, s>>>(b, bc, P, part);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

// packed real engine (engine.cu): zero the dummy Im part; unpack a stack of
// nzl real planes (plane 2k = Re of stack plane k, 2k+1 = Im) to one complex
// plane each (Im = 0)
__global__ void k_zero_imag(float2* __restrict__ x, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i].y = 0.f;
}
__global__ void k_unpack_real(const float2* __restrict__ x, float2* __restrict__ out, int nzl, long long P) {
  const long long n = (long long)((nzl + 1) / 2) * P;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long k = i / P, e = i - k * P;
    const float2 v = x[i];
    out[2 * k * P + e] = make_float2(v.x, 0.f);
    if (2 * k + 1 < nzl) out[(2 * k + 1) * P + e] = make_float2(v.y, 0.f);
  }
}
cudaError_t zero_imag(float2* x, long long n, cudaStream_t s) {
  k_zero_imag<<<grid_for(n, kEltThreads, 148 * 8), kEltThreads, 0, s>>>(x, n);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}
cudaError_t unpack_real(const float2* x, float2* out, int nzl, long long P, cudaStream_t s) {
  k_unpack_real<<<grid_for((long long)((nzl + 1) / 2) * P, kEltThreads, 148 * 8), kEltThreads, 0, s>>>(x, out, nzl, P);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t real_part(const float2* in, float* out, long long n, float scale, cudaStream_t s) {
  k_real_part<<<grid_for(n, kEltThreads), kEltThreads, 0, s>>>(in, out, n, scale);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t real_to_complex(const float* in, float2* out, long long n, cudaStream_t s) {
  k_real_to_complex<<<grid_for(n, kEltThreads), kEltThreads, 0, s>>>(in, out, n);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t apply_mask(const Plan& p, float2* spec, int nplanes, cudaStream_t s) {
  const long long n = p.P * nplanes;
  k_apply_mask<<<grid_for(n, kEltThreads), kEltThreads, 0, s>>>(spec, p.mask, p.P, n);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t transfer_stack(const Plan& p, int k0, int k1, bool conj, float2* out, cudaStream_t s) {
  const long long n = p.P * (k1 - k0);
  k_transfer<<<grid_for(n, kEltThreads), kEltThreads, 0, s>>>(p.phase, p.mask, p.circle, p.P, k0, k1 - k0,
                                                              conj ? 1 : 0, out);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t spec_combine(const Plan& p, const float2* Sa, const float2* Sb, float ca, float cb, float2* out,
                         cudaStream_t s) {
  k_spec_combine<<<grid_for(p.P, kEltThreads), kEltThreads, 0, s>>>(Sa, Sb, ca, cb, out, p.P);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t real_opnorm(const Plan& p, int nz, double* d_out, cudaStream_t s) {
  const int nb = 148 * 2;
  double* part = nullptr;
  cudaError_t e = cudaMallocAsync(&part, sizeof(double) * nb, s);
  if (e) return e;
  k_real_opnorm<<<nb, 256, 0, s>>>(p.phase, p.mask, p.circle, p.P, nz, part);
  COUNT_LAUNCH(1);
  k_max_final<<<1, 32, 0, s>>>(part, nb, d_out);
  COUNT_LAUNCH(1);
  cudaFreeAsync(part, s);
  return cudaGetLastError();
}

int vol_norm2_blocks(long long n) { return grid_for(n, 256, 148 * 4); }

cudaError_t vol_norm2(const float2* x, long long n, double* part, cudaStream_t s) {
  k_vol_norm2<<<vol_norm2_blocks(n), 256, 0, s>>>(x, n, part);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t vol_rescale(float2* x, long long n, const double* nrm2, int real, cudaStream_t s) {
  k_vol_rescale<<<grid_for(n, 256), 256, 0, s>>>(x, n, nrm2, real);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

int coo_chunks(long long P, int nplanes) { return (int)((P + kCooChunk - 1) / kCooChunk) * nplanes; }

cudaError_t coo_count(const float2* x, long long P, int nplanes, int* chunk_counts, cudaStream_t s) {
  const int cpp = (int)((P + kCooChunk - 1) / kCooChunk);
  k_coo_count<<<dim3(cpp, nplanes), kCooThreads, 0, s>>>(x, P, cpp, chunk_counts);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

cudaError_t coo_compact(const float2* x, long long P, int nx, int nplanes, const long long* chunk_offsets, int* rows,
                        int* cols, float2* vals, double2* vals64, cudaStream_t s) {
  const int cpp = (int)((P + kCooChunk - 1) / kCooChunk);
  k_coo_compact<<<dim3(cpp, nplanes), kCooThreads, 0, s>>>(x, P, nx, cpp, chunk_offsets, rows, cols, vals, vals64);
  COUNT_LAUNCH(1);
  return cudaGetLastError();
}

}  // namespace holo
