// General plane sizes: mixed-radix transforms for planes whose sides are not
// powers of two (the reference's numpy FFTs take any size, optics.py:119-122,
// solver.py:117-132).  The power-of-two path (fft.cuh, the fused TMA column
// passes) stays the production path; a plane with a side that is not a power
// of two runs every pass through the kernels below instead, with the same
// semantics as fft_rows / fft_cols / adj_cols / fwd_cols (kernels.cuh):
//
//  * each line (row or column) is transformed in shared memory by a Stockham
//    autosort over the factors of N (radix 8, then 4, for the 2s): stage
//    (R, Ns) maps butterfly j to outputs (j / Ns) Ns R + j % Ns + q Ns with the
//    combined twiddle W_N^(r (j % Ns + q Ns) N / (Ns R)) from one fp64-exact
//    table of the N roots of unity: a stage twiddle per input, then an
//    in-register radix-2/3/4/8 (closed form) or radix-5/7 (table) DFT; a larger
//    prime factor R gives each thread one output of R table MACs over
//    re-read inputs (a prime side is a direct DFT of its lines);
//  * the adjoint multiplies R by the plane weight U_k on the load (complex
//    engine: H_{k0+k}; packed real engine: Re H_j + i Re H_{j+1}, j = k0 + 2k),
//    the forward accumulates colFFT(v_k) conj(U_k) over a CTA's plane group in
//    registers (no Horner recurrence: U_k is evaluated exactly per plane
//    from the 64-bit phase), all-zero planes (live[k] == 0) skipped.
//
// Throughput is not the point of this path (the lines are smem-latency bound);
// it exists so that any camera frame (1000x1000, 1280x1024, ...) reconstructs
// on the GPU with the reference's results.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace holo {

namespace {

constexpr int kGThreads = 256;
#ifndef HOLO_GLINE
#define HOLO_GLINE 4096  // 2048 (more CTAs per SM, half-sector column segments) measured 7-20 % slower
#endif
constexpr int kGLineElems = HOLO_GLINE;  // target elements per CTA (lines x N; one line if N is larger)
constexpr int kGMaxN = 4096;

// per-stage constants; m*: exact reciprocals for x < 2^12 (q = umulhi(x, m), d >= 2)
struct Radices {
  int n = 0;
  int r[24] = {};
  int M[24] = {}, Ns[24] = {}, step[24] = {};
  unsigned mM[24] = {}, mNs[24] = {}, mR[24] = {};
};

unsigned magic(int d) { return d >= 2 ? (unsigned)((0x100000000ull + (unsigned long long)d - 1) / (unsigned long long)d) : 0u; }

Radices factor(int N) {
  Radices f;
  int n = N;
  while (n % 8 == 0 && n > 8) { f.r[f.n++] = 8; n /= 8; }
  while (n % 4 == 0 && n > 4) { f.r[f.n++] = 4; n /= 4; }
  for (int p = 2; n > 1; ++p)
    while (n % p == 0) { f.r[f.n++] = p; n /= p; }
  int ns = 1;
  for (int s = 0; s < f.n; ++s) {
    f.M[s] = N / f.r[s];
    f.Ns[s] = ns;
    f.step[s] = N / (ns * f.r[s]);
    f.mM[s] = magic(f.M[s]);
    f.mNs[s] = magic(ns);
    f.mR[s] = magic(f.r[s]);
    ns *= f.r[s];
  }
  return f;
}

// x / d for 0 <= x < 2^12 (d = 1: x)
__device__ __forceinline__ int udiv(int x, int d, unsigned m) { return d == 1 ? x : (int)__umulhi((unsigned)x, m); }

int largest_prime(int N) {
  int best = 1, n = N;
  for (int p = 2; n > 1; ++p)
    while (n % p == 0) { best = p; n /= p; }
  return best;
}

// W[m] = exp(-2 pi i m / N), fp64 argument reduced exactly
__global__ void k_groots(float2* W, int N) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= N) return;
  double s, c;
  sincospi(-2.0 * (double)m / (double)N, &s, &c);
  W[m] = make_float2((float)c, (float)s);
}

HD float2 conj_if(float2 w, bool inv) { return inv ? make_float2(w.x, -w.y) : w; }

// In-register butterfly of radix R (R = 2, 3, 4 closed form; others by table):
// x_r <- x_r W_N^(r jm step) (stage twiddle), then y_q = sum_r x_r W_R^(r q).
template <int R>
__device__ __forceinline__ void bfly(const float2* sl, float2* dl, int j, int M, int jm, int Ns, int step, int base,
                                     const float2* W, bool inv, int N) {
  float2 x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) x[r] = sl[j + r * M];
  const int e = jm * step;
  int m = e;
#pragma unroll
  for (int r = 1; r < R; ++r) {
    x[r] = cmul(x[r], conj_if(W[m], inv));
    m += e;
    if (m >= N) m -= N;
  }
  if constexpr (R == 2) {
    const float2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const float2 a = cadd(x[0], x[2]), b = csub(x[0], x[2]), c = cadd(x[1], x[3]), d = csub(x[1], x[3]);
    const float2 di = inv ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);  // W_4 d = -+ i d
    x[0] = cadd(a, c);
    x[2] = csub(a, c);
    x[1] = cadd(b, di);
    x[3] = csub(b, di);
  } else if constexpr (R == 8) {  // two 4-point DFTs (even / odd inputs) and W_8^q
    float2 ev[4] = {x[0], x[2], x[4], x[6]}, od[4] = {x[1], x[3], x[5], x[7]};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float2* v = h ? od : ev;
      const float2 a = cadd(v[0], v[2]), b = csub(v[0], v[2]), c = cadd(v[1], v[3]), d = csub(v[1], v[3]);
      const float2 di = inv ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);
      v[0] = cadd(a, c);
      v[2] = csub(a, c);
      v[1] = cadd(b, di);
      v[3] = csub(b, di);
    }
    const float h = 0.70710678118654752f, sg = inv ? 1.f : -1.f;
    const float2 o1 = make_float2(h * (od[1].x - sg * od[1].y), h * (od[1].y + sg * od[1].x));   // W_8 o1
    const float2 o2 = make_float2(-sg * od[2].y, sg * od[2].x);                                  // W_8^2 o2
    const float2 o3 = make_float2(h * (-od[3].x - sg * od[3].y), h * (-od[3].y + sg * od[3].x));  // W_8^3 o3
    x[0] = cadd(ev[0], od[0]);
    x[4] = csub(ev[0], od[0]);
    x[1] = cadd(ev[1], o1);
    x[5] = csub(ev[1], o1);
    x[2] = cadd(ev[2], o2);
    x[6] = csub(ev[2], o2);
    x[3] = cadd(ev[3], o3);
    x[7] = csub(ev[3], o3);
  } else if constexpr (R == 3) {
    const float sn = inv ? 0.86602540378443865f : -0.86602540378443865f;  // Im W_3
    const float2 t = cadd(x[1], x[2]), u = csub(x[1], x[2]);
    const float2 c = make_float2(fmaf(-0.5f, t.x, x[0].x), fmaf(-0.5f, t.y, x[0].y));
    const float2 iu = make_float2(-sn * u.y, sn * u.x);
    x[0] = cadd(x[0], t);
    x[1] = cadd(c, iu);
    x[2] = csub(c, iu);
  } else {
    float2 y[R];
    const int nr = N / R;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      float2 acc = x[0];
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const float2 w = conj_if(W[((r * q) % R) * nr], inv);
        acc = make_float2(fmaf(x[r].x, w.x, fmaf(-x[r].y, w.y, acc.x)), fmaf(x[r].x, w.y, fmaf(x[r].y, w.x, acc.y)));
      }
      y[q] = acc;
    }
#pragma unroll
    for (int q = 0; q < R; ++q) x[q] = y[q];
  }
#pragma unroll
  for (int q = 0; q < R; ++q) dl[base + q * Ns] = x[q];
}

// large prime radix: one output q of butterfly j per call (so a prime side's
// R outputs spread over R threads), R table MACs re-reading the inputs
__device__ void bfly_one(const float2* sl, float2* dl, int j, int q, int M, int jm, int Ns, int step, int base, int R,
                         const float2* W, bool inv, int N) {
  const int e = (jm + q * Ns) * step;  // < N
  float2 acc = czero();
  int m = 0;
  for (int r = 0; r < R; ++r) {
    const float2 x = sl[j + r * M];
    const float2 w = conj_if(W[m], inv);
    acc = make_float2(fmaf(x.x, w.x, fmaf(-x.y, w.y, acc.x)), fmaf(x.x, w.y, fmaf(x.y, w.x, acc.y)));
    m += e;
    if (m >= N) m -= N;
  }
  dl[base + q * Ns] = acc;
}

// L lines of N points in a (line-major [L][N]); returns the buffer holding the result
__device__ float2* stockham(float2* a, float2* b, int N, int L, const Radices& rad, const float2* W, bool inv) {
  float2* src = a;
  float2* dst = b;
  for (int s = 0; s < rad.n; ++s) {
    const int R = rad.r[s], M = rad.M[s], Ns = rad.Ns[s], step = rad.step[s];
    const unsigned mM = rad.mM[s], mNs = rad.mNs[s];
    if (R <= 8) {
      for (int t = threadIdx.x; t < L * M; t += blockDim.x) {
        const int line = udiv(t, M, mM), j = t - line * M;
        const float2* sl = src + line * N;
        float2* dl = dst + line * N;
        const int jq = udiv(j, Ns, mNs), jm = j - jq * Ns, base = jq * Ns * R + jm;
        switch (R) {
          case 2: bfly<2>(sl, dl, j, M, jm, Ns, step, base, W, inv, N); break;
          case 3: bfly<3>(sl, dl, j, M, jm, Ns, step, base, W, inv, N); break;
          case 4: bfly<4>(sl, dl, j, M, jm, Ns, step, base, W, inv, N); break;
          case 5: bfly<5>(sl, dl, j, M, jm, Ns, step, base, W, inv, N); break;
          case 7: bfly<7>(sl, dl, j, M, jm, Ns, step, base, W, inv, N); break;
          default: bfly<8>(sl, dl, j, M, jm, Ns, step, base, W, inv, N);
        }
      }
    } else {  // prime R > 7: tasks are (line, butterfly, output), L N of them
      const unsigned mR = rad.mR[s];
      for (int t = threadIdx.x; t < L * N; t += blockDim.x) {
        const int lj = udiv(t, R, mR), q = t - lj * R;
        const int line = udiv(lj, M, mM), j = lj - line * M;
        const int jq = udiv(j, Ns, mNs), jm = j - jq * Ns, base = jq * Ns * R + jm;
        bfly_one(src + line * N, dst + line * N, j, q, M, jm, Ns, step, base, R, W, inv, N);
      }
    }
    __syncthreads();
    float2* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

__device__ void load_roots(float2* Ws, const float2* Wg, int N) {
  for (int i = threadIdx.x; i < N; i += blockDim.x) Ws[i] = Wg[i];
}

// plane weight U_k at pixel phase t (see the file comment)
__device__ float2 plane_weight(uint64_t t, int k0, int k, bool packed, const float2* circ) {
  if (packed) {
    const int j = k0 + 2 * k;
    return make_float2(cis_cycles(plane_phase(t, j), circ).x, cis_cycles(plane_phase(t, j + 1), circ).x);
  }
  return cis_cycles(plane_phase(t, k0 + k), circ);
}

// rows: CTA = L consecutive rows of N = nx points
__global__ void __launch_bounds__(kGThreads) k_grows(const float2* in, float2* out, long long nrows, int N, int L,
                                                     Radices rad, const float2* __restrict__ Wg, bool inv,
                                                     float scale, const uint8_t* __restrict__ live,
                                                     int rows_per_plane) {
  extern __shared__ __align__(16) float2 gsm[];
  poison_dyn_smem();
  float2* W = gsm;
  float2* a = gsm + N;
  float2* b = a + (size_t)L * N;
  load_roots(W, Wg, N);
  const long long r0 = (long long)blockIdx.x * L;
  for (int l = 0; l < L; ++l) {
    const long long row = r0 + l;
    const bool on = row < nrows && !(live && !live[row / rows_per_plane]);
    HOLO_DCHECK(!on || (row + 1) * N <= nrows * N, CK_ROWS);
    for (int i = threadIdx.x; i < N; i += blockDim.x) a[l * N + i] = on ? in[row * N + i] : czero();
  }
  __syncthreads();
  const float2* res = stockham(a, b, N, L, rad, W, inv);
  for (int l = 0; l < L; ++l) {
    const long long row = r0 + l;
    if (row < nrows && !(live && !live[row / rows_per_plane]))
      for (int i = threadIdx.x; i < N; i += blockDim.x) out[row * N + i] = cscale(res[l * N + i], scale);
  }
}

// columns: CTA = L adjacent columns of one plane (blockIdx.y), N = ny points:
// out[k] = scale * colFFT(in[k])
__global__ void __launch_bounds__(kGThreads) k_gcols(const float2* in, float2* out, int nx, int N, int L, Radices rad,
                                                     const float2* __restrict__ Wg, bool inv, float scale) {
  extern __shared__ __align__(16) float2 gsm[];
  poison_dyn_smem();
  float2* W = gsm;
  float2* a = gsm + N;
  float2* b = a + (size_t)L * N;
  load_roots(W, Wg, N);
  const int lgL = __ffs(L) - 1;  // L is a power of two
  const int c0 = blockIdx.x * L, k = blockIdx.y;
  const long long P = (long long)nx * N;
  const float2* src = in + (long long)k * P;
  for (int t = threadIdx.x; t < L * N; t += blockDim.x) {
    const int l = t & (L - 1), i = t >> lgL, c = c0 + l;
    a[l * N + i] = c < nx ? src[(long long)i * nx + c] : czero();
  }
  __syncthreads();
  const float2* res = stockham(a, b, N, L, rad, W, inv);
  float2* dst = out + (long long)k * P;
  for (int t = threadIdx.x; t < L * N; t += blockDim.x) {
    const int l = t & (L - 1), i = t >> lgL, c = c0 + l;
    HOLO_DCHECK(i < N, CK_COLS);
    if (c < nx) dst[(long long)i * nx + c] = cscale(res[l * N + i], scale);
  }
}

// adjoint: out[k] = colIFFT(U_k R) for the CTA's planes [kb, ke); R and the
// phase are plane-independent and stay in registers across the planes
__global__ void __launch_bounds__(kGThreads, 2) k_gadj(const float2* __restrict__ R, float2* out, int nx, int N, int L,
                                                       Radices rad, const float2* __restrict__ Wg, int nzl, int ppc,
                                                       const uint64_t* __restrict__ tab,
                                                       const float2* __restrict__ circ, int k0, bool packed) {
  extern __shared__ __align__(16) float2 gsm[];
  poison_dyn_smem();
  float2* W = gsm;
  float2* a = gsm + N;
  float2* b = a + (size_t)L * N;
  load_roots(W, Wg, N);
  const int lgL = __ffs(L) - 1;  // L is a power of two
  const int c0 = blockIdx.x * L, kb = blockIdx.y * ppc, ke = min(nzl, kb + ppc);
  const long long P = (long long)nx * N;
  constexpr int kReg = (kGLineElems > kGMaxN ? kGLineElems : kGMaxN) / kGThreads;
  float2 rv[kReg];
  uint64_t ph[kReg];
#pragma unroll
  for (int n = 0; n < kReg; ++n) {
    const int t = threadIdx.x + n * kGThreads;
    const int l = t & (L - 1), i = t >> lgL, c = c0 + l;
    const bool on = t < L * N && c < nx;
    rv[n] = on ? R[(long long)i * nx + c] : czero();
    ph[n] = on ? tab[(long long)i * nx + c] : 0ull;
  }
  for (int k = kb; k < ke; ++k) {
    __syncthreads();  // the previous plane's result buffer has been stored
#pragma unroll
    for (int n = 0; n < kReg; ++n) {
      const int t = threadIdx.x + n * kGThreads;
      const int l = t & (L - 1), i = t >> lgL;
      if (t < L * N) a[l * N + i] = cmul(rv[n], plane_weight(ph[n], k0, k, packed, circ));
    }
    __syncthreads();
    const float2* res = stockham(a, b, N, L, rad, W, true);
    float2* dst = out + (long long)k * P;
    for (int t = threadIdx.x; t < L * N; t += blockDim.x) {
      const int l = t & (L - 1), i = t >> lgL, c = c0 + l;
      HOLO_DCHECK(i < N && k < nzl, CK_COLS);
      if (c < nx) dst[(long long)i * nx + c] = res[l * N + i];
    }
  }
}

// forward: Spart[g] = sum_{k in group g, live} colFFT(in[k]) conj(U_k)
__global__ void __launch_bounds__(kGThreads, 3) k_gfwd(const float2* in, float2* Spart, int nx, int N, int L, Radices rad,
                                                    const float2* __restrict__ Wg, int nzl, int ppg,
                                                    const uint64_t* __restrict__ tab,
                                                    const float2* __restrict__ circ, int k0, bool packed,
                                                    const uint8_t* __restrict__ live) {
  extern __shared__ __align__(16) float2 gsm[];
  poison_dyn_smem();
  float2* W = gsm;
  float2* a = gsm + N;
  float2* b = a + (size_t)L * N;
  load_roots(W, Wg, N);
  const int lgL = __ffs(L) - 1;  // L is a power of two
  const int c0 = blockIdx.x * L, kb = blockIdx.y * ppg, ke = min(nzl, kb + ppg);
  const long long P = (long long)nx * N;
  // the plane sum stays in registers: thread owns elements t = threadIdx.x + n blockDim.x
  constexpr int kAcc = (kGLineElems > kGMaxN ? kGLineElems : kGMaxN) / kGThreads;
  float2 acc[kAcc];
#pragma unroll
  for (int n = 0; n < kAcc; ++n) acc[n] = czero();
  for (int k = kb; k < ke; ++k) {
    if (live && !live[k]) continue;
    __syncthreads();  // the previous plane's accumulate read its result buffer
    for (int t = threadIdx.x; t < L * N; t += blockDim.x) {
      const int l = t & (L - 1), i = t >> lgL, c = c0 + l;
      a[l * N + i] = c < nx ? in[(long long)k * P + (long long)i * nx + c] : czero();
    }
    __syncthreads();
    const float2* res = stockham(a, b, N, L, rad, W, false);
#pragma unroll
    for (int n = 0; n < kAcc; ++n) {
      const int t = threadIdx.x + n * kGThreads;
      const int l = t & (L - 1), i = t >> lgL, c = c0 + l;
      if (t < L * N && c < nx) {
        const float2 u = plane_weight(tab[(long long)i * nx + c], k0, k, packed, circ);
        const float2 v = res[l * N + i];
        acc[n] = cadd(acc[n], make_float2(v.x * u.x + v.y * u.y, v.y * u.x - v.x * u.y));  // v conj(u)
      }
    }
  }
  float2* dst = Spart + (long long)blockIdx.y * P;
#pragma unroll
  for (int n = 0; n < kAcc; ++n) {
    const int t = threadIdx.x + n * kGThreads;
    const int l = t & (L - 1), i = t >> lgL, c = c0 + l;
    HOLO_DCHECK(t >= L * N || i < N, CK_COLS);
    if (t < L * N && c < nx) dst[(long long)i * nx + c] = acc[n];
  }
}

int lines_per_cta(int N) {  // a power of two (t % L, t / L in the column kernels)
  int L = 1;
  while (L < 16 && 2 * L * N <= kGLineElems) L *= 2;
  return L;
}

size_t smem_bytes(int N, int L, int bufs) { return sizeof(float2) * ((size_t)N + (size_t)bufs * L * N); }

template <class K>
cudaError_t allow_smem(K kern, size_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

HOLO_CHECK_TU(check_bits_gfft)

bool pow2_side(int n) { return n >= 8 && n <= 4096 && (n & (n - 1)) == 0; }

bool generic_side(int n) { return n >= 8 && n <= 4096 && largest_prime(n) <= kMaxPrime; }

cudaError_t gplan_build(Plan& p, cudaStream_t s) {
  cudaError_t e;
  if ((e = cudaMalloc(&p.groots_x, sizeof(float2) * p.nx))) return e;
  if ((e = cudaMalloc(&p.groots_y, sizeof(float2) * p.ny))) return e;
  k_groots<<<(p.nx + 255) / 256, 256, 0, s>>>(p.groots_x, p.nx);
  k_groots<<<(p.ny + 255) / 256, 256, 0, s>>>(p.groots_y, p.ny);
  add_launches(2);
  return cudaGetLastError();
}

cudaError_t g_fft_rows(const Plan& p, const float2* in, float2* out, long long nrows, bool inverse, float scale,
                       cudaStream_t s, const uint8_t* live, int rows_per_plane) {
  const int N = p.nx, L = lines_per_cta(N);
  const size_t smem = smem_bytes(N, L, 2);
  cudaError_t e = allow_smem(k_grows, smem);
  if (e) return e;
  const long long blocks = (nrows + L - 1) / L;
  if (blocks <= 0) return cudaSuccess;
  k_grows<<<(unsigned)blocks, kGThreads, smem, s>>>(in, out, nrows, N, L, factor(N), p.groots_x, inverse, scale, live,
                                                    std::max(rows_per_plane, 1));
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t g_fft_cols(const Plan& p, const float2* in, float2* out, int nplanes, bool inverse, float scale,
                       cudaStream_t s) {
  const int N = p.ny, L = lines_per_cta(N);
  const size_t smem = smem_bytes(N, L, 2);
  cudaError_t e = allow_smem(k_gcols, smem);
  if (e) return e;
  if (nplanes <= 0) return cudaSuccess;
  dim3 grid((p.nx + L - 1) / L, nplanes);
  k_gcols<<<grid, kGThreads, smem, s>>>(in, out, p.nx, N, L, factor(N), p.groots_y, inverse, scale);
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t g_adj_cols(const Plan& p, const float2* R, float2* out, int nzl, int k0, cudaStream_t s, bool packed) {
  const int N = p.ny, L = lines_per_cta(N);
  const size_t smem = smem_bytes(N, L, 2);
  cudaError_t e = allow_smem(k_gadj, smem);
  if (e) return e;
  if (nzl <= 0) return cudaSuccess;
  const int bx = (p.nx + L - 1) / L;
  // plane groups: ~8 waves of 2 CTAs per SM, R and the phase reused across a group
  const int groups = std::max(1, std::min(nzl, (148 * 2 * 8 + bx - 1) / bx));
  const int ppc = (nzl + groups - 1) / groups;
  dim3 grid(bx, (nzl + ppc - 1) / ppc);
  k_gadj<<<grid, kGThreads, smem, s>>>(R, out, p.nx, N, L, factor(N), p.groots_y, nzl, ppc, p.phase, p.circle, k0,
                                       packed);
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t g_fwd_cols(const Plan& p, const float2* in, float2* Spart, int nzl, int k0, int groups, cudaStream_t s,
                       bool packed, const uint8_t* live) {
  const int N = p.ny, L = lines_per_cta(N);
  const size_t smem = smem_bytes(N, L, 2);
  cudaError_t e = allow_smem(k_gfwd, smem);
  if (e) return e;
  groups = std::max(groups, 1);
  const int ppg = std::max(1, (nzl + groups - 1) / groups);
  dim3 grid((p.nx + L - 1) / L, groups);
  k_gfwd<<<grid, kGThreads, smem, s>>>(in, Spart, p.nx, N, L, factor(N), p.groots_y, nzl, ppg, p.phase, p.circle, k0,
                                       packed, live);
  add_launches(1);
  return cudaGetLastError();
}

}  // namespace holo
