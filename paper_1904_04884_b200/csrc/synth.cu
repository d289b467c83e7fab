// Input side: GPU hologram rendering and background removal.
//
// render: synth.py:161-181 computes spec = sum_p fft2(mask_p) * H(-z_p), one
// full-plane FFT per particle (0.1 s/particle on the CPU).  A particle's mask
// is a handful of pixels, so fft2(mask_p)(f) = sum_pix a_p exp(-2 pi i (fy y /
// ny + fx x / nx)) is a short sum of exact-rational twiddles, and the spectrum
// is accumulated per frequency, particle by particle in the reference's order,
// in fp64 (the reference's precision): phase (z_p / lam) * sqrt(arg) in fp64,
// cis by sincospi.  The caller inverts with holo_op_fft2.
//
// background: preprocess.py:17-38 (I - M) / sqrt(M), M the sliding temporal
// mean excluding the frame itself, window truncated at the stack ends.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/holo_b200.h"

namespace holo {
namespace {

constexpr int kRenderThreads = 256;
constexpr int kBatch = 128;  // particles staged in shared memory per pass

// exp(-2 pi i t / n), t < n, fp64
__global__ void k_unit_roots(double2* __restrict__ w, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    double sn, cs;
    sincospi(-2.0 * (double)t / (double)n, &sn, &cs);
    w[t] = make_double2(cs, sn);
  }
}

__global__ void __launch_bounds__(kRenderThreads) k_render_spectrum(
    const double* __restrict__ zl, const int32_t* __restrict__ pix_off, const int32_t* __restrict__ pix_yx,
    const double* __restrict__ pix_a, int n, int ny, int nx, double pitch, double lam,
    const double2* __restrict__ wy, const double2* __restrict__ wx, double2* __restrict__ spec) {
  __shared__ double s_zl[kBatch];
  __shared__ int s_off[kBatch + 1];
  const long long P = (long long)ny * nx;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = p < P;
  int iy = 0, ix = 0;
  double root = 0.0;
  bool prop = false;
  if (active) {
    iy = (int)(p / nx);
    ix = (int)(p - (long long)iy * nx);
    const int ky = (iy <= (ny - 1) / 2) ? iy : iy - ny, kx = (ix <= (nx - 1) / 2) ? ix : ix - nx;
    const double fy = (double)ky * (1.0 / ((double)ny * pitch)), fx = (double)kx * (1.0 / ((double)nx * pitch));
    const double arg = 1.0 - (lam * fx) * (lam * fx) - (lam * fy) * (lam * fy);
    prop = arg >= 0.0;
    root = prop ? sqrt(arg) : 0.0;
  }
  const bool pow2y = (ny & (ny - 1)) == 0, pow2x = (nx & (nx - 1)) == 0;  // iy*y < 2^31 for n <= 46340
  double re = 0.0, im = 0.0;
  for (int b0 = 0; b0 < n; b0 += kBatch) {
    const int nb = min(kBatch, n - b0);
    __syncthreads();
    for (int t = threadIdx.x; t < nb; t += blockDim.x) s_zl[t] = zl[b0 + t];
    for (int t = threadIdx.x; t <= nb; t += blockDim.x) s_off[t] = pix_off[b0 + t];
    __syncthreads();
    if (!active || !prop) continue;
    for (int q = 0; q < nb; ++q) {
      // mask spectrum: sum over the particle's pixels of a * exp(-2 pi i (iy y / ny + ix x / nx))
      double mr = 0.0, mi = 0.0;
      for (int e = s_off[q]; e < s_off[q + 1]; ++e) {
        const int y = pix_yx[2 * e], x = pix_yx[2 * e + 1];
        // exact rational phase: (iy*y mod ny)/ny + (ix*x mod nx)/nx, in units of pi
        const int ty = pow2y ? ((iy * y) & (ny - 1)) : (iy * y) % ny;
        const int tx = pow2x ? ((ix * x) & (nx - 1)) : (ix * x) % nx;
        const double2 a = __ldg(wy + ty), b = __ldg(wx + tx);
        const double cr = a.x * b.x - a.y * b.y, ci = a.x * b.y + a.y * b.x;
        mr = fma(pix_a[e], cr, mr);
        mi = fma(pix_a[e], ci, mi);
      }
      // H(-z) = exp(-i 2 pi (z / lam) root)
      const double ph = s_zl[q] * root;
      double hs, hc;
      sincospi(-2.0 * (ph - floor(ph)), &hs, &hc);
      re += mr * hc - mi * hs;
      im += mr * hs + mi * hc;
    }
  }
  if (active) spec[p] = make_double2(re, im);
}

__global__ void k_background(const double* __restrict__ img, long long P, int T, int half, double floor_,
                             double* __restrict__ out) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    // running window sum over frames [lo, hi) with the frame itself excluded
    double sum = 0.0;
    int lo = 0, hi = 0;
    for (int t = 0; t < T; ++t) {
      const int nlo = max(0, t - half), nhi = min(T, t + half + 1);
      while (hi < nhi) sum += img[(long long)(hi++) * P + p];
      while (lo < nlo) sum -= img[(long long)(lo++) * P + p];
      const double cur = img[(long long)t * P + p];
      const double mean = (sum - cur) / (double)(hi - lo - 1);
      out[(long long)t * P + p] = (cur - mean) / sqrt(fmax(mean, floor_));
    }
  }
}

}  // namespace
}  // namespace holo

extern "C" int holo_render_spectrum(const double* z_over_lam, const int32_t* pix_off, const int32_t* pix_yx,
                                    const double* pix_a, int32_t n, int32_t ny, int32_t nx, double pitch,
                                    double wavelength, void* spec, void* stream) {
  if (n < 0 || ny < 1 || nx < 1 || ny > 46340 || nx > 46340 || !(pitch > 0) || !(wavelength > 0) || !spec)
    return HOLO_ERR_INVALID;
  if (n > 0 && (!z_over_lam || !pix_off || !pix_yx || !pix_a)) return HOLO_ERR_INVALID;
  const long long P = (long long)ny * nx;
  cudaStream_t s = (cudaStream_t)stream;
  double2 *wy = nullptr, *wx = nullptr;
  if (cudaMallocAsync(&wy, sizeof(double2) * ny, s) || cudaMallocAsync(&wx, sizeof(double2) * nx, s))
    return HOLO_ERR_CUDA;
  holo::k_unit_roots<<<(ny + 255) / 256, 256, 0, s>>>(wy, ny);
  holo::k_unit_roots<<<(nx + 255) / 256, 256, 0, s>>>(wx, nx);
  const int grid = (int)((P + holo::kRenderThreads - 1) / holo::kRenderThreads);
  holo::k_render_spectrum<<<grid, holo::kRenderThreads, 0, s>>>(z_over_lam, pix_off, pix_yx, pix_a, n, ny, nx, pitch,
                                                                   wavelength, wy, wx, (double2*)spec);
  cudaFreeAsync(wy, s);
  cudaFreeAsync(wx, s);
  return cudaGetLastError() == cudaSuccess ? HOLO_OK : HOLO_ERR_CUDA;
}

extern "C" int holo_background(const double* images, int32_t T, int32_t ny, int32_t nx, int32_t window, double* out,
                               void* stream) {
  if (!images || !out || ny < 1 || nx < 1 || window % 2 != 1 || window < 3 || window > T) return HOLO_ERR_INVALID;
  const long long P = (long long)ny * nx;
  const int grid = (int)std::min<long long>((P + 255) / 256, 148 * 16);
  holo::k_background<<<grid, 256, 0, (cudaStream_t)stream>>>(images, P, T, window / 2, 1e-12, out);
  return cudaGetLastError() == cudaSuccess ? HOLO_OK : HOLO_ERR_CUDA;
}
