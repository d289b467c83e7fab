// Host-side launch interface of the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace holo {

// Device tables for one geometry; built once by plan_build().
struct Plan {
  int nx = 0, ny = 0, nz = 0;  // nz = global plane count (plane index k in the phase)
  long long P = 0;             // ny * nx
  double pitch = 0, dz = 0, z0 = 0, lam = 0;
  int col_c = 8;                // interleaved columns per column-pass CTA
  float4* tw_x[2] = {nullptr, nullptr};  // per-pass (w, conj w) tables for nx: [0] E=16, [1] E=32
  float4* tw_y[2] = {nullptr, nullptr};  // same for ny
  float2* circle = nullptr;     // exp(2 pi i m / 256)
  uint64_t* phase = nullptr;    // per pixel packed (frac(z0 q), frac(dz q)) cycle fractions (plane_phase)
  uint8_t* mask = nullptr;      // per pixel 1 = propagating (arg >= 0)
  int any_propagating = 0;
  // general plane sizes (gfft.cu): a side that is not a power of two runs every
  // pass through the mixed-radix kernels; W_N roots per side
  int generic = 0;    // either side runs gfft.cu
  int generic_x = 0;  // rows (nx not a power of two)
  int generic_y = 0;  // columns (ny not a power of two, or nx not a multiple of the fused passes' 8 columns)
  float2* groots_x = nullptr;
  float2* groots_y = nullptr;
};

constexpr int kProxParts = 6;  // per-tile fp64 partial sums written by the prox kernel
// indices into a tile's partials
// G = tau TV(w) + |w - v|^2 / 2 - tau TV(v) per (re, im) part: the TV guard
// (prox.py:138-147) fires where G > 0; TVX = TV(Re x_new) + TV(Im x_new)
enum ProxPart { PT_G_R = 0, PT_G_I, PT_IP, PT_DX2, PT_L1, PT_TVX };

struct ProxArgs {
  const float2* x = nullptr;     // state x_k
  const float2* xp = nullptr;    // state x_{k-1} (read only if beta != 0)
  const float2* grad = nullptr;  // 2 A^H (A y - b) (nullptr: pure prox of y)
  float2* xnew = nullptr;
  long long P = 0;
  int ny = 0, nx = 0, nplanes = 0;
  float beta = 0.f, step = 0.f;  // y = (1+beta) x - beta xp ; v = y - step * grad
  float tau_l1 = 0.f, tau_tv = 0.f, lr_tv = 0.f;
  int real_mode = 0;  // packed real engine: Re / Im are two real planes, x = max(w - tau_l1, 0) per part
  int inner = 0, halo = 0, tile = 0, tiles_x = 0, tiles_per_plane = 0;
  int kind = 0;  // 0: generic tile kernel, 1: 64x64 register-strip kernel
  const float* fgp_beta = nullptr;  // [inner] FGP momentum schedule (device)
  float fgpb[16] = {};              // same schedule by value (strip kernel, inner <= 12)
  const uint8_t* force = nullptr;   // guard fix-up pass: per plane bit0 re / bit1 im -> identity
  double* part = nullptr;           // [nplanes][tiles_per_plane][kProxParts] doubles, or (part_warps > 0)
                                    // [nplanes][kProxParts][tiles_per_plane][part_warps] floats
  int part_warps = 0;
  int walk = 0;                      // strip kernel: column-strip walk (multi-pass FGP), see prox_strip.cu
  int ky = 1;                        // strip kernel: regions per column strip (tiles_per_plane = tiles_x * ky)
  float rcp_ky = 1.f;
  // multi-pass FGP (strip kernel, large T): this launch runs iterations [t0, t1);
  // the dual state crosses launches through HBM (interior pixels written,
  // region + halo read back by the next pass)
  int tile_h = 0;                   // strip kernel: tile height (tile = width)
  float rcp_tx = 0.f, rcp_tpp = 0.f;  // strip kernel: 1/tiles_x, 1/tiles_per_plane (fast division)
  int ipdx = 1;                      // 0: skip <g, dx> and |dx|^2 (no evaluated backtracking test)
  int t0 = 0, t1 = 0, pass_len = 0;  // pass_len 0: single pass
  float2* vbuf = nullptr;            // v = y - step grad (first pass writes)
  float4* sbuf = nullptr;            // (p, q) per pixel, two halves (pass parity)
  float4* rbuf = nullptr;            // extrapolated (rp, rq) per pixel, two halves
  long long sstride = 0;             // elements per half: pass i writes half i&1, reads (i-1)&1
  float* tvv = nullptr;              // per-tile TV(v) partials [tile][2], first pass -> last pass
  // strip kernel, single pass: tiles [ix0, ix1) x [iy0, iy1) are interior (their
  // regions touch no plane edge); ordered launches visit those first
  int ix0 = 0, ix1 = 0, iy0 = 0, iy1 = 0, icnt = 0;
  float rcp_icnt = 0.f, rcp_ecnt = 0.f, rcp_nix = 0.f, rcp_ew = 0.f;
  // strip kernel, single pass: top halo rows (halo_y) and the boundary-row
  // statistics.  tvfix: the top halo is T instead of T + 1, so a tile's first
  // row has no valid row above it in its own region; its TV(w) / TV(x_new)
  // terms are left out there and added by k_prox_tvfix from wside (every
  // tile's first and last rows of w) and x_new, into bpart [plane][3][tile]
  int halo_y = 0, tvfix = 0;
  float4* wside = nullptr;  // [nplanes][tiles_per_plane][2][32] float4 (64 complex per row)
  float* bpart = nullptr;   // [nplanes][3 (G_R, G_I, TVX)][tiles_per_plane]
};

// the launch's boundary-row statistics come from k_prox_tvfix
inline bool prox_tvfix_launch(const ProxArgs& a) {
  return a.tvfix && a.kind == 1 && !a.pass_len && a.tau_tv > 0.f && a.wside && a.bpart;
}

// Peer-memory spectrum reduction (peer.cu): every rank's symmetric buffers.
constexpr int kMaxPeers = 8;
struct PeerSet {
  float2* inbox[kMaxPeers] = {};               // [nranks][L]
  float2* result[kMaxPeers] = {};              // [nranks * L]
  unsigned long long* flags[kMaxPeers] = {};   // [2][kMaxPeers] epoch counters
  int nranks = 0, rank = 0;
  long long L = 0;                             // slice length, nranks * L >= P
};
long long peer_slice(long long P, int nranks);
cudaError_t peer_scatter(const float2* Spart, int groups, long long P, const PeerSet& ps, unsigned long long epoch,
                         unsigned* counter, cudaStream_t s);
cudaError_t peer_wait(const PeerSet& ps, int which, unsigned long long epoch, long long max_polls, int* err,
                      cudaStream_t s);
cudaError_t peer_gather(long long P, const PeerSet& ps, unsigned long long epoch, unsigned* counter, cudaStream_t s);

// 2D tiled TMA descriptor over float rows (kernels.cu); nonzero on failure
int encode_tiled_2d(CUtensorMap* m, const void* base, long long inner, long long rows, int box_inner, int box_rows);
bool plan_supported(int nx, int ny);
// gfft.cu: general plane sizes (mixed radix; a prime factor above 7 costs R^2
// table MACs per R outputs, so a prime side is a direct DFT of its lines)
constexpr int kMaxPrime = 4096;
bool pow2_side(int n);
bool generic_side(int n);
cudaError_t gplan_build(Plan& p, cudaStream_t s);
cudaError_t g_fft_rows(const Plan& p, const float2* in, float2* out, long long nrows, bool inverse, float scale,
                       cudaStream_t s, const uint8_t* live, int rows_per_plane);
cudaError_t g_fft_cols(const Plan& p, const float2* in, float2* out, int nplanes, bool inverse, float scale,
                       cudaStream_t s);
cudaError_t g_adj_cols(const Plan& p, const float2* R, float2* out, int nzl, int k0, cudaStream_t s, bool packed);
cudaError_t g_fwd_cols(const Plan& p, const float2* in, float2* Spart, int nzl, int k0, int groups, cudaStream_t s,
                       bool packed, const uint8_t* live);
void add_launches(long long n);
long long launch_count();  // kernels launched by this library since load
cudaError_t plan_build(Plan& p, int nx, int ny, int nz, double pitch, double dz, double z0, double lam,
                       cudaStream_t s);
void plan_free(Plan& p);

// checked build (HOLO_CHECKS): read-and-clear the violation bits of each
// translation unit (HoloCheckBit, common.cuh); 0 in the normal build
unsigned check_bits_kernels();
unsigned check_bits_prox();
unsigned check_bits_gfft();

// batched 1D transforms (unnormalised; `scale` multiplies the output)
// live (optional, forward rows): live[row / rows_per_plane] == 0 marks an
// all-zero plane whose rows are neither read, transformed nor written
cudaError_t fft_rows(const Plan& p, const float2* in, float2* out, long long nrows, bool inverse, float scale,
                     cudaStream_t s, const uint8_t* live = nullptr, int rows_per_plane = 0);
cudaError_t fft_cols(const Plan& p, const float2* in, float2* out, int nplanes, bool inverse, float scale,
                     cudaStream_t s);
// adjoint column pass: out[k] = colIFFT(H_{k0+k} * R), k < nzl (R already band-masked)
cudaError_t adj_cols(const Plan& p, const float2* R, float2* out, int nzl, int k0, cudaStream_t s,
                     bool packed = false);  // packed: the packed real engine's stack (engine.cu)
// forward column pass: Spart[g] = sum_{k in group g} colFFT(in[k]) * conj(H_{k0+k});
// planes with live[k] == 0 (optional) are all zero and skipped (solver.py:115-119)
cudaError_t fwd_cols(const Plan& p, const float2* in, float2* Spart, int nzl, int k0, int groups, cudaStream_t s,
                     bool packed = false, const uint8_t* live = nullptr);
int fwd_groups(const Plan& p, int nzl);
cudaError_t sum_groups(const Plan& p, const float2* Spart, int groups, float2* S, cudaStream_t s);

// residual spectrum R = m * (0.5 (S(f) + conj S(-f))) - B with S = ca Sa + cb Sb;
// writes m*R to Rout (if non-null) and per-block sum |R|^2 to part; returns #blocks.
int sensor_blocks(const Plan& p);
cudaError_t sensor(const Plan& p, const float2* Sa, const float2* Sb, float ca, float cb, const float2* B,
                   float2* Rout, double* part, cudaStream_t s);
// out[slot] = scale * sum(part[0..n))  (fixed order, one block)
cudaError_t final_sum(const double* part, int n, double scale, double* out, cudaStream_t s);

// prox: tile geometry chosen by prox_setup (fills halo/tile/tiles_*); returns smem bytes
size_t prox_setup(ProxArgs& a, int ny, int nx, int inner);
bool prox_supported(int ny, int nx, int inner);
// register-strip prox (prox_strip.cu): used when the halo T+2 <= prox_strip_max_halo()
int prox_strip_max_halo();
bool prox_strip_applicable(int ny, int nx, int inner);
int prox_strip_pass_len(int inner);  // 0: single pass; else FGP iterations per pass
void prox_strip_setup(ProxArgs& a, int ny, int nx, int inner);
cudaError_t prox_strip(const ProxArgs& a, cudaStream_t s);
cudaError_t prox(const ProxArgs& a, cudaStream_t s);
// per-plane reduction of the prox partials + guard check.  force_acc[plane]
// accumulates the guard bits; plane_out[plane*4 + {0..3}] = ip, dx2, l1, tv;
// new_fail[plane] = 1 when a guard bit was newly raised.  live (optional):
// live[plane] = 0 when skip_ok and the plane's sum |x_new| is exactly 0, i.e.
// every x_new of the plane is zero (the caller sets skip_ok only where a
// nonzero pixel cannot contribute an underflowed 0 to that sum).
cudaError_t prox_reduce(const ProxArgs& a, double tau_tv, int tv_on, uint8_t* force_acc, double* plane_out,
                        int* new_fail, cudaStream_t s, uint8_t* live = nullptr, int skip_ok = 0);
// scalars[0..3] += sums of plane_out over planes (fixed order); scalars[4] = #new guard failures;
// scalars[5] = #planes with live == 0 (0 without live)
cudaError_t plane_total(const double* plane_out, const int* new_fail, int nplanes, double* scalars,
                        cudaStream_t s, const uint8_t* live = nullptr);

// b (fp64, host layout) -> fp32 complex plane (imag 0), per-block sum b^2
cudaError_t load_hologram(const double* b, float2* bc, long long P, double* part, int* nblocks, cudaStream_t s);
// real part extraction with scale (for forward-operator output)
cudaError_t zero_imag(float2* x, long long n, cudaStream_t s);
cudaError_t unpack_real(const float2* x, float2* out, int nzl, long long P, cudaStream_t s);
cudaError_t real_part(const float2* in, float* out, long long n, float scale, cudaStream_t s);
cudaError_t real_to_complex(const float* in, float2* out, long long n, cudaStream_t s);
// mask a spectrum in place (m = 0 -> 0)
cudaError_t apply_mask(const Plan& p, float2* spec, int nplanes, cudaStream_t s);
// transfer stack H_k (k = k0..k1-1), optionally conjugated
cudaError_t transfer_stack(const Plan& p, int k0, int k1, bool conj, float2* out, cudaStream_t s);
// S_out = ca * Sa + cb * Sb (elementwise)
cudaError_t spec_combine(const Plan& p, const float2* Sa, const float2* Sb, float ca, float cb, float2* out,
                         cudaStream_t s);

// ||A_real||^2 = max_f sum_k cos^2(phase_k(f)) over the propagating band (real engine)
cudaError_t real_opnorm(const Plan& p, int nz, double* d_out, cudaStream_t s);
// sum |x|^2 over n complex elements -> per-block partials (returns #blocks)
int vol_norm2_blocks(long long n);
cudaError_t vol_norm2(const float2* x, long long n, double* part, cudaStream_t s);
// x = scale * (real ? (Re x, 0) : x), scale read from device (1/sqrt(*nrm2)) or 1 if null
cudaError_t vol_rescale(float2* x, long long n, const double* nrm2, int real, cudaStream_t s);

// COO export: count nonzeros per chunk, then compact in row-major order.
int coo_chunks(long long P, int nplanes);
cudaError_t coo_count(const float2* x, long long P, int nplanes, int* chunk_counts, cudaStream_t s);
cudaError_t coo_compact(const float2* x, long long P, int nx, int nplanes, const long long* chunk_offsets,
                        int* rows, int* cols, float2* vals, double2* vals64, cudaStream_t s);

}  // namespace holo
