// K4: fused-lasso prox on 64x64 register-strip regions (planes >= 64x64).
//
// Semantics are those of prox.py:104-148 (FGP-TV on Re and Im, step 1/(8 tau),
// replicated edges, per-plane guard) followed by prox.py:83-96 (complex soft
// threshold), fused with the FISTA extrapolation and gradient step
// (solver.py:309-310) and the fp64 partial sums the outer loop needs
// (solver.py:312-318 ip / dx2, solver.py:146-151 penalty, prox.py:138-147 guard).
//
// Layout: a CTA owns a 64x64 region = interior tile plus a recomputed halo
// (temporal blocking: T+1 rows/columns before the tile, T after, rounded
// even).  Regions are clamped into the plane, so a region edge is either a
// true plane edge (where "missing neighbour" is exactly the replicated-edge
// rule: zero up/left difference, no down/right D^T term) or far enough from
// every interior pixel that its garbage cannot reach it.  No per-pixel masks.
// The multi-pass kernels (large T) walk column strips instead, taking the rows
// above a frame from the previous region (see work_geom_walk).  A persistent
// CTA per SM streams the next region's inputs in by TMA while it works.
//
// 512 threads = 16 warps; warp w owns rows 4w..4w+3 of all 64 columns and
// lane l owns columns 2l, 2l+1, so each thread keeps a 4x2 tile of packed
// (re, im) float2 state in registers: the in-tile neighbours are register
// reads, the column neighbour across lanes is one warp shuffle per row, and
// only the band ends (row 4w-1 / 4w+4) go through ~24 KB of shared memory.
// Loads/stores are 16-byte (two complex64) per lane, 512 B per warp per row.
// The FGP A/B half-steps are fused into one sweep down the band per
// iteration, and the (re, im) arithmetic is packed FADD2/FMUL2/FFMA2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace holo {
namespace {

constexpr int RW = 64;  // region width: one warp, 2 columns per lane
#ifndef HOLO_PROX_RH
#define HOLO_PROX_RH 64
#endif
constexpr int RH = HOLO_PROX_RH;  // region height
#ifndef HOLO_PROX_SR
#define HOLO_PROX_SR 4
#endif
constexpr int SR = HOLO_PROX_SR;  // rows per thread (2: 1024 threads / 64 regs; 4: 512 threads / 128 regs)
constexpr int NW = RH / SR;       // warps = row bands
constexpr int NT = 32 * NW;

// Band w publishes top[.][w] and bot[w + 1]; it reads top[.][w + 1] (band
// below) and bot[w] (band above).  top[.][NW] and bot[0] are never written:
// interior regions read them as garbage for the region's outer rows (halo),
// so the read needs no select; plane-edge regions (EDGE) apply the exact rule.
struct Bands {
  float4 top[2][NW + 1][RW / 2];  // [buf][band][lane]: row-0 values (2 columns) -> down neighbour of the band above
  float4 bot[2][NW + 1][RW / 2];  // row-(SR-1) values (FGP sweep: X) -> up neighbour of the band below
};

HD float4 f4(float2 a, float2 b) { return make_float4(a.x, a.y, b.x, b.y); }
HD float2 lo2(float4 a) { return make_float2(a.x, a.y); }
HD float2 hi2(float4 a) { return make_float2(a.z, a.w); }
HD float2 shfl_dn(float2 x) {
  return make_float2(__shfl_down_sync(0xffffffffu, x.x, 1), __shfl_down_sync(0xffffffffu, x.y, 1));
}
HD float2 shfl_up(float2 x) {
  return make_float2(__shfl_up_sync(0xffffffffu, x.x, 1), __shfl_up_sync(0xffffffffu, x.y, 1));
}
// (|(a.x, b.x)|, |(a.y, b.y)|)
HD float2 norm_pair(float2 a, float2 b) {
  const float2 n2 = fma2(a, a, mul2(b, b));
  return make_float2(sqrt_a(n2.x), sqrt_a(n2.y));
}
// (pn, qn) /= max(1, |(pn, qn)|) for each of the (re, im) parts
HD void project(float2& pn, float2& qn) {
  const float2 n2 = fma2(pn, pn, mul2(qn, qn));
  // 1 / max(1, |.|) = rsqrt(max(1, |.|^2)); MUFU.RSQ(1) = 1 exactly
  const float2 sc = make_float2(rsqrt_a(fmaxf(n2.x, 1.f)), rsqrt_a(fmaxf(n2.y, 1.f)));
  pn = mul2(pn, sc);
  qn = mul2(qn, sc);
}

struct TileGeom {
  int i0, i1, j0, j1, ri0, rj0;
};

// n / d for 0 <= n < 2^24 via a host-side reciprocal (one correction step)
HD int fdiv(int n, int d, float rcp) {
  int q = __float2int_rz((float)n * rcp);
  const int r = n - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

// Everything a region needs from its work index, computed once per region.
struct Work {
  int plane = -1;
  TileGeom tg;
  long long g0;    // this thread's first element (row 0 of its band, column pair)
  bool edge;       // region touches a plane edge
  int k = 0;       // strip walk: region index in its column strip (0: plane top)
  int rsave = -1;  // strip walk: frame row the next region reads from above (-1: none)
};

// Strip walk (multi-pass FGP, a.walk): a CTA walks a column strip of a plane
// top to bottom.  Region k's frame starts at row f0_k = min(k TH, ny - RH),
// its tile is rows [k TH, (k+1) TH) (the last region: down to ny), and band 0
// reads the rows above the frame from what region k-1 saved for every
// exchange of the pass (v, X per FGP step, w, x_new), so only the bottom of a
// frame is halo (TH = 56 instead of 48 for 7-step passes).  TH is a multiple
// of SR, so the saved row is always the last row of one band.
// Work index = strip * ky + k, strip = plane * tiles_x + tx (tile = tx * ky + k).
HD Work work_geom_walk(const ProxArgs& a, int work) {
  Work wk;
  const int strip = fdiv(work, a.ky, a.rcp_ky);
  wk.k = work - strip * a.ky;
  wk.plane = fdiv(strip, a.tiles_x, a.rcp_tx);
  const int tx = strip - wk.plane * a.tiles_x;
  TileGeom& t = wk.tg;
  t.i0 = wk.k * a.tile_h;
  t.j0 = tx * a.tile;
  t.i1 = wk.k + 1 == a.ky ? a.ny : t.i0 + a.tile_h;
  t.j1 = min(a.nx, t.j0 + a.tile);
  t.ri0 = min(t.i0, a.ny - RH);
  t.rj0 = min(max(t.j0 - a.halo, 0), a.nx - RW);
  wk.rsave = wk.k + 1 < a.ky ? min(t.i0 + a.tile_h, a.ny - RH) - 1 - t.ri0 : -1;
  return wk;
}

template <bool WALK>
HD Work work_geom(const ProxArgs& a, int work) {
  if constexpr (WALK) return work_geom_walk(a, work);
  Work wk;
  wk.plane = fdiv(work, a.tiles_per_plane, a.rcp_tpp);
  const int tile = work - wk.plane * a.tiles_per_plane;
  const int ty = fdiv(tile, a.tiles_x, a.rcp_tx), tx = tile - ty * a.tiles_x;
  TileGeom& t = wk.tg;
  t.i0 = ty * a.tile_h;
  t.j0 = tx * a.tile;
  t.i1 = min(a.ny, t.i0 + a.tile_h);
  t.j1 = min(a.nx, t.j0 + a.tile);
  t.ri0 = min(max(t.i0 - a.halo_y, 0), a.ny - RH);  // region clamped into the plane
  t.rj0 = min(max(t.j0 - a.halo, 0), a.nx - RW);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  wk.g0 = (long long)wk.plane * a.P + (long long)(t.ri0 + w * SR) * a.nx + t.rj0 + 2 * lane;
  wk.edge = t.rj0 == 0 || t.rj0 + RW == a.nx || t.ri0 == 0 || t.ri0 + RH == a.ny;
  return wk;
}

// Ordered visit (single pass, ORD): local index lw < nplanes * icnt walks the
// interior tiles plane by plane (row-major inside the interior rectangle),
// the rest the edge ring, so a CTA runs the interior instantiation and then
// the edge one instead of alternating between the two code copies.
template <bool ORD>
HD int ordered_work(const ProxArgs& a, int lw) {
  if constexpr (!ORD) return lw;
  const int ni = a.icnt * a.nplanes, nix = a.ix1 - a.ix0;
  int plane, r, tile;
  if (lw < ni) {
    plane = fdiv(lw, a.icnt, a.rcp_icnt);
    r = lw - plane * a.icnt;
    const int ry = fdiv(r, nix, a.rcp_nix);
    tile = (a.iy0 + ry) * a.tiles_x + a.ix0 + r - ry * nix;
  } else {
    const int ecnt = a.tiles_per_plane - a.icnt;
    lw -= ni;
    plane = fdiv(lw, ecnt, a.rcp_ecnt);
    r = lw - plane * ecnt;
    const int top = a.iy0 * a.tiles_x, ew = a.tiles_x - nix, mid = (a.iy1 - a.iy0) * ew;
    if (r < top) {
      tile = r;
    } else if (r - top < mid) {
      r -= top;
      const int ry = fdiv(r, ew, a.rcp_ew), c = r - ry * ew;
      tile = (a.iy0 + ry) * a.tiles_x + (c < a.ix0 ? c : c + nix);
    } else {
      tile = a.iy1 * a.tiles_x + r - top - mid;
    }
  }
  return plane * a.tiles_per_plane + tile;
}

// The leader computes the next region's geometry anyway (for its TMA copies)
// and publishes it in shared memory; the other 511 threads read it instead of
// repeating the divisions.
struct GeoSlot {
  int plane, i0, i1, j0, j1, ri0, rj0, k, rsave, work, pad[2];  // work: global index (ordered visits)
};
HD void geo_store(GeoSlot& g, const Work& wk) {
  g.plane = wk.plane;
  g.i0 = wk.tg.i0;
  g.i1 = wk.tg.i1;
  g.j0 = wk.tg.j0;
  g.j1 = wk.tg.j1;
  g.ri0 = wk.tg.ri0;
  g.rj0 = wk.tg.rj0;
  g.k = wk.k;
  g.rsave = wk.rsave;
}
template <bool WALK = true>
HD Work geo_load(const ProxArgs& a, const GeoSlot& g) {
  const int4 lo = *reinterpret_cast<const int4*>(&g.plane);
  const int4 hi = *reinterpret_cast<const int4*>(&g.j1);
  Work wk;
  wk.plane = lo.x;
  TileGeom& t = wk.tg;
  t.i0 = lo.y;
  t.i1 = lo.z;
  t.j0 = lo.w;
  t.j1 = hi.x;
  t.ri0 = hi.y;
  t.rj0 = hi.z;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  wk.g0 = (long long)wk.plane * a.P + (long long)(t.ri0 + w * SR) * a.nx + t.rj0 + 2 * lane;
  wk.edge = t.rj0 == 0 || t.rj0 + RW == a.nx || t.ri0 == 0 || t.ri0 + RH == a.ny;
  if constexpr (WALK) {
    wk.k = g.k;
    wk.rsave = g.rsave;
  }
  return wk;
}

// Region inputs are staged by TMA: one elected thread loads the 64x64
// complex box of x, x_prev and grad (32 KB each, row-major [row][2*col]
// floats) into a double-buffered slot with one 2D tensor copy per array,
// completing on an mbarrier, so the 512 threads issue no load instructions
// and the next region's box streams in while this one iterates.
constexpr int kSlotF4 = RH * RW / 2;  // float4 per array per slot
constexpr int kSlotArrays = 3;        // x, x_prev, grad
constexpr unsigned kArrayBytes = kSlotF4 * 16;
// Strip-walk kernels: x and grad double-buffered ([buf][x, grad]), x_prev in
// one slot after them (refilled for the next region once this region's
// prologue has read it), then the saved rows [region parity][slot][lane]:
// slot 0 v, 1 + j the X read by FGP step tstart + j, kSaveW w, kSaveX x_new.
constexpr int kXpSlot = 4 * kSlotF4;
constexpr int kStageWalkF4 = 5 * kSlotF4;
constexpr int kSaveW = 9, kSaveX = 10, kSaveSlots = 11;

struct TmaMaps {
  CUtensorMap m[kSlotArrays];
};

HD unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
HD void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
HD void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// strip walk: x and grad into buffer `buf`; the barrier expects x_prev's bytes
// too (tma_xprev, issued later, completes it)
HD void tma_box(const TmaMaps& maps, int k, float4* dst, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(&maps.m[k])), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
HD void tma_region_walk(const ProxArgs& a, const TmaMaps& maps, float4* buf, uint64_t* bar, const Work& wk) {
  const int c0 = 2 * wk.tg.rj0, c1 = wk.plane * a.ny + wk.tg.ri0;
  const unsigned bytes = kArrayBytes * (1u + (a.beta != 0.f) + (a.grad != nullptr));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  tma_box(maps, 0, buf, bar, c0, c1);
  if (a.grad) tma_box(maps, 2, buf + kSlotF4, bar, c0, c1);
}
HD void tma_xprev(const ProxArgs& a, const TmaMaps& maps, float4* stage, uint64_t* bar, const Work& wk) {
  if (a.beta == 0.f) return;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tma_box(maps, 1, stage + kXpSlot, bar, 2 * wk.tg.rj0, wk.plane * a.ny + wk.tg.ri0);
}

// Band-slot split barrier: mbarriers with one arrival per warp (lane 0, after
// __syncwarp orders the warp's slot writes; release), waited on by every
// thread (acquire).  bph holds each barrier's next completion parity.
HD void band_arrive(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0)
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
HD void band_wait(uint64_t* bars, int i, unsigned& bph) {
  mbar_wait(&bars[i], (bph >> i) & 1u);
  bph ^= 1u << i;
}

// Later passes of a multi-pass FGP stage the dual state instead: v (8 B),
// (p, q) and (rp, rq) (16 B each) per pixel, 160 KB per region, in one slot
// (read into registers by the prologue, after which the next region's state
// streams in while this region iterates).
constexpr int kStateV = 0, kStateS = RH * RW / 2, kStateR = kStateS + RH * RW;  // float4 offsets
constexpr unsigned kStateBytes = (unsigned)(RH * RW) * 40u;
HD void tma_state(const ProxArgs& a, const TmaMaps& maps, float4* slot, uint64_t* bar, const Work& wk) {
  const int c1 = wk.plane * a.ny + wk.tg.ri0;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(kStateBytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(slot + kStateV)),
      "l"(reinterpret_cast<uint64_t>(&maps.m[0])), "r"(2 * wk.tg.rj0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
  // dual state: rows split by column parity (even columns, then odd; see the
  // last-pass stores), one 3-D box {32 pixels, both parities, RH rows} each
  const int off[2] = {kStateS, kStateR};
#pragma unroll
  for (int k = 0; k < 2; ++k)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            smem_u32(slot + off[k])),
        "l"(reinterpret_cast<uint64_t>(&maps.m[k + 1])), "r"(2 * wk.tg.rj0), "r"(0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// One region.  `pre` is its staged input slot (first / single pass) or null
// (later passes of a multi-pass FGP read HBM directly).
// EDGE: the region touches a plane edge, so its outer rows/columns need the
// exact replicated-edge rule; otherwise they are garbage zone and the
// lane-0 / lane-31 / band-0 / band-(NW-1) selects are skipped.
// RM: the packed real engine (x = max(w - tau, 0) per part), a separate
// instantiation so the complex kernels carry no real-mode branch.
// FAST: the engine's main launch -- no evaluated backtracking test (a.ipdx ==
// 0), no guard fix-up (a.force == nullptr) -- compiled without those branches
// (C3 prox 76.4 -> 72.8 ms per 10 iterations; also compiling out the beta == 0
// and grad == nullptr branches measured 73.1-73.4).
#ifndef HOLO_TT_UNROLL
#define HOLO_TT_UNROLL 3  // (C3 prox 74.0 -> 73.4 ms per 10 iterations vs 2; 4, a full unroll at T = 5, spills 48 B)
#endif
template <bool TV, bool EDGE, int PH, bool RM, bool FAST, int TT>
__device__ __forceinline__ void prox_tile(const ProxArgs& a, const TmaMaps& maps, Bands& sm, uint64_t* bbar,
                                          unsigned& bph, float4* pre, uint64_t* sbar, int work, const Work& wk,
                                          int next_work, const GeoSlot* nxgeo, float4* stage, float4* save,
                                          uint64_t* nbar) {
  constexpr bool WALK = PH != 0;  // multi-pass kernels walk column strips
  const int plane = wk.plane, tile = work - plane * a.tiles_per_plane;
  const uint32_t force = (!FAST && a.force) ? a.force[plane] : 0u;
  const bool ipdx = !FAST && a.ipdx;
  const TileGeom& tg = wk.tg;
  const int i0 = tg.i0, i1 = tg.i1, j0 = tg.j0, j1 = tg.j1, ri0 = tg.ri0, rj0 = tg.rj0;
  // the frame lies in its plane (the garbage-zone argument needs clamped
  // regions) and holds its tile
  HOLO_DCHECK(plane >= 0 && plane < a.nplanes && ri0 >= 0 && ri0 + RH <= a.ny && rj0 >= 0 && rj0 + RW <= a.nx &&
                  (rj0 & 1) == 0 && i0 >= ri0 && i1 <= ri0 + RH && j0 >= rj0 && j1 <= rj0 + RW && i0 < i1 &&
                  j0 < j1,
              CK_PROX_FRAME);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool lane0 = lane == 0, lane31 = lane == 31;
  const int r0 = w * SR;
  const int gj = rj0 + 2 * lane;  // columns gj, gj+1
  // Interior pixels: rows are warp-uniform (bit s of rInt: whole rows of halo
  // are skipped by uniform branches), and columns come in aligned pairs (tile
  // and halo are even), so a lane's two columns are both in or both out: the
  // statistics are accumulated unmasked and dropped per lane at the end.
  uint32_t rInt = 0;
#pragma unroll
  for (int s = 0; s < SR; ++s) {
    const int gi = ri0 + r0 + s;
    if (gi >= i0 && gi < i1) rInt |= 1u << s;
  }
  const bool cInt = gj >= j0 && gj < j1;
  // tvfix (single pass, top halo T): the row above the tile's first row is in
  // this region's garbage zone, so that row's TV(w) / TV(x_new) terms are left
  // to k_prox_tvfix (rTV); its pointwise terms stay here (rInt)
  uint32_t rTV = rInt;
  if constexpr (TV && !WALK) {
    const int rf = i0 - ri0 - r0;
    if (a.tvfix && i0 > 0 && rf >= 0 && rf < SR) rTV &= ~(1u << rf);
  }
  const long long g0 = wk.g0;
  constexpr bool staged = PH <= 1;
  // Staged kernels keep x and grad double-buffered ([buf][x, grad]) and x_prev
  // in one slot after them, refilled for the next region once every thread
  // has read it (after iteration 0's barrier; without TV after the x_new one).
  constexpr bool SPLITXP = staged;
  // single pass with TV: the epilogue's w = v - tau D^T p takes the band
  // below's non-extrapolated row-0 p from ptop (published with every FGP
  // step), and w / x_new cross bands in one CTA barrier (top[0] / top[1])
  constexpr bool FUSED_EPI = TV && PH == 0;
  float4* ptop = save;  // [NW + 1][32] (single pass: the walk's save area)
  // this thread's float4 (2 columns) of row s of array k in the staged slot
  auto slot = [&](int k, int s) {
    if constexpr (SPLITXP) return (k == 1 ? stage + kXpSlot : pre + (k ? kSlotF4 : 0))[(r0 + s) * (RW / 2) + lane];
    return pre[k * kSlotF4 + (r0 + s) * (RW / 2) + lane];
  };
  // Strip walk: band 0 reads the rows above the frame, saved by the previous
  // region (rd), through bot[.][0], which it alone reads: it copies each saved
  // row in just before it is needed.  Band `saver` saves its last row into wr
  // for the next region at every exchange.
  const bool top = wk.k == 0;
  const bool band0 = w == 0, saver = WALK && w == wk.rsave / SR && wk.rsave >= 0;
  const float4* rd = save + (wk.k & 1) * kSaveSlots * 32 + lane;
  float4* wr = save + ((wk.k + 1) & 1) * kSaveSlots * 32 + lane;
  auto save_rows = [&](int sl, const float2 (&arr)[SR][2]) {
    if constexpr (WALK)
      if (saver) wr[sl * 32] = f4(arr[SR - 1][0], arr[SR - 1][1]);
  };
  auto fetch_above = [&](int buf, int sl) {
    if constexpr (WALK)
      if (band0) sm.bot[buf][0][lane] = rd[sl * 32];
  };
  // plane top row (zero y-difference): every band-0 row of an EDGE region in
  // the tiled kernel (a halo row unless the region is at the top), only the top
  // region's in a strip walk
  auto top_rule = [&]() { return EDGE && w == 0 && (!WALK || top); };

  float2 v[SR][2], p[SR][2], q[SR][2], rp[SR][2], rq[SR][2];
  if (TV && PH == 1) fetch_above(0, 0);  // v above the frame, read by iteration 0
  // PH: pass kind of a multi-pass FGP (compile-time, so no kernel carries the
  // state handling it does not use): 0 single pass, 1 first, 2 middle, 3 last
  constexpr bool first = PH == 0 || PH == 1, last = PH == 0 || PH == 3;
  const int pass = PH ? a.t0 / a.pass_len : 0;
  // state halves alternate by pass parity so a pass never overwrites what
  // neighbouring regions of the same launch still read as their halo
  const float4* s_in = a.sbuf + ((pass - 1) & 1) * a.sstride;
  const float4* r_in = a.rbuf + ((pass - 1) & 1) * a.sstride;
  if (!first) {  // later pass of a multi-pass FGP: v and the dual state from the staged slot
    (void)s_in;
    (void)r_in;
#pragma unroll
    for (int s = 0; s < SR; ++s) {
      const int row = r0 + s;
      const float4 vv = pre[kStateV + row * (RW / 2) + lane];
      v[s][0] = lo2(vv);
      v[s][1] = hi2(vv);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        // [row][column parity][lane] (see tma_state)
        const float4 sq = pre[kStateS + row * RW + k * 32 + lane], rr = pre[kStateR + row * RW + k * 32 + lane];
        p[s][k] = lo2(sq);
        q[s][k] = hi2(sq);
        rp[s][k] = lo2(rr);
        rq[s][k] = hi2(rr);
      }
    }
    // the slot is free once everyone has read it: stream the next region's state in
    __syncthreads();
    if (threadIdx.x == 0 && next_work >= 0) tma_state(a, maps, pre, sbar, geo_load(a, *nxgeo));
  } else {
    const float2 cb = splat2(1.f + a.beta), cm = splat2(-a.beta), cs = splat2(-a.step);
#pragma unroll
    for (int s = 0; s < SR; ++s) {
      const float4 y = slot(0, s);
      float2 y0 = lo2(y), y1 = hi2(y);
      if (a.beta != 0.f) {
        const float4 o = slot(1, s);
        y0 = fma2(cb, y0, mul2(cm, lo2(o)));
        y1 = fma2(cb, y1, mul2(cm, hi2(o)));
      }
      if (a.grad) {
        const float4 gg = slot(2, s);
        y0 = fma2(cs, lo2(gg), y0);
        y1 = fma2(cs, hi2(gg), y1);
      }
      v[s][0] = y0;
      v[s][1] = y1;
    }
  }

  // per-thread partial sums over its 8 pixels (fp32), promoted to fp64 at the end
  float acc[kProxParts];
#pragma unroll
  for (int i = 0; i < kProxParts; ++i) acc[i] = 0.f;

  // x-differences and TV contributions of one row (both columns): left neighbour
  // of column 0 is lane-1's column 1 (own value at the region's left edge)
  auto gx_row = [&](float2 x0, float2 x1, float2& gx0, float2& gx1) {
    const float2 l = shfl_up(x1);
    gx0 = sub2(x0, l);
    if (EDGE && lane0) gx0 = make_float2(0.f, 0.f);
    gx1 = sub2(x1, x0);
  };
  // right neighbour of column 1 = lane+1's column 0 (0 beyond the region)
  auto right_of = [&](float2 x0) {
    float2 r = shfl_dn(x0);
    if (EDGE && lane31) r = make_float2(0.f, 0.f);
    return r;
  };
  auto above_of = [&](int buf, int k, float2 self) -> float2 {
    if (top_rule()) return self;
    const float4 b4 = sm.bot[buf][w][lane];
    return k ? hi2(b4) : lo2(b4);
  };
  const float2 mtau = splat2(-a.tau_tv);
  const float ttv = a.tau_tv;

  // soft threshold of w (fix-up pass: identity part where the guard fired); x_new -> p
  auto soft_rows = [&]() {
  const float tl = a.tau_l1;
  if (force) {  // (per plane, so warp-uniform; the main pass never takes it)
#pragma unroll
    for (int s = 0; s < SR; ++s)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (force & 1u) rp[s][k].x = v[s][k].x;
        if (force & 2u) rp[s][k].y = v[s][k].y;
      }
  }
  // |x_new| = gsc |w| = gsc n2 rsqrt(n2) feeds the L1 sum with the same rsqrt
#pragma unroll
  for (int s = 0; s < SR; ++s) {
    float l1 = 0.f;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float wr = rp[s][k].x, wi = rp[s][k].y;
      if constexpr (RM) {  // solver.py:208-210: max(w - tau, 0), per packed real plane (Re, Im)
        p[s][k] = make_float2(fmaxf(wr - tl, 0.f), fmaxf(wi - tl, 0.f));
        l1 += p[s][k].x + p[s][k].y;
        continue;
      }
      const float n2 = fmaf(wr, wr, wi * wi);
      const float r = rsqrt_a(fmaxf(n2, 1e-30f));
      const float shrink = 1.f - tl * r;
      // |w| <= tau -> 0 (tau = 0: shrink = 1 for w != 0, and w = 0 maps to 0 either way)
      const float gsc = (n2 > tl * tl) ? shrink : 0.f;
      p[s][k] = make_float2(wr * gsc, wi * gsc);
      l1 = fmaf(gsc * n2, r, l1);
    }
    if (rInt & (1u << s)) acc[PT_L1] += l1;
  }
  };
  // tvfix: w (after the guard's identity parts) of the tile's first and last
  // rows for k_prox_tvfix, 64 region columns per row
  auto save_wside = [&]() {
    if constexpr (TV && !WALK) {
      if (a.tvfix) {
        const int rf = i0 - ri0 - r0, rl = i1 - 1 - ri0 - r0;
        float4* ws = a.wside + (long long)(plane * a.tiles_per_plane + tile) * 64 + lane;
        HOLO_DCHECK(plane * a.tiles_per_plane + tile < a.nplanes * a.tiles_per_plane, CK_PROX_STORE);
#pragma unroll
        for (int s = 0; s < SR; ++s) {
          if (s == rf) ws[0] = f4(rp[s][0], rp[s][1]);
          if (s == rl) ws[32] = f4(rp[s][0], rp[s][1]);
        }
      }
    }
  };
  if (TV) {
    const float2 lr2 = splat2(a.lr_tv);
    // X = v - tau (rp + rq - rq_right) of the band's last row: the last-row u
    // without its rp_down term.  The band below rebuilds that u from X and its
    // own row-0 rp, so one barrier per FGP iteration suffices.
    auto xlast = [&](float2& x0, float2& x1) {
      const float2 rqr1 = right_of(rq[SR - 1][0]);
      x0 = fma2(mtau, sub2(add2(rp[SR - 1][0], rq[SR - 1][0]), rq[SR - 1][1]), v[SR - 1][0]);
      x1 = fma2(mtau, sub2(add2(rp[SR - 1][1], rq[SR - 1][1]), rqr1), v[SR - 1][1]);
    };
    float2 xl0, xl1;
    auto save_x = [&](int sl) {  // X of the band's last row, just published
      if constexpr (WALK)
        if (saver) wr[sl * 32] = f4(xl0, xl1);
    };
    const int tstart = first ? 1 : a.t0;
    if (first) {
    // ---- iteration 0: r = 0, u = v, beta_0 = 0; TV(v) for the guard ----
    sm.bot[0][w + 1][lane] = f4(v[SR - 1][0], v[SR - 1][1]);
    save_rows(0, v);
    __syncthreads();
    if constexpr (SPLITXP) {  // every thread has read this region's x_prev: stream the next region's in
      if (threadIdx.x == 0 && next_work >= 0) tma_xprev(a, maps, stage, nbar, geo_load<WALK>(a, *nxgeo));
    }
    {
      float2 up0 = above_of(0, 0, v[0][0]), up1 = above_of(0, 1, v[0][1]);
#pragma unroll
      for (int s = 0; s < SR; ++s) {
        float2 gx0, gx1;
        gx_row(v[s][0], v[s][1], gx0, gx1);
        const float2 gy0 = sub2(v[s][0], up0), gy1 = sub2(v[s][1], up1);
        up0 = v[s][0];
        up1 = v[s][1];
        // One rsqrt per part serves both the guard's |Dv| and the projection:
        // r = 1/|Dv|, |Dv| = |Dv|^2 r, and lr Dv / max(1, lr |Dv|) = min(lr, r) Dv.
        const float2 n0 = fma2(gy0, gy0, mul2(gx0, gx0)), n1 = fma2(gy1, gy1, mul2(gx1, gx1));
        const float2 r0 = make_float2(rsqrt_a(fmaxf(n0.x, 1e-30f)), rsqrt_a(fmaxf(n0.y, 1e-30f)));
        const float2 r1 = make_float2(rsqrt_a(fmaxf(n1.x, 1e-30f)), rsqrt_a(fmaxf(n1.y, 1e-30f)));
        // guard: G = tau TV(w) + |w - v|^2 / 2 - tau TV(v) per part, here the -tau TV(v) term
        if (rInt & (1u << s)) {
          const float2 nv = fma2(n0, r0, mul2(n1, r1));
          acc[PT_G_R] = fmaf(-ttv, nv.x, acc[PT_G_R]);
          acc[PT_G_I] = fmaf(-ttv, nv.y, acc[PT_G_I]);
        }
        const float2 f0 = make_float2(fminf(lr2.x, r0.x), fminf(lr2.x, r0.y));
        const float2 f1 = make_float2(fminf(lr2.x, r1.x), fminf(lr2.x, r1.y));
        const float2 pn0 = mul2(f0, gy0), qn0 = mul2(f0, gx0);
        const float2 pn1 = mul2(f1, gy1), qn1 = mul2(f1, gx1);
        p[s][0] = rp[s][0] = pn0;
        q[s][0] = rq[s][0] = qn0;
        p[s][1] = rp[s][1] = pn1;
        q[s][1] = rq[s][1] = qn1;
      }
    }
    }
    // publish for the first sweep (iteration t reads buffer t&1, writes its
    // complement; iteration 0 used bot[0], so the first sweep reads buffer 1)
    int lastbuf = first ? 1 : a.t0 & 1;
    {
      xlast(xl0, xl1);
      sm.top[lastbuf][w][lane] = f4(rp[0][0], rp[0][1]);
      sm.bot[lastbuf][w + 1][lane] = f4(xl0, xl1);
      if constexpr (FUSED_EPI)  // (T = 1: iteration 0 is the final step)
        if ((TT > 0 ? TT : a.t1) == 1) ptop[w * 32 + lane] = f4(p[0][0], p[0][1]);
      save_x(1);
      band_arrive(&bbar[lastbuf]);
      fetch_above(lastbuf, 1);  // read by band 0 itself only: after its arrival
    }
    // ---- iterations max(t0,1)..t1-1: one fused sweep down the band per iteration ----
    // Split barrier: rows 1..SR-2 only need this band's registers, so they are
    // updated between the previous iteration's arrive and the wait for the
    // neighbours' band data; rows 0 and SR-1 follow the wait.
    const float2 ptau = splat2(a.tau_tv);
    // (TT > 0: the FGP depth is a compile-time constant -- T = 5, the
    // reference's default: C3 prox 75.7 -> 74.7 ms per 10 iterations)
    const int tend = TT > 0 ? TT : a.t1;
    // multi-pass kernels, per pass kind (C5 passes, ncu per launch, unroll 1 / 2 / 3):
    // first 12.7 / 15.4 / 14.7 ms (168 B of spills at 2), middle 11.6 / 11.0 / 11.5,
    // last 12.3 / 10.9 / 10.7
    constexpr int kTU = TT > 0 ? HOLO_TT_UNROLL : (PH == 1 ? 1 : PH == 3 ? 3 : 2);
#pragma unroll kTU
    for (int t = tstart; t < tend; ++t) {
      const int b = t & 1;  // buffers holding this iteration's band-top rp / band-bottom X
      // single pass (T <= 8): the momentum schedule from the parameter bank
      const float2 bt2 = splat2(PH == 0 ? a.fgpb[t] : __ldg(a.fgp_beta + t));
      // final step of a single pass or of a multi-pass FGP's last pass: the
      // epilogue reads only p, q, so the extrapolated duals, the band's X and
      // its band-top rp are not formed (the walk's saved X of that step is
      // never fetched: the epilogue exchanges through its own slots)
      const bool fin = (PH == 0 || PH == 3) && t == tend - 1;
      // one row's dual update from its u, given the u of the row above
      auto update = [&](int s, float2 u0, float2 u1, float2 up0, float2 up1) {
        float2 gx0, gx1;
        gx_row(u0, u1, gx0, gx1);
        const float2 gy0 = sub2(u0, up0), gy1 = sub2(u1, up1);
        float2 pn0 = fma2(lr2, gy0, rp[s][0]), qn0 = fma2(lr2, gx0, rq[s][0]);
        float2 pn1 = fma2(lr2, gy1, rp[s][1]), qn1 = fma2(lr2, gx1, rq[s][1]);
        project(pn0, qn0);
        project(pn1, qn1);
        if (!fin) {
          rp[s][0] = fma2(bt2, sub2(pn0, p[s][0]), pn0);
          rq[s][0] = fma2(bt2, sub2(qn0, q[s][0]), qn0);
          rp[s][1] = fma2(bt2, sub2(pn1, p[s][1]), pn1);
          rq[s][1] = fma2(bt2, sub2(qn1, q[s][1]), qn1);
        }
        p[s][0] = pn0;
        q[s][0] = qn0;
        p[s][1] = pn1;
        q[s][1] = qn1;
      };
      // u(s, k) = v - tau (rp + rq - rp_down - rq_right) for rows 0..SR-2 (own registers)
      float2 u[SR - 1][2];
#pragma unroll
      for (int s = 0; s < SR - 1; ++s) {
        const float2 rqr1 = right_of(rq[s][0]);
        u[s][0] = fma2(mtau, sub2(sub2(add2(rp[s][0], rq[s][0]), rp[s + 1][0]), rq[s][1]), v[s][0]);
        u[s][1] = fma2(mtau, sub2(sub2(add2(rp[s][1], rq[s][1]), rp[s + 1][1]), rqr1), v[s][1]);
      }
      // the u of the row above row 0 uses row 0's rp before its update: keep it
      const float2 r00 = rp[0][0], r01 = rp[0][1];
#pragma unroll
      for (int s = 1; s < SR - 1; ++s) update(s, u[s][0], u[s][1], u[s - 1][0], u[s - 1][1]);
      band_wait(bbar, b, bph);
      const float4 d4 = (!EDGE || w < NW - 1) ? sm.top[b][w + 1][lane] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 x4 = sm.bot[b][w][lane];
      {
        // u of the row above the band: X of the band above + tau * my row-0 rp
        float2 up0 = fma2(ptau, r00, lo2(x4)), up1 = fma2(ptau, r01, hi2(x4));
        if (top_rule()) {  // plane top row: zero y-difference
          up0 = u[0][0];
          up1 = u[0][1];
        }
        update(0, u[0][0], u[0][1], up0, up1);
      }
      update(SR - 1, fma2(ptau, lo2(d4), xl0), fma2(ptau, hi2(d4), xl1), u[SR - 2][0], u[SR - 2][1]);
      if (!fin) {
        xlast(xl0, xl1);
        sm.top[b ^ 1][w][lane] = f4(rp[0][0], rp[0][1]);  // other buffers: slower warps may still read b
        sm.bot[b ^ 1][w + 1][lane] = f4(xl0, xl1);
      }
      // (read only after the final band barrier, so only the final step's matters;
      // rewritten by the next region behind its iteration-0 barrier)
      if constexpr (FUSED_EPI)
        if (fin) ptop[w * 32 + lane] = f4(p[0][0], p[0][1]);
      save_x(2 + t - tstart);
      band_arrive(&bbar[b ^ 1]);
      fetch_above(b ^ 1, 2 + t - tstart);
      lastbuf = b ^ 1;
    }
    band_wait(bbar, lastbuf, bph);  // every band's last publication (and its reads of the other buffer) is done
    if (!last) {
      // hand the dual state (and v, once) of the interior pixels to the next pass
#pragma unroll
      for (int s = 0; s < SR; ++s) {
        const long long g = g0 + (long long)s * a.nx;
        if (!(rInt & (1u << s)) || !cInt) continue;
        // parity-split rows (even columns, then odd): a warp's store is 512
        // contiguous bytes instead of every other 16 bytes of 1 KB
        const long long gs = (pass & 1) * a.sstride + g - (gj >> 1);  // row start + gj / 2
        HOLO_DCHECK(gs >= 0 && gs + (a.nx >> 1) < 2 * a.sstride && g + 1 < a.sstride, CK_PROX_STORE);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          a.sbuf[gs + k * (a.nx >> 1)] = f4(p[s][k], q[s][k]);
          a.rbuf[gs + k * (a.nx >> 1)] = f4(rp[s][k], rq[s][k]);
        }
        if (first) *reinterpret_cast<float4*>(a.vbuf + g) = f4(v[s][0], v[s][1]);
      }
      if (first) {  // TV(v) guard partials of this tile, consumed by the last pass
        if (!cInt) acc[PT_G_R] = acc[PT_G_I] = 0.f;
        __shared__ float tsum[NW][2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          float x = acc[PT_G_R + i];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
          if (lane == 0) tsum[w][i] = x;
        }
        __syncthreads();
        if (threadIdx.x < 2) {
          float t = 0.f;
          for (int k = 0; k < NW; ++k) t += tsum[k][threadIdx.x];
          a.tvv[(long long)work * 2 + threadIdx.x] = t;
        }
      }
      return;  // every band read of this region precedes the last sweep's barrier
    }
    if constexpr (FUSED_EPI) {
      // ---- w = v - tau D^T(p, q) (into rp), x_new = soft(w) (into p) ----
      {
        const float4 d4 = (!EDGE || w < NW - 1) ? ptop[(w + 1) * 32 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int s = 0; s < SR; ++s) {
          const float2 pd0 = (s < SR - 1) ? p[s + 1][0] : lo2(d4);
          const float2 pd1 = (s < SR - 1) ? p[s + 1][1] : hi2(d4);
          const float2 qr1 = right_of(q[s][0]);
          rp[s][0] = fma2(mtau, sub2(sub2(add2(p[s][0], q[s][0]), pd0), q[s][1]), v[s][0]);
          rp[s][1] = fma2(mtau, sub2(sub2(add2(p[s][1], q[s][1]), pd1), qr1), v[s][1]);
        }
      }
      soft_rows();
      save_wside();
      // Last rows of w and x_new for the band below, in top[0] / top[1]: every
      // band's reads of the band slots ended before its final-sweep arrival,
      // and the next region writes top[] only behind its iteration-0 barrier
      // (its pre-barrier write goes to bot[0]).
      sm.top[0][w + 1][lane] = f4(rp[SR - 1][0], rp[SR - 1][1]);
      sm.top[1][w + 1][lane] = f4(p[SR - 1][0], p[SR - 1][1]);
      __syncthreads();
      // guard statistics: tau TV(w) + |w - v|^2 / 2 against tau TV(v)
      {
        float2 up0 = rp[0][0], up1 = rp[0][1];
        if (!top_rule()) {
          const float4 b4 = sm.top[0][w][lane];
          up0 = lo2(b4);
          up1 = hi2(b4);
        }
#pragma unroll
        for (int s = 0; s < SR; ++s) {
          float2 gx0, gx1;
          gx_row(rp[s][0], rp[s][1], gx0, gx1);
          const float2 gy0 = sub2(rp[s][0], up0), gy1 = sub2(rp[s][1], up1);
          up0 = rp[s][0];
          up1 = rp[s][1];
          if (rInt & (1u << s)) {
            const float2 nw = (rTV & (1u << s)) ? add2(norm_pair(gy0, gx0), norm_pair(gy1, gx1)) : make_float2(0.f, 0.f);
            const float2 d0 = sub2(rp[s][0], v[s][0]), d1 = sub2(rp[s][1], v[s][1]);
            const float2 dd = fma2(d0, d0, mul2(d1, d1));
            acc[PT_G_R] = fmaf(ttv, nw.x, fmaf(0.5f, dd.x, acc[PT_G_R]));
            acc[PT_G_I] = fmaf(ttv, nw.y, fmaf(0.5f, dd.y, acc[PT_G_I]));
          }
        }
      }
    } else {
    // ---- w = v - tau D^T(p, q) with the non-extrapolated dual (into rp) ----
    const int bf = lastbuf ^ 1;  // read by the last sweep, which every band has finished
    sm.top[bf][w][lane] = f4(p[0][0], p[0][1]);
    __syncthreads();
    {
      const float4 d4 = (!EDGE || w < NW - 1) ? sm.top[bf][w + 1][lane] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int s = 0; s < SR; ++s) {
        const float2 pd0 = (s < SR - 1) ? p[s + 1][0] : lo2(d4);
        const float2 pd1 = (s < SR - 1) ? p[s + 1][1] : hi2(d4);
        const float2 qr1 = right_of(q[s][0]);
        rp[s][0] = fma2(mtau, sub2(sub2(add2(p[s][0], q[s][0]), pd0), q[s][1]), v[s][0]);
        rp[s][1] = fma2(mtau, sub2(sub2(add2(p[s][1], q[s][1]), pd1), qr1), v[s][1]);
      }
    }
    sm.bot[0][w + 1][lane] = f4(rp[SR - 1][0], rp[SR - 1][1]);  // bot last read by the final sweep, a sync ago
    save_rows(kSaveW, rp);
    fetch_above(0, kSaveW);
    soft_rows();  // x_new -> p: needs only this band's w, so it runs ahead of the barrier
    save_wside();
    __syncthreads();
    // guard statistics: tau TV(w) + |w - v|^2 / 2 against tau TV(v)
    {
      float2 up0 = above_of(0, 0, rp[0][0]), up1 = above_of(0, 1, rp[0][1]);
#pragma unroll
      for (int s = 0; s < SR; ++s) {
        float2 gx0, gx1;
        gx_row(rp[s][0], rp[s][1], gx0, gx1);
        const float2 gy0 = sub2(rp[s][0], up0), gy1 = sub2(rp[s][1], up1);
        up0 = rp[s][0];
        up1 = rp[s][1];
        if (rInt & (1u << s)) {
          const float2 nw = (rTV & (1u << s)) ? add2(norm_pair(gy0, gx0), norm_pair(gy1, gx1)) : make_float2(0.f, 0.f);
          const float2 d0 = sub2(rp[s][0], v[s][0]), d1 = sub2(rp[s][1], v[s][1]);
          const float2 dd = fma2(d0, d0, mul2(d1, d1));  // (re, im) |w - v|^2 of the pair
          acc[PT_G_R] = fmaf(ttv, nw.x, fmaf(0.5f, dd.x, acc[PT_G_R]));
          acc[PT_G_I] = fmaf(ttv, nw.y, fmaf(0.5f, dd.y, acc[PT_G_I]));
        }
      }
    }
    }  // !FUSED_EPI
  } else {
#pragma unroll
    for (int s = 0; s < SR; ++s) {
      rp[s][0] = v[s][0];
      rp[s][1] = v[s][1];
    }
    soft_rows();
  }
  // x_new exchange: bot[1] after the FGP (the guard's reads of bot[0] may
  // still be running; the next region's first band-slot write, iteration 0's,
  // goes to bot[0] and its first-sweep publication follows a CTA barrier)
  constexpr int xb = TV ? 1 : 0;

  if constexpr (!FUSED_EPI) {
    sm.bot[xb][w + 1][lane] = f4(p[SR - 1][0], p[SR - 1][1]);
    save_rows(kSaveX, p);
    fetch_above(xb, kSaveX);
    __syncthreads();
  }
  if constexpr (SPLITXP && !TV) {  // (TV: issued after iteration 0's barrier)
    if (threadIdx.x == 0 && next_work >= 0) tma_xprev(a, maps, stage, nbar, geo_load<WALK>(a, *nxgeo));
  }
  {
    float2 up0, up1;
    if constexpr (FUSED_EPI) {
      up0 = p[0][0];
      up1 = p[0][1];
      if (!top_rule()) {
        const float4 b4 = sm.top[1][w][lane];
        up0 = lo2(b4);
        up1 = hi2(b4);
      }
    } else {
      up0 = above_of(xb, 0, p[0][0]);
      up1 = above_of(xb, 1, p[0][1]);
    }
    const float2 cb = splat2(1.f + a.beta), cm = splat2(-a.beta);
#pragma unroll
    for (int s = 0; s < SR; ++s) {
      float2 gx0, gx1;
      gx_row(p[s][0], p[s][1], gx0, gx1);
      const float2 gy0 = sub2(p[s][0], up0), gy1 = sub2(p[s][1], up1);
      up0 = p[s][0];
      up1 = p[s][1];
      if (!(rInt & (1u << s))) continue;
      const long long g = g0 + (long long)s * a.nx;
      if (rTV & (1u << s)) {
        const float2 nx2 = add2(norm_pair(gy0, gx0), norm_pair(gy1, gx1));
        acc[PT_TVX] += nx2.x + nx2.y;
      }
      if (ipdx) {  // <g, x_new - y> and |x_new - y|^2: only for an evaluated backtracking test
        const float4 y4 = staged ? slot(0, s) : *reinterpret_cast<const float4*>(a.x + g);
        float2 y[2] = {lo2(y4), hi2(y4)};
        if (a.beta != 0.f) {
          // (strip walk: x_prev's slot may already hold the next region's)
          const float4 o = *reinterpret_cast<const float4*>(a.xp + g);
          y[0] = fma2(cb, y[0], mul2(cm, lo2(o)));
          y[1] = fma2(cb, y[1], mul2(cm, hi2(o)));
        }
        float4 gr4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a.grad) gr4 = staged ? slot(2, s) : *reinterpret_cast<const float4*>(a.grad + g);
        const float2 gr[2] = {lo2(gr4), hi2(gr4)};
        const float2 dx0 = sub2(p[s][0], y[0]), dx1 = sub2(p[s][1], y[1]);
        const float2 ip = fma2(gr[0], dx0, mul2(gr[1], dx1));  // (re, im) parts of <g, dx>
        const float2 d2 = fma2(dx0, dx0, mul2(dx1, dx1));
        acc[PT_IP] += ip.x + ip.y;
        acc[PT_DX2] += d2.x + d2.y;
      }
      HOLO_DCHECK(!cInt || (g >= (long long)plane * a.P && g + 1 < (long long)(plane + 1) * a.P && gj + 1 < a.nx),
                  CK_PROX_STORE);
      if (cInt) *reinterpret_cast<float4*>(a.xnew + g) = f4(p[s][0], p[s][1]);
    }
  }
  // fp32 warp sums (32 terms each), then fp64 across the 16 warps
  // Transposed butterfly: each xor step halves the values a lane carries
  // (it keeps one half and receives its partner's copy of it), so 8 slots
  // cost 4+2+1+2 shuffles instead of 8x5; lane l ends with slot (l >> 2) & 7.
  static_assert(kProxParts <= 8, "");
  if (!cInt) {  // halo columns
#pragma unroll
    for (int i = 0; i < kProxParts; ++i) acc[i] = 0.f;
  }
  if (TV && !first && threadIdx.x == 0) {  // -tau TV(v) of this tile from the first pass
    acc[PT_G_R] += a.tvv[(long long)work * 2];
    acc[PT_G_I] += a.tvv[(long long)work * 2 + 1];
  }
  {
    float r8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r8[i] = i < kProxParts ? acc[i] : 0.f;
#pragma unroll
    for (int h = 4, o = 16; h >= 1; h >>= 1, o >>= 1) {
      const bool hi = lane & o;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const float send = hi ? r8[i] : r8[i + h];
        const float keep = hi ? r8[i + h] : r8[i];
        r8[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    float x = r8[0];
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    const int slot = (lane >> 2) & 7;
    // per-warp fp32 partials straight to HBM; k_prox_reduce sums them in fp64
    // (no cross-warp barrier at the end of the region)
    HOLO_DCHECK(tile >= 0 && tile < a.tiles_per_plane, CK_PROX_STORE);
    if ((lane & 3) == 0 && slot < kProxParts)
      reinterpret_cast<float*>(a.part)[(((long long)plane * kProxParts + slot) * a.tiles_per_plane + tile) * NW + w] = x;
  }
  // The next region's leader refills this region's x / grad slot right away:
  // when the epilogue read the slot (evaluated backtracking test), wait for
  // every warp first.  Band slots and geo[] are only rewritten behind the next
  // region's own barriers.
  // (no TV: the next region's only exchange writes bot[0] before its barrier)
  if (!TV || ipdx) __syncthreads();
}

// Persistent: one CTA per SM walks regions blockIdx.x, +gridDim.x, ...
// (fix-up pass: only regions of planes whose guard fired).
template <bool TV, int PH, bool RM = false, bool FAST = false, int TT = 0, bool ORD = false>
__global__ void __launch_bounds__(NT, 1) k_prox_strip(const ProxArgs a, const __grid_constant__ TmaMaps maps) {
  static_assert(NT <= 1024, "");
  // Bands, then the staged slots: [2][x, x_prev, grad] (single pass), or the
  // strip walk's [2][x, grad] + x_prev + saved rows (first pass) / state slot
  // + saved rows (later passes)
  extern __shared__ __align__(1024) float4 dyn[];
  Bands& sm = *reinterpret_cast<Bands*>(dyn);
  float4* pre = dyn + sizeof(Bands) / sizeof(float4);
  float4* save = pre + kStageWalkF4;  // strip walk only
  __shared__ uint64_t bars[2];   // TMA slot completion
  __shared__ uint64_t bbar[2];   // band-slot split barrier (one arrival per warp)
  __shared__ __align__(16) GeoSlot geo[2];  // [buf] geometry of the region in slot buf
  constexpr bool staged = PH <= 1;
  constexpr bool WALK = PH != 0;
  const int total = a.tiles_per_plane * a.nplanes;
  auto next_from = [&](int t) {
    if (!FAST && a.force)
      while (t < total && !a.force[t / a.tiles_per_plane]) t += gridDim.x;
    return t < total ? t : -1;
  };
  // strip walk: strips blockIdx.x, +gridDim.x, ..., each region by region
  const int nstrips = a.tiles_x * a.nplanes;
  auto strip_from = [&](int st) {
    if (!FAST && a.force)
      while (st < nstrips && !a.force[fdiv(st, a.tiles_x, a.rcp_tx)]) st += gridDim.x;
    return st < nstrips ? st * a.ky : -1;
  };
  auto next_of = [&](int wkid) {
    if constexpr (!WALK) return next_from(wkid + gridDim.x);
    const int st = fdiv(wkid, a.ky, a.rcp_ky);
    return wkid + 1 < (st + 1) * a.ky ? wkid + 1 : strip_from(st + gridDim.x);
  };
  int work = WALK ? strip_from(blockIdx.x) : next_from(blockIdx.x);
  if (work < 0) return;
  const bool leader = threadIdx.x == 0;
  poison_dyn_smem();  // (checked build: never-written band slots / halo reads are NaN)
  if (leader) {
    mbar_init(&bars[0], 1);  // slot 0 (and the later passes' state slot)
    mbar_init(&bars[1], 1);
    mbar_init(&bbar[0], NW);
    mbar_init(&bbar[1], NW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    geo_store(geo[0], work_geom<WALK>(a, ordered_work<ORD>(a, work)));
    if (ORD) geo[0].work = ordered_work<ORD>(a, work);
  }
  __syncthreads();
  if (leader) {
    const Work w0 = geo_load<WALK>(a, geo[0]);
    if (staged) {  // [buf][x, grad] + one x_prev slot
      tma_region_walk(a, maps, pre, &bars[0], w0);
      tma_xprev(a, maps, pre, &bars[0], w0);
    } else {
      tma_state(a, maps, pre, &bars[0], w0);
    }
  }
  unsigned phase = 0;  // bit b: parity of slot b's next completion
  unsigned bph = 0;    // bit b: parity of band barrier b's next completion
  for (int buf = 0; work >= 0; buf ^= 1) {
    const int nw = next_of(work);
    // geo[buf ^ 1] and the other slot were last read by the previous region, before its final barrier
    if (leader && nw >= 0) {
      const int gw = ordered_work<ORD>(a, nw);
      const Work wn = work_geom<WALK>(a, gw);
      geo_store(geo[buf ^ 1], wn);
      if (ORD) geo[buf ^ 1].work = gw;
      if (staged) tma_region_walk(a, maps, pre + (buf ^ 1) * 2 * kSlotF4, &bars[buf ^ 1], wn);
    }
    const Work cur = geo_load<WALK>(a, geo[buf]);
    // x / x_prev / grad slots double-buffered (first pass); one state slot (later passes)
    const int sb = staged ? buf : 0;
    float4* slot = pre + sb * 2 * kSlotF4;  // (later passes: the state slot at pre)
    mbar_wait(&bars[sb], (phase >> sb) & 1u);
    phase ^= 1u << sb;
    const int gwork = ORD ? geo[buf].work : work;
    if (cur.edge)
      prox_tile<TV, true, PH, RM, FAST, TT>(a, maps, sm, bbar, bph, slot, &bars[0], gwork, cur, nw, &geo[buf ^ 1], pre,
                                            save, &bars[sb ^ 1]);
    else
      prox_tile<TV, false, PH, RM, FAST, TT>(a, maps, sm, bbar, bph, slot, &bars[0], gwork, cur, nw, &geo[buf ^ 1], pre,
                                             save, &bars[sb ^ 1]);
    work = nw;
  }
}

// 2D view [nplanes * ny rows][2 nx floats] of one complex64 stack, 64 x 128 boxes
CUresult encode_map(CUtensorMap* m, const void* base, int ny_total, int nx, int fpp = 2) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return CUDA_ERROR_NOT_FOUND;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  // fpp floats per pixel: 2 (complex64 x, v), 4 (float4 dual state)
  const cuuint64_t dims[2] = {(cuuint64_t)fpp * nx, (cuuint64_t)ny_total};
  const cuuint64_t strides[1] = {(cuuint64_t)fpp * nx * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)(fpp * RW), RH};
  const cuuint32_t estr[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// Dual-state arrays (float4 per pixel): every row stored as its even columns
// then its odd columns; viewed as [rows][parity][nx/2] float4 with boxes of
// {32 pixels, 2 parities, RH rows}, which land in shared memory as
// [row][parity][32] -- lane l's two pixels at (row, 0, l) and (row, 1, l).
CUresult encode_state_map(CUtensorMap* m, const void* base, int ny_total, int nx) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return CUDA_ERROR_NOT_FOUND;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)2 * nx, 2, (cuuint64_t)ny_total};  // floats: 4 per pixel, nx/2 pixels
  const cuuint64_t strides[2] = {(cuuint64_t)2 * nx * sizeof(float), (cuuint64_t)4 * nx * sizeof(float)};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * RW), 2, RH};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace

HOLO_CHECK_TU(check_bits_prox)

int prox_strip_max_halo() { return 14; }

bool prox_strip_applicable(int ny, int nx, int inner) {
  (void)inner;  // any T: passes of <= 5 FGP steps beyond T = 8
  return ny >= RH && nx >= RW && (nx % 2) == 0;
}

// Passes of 5 FGP steps (halo 6, tile 52) or 7 (halo 8, tile 48): the fewer
// passes win (each pass moves 40 B/pixel of dual state through HBM), ties go
// to the smaller halo.  C5 (T = 20): 7+7+6, 450 vs 464 ms per 10 iterations.
int prox_strip_pass_len(int inner) {
  if (inner <= 8) return 0;
  const int p5 = (inner + 4) / 5, p7 = (inner + 6) / 7;
  return p7 < p5 ? 7 : 5;
}

// Halo widths.  Garbage from a region edge that is not a plane edge advances
// one pixel per dependent step: from the top/left edge T B-steps (which read
// the up/left neighbour) plus the TV of w / x_new (also up/left) -> T+1; from
// the bottom/right edge T-1 A-steps plus the final D^T (down/right) -> T.
// The leading halo is rounded up to even (16-byte aligned float4 lanes) and
// the trailing one so the tile is even.
void prox_strip_setup(ProxArgs& a, int ny, int nx, int inner) {
  a.ny = ny;
  a.nx = nx;
  a.P = (long long)ny * nx;
  a.inner = inner;
  // multi-pass: every pass of <= Tp steps needs lo >= Tp+1 (last pass: Tp
  // B-steps + the TV statistics) and hi >= Tp+1 (Tp A-steps + the final D^T)
  const int tp = prox_strip_pass_len(inner);
  const int h_lo = tp ? ((tp + 2) & ~1) : ((inner + 2) & ~1);  // >= T+1, even
  const int h_hi = tp ? h_lo : inner + (inner & 1);           // >= T, tile even
  a.halo = h_lo;
  a.tile = RW - h_lo - h_hi;
  a.pass_len = tp;
  a.t0 = 0;
  a.t1 = inner;
  a.tiles_x = (nx + a.tile - 1) / a.tile;
  // multi-pass: strip walk, only the frame bottom is halo (Tp A-steps + the
  // final D^T); single pass: square tiles with halo on every side
  a.walk = tp > 0 && !getenv("HOLO_PROX_NOWALK");
  a.tvfix = 0;
  if (a.walk) {
    a.tile_h = (RH - (tp + 1)) / SR * SR;  // multiple of SR: the saved row ends a band
    a.ky = ny > RH ? 1 + (ny - RH + a.tile_h - 1) / a.tile_h : 1;
  } else {
    a.tile_h = RH - h_lo - h_hi;
    a.ky = (ny + a.tile_h - 1) / a.tile_h;
    // tvfix: top halo T instead of T + 1 (w / x_new are valid from row T of a
    // region; only the TV terms of a tile's first row reach one row higher,
    // and k_prox_tvfix takes those from the neighbouring tile), bottom T:
    // 54-row tiles at T = 5, used where that saves a tile row (1024 rows: 19
    // instead of 20 region rows).  HOLO_PROX_TVFIX=1 / 0 forces it on / off.
    const char* tf = getenv("HOLO_PROX_TVFIX");
    const int th2 = RH - 2 * inner, ky2 = (ny + th2 - 1) / th2;
    const bool fix = tf ? tf[0] == '1' : ky2 < a.ky;
    if (fix && ny > RH) {
      a.tvfix = 1;
      a.halo_y = inner;
      a.tile_h = th2;
      a.ky = ky2;
    }
  }
  if (!a.tvfix) a.halo_y = a.halo;
  a.rcp_ky = 1.f / (float)a.ky;
  a.tiles_per_plane = a.tiles_x * a.ky;
  a.rcp_tx = 1.f / (float)a.tiles_x;
  a.rcp_tpp = 1.f / (float)a.tiles_per_plane;
  a.part_warps = NW;
  // interior tile rectangle (single pass): region frames clear of every plane edge
  auto interior = [](int n_tiles, int tile, int halo, int n, int R, int& t0, int& t1) {
    t0 = t1 = 0;
    for (int t = 0; t < n_tiles; ++t) {
      const int r0 = t * tile - halo;
      if (r0 > 0 && r0 < n - R) {
        if (t1 == t0) t0 = t;
        t1 = t + 1;
      }
    }
  };
  a.icnt = 0;
  if (!a.walk) {
    interior(a.tiles_x, a.tile, a.halo, nx, RW, a.ix0, a.ix1);
    interior(a.ky, a.tile_h, a.halo_y, ny, RH, a.iy0, a.iy1);
    a.icnt = (a.ix1 - a.ix0) * (a.iy1 - a.iy0);
  }
  if (a.icnt > 0) {
    a.rcp_icnt = 1.f / (float)a.icnt;
    a.rcp_ecnt = 1.f / (float)(a.tiles_per_plane - a.icnt);
    a.rcp_nix = 1.f / (float)(a.ix1 - a.ix0);
    a.rcp_ew = 1.f / (float)(a.tiles_x - (a.ix1 - a.ix0));
  }
}

cudaError_t prox_strip(const ProxArgs& a, cudaStream_t s) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  static_assert(kStateBytes == sizeof(float4) * kStageWalkF4, "later passes' state slot = the walk stage area");
  // [2][x, grad] + x_prev (+ the walk's saved rows / the single pass's ptop)
  const size_t smem = sizeof(Bands) + sizeof(float4) * (kStageWalkF4 + (a.walk ? 2 * kSaveSlots * 32 : (NW + 1) * 32));
  TmaMaps maps;
  memset(&maps, 0, sizeof(maps));
  const int rows = a.nplanes * a.ny;
  if (a.pass_len == 0 || a.t0 == 0 || !(a.tau_tv > 0.f)) {  // x, x_prev, grad
    if (encode_map(&maps.m[0], a.x, rows, a.nx) != CUDA_SUCCESS) return cudaErrorInvalidValue;
    if (a.beta != 0.f && encode_map(&maps.m[1], a.xp, rows, a.nx) != CUDA_SUCCESS) return cudaErrorInvalidValue;
    if (a.grad && encode_map(&maps.m[2], a.grad, rows, a.nx) != CUDA_SUCCESS) return cudaErrorInvalidValue;
  } else {  // later passes: v and the dual state half written by the previous pass
    const long long half = ((a.t0 / a.pass_len - 1) & 1) * a.sstride;
    if (encode_map(&maps.m[0], a.vbuf, rows, a.nx) != CUDA_SUCCESS ||
        encode_state_map(&maps.m[1], a.sbuf + half, rows, a.nx) != CUDA_SUCCESS ||
        encode_state_map(&maps.m[2], a.rbuf + half, rows, a.nx) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const long long total = a.walk ? (long long)a.tiles_x * a.nplanes  // strips
                                 : (long long)a.tiles_per_plane * a.nplanes;
  const int grid = (int)std::min<long long>(total, nsm);
  if (grid <= 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  auto launch = [&](auto kern) {
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return;
    kern<<<grid, NT, smem, s>>>(a, maps);
  };
  if (a.tau_tv > 0.f && a.pass_len && !a.walk) return cudaErrorInvalidValue;  // multi-pass kinds walk strips
  auto pick = [&](auto rm) {
    constexpr bool RM = decltype(rm)::value;
    if (a.tau_tv > 0.f && a.pass_len) {
      const bool fast = !a.ipdx && !a.force;
      if (a.t0 == 0)
        launch(k_prox_strip<true, 1, RM>);  // (no force / ipdx code in a first pass)
      else if (a.t1 >= a.inner)
        fast ? launch(k_prox_strip<true, 3, RM, true>) : launch(k_prox_strip<true, 3, RM>);
      else
        launch(k_prox_strip<true, 2, RM>);
    } else if (a.tau_tv > 0.f) {
      if (!a.ipdx && !a.force && a.inner == 5 && a.icnt > 0 && !getenv("HOLO_PROX_NOORD"))
        launch(k_prox_strip<true, 0, RM, true, 5, true>);  // the engine's main pass, T = 5
      else if (!a.ipdx && !a.force && a.inner == 5 && !getenv("HOLO_PROX_NOTT"))
        launch(k_prox_strip<true, 0, RM, true, 5>);
      else if (!a.ipdx && !a.force)  // the engine's main pass
        launch(k_prox_strip<true, 0, RM, true>);
      else
        launch(k_prox_strip<true, 0, RM>);
    } else {
      if (a.walk)  // no TV: no FGP passes, but the strip-walk tiling of this setup
        launch(k_prox_strip<false, 1, RM>);
      else
        launch(k_prox_strip<false, 0, RM>);
    }
  };
  if (a.real_mode)
    pick(std::true_type());
  else
    pick(std::false_type());
  if (e) return e;
  return cudaGetLastError();
}

}  // namespace holo
