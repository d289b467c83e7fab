// K4 (v3): fused-lasso prox on 64x64 register-strip regions (planes >= 64x64).
//
// Semantics are those of prox.py:104-148 (FGP-TV on Re and Im, step 1/(8 tau),
// replicated edges, per-plane guard) followed by prox.py:83-96 (complex soft
// threshold), fused with the FISTA extrapolation and gradient step
// (solver.py:309-310) and the fp64 partial sums the outer loop needs
// (solver.py:312-318 ip / dx2, solver.py:146-151 penalty, prox.py:138-147 guard).
//
// Layout: a CTA owns a 64x64 region = interior tile (64-2H)^2 plus a halo
// H = T+2 that is recomputed (temporal blocking).  Regions are clamped into
// the plane, so a region edge is either a true plane edge (where "missing
// neighbour" is exactly the replicated-edge rule: zero up/left difference,
// no down/right D^T term) or at least H pixels from every interior pixel
// (garbage that cannot reach the interior in T+2 steps).  No per-pixel masks.
//
// 512 threads = 16 warps: warp w covers columns 32*(w&1)..+32 (lane = column)
// and rows 8*(w>>1)..+8; each thread keeps its 8-pixel vertical strip in
// registers as packed (re, im) float2, so vertical neighbours are free,
// horizontal neighbours are warp shuffles, and only the warp seam (columns
// 31|32) and the strip ends go through ~10 KB of shared memory.  The (re, im)
// pairs run the same formula, so the arithmetic is FADD2/FMUL2/FFMA2.
#include "common.cuh"
#include "kernels.cuh"

namespace holo {
namespace {

constexpr int RW = 64;  // region width: 2 warps of 32 columns
constexpr int SR = 8;   // rows per thread strip
constexpr int NS = 8;   // strips (warp rows)
constexpr int RH = SR * NS;
constexpr int NT = 2 * 32 * NS;

struct Seams {
  float2 colR[2][2][RH];  // [buf][wx]: wx=0: column 32 values (right neighbour of column 31); wx=1: zeros
  float2 colL[RH];        // column 31 values -> left neighbour of column 32
  float2 top[2][NS][RW];  // [buf] strip top-row values -> down neighbour of the strip above
  float2 bot[NS][RW];     // strip bottom-row values -> up neighbour of the strip below
};

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
// projection of the dual pair onto the unit ball, per part: (pn, qn) /= max(1, |(pn, qn)|)
HD void project(float2& pn, float2& qn) {
  const float2 n2 = fma2(pn, pn, mul2(qn, qn));
  const float rx = rsqrt_a(n2.x), ry = rsqrt_a(n2.y);  // unconditional MUFU, then select
  const float2 sc = make_float2(n2.x > 1.f ? rx : 1.f, n2.y > 1.f ? ry : 1.f);
  pn = mul2(pn, sc);
  qn = mul2(qn, sc);
}

template <bool TV>
__global__ void __launch_bounds__(NT, 1) k_prox_strip(const ProxArgs a) {
  const int plane = blockIdx.y, tile = blockIdx.x;
  uint32_t force = 0;
  if (a.force) {
    force = a.force[plane];
    if (!force) return;  // fix-up pass: only planes whose guard fired
  }
  __shared__ Seams sm;
  const int TI = a.tile, H = a.halo;
  const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
  const int i0 = ty * TI, j0 = tx * TI;
  const int i1 = min(a.ny, i0 + TI), j1 = min(a.nx, j0 + TI);
  const int ri0 = min(max(i0 - H, 0), a.ny - RH);  // region clamped into the plane
  const int rj0 = min(max(j0 - H, 0), a.nx - RW);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wx = w & 1, wy = w >> 1;
  const int c = wx * 32 + lane, r0 = wy * SR;
  const bool lane0 = lane == 0, lane31 = lane == 31;
  const bool seam_w = (wx == 0) && lane31;  // writes column 31 (left-neighbour seam)
  const bool seam_e = (wx == 1) && lane0;   // writes column 32 (right-neighbour seam)
  const bool self_left = lane0 && wx == 0;  // region's left column: zero x-difference
  const int gj = rj0 + c;
  const bool colInt = gj >= j0 && gj < j1;
  uint32_t mInt = 0;
#pragma unroll
  for (int s = 0; s < SR; ++s) {
    const int gi = ri0 + r0 + s;
    if (colInt && gi >= i0 && gi < i1) mInt |= 1u << s;
  }
  if (threadIdx.x < RH) {
    sm.colR[0][1][threadIdx.x] = make_float2(0.f, 0.f);
    sm.colR[1][1][threadIdx.x] = make_float2(0.f, 0.f);
  }
  const long long g0 = (long long)plane * a.P + (long long)(ri0 + r0) * a.nx + gj;

  float2 v[SR], p[SR], q[SR], rp[SR], rq[SR];
  {
    const float2 cb = splat2(1.f + a.beta), cm = splat2(-a.beta), cs = splat2(-a.step);
#pragma unroll
    for (int s = 0; s < SR; ++s) {
      const long long g = g0 + (long long)s * a.nx;
      float2 y = a.x[g];
      if (a.beta != 0.f) y = fma2(cb, y, mul2(cm, a.xp[g]));
      if (a.grad) y = fma2(cs, a.grad[g], y);
      v[s] = y;
    }
  }

  // per-thread partial sums over its <= 8 pixels (fp32), promoted to fp64 at the end
  float acc[kProxParts];
#pragma unroll
  for (int i = 0; i < kProxParts; ++i) acc[i] = 0.f;

  // values other threads read as "up" (strip bottom row) and "left" (seam column 31)
  auto publish_ul = [&](const float2 (&x)[SR]) {
    sm.bot[wy][c] = x[SR - 1];
    if (seam_w) {
#pragma unroll
      for (int s = 0; s < SR; ++s) sm.colL[r0 + s] = x[s];
    }
  };
  // values other threads read as "down" (strip top row) and "right" (seam column 32)
  auto publish_dr = [&](int b, const float2 (&dn)[SR], const float2 (&rt)[SR]) {
    sm.top[b][wy][c] = dn[0];
    if (seam_e) {
#pragma unroll
      for (int s = 0; s < SR; ++s) sm.colR[b][0][r0 + s] = rt[s];
    }
  };
  // left neighbour of row s (own value at the region's left edge: zero difference)
  auto left_of = [&](float2 x, int s) {
    const float2 l = shfl_up(x);
    if (lane0) return self_left ? x : sm.colL[r0 + s];
    return l;
  };
  const float2 mtau = splat2(-a.tau_tv);

  if (TV) {
    const float2 lr2 = splat2(a.lr_tv);
    // ---- iteration 0: r = 0, u = v, beta_0 = 0; TV(v) for the guard ----
    publish_ul(v);
    __syncthreads();
    {
      float2 up = (wy > 0) ? sm.bot[wy - 1][c] : v[0];
#pragma unroll
      for (int s = 0; s < SR; ++s) {
        const float2 gy = sub2(v[s], up);
        const float2 gx = sub2(v[s], left_of(v[s], s));
        up = v[s];
        if (mInt & (1u << s)) {
          const float2 nv = norm_pair(gy, gx);
          acc[PT_TVV_R] += nv.x;
          acc[PT_TVV_I] += nv.y;
        }
        float2 pn = mul2(lr2, gy), qn = mul2(lr2, gx);
        project(pn, qn);
        p[s] = rp[s] = pn;
        q[s] = rq[s] = qn;
      }
    }
    publish_dr(0, rp, rq);
    __syncthreads();
    // ---- iterations 1..T-1: one fused sweep down the strip per iteration ----
    for (int t = 1; t < a.inner; ++t) {
      const int b = (t - 1) & 1;  // buffer holding this iteration's rp-top / rq-seam
      const float2 bt2 = splat2(__ldg(a.fgp_beta + t));
      // u of row s = v - tau (rp[s] + rq[s] - rp[s+1] - rq_right[s])
      auto urow = [&](int s, float2 rp_next, float2 rq_right) {
        return fma2(mtau, sub2(sub2(add2(rp[s], rq[s]), rp_next), rq_right), v[s]);
      };
      // pre-pass: the rows other threads need before the sweep (strip bottom, seam column)
      const float2 rp_below = (wy < NS - 1) ? sm.top[b][wy + 1][c] : make_float2(0.f, 0.f);
      float2 rq_r7 = shfl_dn(rq[SR - 1]);
      if (lane31) rq_r7 = sm.colR[b][wx][r0 + SR - 1];
      const float2 u7 = urow(SR - 1, rp_below, rq_r7);
      sm.bot[wy][c] = u7;
      if (seam_w) {
#pragma unroll
        for (int s = 0; s < SR - 1; ++s) sm.colL[r0 + s] = urow(s, rp[s + 1], sm.colR[b][0][r0 + s]);
        sm.colL[r0 + SR - 1] = u7;
      }
      __syncthreads();
      float2 up = (wy > 0) ? sm.bot[wy - 1][c] : make_float2(0.f, 0.f);
#pragma unroll
      for (int s = 0; s < SR; ++s) {
        float2 u;
        if (s == SR - 1) {
          u = u7;
        } else {
          float2 rq_r = shfl_dn(rq[s]);
          if (lane31) rq_r = sm.colR[b][wx][r0 + s];
          u = urow(s, rp[s + 1], rq_r);
        }
        if (s == 0 && wy == 0) up = u;  // region top row: zero y-difference
        const float2 gy = sub2(u, up);
        const float2 gx = sub2(u, left_of(u, s));
        up = u;
        float2 pn = fma2(lr2, gy, rp[s]);
        float2 qn = fma2(lr2, gx, rq[s]);
        project(pn, qn);
        rp[s] = fma2(bt2, sub2(pn, p[s]), pn);
        rq[s] = fma2(bt2, sub2(qn, q[s]), qn);
        p[s] = pn;
        q[s] = qn;
      }
      publish_dr(b ^ 1, rp, rq);  // other buffer: slower warps may still read buffer b
      __syncthreads();
    }
    // ---- w = v - tau D^T(p, q) with the non-extrapolated dual (into rp) ----
    const int bf = (a.inner - 1) & 1;  // the buffer not read by the last sweep
    publish_dr(bf ^ 1, p, q);
    __syncthreads();
    {
      const float2 p_below = (wy < NS - 1) ? sm.top[bf ^ 1][wy + 1][c] : make_float2(0.f, 0.f);
#pragma unroll
      for (int s = 0; s < SR; ++s) {
        float2 q_r = shfl_dn(q[s]);
        if (lane31) q_r = sm.colR[bf ^ 1][wx][r0 + s];
        const float2 pd = (s < SR - 1) ? p[s + 1] : p_below;
        rp[s] = fma2(mtau, sub2(sub2(add2(p[s], q[s]), pd), q_r), v[s]);
      }
    }
    publish_ul(rp);  // bot/colL last read by the final sweep, a sync ago
    __syncthreads();
    // guard statistics: tau TV(w) + |w - v|^2 / 2 against tau TV(v)
    {
      float2 up = (wy > 0) ? sm.bot[wy - 1][c] : rp[0];
#pragma unroll
      for (int s = 0; s < SR; ++s) {
        const float2 gy = sub2(rp[s], up);
        const float2 gx = sub2(rp[s], left_of(rp[s], s));
        up = rp[s];
        if (mInt & (1u << s)) {
          const float2 nw = norm_pair(gy, gx);
          const float2 dv = sub2(rp[s], v[s]);
          acc[PT_TVW_R] += nw.x;
          acc[PT_TVW_I] += nw.y;
          acc[PT_D2_R] += dv.x * dv.x;
          acc[PT_D2_I] += dv.y * dv.y;
        }
      }
    }
    __syncthreads();  // bot/colL reads done before x_new is published
  } else {
#pragma unroll
    for (int s = 0; s < SR; ++s) rp[s] = v[s];
  }

  // soft threshold of w (fix-up pass: identity part where the guard fired); x_new -> p
  const float tl = a.tau_l1;
#pragma unroll
  for (int s = 0; s < SR; ++s) {
    const float wr = (force & 1u) ? v[s].x : rp[s].x;
    const float wi = (force & 2u) ? v[s].y : rp[s].y;
    const float n2 = fmaf(wr, wr, wi * wi);
    const float shrink = 1.f - tl * rsqrt_a(n2);
    const float gsc = (tl > 0.f) ? ((n2 > tl * tl) ? shrink : 0.f) : 1.f;
    p[s] = make_float2(wr * gsc, wi * gsc);
  }
  publish_ul(p);
  __syncthreads();
  {
    float2 up = (wy > 0) ? sm.bot[wy - 1][c] : p[0];
    const float2 cb = splat2(1.f + a.beta), cm = splat2(-a.beta);
#pragma unroll
    for (int s = 0; s < SR; ++s) {
      const float2 gy = sub2(p[s], up);
      const float2 gx = sub2(p[s], left_of(p[s], s));
      up = p[s];
      if (!(mInt & (1u << s))) continue;
      const float2 nx2 = norm_pair(gy, gx);
      acc[PT_TVX_R] += nx2.x;
      acc[PT_TVX_I] += nx2.y;
      acc[PT_L1] += sqrt_a(fmaf(p[s].x, p[s].x, p[s].y * p[s].y));
      const long long g = g0 + (long long)s * a.nx;
      float2 y = a.x[g];
      if (a.beta != 0.f) y = fma2(cb, y, mul2(cm, a.xp[g]));
      const float2 dx = sub2(p[s], y);
      if (a.grad) {
        const float2 gg = a.grad[g];
        acc[PT_IP] += fmaf(gg.x, dx.x, gg.y * dx.y);
      }
      acc[PT_DX2] += fmaf(dx.x, dx.x, dx.y * dx.y);
      a.xnew[g] = p[s];
    }
  }
  double accd[kProxParts];
#pragma unroll
  for (int i = 0; i < kProxParts; ++i) accd[i] = (double)acc[i];
  block_sum<kProxParts, NT>(accd, a.part + ((long long)plane * a.tiles_per_plane + tile) * kProxParts);
}

}  // namespace

int prox_strip_max_halo() { return 14; }

bool prox_strip_applicable(int ny, int nx, int inner) {
  return ny >= RH && nx >= RW && inner + 2 <= prox_strip_max_halo() && inner <= 16;
}

void prox_strip_setup(ProxArgs& a, int ny, int nx, int inner) {
  a.ny = ny;
  a.nx = nx;
  a.P = (long long)ny * nx;
  a.inner = inner;
  a.halo = inner + 2;
  a.tile = RW - 2 * a.halo;
  a.tiles_x = (nx + a.tile - 1) / a.tile;
  a.tiles_per_plane = a.tiles_x * ((ny + a.tile - 1) / a.tile);
}

cudaError_t prox_strip(const ProxArgs& a, cudaStream_t s) {
  dim3 grid(a.tiles_per_plane, a.nplanes);
  if (a.tau_tv > 0.f)
    k_prox_strip<true><<<grid, NT, 0, s>>>(a);
  else
    k_prox_strip<false><<<grid, NT, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace holo
