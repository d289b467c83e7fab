// Shared-memory batched 1D FFTs (power-of-two N, 8..4096), register radix-16
// Stockham passes.  No host cuFFT anywhere on the hot path.
//
// Data distribution: the FFT of one line is computed by TPF = N/E threads
// ("j" = 0..TPF-1), each holding E = min(16, N) elements in registers.  On
// entry AND on exit thread j holds elements  j + m*TPF,  m = 0..E-1
// ("natural distribution"), so callers load/store global memory directly
// from registers with coalesced addresses and can fuse pre/post operations
// (transfer multiply, scaling, accumulation) element by element.
//
// Passes: radix 16 while N/NS is a multiple of 16, then one pass of the
// remaining radix (2, 4 or 8).  Between passes the line goes through shared
// memory; element i of a line lives at buf[pad(i) * S] (S = element stride,
// 1 for row-contiguous lines, C for C interleaved column lines).  pad(i) =
// i + i/16 keeps the radix-16 scatter conflict-free.
//
// Sign convention (numpy): forward X[k] = sum x[n] exp(-2 pi i nk/N); the
// inverse uses +i and is NOT scaled here (callers fold 1/N into their
// epilogue).  Twiddles come from a table tw[m] = (w, conj w), w = exp(-2 pi i
// m/N) (fp64-exact entries rounded to fp32) held in shared memory, so a table
// twiddle multiply is one FMUL2 + one FFMA2.
#pragma once
#include "common.cuh"

namespace holo {

template <int N>
struct FftShape {
  static_assert(N >= 8 && N <= 4096 && (N & (N - 1)) == 0, "N must be a power of two in [8, 4096]");
  static constexpr int E = N >= 16 ? 16 : N;
  static constexpr int TPF = N / E;
  // padded line length in elements; the +2/+TPF term staggers consecutive
  // lines across banks (see kernels: lines of one warp start on distinct banks)
  static constexpr int PADN = N + N / 16 + (TPF >= 16 ? 2 : TPF);
};

// Twiddle tables are stored per pass as [r-1][kk] (kk = butterfly index mod
// NS), so the lanes of a warp (consecutive kk) read consecutive entries:
// conflict-free, or broadcast.  Entry = (w, conj w), w = exp(-2 pi i kk r/(NS R)).
template <int N>
struct TwLayout {
  static constexpr int radix(int ns) { return ((N / ns) % 16 == 0) ? 16 : N / ns; }
  // offset of the table of the pass whose product of earlier radices is ns
  static constexpr int offset(int ns) {
    int off = 0;
    for (int s = 16; s < ns; s *= radix(s)) off += (radix(s) - 1) * s;
    return off;
  }
  static constexpr int size() {
    if (N <= 16) return 1;
    int off = 0;
    for (int s = 16; s < N; s *= radix(s)) off += (radix(s) - 1) * s;
    return off;
  }
};

HD int fft_pad(int i) { return i + (i >> 4); }
// pad(i + d) - pad(i) for a compile-time d that is a multiple of 16 (any i >= 0)
template <int D>
struct PadStep {
  static_assert(D % 16 == 0, "");
  static constexpr int value = D + D / 16;
};

// Complex arithmetic on packed f32x2 pairs (FADD2/FMUL2/FFMA2); the (re, im)
// swap below compiles to the .LO_HI operand selector, not a move.
HD float2 swp(float2 a) { return make_float2(a.y, a.x); }

// c + (-i) d  (forward)  or  c + (+i) d  (inverse):  one FFMA2
template <bool INV>
HD float2 add_ni(float2 c, float2 d) {
  return fma2(swp(d), INV ? make_float2(-1.f, 1.f) : make_float2(1.f, -1.f), c);
}
// multiply by -i (forward) or +i (inverse)
template <bool INV>
HD float2 mul_ni(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

template <bool INV>
HD void dft2(float2& a, float2& b) {
  const float2 t = a;
  a = add2(t, b);
  b = sub2(t, b);
}

template <bool INV>
HD void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
  const float2 t0 = add2(a0, a2), t1 = sub2(a0, a2);
  const float2 t2 = add2(a1, a3), t3 = sub2(a1, a3);
  a0 = add2(t0, t2);
  a2 = sub2(t0, t2);
  a1 = add_ni<INV>(t1, t3);
  a3 = add_ni<!INV>(t1, t3);
}

// x * exp(-/+ 2 pi i e / 16), e in [0, 16) compile-time
template <bool INV, int e>
HD float2 rot16(float2 x) {
  constexpr float C1 = 0.92387953251128674f, S1 = 0.38268343236508978f, R2 = 0.70710678118654752f;
  constexpr int ee = e & 15;
  if constexpr (ee == 0) {
    return x;
  } else if constexpr (ee == 4) {
    return mul_ni<INV>(x);
  } else if constexpr (ee == 8) {
    return make_float2(-x.x, -x.y);
  } else if constexpr (ee == 12) {
    return mul_ni<!INV>(x);
  } else {
    // cos/sin of pi*ee/8
    constexpr float cs = (ee == 1 || ee == 15) ? C1 : (ee == 2 || ee == 14) ? R2 : (ee == 3 || ee == 13) ? S1
                       : (ee == 5 || ee == 11) ? -S1 : (ee == 6 || ee == 10) ? -R2 : -C1;
    constexpr float sn = (ee == 1 || ee == 7) ? S1 : (ee == 2 || ee == 6) ? R2 : (ee == 3 || ee == 5) ? C1
                       : (ee == 9 || ee == 15) ? -S1 : (ee == 10 || ee == 14) ? -R2 : -C1;
    // forward: multiply by (cs, -sn); inverse: (cs, +sn)
    //   x (cs + i s) = x * cs + swap(x) * (-s, s)
    constexpr float s = INV ? sn : -sn;
    return fma2(swp(x), make_float2(-s, s), mul2(x, make_float2(cs, cs)));
  }
}

// a * w (forward) or a * conj(w) (inverse) with the table entry t = (w, conj w):
//   a w      = a.x (w)      + a.y swap(conj w)
//   a conj w = a.x (conj w) + a.y swap(w)
template <bool INV>
HD float2 twiddle(float2 a, float4 t) {
  const float2 w = make_float2(t.x, t.y), cw = make_float2(t.z, t.w);
  return INV ? fma2(make_float2(a.y, a.y), swp(w), mul2(make_float2(a.x, a.x), cw))
             : fma2(make_float2(a.y, a.y), swp(cw), mul2(make_float2(a.x, a.x), w));
}

template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<2, INV> {
  static HD void run(float2 (&a)[2]) { dft2<INV>(a[0], a[1]); }
};
template <bool INV>
struct Dft<4, INV> {
  static HD void run(float2 (&a)[4]) { dft4<INV>(a[0], a[1], a[2], a[3]); }
};
template <bool INV>
struct Dft<8, INV> {
  static HD void run(float2 (&a)[8]) {
    dft4<INV>(a[0], a[2], a[4], a[6]);
    dft4<INV>(a[1], a[3], a[5], a[7]);
    float2 o1 = rot16<INV, 2>(a[3]), o2 = rot16<INV, 4>(a[5]), o3 = rot16<INV, 6>(a[7]);
    float2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6], o0 = a[1];
    a[0] = add2(e0, o0); a[4] = sub2(e0, o0);
    a[1] = add2(e1, o1); a[5] = sub2(e1, o1);
    a[2] = add2(e2, o2); a[6] = sub2(e2, o2);
    a[3] = add2(e3, o3); a[7] = sub2(e3, o3);
  }
};
// 16 = 4 x 4: DFT4 over a (stride 4), twiddle w16^(b*k1), DFT4 over b, transpose.
template <bool INV>
struct Dft<16, INV> {
  static HD void run(float2 (&a)[16]) {
#pragma unroll
    for (int b = 0; b < 4; ++b) dft4<INV>(a[b], a[b + 4], a[b + 8], a[b + 12]);
    // a[b + 4*k1] now holds Y_b[k1]
    a[5] = rot16<INV, 1>(a[5]);
    a[9] = rot16<INV, 2>(a[9]);
    a[13] = rot16<INV, 3>(a[13]);
    a[6] = rot16<INV, 2>(a[6]);
    a[10] = rot16<INV, 4>(a[10]);
    a[14] = rot16<INV, 6>(a[14]);
    a[7] = rot16<INV, 3>(a[7]);
    a[11] = rot16<INV, 6>(a[11]);
    a[15] = rot16<INV, 9>(a[15]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(a[4 * k1], a[4 * k1 + 1], a[4 * k1 + 2], a[4 * k1 + 3]);
    // X[k1 + 4*k2] sits at a[4*k1 + k2]: transpose to natural order
    float2 t[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) t[k1 + 4 * k2] = a[4 * k1 + k2];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = t[i];
  }
};

// One Stockham pass of radix R with NS = product of earlier radices.
template <int N, int R, int NS, bool INV, bool FIRST, bool LAST>
HD void fft_pass(float2 (&v)[FftShape<N>::E], int j, float2* buf, int S, const float4* __restrict__ tw) {
  constexpr int E = FftShape<N>::E, TPF = FftShape<N>::TPF, BPT = E / R;
  static_assert(E % R == 0, "radix must divide E");
  if constexpr (!FIRST) {
    if constexpr (TPF % 16 == 0) {
      const float2* rp = buf + fft_pad(j) * S;  // one address, immediate offsets
#pragma unroll
      for (int m = 0; m < E; ++m) v[m] = rp[m * PadStep<TPF>::value * S];
    } else {
#pragma unroll
      for (int m = 0; m < E; ++m) v[m] = buf[fft_pad(j + m * TPF) * S];
    }
    if constexpr (!LAST) __syncthreads();  // everyone has read before anyone writes
  } else if constexpr (!LAST) {
    __syncthreads();  // buffer may still be read by a previous transform's last pass
  }
#pragma unroll
  for (int s = 0; s < BPT; ++s) {
    const int b = j + s * TPF;
    float2 a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = v[s + r * BPT];
    if constexpr (NS > 1) {
      const int kk = b % NS;
      const float4* tp = tw + TwLayout<N>::offset(NS) + kk;
      // groups of 4 twiddles: bounds the 4-register table entries in flight
#pragma unroll
      for (int r0 = 1; r0 < R; r0 += 4) {
#pragma unroll
        for (int r = r0; r < r0 + 4 && r < R; ++r) a[r] = twiddle<INV>(a[r], tp[(r - 1) * NS]);
        if (R > 4) asm volatile("" ::: "memory");
      }
    }
    Dft<R, INV>::run(a);
    if constexpr (LAST) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[s + r * BPT] = a[r];
    } else {
      const int base = (b / NS) * NS * R + (b % NS);
      float2* wp = buf + fft_pad(base) * S;
      if constexpr (NS % 16 == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) wp[r * PadStep<NS>::value * S] = a[r];
      } else if constexpr (NS == 1 && R == 16) {  // base = 16 b: pad(base + r) = pad(base) + r
#pragma unroll
        for (int r = 0; r < R; ++r) wp[r * S] = a[r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) buf[fft_pad(base + r * NS) * S] = a[r];
      }
    }
  }
  if constexpr (!LAST) __syncthreads();
}

template <int N, int NS, bool INV, bool FIRST>
HD void fft_passes(float2 (&v)[FftShape<N>::E], int j, float2* buf, int S, const float4* __restrict__ tw) {
  constexpr int REM = N / NS;
  constexpr int R = (REM % 16 == 0) ? 16 : REM;
  constexpr bool LAST = (NS * R == N);
  fft_pass<N, R, NS, INV, FIRST, LAST>(v, j, buf, S, tw);
  if constexpr (!LAST) fft_passes<N, NS * R, INV, false>(v, j, buf, S, tw);
}

// Full length-N transform of the line held by the TPF threads j=0..TPF-1.
// Contains __syncthreads(): every thread of the block must call it.
template <int N, bool INV>
HD void fft_line(float2 (&v)[FftShape<N>::E], int j, float2* buf, int S, const float4* __restrict__ tw) {
  fft_passes<N, 1, INV, true>(v, j, buf, S, tw);
}

}  // namespace holo
