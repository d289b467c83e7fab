// Shared-memory batched 1D FFTs (power-of-two N, 8..4096), register Stockham
// passes of radix E (16 or 32).  No host cuFFT anywhere on the hot path.
//
// Data distribution: the FFT of one line is computed by TPF = N/E threads
// ("j" = 0..TPF-1), each holding E elements in registers.  On entry AND on
// exit thread j holds elements  j + m*TPF,  m = 0..E-1  ("natural
// distribution"), so callers load/store global memory directly from registers
// with coalesced addresses and fuse pre/post operations (transfer multiply,
// scaling, accumulation) element by element.
//
// Passes: radix E while N/NS is a multiple of E, then one pass of the
// remaining radix.  Between passes the line goes through shared memory;
// element i of a line lives at buf[pad(i) * S] (S = element stride: 1 for
// row-contiguous lines, C for C interleaved column lines), pad(i) = i + i/E,
// which keeps the radix-E scatter and the strided reads conflict-free.
// E = 32 halves the shared-memory exchanges of a 1024-point line (32 x 32:
// one exchange, one twiddle pass) at the cost of 64 data registers.
//
// Sign convention (numpy): forward X[k] = sum x[n] exp(-2 pi i nk/N); the
// inverse uses +i and is NOT scaled here (callers fold 1/N into their
// epilogue).  Twiddles come from per-pass tables of (w, conj w), w = exp(-2
// pi i m/N) (fp64-exact entries rounded to fp32) held in shared memory, so a
// table twiddle multiply is one FMUL2 + one FFMA2.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace holo {

template <int N>
struct DefaultE {
  static constexpr int value = N >= 16 ? 16 : N;
};

template <int N, int EE = DefaultE<N>::value>
struct FftShape {
  static_assert(N >= 8 && N <= 4096 && (N & (N - 1)) == 0, "N must be a power of two in [8, 4096]");
  static_assert(EE <= N && (EE == 8 || EE == 16 || EE == 32 || EE == 64 || EE == N), "E must be 8, 16, 32 or 64");
  static constexpr int E = EE;
  static constexpr int TPF = N / E;
  static constexpr int SH = E == 64 ? 6 : E == 32 ? 5 : E == 16 ? 4 : E == 8 ? 3 : E == 4 ? 2 : 1;  // log2 E  // log2 E
  // padded line length in elements; the +2/+TPF term staggers consecutive
  // lines across banks (lines of one warp start on distinct banks)
  static constexpr int PADN = N + N / E + (TPF >= 16 ? 2 : TPF);
};

// Twiddle tables are stored per pass as [row][kk] (kk = butterfly index mod
// NS), so the lanes of a warp (consecutive kk) read consecutive entries:
// conflict-free, or broadcast.  Entry = (w, conj w), w = exp(-2 pi i kk r/(NS R)).
// Only the twiddles fft_pass loads are stored (compact, so the row kernel's
// shared copy is small):
// * the last pass with several butterflies per thread (rotlast): rows
//   r = 1..R-1, kk < TPF only (the other butterflies rotate these);
// * radix-16 / -32 passes (split): rows r = 1, 2, 3 then r = 4, 8, ..., R-4;
// * other passes: rows r = 1..R-1.
template <int N, int E = DefaultE<N>::value>
struct TwLayout {
  static constexpr int radix(int ns) { return ((N / ns) % E == 0) ? E : N / ns; }
  static constexpr bool rotlast(int ns) { return ns * radix(ns) == N && E / radix(ns) > 1; }
  static constexpr bool split(int ns) { return !rotlast(ns) && (radix(ns) == 16 || radix(ns) == 32); }
  static constexpr int rows(int ns) { return split(ns) ? radix(ns) / 4 + 2 : radix(ns) - 1; }
  static constexpr int cols(int ns) { return rotlast(ns) ? N / E : ns; }
  // table row of twiddle power r (split passes)
  static constexpr int row_of(int ns, int r) { return split(ns) ? (r < 4 ? r - 1 : 2 + r / 4) : r - 1; }
  // offset of the table of the pass whose product of earlier radices is ns
  static constexpr int offset(int ns) {
    int off = 0;
    for (int s = E; s < ns; s *= radix(s)) off += rows(s) * cols(s);
    return off;
  }
  static constexpr int size() {
    if (N <= E) return 1;
    int off = 0;
    for (int s = E; s < N; s *= radix(s)) off += rows(s) * cols(s);
    return off;
  }
};
// float2 slots of a kernel's shared copy of the table (128-byte multiple)
template <int N, int E>
constexpr int tw_f2() {
  return (2 * TwLayout<N, E>::size() + 15) & ~15;
}

template <int SH>
HD int fft_pad(int i) { return i + (i >> SH); }

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

// cos / sin of pi k / 16, k = 0..15 (fp64 values rounded to fp32)
struct Trig32 {
  static constexpr float c[16] = {1.0f, 0.98078528040323043f, 0.92387953251128674f, 0.83146961230254524f,
                                  0.70710678118654757f, 0.55557023301960229f, 0.38268343236508984f,
                                  0.19509032201612833f, 0.0f, -0.19509032201612819f, -0.38268343236508973f,
                                  -0.55557023301960196f, -0.70710678118654746f, -0.83146961230254535f,
                                  -0.92387953251128674f, -0.98078528040323043f};
  static constexpr float s[16] = {0.0f, 0.19509032201612825f, 0.38268343236508978f, 0.55557023301960218f,
                                  0.70710678118654746f, 0.83146961230254524f, 0.92387953251128674f,
                                  0.98078528040323043f, 1.0f, 0.98078528040323043f, 0.92387953251128674f,
                                  0.83146961230254546f, 0.70710678118654757f, 0.55557023301960218f,
                                  0.38268343236508989f, 0.19509032201612861f};
};

// x * exp(-/+ 2 pi i e / 32), e compile-time
template <bool INV, int e>
HD float2 rot32(float2 x) {
  constexpr int ee = e & 31;
  if constexpr (ee == 0) {
    return x;
  } else if constexpr (ee == 8) {
    return mul_ni<INV>(x);
  } else if constexpr (ee == 16) {
    return make_float2(-x.x, -x.y);
  } else if constexpr (ee == 24) {
    return mul_ni<!INV>(x);
  } else {
    // angle pi ee / 16 in [0, 2 pi): the second half-turn negates the first
    constexpr int h = ee & 15;
    constexpr float cs = (ee < 16) ? Trig32::c[h] : -Trig32::c[h];
    constexpr float sn = (ee < 16) ? Trig32::s[h] : -Trig32::s[h];
    // forward: multiply by (cs, -sn); inverse: (cs, +sn)
    //   x (cs + i s) = x * cs + swap(x) * (-s, s)
    constexpr float s = INV ? sn : -sn;
    return fma2(swp(x), make_float2(-s, s), mul2(x, make_float2(cs, cs)));
  }
}
template <bool INV, int e>
HD float2 rot16(float2 x) {
  return rot32<INV, 2 * e>(x);
}
// cos / sin of pi k / 32, k = 0..31 (fp32-rounded)
struct Trig64 {
  static constexpr float c[32] = {1.0f, 0.9951847195625305f, 0.9807852506637573f, 0.9569403529167175f, 0.9238795042037964f, 0.8819212913513184f, 0.8314695954322815f, 0.7730104327201843f, 0.7071067690849304f, 0.6343932747840881f, 0.5555702447891235f, 0.4713967442512512f, 0.3826834261417389f, 0.290284663438797f, 0.19509032368659973f, 0.0980171412229538f, 6.123234262925839e-17f, -0.0980171412229538f, -0.19509032368659973f, -0.290284663438797f, -0.3826834261417389f, -0.4713967442512512f, -0.5555702447891235f, -0.6343932747840881f, -0.7071067690849304f, -0.7730104327201843f, -0.8314695954322815f, -0.8819212913513184f, -0.9238795042037964f, -0.9569403529167175f, -0.9807852506637573f, -0.9951847195625305f};
  static constexpr float s[32] = {0.0f, 0.0980171412229538f, 0.19509032368659973f, 0.290284663438797f, 0.3826834261417389f, 0.4713967442512512f, 0.5555702447891235f, 0.6343932747840881f, 0.7071067690849304f, 0.7730104327201843f, 0.8314695954322815f, 0.8819212913513184f, 0.9238795042037964f, 0.9569403529167175f, 0.9807852506637573f, 0.9951847195625305f, 1.0f, 0.9951847195625305f, 0.9807852506637573f, 0.9569403529167175f, 0.9238795042037964f, 0.8819212913513184f, 0.8314695954322815f, 0.7730104327201843f, 0.7071067690849304f, 0.6343932747840881f, 0.5555702447891235f, 0.4713967442512512f, 0.3826834261417389f, 0.290284663438797f, 0.19509032368659973f, 0.0980171412229538f};
};
// x * exp(-/+ 2 pi i e / 64), e compile-time
template <bool INV, int e>
HD float2 rot64(float2 x) {
  constexpr int ee = e & 63;
  if constexpr ((ee & 1) == 0) {
    return rot32<INV, ee / 2>(x);
  } else {
    constexpr int h = ee & 31;
    constexpr float cs = (ee < 32) ? Trig64::c[h] : -Trig64::c[h];
    constexpr float sn = (ee < 32) ? Trig64::s[h] : -Trig64::s[h];
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
// 32 = 2 x 16: DFT16 of the even and odd samples, X[k] = E[k] +- w32^k O[k].
template <bool INV>
struct Dft<32, INV> {
  template <int K>
  static HD void combine(float2 (&ev)[16], float2 (&od)[16], float2 (&a)[32]) {
    if constexpr (K < 16) {
      const float2 o = rot32<INV, K>(od[K]);
      a[K] = add2(ev[K], o);
      a[K + 16] = sub2(ev[K], o);
      combine<K + 1>(ev, od, a);
    }
  }
  static HD void run(float2 (&a)[32]) {
    float2 ev[16], od[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      ev[i] = a[2 * i];
      od[i] = a[2 * i + 1];
    }
    Dft<16, INV>::run(ev);
    Dft<16, INV>::run(od);
    combine<0>(ev, od, a);
  }
};

// 64 = 2 x 32: DFT32 of the even and odd samples, X[k] = E[k] +- w64^k O[k].
template <bool INV>
struct Dft<64, INV> {
  template <int K>
  static HD void combine(float2 (&ev)[32], float2 (&od)[32], float2 (&a)[64]) {
    if constexpr (K < 32) {
      const float2 o = rot64<INV, K>(od[K]);
      a[K] = add2(ev[K], o);
      a[K + 32] = sub2(ev[K], o);
      combine<K + 1>(ev, od, a);
    }
  }
  static HD void run(float2 (&a)[64]) {
    float2 ev[32], od[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      ev[i] = a[2 * i];
      od[i] = a[2 * i + 1];
    }
    Dft<32, INV>::run(ev);
    Dft<32, INV>::run(od);
    combine<0>(ev, od, a);
  }
};
template <bool INV, int E, int R, int S, int RR>
HD void rot_apply(float2 (&a)[R]);
// x * exp(-/+ 2 pi i e / E), e compile-time, E in {8, 16, 32, 64}
template <bool INV, int E, int e>
HD float2 rotE(float2 x) {
  if constexpr (E == 64)
    return rot64<INV, e>(x);
  else
    return rot32<INV, e * (32 / E)>(x);
}
template <bool INV, int E, int R, int S, int RR>
HD void rot_apply(float2 (&a)[R]) {
  if constexpr (RR < R) {
    a[RR] = rotE<INV, E, (S * RR) % E>(a[RR]);
    rot_apply<INV, E, R, S, RR + 1>(a);
  }
}
// last-pass twiddles of butterfly s: table twiddle of butterfly 0 (t0[r-1]),
// then the compile-time rotation by s r / E turns (S runs over 0..E-1 so s
// can be matched against a template argument)
template <bool INV, int E, int R, int S>
HD void rot_twiddles(float2 (&a)[R], const float4 (&t0)[R - 1], std::integral_constant<int, S>, int s) {
  if constexpr (S < E / R) {
    if (s == S) {
#pragma unroll
      for (int r = 1; r < R; ++r) a[r] = twiddle<INV>(a[r], t0[r - 1]);
      rot_apply<INV, E, R, S, 1>(a);
    } else {
      rot_twiddles<INV, E, R, S + 1>(a, t0, std::integral_constant<int, S + 1>(), s);
    }
  }
}

// One Stockham pass of radix R with NS = product of earlier radices.
template <int N, int E, int R, int NS, bool INV, bool FIRST, bool LAST>
HD void fft_pass(float2 (&v)[E], int j, float2* buf, int S, const float4* __restrict__ tw) {
  using Sh = FftShape<N, E>;
  constexpr int TPF = Sh::TPF, BPT = E / R, SH = Sh::SH;
  static_assert(E % R == 0, "radix must divide E");
  if constexpr (!FIRST) {
    if constexpr (TPF % E == 0) {
      // pad(j + m TPF) = pad(j) + m (TPF + TPF/E): one address, immediate offsets
      const float2* rp = buf + fft_pad<SH>(j) * S;
#pragma unroll
      for (int m = 0; m < E; ++m) v[m] = rp[m * (TPF + TPF / E) * S];
    } else {
#pragma unroll
      for (int m = 0; m < E; ++m) v[m] = buf[fft_pad<SH>(j + m * TPF) * S];
    }
    if constexpr (!LAST) __syncthreads();  // everyone has read before anyone writes
  } else if constexpr (!LAST) {
    __syncthreads();  // buffer may still be read by a previous transform's last pass
  }
  // Twiddle loads are shared-memory wavefronts, the bound of the column
  // passes (a quarter of their wavefronts at N = 1024, E = 16), so:
  // * the last pass with several butterflies per thread (BPT > 1) loads the
  //   s = 0 butterfly's R-1 twiddles once: butterfly s has kk = j + s TPF < NS
  //   and w^(kk r) = w^(j r) exp(-/+ 2 pi i s r / E), a compile-time rotation;
  // * a radix-16 / radix-32 pass factors w^(kk r) = w^(kk r1) w^(kk 4 r2),
  //   r = r1 + 4 r2: 6 (10) table loads instead of 15 (31), one more rounding
  //   where both factors are nonzero.  Measured (C3, 10 iterations): adjoint
  //   columns 12.18 -> 11.16 ms, forward columns 12.34 -> 12.08, row passes
  //   15.22 / 14.97 -> 14.49 / 14.24.
  using TL = TwLayout<N, E>;
  constexpr bool kRotLast = NS > 1 && TL::rotlast(NS);
  constexpr bool kSplit = NS > 1 && TL::split(NS);
  static_assert(!kRotLast || (LAST && BPT > 1), "");
  float4 t0[kRotLast ? R - 1 : 1];
  if constexpr (kRotLast) {
    const float4* tp = tw + TL::offset(NS) + j;  // kk of butterfly s = 0
#pragma unroll
    for (int r = 1; r < R; ++r) t0[r - 1] = tp[(r - 1) * TL::cols(NS)];
  }
#pragma unroll
  for (int s = 0; s < BPT; ++s) {
    const int b = j + s * TPF;
    float2 a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = v[s + r * BPT];
    if constexpr (kRotLast) {
      rot_twiddles<INV, E, R>(a, t0, std::integral_constant<int, 0>(), s);
    } else if constexpr (kSplit) {
      const int kk = b % NS;
      const float4* tp = tw + TL::offset(NS) + kk;
      {  // w^(kk 4 r2), r2 = 1..R/4-1, on a[4 r2 .. 4 r2 + 3]
        float4 th[R / 4 - 1];
#pragma unroll
        for (int r2 = 1; r2 < R / 4; ++r2) th[r2 - 1] = tp[TL::row_of(NS, 4 * r2) * NS];
#pragma unroll
        for (int r = 4; r < R; ++r) a[r] = twiddle<INV>(a[r], th[r / 4 - 1]);
      }
      asm volatile("" ::: "memory");
      {  // w^(kk r1), r1 = 1..3, on a[r1 + 4 r2]
        float4 tl[3];
#pragma unroll
        for (int r1 = 1; r1 < 4; ++r1) tl[r1 - 1] = tp[TL::row_of(NS, r1) * NS];
#pragma unroll
        for (int r = 1; r < R; ++r)
          if (r % 4) a[r] = twiddle<INV>(a[r], tl[r % 4 - 1]);
      }
    } else if constexpr (NS > 1) {
      const int kk = b % NS;
      const float4* tp = tw + TL::offset(NS) + kk;
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
      float2* wp = buf + fft_pad<SH>(base) * S;
      if constexpr (NS % E == 0) {  // pad(base + r NS) = pad(base) + r (NS + NS/E)
#pragma unroll
        for (int r = 0; r < R; ++r) wp[r * (NS + NS / E) * S] = a[r];
      } else if constexpr (NS == 1 && R == E) {  // base = E b: pad(base + r) = pad(base) + r
#pragma unroll
        for (int r = 0; r < R; ++r) wp[r * S] = a[r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) buf[fft_pad<SH>(base + r * NS) * S] = a[r];
      }
    }
  }
  if constexpr (!LAST) __syncthreads();
}

template <int N, int E, int NS, bool INV, bool FIRST>
HD void fft_passes(float2 (&v)[E], int j, float2* buf, int S, const float4* __restrict__ tw) {
  constexpr int REM = N / NS;
  constexpr int R = (REM % E == 0) ? E : REM;
  constexpr bool LAST = (NS * R == N);
  fft_pass<N, E, R, NS, INV, FIRST, LAST>(v, j, buf, S, tw);
  if constexpr (!LAST) fft_passes<N, E, NS * R, INV, false>(v, j, buf, S, tw);
}

// Full length-N transform of the line held by the TPF threads j=0..TPF-1.
// Contains __syncthreads(): every thread of the block must call it.
template <int N, bool INV, int E = DefaultE<N>::value>
HD void fft_line(float2 (&v)[E], int j, float2* buf, int S, const float4* __restrict__ tw) {
  fft_passes<N, E, 1, INV, true>(v, j, buf, S, tw);
}

}  // namespace holo
