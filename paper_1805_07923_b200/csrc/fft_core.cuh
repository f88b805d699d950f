// In-place mixed-radix FFT on shared memory, fp64.
//
// Replaces the reference's longitude transforms np.fft.rfft / np.fft.irfft
// (spharm.py:210-222).  One "ring" of n_lon points lives in shared memory as
// complex (double2) values; two real latitude rings (a north/south mirror
// pair) are packed into one complex ring z = g_north + i g_south so a single
// complex FFT serves both (see fourier.cu).
//
// Both directions run decimation in time: digit-reversed input (the loaders
// scatter through a permutation table), natural-order output, twiddles
// applied before each butterfly (exp(-2 pi i e / N) forward, conjugate
// inverse).  A DIF variant (natural in, digit-reversed out) is kept for the
// self-test.
//
// Stages use radix 16, 8, 4, 2, 3, 5 (register butterflies; 16 and 8 are
// 4x4 / 2x4 decompositions with constant inner twiddles) and 7, 11, 13 via a
// direct DFT, so every n_lon with prime factors <= 13 works.  Ring storage is
// padded (one slot per 16 points) so strided butterfly accesses are free of
// shared-memory bank conflicts; block/offset indices use precomputed
// multiply-high reciprocals instead of integer division.  The index math is
// __host__ __device__ so tests/csrc/fft_selftest.cpp checks it against a naive
// DFT on the CPU.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define SW_HD __host__ __device__ __forceinline__
#else
#define SW_HD inline
#include <cmath>
struct double2 { double x, y; };
#endif

namespace swfft {

constexpr int kMaxStages = 16;

struct FftPlan {
  int n;                    // ring length
  int nstage;               // number of radix stages
  int radix[kMaxStages];    // radix of stage s (stage 0 splits n first in DIF)
  int span[kMaxStages];     // block length L at stage s (L_0 = n, L_{s+1} = L_s / radix_s)
  uint32_t mmag[kMaxStages];  // umulhi reciprocal of m_s = span_s / radix_s
  uint32_t bmag[kMaxStages];  // umulhi reciprocal of n / radix_s (butterflies per ring)
};

// Padded ring slot of point i: one spare slot per 16 points.
SW_HD int pad_idx(int i) { return i + (i >> 4); }
SW_HD int padded_len(int n) { return n + (n >> 4) + 1; }

// floor(x / d) for x < 2^32 / d via multiply-high with mag = ceil(2^32 / d).
SW_HD uint32_t udiv(uint32_t x, uint32_t mag) {
#ifdef __CUDA_ARCH__
  return __umulhi(x, mag);
#else
  return (uint32_t)(((uint64_t)x * mag) >> 32);
#endif
}
inline uint32_t magic_for(uint32_t d) {
  return d == 1 ? 0xFFFFFFFFu : (uint32_t)((((uint64_t)1 << 32) + d - 1) / d);
}

// Factor n into stage radices: 16s, then one 8/4/2 for the remaining power of
// two, then 3, 5, 7, 11, 13.
inline FftPlan make_fft_plan(int n, int max_radix = 16) {
  FftPlan p{};
  p.n = n;
  int m = n, k = 0;
  int rad[64];
  while (max_radix >= 16 && m % 16 == 0) { rad[k++] = 16; m /= 16; }
  while (max_radix == 8 && m % 8 == 0) { rad[k++] = 8; m /= 8; }
  if (m % 8 == 0) { rad[k++] = 8; m /= 8; }
  if (m % 4 == 0) { rad[k++] = 4; m /= 4; }
  if (m % 2 == 0) { rad[k++] = 2; m /= 2; }
  for (int f : {3, 5, 7, 11, 13})
    while (m % f == 0) { rad[k++] = f; m /= f; }
  if (m != 1 || k > kMaxStages) { p.nstage = -1; return p; }
  p.nstage = k;
  int L = n;
  for (int s = 0; s < k; ++s) {
    p.radix[s] = rad[s];
    p.span[s] = L;
    p.mmag[s] = magic_for((uint32_t)(L / rad[s]));
    p.bmag[s] = magic_for((uint32_t)(n / rad[s]));
    L /= rad[s];
  }
  return p;
}

// True when every prime factor of n is <= 13.
inline bool fft_supported(int n) {
  if (n < 1) return false;
  for (int f : {2, 3, 5, 7, 11, 13}) while (n % f == 0) n /= f;
  return n == 1;
}

// True when n needs one of the prime radices 7, 11, 13.
inline bool fft_needs_bigp(int n) {
  for (int f : {2, 3, 5}) while (n % f == 0) n /= f;
  return n != 1;
}

// Position of frequency k in the digit-reversed DIF output.
// k = k_0 + p_0 (k_1 + p_1 (k_2 + ...)),  pos = sum_s k_s * (n / (p_0 ... p_s)).
SW_HD int digit_rev(const FftPlan& p, int k) {
  int pos = 0;
  for (int s = 0; s < p.nstage; ++s) {
    const int r = p.radix[s];
    pos += (k % r) * (p.span[s] / r);
    k /= r;
  }
  return pos;
}

SW_HD double2 cmul(double2 a, double2 b) {
  double2 c;
  c.x = a.x * b.x - a.y * b.y;
  c.y = a.x * b.y + a.y * b.x;
  return c;
}
SW_HD double2 cadd(double2 a, double2 b) { double2 c; c.x = a.x + b.x; c.y = a.y + b.y; return c; }
SW_HD double2 csub(double2 a, double2 b) { double2 c; c.x = a.x - b.x; c.y = a.y - b.y; return c; }
SW_HD double2 conj2(double2 a) { a.y = -a.y; return a; }
SW_HD double2 mk2(double x, double y) { double2 c; c.x = x; c.y = y; return c; }

// multiply by -i (forward) / +i (inverse)
SW_HD double2 rot_mi(double2 a, bool inverse) {
  return inverse ? mk2(-a.y, a.x) : mk2(a.y, -a.x);
}

SW_HD void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

// 4-point DFT of (a0, a1, a2, a3) in natural order.
SW_HD void dft4(double2& a0, double2& a1, double2& a2, double2& a3, bool inverse) {
  double2 s0 = cadd(a0, a2), d0 = csub(a0, a2);
  double2 s1 = cadd(a1, a3), d1 = rot_mi(csub(a1, a3), inverse);
  a0 = cadd(s0, s1);
  a2 = csub(s0, s1);
  a1 = cadd(d0, d1);
  a3 = csub(d0, d1);
}

// Small DFT of radix R on v[0..R-1] in place.  inverse=false: exp(-2 pi i ...).
template <int R>
SW_HD void small_dft(double2* v, bool inverse) {
  if (R == 2) {
    dft2(v[0], v[1]);
  } else if (R == 4) {
    dft4(v[0], v[1], v[2], v[3], inverse);
  } else if (R == 8) {
    // X[k] = E[k] + w^k O[k], X[k+4] = E[k] - w^k O[k]
    const double h = 0.70710678118654752440;
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4(e0, e1, e2, e3, inverse);
    dft4(o0, o1, o2, o3, inverse);
    const double sg = inverse ? 1.0 : -1.0;
    // w^1 = (1 + sg i) h, w^2 = sg i, w^3 = (-1 + sg i) h
    double2 t1 = mk2(h * (o1.x - sg * o1.y), h * (o1.y + sg * o1.x));
    double2 t2 = mk2(-sg * o2.y, sg * o2.x);
    double2 t3 = mk2(h * (-o3.x - sg * o3.y), h * (-o3.y + sg * o3.x));
    v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
    v[1] = cadd(e1, t1); v[5] = csub(e1, t1);
    v[2] = cadd(e2, t2); v[6] = csub(e2, t2);
    v[3] = cadd(e3, t3); v[7] = csub(e3, t3);
  } else if (R == 16) {
    // n = n1 + 4 n2, k = k1 + 4 k2: DFT4 over n2, twiddle w16^(n1 k1), DFT4 over
    // n1.  Output X[k1 + 4 k2] is left at v[4 k1 + k2] (transposed); callers
    // use out16() to read it back in natural order.
    const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
    const double c2 = 0.70710678118654752440;
    const double sg = inverse ? 1.0 : -1.0;
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) dft4(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12], inverse);
    const double wc[10] = {1.0, c1, c2, s1, 0.0, -s1, -c2, -c1, -1.0, -c1};
    const double ws[10] = {0.0, s1, c2, c1, 1.0, c1, c2, s1, 0.0, -s1};
#pragma unroll
    for (int n1 = 1; n1 < 4; ++n1)
#pragma unroll
      for (int k1 = 1; k1 < 4; ++k1) {
        const int e = n1 * k1;
        v[n1 + 4 * k1] = cmul(v[n1 + 4 * k1], mk2(wc[e], sg * ws[e]));
      }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3], inverse);
  } else if (R == 3) {
    const double c1 = -0.5;
    const double s1 = inverse ? 0.86602540378443864676 : -0.86602540378443864676;
    double2 t = cadd(v[1], v[2]), d = csub(v[1], v[2]);
    double2 m = mk2(v[0].x + c1 * t.x, v[0].y + c1 * t.y);
    double2 js = mk2(-s1 * d.y, s1 * d.x);  // i*s1*d
    v[0] = cadd(v[0], t);
    v[1] = cadd(m, js);
    v[2] = csub(m, js);
  } else if (R == 5) {
    const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    const double sg = inverse ? 1.0 : -1.0;
    const double s1 = sg * 0.95105651629515357212, s2 = sg * 0.58778525229247312917;
    double2 t1 = cadd(v[1], v[4]), d1 = csub(v[1], v[4]);
    double2 t2 = cadd(v[2], v[3]), d2 = csub(v[2], v[3]);
    double2 m1 = mk2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
    double2 m2 = mk2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
    double2 n1 = mk2(-(s1 * d1.y + s2 * d2.y), s1 * d1.x + s2 * d2.x);
    double2 n2 = mk2(-(s2 * d1.y - s1 * d2.y), s2 * d1.x - s1 * d2.x);
    v[0] = mk2(v[0].x + t1.x + t2.x, v[0].y + t1.y + t2.y);
    v[1] = cadd(m1, n1); v[4] = csub(m1, n1);
    v[2] = cadd(m2, n2); v[3] = csub(m2, n2);
  }
}

// Register slot of DFT output q after small_dft<R> (radix 16 leaves it transposed).
template <int R>
SW_HD constexpr int out_slot(int q) { return R == 16 ? 4 * (q & 3) + (q >> 2) : q; }

// Direct DFT for a prime radix R (7, 11, 13) through the n-point twiddle table.
template <int R>
SW_HD void prime_dft(double2* v, const double2* tw, int n, bool inverse) {
  const int step = n / R;
  double2 tmp[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    double2 acc = v[0];
#pragma unroll
    for (int t = 1; t < R; ++t) {
      double2 w = tw[((q * t) % R) * step];
      if (inverse) w.y = -w.y;
      acc = cadd(acc, cmul(v[t], w));
    }
    tmp[q] = acc;
  }
#pragma unroll
  for (int q = 0; q < R; ++q) v[q] = tmp[q];
}

// Twiddles w[q] = W_n^{q e1} (conjugated for the inverse), q = 1..R-1, from the
// table tw[e] = exp(-2 pi i e / n) (q e1 < n always).  Powers beyond the
// loaded ones are formed by at most three complex products.
template <int R>
SW_HD void twiddles(double2* w, const double2* tw, int e1, bool inverse) {
  if (R == 8) {
    w[1] = tw[e1]; w[2] = tw[2 * e1]; w[4] = tw[4 * e1];
    w[3] = cmul(w[1], w[2]); w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]); w[7] = cmul(w[3], w[4]);
  } else if (R == 16) {
    w[1] = tw[e1]; w[2] = tw[2 * e1]; w[4] = tw[4 * e1]; w[8] = tw[8 * e1];
    w[3] = cmul(w[1], w[2]); w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]); w[7] = cmul(w[3], w[4]);
#pragma unroll
    for (int q = 9; q < 16; ++q) w[q] = cmul(w[8], w[q - 8]);
  } else {
#pragma unroll
    for (int q = 1; q < R; ++q) w[q] = tw[q * e1];
  }
  if (inverse) {
#pragma unroll
    for (int q = 1; q < R; ++q) w[q].y = -w[q].y;
  }
}

// One butterfly of stage s on a padded ring, butterfly index b in [0, n/R).
// DIF (forward): load, DFT, twiddle, store.  DIT (inverse): load, twiddle, DFT, store.
// DIT: twiddle-before (digit-reversed input, natural output when the stages
// run last to first); otherwise DIF twiddle-after (natural input, digit-
// reversed output, stages first to last).  CONJ selects exp(+2 pi i ...).
template <int R, bool DIT, bool CONJ>
SW_HD void stage_butterfly_t(double2* buf, const FftPlan& p, int s, int b, const double2* tw) {
  constexpr bool inverse = CONJ;
  const int L = p.span[s];
  const int m = L / R;
  const int blk = (m == 1) ? b : (int)udiv((uint32_t)b, p.mmag[s]);
  const int j = b - blk * m;
  const int base = blk * L + j;
  double2 v[R];
#pragma unroll
  for (int q = 0; q < R; ++q) v[q] = buf[pad_idx(base + q * m)];
  if (R == 16) {
    // twiddles streamed from w^1, w^2, w^4, w^8 to keep register pressure low
    double2 w1 = mk2(1.0, 0.0), w2 = w1, w4 = w1, w8 = w1;
    if (j != 0) {
      const int e1 = j * (p.n / L);
      w1 = tw[e1]; w2 = tw[2 * e1]; w4 = tw[4 * e1]; w8 = tw[8 * e1];
      if (inverse) { w1.y = -w1.y; w2.y = -w2.y; w4.y = -w4.y; w8.y = -w8.y; }
    }
    if (DIT && j != 0) {
#pragma unroll
      for (int q = 1; q < 16; ++q) {
        double2 w = (q & 1) ? w1 : mk2(1.0, 0.0);
        if (q & 2) w = (q & 1) ? cmul(w, w2) : w2;
        if (q & 4) w = (q & 3) ? cmul(w, w4) : w4;
        if (q & 8) w = (q & 7) ? cmul(w, w8) : w8;
        v[q] = cmul(v[q], w);
      }
    }
    small_dft<16>(v, inverse);
    if (!DIT && j != 0) {
#pragma unroll
      for (int q = 1; q < 16; ++q) {
        double2 w = (q & 1) ? w1 : mk2(1.0, 0.0);
        if (q & 2) w = (q & 1) ? cmul(w, w2) : w2;
        if (q & 4) w = (q & 3) ? cmul(w, w4) : w4;
        if (q & 8) w = (q & 7) ? cmul(w, w8) : w8;
        v[out_slot<16>(q)] = cmul(v[out_slot<16>(q)], w);
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) buf[pad_idx(base + q * m)] = v[out_slot<16>(q)];
    return;
  }
  double2 w[R];
  if (j != 0) twiddles<R>(w, tw, j * (p.n / L), inverse);
  if (DIT && j != 0) {
#pragma unroll
    for (int q = 1; q < R; ++q) v[q] = cmul(v[q], w[q]);
  }
  if (R == 7 || R == 11 || R == 13) prime_dft<R>(v, tw, p.n, inverse);
  else small_dft<R>(v, inverse);
  if (!DIT && j != 0) {
#pragma unroll
    for (int q = 1; q < R; ++q) v[q] = cmul(v[q], w[q]);
  }
#pragma unroll
  for (int q = 0; q < R; ++q) buf[pad_idx(base + q * m)] = v[q];
}

// BIGP selects whether the rare prime radices 7, 11, 13 are compiled in (they
// raise register pressure, so kernels are instantiated both ways).
template <bool BIGP, bool DIT, bool CONJ>
SW_HD void stage_butterfly(double2* buf, const FftPlan& p, int s, int b, const double2* tw) {
  switch (p.radix[s]) {
    case 16: stage_butterfly_t<16, DIT, CONJ>(buf, p, s, b, tw); break;
    case 8: stage_butterfly_t<8, DIT, CONJ>(buf, p, s, b, tw); break;
    case 4: stage_butterfly_t<4, DIT, CONJ>(buf, p, s, b, tw); break;
    case 2: stage_butterfly_t<2, DIT, CONJ>(buf, p, s, b, tw); break;
    case 3: stage_butterfly_t<3, DIT, CONJ>(buf, p, s, b, tw); break;
    case 5: stage_butterfly_t<5, DIT, CONJ>(buf, p, s, b, tw); break;
    default:
      if (BIGP) {
        if (p.radix[s] == 7) stage_butterfly_t<7, DIT, CONJ>(buf, p, s, b, tw);
        else if (p.radix[s] == 11) stage_butterfly_t<11, DIT, CONJ>(buf, p, s, b, tw);
        else stage_butterfly_t<13, DIT, CONJ>(buf, p, s, b, tw);
      }
  }
}

// Whole transforms on one padded ring, sequentially (host self-test).
// DIF forward: natural in, digit-reversed out.
inline void fft_forward_dif_serial(double2* buf, const FftPlan& p, const double2* tw) {
  for (int s = 0; s < p.nstage; ++s)
    for (int b = 0; b < p.n / p.radix[s]; ++b) stage_butterfly<true, false, false>(buf, p, s, b, tw);
}
// DIT (what the kernels run): digit-reversed in, natural out; CONJ = inverse.
template <bool CONJ>
inline void fft_dit_serial(double2* buf, const FftPlan& p, const double2* tw) {
  for (int s = p.nstage - 1; s >= 0; --s)
    for (int b = 0; b < p.n / p.radix[s]; ++b) stage_butterfly<true, true, CONJ>(buf, p, s, b, tw);
}

}  // namespace swfft
