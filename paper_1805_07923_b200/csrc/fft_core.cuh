// In-place mixed-radix FFT on shared memory, fp64.
//
// Replaces the reference's longitude transforms np.fft.rfft / np.fft.irfft
// (spharm.py:210-222).  One "ring" of n_lon points lives in shared memory as
// complex (double2) values; two real latitude rings (a north/south mirror
// pair) are packed into one complex ring z = g_north + i g_south so a single
// complex FFT serves both (see fourier.cu).
//
//   forward  : decimation in frequency, natural-order input, digit-reversed
//              output, twiddles exp(-2 pi i e / N)
//   inverse  : decimation in time, digit-reversed input, natural-order output,
//              conjugate twiddles
//
// Radices: 4, 2, 3, 5 specialised, any other prime via a direct DFT, so every
// n_lon works (the reference accepts any n_lon >= 2R+1, spharm.py:192-195).
// The index math is __host__ __device__ so tests/fft_selftest.cpp checks it
// against a naive DFT on the CPU.
#pragma once

#ifdef __CUDACC__
#define SW_HD __host__ __device__ __forceinline__
#else
#define SW_HD inline
#include <cmath>
struct double2 { double x, y; };
#endif

namespace swfft {

constexpr int kMaxStages = 24;

struct FftPlan {
  int n;                    // ring length
  int nstage;               // number of radix stages
  int radix[kMaxStages];    // radix of stage s (stage 0 splits n first in DIF)
  int span[kMaxStages];     // block length L at stage s (L_0 = n, L_{s+1} = L_s / radix_s)
};

// Factor n: as many 4s as possible, then a 2, then 3s, 5s, then other primes.
inline FftPlan make_fft_plan(int n) {
  FftPlan p{};
  p.n = n;
  int m = n, k = 0;
  int rad[kMaxStages];
  while (m % 4 == 0) { rad[k++] = 4; m /= 4; }
  while (m % 2 == 0) { rad[k++] = 2; m /= 2; }
  while (m % 3 == 0) { rad[k++] = 3; m /= 3; }
  while (m % 5 == 0) { rad[k++] = 5; m /= 5; }
  for (int f = 7; m > 1; f += 2) {
    while (m % f == 0) { rad[k++] = f; m /= f; }
  }
  p.nstage = k;
  int L = n;
  for (int s = 0; s < k; ++s) {
    p.radix[s] = rad[s];
    p.span[s] = L;
    L /= rad[s];
  }
  return p;
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

// twiddle exp(sign * 2 pi i e / n) from the table tw[e] = exp(-2 pi i e / n)
SW_HD double2 twid(const double2* tw, int n, long long e, bool inverse) {
  int idx = (int)(e % n);
  double2 w = tw[idx];
  if (inverse) w.y = -w.y;
  return w;
}

// Small DFT of radix r on v[0..r-1] in place.  inverse=false: exp(-2 pi i ...).
template <int R>
SW_HD void small_dft(double2* v, bool inverse) {
  if (R == 2) {
    double2 a = v[0], b = v[1];
    v[0] = cadd(a, b); v[1] = csub(a, b);
  } else if (R == 4) {
    double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    double2 a2 = cadd(v[1], v[3]), a3 = csub(v[1], v[3]);
    // -i * a3 (forward) or +i * a3 (inverse)
    double2 j3;
    if (!inverse) { j3.x = a3.y; j3.y = -a3.x; } else { j3.x = -a3.y; j3.y = a3.x; }
    v[0] = cadd(a0, a2); v[2] = csub(a0, a2);
    v[1] = cadd(a1, j3); v[3] = csub(a1, j3);
  } else if (R == 3) {
    const double c1 = -0.5;
    const double s1 = inverse ? 0.86602540378443864676 : -0.86602540378443864676;
    double2 t = cadd(v[1], v[2]), d = csub(v[1], v[2]);
    double2 m; m.x = v[0].x + c1 * t.x; m.y = v[0].y + c1 * t.y;
    double2 js; js.x = -s1 * d.y; js.y = s1 * d.x;  // i*s1*d
    v[0] = cadd(v[0], t);
    v[1] = cadd(m, js);
    v[2] = csub(m, js);
  } else if (R == 5) {
    const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    const double sg = inverse ? 1.0 : -1.0;
    const double s1 = sg * 0.95105651629515357212, s2 = sg * 0.58778525229247312917;
    double2 t1 = cadd(v[1], v[4]), d1 = csub(v[1], v[4]);
    double2 t2 = cadd(v[2], v[3]), d2 = csub(v[2], v[3]);
    double2 m1, m2;
    m1.x = v[0].x + c1 * t1.x + c2 * t2.x; m1.y = v[0].y + c1 * t1.y + c2 * t2.y;
    m2.x = v[0].x + c2 * t1.x + c1 * t2.x; m2.y = v[0].y + c2 * t1.y + c1 * t2.y;
    double2 n1, n2;  // i*(s1 d1 + s2 d2), i*(s2 d1 - s1 d2)
    n1.x = -(s1 * d1.y + s2 * d2.y); n1.y = s1 * d1.x + s2 * d2.x;
    n2.x = -(s2 * d1.y - s1 * d2.y); n2.y = s2 * d1.x - s1 * d2.x;
    v[0].x = v[0].x + t1.x + t2.x; v[0].y = v[0].y + t1.y + t2.y;
    v[1] = cadd(m1, n1); v[4] = csub(m1, n1);
    v[2] = cadd(m2, n2); v[3] = csub(m2, n2);
  }
}

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
      double2 w = twid(tw, n, (long long)((q * t) % R) * step, inverse);
      acc = cadd(acc, cmul(v[t], w));
    }
    tmp[q] = acc;
  }
#pragma unroll
  for (int q = 0; q < R; ++q) v[q] = tmp[q];
}

// Largest prime factor of n_lon supported (plan creation rejects others).
constexpr int kMaxPrime = 13;

// One butterfly of stage s, butterfly index b in [0, n/radix), radix fixed at
// compile time.  DIF (forward): load, DFT, twiddle, store.
// DIT (inverse): load, twiddle, DFT, store.
template <int R>
SW_HD void stage_butterfly_t(double2* buf, const FftPlan& p, int s, int b, const double2* tw,
                             bool inverse) {
  const int L = p.span[s];
  const int m = L / R;
  const int blk = b / m, j = b - blk * m;
  const int base = blk * L + j;
  const long long tstep = (long long)(p.n / L) * j;  // W_L^{j q} = W_n^{q j n/L}
  double2 v[R];
#pragma unroll
  for (int q = 0; q < R; ++q) v[q] = buf[base + q * m];
  if (inverse && j != 0) {
#pragma unroll
    for (int q = 1; q < R; ++q) v[q] = cmul(v[q], twid(tw, p.n, tstep * q, true));
  }
  if (R <= 5) small_dft<R>(v, inverse);
  else prime_dft<R>(v, tw, p.n, inverse);
  if (!inverse && j != 0) {
#pragma unroll
    for (int q = 1; q < R; ++q) v[q] = cmul(v[q], twid(tw, p.n, tstep * q, false));
  }
#pragma unroll
  for (int q = 0; q < R; ++q) buf[base + q * m] = v[q];
}

// BIGP selects whether the rare prime radices 7, 11, 13 are compiled in (they
// raise register pressure, so kernels are instantiated both ways).
template <bool BIGP = true>
SW_HD void stage_butterfly(double2* buf, const FftPlan& p, int s, int b, const double2* tw,
                           bool inverse) {
  switch (p.radix[s]) {
    case 4: stage_butterfly_t<4>(buf, p, s, b, tw, inverse); break;
    case 2: stage_butterfly_t<2>(buf, p, s, b, tw, inverse); break;
    case 3: stage_butterfly_t<3>(buf, p, s, b, tw, inverse); break;
    case 5: stage_butterfly_t<5>(buf, p, s, b, tw, inverse); break;
    default:
      if (BIGP) {
        if (p.radix[s] == 7) stage_butterfly_t<7>(buf, p, s, b, tw, inverse);
        else if (p.radix[s] == 11) stage_butterfly_t<11>(buf, p, s, b, tw, inverse);
        else stage_butterfly_t<13>(buf, p, s, b, tw, inverse);
      }
  }
}

// True when n needs one of the prime radices 7, 11, 13.
inline bool fft_needs_bigp(int n) {
  for (int f : {2, 3, 5}) while (n % f == 0) n /= f;
  return n != 1;
}

// True when every prime factor of n is <= kMaxPrime.
inline bool fft_supported(int n) {
  if (n < 1) return false;
  for (int f : {2, 3, 5, 7, 11, 13}) while (n % f == 0) n /= f;
  return n == 1;
}

// Whole transform on one ring, sequentially (host self-test and reference).
inline void fft_forward_serial(double2* buf, const FftPlan& p, const double2* tw) {
  for (int s = 0; s < p.nstage; ++s)
    for (int b = 0; b < p.n / p.radix[s]; ++b) stage_butterfly(buf, p, s, b, tw, false);
}
inline void fft_inverse_serial(double2* buf, const FftPlan& p, const double2* tw) {
  for (int s = p.nstage - 1; s >= 0; --s)
    for (int b = 0; b < p.n / p.radix[s]; ++b) stage_butterfly(buf, p, s, b, tw, true);
}

}  // namespace swfft
