// Register-resident complex FFT of one ring of N = 32 K points per warp.
//
// Lane l holds x[32 k + l] in v[k] (k < K).  With m = m1 + K m2,
//   X[m] = sum_l W_32^(l m2) W_N^(l m1) sum_k x[32 k + l] W_K^(k m1),
// so the transform is (A) a K-point DFT over the lane's own registers,
// (B) the twiddle W_N^(l m1) on slot m1, (C) a 32-point DFT across the lanes
// (radix-2 decimation in frequency over shfl.xor; half exchanges for even K,
// see below).  Afterwards slot q of lane l holds X[ring_out_index(l, q)]
// (odd K: X[q + K brev5(l)]).  No shared memory and no barriers: the only
// latency is the shuffles', and every stage has K (or K/2) independent chains.
// ring_fft_dit is the transposed transform (input in that order, natural out).
//
// Twiddles come from the plan table tw[e] = exp(-2 pi i e / N) (capi.cu),
// conjugated for the inverse: W_K^e = tw[32 e], W_32^e = tw[K e].
#pragma once

#include "fft_core.cuh"

namespace swfft {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double2 tw_at(const double2* tw, int e, bool inverse) {
  double2 w = tw[e];
  if (inverse) w.y = -w.y;
  return w;
}

// W_K^e (conjugated for the inverse) for K dividing 24 or 20, as compile-time
// constants: inside the unrolled DFTs e is a constant, so these fold into
// immediates instead of table loads.
template <int K, bool INV>
__device__ __forceinline__ double2 wk(int e) {
  constexpr double h = 0.70710678118654752440, r3 = 0.86602540378443864676;
  constexpr double a15 = 0.96592582628906828675, b15 = 0.25881904510252076235;
  if constexpr (24 % K == 0) {
    constexpr double c[24] = {1.0, a15, r3, h, 0.5, b15, 0.0, -b15, -0.5, -h, -r3, -a15,
                              -1.0, -a15, -r3, -h, -0.5, -b15, 0.0, b15, 0.5, h, r3, a15};
    constexpr double s[24] = {0.0, -b15, -0.5, -h, -r3, -a15, -1.0, -a15, -r3, -h, -0.5, -b15,
                              0.0, b15, 0.5, h, r3, a15, 1.0, a15, r3, h, 0.5, b15};
    const int i = (e * (24 / K)) % 24;
    return mk2(c[i], INV ? -s[i] : s[i]);
  } else {
    static_assert(20 % K == 0, "twiddle constants cover K | 24 and K | 20");
    constexpr double c1 = 0.95105651629515357212, s1 = 0.30901699437494742410;
    constexpr double c2 = 0.80901699437494742410, s2 = 0.58778525229247312917;
    constexpr double c[20] = {1.0, c1, c2, s2, s1, 0.0, -s1, -s2, -c2, -c1,
                              -1.0, -c1, -c2, -s2, -s1, 0.0, s1, s2, c2, c1};
    constexpr double s[20] = {0.0, -s1, -s2, -c2, -c1, -1.0, -c1, -c2, -s2, -s1,
                              0.0, s1, s2, c2, c1, 1.0, c1, c2, s2, s1};
    const int i = (e * (20 / K)) % 20;
    return mk2(c[i], INV ? -s[i] : s[i]);
  }
}

// K = A * B: A-point DFTs over stride-B subsequences, twiddles W_K^(kb ma),
// B-point DFTs; natural order in and out.
template <int A, int B, bool INV>
__device__ __forceinline__ void dft_ab(double2* v, const double2* tw) {
  double2 t[A * B];
#pragma unroll
  for (int kb = 0; kb < B; ++kb) {
    double2 a[A];
#pragma unroll
    for (int ka = 0; ka < A; ++ka) a[ka] = v[B * ka + kb];
    small_dft<A>(a, INV);
#pragma unroll
    for (int ma = 0; ma < A; ++ma) {
      double2 z = a[out_slot<A>(ma)];
      if (kb * ma != 0) z = cmul(z, wk<A * B, INV>(kb * ma));
      t[kb * A + ma] = z;
    }
  }
#pragma unroll
  for (int ma = 0; ma < A; ++ma) {
    double2 b[B];
#pragma unroll
    for (int kb = 0; kb < B; ++kb) b[kb] = t[kb * A + ma];
    small_dft<B>(b, INV);
#pragma unroll
    for (int mb = 0; mb < B; ++mb) v[ma + A * mb] = b[out_slot<B>(mb)];
  }
}

// K-point DFT in registers, natural order in and out.
template <int K, bool INV>
__device__ __forceinline__ void dft_k(double2* v, const double2* tw) {
  if constexpr (K == 1) {
  } else if constexpr (K == 2 || K == 3 || K == 4 || K == 5 || K == 8) {
    small_dft<K>(v, INV);
  } else if constexpr (K == 16) {
    small_dft<16>(v, INV);
    double2 t[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) t[q] = v[out_slot<16>(q)];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = t[q];
  } else if constexpr (K == 6) {
    dft_ab<3, 2, INV>(v, tw);
  } else if constexpr (K == 10) {
    dft_ab<5, 2, INV>(v, tw);
  } else if constexpr (K == 12) {
    dft_ab<3, 4, INV>(v, tw);
  } else if constexpr (K == 20) {
    dft_ab<5, 4, INV>(v, tw);
  } else if constexpr (K == 24) {
    dft_ab<3, 8, INV>(v, tw);
  } else {
    static_assert(K == 1, "unsupported register-FFT size");
  }
}

// Ring lengths N = 32 K with a register FFT (K <= 24 keeps v[] at 96 registers).
__host__ __device__ constexpr bool reg_fft_k_ok(int K) {
  return K == 1 || K == 2 || K == 3 || K == 4 || K == 5 || K == 6 || K == 8 || K == 10 ||
         K == 12 || K == 16 || K == 20 || K == 24;
}

// Cross-lane stages come in two forms.  Odd K: every lane exchanges all K slots with
// its partner and computes one output of each butterfly (own + partner on the lower
// lane, (partner - own) * twiddle on the upper one).  Even K (half exchange): a lane
// pair splits the K butterflies -- the lower lane sends its upper register half
// (slots >= K/2) and receives the partner's lower half, the upper lane the reverse
// -- so each lane holds both inputs of K/2 butterflies and computes both outputs:
// half the shuffles (2 K instead of 4 K 32-bit shuffles per stage) and no multiply
// by 1 on the lower lanes.  Sums go to slot u, differences to slot u + K/2, which
// swaps the lane bit with the register-half bit; see ring_out_index for where the
// spectrum ends up.
#ifndef SWSDC_FFT_HX
#define SWSDC_FFT_HX 1   // build with -DSWSDC_FFT_HX=0 for the full-exchange stages (same-box A/B)
#endif
template <int K>
__host__ __device__ constexpr bool half_exchange() { return SWSDC_FFT_HX != 0 && K % 2 == 0; }

// Per-lane twiddles of the cross-lane stages h = 16, 8, 4: W_{2h}^(l mod h).
// Odd K: on the upper lane of each pair, 1 on the lower one.  Half exchange: on
// both lanes (they share l mod h), negated on the upper lane whose difference is
// formed as own - partner.
// tws: stride of tw relative to an N-point table (a sub-transform of a longer
// ring reads the longer ring's table: W_N^e = tw[e * tws]).
//
// Twiddle cache (TWC): the lane-gathered table reads of one transform -- the powers
// W_N^(lane 2^b), b < NB, and the three stage twiddles -- touch ~9 K sectors, one
// LSU wavefront each, and every warp of a CTA gathers the same values.  A CTA that
// runs several transforms fills a [NB + 3][32] cache in shared memory once
// (fill_twiddle_cache) and its transforms read their lane's entries from it (4
// wavefronts per read); `tw` is then the cache, forward values, conjugated on use.
template <int K>
__host__ __device__ constexpr int tw_powers() { return K > 16 ? 5 : K > 8 ? 4 : K > 4 ? 3 : K > 2 ? 2 : 1; }
template <int K>
__host__ __device__ constexpr int tw_cache_entries() { return (tw_powers<K>() + 3) * 32; }

template <int K>
__device__ __forceinline__ void fill_twiddle_cache(double2* cache, const double2* tw, int tid,
                                                   int nthreads) {
  constexpr int NB = tw_powers<K>();
  for (int i = tid; i < (NB + 3) * 32; i += nthreads) {
    const int e = i >> 5, lane = i & 31;
    int idx;
    if (e < NB) {
      idx = lane << e;
    } else {
      const int h = 16 >> (e - NB);
      idx = (lane & (h - 1)) * (16 / h) * K;
    }
    cache[i] = tw[idx];
  }
}

// stage twiddle W_{2h}^(lane mod h), h = 16 >> st
template <int K, bool INV, bool TWC>
__device__ __forceinline__ double2 stage_twiddle(const double2* tw, int lane, int st, int tws) {
  if constexpr (TWC) {
    return tw_at(tw, (tw_powers<K>() + st) * 32 + lane, INV);
  } else {
    const int h = 16 >> st;
    return tw_at(tw, (lane & (h - 1)) * (16 / h) * K * tws, INV);
  }
}
// power W_N^(lane 2^b)
template <int K, bool INV, bool TWC>
__device__ __forceinline__ double2 power_twiddle(const double2* tw, int lane, int b, int tws) {
  if constexpr (TWC) return tw_at(tw, b * 32 + lane, INV);
  else return tw_at(tw, (lane << b) * tws, INV);
}

template <int K, bool INV, bool TWC = false>
__device__ __forceinline__ void cross_twiddles(double2 (&wst)[3], const double2* tw, int lane,
                                               int tws = 1) {
#pragma unroll
  for (int st = 0; st < 3; ++st) {
    const int h = 16 >> st;
    if constexpr (half_exchange<K>()) {
      const double2 w = stage_twiddle<K, INV, TWC>(tw, lane, st, tws);
      wst[st] = (lane & h) ? mk2(-w.x, -w.y) : w;
    } else {
      wst[st] = (lane & h) ? stage_twiddle<K, INV, TWC>(tw, lane, st, tws) : mk2(1.0, 0.0);
    }
  }
}

// Full N-point transform (see the header comment); wst from cross_twiddles.
template <int K, bool INV, bool TWC = false>
__device__ __forceinline__ void ring_fft(double2 (&v)[K], const double2* tw, int lane,
                                         const double2 (&wst)[3], int tws = 1) {
  dft_k<K, INV>(v, tw);
  // W_N^(lane m1) from the gathered powers W_N^(lane 2^b) (2^b < K, so
  // lane 2^b < N) by at most 4 products: 5 table gathers instead of K - 1
  constexpr int NB = tw_powers<K>();
  double2 wp[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) wp[b] = power_twiddle<K, INV, TWC>(tw, lane, b, tws);
#pragma unroll
  for (int m1 = 1; m1 < K; ++m1) {
    double2 w = mk2(1.0, 0.0);
    bool first = true;
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if ((m1 >> b) & 1) {
        w = first ? wp[b] : cmul(w, wp[b]);
        first = false;
      }
    v[m1] = cmul(v[m1], w);
  }
  if constexpr (half_exchange<K>()) {
    constexpr int H = K / 2;
#pragma unroll
    for (int st = 0; st < 5; ++st) {
      const int h = 16 >> st;
      const bool up = (lane & h) != 0;
      const double sg = up ? -1.0 : 1.0;
      const bool rot = (st == 3) && (lane & 1);   // h = 2: W_4^1 on odd lanes
#pragma unroll
      for (int u = 0; u < H; ++u) {
        const double2 kept = up ? v[u + H] : v[u];
        const double2 send = up ? v[u] : v[u + H];
        double2 p;
        p.x = __shfl_xor_sync(kFull, send.x, h);
        p.y = __shfl_xor_sync(kFull, send.y, h);
        v[u] = mk2(kept.x + p.x, kept.y + p.y);
        double2 d = mk2(kept.x - p.x, kept.y - p.y);   // upper lane: -(a - b)
        if (st < 3) {
          d = cmul(d, wst[st]);
        } else {
          d = mk2(sg * d.x, sg * d.y);
          if (st == 3) {
            const double2 r = rot_mi(d, INV);
            d = rot ? r : d;
          }
        }
        v[u + H] = d;
      }
    }
  } else {
#pragma unroll
    for (int st = 0; st < 5; ++st) {
      const int h = 16 >> st;
      const bool up = (lane & h) != 0;
      const double sg = up ? -1.0 : 1.0;
      const bool rot = (st == 3) && up && (lane & 1);   // h = 2: W_4^1 on odd upper lanes
#pragma unroll
      for (int q = 0; q < K; ++q) {
        double2 p;
        p.x = __shfl_xor_sync(kFull, v[q].x, h);
        p.y = __shfl_xor_sync(kFull, v[q].y, h);
        // lower lane: own + partner; upper lane: (partner - own) * twiddle
        double2 d = mk2(fma(sg, v[q].x, p.x), fma(sg, v[q].y, p.y));
        if (st < 3) {
          d = cmul(d, wst[st]);
        } else if (st == 3) {
          const double2 r = rot_mi(d, INV);
          d = rot ? r : d;
        }
        v[q] = d;
      }
    }
  }
}

// Decimation-in-time counterpart: the transpose of ring_fft.  Lane l enters with
// y[ring_out_index<K>(l, q)] in v[q] (exactly what ring_fft leaves behind) and ends
// with Y[32 k + l] in v[k]: the cross-lane stages run in reverse order (h = 1 .. 16,
// butterflies a + w b, a - w b), then the twiddle W_N^(l m1), then the in-lane K-point
// DFT (symmetric, so its own transpose).  A DIF transform followed by pointwise work
// and a DIT transform needs no reordering in between, and a transform whose input is
// gathered anyway (the packed spectrum of a latitude pair) ends in the order in which
// rings are stored: neither scatters through shared memory.
// wd from cross_twiddles_dit: W_{2h}^(l mod h), on every lane for the half exchange,
// on the upper lane of each pair (1 on the lower) otherwise.
template <int K, bool INV, bool TWC = false>
__device__ __forceinline__ void cross_twiddles_dit(double2 (&wd)[3], const double2* tw, int lane,
                                                   int tws = 1) {
#pragma unroll
  for (int st = 0; st < 3; ++st) {
    const int h = 16 >> st;
    const double2 w = stage_twiddle<K, INV, TWC>(tw, lane, st, tws);
    wd[st] = (half_exchange<K>() || (lane & h)) ? w : mk2(1.0, 0.0);
  }
}

template <int K, bool INV, bool TWC = false>
__device__ __forceinline__ void ring_fft_dit(double2 (&v)[K], const double2* tw, int lane,
                                             const double2 (&wd)[3], int tws = 1) {
  if constexpr (half_exchange<K>()) {
    constexpr int H = K / 2;
#pragma unroll
    for (int st = 4; st >= 0; --st) {
      const int h = 16 >> st;
      const bool up = (lane & h) != 0;
      const bool rot = (st == 3) && (lane & 1);   // h = 2: W_4^1 on odd lanes
#pragma unroll
      for (int u = 0; u < H; ++u) {
        double2 d = v[u + H];
        if (st < 3) {
          d = cmul(d, wd[st]);
        } else if (st == 3) {
          const double2 r = rot_mi(d, INV);
          d = rot ? r : d;
        }
        const double2 a = mk2(v[u].x + d.x, v[u].y + d.y);
        const double2 b = mk2(v[u].x - d.x, v[u].y - d.y);
        // the lower lane keeps a (slot u) and takes the partner's a into slot u + H;
        // the upper lane keeps b (slot u + H) and takes the partner's b into slot u
        const double2 send = up ? a : b;
        double2 p;
        p.x = __shfl_xor_sync(kFull, send.x, h);
        p.y = __shfl_xor_sync(kFull, send.y, h);
        v[u] = up ? p : a;
        v[u + H] = up ? b : p;
      }
    }
  } else {
#pragma unroll
    for (int st = 4; st >= 0; --st) {
      const int h = 16 >> st;
      const bool up = (lane & h) != 0;
      const double sg = up ? -1.0 : 1.0;
      const bool rot = (st == 3) && up && (lane & 1);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        double2 t = v[q];
        if (st < 3) {
          t = cmul(t, wd[st]);
        } else if (st == 3) {
          const double2 r = rot_mi(t, INV);
          t = rot ? r : t;
        }
        double2 p;
        p.x = __shfl_xor_sync(kFull, t.x, h);
        p.y = __shfl_xor_sync(kFull, t.y, h);
        // lower lane: own + w partner; upper lane: partner - w own
        v[q] = mk2(fma(sg, t.x, p.x), fma(sg, t.y, p.y));
      }
    }
  }
  constexpr int NB = tw_powers<K>();
  double2 wp[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) wp[b] = power_twiddle<K, INV, TWC>(tw, lane, b, tws);
#pragma unroll
  for (int m1 = 1; m1 < K; ++m1) {
    double2 w = mk2(1.0, 0.0);
    bool first = true;
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if ((m1 >> b) & 1) {
        w = first ? wp[b] : cmul(w, wp[b]);
        first = false;
      }
    v[m1] = cmul(v[m1], w);
  }
  dft_k<K, INV>(v, tw);
}

template <int K>
__device__ __forceinline__ int ring_out_index(int lane, int q);

// 15-point DFT in registers, natural order in and out: prime-factor
// (Good-Thomas) 3 x 5 with no twiddles -- input n = (5 na + 3 nb) mod 15,
// output k = (10 ka + 6 kb) mod 15.
template <bool INV>
__device__ __forceinline__ void dft15(double2 (&v)[15]) {
  double2 t[3][5];
#pragma unroll
  for (int na = 0; na < 3; ++na) {
#pragma unroll
    for (int nb = 0; nb < 5; ++nb) t[na][nb] = v[(5 * na + 3 * nb) % 15];
    small_dft<5>(t[na], INV);
  }
#pragma unroll
  for (int kb = 0; kb < 5; ++kb) {
    double2 u[3] = {t[0][kb], t[1][kb], t[2][kb]};
    small_dft<3>(u, INV);
#pragma unroll
    for (int ka = 0; ka < 3; ++ka) v[(10 * ka + 6 * kb) % 15] = u[ka];
  }
}

// In-place FFT of one ring of N = 15 * 32 K points in shared memory (padded
// slots pad_idx, natural order in and out), by a CTA of >= 256 threads:
// N = N1 x 15 with N1 = 32 K, n = n1 + N1 n2, k = k2 + 15 k1.
//   A. thread n1: 15-point DFT over n2 in registers, twiddle W_N^(n1 k2),
//      written back to the same slots (no barrier between read and write);
//   B. warp: column k2 (contiguous N1 points) through the register FFT
//      ring_fft<K> on the N-point table at stride 15, results scattered to
//      k2 + 15 k1 once every column has been read.
// Three CTA barriers instead of one per radix stage, and no digit reversal.
template <int K, bool INV>
__device__ void ring_fft15(double2* ring, const double2* tw) {
  constexpr int N1 = 32 * K;
  const int nthr = blockDim.x;
  for (int n1 = threadIdx.x; n1 < N1; n1 += nthr) {
    double2 v[15];
#pragma unroll
    for (int n2 = 0; n2 < 15; ++n2) v[n2] = ring[pad_idx(n1 + N1 * n2)];
    dft15<INV>(v);
#pragma unroll
    for (int k2 = 1; k2 < 15; ++k2)
      if (n1 != 0) v[k2] = cmul(v[k2], tw_at(tw, n1 * k2, INV));
#pragma unroll
    for (int k2 = 0; k2 < 15; ++k2) ring[pad_idx(n1 + N1 * k2)] = v[k2];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = nthr >> 5;
  double2 c[2][K];   // nw >= 8: at most two of the 15 columns per warp
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int k2 = warp + i * nw;
    if (k2 < 15) {
#pragma unroll
      for (int k = 0; k < K; ++k) c[i][k] = ring[pad_idx(N1 * k2 + 32 * k + lane)];
    }
  }
  __syncthreads();
  double2 wst[3];
  cross_twiddles<K, INV>(wst, tw, lane, 15);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int k2 = warp + i * nw;
    if (k2 < 15) {
      ring_fft<K, INV>(c[i], tw, lane, wst, 15);
#pragma unroll
      for (int m1 = 0; m1 < K; ++m1) ring[pad_idx(k2 + 15 * ring_out_index<K>(lane, m1))] = c[i][m1];
    }
  }
  __syncthreads();
}

// Ring length with a ring_fft15 path: N = 15 * 32 K, K a power of two <= 16.
__host__ __device__ constexpr int fft15_k(int n) {
  return (n % 480 == 0 && (n / 480 == 1 || n / 480 == 2 || n / 480 == 4 || n / 480 == 8 ||
                           n / 480 == 16)) ? n / 480 : 0;
}

// Output index held by (lane, slot q) after ring_fft.  Odd K: m1 = q and the
// radix-2 DIF leaves m2 = brev5(lane).  Half exchange: each stage swapped its lane
// bit with the register-half bit t = q >= K/2, so with b = brev5(lane) the column is
// m1 = (b & 1) K/2 + (q mod K/2) and m2 = (b >> 1) + 16 t.
template <int K>
__device__ __forceinline__ int ring_out_index(int lane, int q) {
  const int b = (int)(__brev((unsigned)lane) >> 27);
  if constexpr (half_exchange<K>()) {
    constexpr int H = K / 2;
    const int t = q >= H ? 1 : 0;
    return (b & 1) * H + (q - t * H) + K * ((b >> 1) + 16 * t);
  } else {
    return q + K * b;
  }
}

// Transform the warp's ring held in v (lane l: points 32 k + l) and store the
// spectrum to ring in natural order (padded slots).  ring may be the buffer v
// was loaded from.  (A quad-split variant -- the 32-point cross-lane DFT as a
// transpose through the ring, in-lane 8-point DFTs and two shuffle stages --
// won in the fused F_E kernel at K = 24 against full-exchange shuffle stages and
// lost to the half exchange: profiles/r01 and r02 experiments.md.)
template <int K, bool INV, bool TWC = false>
__device__ __forceinline__ void ring_fft_to(double2 (&v)[K], const double2* tw, int lane,
                                            const double2 (&wst)[3], double2* ring) {
  ring_fft<K, INV, TWC>(v, tw, lane, wst);
  __syncwarp();
#pragma unroll
  for (int m1 = 0; m1 < K; ++m1) ring[pad_idx(ring_out_index<K>(lane, m1))] = v[m1];
}

}  // namespace swfft
