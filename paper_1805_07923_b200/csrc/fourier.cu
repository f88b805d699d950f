// Longitude (zonal Fourier) stage on B200, fp64, plus the fused grid-space
// nonlinear terms of the shallow-water explicit tendency.
//
// Reference counterparts:
//   _grid_to_fourier  rfft(field, axis=0)[:R+1] / n_lon          (spharm.py:210-217)
//   _fourier_to_grid  irfft(pad(F) * n_lon, n=n_lon, axis=0)      (spharm.py:219-222)
//   grid products of ShallowWaterRHS.eval_f_e                     (swe.py:258-274)
//
// A latitude pair (north jn, mirror js) is one complex ring z = g_n + i g_s of
// n_lon points in shared memory; one in-place complex FFT (fft_core.cuh)
// transforms both latitudes.  The Legendre side hands over even/odd partial
// sums (E, O) so the pair's spectra are F_n = E + O, F_s = E - O; the
// analysis side receives S = v_n + v_s and D = v_n - v_s of each weighted
// Fourier vector v.  As in the reference's irfft, the imaginary part of the
// r = 0 coefficient is ignored on synthesis.
//
// In the fused SWE kernel the grids never leave shared memory: 5 inverse FFTs
// (U/a, V/a, zeta, delta, phi'), pointwise products, 7 forward FFTs, and the
// Fourier-space weights (w, w/(1-mu^2), i r, 1/a) of the div/curl/analysis
// contractions (spharm.py:201-205, 281-300) are applied before the result is
// written for the Legendre analysis.
//
// Rings are padded (fft_core.cuh) with a ring stride == 1 (mod 8) double2, so
// both the butterflies and the cross-ring grid transposes are bank-conflict
// free.  Pairs per CTA (np) is a power of two.
#include <algorithm>
#include <type_traits>

#include <cooperative_groups.h>

#include "common.cuh"
#include "fourier.cuh"
#include "reg_fft.cuh"

namespace swsdc {
namespace cg = cooperative_groups;
#ifdef GRID_TRACE
// debug build only (tools/grid_trace.py): per-CTA %globaltimer stamps of the
// fused F_E grid kernel's phases, read back with swsdc_debug_grid_trace
__device__ unsigned long long g_grid_trace[16384][8];
__device__ __forceinline__ unsigned long long gtime_g() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GRID_STAMP(k) do { if (threadIdx.x == 0) { const int cid_ = blockIdx.y * gridDim.x + blockIdx.x; if (cid_ < 16384) g_grid_trace[cid_][k] = gtime_g(); } } while (0)
#else
#define GRID_STAMP(k) do {} while (0)
#endif
namespace {

constexpr int kSweMaxPts = 4;   // grid points per thread in the fused SWE kernel

template <bool BIGP, bool CONJ>
__device__ __forceinline__ void fft_stage_all(double2* rings, int nrings, const PlanDev& P, int s) {
  const swfft::FftPlan& fp = P.fft;
  const int r = fp.radix[s];
  const int nb = fp.n / r;
  const int total = nrings * nb;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int q = (nb == 1) ? t : (int)swfft::udiv((uint32_t)t, fp.bmag[s]);
    const int b = t - q * nb;
    swfft::stage_butterfly<BIGP, true, CONJ>(rings + (size_t)q * P.ring_stride, fp, s, b, P.tw);
  }
}

// Both directions are decimation in time: input in digit-reversed slots
// (P.rev), output in natural order.  Caller synchronises before.
// Forward: exp(-2 pi i k n / I).
template <bool BIGP>
__device__ void fft_forward(double2* rings, int nrings, const PlanDev& P) {
  for (int s = P.fft.nstage - 1; s >= 0; --s) {
    fft_stage_all<BIGP, false>(rings, nrings, P, s);
    __syncthreads();
  }
}
// Inverse (unnormalised): exp(+2 pi i k n / I).
template <bool BIGP>
__device__ void fft_inverse(double2* rings, int nrings, const PlanDev& P) {
  for (int s = P.fft.nstage - 1; s >= 0; --s) {
    fft_stage_all<BIGP, true>(rings, nrings, P, s);
    __syncthreads();
  }
}

__device__ __forceinline__ double2 d2(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return d2(a.x * s, a.y * s); }
// i r s * a
__device__ __forceinline__ double2 ir_scale(double2 a, double rs) { return d2(-a.y * rs, a.x * rs); }
__device__ __forceinline__ double2 cadd2(double2 a, double2 b) { return d2(a.x + b.x, a.y + b.y); }

// 32-byte global accesses (sm_100 LDG / STG .256): one sector, one LSU data-pipe
// wavefront, where two 16-byte accesses of the same sector cost two.
__device__ __forceinline__ void ld_global_256(const double2* p, double2& a, double2& b) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(p));
}
__device__ __forceinline__ void st_global_256(double* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y) : "memory");
}

// Packed ring values at +r and -r from a pair's (E, O) partial sums.
__device__ __forceinline__ void pair_spectrum(double2 E, double2 O, int r, double2& zp,
                                              double2& zm) {
  const double2 Fn = d2(E.x + O.x, E.y + O.y), Fs = d2(E.x - O.x, E.y - O.y);
  if (r == 0) {
    zp = d2(Fn.x, Fs.x);  // irfft drops Im of the DC bin
    zm = zp;
  } else {
    zp = d2(Fn.x - Fs.y, Fn.y + Fs.x);   // F_n + i F_s
    zm = d2(Fn.x + Fs.y, Fs.x - Fn.y);   // conj(F_n) + i conj(F_s)
  }
}

// Fill nr rings (ring q of CTA-local pair i at rings[(q*np + i) * RS]) from
// (E, O) rows eo[q][r][jh0 + i]; every slot is written (zeros off-band).
// Loads are issued kU at a time before use so each thread keeps several
// global reads in flight.
// One pair (np = 1, natural order), NR rings: thread t takes the rows
// r = t, t + nt, ... of every field -- no index division -- with all its
// loads in flight before the spectra are formed.
template <int NR>
__device__ __forceinline__ void fill_rings_pair(double2* rings, const PlanDev& P, const double2* eo,
                                                size_t fstride) {
  const int R = P.R, I = P.I, RS = P.ring_stride, nt = blockDim.x;
  for (int r0 = threadIdx.x; r0 <= R; r0 += 2 * nt) {
    double2 E[2][NR], O[2][NR];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = r0 + h * nt;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        E[h][q] = O[h][q] = d2(0.0, 0.0);
        if (r <= R) {
          ld_global_256(eo + q * fstride + (size_t)r * P.Jh * 2, E[h][q], O[h][q]);
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = r0 + h * nt;
      if (r <= R) {
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          double2 zp, zm;
          pair_spectrum(E[h][q], O[h][q], r, zp, zm);
          double2* ring = rings + (size_t)q * RS;
          ring[swfft::pad_idx(r)] = zp;
          if (r != 0) ring[swfft::pad_idx(I - r)] = zm;
        }
      }
    }
  }
  for (int k = R + 1 + threadIdx.x; k < I - R; k += nt)
#pragma unroll
    for (int q = 0; q < NR; ++q) rings[(size_t)q * RS + swfft::pad_idx(k)] = d2(0.0, 0.0);
}

__device__ __forceinline__ void fill_rings(double2* rings, const PlanDev& P, const double2* eo,
                                           size_t fstride, int nr, int np, int lnp, int jh0,
                                           bool natural = false) {
  constexpr int kU = 8;
  const int R = P.R, I = P.I, RS = P.ring_stride;
  const int nband = (nr * (R + 1)) << lnp;
  const int nmid = I - 2 * R - 1;
  const int nzero = (nr * nmid) << lnp;
  const int nt = blockDim.x;
  for (int base = threadIdx.x; base < nband; base += kU * nt) {
    double2 E[kU], O[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = base + u * nt;
      E[u] = O[u] = d2(0.0, 0.0);
      if (idx < nband) {
        const int i = idx & (np - 1), qr = idx >> lnp;
        const int q = qr / (R + 1), r = qr - q * (R + 1);
        if (jh0 + i < P.Jh) {
          ld_global_256(eo + q * fstride + ((size_t)r * P.Jh + jh0 + i) * 2, E[u], O[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = base + u * nt;
      if (idx < nband) {
        const int i = idx & (np - 1), qr = idx >> lnp;
        const int q = qr / (R + 1), r = qr - q * (R + 1);
        double2 zp, zm;
        pair_spectrum(E[u], O[u], r, zp, zm);
        double2* ring = rings + (size_t)(q * np + i) * RS;
        ring[natural ? swfft::pad_idx(r) : P.rev[r]] = zp;
        if (r != 0) ring[natural ? swfft::pad_idx(I - r) : P.rev[I - r]] = zm;
      }
    }
  }
  for (int z = threadIdx.x; z < nzero; z += nt) {
    const int i = z & (np - 1);
    const int qk = z >> lnp;
    const int q = qk / nmid, k = R + 1 + (qk - q * nmid);
    rings[(size_t)(q * np + i) * RS + (natural ? swfft::pad_idx(k) : P.rev[k])] = d2(0.0, 0.0);
  }
}

// Unpack F_n, F_s (already divided by n_lon) at wavenumber r from a forward-
// transformed packed ring (natural order).
__device__ __forceinline__ void get_pair(const double2* ring, const PlanDev& P, int r, double2& Fn,
                                         double2& Fs) {
  const double2 zk = ring[swfft::pad_idx(r)];
  const double2 zm = ring[swfft::pad_idx(r == 0 ? 0 : P.I - r)];
  const double h = 0.5 / P.I;
  Fn = d2((zk.x + zm.x) * h, (zk.y - zm.y) * h);
  Fs = d2((zk.y + zm.y) * h, (zm.x - zk.x) * h);
}

// Write analysis vector v at (r, jh): S = v_n + v_s, D = v_n - v_s (equator:
// S = v_n, D = 0) into the fragment-native layout (common.cuh XLayout).
__device__ __forceinline__ void put_x(double* x, const XLayout& L, int v, int r, int jh,
                                      double2 vn, double2 vs, bool equator) {
  double2 S, D;
  if (equator) {
    S = vn;
    D = d2(0.0, 0.0);
  } else {
    S = d2(vn.x + vs.x, vn.y + vs.y);
    D = d2(vn.x - vs.x, vn.y - vs.y);
  }
  if (L.pm) {   // re / im columns adjacent: one 16-byte store per parity
    *reinterpret_cast<double2*>(x + L.idx(v, 0, r, jh, 0)) = S;
    *reinterpret_cast<double2*>(x + L.idx(v, 0, r, jh, 1)) = D;
    return;
  }
  x[L.idx(v, 0, r, jh, 0)] = S.x;
  x[L.idx(v, 1, r, jh, 0)] = S.y;
  x[L.idx(v, 0, r, jh, 1)] = D.x;
  x[L.idx(v, 1, r, jh, 1)] = D.y;
}

// ---------------------------------------------------------------------------
// (E, O) -> grid, np pairs per CTA.  grid: [f][I][J]
// ---------------------------------------------------------------------------
// RINGS: write each pair's ring (north, south) contiguously, rings_out[f][jh][il]
// (double2, grid_fstride in double2), the layout swe_prod_kernel reads coalesced.
// K15 > 0: n_lon = 15 * 32 K15, one pair per CTA, 256 threads: the ring is
// filled in natural order and transformed by swfft::ring_fft15 (reg_fft.cuh).
template <bool BIGP, bool RINGS = false, int K15 = 0>
__global__ void __launch_bounds__(256, 2) f2g_kernel(PlanDev P, const double2* eo, long long eo_fstride, double* grid,
                           long long grid_fstride, int lnp, int jh_begin, int jh_end) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double2 rings[];
  const int np = 1 << lnp;
  const int f = blockIdx.y;
  const int jh0 = jh_begin + blockIdx.x * np;
  PlanDev Q = P;
  Q.Jh = jh_end;  // pairs >= jh_end are not this launch's (fill_rings bounds on Q.Jh)
  fill_rings(rings, Q, eo + (size_t)f * eo_fstride, 0, 1, np, lnp, jh0, K15 > 0);
  __syncthreads();
  if constexpr (K15 > 0) swfft::ring_fft15<K15, true>(rings, P.tw);
  else fft_inverse<BIGP>(rings, np, P);
  if (RINGS) {
    double2* out = reinterpret_cast<double2*>(grid) + (size_t)f * grid_fstride;
    for (int i = 0; i < np && jh0 + i < jh_end; ++i) {
      const double2* ring = rings + (size_t)i * P.ring_stride;
      double2* dst = out + (size_t)(jh0 + i) * P.I;
      for (int il = threadIdx.x; il < P.I; il += blockDim.x) dst[il] = ring[swfft::pad_idx(il)];
    }
    return;
  }
  double* g = grid + (size_t)f * grid_fstride;
  for (int idx = threadIdx.x; idx < (P.I << lnp); idx += blockDim.x) {
    const int il = idx >> lnp, i = idx & (np - 1);
    const int jh = jh0 + i;
    if (jh >= jh_end) continue;
    const double2 z = rings[(size_t)i * P.ring_stride + swfft::pad_idx(il)];
    const int jn = jn_of(P, jh), js = js_of(P, jh);
    g[(size_t)il * P.J + jn] = z.x;
    if (js != jn) g[(size_t)il * P.J + js] = z.y;
  }
}

// ---------------------------------------------------------------------------
// grid -> weighted (S, D) vectors.  MODE 0: plain analysis (1 field -> 1
// vector, weight w).  MODE 1: div/curl (fields U, V -> 4 vectors
// [P-div, H-div, P-curl, H-curl], weight w / (1 - mu^2)).
// ---------------------------------------------------------------------------
template <int MODE, bool BIGP, int K15 = 0>
__global__ void __launch_bounds__(256, 2) g2f_kernel(PlanDev P, const double* grid, const double* grid2,
                           long long grid_fstride, double* x, XLayout xl, int lnp) {
  pdl_wait();
  pdl_trigger();
  constexpr int NIN = (MODE == 0) ? 1 : 2;
  extern __shared__ __align__(16) double2 rings[];  // [NIN][np][RS]
  const int np = 1 << lnp;
  const int f = blockIdx.y;
  const int jh0 = blockIdx.x * np;
  const double* gin[2] = {grid + (size_t)f * grid_fstride,
                          (MODE == 0 ? grid : grid2) + (size_t)f * grid_fstride};
  {
    constexpr int kU = 4;
    const int ntot = NIN * (P.I << lnp), nt = blockDim.x;
    for (int base = threadIdx.x; base < ntot; base += kU * nt) {
      double2 z[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int idx = base + u * nt;
        z[u] = d2(0.0, 0.0);
        if (idx < ntot) {
          const int q = (NIN == 1) ? 0 : idx / (P.I << lnp);
          const int rem = idx - q * (P.I << lnp);
          const int il = rem >> lnp, i = rem & (np - 1);
          const int jh = jh0 + i;
          if (jh < P.Jh) {
            const double* gq = gin[q] + (size_t)il * P.J;
            z[u] = d2(gq[jn_of(P, jh)], gq[js_of(P, jh)]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int idx = base + u * nt;
        if (idx < ntot) {
          const int q = (NIN == 1) ? 0 : idx / (P.I << lnp);
          const int rem = idx - q * (P.I << lnp);
          const int il = rem >> lnp, i = rem & (np - 1);
          rings[(size_t)(q * np + i) * P.ring_stride + (K15 > 0 ? swfft::pad_idx(il) : P.rev[il])] = z[u];
        }
      }
    }
  }
  __syncthreads();
  if constexpr (K15 > 0) {
#pragma unroll 1
    for (int q = 0; q < NIN; ++q) swfft::ring_fft15<K15, false>(rings + (size_t)q * P.ring_stride, P.tw);
  } else {
    fft_forward<BIGP>(rings, NIN * np, P);
  }
  // mode 0: field f is vector f of one member; mode 1: pair f is member f (4 vectors)
  double* xf = x + (MODE == 0 ? 0 : (size_t)f * xl.mstride);
  for (int idx = threadIdx.x; idx < ((P.R + 1) << lnp); idx += blockDim.x) {
    const int r = idx >> lnp, i = idx & (np - 1);
    const int jh = jh0 + i;
    if (jh >= P.Jh) continue;
    const bool eq = (jn_of(P, jh) == js_of(P, jh));
    const double mu = P.mu_n[jh], w = P.w_n[jh];
    if (MODE == 0) {
      double2 Fn, Fs;
      get_pair(rings + (size_t)i * P.ring_stride, P, r, Fn, Fs);
      put_x(xf, xl, f, r, jh, cscale(Fn, w), cscale(Fs, w), eq);
    } else {
      double2 Un, Us, Vn, Vs;
      get_pair(rings + (size_t)i * P.ring_stride, P, r, Un, Us);
      get_pair(rings + (size_t)(np + i) * P.ring_stride, P, r, Vn, Vs);
      const double wc = w / (1.0 - mu * mu);
      const double rw = r * wc;
      // div = Pwc2 (i r F_U) - Hwc2 F_V ; curl = Pwc2 (i r F_V) + Hwc2 F_U  (spharm.py:294-299)
      put_x(xf, xl, 0, r, jh, ir_scale(Un, rw), ir_scale(Us, rw), eq);
      put_x(xf, xl, 1, r, jh, cscale(Vn, -wc), cscale(Vs, -wc), eq);
      put_x(xf, xl, 2, r, jh, ir_scale(Vn, rw), ir_scale(Vs, rw), eq);
      put_x(xf, xl, 3, r, jh, cscale(Un, wc), cscale(Us, wc), eq);
    }
  }
}

// ---------------------------------------------------------------------------
// Register-FFT variants (n_lon = 32 K, reg_fft.cuh): warp w of the CTA owns
// ring w.  Shared memory only carries the coalesced grid loads/stores and the
// analysis-layout writes (rings in natural order, padded); the transforms run
// in registers with no CTA barriers between stages.
// ---------------------------------------------------------------------------
// Warp index as a value the compiler knows to be warp-uniform: code under
// `if (warp < n)` then keeps plain shuffles (no divergence check with an
// out-of-line WARPSYNC.COLLECTIVE path per shuffle).
__device__ __forceinline__ int uniform_warp() {
  return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// E/O staging row stride (double2) for np pairs: 2 np + 1 keeps the lanes'
// reads of consecutive wavenumbers in distinct bank groups.
__host__ __device__ inline int eo_row(int np) { return 2 * np + 1; }
// f2g_reg_kernel: double2 slots of the staging / rings region
__host__ __device__ inline size_t f2g_reg_elems(const PlanDev& P, int np) {
  const size_t a = (size_t)np * P.ring_stride, b = (size_t)(P.R + 1) * eo_row(np);
  return a > b ? a : b;
}

// K >= 16: 4 pairs (128 threads) per CTA, registers capped for 3 CTAs/SM;
// smaller rings: up to 8 pairs (256 threads).
#define SWSDC_REG_BOUNDS(K) __launch_bounds__((K) >= 16 ? 128 : 256, (K) >= 16 ? 3 : 2)

// RINGS: instead of the (n_lon, n_lat) grid, write each pair's ring (north,
// south) contiguously: rings_out[f][jh][il] (double2), the internal layout of
// the split F_E path whose consumer then reads whole rings coalesced.
template <int K, bool RINGS = false>
__global__ void SWSDC_REG_BOUNDS(K) f2g_reg_kernel(PlanDev P, const double2* eo,
                                                      long long eo_fstride, double* grid,
                                                      long long grid_fstride, int lnp,
                                                      int jh_begin, int jh_end) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double2 rings[];
  const int np = 1 << lnp;
  const int lane = threadIdx.x & 31, warp = uniform_warp();
  const int f = blockIdx.y;
  const int jh0 = jh_begin + blockIdx.x * np;
  const int R = P.R, I = P.I, row = eo_row(np);
  // 1. stage the CTA's (E, O) rows with async copies: for each r, np pairs x
  //    (E, O) = 32 np contiguous bytes; every copy is in flight at once
  {
    const double2* e = eo + (size_t)f * eo_fstride;
    const int per_r = 2 * np, total = (R + 1) * per_r;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int r = idx >> (lnp + 1), c = idx & (per_r - 1);   // c = 2 i + (E|O)
      const int jh = jh0 + (c >> 1);
      double2* dst = rings + (size_t)r * row + c;
      if (jh < jh_end) cp_async16(dst, e + ((size_t)r * P.Jh + jh) * 2 + (c & 1));
      else *dst = d2(0.0, 0.0);
    }
    cp_async_wait_all();
  }
  __syncthreads();
  // 2. each warp assembles its pair's packed spectrum in registers and transforms it
  //    (the decimation-in-time variant with its gathered input order measured slower
  //    here: 35.2 vs 27.1 us at config 1, profiles/r02/experiments.md)
  const int jhw = jh0 + warp;
  double2 v[K];
  double2 wst[3];
  swfft::cross_twiddles<K, true>(wst, P.tw, lane);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int n = 32 * k + lane;
    const bool lo = n <= R, hi = n >= I - R;
    const int r = lo ? n : I - n;
    v[k] = d2(0.0, 0.0);
    if (lo || hi) {
      const double2* src = rings + (size_t)r * row + 2 * warp;
      double2 zp, zm;
      pair_spectrum(src[0], src[1], r, zp, zm);
      v[k] = lo ? zp : zm;
    }
  }
  __syncthreads();   // staging consumed; the rings reuse its space
  if (jhw < jh_end) {
    double2* ring = rings + (size_t)warp * P.ring_stride;
    swfft::ring_fft_to<K, true>(v, P.tw, lane, wst, ring);
    if (RINGS) {
      __syncwarp();
      double2* dst = reinterpret_cast<double2*>(grid) + (size_t)f * grid_fstride + (size_t)jhw * P.I;
      for (int il = lane; il < P.I; il += 32) dst[il] = ring[swfft::pad_idx(il)];
    }
  }
  if (RINGS) return;
  __syncthreads();
  {
    // thread -> fixed pair i, longitudes il0, il0 + step, ...: np consecutive
    // threads write np consecutive latitudes of one longitude row
    const int i = threadIdx.x & (np - 1), step = blockDim.x >> lnp;
    const int jh = jh0 + i;
    if (jh < jh_end) {
      const int jn = jn_of(P, jh), js = js_of(P, jh);
      double* gn = grid + (size_t)f * grid_fstride + jn;
      const long long dj = (long long)(js - jn);
      const double2* ring = rings + (size_t)i * P.ring_stride;
      for (int il = threadIdx.x >> lnp; il < P.I; il += step) {
        const double2 z = ring[swfft::pad_idx(il)];
        double* gp = gn + (size_t)il * P.J;
        gp[0] = z.x;
        if (dj != 0) gp[dj] = z.y;
      }
    }
  }
}

template <int K, int MODE>
__global__ void SWSDC_REG_BOUNDS(K) g2f_reg_kernel(PlanDev P, const double* grid,
                                                      const double* grid2, long long grid_fstride,
                                                      double* x, XLayout xl, int lnp) {
  pdl_wait();
  pdl_trigger();
  constexpr int NIN = (MODE == 0) ? 1 : 2;
  extern __shared__ __align__(16) double2 rings[];  // [NIN][np][RS], natural order
  const int np = 1 << lnp;
  const int lane = threadIdx.x & 31, warp = uniform_warp();
  const int f = blockIdx.y;
  const int jh0 = blockIdx.x * np;
  const double* gin[2] = {grid + (size_t)f * grid_fstride,
                          (MODE == 0 ? grid : grid2) + (size_t)f * grid_fstride};
  {
    // async 8-byte copies straight into the natural-order rings: thread ->
    // fixed (ring q, pair i, side) slot, strided over longitudes; 2 np
    // consecutive threads read 2 x np consecutive latitudes of one row
    const int nslot = 2 * np * NIN, slot = threadIdx.x % nslot, step = blockDim.x / nslot;
    const int q = slot / (2 * np), c = slot - q * 2 * np, i = c >> 1, side = c & 1;
    const int jh = jh0 + i;
    double* dst0 = reinterpret_cast<double*>(rings + (size_t)(q * np + i) * P.ring_stride) + side;
    if (jh < P.Jh) {
      const double* src0 = gin[q] + (side ? js_of(P, jh) : jn_of(P, jh));
      for (int il = threadIdx.x / nslot; il < P.I; il += step)
        cp_async8(dst0 + 2 * swfft::pad_idx(il), src0 + (size_t)il * P.J);
    } else {
      for (int il = threadIdx.x / nslot; il < P.I; il += step) dst0[2 * swfft::pad_idx(il)] = 0.0;
    }
    cp_async_wait_all();
  }
  __syncthreads();
  {
    // warp w transforms ring w (q = w / np, pair w % np)
    double2 wst[3];
    swfft::cross_twiddles<K, false>(wst, P.tw, lane);
    double2* ring = rings + (size_t)warp * P.ring_stride;
    double2 v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = ring[swfft::pad_idx(32 * k + lane)];
    swfft::ring_fft_to<K, false>(v, P.tw, lane, wst, ring);
  }
  __syncthreads();
  double* xf = x + (MODE == 0 ? 0 : (size_t)f * xl.mstride);
  {
    // thread -> fixed pair i, wavenumbers r0, r0 + step, ...: np consecutive
    // threads write np consecutive latitudes of one (vector, r) x row
    const int i = threadIdx.x & (np - 1), step = blockDim.x >> lnp;
    const int jh = jh0 + i;
    if (jh < P.Jh) {
      const bool eq = (jn_of(P, jh) == js_of(P, jh));
      const double mu = P.mu_n[jh], w = P.w_n[jh];
      const double wc = w / (1.0 - mu * mu);
      for (int r = threadIdx.x >> lnp; r <= P.R; r += step) {
        if (MODE == 0) {
          double2 Fn, Fs;
          get_pair(rings + (size_t)i * P.ring_stride, P, r, Fn, Fs);
          put_x(xf, xl, f, r, jh, cscale(Fn, w), cscale(Fs, w), eq);
        } else {
          double2 Un, Us, Vn, Vs;
          get_pair(rings + (size_t)i * P.ring_stride, P, r, Un, Us);
          get_pair(rings + (size_t)(np + i) * P.ring_stride, P, r, Vn, Vs);
          const double rw = r * wc;
          // div = Pwc2 (i r F_U) - Hwc2 F_V ; curl = Pwc2 (i r F_V) + Hwc2 F_U  (spharm.py:294-299)
          put_x(xf, xl, 0, r, jh, ir_scale(Un, rw), ir_scale(Us, rw), eq);
          put_x(xf, xl, 1, r, jh, cscale(Vn, -wc), cscale(Vs, -wc), eq);
          put_x(xf, xl, 2, r, jh, ir_scale(Vn, rw), ir_scale(Vs, rw), eq);
          put_x(xf, xl, 3, r, jh, cscale(Un, wc), cscale(Us, wc), eq);
        }
      }
    }
  }
}

// Output stage shared by the fused SWE kernels: weighted analysis vectors at
// wavenumber r of latitude pair jh from its 7 (or 2) forward-transformed
// product rings (natural order) into x.
template <bool NONLIN>
__device__ __forceinline__ void swe_out_one(const double2* rings, const PlanDev& P, double* xm,
                                            const XLayout& xl, int r, int jh, double w, double wc,
                                            double ia, bool eq) {
  const int RS = P.ring_stride;
  double2 A1n, A1s, A2n, A2s;
  get_pair(rings, P, r, A1n, A1s);
  get_pair(rings + RS, P, r, A2n, A2s);
  if (!NONLIN) {
    put_x(xm, xl, 0, r, jh, cscale(A1n, w), cscale(A1s, w), eq);
    put_x(xm, xl, 1, r, jh, cscale(A2n, w), cscale(A2s, w), eq);
  } else {
    double2 PUn, PUs, PVn, PVs, ZUn, ZUs, ZVn, ZVs, Kn, Ks;
    get_pair(rings + 2 * RS, P, r, PUn, PUs);
    get_pair(rings + 3 * RS, P, r, PVn, PVs);
    get_pair(rings + 4 * RS, P, r, ZUn, ZUs);
    get_pair(rings + 5 * RS, P, r, ZVn, ZVs);
    get_pair(rings + 6 * RS, P, r, Kn, Ks);
    const double rwa = r * wc * ia, wa = wc * ia;
    // P-vectors: phi, zeta, delta, ke ; H-vectors: phi, zeta, delta
    put_x(xm, xl, 0, r, jh, ir_scale(PUn, -rwa), ir_scale(PUs, -rwa), eq);
    put_x(xm, xl, 1, r, jh, cadd2(cscale(A1n, w), ir_scale(ZUn, -rwa)),
          cadd2(cscale(A1s, w), ir_scale(ZUs, -rwa)), eq);
    put_x(xm, xl, 2, r, jh, cadd2(cscale(A2n, w), ir_scale(ZVn, rwa)),
          cadd2(cscale(A2s, w), ir_scale(ZVs, rwa)), eq);
    put_x(xm, xl, 3, r, jh, cscale(Kn, w), cscale(Ks, w), eq);
    put_x(xm, xl, 4, r, jh, cscale(PVn, wa), cscale(PVs, wa), eq);
    put_x(xm, xl, 5, r, jh, cscale(ZVn, wa), cscale(ZVs, wa), eq);
    put_x(xm, xl, 6, r, jh, cscale(ZUn, wa), cscale(ZUs, wa), eq);
  }
}

template <bool NONLIN>
__device__ __forceinline__ void swe_grid_output(const double2* rings, const PlanDev& P, double* xm,
                                                const XLayout& xl, int jh, double w, double wc,
                                                double ia) {
  const bool eq = (jn_of(P, jh) == js_of(P, jh));
  for (int r = threadIdx.x; r <= P.R; r += blockDim.x)
    swe_out_one<NONLIN>(rings, P, xm, xl, r, jh, w, wc, ia, eq);
}

// Fused SWE grid stage with register FFTs (n_lon = 32 K), one latitude pair per
// CTA.  Rings stay in natural order, so the pointwise products are computed in
// place (each thread reads and rewrites its own grid points: no barrier, no
// register staging), and warp w transforms rings w, w + nwarps, ...
// K >= 16: 6 warps (5 inverse FFTs in one round) at <= 170 registers so two
// CTAs share an SM; smaller rings: 8 warps.
//
// CL: the CTA is one of a cluster of 4 covering one 4-latitude block of x.
// After the forward FFTs the cluster synchronises and CTA c computes the
// vectors of wavenumbers [c (R+1)/4, (c+1)(R+1)/4) for all 4 latitude pairs,
// reading the other CTAs' spectra through distributed shared memory, so 4
// consecutive threads write each 32-byte x sector whole (one pair per CTA
// would write 8-byte quarters of it); a second cluster barrier keeps every
// CTA's rings alive until the others have read them.
template <int K, bool NONLIN, bool CL = false>
__global__ void __launch_bounds__((K) >= 20 ? 192 : (K) == 16 ? 224 : 256, 2) swe_grid_reg_kernel(PlanDev P, const double2* eo,
                                                        long long eo_mstride, double* x,
                                                        XLayout xl, double omega, double radius,
                                                        int jh_begin) {
  pdl_wait();
  pdl_trigger();
  constexpr int NIN = NONLIN ? 5 : 4;
  constexpr int NPROD = NONLIN ? 7 : 2;
  extern __shared__ __align__(16) double2 rings[];  // [7 or 4][RS]
  const int jh = jh_begin + blockIdx.x;
  const int m = blockIdx.y;
  const int RS = P.ring_stride;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const size_t fstride = (size_t)(P.R + 1) * P.Jh * 2;
  GRID_STAMP(0);
  fill_rings_pair<NIN>(rings, P, eo + (size_t)m * eo_mstride + (size_t)jh * 2, fstride);
  __syncthreads();
  GRID_STAMP(1);
  {
    double2 wst[3];
    swfft::cross_twiddles<K, true>(wst, P.tw, lane);
    for (int q = warp; q < NIN; q += nwarp) {
      double2* ring = rings + (size_t)q * RS;
      double2 v[K];
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = ring[swfft::pad_idx(32 * k + lane)];
      swfft::ring_fft_to<K, true>(v, P.tw, lane, wst, ring);
    }
  }
  __syncthreads();
  GRID_STAMP(2);
  const double mu = P.mu_n[jh];
  const double fn = 2.0 * omega * mu;         // f = 2 Omega mu (swe.py:178); south: -fn
  const double c2o = 2.0 * omega / radius;    // swe.py:179
  const double ic2 = 1.0 / (1.0 - mu * mu);   // swe.py:180
  for (int il = threadIdx.x; il < P.I; il += blockDim.x) {
    const int p = swfft::pad_idx(il);
    const double2 U = rings[p], V = rings[RS + p], Z = rings[2 * RS + p], D = rings[3 * RS + p];
    // swe.py:262,265 : tend_zeta grid = -f delta - (2 Omega/a) V ; tend_delta grid = f zeta - (2 Omega/a) U
    rings[p] = d2(-fn * D.x - c2o * V.x, fn * D.y - c2o * V.y);
    rings[RS + p] = d2(fn * Z.x - c2o * U.x, -fn * Z.y - c2o * U.y);
    if (NONLIN) {
      const double2 Ph = rings[(NIN - 1) * RS + p];
      // swe.py:271-273 : Phi U, Phi V, zeta U, zeta V, KE = (U^2 + V^2) / (2 (1 - mu^2))
      rings[2 * RS + p] = d2(Ph.x * U.x, Ph.y * U.y);
      rings[3 * RS + p] = d2(Ph.x * V.x, Ph.y * V.y);
      rings[4 * RS + p] = d2(Z.x * U.x, Z.y * U.y);
      rings[5 * RS + p] = d2(Z.x * V.x, Z.y * V.y);
      rings[6 * RS + p] = d2(0.5 * (U.x * U.x + V.x * V.x) * ic2, 0.5 * (U.y * U.y + V.y * V.y) * ic2);
    }
  }
  __syncthreads();
  GRID_STAMP(3);
  {
    double2 wst[3];
    swfft::cross_twiddles<K, false>(wst, P.tw, lane);
    for (int q = warp; q < NPROD; q += nwarp) {
      double2* ring = rings + (size_t)q * RS;
      double2 v[K];
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = ring[swfft::pad_idx(32 * k + lane)];
      swfft::ring_fft_to<K, false>(v, P.tw, lane, wst, ring);
    }
  }
  __syncthreads();
  GRID_STAMP(4);
  if constexpr (!CL) {
    const double w = P.w_n[jh];
    swe_grid_output<NONLIN>(rings, P, x + (size_t)m * xl.mstride, xl, jh, w, w * ic2, 1.0 / radius);
  } else {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    GRID_STAMP(5);
    const int c = (int)cl.block_rank();
    const int jb0 = jh - c;                  // first latitude pair of this cluster's block
    const int nr = P.R + 1, r_lo = c * nr / 4, r_hi = (c + 1) * nr / 4;
    double* xm = x + (size_t)m * xl.mstride;
    const double ia = 1.0 / radius;
    for (int idx = threadIdx.x; idx < (r_hi - r_lo) * 4; idx += blockDim.x) {
      const int i = idx & 3, r = r_lo + (idx >> 2);
      const int jhi = jb0 + i;
      const double mui = P.mu_n[jhi], wi = P.w_n[jhi];
      const double2* ri = cl.map_shared_rank(rings, i);
      swe_out_one<NONLIN>(ri, P, xm, xl, r, jhi, wi, wi / (1.0 - mui * mui), ia,
                          jn_of(P, jhi) == js_of(P, jhi));
    }
    GRID_STAMP(6);
    // only the remote shared-memory reads above must be complete before a CTA
    // may exit, and they are (their values were consumed): a relaxed arrive
    // does not wait for this CTA's outstanding x stores as cl.sync()'s release would
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    GRID_STAMP(7);
  }
}

// ---------------------------------------------------------------------------
// Fused SWE grid stage, 9 register FFTs per latitude pair (default for the
// nonlinear F_E).  The Coriolis terms of swe.py:262-265,
//   A1 = -f delta - (2 Omega / a) V,   A2 = f zeta - (2 Omega / a) U,
// are linear in the fields with coefficients constant along a latitude, so
// their Fourier coefficients are formed directly from the input spectra
// (kept in shared memory as cf) instead of by a grid round trip: the delta
// grid is never synthesised (4 inverse FFTs: U/a, V/a, zeta, phi') and only
// the 5 true products (phi U, phi V, zeta U, zeta V, KE) are transformed back
// (5 forward FFTs) -- 9 FFTs instead of 12, 5 rings instead of 7, and every
// FFT round keeps 4-5 of the CTA's 5 warps busy.  Mathematically identical
// to the grid round trip (band-limited input, r <= R < n_lon / 2): only the
// rounding differs.
// ---------------------------------------------------------------------------
constexpr int kG5Rings = 5;
constexpr int kG5Threads = 160;

// Fill rings 0..3 with the packed spectra of fields U, V, zeta, phi' (eo
// fields 0, 1, 2, 4) and cf[q][r] = (F_n, F_s) of fields U, V, zeta, delta
// (eo fields 0..3) with Im dropped at r = 0, as the grid round trip would
// (cf[2 q + side][r], so consecutive lanes touch consecutive 16-byte slots).
__device__ __forceinline__ void fill_g5(double2* rings, double2* cf, const PlanDev& P,
                                        const double2* eo, size_t fstride) {
  const int R = P.R, I = P.I, RS = P.ring_stride, nt = blockDim.x;
  for (int r = threadIdx.x; r <= R; r += nt) {
    double2 E[5], O[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      ld_global_256(eo + q * fstride + (size_t)r * P.Jh * 2, E[q], O[q]);
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      if (q < 4) {
        double2 Fn = d2(E[q].x + O[q].x, E[q].y + O[q].y);
        double2 Fs = d2(E[q].x - O[q].x, E[q].y - O[q].y);
        if (r == 0) { Fn.y = 0.0; Fs.y = 0.0; }
        cf[(2 * q) * (R + 1) + r] = Fn;        // [field][north | south][r]: lanes 16 B apart
        cf[(2 * q + 1) * (R + 1) + r] = Fs;
      }
      if (q == 3) continue;            // no delta ring
      const int ring = q == 4 ? 3 : q;
      double2 zp, zm;
      pair_spectrum(E[q], O[q], r, zp, zm);
      double2* rg = rings + (size_t)ring * RS;
      rg[swfft::pad_idx(r)] = zp;
      if (r != 0) rg[swfft::pad_idx(I - r)] = zm;
    }
  }
  for (int k = R + 1 + threadIdx.x; k < I - R; k += nt)
#pragma unroll
    for (int q = 0; q < 4; ++q) rings[(size_t)q * RS + swfft::pad_idx(k)] = d2(0.0, 0.0);
}

// Analysis vectors at (r, jh) from the 5 forward-transformed product rings
// (PU, PV, ZU, ZV, KE) and the input spectra cf (U, V, zeta, delta); same
// vectors and weights as swe_out_one.
__device__ __forceinline__ void swe_out_g5(const double2* rings, const double2* cf,
                                           const PlanDev& P, double* xm, const XLayout& xl, int r,
                                           int jh, double w, double wc, double ia, double fn,
                                           double c2o, bool eq) {
  const int RS = P.ring_stride, R1 = P.R + 1;
  double2 PUn, PUs, PVn, PVs, ZUn, ZUs, ZVn, ZVs, Kn, Ks;
  get_pair(rings, P, r, PUn, PUs);
  get_pair(rings + RS, P, r, PVn, PVs);
  get_pair(rings + 2 * RS, P, r, ZUn, ZUs);
  get_pair(rings + 3 * RS, P, r, ZVn, ZVs);
  get_pair(rings + 4 * RS, P, r, Kn, Ks);
  const double2 Un = cf[r], Us = cf[R1 + r];
  const double2 Vn = cf[2 * R1 + r], Vs = cf[3 * R1 + r];
  const double2 Zn = cf[4 * R1 + r], Zs = cf[5 * R1 + r];
  const double2 Dn = cf[6 * R1 + r], Ds = cf[7 * R1 + r];
  // swe.py:262,265 in Fourier space; f = fn north, -fn south
  const double2 A1n = d2(-fn * Dn.x - c2o * Vn.x, -fn * Dn.y - c2o * Vn.y);
  const double2 A1s = d2(fn * Ds.x - c2o * Vs.x, fn * Ds.y - c2o * Vs.y);
  const double2 A2n = d2(fn * Zn.x - c2o * Un.x, fn * Zn.y - c2o * Un.y);
  const double2 A2s = d2(-fn * Zs.x - c2o * Us.x, -fn * Zs.y - c2o * Us.y);
  const double rwa = r * wc * ia, wa = wc * ia;
  // P-vectors: phi, zeta, delta, ke ; H-vectors: phi, zeta, delta
  const double2 vn[7] = {ir_scale(PUn, -rwa), cadd2(cscale(A1n, w), ir_scale(ZUn, -rwa)),
                         cadd2(cscale(A2n, w), ir_scale(ZVn, rwa)), cscale(Kn, w),
                         cscale(PVn, wa), cscale(ZVn, wa), cscale(ZUn, wa)};
  const double2 vs[7] = {ir_scale(PUs, -rwa), cadd2(cscale(A1s, w), ir_scale(ZUs, -rwa)),
                         cadd2(cscale(A2s, w), ir_scale(ZVs, rwa)), cscale(Ks, w),
                         cscale(PVs, wa), cscale(ZVs, wa), cscale(ZUs, wa)};
  if (xl.pm) {
    // pair-major: the 16 columns of (r, jh, parity) are one 128-byte row -- four
    // 32-byte stores per parity (vector pairs; column 14-15 is padding, zeroed)
    double2 S[8], D[8];
#pragma unroll
    for (int v = 0; v < 7; ++v) {
      S[v] = eq ? vn[v] : d2(vn[v].x + vs[v].x, vn[v].y + vs[v].y);
      D[v] = eq ? d2(0.0, 0.0) : d2(vn[v].x - vs[v].x, vn[v].y - vs[v].y);
    }
    S[7] = d2(0.0, 0.0);
    D[7] = d2(0.0, 0.0);
    double* rs = xm + xl.idx(0, 0, r, jh, 0);
    double* rd = xm + xl.idx(0, 0, r, jh, 1);
#pragma unroll
    for (int v = 0; v < 8; v += 2) {
      st_global_256(rs + 2 * v, S[v], S[v + 1]);
      st_global_256(rd + 2 * v, D[v], D[v + 1]);
    }
    return;
  }
#pragma unroll
  for (int v = 0; v < 7; ++v) put_x(xm, xl, v, r, jh, vn[v], vs[v], eq);
}

template <int K>
__host__ __device__ constexpr int g5_min_blocks() { return K >= 20 ? 2 : K == 16 ? 3 : 4; }

// One latitude pair per CTA of 5 warps; CL as in swe_grid_reg_kernel (4-CTA
// clusters write whole x sectors over DSMEM).  Shared memory: 5 rings, then cf.
template <int K, bool CL>
__global__ void __launch_bounds__(kG5Threads, g5_min_blocks<K>()) swe_grid5_kernel(
    PlanDev P, const double2* eo, long long eo_mstride, double* x, XLayout xl, double omega,
    double radius, int jh_begin) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double2 rings[];   // [5][RS], then cf [4][R+1][2]
  const int jh = jh_begin + blockIdx.x;
  const int m = blockIdx.y;
  const int RS = P.ring_stride;
  double2* cf = rings + (size_t)kG5Rings * RS;
  double2* twc = cf + 8 * (size_t)(P.R + 1);          // twiddle cache (reg_fft.cuh)
  const int lane = threadIdx.x & 31, warp = uniform_warp();
  const size_t fstride = (size_t)(P.R + 1) * P.Jh * 2;
  GRID_STAMP(0);
  swfft::fill_twiddle_cache<K>(twc, P.tw, threadIdx.x, blockDim.x);
  fill_g5(rings, cf, P, eo + (size_t)m * eo_mstride + (size_t)jh * 2, fstride);
  __syncthreads();
  GRID_STAMP(1);
  // Inverse transforms decimate in frequency and leave each grid in the transform's
  // own output order, stored register-major (slot q of lane l at 32 q + l: conflict-
  // free, no padding); the products are pointwise, so they run in that order, and
  // the forward transforms decimate in time from it (ring_fft_dit), ending in natural
  // order for the output stage: no scatter through shared memory in either direction.
  if (warp < 4) {   // U/a, V/a, zeta, phi' to the grid
    double2 wst[3];
    swfft::cross_twiddles<K, true, true>(wst, twc, lane);
    double2* ring = rings + (size_t)warp * RS;
    double2 v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = ring[swfft::pad_idx(32 * k + lane)];
    swfft::ring_fft<K, true, true>(v, twc, lane, wst);
    __syncwarp();
#pragma unroll
    for (int q = 0; q < K; ++q) ring[32 * q + lane] = v[q];
  }
  __syncthreads();
  GRID_STAMP(2);
  const double mu = P.mu_n[jh];
  const double ic2 = 1.0 / (1.0 - mu * mu);   // swe.py:180
  if constexpr (K >= 20) {
    // Products formed in registers on the way into the forward transforms (swe.py:271-273):
    // warp w reads its two factor grids in transform order and multiplies pointwise --
    // Phi U, Phi V, zeta U, zeta V, KE = (U^2 + V^2) / (2 (1 - mu^2)) -- instead of a
    // separate pass that rewrites the rings; every read ends before any ring is rewritten.
    // Measured per ring length: config 2 (K = 24) -1.5%, config 4 (K = 16 / 8) +0.4%, so
    // the shorter rings keep the separate pass below.
    double2 wst[3];
    swfft::cross_twiddles_dit<K, false, true>(wst, twc, lane);
    const int fa = (warp == 4) ? 0 : (warp < 2 ? 3 : 2);       // Phi', Phi', zeta, zeta, U
    const int fb = (warp == 4) ? 1 : (warp & 1);               // U, V, U, V, V
    const double2* ra = rings + (size_t)fa * RS;
    const double2* rb = rings + (size_t)fb * RS;
    double2 v[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const double2 a = ra[32 * q + lane], b = rb[32 * q + lane];
      v[q] = (warp == 4) ? d2(0.5 * (a.x * a.x + b.x * b.x) * ic2, 0.5 * (a.y * a.y + b.y * b.y) * ic2)
                         : d2(a.x * b.x, a.y * b.y);
    }
    __syncthreads();
    GRID_STAMP(3);
    double2* ring = rings + (size_t)warp * RS;
    swfft::ring_fft_dit<K, false, true>(v, twc, lane, wst);
#pragma unroll
    for (int k = 0; k < K; ++k) ring[swfft::pad_idx(32 * k + lane)] = v[k];
  } else {
    for (int p = threadIdx.x; p < P.I; p += blockDim.x) {
      const double2 U = rings[p], V = rings[RS + p], Z = rings[2 * RS + p], Ph = rings[3 * RS + p];
      // swe.py:271-273 : Phi U, Phi V, zeta U, zeta V, KE = (U^2 + V^2) / (2 (1 - mu^2))
      rings[p] = d2(Ph.x * U.x, Ph.y * U.y);
      rings[RS + p] = d2(Ph.x * V.x, Ph.y * V.y);
      rings[2 * RS + p] = d2(Z.x * U.x, Z.y * U.y);
      rings[3 * RS + p] = d2(Z.x * V.x, Z.y * V.y);
      rings[4 * RS + p] = d2(0.5 * (U.x * U.x + V.x * V.x) * ic2, 0.5 * (U.y * U.y + V.y * V.y) * ic2);
    }
    __syncthreads();
    GRID_STAMP(3);
    double2 wst[3];
    swfft::cross_twiddles_dit<K, false, true>(wst, twc, lane);
    double2* ring = rings + (size_t)warp * RS;
    double2 v[K];
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = ring[32 * q + lane];
    swfft::ring_fft_dit<K, false, true>(v, twc, lane, wst);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) ring[swfft::pad_idx(32 * k + lane)] = v[k];
  }
  __syncthreads();
  GRID_STAMP(4);
  const double c2o = 2.0 * omega / radius;    // swe.py:179
  const double ia = 1.0 / radius;
  if constexpr (!CL) {
    const double w = P.w_n[jh];
    const bool eq = (jn_of(P, jh) == js_of(P, jh));
    double* xm = x + (size_t)m * xl.mstride;
    for (int r = threadIdx.x; r <= P.R; r += blockDim.x)
      swe_out_g5(rings, cf, P, xm, xl, r, jh, w, w * ic2, ia, 2.0 * omega * mu, c2o, eq);
    GRID_STAMP(6);
  } else {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    GRID_STAMP(5);
    const int c = (int)cl.block_rank();
    const int jb0 = jh - c;
    const int nr = P.R + 1, r_lo = c * nr / 4, r_hi = (c + 1) * nr / 4;
    double* xm = x + (size_t)m * xl.mstride;
    for (int idx = threadIdx.x; idx < (r_hi - r_lo) * 4; idx += blockDim.x) {
      const int i = idx & 3, r = r_lo + (idx >> 2);
      const int jhi = jb0 + i;
      const double mui = P.mu_n[jhi], wi = P.w_n[jhi];
      const double2* ri = cl.map_shared_rank(rings, i);
      const double2* ci = cl.map_shared_rank(cf, i);
      swe_out_g5(ri, ci, P, xm, xl, r, jhi, wi, wi / (1.0 - mui * mui), ia, 2.0 * omega * mui, c2o,
                 jn_of(P, jhi) == js_of(P, jhi));
    }
    GRID_STAMP(6);
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    GRID_STAMP(7);
  }
}

// Split SWE grid stage, second kernel (register FFTs): the 5 grids come from
// HBM/L2 (written by f2g_reg_kernel); CTA (pair, member, role) stages the grid
// rows it needs with async copies, each warp forms one product ring in
// registers and transforms it, and the CTA writes the analysis vectors of its
// role.  Role 0: A1, ZU, A2, ZV -> vectors 1, 2, 5, 6 (linear: A1, A2 -> 0, 1);
// role 1: PU, PV, KE -> vectors 0, 4, 3.  Twice the CTAs of the fused kernel
// and no inverse FFTs: for batches too small to fill the GPU one pair per CTA.
template <int K, bool NONLIN>
__global__ void __launch_bounds__(128) swe_fwd_reg_kernel(PlanDev P, const double2* gr,
                                                          long long gfield, long long gmember,
                                                          double* x, XLayout xl, double omega,
                                                          double radius, int jh_begin) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double2 rings[];  // [4][RS] product spectra
  const int jh = jh_begin + blockIdx.x, m = blockIdx.y, role = blockIdx.z;
  const int RS = P.ring_stride;
  const int lane = threadIdx.x & 31, warp = uniform_warp();
  const int jn = jn_of(P, jh), js = js_of(P, jh);
  // this pair's ring of field q (U/a, V/a, zeta, delta, phi'): I contiguous (north, south);
  // the role's fields are staged whole (coalesced 16-byte async copies, all in
  // flight at once): role 0 -> U, V, zeta, delta ; role 1 -> U, V, phi'
  const double2* gp = gr + (size_t)m * gmember + (size_t)jh * P.I;
  const int nst = role == 0 ? 4 : 3;
  for (int idx = threadIdx.x; idx < nst * P.I; idx += blockDim.x) {
    const int sidx = idx / P.I, il = idx - sidx * P.I;
    const int q = (role == 1 && sidx == 2) ? 4 : sidx;
    cp_async16(rings + idx, gp + (size_t)q * gfield + il);
  }
  cp_async_wait_all();
  __syncthreads();
  const double2* stg = rings;   // [nst][I], unpadded
  const double mu = P.mu_n[jh];
  const double fn = 2.0 * omega * mu;         // f = 2 Omega mu (swe.py:178); south: -fn
  const double c2o = 2.0 * omega / radius;    // swe.py:179
  const double ic2 = 1.0 / (1.0 - mu * mu);   // swe.py:180
  const int nprod = role == 0 ? (NONLIN ? 4 : 2) : 3;
  double2 v[K];
  const bool busy = warp < nprod;
  if (busy) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int il = 32 * k + lane;
      const double2 U = stg[il], V = stg[P.I + il];
      double2 z;
      if (role == 0) {
        const double2 Z = stg[2 * P.I + il], D = stg[3 * P.I + il];
        // swe.py:262,265,273 : A1 = -f delta - c2o V ; ZU = zeta U ; A2 = f zeta - c2o U ; ZV = zeta V
        const int w = NONLIN ? warp : 2 * warp;   // linear: A1, A2 only
        if (w == 0) z = d2(-fn * D.x - c2o * V.x, fn * D.y - c2o * V.y);
        else if (w == 1) z = d2(Z.x * U.x, Z.y * U.y);
        else if (w == 2) z = d2(fn * Z.x - c2o * U.x, -fn * Z.y - c2o * U.y);
        else z = d2(Z.x * V.x, Z.y * V.y);
      } else {
        const double2 Ph = stg[2 * P.I + il];
        // swe.py:271-272 : Phi U, Phi V, KE = (U^2 + V^2) / (2 (1 - mu^2))
        if (warp == 0) z = d2(Ph.x * U.x, Ph.y * U.y);
        else if (warp == 1) z = d2(Ph.x * V.x, Ph.y * V.y);
        else z = d2(0.5 * (U.x * U.x + V.x * V.x) * ic2, 0.5 * (U.y * U.y + V.y * V.y) * ic2);
      }
      v[k] = z;
    }
    double2 wst[3];
    swfft::cross_twiddles<K, false>(wst, P.tw, lane);
    swfft::ring_fft<K, false>(v, P.tw, lane, wst);
  }
  __syncthreads();   // staging consumed; the product rings reuse it
  if (busy) {
    double2* ring = rings + (size_t)warp * RS;
#pragma unroll
    for (int m1 = 0; m1 < K; ++m1) ring[swfft::pad_idx(swfft::ring_out_index<K>(lane, m1))] = v[m1];
  }
  __syncthreads();
  const bool eq = (jn == js);
  const double w = P.w_n[jh], wc = w * ic2, ia = 1.0 / radius;
  const double rwa_base = wc * ia, wa = wc * ia;
  double* xm = x + (size_t)m * xl.mstride;
  for (int r = threadIdx.x; r <= P.R; r += blockDim.x) {
    const double rwa = r * rwa_base;
    if (role == 0 && !NONLIN) {
      double2 A1n, A1s, A2n, A2s;
      get_pair(rings, P, r, A1n, A1s);
      get_pair(rings + RS, P, r, A2n, A2s);
      put_x(xm, xl, 0, r, jh, cscale(A1n, w), cscale(A1s, w), eq);
      put_x(xm, xl, 1, r, jh, cscale(A2n, w), cscale(A2s, w), eq);
    } else if (role == 0) {
      double2 A1n, A1s, ZUn, ZUs, A2n, A2s, ZVn, ZVs;
      get_pair(rings, P, r, A1n, A1s);
      get_pair(rings + RS, P, r, ZUn, ZUs);
      get_pair(rings + 2 * RS, P, r, A2n, A2s);
      get_pair(rings + 3 * RS, P, r, ZVn, ZVs);
      put_x(xm, xl, 1, r, jh, cadd2(cscale(A1n, w), ir_scale(ZUn, -rwa)),
            cadd2(cscale(A1s, w), ir_scale(ZUs, -rwa)), eq);
      put_x(xm, xl, 2, r, jh, cadd2(cscale(A2n, w), ir_scale(ZVn, rwa)),
            cadd2(cscale(A2s, w), ir_scale(ZVs, rwa)), eq);
      put_x(xm, xl, 5, r, jh, cscale(ZVn, wa), cscale(ZVs, wa), eq);
      put_x(xm, xl, 6, r, jh, cscale(ZUn, wa), cscale(ZUs, wa), eq);
    } else {
      double2 PUn, PUs, PVn, PVs, Kn, Ks;
      get_pair(rings, P, r, PUn, PUs);
      get_pair(rings + RS, P, r, PVn, PVs);
      get_pair(rings + 2 * RS, P, r, Kn, Ks);
      put_x(xm, xl, 0, r, jh, ir_scale(PUn, -rwa), ir_scale(PUs, -rwa), eq);
      put_x(xm, xl, 3, r, jh, cscale(Kn, w), cscale(Ks, w), eq);
      put_x(xm, xl, 4, r, jh, cscale(PVn, wa), cscale(PVs, wa), eq);
    }
  }
}

// ---------------------------------------------------------------------------
// Fused explicit-tendency grid stage, one latitude pair per CTA.
//   in : eo[m][5][R+1][Jh][2] for (U/a, V/a, zeta, delta, phi')
//   out: x[m][NV][R+1][Jh][2], NV = 7 (nonlinear) or 2 (linear only)
// ---------------------------------------------------------------------------
template <bool NONLIN, bool BIGP>
__global__ void __launch_bounds__(256, 2) swe_grid_kernel(PlanDev P, const double2* eo, long long eo_mstride, double* x,
                                XLayout xl, double omega, double radius, int jh_begin) {
  pdl_wait();
  pdl_trigger();
  constexpr int NIN = NONLIN ? 5 : 4;
  constexpr int NPROD = NONLIN ? 7 : 2;
  extern __shared__ __align__(16) double2 rings[];  // [7 or 4][RS]
  const int jh = jh_begin + blockIdx.x;
  const int m = blockIdx.y;
  const int RS = P.ring_stride;
  const size_t fstride = (size_t)(P.R + 1) * P.Jh * 2;
  fill_rings(rings, P, eo + (size_t)m * eo_mstride + (size_t)jh * 2, fstride, NIN, 1, 0, 0);
  __syncthreads();
  fft_inverse<BIGP>(rings, NIN, P);

  const double mu = P.mu_n[jh];
  const double fn = 2.0 * omega * mu;         // f = 2 Omega mu (swe.py:178); south: -fn
  const double c2o = 2.0 * omega / radius;    // swe.py:179
  const double ic2 = 1.0 / (1.0 - mu * mu);   // swe.py:180
  // the forward FFT wants its input in digit-reversed slots: read every grid
  // point this thread owns, barrier, then write the products permuted
  double2 gv[kSweMaxPts][NIN];
#pragma unroll
  for (int u = 0; u < kSweMaxPts; ++u) {
    const int il = threadIdx.x + u * blockDim.x;
    if (il < P.I) {
      const int p = swfft::pad_idx(il);
#pragma unroll
      for (int q = 0; q < NIN; ++q) gv[u][q] = rings[q * RS + p];
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kSweMaxPts; ++u) {
    const int il = threadIdx.x + u * blockDim.x;
    if (il >= P.I) continue;
    const int p = P.rev[il];
    const double2 U = gv[u][0], V = gv[u][1], Z = gv[u][2], D = gv[u][3];
    // swe.py:262,265 : tend_zeta grid = -f delta - (2 Omega/a) V ; tend_delta grid = f zeta - (2 Omega/a) U
    rings[p] = d2(-fn * D.x - c2o * V.x, fn * D.y - c2o * V.y);
    rings[RS + p] = d2(fn * Z.x - c2o * U.x, -fn * Z.y - c2o * U.y);
    if (NONLIN) {
      const double2 Ph = gv[u][NIN - 1];
      // swe.py:271-273 : Phi U, Phi V, zeta U, zeta V, KE = (U^2 + V^2) / (2 (1 - mu^2))
      rings[2 * RS + p] = d2(Ph.x * U.x, Ph.y * U.y);
      rings[3 * RS + p] = d2(Ph.x * V.x, Ph.y * V.y);
      rings[4 * RS + p] = d2(Z.x * U.x, Z.y * U.y);
      rings[5 * RS + p] = d2(Z.x * V.x, Z.y * V.y);
      rings[6 * RS + p] = d2(0.5 * (U.x * U.x + V.x * V.x) * ic2, 0.5 * (U.y * U.y + V.y * V.y) * ic2);
    }
  }
  __syncthreads();
  fft_forward<BIGP>(rings, NPROD, P);

  const bool eq = (jn_of(P, jh) == js_of(P, jh));
  const double w = P.w_n[jh];
  const double wc = w * ic2;
  const double ia = 1.0 / radius;
  double* xm = x + (size_t)m * xl.mstride;
  for (int r = threadIdx.x; r <= P.R; r += blockDim.x) {
    double2 A1n, A1s, A2n, A2s;
    get_pair(rings, P, r, A1n, A1s);
    get_pair(rings + RS, P, r, A2n, A2s);
    if (!NONLIN) {
      put_x(xm, xl, 0, r, jh, cscale(A1n, w), cscale(A1s, w), eq);
      put_x(xm, xl, 1, r, jh, cscale(A2n, w), cscale(A2s, w), eq);
    } else {
      double2 PUn, PUs, PVn, PVs, ZUn, ZUs, ZVn, ZVs, Kn, Ks;
      get_pair(rings + 2 * RS, P, r, PUn, PUs);
      get_pair(rings + 3 * RS, P, r, PVn, PVs);
      get_pair(rings + 4 * RS, P, r, ZUn, ZUs);
      get_pair(rings + 5 * RS, P, r, ZVn, ZVs);
      get_pair(rings + 6 * RS, P, r, Kn, Ks);
      const double rwa = r * wc * ia, wa = wc * ia;
      // P-vectors: phi, zeta, delta, ke ; H-vectors: phi, zeta, delta
      put_x(xm, xl, 0, r, jh, ir_scale(PUn, -rwa), ir_scale(PUs, -rwa), eq);
      put_x(xm, xl, 1, r, jh, cadd2(cscale(A1n, w), ir_scale(ZUn, -rwa)),
            cadd2(cscale(A1s, w), ir_scale(ZUs, -rwa)), eq);
      put_x(xm, xl, 2, r, jh, cadd2(cscale(A2n, w), ir_scale(ZVn, rwa)),
            cadd2(cscale(A2s, w), ir_scale(ZVs, rwa)), eq);
      put_x(xm, xl, 3, r, jh, cscale(Kn, w), cscale(Ks, w), eq);
      put_x(xm, xl, 4, r, jh, cscale(PVn, wa), cscale(PVs, wa), eq);
      put_x(xm, xl, 5, r, jh, cscale(ZVn, wa), cscale(ZVs, wa), eq);
      put_x(xm, xl, 6, r, jh, cscale(ZUn, wa), cscale(ZUs, wa), eq);
    }
  }
}

// ---------------------------------------------------------------------------
// Large-n_lon variant of the fused grid stage: the grids (U/a, V/a, zeta,
// phi') come from HBM (written by f2g_kernel) and the 5 products are
// transformed pairwise through 2 rings, each pair completing its analysis
// vectors: (ZU, ZV) -> v1, v6, v2, v5; (PU, PV) -> v0, v4; KE -> v3.  As in
// swe_grid5_kernel, the Coriolis terms A1 / A2 of v1 / v2 are formed in
// Fourier space from the input spectra (E, O partial sums at eo) instead of
// by two more forward transforms.
// ---------------------------------------------------------------------------
template <bool NONLIN, bool BIGP, bool RINGS = false, int K15 = 0>
__global__ void __launch_bounds__(256, 1) swe_prod_kernel(PlanDev P, const double* grids,
                                                          long long gfield, long long gmember,
                                                          const double2* eo, long long eo_fstride,
                                                          double* x, XLayout xl, double omega,
                                                          double radius, int jh_begin) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double2 rings[];  // [2][RS]
  const int jh = jh_begin + blockIdx.x, m = blockIdx.y;
  const int RS = P.ring_stride, I = P.I;
  const int jn = jn_of(P, jh), js = js_of(P, jh);
  const bool eq = (jn == js);
  const double* gm = grids + (size_t)m * gmember;
  const double mu = P.mu_n[jh];
  const double fn = 2.0 * omega * mu, c2o = 2.0 * omega / radius, ic2 = 1.0 / (1.0 - mu * mu);
  const double w = P.w_n[jh], wc = w * ic2, ia = 1.0 / radius;
  double* xm = x + (size_t)m * xl.mstride;
  // grid value of field q at longitude il, north (x) and south (y); RINGS:
  // rings[m][q][jh][il] (double2; gfield, gmember in double2)
  const double2* gr = reinterpret_cast<const double2*>(grids) + (size_t)m * gmember + (size_t)jh * I;
  auto gv = [&](int q, int il) {
    if (RINGS) return gr[(size_t)q * gfield + il];
    const double* g = gm + (size_t)q * gfield + (size_t)il * P.J;
    return d2(g[jn], g[js]);
  };
  // input spectra (F_n, F_s) of field q at wavenumber r (Im dropped at r = 0,
  // as the grid round trip would): eo fields U/a, V/a, zeta, delta, phi'
  const double2* em = eo + (size_t)m * 5 * eo_fstride + (size_t)jh * 2;
  auto coef = [&](int q, int r, double2& Fn, double2& Fs) {
    double2 E, O;
    ld_global_256(em + (size_t)q * eo_fstride + (size_t)r * P.Jh * 2, E, O);
    Fn = d2(E.x + O.x, r == 0 ? 0.0 : E.y + O.y);
    Fs = d2(E.x - O.x, r == 0 ? 0.0 : E.y - O.y);
  };
  // Passes over the grids (each ends with the forward FFTs of its rings and the
  // analysis vectors they complete): nonlinear -- pass 0: ZU, ZV, KE (3 rings)
  // -> v1, v6, v2, v5, v3; pass 1: PU, PV -> v0, v4 (U and V are read twice, not
  // three times); linear only (include_nonlinear=False): pass 4: A1, A2 -> v0, v1.
  for (int pass = NONLIN ? 0 : 4; pass < (NONLIN ? 2 : 5); ++pass) {
    const int nr = (pass == 0) ? 3 : 2;
#pragma unroll 4
    for (int il = threadIdx.x; il < I; il += blockDim.x) {
      const double2 U = gv(0, il), V = gv(1, il);
      double2 a, b, c = d2(0.0, 0.0);
      if (pass == 0) {          // ZU = zeta U ; ZV = zeta V ; KE = (U^2 + V^2) / (2 (1 - mu^2))
        const double2 Z = gv(2, il);
        a = d2(Z.x * U.x, Z.y * U.y);
        b = d2(Z.x * V.x, Z.y * V.y);
        c = d2(0.5 * (U.x * U.x + V.x * V.x) * ic2, 0.5 * (U.y * U.y + V.y * V.y) * ic2);
      } else if (pass == 1) {   // PU = phi U ; PV = phi V
        const double2 Ph = gv(4, il);
        a = d2(Ph.x * U.x, Ph.y * U.y);
        b = d2(Ph.x * V.x, Ph.y * V.y);
      } else {                  // linear: A1, A2
        const double2 D = gv(3, il), Z = gv(2, il);
        a = d2(-fn * D.x - c2o * V.x, fn * D.y - c2o * V.y);
        b = d2(fn * Z.x - c2o * U.x, -fn * Z.y - c2o * U.y);
      }
      const int p = K15 > 0 ? swfft::pad_idx(il) : P.rev[il];
      rings[p] = a;
      rings[RS + p] = b;
      if (nr == 3) rings[2 * RS + p] = c;
    }
    __syncthreads();
    if constexpr (K15 > 0) {
      for (int q = 0; q < nr; ++q) swfft::ring_fft15<K15, false>(rings + (size_t)q * RS, P.tw);
    } else {
      fft_forward<BIGP>(rings, nr, P);
    }
    for (int r = threadIdx.x; r <= P.R; r += blockDim.x) {
      double2 An, As, Bn, Bs;
      get_pair(rings, P, r, An, As);
      get_pair(rings + RS, P, r, Bn, Bs);
      const double rwa = r * wc * ia, wa = wc * ia;
      if (pass == 0) {
        // swe.py:262,265 in Fourier space (f = fn north, -fn south)
        double2 Un, Us, Vn, Vs, Zn, Zs, Dn, Ds, Kn, Ks;
        get_pair(rings + 2 * RS, P, r, Kn, Ks);
        coef(0, r, Un, Us);
        coef(1, r, Vn, Vs);
        coef(2, r, Zn, Zs);
        coef(3, r, Dn, Ds);
        const double2 A1n = d2(-fn * Dn.x - c2o * Vn.x, -fn * Dn.y - c2o * Vn.y);
        const double2 A1s = d2(fn * Ds.x - c2o * Vs.x, fn * Ds.y - c2o * Vs.y);
        const double2 A2n = d2(fn * Zn.x - c2o * Un.x, fn * Zn.y - c2o * Un.y);
        const double2 A2s = d2(-fn * Zs.x - c2o * Us.x, -fn * Zs.y - c2o * Us.y);
        put_x(xm, xl, 1, r, jh, cadd2(cscale(A1n, w), ir_scale(An, -rwa)),
              cadd2(cscale(A1s, w), ir_scale(As, -rwa)), eq);
        put_x(xm, xl, 6, r, jh, cscale(An, wa), cscale(As, wa), eq);
        put_x(xm, xl, 2, r, jh, cadd2(cscale(A2n, w), ir_scale(Bn, rwa)),
              cadd2(cscale(A2s, w), ir_scale(Bs, rwa)), eq);
        put_x(xm, xl, 5, r, jh, cscale(Bn, wa), cscale(Bs, wa), eq);
        put_x(xm, xl, 3, r, jh, cscale(Kn, w), cscale(Ks, w), eq);
      } else if (pass == 1) {
        put_x(xm, xl, 0, r, jh, ir_scale(An, -rwa), ir_scale(As, -rwa), eq);
        put_x(xm, xl, 4, r, jh, cscale(Bn, wa), cscale(Bs, wa), eq);
      } else {
        put_x(xm, xl, 0, r, jh, cscale(An, w), cscale(As, w), eq);
        put_x(xm, xl, 1, r, jh, cscale(Bn, w), cscale(Bs, w), eq);
      }
    }
    __syncthreads();
  }
}

int pick_threads(int work, bool bigp) {
  if (bigp) return work >= 128 ? 128 : 64;
  if (work >= 256) return 256;
  if (work >= 128) return 128;
  return 64;
}

int max_butterflies(const PlanDev& P) {
  int mx = 1;
  for (int s = 0; s < P.fft.nstage; ++s) mx = std::max(mx, P.fft.n / P.fft.radix[s]);
  return mx;
}

int set_smem(const void* kern, size_t smem) {
  if (smem > 227 * 1024) {
    set_error("longitude ring does not fit in shared memory (n_lon too large for this kernel)");
    return kUsage;
  }
  return set_max_dyn_smem(kern, smem);
}

// log2 of pairs per CTA: rings <= ~56 KB (4 CTAs/SM), at most 8 pairs
int pairs_log2(const PlanDev& P, int nin) {
  const size_t ring = sizeof(double2) * P.ring_stride * nin;
  int l = 0;
  while (l < 3 && ring * (2 << l) <= 56 * 1024 && (2 << l) <= P.Jh) ++l;
  return l;
}

// Register-FFT dispatch: n_lon = 32 K with K in reg_fft_k_ok (SWSDC_REG_FFT=0 disables).
bool use_reg_fft(const PlanDev& P) {
  static const int knob = env_int("SWSDC_REG_FFT", 1);
  return knob != 0 && P.I % 32 == 0 && swfft::reg_fft_k_ok(P.I / 32);
}

template <int K>
int f2g_reg_launch(const PlanDev& P, const double2* eo, long long eo_fstride, double* grid,
                   long long grid_fstride, int nf, int jh_begin, int jh_end, cudaStream_t st) {
  const int lnp = pairs_log2(P, 1), np = 1 << lnp;
  const size_t smem = sizeof(double2) * f2g_reg_elems(P, np);
  SW_TRY(set_smem((const void*)f2g_reg_kernel<K>, smem));
  dim3 gridDim((jh_end - jh_begin + np - 1) / np, nf);
  if (gridDim.x == 0) return kOk;
  StageScope sc("fourier_to_grid", st);
  SW_CUDA(launch_pdl(f2g_reg_kernel<K>, dim3(gridDim), dim3(32 * np), smem, st, P, eo, eo_fstride, grid, grid_fstride, lnp, jh_begin, jh_end));
  SW_LAUNCH_CHECK();
  return kOk;
}

template <int K, int MODE>
int g2f_reg_launch(const PlanDev& P, const double* grid, const double* grid2,
                   long long grid_fstride, double* x, const XLayout& xl, int nf, cudaStream_t st) {
  const int nin = MODE == 0 ? 1 : 2;
  const int lnp = std::min(pairs_log2(P, nin), 3 - (nin - 1)), np = 1 << lnp;   // <= 8 warps
  const size_t smem = sizeof(double2) * nin * np * P.ring_stride;
  dim3 gridDim((P.Jh + np - 1) / np, nf);
  SW_TRY(set_smem((const void*)g2f_reg_kernel<K, MODE>, smem));
  StageScope sc(MODE == 0 ? "grid_to_fourier" : "grid_to_fourier_divcurl", st);
  SW_CUDA(launch_pdl(g2f_reg_kernel<K, MODE>, dim3(gridDim), dim3(32 * nin * np), smem, st, P, grid, grid2, grid_fstride, x, xl, lnp));
  SW_LAUNCH_CHECK();
  return kOk;
}

#define SWSDC_REG_K_SWITCH(K_, CALL)                                              \
  switch (K_) {                                                                   \
    case 1: { constexpr int KK = 1; return CALL; }                                \
    case 2: { constexpr int KK = 2; return CALL; }                                \
    case 3: { constexpr int KK = 3; return CALL; }                                \
    case 4: { constexpr int KK = 4; return CALL; }                                \
    case 5: { constexpr int KK = 5; return CALL; }                                \
    case 6: { constexpr int KK = 6; return CALL; }                                \
    case 8: { constexpr int KK = 8; return CALL; }                                \
    case 10: { constexpr int KK = 10; return CALL; }                              \
    case 12: { constexpr int KK = 12; return CALL; }                              \
    case 16: { constexpr int KK = 16; return CALL; }                              \
    case 20: { constexpr int KK = 20; return CALL; }                              \
    case 24: { constexpr int KK = 24; return CALL; }                              \
  }

// n_lon = 15 * 32 K with one pair per CTA: the ring_fft15 kernels (SWSDC_FFT15=0 disables)
int fft15_path(const PlanDev& P, int lnp) {
  static const int knob = env_int("SWSDC_FFT15", 1);
  return (knob != 0 && lnp == 0) ? swfft::fft15_k(P.I) : 0;
}

#define SWSDC_K15_SWITCH(K_, CALL)                                                \
  switch (K_) {                                                                   \
    case 1: { constexpr int KK = 1; return CALL; }                                \
    case 2: { constexpr int KK = 2; return CALL; }                                \
    case 4: { constexpr int KK = 4; return CALL; }                                \
    case 8: { constexpr int KK = 8; return CALL; }                                \
    case 16: { constexpr int KK = 16; return CALL; }                              \
  }

template <bool BIGP, bool RINGS, int K15>
int f2g_launch_k(const PlanDev& P, const double2* eo, long long eo_fstride, double* grid,
                 long long grid_fstride, int nf, int jh_begin, int jh_end, int lnp, int threads,
                 cudaStream_t st) {
  const int np = 1 << lnp;
  const size_t smem = sizeof(double2) * np * P.ring_stride;
  SW_TRY(set_smem((const void*)f2g_kernel<BIGP, RINGS, K15>, smem));
  dim3 gridDim((jh_end - jh_begin + np - 1) / np, nf);
  if (gridDim.x == 0) return kOk;
  StageScope sc("fourier_to_grid", st);
  SW_CUDA(launch_pdl(f2g_kernel<BIGP, RINGS, K15>, dim3(gridDim), dim3(threads), smem, st, P, eo, eo_fstride, grid, grid_fstride, lnp, jh_begin, jh_end));
  SW_LAUNCH_CHECK();
  return kOk;
}

template <bool BIGP, bool RINGS = false>
int f2g_launch(const PlanDev& P, const double2* eo, long long eo_fstride, double* grid,
               long long grid_fstride, int nf, int jh_begin, int jh_end, cudaStream_t st) {
  const int lnp = pairs_log2(P, 1), np = 1 << lnp;
  SWSDC_K15_SWITCH(fft15_path(P, lnp), (f2g_launch_k<false, RINGS, KK>(P, eo, eo_fstride, grid, grid_fstride, nf, jh_begin, jh_end, lnp, 256, st)));
  return f2g_launch_k<BIGP, RINGS, 0>(P, eo, eo_fstride, grid, grid_fstride, nf, jh_begin, jh_end,
                                      lnp, pick_threads(np * max_butterflies(P), BIGP), st);
}

template <int MODE, bool BIGP, int K15>
int g2f_launch_k(const PlanDev& P, const double* grid, const double* grid2, long long grid_fstride,
                 double* x, const XLayout& xl, int nf, int lnp, int threads, cudaStream_t st) {
  const int nin = MODE == 0 ? 1 : 2;
  const int np = 1 << lnp;
  const size_t smem = sizeof(double2) * nin * np * P.ring_stride;
  dim3 gridDim((P.Jh + np - 1) / np, nf);
  SW_TRY(set_smem((const void*)g2f_kernel<MODE, BIGP, K15>, smem));
  StageScope sc(MODE == 0 ? "grid_to_fourier" : "grid_to_fourier_divcurl", st);
  SW_CUDA(launch_pdl(g2f_kernel<MODE, BIGP, K15>, dim3(gridDim), dim3(threads), smem, st, P, grid, grid2, grid_fstride, x, xl, lnp));
  SW_LAUNCH_CHECK();
  return kOk;
}

template <int MODE, bool BIGP>
int g2f_launch(const PlanDev& P, const double* grid, const double* grid2, long long grid_fstride,
               double* x, const XLayout& xl, int nf, cudaStream_t st) {
  const int nin = MODE == 0 ? 1 : 2;
  const int lnp = pairs_log2(P, nin), np = 1 << lnp;
  SWSDC_K15_SWITCH(fft15_path(P, lnp), (g2f_launch_k<MODE, false, KK>(P, grid, grid2, grid_fstride, x, xl, nf, lnp, 256, st)));
  return g2f_launch_k<MODE, BIGP, 0>(P, grid, grid2, grid_fstride, x, xl, nf, lnp,
                                     pick_threads(nin * np * max_butterflies(P), BIGP), st);
}

template <bool NONLIN, bool BIGP>
int swe_launch(const PlanDev& P, const double2* eo, long long eo_mstride, double* x,
               const XLayout& xl, int nmembers, double omega, double radius, int jh_begin,
               int jh_end, cudaStream_t st) {
  const int nr = NONLIN ? 7 : 4;
  const size_t smem = sizeof(double2) * nr * P.ring_stride;
  dim3 gridDim(jh_end - jh_begin, nmembers);
  if (gridDim.x == 0) return kOk;
  SW_TRY(set_smem((const void*)swe_grid_kernel<NONLIN, BIGP>, smem));
  int threads = pick_threads(nr * max_butterflies(P), BIGP);
  while (threads * kSweMaxPts < P.I && threads < 256) threads *= 2;
  if (threads * kSweMaxPts < P.I) {
    set_error("n_lon too large for the fused grid kernel");
    return kUsage;
  }
  StageScope sc("swe_grid", st);
  SW_CUDA(launch_pdl(swe_grid_kernel<NONLIN, BIGP>, dim3(gridDim), dim3(threads), smem, st, P, eo, eo_mstride, x, xl, omega, radius, jh_begin));
  SW_LAUNCH_CHECK();
  return kOk;
}

template <int K, bool NONLIN>
int swe_reg_launch(const PlanDev& P, const double2* eo, long long eo_mstride, double* x,
                   const XLayout& xl, int nmembers, double omega, double radius, int jh_begin,
                   int jh_end, cudaStream_t st) {
  const int nr = NONLIN ? 7 : 4;
  const size_t smem = sizeof(double2) * nr * P.ring_stride;
  dim3 gridDim(jh_end - jh_begin, nmembers);
  if (gridDim.x == 0) return kOk;
  static const int cl_knob = env_int("SWSDC_SWE_CLUSTER", 1);
  // the cluster only serves the column-major layout's 32-byte sectors; pair-major
  // x is written whole-sector by each pair's CTA
  const bool cl = cl_knob && !xl.pm && (jh_begin % 4 == 0) && ((jh_end - jh_begin) % 4 == 0);
  static const int g5 = env_int("SWSDC_SWE_G5", 1);   // 0: the 12-FFT kernel below
  if (NONLIN && g5) {
    const size_t smem5 = sizeof(double2) * ((size_t)kG5Rings * P.ring_stride + 8 * (P.R + 1) +
                                           swfft::tw_cache_entries<K>());
    StageScope sc("swe_grid", st);
    if (cl) {
      SW_TRY(set_smem((const void*)swe_grid5_kernel<K, true>, smem5));
      SW_CUDA(launch_pdl_cluster(swe_grid5_kernel<K, true>, dim3(gridDim), dim3(kG5Threads), smem5,
                                 st, 4, P, eo, eo_mstride, x, xl, omega, radius, jh_begin));
    } else {
      SW_TRY(set_smem((const void*)swe_grid5_kernel<K, false>, smem5));
      SW_CUDA(launch_pdl(swe_grid5_kernel<K, false>, dim3(gridDim), dim3(kG5Threads), smem5, st, P,
                         eo, eo_mstride, x, xl, omega, radius, jh_begin));
    }
    SW_LAUNCH_CHECK();
    return kOk;
  }
  // warps: 6 for K >= 20 (registers), 7 for K = 16 (all forward FFTs in one round), 8 below
  const int threads = K >= 20 ? 192 : K == 16 ? 224 : 256;
  if (cl) {
    SW_TRY(set_smem((const void*)swe_grid_reg_kernel<K, NONLIN, true>, smem));
    StageScope sc("swe_grid", st);
    SW_CUDA(launch_pdl_cluster(swe_grid_reg_kernel<K, NONLIN, true>, dim3(gridDim), dim3(threads),
                               smem, st, 4, P, eo, eo_mstride, x, xl, omega, radius, jh_begin));
    SW_LAUNCH_CHECK();
    return kOk;
  }
  SW_TRY(set_smem((const void*)swe_grid_reg_kernel<K, NONLIN>, smem));
  StageScope sc("swe_grid", st);
  SW_CUDA(launch_pdl(swe_grid_reg_kernel<K, NONLIN>, dim3(gridDim), dim3(threads), smem, st, P, eo, eo_mstride, x, xl, omega, radius, jh_begin));
  SW_LAUNCH_CHECK();
  return kOk;
}

template <int K, bool NONLIN>
int swe_fwd_reg_launch(const PlanDev& P, const double2* grids, long long gfield, long long gmember,
                       double* x, const XLayout& xl, int nmembers, double omega, double radius,
                       int jh_begin, int jh_end, cudaStream_t st) {
  const size_t smem = sizeof(double2) * 4 * P.ring_stride;
  SW_TRY(set_smem((const void*)swe_fwd_reg_kernel<K, NONLIN>, smem));
  dim3 gridDim(jh_end - jh_begin, nmembers, NONLIN ? 2 : 1);
  if (gridDim.x == 0) return kOk;
  StageScope sc("swe_products", st);
  SW_CUDA(launch_pdl(swe_fwd_reg_kernel<K, NONLIN>, dim3(gridDim), dim3(128), smem, st, P, grids, gfield, gmember, x, xl, omega, radius, jh_begin));
  SW_LAUNCH_CHECK();
  return kOk;
}

template <bool NONLIN, bool BIGP, int K15>
int swe_prod_launch_k(const PlanDev& P, const double* grids, long long gfield, long long gmember,
                      const double2* eo, long long eo_fstride, double* x, const XLayout& xl,
                      int nmembers, double omega, double radius, int jh_begin, int jh_end,
                      cudaStream_t st) {
  // grids in the ring layout (f2g_kernel<., true>): gfield / gmember in double2;
  // 3 rings for the nonlinear first pass (ZU, ZV, KE)
  const size_t smem = sizeof(double2) * (NONLIN ? 3 : 2) * P.ring_stride;
  SW_TRY(set_smem((const void*)swe_prod_kernel<NONLIN, BIGP, true, K15>, smem));
  dim3 gridDim(jh_end - jh_begin, nmembers);
  if (gridDim.x == 0) return kOk;
  StageScope sc("swe_products", st);
  SW_CUDA(launch_pdl(swe_prod_kernel<NONLIN, BIGP, true, K15>, dim3(gridDim), dim3(BIGP && K15 == 0 ? 128 : 256), smem, st, P, grids, gfield, gmember, eo, eo_fstride, x, xl, omega, radius, jh_begin));
  SW_LAUNCH_CHECK();
  return kOk;
}

template <bool NONLIN, bool BIGP>
int swe_prod_launch(const PlanDev& P, const double* grids, long long gfield, long long gmember,
                    const double2* eo, long long eo_fstride, double* x, const XLayout& xl,
                    int nmembers, double omega, double radius, int jh_begin, int jh_end,
                    cudaStream_t st) {
  SWSDC_K15_SWITCH(fft15_path(P, 0), (swe_prod_launch_k<NONLIN, false, KK>(P, grids, gfield, gmember, eo, eo_fstride, x, xl, nmembers, omega, radius, jh_begin, jh_end, st)));
  return swe_prod_launch_k<NONLIN, BIGP, 0>(P, grids, gfield, gmember, eo, eo_fstride, x, xl,
                                            nmembers, omega, radius, jh_begin, jh_end, st);
}

}  // namespace

// Split F_E path with register FFTs: E/O -> 5 rings per pair (ring layout,
// rings[m][q][jh][il]) -> products, forward FFTs, analysis vectors.
int launch_swe_split_reg(const PlanDev& P, bool nonlinear, const double2* eo, long long eo_fstride,
                         double2* ring_ws, double* x, const XLayout& xl, int nmembers,
                         double omega, double radius, cudaStream_t st, int jh_begin, int jh_end) {
  const long long gfield = (long long)P.Jh * P.I;   // double2 per field ring block
  const int lnp = pairs_log2(P, 1), np = 1 << lnp;
  dim3 g1((jh_end - jh_begin + np - 1) / np, 5 * nmembers);
  int st1 = kOk;
  auto first = [&](auto kk) -> int {
    constexpr int KK = decltype(kk)::value;
    const size_t smem1 = sizeof(double2) * f2g_reg_elems(P, np);
    SW_TRY(set_smem((const void*)f2g_reg_kernel<KK, true>, smem1));
    StageScope sc("fourier_to_grid", st);
    SW_CUDA(launch_pdl(f2g_reg_kernel<KK, true>, dim3(g1), dim3(32 * np), smem1, st, P, eo, eo_fstride, reinterpret_cast<double*>(ring_ws), gfield, lnp, jh_begin, jh_end));
    SW_LAUNCH_CHECK();
    if (nonlinear)
      return swe_fwd_reg_launch<KK, true>(P, ring_ws, gfield, 5 * gfield, x, xl, nmembers, omega,
                                          radius, jh_begin, jh_end, st);
    return swe_fwd_reg_launch<KK, false>(P, ring_ws, gfield, 5 * gfield, x, xl, nmembers, omega,
                                         radius, jh_begin, jh_end, st);
  };
  if (g1.x == 0) return kOk;
  switch (P.I / 32) {
    case 1: st1 = first(std::integral_constant<int, 1>()); break;
    case 2: st1 = first(std::integral_constant<int, 2>()); break;
    case 3: st1 = first(std::integral_constant<int, 3>()); break;
    case 4: st1 = first(std::integral_constant<int, 4>()); break;
    case 5: st1 = first(std::integral_constant<int, 5>()); break;
    case 6: st1 = first(std::integral_constant<int, 6>()); break;
    case 8: st1 = first(std::integral_constant<int, 8>()); break;
    case 10: st1 = first(std::integral_constant<int, 10>()); break;
    case 12: st1 = first(std::integral_constant<int, 12>()); break;
    case 16: st1 = first(std::integral_constant<int, 16>()); break;
    case 20: st1 = first(std::integral_constant<int, 20>()); break;
    case 24: st1 = first(std::integral_constant<int, 24>()); break;
    default: set_error("register FFT size not supported"); return kUsage;
  }
  return st1;
}

bool fourier_reg_fft(const PlanDev& P) { return use_reg_fft(P); }

bool swe_grid_fits(const PlanDev& P) {
  return sizeof(double2) * 7 * (size_t)P.ring_stride <= 160 * 1024;
}

// Small batches (few latitude pairs x members) leave the one-pair-per-CTA fused
// kernel short of CTAs; the split path (f2g of the 5 grids, then the role-split
// forward kernel) runs ~3x more warps.  SWSDC_SWE_SPLIT: 0 never (default),
// 1 below SMs/2 pairs x members, 2 always.
bool swe_split_preferred(const PlanDev& P, long long pair_members) {
  // default off: with the cluster output and PDL the fused kernel is as fast
  // even for config 0's tiny grids (0.266 vs 0.268 ms/step, same-box A/B)
  static const int knob = env_int("SWSDC_SWE_SPLIT", 0);
  if (knob == 0 || !use_reg_fft(P)) return false;
  if (knob == 2) return true;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  // measured (config 0 / 2): the split path wins only when the fused kernel
  // would run well under one CTA per SM
  return 2 * pair_members <= sms;
}

int launch_swe_products(const PlanDev& P, bool nonlinear, const double* grids, long long gfield,
                        long long gmember, const double2* eo, long long eo_fstride, double* x,
                        const XLayout& xl, int nmembers, double omega, double radius,
                        cudaStream_t st, int jh_begin, int jh_end) {
  if (jh_end < 0) jh_end = P.Jh;
  const bool big = swfft::fft_needs_bigp(P.I);
  if (nonlinear) {
    if (big) return swe_prod_launch<true, true>(P, grids, gfield, gmember, eo, eo_fstride, x, xl, nmembers, omega, radius, jh_begin, jh_end, st);
    return swe_prod_launch<true, false>(P, grids, gfield, gmember, eo, eo_fstride, x, xl, nmembers, omega, radius, jh_begin, jh_end, st);
  }
  if (big) return swe_prod_launch<false, true>(P, grids, gfield, gmember, eo, eo_fstride, x, xl, nmembers, omega, radius, jh_begin, jh_end, st);
  return swe_prod_launch<false, false>(P, grids, gfield, gmember, eo, eo_fstride, x, xl, nmembers, omega, radius, jh_begin, jh_end, st);
}

// Smem-FFT inverse of nf (E, O) fields into the ring layout rings[f][jh][il]
// (double2, ring_fstride in double2): the grid stage of the split F_E path.
int launch_fourier_to_rings(const PlanDev& P, const double2* eo, long long eo_fstride,
                            double2* rings, long long ring_fstride, int nf, cudaStream_t st,
                            int jh_begin, int jh_end) {
  if (jh_end < 0) jh_end = P.Jh;
  double* g = reinterpret_cast<double*>(rings);
  if (swfft::fft_needs_bigp(P.I))
    return f2g_launch<true, true>(P, eo, eo_fstride, g, ring_fstride, nf, jh_begin, jh_end, st);
  return f2g_launch<false, true>(P, eo, eo_fstride, g, ring_fstride, nf, jh_begin, jh_end, st);
}

int launch_fourier_to_grid(const PlanDev& P, const double2* eo, long long eo_fstride, double* grid,
                           long long grid_fstride, int nf, cudaStream_t st, int jh_begin,
                           int jh_end) {
  if (jh_end < 0) jh_end = P.Jh;
  if (use_reg_fft(P)) {
    SWSDC_REG_K_SWITCH(P.I / 32, (f2g_reg_launch<KK>(P, eo, eo_fstride, grid, grid_fstride, nf,
                                                     jh_begin, jh_end, st)));
  }
  if (swfft::fft_needs_bigp(P.I))
    return f2g_launch<true>(P, eo, eo_fstride, grid, grid_fstride, nf, jh_begin, jh_end, st);
  return f2g_launch<false>(P, eo, eo_fstride, grid, grid_fstride, nf, jh_begin, jh_end, st);
}

int launch_grid_to_fourier(const PlanDev& P, int mode, const double* grid, const double* grid2,
                           long long grid_fstride, double* x, const XLayout& xl, int nf,
                           cudaStream_t st) {
  if (use_reg_fft(P)) {
    if (mode == 0) {
      SWSDC_REG_K_SWITCH(P.I / 32, (g2f_reg_launch<KK, 0>(P, grid, grid2, grid_fstride, x, xl, nf, st)));
    } else {
      SWSDC_REG_K_SWITCH(P.I / 32, (g2f_reg_launch<KK, 1>(P, grid, grid2, grid_fstride, x, xl, nf, st)));
    }
  }
  const bool big = swfft::fft_needs_bigp(P.I);
  if (mode == 0) {
    if (big) return g2f_launch<0, true>(P, grid, grid2, grid_fstride, x, xl, nf, st);
    return g2f_launch<0, false>(P, grid, grid2, grid_fstride, x, xl, nf, st);
  }
  if (big) return g2f_launch<1, true>(P, grid, grid2, grid_fstride, x, xl, nf, st);
  return g2f_launch<1, false>(P, grid, grid2, grid_fstride, x, xl, nf, st);
}

int launch_swe_grid(const PlanDev& P, bool nonlinear, const double2* eo, long long eo_mstride,
                    double* x, const XLayout& xl, int nmembers, double omega, double radius,
                    cudaStream_t st, int jh_begin, int jh_end) {
  if (jh_end < 0) jh_end = P.Jh;
  if (use_reg_fft(P)) {
    if (nonlinear) {
      SWSDC_REG_K_SWITCH(P.I / 32, (swe_reg_launch<KK, true>(P, eo, eo_mstride, x, xl, nmembers,
                                                             omega, radius, jh_begin, jh_end, st)));
    } else {
      SWSDC_REG_K_SWITCH(P.I / 32, (swe_reg_launch<KK, false>(P, eo, eo_mstride, x, xl, nmembers,
                                                              omega, radius, jh_begin, jh_end, st)));
    }
  }
  const bool big = swfft::fft_needs_bigp(P.I);
  if (nonlinear) {
    if (big) return swe_launch<true, true>(P, eo, eo_mstride, x, xl, nmembers, omega, radius, jh_begin, jh_end, st);
    return swe_launch<true, false>(P, eo, eo_mstride, x, xl, nmembers, omega, radius, jh_begin, jh_end, st);
  }
  if (big) return swe_launch<false, true>(P, eo, eo_mstride, x, xl, nmembers, omega, radius, jh_begin, jh_end, st);
  return swe_launch<false, false>(P, eo, eo_mstride, x, xl, nmembers, omega, radius, jh_begin, jh_end, st);
}

}  // namespace swsdc

#ifdef GRID_TRACE
extern "C" int swsdc_debug_grid_trace(unsigned long long* host, int clear) {
  if (clear) {
    static unsigned long long zero[16384][8];
    return cudaMemcpyToSymbol(swsdc::g_grid_trace, zero, sizeof(zero)) == cudaSuccess ? 0 : 3;
  }
  return cudaMemcpyFromSymbol(host, swsdc::g_grid_trace, sizeof(unsigned long long) * 16384 * 8) ==
                 cudaSuccess ? 0 : 3;
}
#endif
