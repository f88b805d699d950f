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
#include "common.cuh"
#include "fourier.cuh"

namespace swsdc {
namespace {

template <bool BIGP>
__device__ __forceinline__ void fft_stage_all(double2* rings, int nrings, const PlanDev& P, int s,
                                              bool inverse) {
  const swfft::FftPlan& fp = P.fft;
  const int r = fp.radix[s];
  const int nb = fp.n / r;
  const int total = nrings * nb;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int q = t / nb, b = t - q * nb;
    double2* ring = rings + (size_t)q * fp.n;
    swfft::stage_butterfly<BIGP>(ring, fp, s, b, P.tw, inverse);
  }
}

// Forward: natural -> digit-reversed.  Caller synchronises before.
template <bool BIGP>
__device__ void fft_forward(double2* rings, int nrings, const PlanDev& P) {
  for (int s = 0; s < P.fft.nstage; ++s) {
    fft_stage_all<BIGP>(rings, nrings, P, s, false);
    __syncthreads();
  }
}
// Inverse (unnormalised): digit-reversed -> natural.
template <bool BIGP>
__device__ void fft_inverse(double2* rings, int nrings, const PlanDev& P) {
  for (int s = P.fft.nstage - 1; s >= 0; --s) {
    fft_stage_all<BIGP>(rings, nrings, P, s, true);
    __syncthreads();
  }
}

__device__ __forceinline__ void zero_rings(double2* rings, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) rings[i] = make_double2(0.0, 0.0);
}

// Place the spectra of a pair (F_n, F_s at wavenumber r) into a packed ring
// in digit-reversed order.
__device__ __forceinline__ void put_pair(double2* ring, const PlanDev& P, int r, double2 Fn,
                                         double2 Fs) {
  if (r == 0) {
    ring[0] = make_double2(Fn.x, Fs.x);  // irfft drops Im of the DC bin
  } else {
    ring[swfft::digit_rev(P.fft, r)] = make_double2(Fn.x - Fs.y, Fn.y + Fs.x);
    ring[swfft::digit_rev(P.fft, P.I - r)] = make_double2(Fn.x + Fs.y, Fs.x - Fn.y);
  }
}

// Unpack F_n, F_s (already divided by n_lon) at wavenumber r from a forward-
// transformed packed ring.
__device__ __forceinline__ void get_pair(const double2* ring, const PlanDev& P, int r, double2& Fn,
                                         double2& Fs) {
  const double2 zk = ring[swfft::digit_rev(P.fft, r)];
  const double2 zm = ring[swfft::digit_rev(P.fft, r == 0 ? 0 : P.I - r)];
  const double h = 0.5 / P.I;
  Fn = make_double2((zk.x + zm.x) * h, (zk.y - zm.y) * h);
  Fs = make_double2((zk.y + zm.y) * h, (zm.x - zk.x) * h);
}

__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// i r s * a
__device__ __forceinline__ double2 ir_scale(double2 a, double rs) { return make_double2(-a.y * rs, a.x * rs); }
__device__ __forceinline__ double2 cadd2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

// Write one analysis vector (S, D) from its north / south values.
__device__ __forceinline__ void put_sd(double2* x, double2 vn, double2 vs, bool equator) {
  if (equator) {
    x[0] = vn;
    x[1] = make_double2(0.0, 0.0);
  } else {
    x[0] = make_double2(vn.x + vs.x, vn.y + vs.y);
    x[1] = make_double2(vn.x - vs.x, vn.y - vs.y);
  }
}

// ---------------------------------------------------------------------------
// (E, O) -> grid, np pairs per CTA.  grid: [f][I][J]
// ---------------------------------------------------------------------------
template <bool BIGP>
__global__ void f2g_kernel(PlanDev P, const double2* eo, long long eo_fstride, double* grid,
                           long long grid_fstride, int np) {
  extern __shared__ __align__(16) double2 rings[];
  const int f = blockIdx.y;
  const int jh0 = blockIdx.x * np;
  const double2* e = eo + (size_t)f * eo_fstride;
  double* g = grid + (size_t)f * grid_fstride;
  zero_rings(rings, np * P.I);
  __syncthreads();
  for (int idx = threadIdx.x; idx < np * (P.R + 1); idx += blockDim.x) {
    const int r = idx / np, i = idx - r * np;
    const int jh = jh0 + i;
    if (jh >= P.Jh) continue;
    const double2* src = e + ((size_t)r * P.Jh + jh) * 2;
    const double2 E = src[0], O = src[1];
    put_pair(rings + (size_t)i * P.I, P, r, make_double2(E.x + O.x, E.y + O.y),
             make_double2(E.x - O.x, E.y - O.y));
  }
  __syncthreads();
  fft_inverse<BIGP>(rings, np, P);
  for (int idx = threadIdx.x; idx < np * P.I; idx += blockDim.x) {
    const int il = idx / np, i = idx - il * np;
    const int jh = jh0 + i;
    if (jh >= P.Jh) continue;
    const double2 z = rings[(size_t)i * P.I + il];
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
template <int MODE, bool BIGP>
__global__ void g2f_kernel(PlanDev P, const double* grid, const double* grid2,
                           long long grid_fstride, double2* x, long long x_fstride, int np) {
  constexpr int NIN = (MODE == 0) ? 1 : 2;
  extern __shared__ __align__(16) double2 rings[];  // [NIN][np][I]
  const int f = blockIdx.y;
  const int jh0 = blockIdx.x * np;
  const double* gin[2] = {grid + (size_t)f * grid_fstride,
                          (MODE == 0 ? grid : grid2) + (size_t)f * grid_fstride};
  for (int idx = threadIdx.x; idx < NIN * np * P.I; idx += blockDim.x) {
    const int q = idx / (np * P.I);
    const int rem = idx - q * np * P.I;
    const int il = rem / np, i = rem - il * np;
    const int jh = jh0 + i;
    double2 z = make_double2(0.0, 0.0);
    if (jh < P.Jh) {
      const double* gq = gin[q] + (size_t)il * P.J;
      z = make_double2(gq[jn_of(P, jh)], gq[js_of(P, jh)]);
    }
    rings[((size_t)q * np + i) * P.I + il] = z;
  }
  __syncthreads();
  fft_forward<BIGP>(rings, NIN * np, P);
  double2* xf = x + (size_t)f * x_fstride;
  const size_t vstride = (size_t)(P.R + 1) * P.Jh * 2;
  for (int idx = threadIdx.x; idx < np * (P.R + 1); idx += blockDim.x) {
    const int r = idx / np, i = idx - r * np;
    const int jh = jh0 + i;
    if (jh >= P.Jh) continue;
    const bool eq = (jn_of(P, jh) == js_of(P, jh));
    const double mu = P.mu_n[jh], w = P.w_n[jh];
    double2* xo = xf + ((size_t)r * P.Jh + jh) * 2;
    if (MODE == 0) {
      double2 Fn, Fs;
      get_pair(rings + (size_t)i * P.I, P, r, Fn, Fs);
      put_sd(xo, cscale(Fn, w), cscale(Fs, w), eq);
    } else {
      double2 Un, Us, Vn, Vs;
      get_pair(rings + (size_t)i * P.I, P, r, Un, Us);
      get_pair(rings + (size_t)(np + i) * P.I, P, r, Vn, Vs);
      const double wc = w / (1.0 - mu * mu);
      const double rw = r * wc;
      // div = Pwc2 (i r F_U) - Hwc2 F_V ; curl = Pwc2 (i r F_V) + Hwc2 F_U  (spharm.py:294-299)
      put_sd(xo, ir_scale(Un, rw), ir_scale(Us, rw), eq);
      put_sd(xo + vstride, cscale(Vn, -wc), cscale(Vs, -wc), eq);
      put_sd(xo + 2 * vstride, ir_scale(Vn, rw), ir_scale(Vs, rw), eq);
      put_sd(xo + 3 * vstride, cscale(Un, wc), cscale(Us, wc), eq);
    }
  }
}

// ---------------------------------------------------------------------------
// Fused explicit-tendency grid stage, one latitude pair per CTA.
//   in : eo[m][5][R+1][Jh][2] for (U/a, V/a, zeta, delta, phi')
//   out: x[m][NV][R+1][Jh][2], NV = 7 (nonlinear) or 2 (linear only)
// ---------------------------------------------------------------------------
template <bool NONLIN, bool BIGP>
__global__ void swe_grid_kernel(PlanDev P, const double2* eo, long long eo_mstride, double2* x,
                                long long x_mstride, double omega, double radius) {
  constexpr int NIN = NONLIN ? 5 : 4;
  constexpr int NPROD = NONLIN ? 7 : 2;
  constexpr int NR = NONLIN ? 7 : 4;
  extern __shared__ __align__(16) double2 rings[];  // [NR][I]
  const int jh = blockIdx.x;
  const int m = blockIdx.y;
  const int I = P.I;
  const double2* e = eo + (size_t)m * eo_mstride;
  const size_t fstride = (size_t)(P.R + 1) * P.Jh * 2;
  zero_rings(rings, NIN * I);
  __syncthreads();
  for (int idx = threadIdx.x; idx < NIN * (P.R + 1); idx += blockDim.x) {
    const int q = idx / (P.R + 1), r = idx - q * (P.R + 1);
    const double2* src = e + q * fstride + ((size_t)r * P.Jh + jh) * 2;
    const double2 E = src[0], O = src[1];
    put_pair(rings + (size_t)q * I, P, r, make_double2(E.x + O.x, E.y + O.y),
             make_double2(E.x - O.x, E.y - O.y));
  }
  __syncthreads();
  fft_inverse<BIGP>(rings, NIN, P);

  const double mu = P.mu_n[jh];
  const double fn = 2.0 * omega * mu;         // f = 2 Omega mu (swe.py:178); south: -fn
  const double c2o = 2.0 * omega / radius;    // swe.py:179
  const double ic2 = 1.0 / (1.0 - mu * mu);   // swe.py:180
  for (int il = threadIdx.x; il < I; il += blockDim.x) {
    const double2 U = rings[il], V = rings[I + il], Z = rings[2 * I + il], D = rings[3 * I + il];
    // swe.py:262,265 : tend_zeta grid = -f delta - (2 Omega/a) V ; tend_delta grid = f zeta - (2 Omega/a) U
    rings[il] = make_double2(-fn * D.x - c2o * V.x, fn * D.y - c2o * V.y);
    rings[I + il] = make_double2(fn * Z.x - c2o * U.x, -fn * Z.y - c2o * U.y);
    if (NONLIN) {
      const double2 Ph = rings[4 * I + il];
      // swe.py:271-273 : Phi U, Phi V, zeta U, zeta V, KE = (U^2 + V^2) / (2 (1 - mu^2))
      rings[2 * I + il] = make_double2(Ph.x * U.x, Ph.y * U.y);
      rings[3 * I + il] = make_double2(Ph.x * V.x, Ph.y * V.y);
      rings[4 * I + il] = make_double2(Z.x * U.x, Z.y * U.y);
      rings[5 * I + il] = make_double2(Z.x * V.x, Z.y * V.y);
      rings[6 * I + il] = make_double2(0.5 * (U.x * U.x + V.x * V.x) * ic2,
                                       0.5 * (U.y * U.y + V.y * V.y) * ic2);
    }
  }
  __syncthreads();
  fft_forward<BIGP>(rings, NPROD, P);

  const bool eq = (jn_of(P, jh) == js_of(P, jh));
  const double w = P.w_n[jh];
  const double wc = w * ic2;
  const double ia = 1.0 / radius;
  double2* xm = x + (size_t)m * x_mstride;
  for (int r = threadIdx.x; r <= P.R; r += blockDim.x) {
    double2 A1n, A1s, A2n, A2s;
    get_pair(rings, P, r, A1n, A1s);
    get_pair(rings + I, P, r, A2n, A2s);
    double2* xo = xm + ((size_t)r * P.Jh + jh) * 2;
    if (!NONLIN) {
      put_sd(xo, cscale(A1n, w), cscale(A1s, w), eq);
      put_sd(xo + fstride, cscale(A2n, w), cscale(A2s, w), eq);
    } else {
      double2 PUn, PUs, PVn, PVs, ZUn, ZUs, ZVn, ZVs, Kn, Ks;
      get_pair(rings + 2 * I, P, r, PUn, PUs);
      get_pair(rings + 3 * I, P, r, PVn, PVs);
      get_pair(rings + 4 * I, P, r, ZUn, ZUs);
      get_pair(rings + 5 * I, P, r, ZVn, ZVs);
      get_pair(rings + 6 * I, P, r, Kn, Ks);
      const double rwa = r * wc * ia, wa = wc * ia;
      // P-vectors: phi, zeta, delta, ke ; H-vectors: phi, zeta, delta
      put_sd(xo, ir_scale(PUn, -rwa), ir_scale(PUs, -rwa), eq);
      put_sd(xo + fstride, cadd2(cscale(A1n, w), ir_scale(ZUn, -rwa)),
             cadd2(cscale(A1s, w), ir_scale(ZUs, -rwa)), eq);
      put_sd(xo + 2 * fstride, cadd2(cscale(A2n, w), ir_scale(ZVn, rwa)),
             cadd2(cscale(A2s, w), ir_scale(ZVs, rwa)), eq);
      put_sd(xo + 3 * fstride, cscale(Kn, w), cscale(Ks, w), eq);
      put_sd(xo + 4 * fstride, cscale(PVn, wa), cscale(PVs, wa), eq);
      put_sd(xo + 5 * fstride, cscale(ZVn, wa), cscale(ZVs, wa), eq);
      put_sd(xo + 6 * fstride, cscale(ZUn, wa), cscale(ZUs, wa), eq);
    }
  }
}

int pick_threads(int work, bool bigp) {
  if (bigp) return work >= 128 ? 128 : 64;
  if (work >= 512) return 256;
  if (work >= 128) return 128;
  return 64;
}

int set_smem(const void* kern, size_t smem) {
  if (smem > 227 * 1024) {
    set_error("longitude ring does not fit in shared memory (n_lon too large for this kernel)");
    return kUsage;
  }
  if (smem > 48 * 1024)
    SW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return kOk;
}

int pairs_per_cta(const PlanDev& P, int nin) {
  // keep the rings at <= ~96 KB so two CTAs fit per SM; at least one pair
  int np = (int)((96 * 1024) / ((size_t)nin * P.I * sizeof(double2)));
  if (np < 1) np = 1;
  if (np > 8) np = 8;
  if (np > P.Jh) np = P.Jh;
  return np;
}

template <bool BIGP>
int f2g_launch(const PlanDev& P, const double2* eo, long long eo_fstride, double* grid,
               long long grid_fstride, int nf, cudaStream_t st) {
  const int np = pairs_per_cta(P, 1);
  const size_t smem = sizeof(double2) * np * P.I;
  SW_TRY(set_smem((const void*)f2g_kernel<BIGP>, smem));
  dim3 gridDim((P.Jh + np - 1) / np, nf);
  StageScope sc("fourier_to_grid", st);
  f2g_kernel<BIGP><<<gridDim, pick_threads(np * P.I / 4, BIGP), smem, st>>>(P, eo, eo_fstride, grid,
                                                                       grid_fstride, np);
  SW_LAUNCH_CHECK();
  return kOk;
}

template <int MODE, bool BIGP>
int g2f_launch(const PlanDev& P, const double* grid, const double* grid2, long long grid_fstride,
               double2* x, long long x_fstride, int nf, cudaStream_t st) {
  const int nin = MODE == 0 ? 1 : 2;
  const int np = pairs_per_cta(P, nin);
  const size_t smem = sizeof(double2) * nin * np * P.I;
  dim3 gridDim((P.Jh + np - 1) / np, nf);
  SW_TRY(set_smem((const void*)g2f_kernel<MODE, BIGP>, smem));
  StageScope sc(MODE == 0 ? "grid_to_fourier" : "grid_to_fourier_divcurl", st);
  g2f_kernel<MODE, BIGP><<<gridDim, pick_threads(nin * np * P.I / 4, BIGP), smem, st>>>(
      P, grid, grid2, grid_fstride, x, x_fstride, np);
  SW_LAUNCH_CHECK();
  return kOk;
}

template <bool NONLIN, bool BIGP>
int swe_launch(const PlanDev& P, const double2* eo, long long eo_mstride, double2* x,
               long long x_mstride, int nmembers, double omega, double radius, cudaStream_t st) {
  const int nr = NONLIN ? 7 : 4;
  const size_t smem = sizeof(double2) * nr * P.I;
  dim3 gridDim(P.Jh, nmembers);
  SW_TRY(set_smem((const void*)swe_grid_kernel<NONLIN, BIGP>, smem));
  StageScope sc("swe_grid", st);
  swe_grid_kernel<NONLIN, BIGP><<<gridDim, pick_threads(nr * P.I / 4, BIGP), smem, st>>>(
      P, eo, eo_mstride, x, x_mstride, omega, radius);
  SW_LAUNCH_CHECK();
  return kOk;
}

}  // namespace

int launch_fourier_to_grid(const PlanDev& P, const double2* eo, long long eo_fstride, double* grid,
                           long long grid_fstride, int nf, cudaStream_t st) {
  if (swfft::fft_needs_bigp(P.I)) return f2g_launch<true>(P, eo, eo_fstride, grid, grid_fstride, nf, st);
  return f2g_launch<false>(P, eo, eo_fstride, grid, grid_fstride, nf, st);
}

int launch_grid_to_fourier(const PlanDev& P, int mode, const double* grid, const double* grid2,
                           long long grid_fstride, double2* x, long long x_fstride, int nf,
                           cudaStream_t st) {
  const bool big = swfft::fft_needs_bigp(P.I);
  if (mode == 0) {
    if (big) return g2f_launch<0, true>(P, grid, grid2, grid_fstride, x, x_fstride, nf, st);
    return g2f_launch<0, false>(P, grid, grid2, grid_fstride, x, x_fstride, nf, st);
  }
  if (big) return g2f_launch<1, true>(P, grid, grid2, grid_fstride, x, x_fstride, nf, st);
  return g2f_launch<1, false>(P, grid, grid2, grid_fstride, x, x_fstride, nf, st);
}

int launch_swe_grid(const PlanDev& P, bool nonlinear, const double2* eo, long long eo_mstride,
                    double2* x, long long x_mstride, int nmembers, double omega, double radius,
                    cudaStream_t st) {
  const bool big = swfft::fft_needs_bigp(P.I);
  if (nonlinear) {
    if (big) return swe_launch<true, true>(P, eo, eo_mstride, x, x_mstride, nmembers, omega, radius, st);
    return swe_launch<true, false>(P, eo, eo_mstride, x, x_mstride, nmembers, omega, radius, st);
  }
  if (big) return swe_launch<false, true>(P, eo, eo_mstride, x, x_mstride, nmembers, omega, radius, st);
  return swe_launch<false, false>(P, eo, eo_mstride, x, x_mstride, nmembers, omega, radius, st);
}

}  // namespace swsdc
