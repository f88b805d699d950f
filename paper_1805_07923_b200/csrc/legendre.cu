// Legendre stage of the SH transform on B200 (sm_100a), fp64.
//
// Replaces the reference's dense-table contractions
//   _contract_synthesis  F[r, j] = sum_s P[r, s, j] c[r, s]     (spharm.py:235-240)
//   _contract_analysis   c[r, s] = sum_j W[r, s, j] F[r, j]     (spharm.py:224-233)
// and the H-table variants used by synthesize_pair_cos_gradient and
// analyze_vector_div_curl (spharm.py:262-300).  Differences in HOW, not WHAT:
//
//  * No (R+1, R+1, J) tables.  Pbar_s^r(mu) is regenerated on the fly from the
//    three-term recurrence of spharm.py:160-168, rescaled so each step is one
//    DMUL + one DFMA:  q_s = mu q_{s-1} - beta_s q_{s-2},  P_s = g_s q_s,
//    beta_s = b_s / (a_s a_{s-1}),  g_s = prod a over the current chunk.
//    Chunks of kChunk degrees restart from checkpoint seeds (exact reference
//    values, see build_checkpoints) so work splits across warps / CTAs.
//  * Even/odd split: only the north half of the latitudes is visited; the
//    mirror latitude follows from Pbar(-mu) = (-1)^(s-r) Pbar(mu).
//  * H = (1-mu^2) dP/dmu is never formed: sum_s H_s c_s = sum_t P_t d_t with
//    d_t = (t+2) eps_{t+1} c_{t+1} - (t-1) eps_t c_{t-1} (synthesis) and
//    sum_j H_s y_j = (s+1) eps_s Y_{s-1} - s eps_{s+1} Y_{s+1} (analysis,
//    applied in spectral.cu), both from spharm.py:171-178.
//
// Synthesis: DFMA register kernel, each lane owns 2 latitudes and runs the
// recurrence in registers; coefficients are warp-uniform smem broadcasts.
// Analysis: the q tile (32 degrees x 128 latitudes) is generated into shared
// memory and contracted over latitude with FP64 tensor-core DMMA
// (mma.sync.m8n8k4.f64), so the latitude reduction happens inside the MMA.
#include "common.cuh"
#include "legendre.cuh"

namespace swsdc {

// ---------------------------------------------------------------------------
// Checkpoint seeds: the reference recurrence (spharm.py:153-169) evaluated
// with the reference's rounding order (no FMA contraction), one thread per
// north latitude; stores (P_{s0}, P_{s0+1} / a_{s0+1}) at every chunk start.
// ---------------------------------------------------------------------------
__global__ void build_checkpoints_kernel(PlanDev P, const double* a_tab, const double* b_tab,
                                         const double* sect_fac, double2* ckpt) {
  const int jh = blockIdx.x * blockDim.x + threadIdx.x;
  if (jh >= P.Jh) return;
  const double mu = P.mu_n[jh];
  const double u = __dsqrt_rn(__dsub_rn(1.0, __dmul_rn(mu, mu)));  // sqrt(1 - mu*mu)
  double sect = 0.70710678118654757;                                // 1/sqrt(2)
  for (int r = 0; r <= P.R; ++r) {
    const int nstep = P.R + 2 - r;  // degrees r .. R+1
    const double* ar = a_tab + (size_t)r * P.ldk;
    const double* br = b_tab + (size_t)r * P.ldk;
    const int off = P.ck_off[r];
    double pm1 = 0.0, pm2 = 0.0;
    for (int k = 0; k <= nstep; ++k) {
      double pk;
      if (k == 0) pk = sect;
      else if (k == 1) pk = __dmul_rn(__dmul_rn(mu, ar[1]), sect);
      else pk = __dsub_rn(__dmul_rn(__dmul_rn(ar[k], mu), pm1), __dmul_rn(br[k], pm2));
      if (k % kChunk == 1) {
        // chunk starting at k-1: seeds (P_{k-1}, P_k / a_k)
        ckpt[(size_t)(off + (k - 1) / kChunk) * P.Jh + jh] = make_double2(pm1, pk / ar[k]);
      }
      pm2 = pm1;
      pm1 = pk;
    }
    sect = __dmul_rn(__dmul_rn(sect, u), sect_fac[r]);
  }
}

int build_checkpoints(const PlanDev& P, const double* a_tab, const double* b_tab,
                      const double* sect_fac, double2* ckpt, cudaStream_t st) {
  const int threads = 64;
  StageScope sc("build_checkpoints", st);
  build_checkpoints_kernel<<<(P.Jh + threads - 1) / threads, threads, 0, st>>>(P, a_tab, b_tab,
                                                                               sect_fac, ckpt);
  SW_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// Synthesis
// ---------------------------------------------------------------------------
namespace {

constexpr int kSynWarps = 4;
constexpr int kSynNL = 2;  // latitudes per lane
constexpr int kSynLat = 32 * kSynNL;

__device__ __forceinline__ double2 fetch_coef(const double2* f, int srcR, int r, int s) {
  if (s < r || s > srcR || r > srcR) return make_double2(0.0, 0.0);
  return f[(size_t)r * (srcR + 1) + s];
}

// d_t = (t+2) eps_{t+1} c_{t+1} - (t-1) eps_t c_{t-1}: H-synthesis folded onto P.
__device__ __forceinline__ double2 h_fold(const double2* f, int srcR, int r, int t,
                                          const double* eps_r, double scale_hi, double scale_lo) {
  const double2 hi = fetch_coef(f, srcR, r, t + 1);
  const double2 lo = fetch_coef(f, srcR, r, t - 1);
  const double ch = (t + 2.0) * eps_r[t + 1] * scale_hi;
  const double cl = (t - 1.0) * eps_r[t] * scale_lo;
  return make_double2(ch * hi.x - cl * lo.x, ch * hi.y - cl * lo.y);
}

__device__ __forceinline__ double inv_lap(int s, double radius) {
  if (s == 0) return 0.0;
  const double lam = (-(double)s * (s + 1.0)) / (radius * radius);
  return 1.0 / lam;
}

template <int B, int MODE>
__device__ __forceinline__ void stage_coefs(const PlanDev& P, const SynArgs& a, int r, int nstep,
                                            int npad, double2* cs) {
  const double* eps_r = P.eps + (size_t)r * P.ldk;
  const double* g_r = P.gsc + (size_t)r * P.ldk;
  for (int idx = threadIdx.x; idx < B * npad; idx += blockDim.x) {
    const int b = idx / npad, k = idx - b * npad;
    double2 v = make_double2(0.0, 0.0);
    if (k < nstep) {
      const int s = r + k;
      if (MODE == kSynPlain) {
        v = fetch_coef(a.src + (size_t)b * a.src_fstride, a.src_R, r, s);
      } else if (MODE == kSynUV) {
        // U = i r chi - d(psi),  V = i r psi + d(chi)   (spharm.py:272-278)
        const double2* psi = a.src;
        const double2* chi = a.src2;
        if (b == 0) {
          const double2 c = fetch_coef(chi, a.src_R, r, s);
          const double2 h = h_fold(psi, a.src_R, r, s, eps_r, 1.0, 1.0);
          v = make_double2(-r * c.y - h.x, r * c.x - h.y);
        } else {
          const double2 c = fetch_coef(psi, a.src_R, r, s);
          const double2 h = h_fold(chi, a.src_R, r, s, eps_r, 1.0, 1.0);
          v = make_double2(-r * c.y + h.x, r * c.x + h.y);
        }
      } else {  // kSynSWE: state (phi, zeta, delta) -> U/a, V/a, zeta, delta, phi
        const double2* phi = a.src;
        const double2* zeta = a.src + a.src_fstride;
        const double2* delta = a.src + 2 * a.src_fstride;
        const double ia = 1.0 / a.radius;
        if (b < 2) {
          // psi = invlap(zeta), chi = invlap(delta)  (swe.py:186-187), then 1/a (swe.py:189)
          const double2* fpsi = zeta;
          const double2* fchi = delta;
          const double2 cmain = fetch_coef(b == 0 ? fchi : fpsi, a.src_R, r, s);
          const double smain = inv_lap(s, a.radius) * ia;
          const double2 hh = h_fold(b == 0 ? fpsi : fchi, a.src_R, r, s, eps_r,
                                    inv_lap(s + 1, a.radius) * ia, inv_lap(s - 1 < 0 ? 0 : s - 1, a.radius) * ia);
          const double sg = (b == 0) ? -1.0 : 1.0;
          v = make_double2(-r * cmain.y * smain + sg * hh.x, r * cmain.x * smain + sg * hh.y);
        } else if (b == 2) {
          v = fetch_coef(zeta, a.src_R, r, s);
        } else if (b == 3) {
          v = fetch_coef(delta, a.src_R, r, s);
        } else {
          v = fetch_coef(phi, a.src_R, r, s);
        }
      }
      const double g = g_r[k];
      v.x *= g;
      v.y *= g;
    }
    cs[idx] = v;
  }
}

template <int B, int MODE>
__global__ void __launch_bounds__(kSynWarps * 32)
syn_kernel(PlanDev P, SynArgs a) {
  extern __shared__ __align__(16) double smem[];
  a.src += (size_t)blockIdx.y * a.src_mstride;
  if (a.src2) a.src2 += (size_t)blockIdx.y * a.src_mstride;
  a.eo += (size_t)blockIdx.y * a.eo_mstride;
  const int r = blockIdx.x / a.nJB;
  const int jb = blockIdx.x - r * a.nJB;
  const int nstep = a.smax - r + 1;
  const int npad = ((nstep + 1) & ~1) + 2;
  double2* cs = reinterpret_cast<double2*>(smem);              // [B][npad]
  double* bs = reinterpret_cast<double*>(cs + B * npad);       // [npad + kChunk + 4]
  double2* red = reinterpret_cast<double2*>(bs + npad + kChunk + 4);  // [B][kSynLat][2]

  stage_coefs<B, MODE>(P, a, r, nstep, npad, cs);
  const double* beta_r = P.beta + (size_t)r * P.ldk;
  for (int k = threadIdx.x; k < npad + kChunk + 4; k += blockDim.x) bs[k] = beta_r[k];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int jh[kSynNL];
  double mu[kSynNL];
#pragma unroll
  for (int l = 0; l < kSynNL; ++l) {
    jh[l] = jb * kSynLat + lane + 32 * l;
    mu[l] = (jh[l] < P.Jh) ? P.mu_n[jh[l]] : 0.0;
  }
  double2 E[B][kSynNL], O[B][kSynNL];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int l = 0; l < kSynNL; ++l) { E[b][l] = make_double2(0.0, 0.0); O[b][l] = E[b][l]; }

  const int nchunk = (nstep + kChunk - 1) / kChunk;
  const int off = P.ck_off[r];
  for (int c = warp; c < nchunk; c += kSynWarps) {
    const int k0 = c * kChunk;
    const int kend = min(k0 + kChunk, nstep);
    double qa[kSynNL], qb[kSynNL];
#pragma unroll
    for (int l = 0; l < kSynNL; ++l) {
      double2 sd = make_double2(0.0, 0.0);
      if (jh[l] < P.Jh) sd = P.ckpt[(size_t)(off + c) * P.Jh + jh[l]];
      qa[l] = sd.x;
      qb[l] = sd.y;
    }
#pragma unroll 2
    for (int k = k0; k < kend; k += 2) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const double2 ce = cs[b * npad + k];
        const double2 co = cs[b * npad + k + 1];
#pragma unroll
        for (int l = 0; l < kSynNL; ++l) {
          E[b][l].x = fma(qa[l], ce.x, E[b][l].x);
          E[b][l].y = fma(qa[l], ce.y, E[b][l].y);
          O[b][l].x = fma(qb[l], co.x, O[b][l].x);
          O[b][l].y = fma(qb[l], co.y, O[b][l].y);
        }
      }
      const double2 bb = *reinterpret_cast<const double2*>(bs + k + 2);
#pragma unroll
      for (int l = 0; l < kSynNL; ++l) {
        qa[l] = fma(mu[l], qb[l], -bb.x * qa[l]);
        qb[l] = fma(mu[l], qa[l], -bb.y * qb[l]);
      }
    }
  }

  // deterministic cross-warp reduction (fixed warp order)
  for (int w = 0; w < kSynWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int l = 0; l < kSynNL; ++l) {
          double2* d = red + ((size_t)b * kSynLat + lane + 32 * l) * 2;
          if (w == 0) {
            d[0] = E[b][l];
            d[1] = O[b][l];
          } else {
            d[0].x += E[b][l].x; d[0].y += E[b][l].y;
            d[1].x += O[b][l].x; d[1].y += O[b][l].y;
          }
        }
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < B * kSynLat; idx += blockDim.x) {
    const int b = idx / kSynLat, lj = idx - b * kSynLat;
    const int j = jb * kSynLat + lj;
    if (j < P.Jh) {
      double2* o = a.eo + (((size_t)b * (P.R + 1) + r) * P.Jh + j) * 2;
      o[0] = red[(size_t)idx * 2];
      o[1] = red[(size_t)idx * 2 + 1];
    }
  }
}

template <int B, int MODE>
int launch_syn_t(const PlanDev& P, const SynArgs& a0, cudaStream_t st) {
  SynArgs a = a0;
  a.nJB = (P.Jh + kSynLat - 1) / kSynLat;
  const int npad_max = ((a.smax + 2) & ~1) + 2;
  const size_t smem = sizeof(double2) * B * npad_max + sizeof(double) * (npad_max + kChunk + 4) +
                      sizeof(double2) * 2 * B * kSynLat;
  auto kern = syn_kernel<B, MODE>;
  if (smem > 48 * 1024) SW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  StageScope sc("legendre_synthesis", st);
  kern<<<dim3((P.R + 1) * a.nJB, a.nmembers), kSynWarps * 32, smem, st>>>(P, a);
  SW_LAUNCH_CHECK();
  return kOk;
}

}  // namespace

int launch_synthesis(const PlanDev& P, const SynArgs& a, int B, int mode, cudaStream_t st) {
  if (mode == kSynUV) return launch_syn_t<2, kSynUV>(P, a, st);
  if (mode == kSynSWE) return launch_syn_t<5, kSynSWE>(P, a, st);
  switch (B) {
    case 1: return launch_syn_t<1, kSynPlain>(P, a, st);
    case 2: return launch_syn_t<2, kSynPlain>(P, a, st);
    case 3: return launch_syn_t<3, kSynPlain>(P, a, st);
    case 4: return launch_syn_t<4, kSynPlain>(P, a, st);
    case 5: return launch_syn_t<5, kSynPlain>(P, a, st);
    case 6: return launch_syn_t<6, kSynPlain>(P, a, st);
    case 7: return launch_syn_t<7, kSynPlain>(P, a, st);
    case 8: return launch_syn_t<8, kSynPlain>(P, a, st);
  }
  set_error("synthesis batch per launch must be 1..8");
  return kUsage;
}

// ---------------------------------------------------------------------------
// Analysis (DMMA)
// ---------------------------------------------------------------------------
namespace {

constexpr int kAnaThreads = 128;
constexpr int kAnaJC = 128;               // latitudes per smem tile
constexpr int kAnaQS = kAnaJC + 4;        // q-tile row stride (doubles), == 4 mod 16

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(kAnaThreads)
ana_kernel(PlanDev P, AnaArgs a) {
  constexpr int XS = 8 * NT + 4;  // x-tile row stride (doubles)
  extern __shared__ __align__(16) double smem[];
  double* qs = smem;                          // [32][kAnaQS]   rows ordered (parity, k/2)
  double* xs = qs + 32 * kAnaQS;              // [2][kAnaJC][XS]  parity 0: S, 1: D
  double* bs = xs + 2 * kAnaJC * XS;          // [kChunk]

  a.x += (size_t)blockIdx.y * a.x_mstride;
  a.out += (size_t)blockIdx.y * a.out_mstride;
  const int2 wk = a.work[blockIdx.x];
  const int r = wk.x, c = wk.y;
  const int k0 = c * kChunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int par = warp & 1, half = warp >> 1;

  for (int i = tid; i < kChunk; i += kAnaThreads) bs[i] = P.beta[(size_t)r * P.ldk + k0 + i];
  // zero the padding columns once
  for (int i = tid; i < 2 * kAnaJC * XS; i += kAnaThreads) xs[i] = 0.0;

  double acc[NT][2];
#pragma unroll
  for (int n = 0; n < NT; ++n) { acc[n][0] = 0.0; acc[n][1] = 0.0; }

  const int off = P.ck_off[r];
  const size_t xrow = (size_t)(P.R + 1) * P.Jh * 2;  // per-vector stride in double2
  for (int jc0 = 0; jc0 < P.Jh; jc0 += kAnaJC) {
    __syncthreads();
    // stage x (S, D) for nv vectors
    for (int idx = tid; idx < kAnaJC * a.nv; idx += kAnaThreads) {
      const int v = idx / kAnaJC, jl = idx - v * kAnaJC;
      const int j = jc0 + jl;
      double2 S = make_double2(0.0, 0.0), D = S;
      if (j < P.Jh) {
        const double2* src = a.x + v * xrow + ((size_t)r * P.Jh + j) * 2;
        S = src[0];
        D = src[1];
      }
      double* x0 = xs + (size_t)jl * XS + 2 * v;
      double* x1 = xs + (size_t)(kAnaJC + jl) * XS + 2 * v;
      x0[0] = S.x; x0[1] = S.y;
      x1[0] = D.x; x1[1] = D.y;
    }
    // generate the q tile for degrees k0 .. k0+31 at latitudes jc0 .. jc0+127
    for (int jl = tid; jl < kAnaJC; jl += kAnaThreads) {
      const int j = jc0 + jl;
      if (j < P.Jh) {
        const double mu = P.mu_n[j];
        const double2 sd = P.ckpt[(size_t)(off + c) * P.Jh + j];
        double qa = sd.x, qb = sd.y;
        qs[0 * kAnaQS + jl] = qa;
        qs[16 * kAnaQS + jl] = qb;
#pragma unroll
        for (int kk = 2; kk < kChunk; kk += 2) {
          qa = fma(mu, qb, -bs[kk] * qa);
          qb = fma(mu, qa, -bs[kk + 1] * qb);
          qs[(kk >> 1) * kAnaQS + jl] = qa;
          qs[(16 + (kk >> 1)) * kAnaQS + jl] = qb;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < kChunk; ++kk) qs[((kk & 1) * 16 + (kk >> 1)) * kAnaQS + jl] = 0.0;
      }
    }
    __syncthreads();
    const double* qrow = qs + (size_t)(par * 16 + half * 8 + g) * kAnaQS + t;
    const double* xcol = xs + (size_t)(par * kAnaJC + t) * XS + g;
#pragma unroll 4
    for (int j0 = 0; j0 < kAnaJC; j0 += 4) {
      const double av = qrow[j0];
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const double bv = xcol[(size_t)j0 * XS + n * 8];
        dmma884(acc[n], av, bv);
      }
    }
  }

  // epilogue: rows k = k0 + par + 2*(8 half + g), cols (re, im) of vector n*4 + t
  const int k = k0 + par + 2 * (8 * half + g);
  const int nout = a.smax - r + 1;
  if (k < nout) {
    const double gs = P.gsc[(size_t)r * P.ldk + k];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int v = n * 4 + t;
      if (v < a.nv) {
        double2 val = make_double2(acc[n][0] * gs, acc[n][1] * gs);
        a.out[(size_t)v * a.out_vstride + (size_t)r * a.out_rstride + r + k] = val;
      }
    }
  }
  if (a.zero_fill && c == 0) {
    for (int idx = tid; idx < a.nv * r; idx += kAnaThreads) {
      const int v = idx / r, s = idx - v * r;
      a.out[(size_t)v * a.out_vstride + (size_t)r * a.out_rstride + s] = make_double2(0.0, 0.0);
    }
  }
}

template <int NT>
int launch_ana_t(const PlanDev& P, const AnaArgs& a, int nwork, cudaStream_t st) {
  constexpr int XS = 8 * NT + 4;
  const size_t smem = sizeof(double) * (32 * kAnaQS + 2 * kAnaJC * XS + kChunk);
  auto kern = ana_kernel<NT>;
  if (smem > 48 * 1024) SW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  StageScope sc("legendre_analysis", st);
  kern<<<dim3(nwork, a.nmembers), kAnaThreads, smem, st>>>(P, a);
  SW_LAUNCH_CHECK();
  return kOk;
}

}  // namespace

int launch_analysis(const PlanDev& P, const AnaArgs& a, int nwork, cudaStream_t st) {
  if (a.nv <= 0) return kOk;
  if (a.nv <= 4) return launch_ana_t<1>(P, a, nwork, st);
  if (a.nv <= 8) return launch_ana_t<2>(P, a, nwork, st);
  if (a.nv <= 16) return launch_ana_t<4>(P, a, nwork, st);
  set_error("analysis vectors per launch must be <= 16");
  return kUsage;
}

}  // namespace swsdc
