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
// recurrence in registers; coefficients are warp-uniform smem broadcasts from a
// warp-private slab refilled chunk by chunk.
// Analysis: the q tile (32 degrees x 128 latitudes) is generated into shared
// memory and contracted over latitude with FP64 tensor-core DMMA
// (mma.sync.m8n8k4.f64), so the latitude reduction happens inside the MMA.
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "legendre.cuh"

namespace swsdc {
#ifdef ANA_TRACE
// debug build only (tools/ana_trace.py): per-warp %globaltimer stamps of the
// analysis phases, read back with swsdc_debug_ana_trace
__device__ unsigned long long g_ana_trace[16384][8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define ANA_STAMP(k) do { if ((threadIdx.x & 31) == 0) { const int wid_ = (blockIdx.y * gridDim.x + blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); if (wid_ < 16384) g_ana_trace[wid_][k] = gtime(); } } while (0)
#else
#define ANA_STAMP(k) do {} while (0)
#endif

// ---------------------------------------------------------------------------
// Checkpoint seeds: the reference recurrence (spharm.py:153-169) evaluated
// with the reference's rounding order (no FMA contraction), one thread per
// north latitude; stores (P_{s0}, P_{s0+1} / a_{s0+1}) at every chunk start.
// ---------------------------------------------------------------------------
__global__ void build_checkpoints_kernel(PlanDev P, const double* a_tab, const double* b_tab,
                                         const double* sect_fac, double2* ckpt) {
  pdl_wait();
  pdl_trigger();
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
  SW_CUDA(launch_pdl(build_checkpoints_kernel, dim3((P.Jh + threads - 1) / threads), dim3(threads), 0, st, P, a_tab, b_tab, sect_fac, ckpt));
  SW_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// Pbar table for the table-fed analysis: the same reference recurrence,
// one thread per (north latitude, r), every degree r .. R+1 stored in the
// analysis A-fragment order -- per (chunk ck = ck_off[r] + (s-r)/32, 4-latitude
// block jb): [parity p][m-tile mt][lane = 4 g + t] = Pbar at degree
// s = r + 32 c + p + 2 (8 mt + g) and latitude jh = 4 jb + t.  Entries past
// R+1 or Jh stay zero (the buffer is zeroed first).
// ---------------------------------------------------------------------------
__global__ void build_ptab_kernel(PlanDev P, const double* a_tab, const double* b_tab,
                                  const double* sect_fac, double* ptab, int syn) {
  pdl_wait();
  pdl_trigger();
  const int jh = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (jh >= P.Jh || r > P.R) return;
  const double mu = P.mu_n[jh];
  const double u = __dsqrt_rn(__dsub_rn(1.0, __dmul_rn(mu, mu)));
  double sect = 0.70710678118654757;   // 1/sqrt(2), then the sectoral chain to row r
  for (int q = 0; q < r; ++q) sect = __dmul_rn(__dmul_rn(sect, u), sect_fac[q]);
  const double* ar = a_tab + (size_t)r * P.ldk;
  const double* br = b_tab + (size_t)r * P.ldk;
  const int jh4 = (P.Jh + 3) >> 2, jb = jh >> 2, tt = jh & 3;
  const int nlb = (P.Jh + 31) >> 5, lb = jh >> 5, lt = (jh >> 3) & 3, gg = jh & 7;
  double pm1 = 0.0, pm2 = 0.0;
  for (int k = 0; k <= P.R + 1 - r; ++k) {
    double pk;
    if (k == 0) pk = sect;
    else if (k == 1) pk = __dmul_rn(__dmul_rn(mu, ar[1]), sect);
    else pk = __dsub_rn(__dmul_rn(__dmul_rn(ar[k], mu), pm1), __dmul_rn(br[k], pm2));
    const int c = k >> 5, kk = k & 31, pp = kk & 1, i = kk >> 1;
    const size_t ck = (size_t)P.ck_off[r] + c;
    if (!syn) {
      // analysis A fragment: [p][m-tile i/8][lane = 4 (i%8) + t], latitude t of block jb
      const int lane = ((i & 7) << 2) | tt;
      ptab[((ck * jh4 + jb) << 7) + ((pp << 1) | (i >> 3)) * 32 + lane] = pk;
    } else {
      // synthesis B fragment: k-step (p, q = i/4), latitude tile lt, lane = 4 g + (i%4)
      ptab[(((ck * nlb + lb) * 8 + (pp * 4 + (i >> 2))) << 7) + lt * 32 + (gg << 2) + (i & 3)] = pk;
    }
    pm2 = pm1;
    pm1 = pk;
  }
}

int build_ptab(const PlanDev& P, const double* a_tab, const double* b_tab, const double* sect_fac,
               double* ptab, cudaStream_t st, int syn) {
  const int threads = 64;
  StageScope sc("build_ptab", st);
  SW_CUDA(launch_pdl(build_ptab_kernel, dim3((P.Jh + threads - 1) / threads, P.R + 1), dim3(threads),
                     0, st, P, a_tab, b_tab, sect_fac, ptab, syn));
  SW_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// Synthesis
//
// One CTA per (r-pair {p, R-p}, latitude group of 64, member): the pair folds
// the triangular work so every CTA carries R+4 recurrence steps.  NSPLIT warps
// share the pair's chunks (a warp never straddles the two rows); each warp is
// autonomous: lane l stages degree k0+l of its chunk (coefficients already
// scaled by g, for B fields) into a warp-private smem slab while the next
// chunk's coefficients, betas and seeds are in flight in registers.  Lanes own
// 2 latitudes each; E/O accumulators stay in registers until the row ends.
// ---------------------------------------------------------------------------
namespace {

constexpr int kSynNL = 2;            // latitudes per lane
constexpr int kSynLat = 32 * kSynNL; // latitudes per latitude group
constexpr int kCS = kChunk + 2;      // staged degrees per chunk (+2 for the pair loop)

__device__ __forceinline__ double2 fetch_coef(const double2* f, int srcR, int r, int s) {
  if (s < r || s > srcR || r > srcR) return make_double2(0.0, 0.0);
  return f[(size_t)r * (srcR + 1) + s];
}

// (1 / lambda_s) / a = -a / (s (s + 1)), lambda_s = -s (s + 1) / a^2 (swe.py:186-189,
// spharm.py:321-333, s = 0 gauged to 0): one division instead of the two of
// forming lambda_s and inverting it
__device__ __forceinline__ double inv_lap_a(int s, double radius) {
  if (s <= 0) return 0.0;
  return -radius / ((double)s * (s + 1.0));
}

// Raw per-lane loads of one chunk (degree s = r + k0 + lane) kept in registers
// while the previous chunk computes; all arithmetic on them is deferred to
// stage_chunk so the loads stay in flight.
//   plain: c_b(s) for B fields
//   UV   : psi, chi at s, s+1, s-1
//   SWE  : zeta, delta at s, s+1, s-1 and phi' at s
template <int B, int MODE>
struct ChunkRegs {
  static constexpr int NRAW = MODE == kSynPlain ? B : (MODE == kSynUV ? 6 : 7);
  double2 raw[NRAW];
  double eps0, eps1, g;    // eps_s, eps_{s+1}, chunk scale g
  double beta, beta_x;     // beta[k0 + lane], beta[k0 + 32 + lane] (lanes 0, 1)
  double2 seed[kSynNL];
};

template <int B, int MODE>
__device__ __forceinline__ void load_chunk(ChunkRegs<B, MODE>& c, const PlanDev& P, const SynArgs& a,
                                           int r, int ci, int nstep, int lane, const int* jh,
                                           int off_r) {
  const int k0 = ci * kChunk;
  const int k = k0 + lane, s = r + k;
  const double* b_r = P.beta + (size_t)r * P.ldk;
  const double* e_r = P.eps + (size_t)r * P.ldk;
  c.g = P.gsc[(size_t)r * P.ldk + k];
  c.eps0 = e_r[s];
  c.eps1 = e_r[s + 1];
  if (MODE == kSynPlain) {
#pragma unroll
    for (int b = 0; b < B; ++b) c.raw[b] = fetch_coef(a.src + (size_t)b * a.src_fstride, a.src_R, r, s);
  } else if (MODE == kSynUV) {
    const double2* f0 = a.src;   // psi
    const double2* f1 = a.src2;  // chi
    c.raw[0] = fetch_coef(f0, a.src_R, r, s);
    c.raw[1] = fetch_coef(f1, a.src_R, r, s);
    c.raw[2] = fetch_coef(f0, a.src_R, r, s + 1);
    c.raw[3] = fetch_coef(f0, a.src_R, r, s - 1);
    c.raw[4] = fetch_coef(f1, a.src_R, r, s + 1);
    c.raw[5] = fetch_coef(f1, a.src_R, r, s - 1);
  } else {
    const double2* zeta = a.src + a.src_fstride;
    const double2* delta = a.src + 2 * a.src_fstride;
    c.raw[0] = fetch_coef(zeta, a.src_R, r, s);
    c.raw[1] = fetch_coef(delta, a.src_R, r, s);
    c.raw[2] = fetch_coef(zeta, a.src_R, r, s + 1);
    c.raw[3] = fetch_coef(zeta, a.src_R, r, s - 1);
    c.raw[4] = fetch_coef(delta, a.src_R, r, s + 1);
    c.raw[5] = fetch_coef(delta, a.src_R, r, s - 1);
    c.raw[6] = fetch_coef(a.src, a.src_R, r, s);
  }
  // degrees past the row end need no masking: fetch_coef returns 0 for s > R_in
  (void)nstep;
  c.beta = b_r[k];
  c.beta_x = (lane < 2) ? b_r[k + kChunk] : 0.0;
  const int off = off_r + ci;
#pragma unroll
  for (int l = 0; l < kSynNL; ++l)
    c.seed[l] = (jh[l] < P.Jh) ? P.ckpt[(size_t)off * P.Jh + jh[l]] : make_double2(0.0, 0.0);
}

// d_t = (t+2) eps_{t+1} c_{t+1} - (t-1) eps_t c_{t-1}: H-synthesis folded onto P.
__device__ __forceinline__ double2 hfold(double2 hi, double2 lo, double e0, double e1, int t,
                                         double shi, double slo) {
  const double ch = (t + 2.0) * e1 * shi, cl = (t - 1.0) * e0 * slo;
  return make_double2(ch * hi.x - cl * lo.x, ch * hi.y - cl * lo.y);
}

// Coefficients of the B synthesis fields at degree s = r + k0 + lane, scaled
// by g, written to the warp's slab cs[b][lane].
// TBL: 1 / (s (s + 1)) from the plan table (no division); measured faster in
// the split (NSPLIT > 1) kernels, while in the NSPLIT = 1 kernel the divisions'
// scheduling barrier keeps the register count (and occupancy) lower.
template <int B, int MODE, bool TBL>
__device__ __forceinline__ void stage_chunk(const ChunkRegs<B, MODE>& c, double2* cs, int r,
                                            int s, double radius, const double* ilap, int lane) {
  double2 v[B];
  if (MODE == kSynPlain) {
#pragma unroll
    for (int b = 0; b < B; ++b) v[b] = c.raw[b];
  } else if (MODE == kSynUV) {
    // U = i r chi - d(psi),  V = i r psi + d(chi)   (spharm.py:272-278)
    const double2 hp = hfold(c.raw[2], c.raw[3], c.eps0, c.eps1, s, 1.0, 1.0);
    const double2 hc = hfold(c.raw[4], c.raw[5], c.eps0, c.eps1, s, 1.0, 1.0);
    v[0] = make_double2(-r * c.raw[1].y - hp.x, r * c.raw[1].x - hp.y);
    v[1] = make_double2(-r * c.raw[0].y + hc.x, r * c.raw[0].x + hc.y);
  } else {
    // psi = invlap(zeta), chi = invlap(delta) (swe.py:186-187), then 1/a (swe.py:189):
    // (1 / lambda_s) / a = -a / (s (s + 1)), lambda_s = -s (s + 1) / a^2
    // (spharm.py:321-333, s = 0 gauged to 0), from the plan table, no division
    // (table read at staging time, not prefetched: it is tiny and L1-resident)
    double s0, sp, sm;
    if (TBL) {
      s0 = -radius * ilap[s];
      sp = -radius * ilap[s + 1];
      sm = s >= 1 ? -radius * ilap[s - 1] : 0.0;
    } else if (s >= 2) {
      // one division for the three scales: q = (s-1) s (s+1) (s+2) is exact in
      // fp64 (s <= ~1300), then -a / (s (s+1)) = -a (s-1)(s+2) / q etc. (each one
      // product more than the direct quotient: <= 1 ulp); three divisions were
      // ~20% of this kernel's stall samples at T1279 (profiles/r02)
      const double q = (double)(s - 1) * (double)s * (s + 1.0) * (s + 2.0);
      const double inv = -radius / q;
      s0 = ((s - 1.0) * (s + 2.0)) * inv;
      sp = ((s - 1.0) * (double)s) * inv;
      sm = ((s + 1.0) * (s + 2.0)) * inv;
    } else {
      s0 = inv_lap_a(s, radius);
      sp = inv_lap_a(s + 1, radius);
      sm = inv_lap_a(s - 1, radius);
    }
    const double2 hpsi = hfold(c.raw[2], c.raw[3], c.eps0, c.eps1, s, sp, sm);
    const double2 hchi = hfold(c.raw[4], c.raw[5], c.eps0, c.eps1, s, sp, sm);
    v[0] = make_double2(-r * c.raw[1].y * s0 - hpsi.x, r * c.raw[1].x * s0 - hpsi.y);  // U/a
    v[1] = make_double2(-r * c.raw[0].y * s0 + hchi.x, r * c.raw[0].x * s0 + hchi.y);  // V/a
    v[2] = c.raw[0];
    v[3] = c.raw[1];
    v[4] = c.raw[6];
  }
#pragma unroll
  for (int b = 0; b < B; ++b) {
    cs[b * kCS + lane] = make_double2(v[b].x * c.g, v[b].y * c.g);
    if (lane < 2) cs[b * kCS + kChunk + lane] = make_double2(0.0, 0.0);
  }
}

// (E, O) of one (field, row, latitude pair): one 32-byte sector, written with one
// 256-bit store (two 16-byte stores would pass the LSU data stage twice)
__device__ __forceinline__ void st_eo(double2* p, double2 e, double2 o) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "d"(e.x), "d"(e.y), "d"(o.x), "d"(o.y) : "memory");
}

template <int B>
__device__ __forceinline__ void flush_row(double2 (&E)[B][kSynNL], double2 (&O)[B][kSynNL],
                                          double2* dst, int lane) {
  // dst: [B][kSynLat][2] (E, O) slab
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int l = 0; l < kSynNL; ++l) {
      double2* d = dst + ((size_t)b * kSynLat + lane + 32 * l) * 2;
      d[0] = E[b][l];
      d[1] = O[b][l];
      E[b][l] = make_double2(0.0, 0.0);
      O[b][l] = make_double2(0.0, 0.0);
    }
}

template <int B, int MODE, int NSPLIT>
__global__ void __launch_bounds__(NSPLIT * 32)
syn_kernel(PlanDev P, SynArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* cs = reinterpret_cast<double2*>(smem) + (size_t)warp * B * kCS;        // [B][kCS]
  double* bs = reinterpret_cast<double*>(reinterpret_cast<double2*>(smem) + NSPLIT * B * kCS) +
               (size_t)warp * kCS;                                               // [kCS]
  double2* red = reinterpret_cast<double2*>(smem) + NSPLIT * B * kCS + (NSPLIT * kCS + 1) / 2;

  a.src += (size_t)blockIdx.z * a.src_mstride;
  if (a.src2) a.src2 += (size_t)blockIdx.z * a.src_mstride;
  a.eo += (size_t)blockIdx.z * a.eo_mstride;

  const int p = blockIdx.x, lg = blockIdx.y;
  const int2 pr = a.pairs ? a.pairs[p] : make_int2(p, P.R - p);
  const int rows[2] = {pr.x, pr.y};
  const bool two = rows[1] > rows[0];
  int nst[2], nch[2];
  for (int i = 0; i < 2; ++i) {
    nst[i] = (i == 0 || two) ? a.smax - rows[i] + 1 : 0;
    nch[i] = (nst[i] + kChunk - 1) / kChunk;
  }
  // warps -> (row, chunk range); a warp never straddles the rows
  int wrow = 0, cb = 0, ce = 0;
  int w1 = NSPLIT;   // warps [0, w1) take row 0, [w1, NSPLIT) row 1
  if (NSPLIT == 1) {
    wrow = -1;  // the single warp walks both rows
  } else {
    w1 = two ? (NSPLIT * nch[0] + (nch[0] + nch[1]) / 2) / (nch[0] + nch[1]) : NSPLIT;
    w1 = max(1, min(w1, two ? NSPLIT - 1 : NSPLIT));
    if (warp < w1) {
      wrow = 0;
      cb = warp * nch[0] / w1;
      ce = (warp + 1) * nch[0] / w1;
    } else {
      wrow = 1;
      const int w2 = NSPLIT - w1, ww = warp - w1;
      cb = ww * nch[1] / w2;
      ce = (ww + 1) * nch[1] / w2;
    }
  }

  int jh[kSynNL];
  double mu[kSynNL];
#pragma unroll
  for (int l = 0; l < kSynNL; ++l) {
    jh[l] = lg * kSynLat + lane + 32 * l;
    mu[l] = (jh[l] < P.Jh) ? P.mu_n[jh[l]] : 0.0;
  }
  double2 E[B][kSynNL], O[B][kSynNL];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int l = 0; l < kSynNL; ++l) { E[b][l] = make_double2(0.0, 0.0); O[b][l] = E[b][l]; }

  const int irow0 = (NSPLIT == 1) ? 0 : wrow;
  const int irow1 = (NSPLIT == 1) ? (two ? 1 : 0) : wrow;
  for (int ir = irow0; ir <= irow1; ++ir) {
    const int r = rows[ir], nstep = nst[ir];
    const int c0 = (NSPLIT == 1) ? 0 : cb, c1 = (NSPLIT == 1) ? nch[ir] : ce;
    if (c0 < c1) {
      const int off_r = P.ck_off[r];
      ChunkRegs<B, MODE> nx;
      load_chunk<B, MODE>(nx, P, a, r, c0, nstep, lane, jh, off_r);
      for (int ci = c0; ci < c1; ++ci) {
        __syncwarp();
        stage_chunk<B, MODE, (NSPLIT > 1)>(nx, cs, r, r + ci * kChunk + lane, a.radius, P.ilap, lane);
        bs[lane] = nx.beta;
        if (lane < 2) bs[kChunk + lane] = nx.beta_x;
        double qa[kSynNL], qb[kSynNL];
#pragma unroll
        for (int l = 0; l < kSynNL; ++l) { qa[l] = nx.seed[l].x; qb[l] = nx.seed[l].y; }
        __syncwarp();
        if (ci + 1 < c1) load_chunk<B, MODE>(nx, P, a, r, ci + 1, nstep, lane, jh, off_r);
        const int kn = min(kChunk, nstep - ci * kChunk);
#pragma unroll 4   // measured: 2 -> 4 saves 4.5%, 8 is slower
        for (int kk = 0; kk < kn; kk += 2) {
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const double2 ce_ = cs[b * kCS + kk];
            const double2 co_ = cs[b * kCS + kk + 1];
#pragma unroll
            for (int l = 0; l < kSynNL; ++l) {
              E[b][l].x = fma(qa[l], ce_.x, E[b][l].x);
              E[b][l].y = fma(qa[l], ce_.y, E[b][l].y);
              O[b][l].x = fma(qb[l], co_.x, O[b][l].x);
              O[b][l].y = fma(qb[l], co_.y, O[b][l].y);
            }
          }
          const double2 bb = *reinterpret_cast<const double2*>(bs + kk + 2);
#pragma unroll
          for (int l = 0; l < kSynNL; ++l) {
            qa[l] = fma(mu[l], qb[l], -bb.x * qa[l]);
            qb[l] = fma(mu[l], qa[l], -bb.y * qb[l]);
          }
        }
      }
    }
    if (NSPLIT == 1) {
      // sole owner of the row: write (E, O) straight out
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int l = 0; l < kSynNL; ++l) {
          if (jh[l] < P.Jh) {
            double2* o = a.eo + (((size_t)b * (P.R + 1) + r) * P.Jh + jh[l]) * 2;
            st_eo(o, E[b][l], O[b][l]);
          }
          E[b][l] = make_double2(0.0, 0.0);
          O[b][l] = make_double2(0.0, 0.0);
        }
    }
  }
  if (NSPLIT > 1) {
    // deterministic reduction of the warps' partial rows (fixed warp order),
    // per row: a row owned by one warp is written straight out; the warps of
    // a shared row meet at a named barrier of their own (1 + row) and split
    // the summation, so neither waits for the other row's warps
    const int wb = wrow == 0 ? 0 : w1, we = wrow == 0 ? w1 : NSPLIT;
    const int nrw = we - wb;
    const int r = rows[wrow];
    if (nrw == 1) {
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int l = 0; l < kSynNL; ++l)
          if (jh[l] < P.Jh) {
            double2* o = a.eo + (((size_t)b * (P.R + 1) + r) * P.Jh + jh[l]) * 2;
            st_eo(o, E[b][l], O[b][l]);
          }
      return;
    }
    flush_row<B>(E, O, red + (size_t)warp * B * kSynLat * 2, lane);
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wrow), "r"(32 * nrw) : "memory");
    for (int idx = (warp - wb) * 32 + lane; idx < B * kSynLat; idx += 32 * nrw) {
      const int b = idx / kSynLat, lj = idx - b * kSynLat;
      const int j = lg * kSynLat + lj;
      if (j >= P.Jh) continue;
      double2 e = make_double2(0.0, 0.0), o = e;
      for (int w = wb; w < we; ++w) {
        const double2* src = red + ((size_t)w * B * kSynLat + (size_t)b * kSynLat + lj) * 2;
        e.x += src[0].x; e.y += src[0].y;
        o.x += src[1].x; o.y += src[1].y;
      }
      double2* dst = a.eo + (((size_t)b * (P.R + 1) + r) * P.Jh + j) * 2;
      st_eo(dst, e, o);
    }
  }
}

template <int B, int MODE, int NSPLIT>
int launch_syn_t(const PlanDev& P, const SynArgs& a, cudaStream_t st) {
  const int npairs = a.pairs ? a.npairs : P.R / 2 + 1;
  if (npairs == 0) return kOk;
  const int nlg = (P.Jh + kSynLat - 1) / kSynLat;
  size_t smem = sizeof(double2) * NSPLIT * B * kCS + sizeof(double) * (NSPLIT * kCS + 2);
  if (NSPLIT > 1) smem += sizeof(double2) * NSPLIT * B * kSynLat * 2;
  auto kern = syn_kernel<B, MODE, NSPLIT>;
  SW_TRY(set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem));
  StageScope sc("legendre_synthesis", st);
  SW_CUDA(launch_pdl(kern, dim3(dim3(npairs, nlg, a.nmembers)), dim3(NSPLIT * 32), smem, st, P, a));
  SW_LAUNCH_CHECK();
  return kOk;
}

// Warps per CTA so the grid offers ~2 resident warps per SM sub-partition.
int pick_split(const PlanDev& P, int npairs, int nmembers) {
  static const int knob = env_int("SWSDC_SYN_SPLIT", 0);   // tuning knob: force 1, 2 or 4
  if (knob == 1 || knob == 2 || knob == 4) return knob;
  const long long base = (long long)npairs * ((P.Jh + kSynLat - 1) / kSynLat) * nmembers;
  if (base >= 1000) return 1;
  if (base >= 500) return 2;
  return 4;
}

template <int B, int MODE>
int launch_syn_b(const PlanDev& P, const SynArgs& a, cudaStream_t st) {
  switch (pick_split(P, a.pairs ? a.npairs : P.R / 2 + 1, a.nmembers)) {
    case 1: return launch_syn_t<B, MODE, 1>(P, a, st);
    case 2: return launch_syn_t<B, MODE, 2>(P, a, st);
    default: return launch_syn_t<B, MODE, 4>(P, a, st);
  }
}

}  // namespace

int launch_synthesis(const PlanDev& P, const SynArgs& a, int B, int mode, cudaStream_t st) {
  if (mode == kSynUV) return launch_syn_b<2, kSynUV>(P, a, st);
  if (mode == kSynSWE) return launch_syn_b<5, kSynSWE>(P, a, st);
  switch (B) {
    case 1: return launch_syn_b<1, kSynPlain>(P, a, st);
    case 2: return launch_syn_b<2, kSynPlain>(P, a, st);
    case 3: return launch_syn_b<3, kSynPlain>(P, a, st);
    case 4: return launch_syn_b<4, kSynPlain>(P, a, st);
    case 5: return launch_syn_b<5, kSynPlain>(P, a, st);
    case 6: return launch_syn_b<6, kSynPlain>(P, a, st);
  }
  set_error("synthesis batch per launch must be 1..6");
  return kUsage;
}
// ---------------------------------------------------------------------------
// Analysis (DMMA)
//
// One warp per (r, 32-degree chunk, member); 4 warps per CTA take consecutive
// chunks of the same r so their x loads hit the same L1 lines.  Each warp
// walks the latitudes in blocks of 32: lane l regenerates q for the chunk's 32
// degrees at latitude 32*jb32 + l (seeded from the checkpoint) into a
// warp-private A tile (rows ordered parity-major), then 8 k-steps of
// mma.sync.m8n8k4.f64 contract 4 latitudes each: A = q (even or odd degrees),
// B = x fragment (one coalesced 256-byte load from the fragment-native layout
// written by fourier.cu), C accumulates (S-parity rows with S, D with D).  No
// CTA barriers; the latitude reduction happens inside the tensor core.
// ---------------------------------------------------------------------------
namespace {

constexpr int kAnaWarps = 4;

// Zeros for s < r of row r (dense output): the CTA's warps take whole vectors,
// lanes consecutive degrees (coalesced 16-byte stores, no index division).
__device__ __forceinline__ void ana_zero_fill(const AnaArgs& a, double2* out, int r, int warp,
                                              int nwarps, int lane) {
  for (int v = warp; v < a.nv; v += nwarps) {
    double2* o = out + (size_t)v * a.out_vstride + (size_t)r * a.out_rstride;
    for (int s = lane; s < r; s += 32) o[s] = make_double2(0.0, 0.0);
  }
}
constexpr int kQS = kChunk + 4;   // A-tile row stride (doubles), == 4 mod 16

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// B fragments (S and D parity) of latitude block jb for the NT n-tiles.
template <int NT>
__device__ __forceinline__ void load_b(double (&bv)[2][NT], const double* xr, int jb, int Jh,
                                       int nc, int ncol, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const bool ok = (jb * 4 + t) < Jh;
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const bool col = (n * 8 + g) < ncol;
      bv[p][n] = (ok && col) ? xr[(((size_t)jb * 2 + p) * nc + n * 8) * 4 + lane] : 0.0;
    }
}

// LSPLIT warps share one chunk, each taking every LSPLIT-th latitude block;
// their accumulators are reduced through shared memory in warp order.
__device__ __forceinline__ void cp_async16_ana(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// B fragments stream through a per-warp shared ring kBDepth k-steps deep
// (cp.async, 2 x NT x 256 contiguous bytes per k-step), so the DMMAs read
// their operands from shared memory instead of waiting on L2.
constexpr int kBDepth = 4;
// A fragments of one k-step in the table-fed variant: [parity][m-tile][lane]
constexpr int kAFrag = 2 * 2 * 32;
// Pair-major x (XLayout::pm): the ring holds each k-step's B block as
// [parity][latitude t][S] rows, S = 8 NT padded to 8 (mod 16) doubles so the
// fragment reads (lane g, t -> row t, column 8 n + g) take the minimum 2
// wavefronts.
template <int NT>
__host__ __device__ constexpr int ana_pm_stride() {
  return (8 * NT + 8) % 16 == 0 ? 8 * NT + 16 : 8 * NT + 8;
}
template <int NT, bool PM>
__host__ __device__ constexpr int ana_bslot() { return PM ? 2 * 4 * ana_pm_stride<NT>() : 2 * NT * 32; }
template <int NT, bool TAB = false, bool PM = false>
__host__ __device__ constexpr int ana_warp_doubles() {
  // TAB: no q tile or betas; the ring carries A and B fragments and, after the
  // k-loop, the epilogue staging ([4 NT][33] double2) and the split reduction
  return TAB ? (kBDepth * (ana_bslot<NT, PM>() + kAFrag) > 4 * NT * 33 * 2
                    ? kBDepth * (ana_bslot<NT, PM>() + kAFrag) : 4 * NT * 33 * 2)
             : kChunk * kQS + kChunk + kBDepth * ana_bslot<NT, PM>();
}

// One work item (r, first chunk, checkpoint index) of member m (one CTA; a
// persistent grid walking the item list was measured in
// profiles/r01/experiments.md and not kept).
// MP = 2: members 2m and 2m + 1 of an ensemble share the CTA -- n-tiles
// [0, NT/2) come from the first member's x, [NT/2, NT) from the second's
// (each member's layout holds NT/2 n-tiles, a.nv <= 4 NT/2 vectors) -- so the
// q tile and the A fragments serve twice the columns.
// TAB: the A operand (Pbar of the chunk's 32 degrees at 4 latitudes per
// k-step) is not regenerated from the recurrence but streamed from the plan's
// fragment-native table P.ptab (reference-rounded values, build_ptab) through
// the same cp.async ring as the B fragments; no seeds, betas, q tile or chunk
// scale g.
template <int NT, int LSPLIT, int MP = 1, bool TAB = false, bool PM = false>
__device__ __forceinline__ void ana_item(const PlanDev& P, const AnaArgs& a, const int4 wk, int m,
                                         double* smem) {
  static_assert(MP == 1 || (MP == 2 && NT % 4 == 0), "member pairs need NT / 2 even");
  constexpr int kWD = ana_warp_doubles<NT, TAB, PM>();
  constexpr int kBS = ana_bslot<NT, PM>();                       // B part of a ring slot
  constexpr int kSlot = kBS + (TAB ? kAFrag : 0);                // ring slot (doubles)
  constexpr int kS = ana_pm_stride<NT>();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* qs = smem + (size_t)warp * kWD;                        // [32][kQS] (TAB: staging only)
  double* bs = qs + kChunk * kQS;                                // [32] betas (not TAB)
  double* bring = TAB ? qs : bs + kChunk;                        // [kBDepth][slot]

  const double* x = a.x + (size_t)(MP * m) * a.xl.mstride;
  double2* out = a.out + (size_t)(MP * m) * a.out_mstride;
  const int r = wk.x, c = wk.y + warp / LSPLIT, half = warp % LSPLIT;
  const int nout = a.smax - r + 1;
  ANA_STAMP(0);

  const bool active = c * kChunk < nout;

  double acc[2][2][NT][2];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int n = 0; n < NT; ++n) { acc[p][mt][n][0] = 0.0; acc[p][mt][n][1] = 0.0; }

  const int k0 = c * kChunk;
  // epilogue scales g of this lane's output rows k0 + p + 2 (8 mt + g), fetched
  // now so the load latency hides behind the contraction (TAB: unscaled, 1)
  double gsv[2][2];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int k = k0 + p + 2 * (8 * mt + g);
      gsv[p][mt] = (active && k < nout) ? (TAB ? 1.0 : P.gsc[(size_t)r * P.ldk + k]) : 0.0;
    }
  // first-block seed and mu of this lane's latitude, loaded together with the
  // betas (one round trip for all the item's table loads; the recurrence of
  // each later block is seeded one block ahead)
  const double2* seeds = P.ckpt + (size_t)(wk.z + (c - wk.y)) * P.Jh;
  double2 sd_nx = make_double2(0.0, 0.0);
  double mu_nx = 0.0;
  if (!TAB && active) {
    const int jh0 = (half << 5) + lane;
    if (jh0 < P.Jh) { sd_nx = seeds[jh0]; mu_nx = P.mu_n[jh0]; }
  }
  if (!TAB && active) bs[lane] = P.beta[(size_t)r * P.ldk + k0 + lane];
  // everything above reads only plan tables; x and out belong to the stream's
  // earlier kernels, so the dependency wait (PDL) sits here: the item's table
  // round trip overlaps the predecessor's tail
  pdl_wait();
  if (a.zero_fill && wk.y == 0) {
#pragma unroll
    for (int h = 0; h < MP; ++h)
      ana_zero_fill(a, out + (size_t)h * a.out_mstride, r, warp, blockDim.x >> 5, lane);
  }
  if (active) {
    const int nc = a.xl.nc, jh4 = a.xl.jh4;
    const double* xr = x + (size_t)r * jh4 * 2 * nc * 4;
    const int nblk = (P.Jh + 31) >> 5;
    const int nmine = (nblk - half + LSPLIT - 1) / LSPLIT;   // latitude blocks of this warp
    const int nks = nmine * 8;
    // Issue side of the x ring: k-steps are issued in order; consecutive k-steps
    // of a latitude block are consecutive 4-latitude blocks jb, this warp's
    // blocks are LSPLIT apart.  A running jb replaces per-step index math, the
    // per-lane copy offsets are loop-invariant, and copies stop at the row's
    // last block (jb < jh4) or after the warp's last k-step.
    static_assert((kBDepth & (kBDepth - 1)) == 0, "ring depth must be a power of 2");
    constexpr int kCp = (2 * NT * 16 + 31) / 32;   // 16-byte copies per lane per k-step
    int coff_d[kCp], coff_s[kCp];
#pragma unroll
    for (int u = 0; u < kCp; ++u) {
      const int cc = lane + 32 * u;
      const int p = cc / (NT * 16), q = cc - p * (NT * 16);
      coff_d[u] = (cc < 2 * NT * 16) ? p * NT * 32 + 2 * q : -1;
      coff_s[u] = p * nc * 4 + 2 * q;
    }
    const size_t jb_stride = (size_t)2 * nc * 4;
    const size_t jump = (size_t)((LSPLIT - 1) * 8 + 1) * jb_stride;
    const size_t poff = (size_t)nc * 4;                       // parity-1 half of a block
    const double* ip = xr + (size_t)(half << 3) * jb_stride;  // block of the next issue
    // pair-major: 16-byte copies of the block's 8 rows [p][t] of nc doubles (MP = 2:
    // nc / 2 of each member) into ring rows of kS; loop-invariant per-lane offsets
    constexpr int kPmCp = PM ? (MP == 2 ? 4 : NT) : 1;
    int pm_s[kPmCp], pm_d[kPmCp];
    if constexpr (PM) {
#pragma unroll
      for (int u = 0; u < kPmCp; ++u) {
        const int cc = lane + 32 * u;
        if constexpr (MP == 2) {
          const int h = cc >> 6, row = (cc >> 3) & 7, q = cc & 7;
          pm_s[u] = row * 16 + 2 * q;   // + member h offset at issue time
          pm_d[u] = row * kS + h * 16 + 2 * q;
        } else {
          const int row = cc / (4 * NT), q = cc - row * (4 * NT);
          pm_s[u] = row * nc + 2 * q;
          pm_d[u] = row * kS + 2 * q;
        }
      }
    }
    // TAB: A fragments of this warp's chunk, kAFrag doubles per 4-latitude block
    const double* ap = TAB ? P.ptab + ((size_t)(wk.z + (c - wk.y)) * jh4 + (half << 3)) * kAFrag
                           : nullptr;
    int iss = 0, ijb = half << 3;
    auto issue_next = [&]() {
      if (iss < nks && ijb < jh4) {
        double* dst = bring + (iss & (kBDepth - 1)) * kSlot;
        if constexpr (TAB) {
          cp_async16_ana(dst + kBS + 2 * lane, ap + 2 * lane);
          cp_async16_ana(dst + kBS + 64 + 2 * lane, ap + 64 + 2 * lane);
        }
        if constexpr (PM) {
#pragma unroll
          for (int u = 0; u < kPmCp; ++u) {
            const size_t mo = (MP == 2 && u >= 2) ? (size_t)a.xl.mstride : 0;
            cp_async16_ana(dst + pm_d[u], ip + mo + pm_s[u]);
          }
        } else if constexpr (NT % 2 == 0) {
          // each parity half is NT/2 copies per lane at fixed offsets from the
          // lane's base: immediate-offset addressing, no per-step index math
          const double* s0 = ip + 2 * lane;
          const double* s1 = s0 + poff;
          double* d0 = dst + 2 * lane;
          // MP = 2: copies u >= NT / 4 read the second member (its tile u - NT / 4)
          constexpr int UM = NT / (2 * MP);
#pragma unroll
          for (int u = 0; u < NT / 2; ++u) {
            const size_t so = (size_t)(u % UM) * 64 + (MP == 2 && u >= UM ? (size_t)a.xl.mstride : 0);
            cp_async16_ana(d0 + 64 * u, s0 + so);
            cp_async16_ana(d0 + NT * 32 + 64 * u, s1 + so);
          }
        } else {
#pragma unroll
          for (int u = 0; u < kCp; ++u)
            if (coff_d[u] >= 0) cp_async16_ana(dst + coff_d[u], ip + coff_s[u]);
        }
      }
      cp_async_commit();
      ++iss;
      const bool blk = (iss & 7) == 0;
      ijb += blk ? (LSPLIT - 1) * 8 + 1 : 1;
      ip += blk ? jump : jb_stride;
      if constexpr (TAB) ap += (blk ? (LSPLIT - 1) * 8 + 1 : 1) * kAFrag;
    };
    ANA_STAMP(1);
#pragma unroll
    for (int d = 0; d < kBDepth - 1; ++d) issue_next();
    int ks = 0;
    // a row's last chunk with <= 16 degrees has an empty upper m-tile (degrees
    // 16..31 of the chunk): its warps run an instantiation without those DMMAs
    // and recurrence steps (decided once per warp, outside the unrolled loops)
    auto blocks = [&](auto mt_count) {
    constexpr int MTN = decltype(mt_count)::value;
    for (int jb32 = half; jb32 < nblk; jb32 += LSPLIT) {
      if constexpr (!TAB) {
      __syncwarp();
      // regenerate q for 32 degrees at latitude jh = 32*jb32 + lane
      const int jh = (jb32 << 5) + lane;
      const double2 sd = sd_nx;
      const double mu = mu_nx;
      {
        const int jn = ((jb32 + LSPLIT) << 5) + lane;
        if (jn < P.Jh) { sd_nx = seeds[jn]; mu_nx = P.mu_n[jn]; }
      }
      if (jh < P.Jh) {
        double qa = sd.x, qb = sd.y;
        qs[lane] = qa;
        qs[16 * kQS + lane] = qb;
#pragma unroll
        for (int kk = 2; kk < (MTN == 2 ? kChunk : kChunk / 2); kk += 2) {
          qa = fma(mu, qb, -bs[kk] * qa);
          qb = fma(mu, qa, -bs[kk + 1] * qb);
          qs[(kk >> 1) * kQS + lane] = qa;
          qs[(16 + (kk >> 1)) * kQS + lane] = qb;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < kChunk; ++kk) qs[((kk & 1) * 16 + (kk >> 1)) * kQS + lane] = 0.0;
      }
      __syncwarp();
      }
      if (jb32 == half) ANA_STAMP(2);
      // k-steps of this block; blocks reaching past Jh (padding rows of x may
      // hold non-finite bits, q = 0 there) take the masked instantiation
      auto ksteps = [&](auto full_c) {
        constexpr bool FULL = decltype(full_c)::value;
#pragma unroll
        for (int s = 0; s < 8; ++s, ++ks) {
          issue_next();
          cp_async_wait<kBDepth - 1>();
          __syncwarp();
          if (ks == 0) ANA_STAMP(3);
          // no column mask: column n of D depends only on column n of B, and
          // columns >= 2 nv only feed accumulators that are never written
          const double* bsrc = bring + (ks & (kBDepth - 1)) * kSlot;
          double bv[2][NT];
          const bool ok = FULL || (((jb32 << 3) + s) * 4 + t) < P.Jh;
#pragma unroll
          for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              const double b = PM ? bsrc[(p * 4 + t) * kS + n * 8 + g] : bsrc[p * NT * 32 + n * 32 + lane];
              bv[p][n] = FULL ? b : (ok ? b : 0.0);
            }
#pragma unroll
          for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int mt = 0; mt < MTN; ++mt) {
              const double av = TAB ? bsrc[kBS + (p * 2 + mt) * 32 + lane]
                                    : qs[(p * 16 + mt * 8 + g) * kQS + s * 4 + t];
#pragma unroll
              for (int n = 0; n < NT; ++n) dmma884(acc[p][mt][n], av, bv[p][n]);
            }
          __syncwarp();   // this slot is refilled kBDepth - 1 k-steps later
        }
      };
      if ((jb32 << 5) + 32 <= P.Jh) ksteps(std::true_type());
      else ksteps(std::false_type());
    }
    };
    if (a.short_tiles && nout - k0 <= kChunk / 2) blocks(std::integral_constant<int, 1>());
    else blocks(std::integral_constant<int, 2>());
    cp_async_wait<0>();
  }
  ANA_STAMP(4);

  // only the LSPLIT warps of one chunk meet: the whole CTA for LSPLIT >= 3 (one
  // chunk per CTA), named barriers 1 / 2 with immediate ids for LSPLIT = 2 -- a
  // register-valued barrier id would reserve all 16 ids and cap the kernel at 4
  // CTAs per SM (ncu: "Block Limit Barriers")
  auto chunk_barrier = [&]() {
    if constexpr (LSPLIT >= 3) {
      __syncthreads();
    } else {
      if (warp < LSPLIT) asm volatile("bar.sync 1, %0;\n" ::"n"(32 * LSPLIT) : "memory");
      else asm volatile("bar.sync 2, %0;\n" ::"n"(32 * LSPLIT) : "memory");
    }
  };
  if (LSPLIT > 1) {
    // warps half > 0 hand their partial sums to the half-0 warp of their chunk
    chunk_barrier();
    double* red = smem + (size_t)warp * ana_warp_doubles<NT, TAB, PM>();
    if (half > 0 && active) {
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const int e = ((p * 2 + mt) * NT + n) * 2;
            red[e * 32 + lane] = acc[p][mt][n][0];
            red[(e + 1) * 32 + lane] = acc[p][mt][n][1];
          }
    }
    chunk_barrier();
    if (!active) return;
    if (half > 0) return;
    for (int h = 1; h < LSPLIT; ++h) {
      const double* src = smem + (size_t)(warp + h) * ana_warp_doubles<NT, TAB, PM>();
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const int e = ((p * 2 + mt) * NT + n) * 2;
            acc[p][mt][n][0] += src[e * 32 + lane];
            acc[p][mt][n][1] += src[(e + 1) * 32 + lane];
          }
    }
  } else if (!active) {
    return;
  }

  ANA_STAMP(5);
  // epilogue: row k = k0 + p + 2 (8 mt + g), column pair (re, im) of staged
  // vector n*4 + t.  The scaled values are transposed through the warp's q
  // tile (free after the k-loop; rows of 33 double2 keep the fragment-order
  // writes conflict-free) so that each vector's 32 degrees leave as one
  // coalesced 512-byte store instead of 16-byte pieces two degrees apart.
  {
    double2* stg = reinterpret_cast<double2*>(qs);   // [4 NT][33] double2 (4 NT * 33 * 2 <= 32 kQS)
    static_assert(4 * NT * 33 * 2 <= (TAB ? ana_warp_doubles<NT, TAB, PM>() : kChunk * kQS),
                  "staging fits the q tile / ring");
    __syncwarp();
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int kl = p + 2 * (8 * mt + g);
        const double gs = gsv[p][mt];
#pragma unroll
        for (int n = 0; n < NT; ++n)
          stg[(n * 4 + t) * 33 + kl] = make_double2(acc[p][mt][n][0] * gs, acc[p][mt][n][1] * gs);
      }
    __syncwarp();
    const bool inrow = k0 + lane < nout;
#pragma unroll
    for (int vs = 0; vs < 4 * NT; ++vs) {
      // MP = 2: staged vectors [2 NT, 4 NT) are the second member's
      const int h = (MP == 2 && vs >= 2 * NT) ? 1 : 0;
      const int v = vs - h * 2 * NT;
      if (v < a.nv && inrow)
        out[(size_t)h * a.out_mstride + (size_t)v * a.out_vstride + (size_t)r * a.out_rstride + r + k0 + lane] =
            stg[vs * 33 + lane];
    }
  }
  ANA_STAMP(6);
}

// One CTA per work item (grid: items x members).
template <int NT, int LSPLIT, int MP = 1, bool TAB = false, bool PM = false>
__global__ void __launch_bounds__(kAnaWarps * 32, 4)
ana_kernel(PlanDev P, AnaArgs a) {
  pdl_trigger();   // pdl_wait() inside ana_item, after the plan-table loads
  extern __shared__ __align__(16) double smem[];
  ana_item<NT, LSPLIT, MP, TAB, PM>(P, a, a.work[blockIdx.x], blockIdx.y, smem);
}

// ---------------------------------------------------------------------------
// Analysis on the FP64 vector pipe (DFMA), for the DMMA-vs-DFMA comparison the
// north star asks for (SWSDC_ANA_DFMA=1).  Same decomposition as ana_kernel
// (work lists, wave-fitted latitude split, q tile, cp.async x ring); lane =
// degree slot of the chunk (lanes 0..15 even degrees, 16..31 odd), holding the
// 4 NT vectors' accumulators.  Per k-step (4 latitudes) a lane reads its q row
// segment (2 x 16 B) and, per vector, the real and imaginary x values of the 4
// latitudes (2 x 16 B half-warp broadcasts: S for even, D for odd degrees).
// ---------------------------------------------------------------------------
constexpr int kQD = kChunk + 2;   // q row stride (doubles): 16-B aligned, conflict-free rows
template <int NT>
__host__ __device__ constexpr int anad_warp_doubles() {
  return kChunk * kQD + kChunk + kBDepth * 2 * NT * 32;
}

template <int NT, int LSPLIT>
__global__ void __launch_bounds__(kAnaWarps * 32)
ana_dfma_kernel(PlanDev P, AnaArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double smem[];
  constexpr int kWD = anad_warp_doubles<NT>();
  constexpr int NV = 4 * NT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* qs = smem + (size_t)warp * kWD;     // [32 degree slots][kQD latitudes]
  double* bs = qs + kChunk * kQD;
  double* bring = bs + kChunk;                // [kBDepth][2][NT * 32]
  const double* x = a.x + (size_t)blockIdx.y * a.xl.mstride;
  double2* out = a.out + (size_t)blockIdx.y * a.out_mstride;
  const int4 wk = a.work[blockIdx.x];
  const int r = wk.x, c = wk.y + warp / LSPLIT, half = warp % LSPLIT;
  const int nout = a.smax - r + 1;
  if (a.zero_fill && wk.y == 0) ana_zero_fill(a, out, r, warp, blockDim.x >> 5, lane);
  const bool active = c * kChunk < nout;
  const int k0 = c * kChunk;
  const int par = lane >> 4;   // degree parity of this lane: x parity S (0) or D (1)
  double acc[NV][2];
#pragma unroll
  for (int v = 0; v < NV; ++v) { acc[v][0] = 0.0; acc[v][1] = 0.0; }
  if (active) {
    bs[lane] = P.beta[(size_t)r * P.ldk + k0 + lane];
    const double2* seeds = P.ckpt + (size_t)(wk.z + (c - wk.y)) * P.Jh;
    const int nc = a.xl.nc, jh4 = a.xl.jh4;
    const double* xr = x + (size_t)r * jh4 * 2 * nc * 4;
    const int nblk = (P.Jh + 31) >> 5;
    const int nmine = (nblk - half + LSPLIT - 1) / LSPLIT;
    const int nks = nmine * 8;
    auto issue = [&](int ks) {
      if (ks < nks) {
        const int jb = ((half + (ks >> 3) * LSPLIT) << 3) + (ks & 7);
        if (jb < jh4) {
          double* dst = bring + (ks % kBDepth) * (2 * NT * 32);
#pragma unroll
          for (int cc = lane; cc < 2 * NT * 16; cc += 32) {
            const int p = cc / (NT * 16), q = cc - p * (NT * 16);
            cp_async16_ana(dst + p * NT * 32 + 2 * q, xr + ((size_t)jb * 2 + p) * nc * 4 + 2 * q);
          }
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int d = 0; d < kBDepth - 1; ++d) issue(d);
    double2 sd_nx = make_double2(0.0, 0.0);
    double mu_nx = 0.0;
    {
      const int jh0 = (half << 5) + lane;
      if (jh0 < P.Jh) { sd_nx = seeds[jh0]; mu_nx = P.mu_n[jh0]; }
    }
    int ks = 0;
    for (int jb32 = half; jb32 < nblk; jb32 += LSPLIT) {
      __syncwarp();
      // q tile: lane = latitude writes its column; row = degree slot (even rows 0..15, odd 16..31)
      const int jh = (jb32 << 5) + lane;
      const double2 sd = sd_nx;
      const double mu = mu_nx;
      {
        const int jn = ((jb32 + LSPLIT) << 5) + lane;
        if (jn < P.Jh) { sd_nx = seeds[jn]; mu_nx = P.mu_n[jn]; }
      }
      double qa = 0.0, qb = 0.0;
      if (jh < P.Jh) { qa = sd.x; qb = sd.y; }
      qs[lane] = qa;
      qs[16 * kQD + lane] = qb;
#pragma unroll
      for (int kk = 2; kk < kChunk; kk += 2) {
        qa = fma(mu, qb, -bs[kk] * qa);
        qb = fma(mu, qa, -bs[kk + 1] * qb);
        qs[(kk >> 1) * kQD + lane] = qa;
        qs[(16 + (kk >> 1)) * kQD + lane] = qb;
      }
      __syncwarp();
      const double* qrow = qs + (size_t)((par << 4) + (lane & 15)) * kQD;
#pragma unroll 1
      for (int s = 0; s < 8; ++s, ++ks) {
        issue(ks + kBDepth - 1);
        cp_async_wait<kBDepth - 1>();
        __syncwarp();
        const double* bsrc = bring + (ks % kBDepth) * (2 * NT * 32) + par * NT * 32;
        const int lat0 = ((jb32 << 3) + s) * 4;
        const double2 q01 = *reinterpret_cast<const double2*>(qrow + s * 4);
        const double2 q23 = *reinterpret_cast<const double2*>(qrow + s * 4 + 2);
        if (lat0 + 3 < P.Jh) {
#pragma unroll
          for (int v = 0; v < NV; ++v) {
#pragma unroll
            for (int ri = 0; ri < 2; ++ri) {
              const int col = 2 * v + ri;
              const double* xc = bsrc + (col >> 3) * 32 + (col & 7) * 4;
              const double2 x01 = *reinterpret_cast<const double2*>(xc);
              const double2 x23 = *reinterpret_cast<const double2*>(xc + 2);
              double t = acc[v][ri];
              t = fma(q01.x, x01.x, t);
              t = fma(q01.y, x01.y, t);
              t = fma(q23.x, x23.x, t);
              acc[v][ri] = fma(q23.y, x23.y, t);
            }
          }
        } else {
          // last latitude block with padding: padded x entries may be garbage
          const double qv[4] = {q01.x, q01.y, q23.x, q23.y};
#pragma unroll
          for (int tt = 0; tt < 4; ++tt) {
            if (lat0 + tt >= P.Jh) break;
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
              for (int ri = 0; ri < 2; ++ri) {
                const int col = 2 * v + ri;
                acc[v][ri] = fma(qv[tt], bsrc[(col >> 3) * 32 + (col & 7) * 4 + tt], acc[v][ri]);
              }
          }
        }
        __syncwarp();
      }
    }
    cp_async_wait<0>();
  }
  if (LSPLIT > 1) {
    const unsigned bar_id = 1 + warp / LSPLIT, bar_n = 32 * LSPLIT;
    asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(bar_n) : "memory");
    double* red = smem + (size_t)warp * kWD;
    if (half > 0 && active) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        red[(2 * v) * 32 + lane] = acc[v][0];
        red[(2 * v + 1) * 32 + lane] = acc[v][1];
      }
    }
    asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(bar_n) : "memory");
    if (half > 0 || !active) return;
    for (int h = 1; h < LSPLIT; ++h) {
      const double* src = smem + (size_t)(warp + h) * kWD;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        acc[v][0] += src[(2 * v) * 32 + lane];
        acc[v][1] += src[(2 * v + 1) * 32 + lane];
      }
    }
  } else if (!active) {
    return;
  }
  // lane -> degree k = k0 + par + 2 (lane & 15)
  const int k = k0 + par + 2 * (lane & 15);
  if (k < nout) {
    const double gs = P.gsc[(size_t)r * P.ldk + k];
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (v < a.nv)
        out[(size_t)v * a.out_vstride + (size_t)r * a.out_rstride + r + k] =
            make_double2(acc[v][0] * gs, acc[v][1] * gs);
  }
}

// CTA = ana_chunks_per_cta(LSPLIT) chunks x LSPLIT latitude splits.
bool ana_dfma() {
  static const int knob = env_int("SWSDC_ANA_DFMA", 0);
  return knob != 0;
}

// Member pairs (a.nmembers pairs of members, a.nv <= 8 vectors each): one
// CTA contracts both members' x with the same q tiles (NT = 4).
template <int LSPLIT>
int launch_ana_pairs_t(const PlanDev& P, const AnaArgs& a, int nwork, cudaStream_t st) {
  const int warps = LSPLIT * ana_chunks_per_cta(LSPLIT);
  const bool tab = ana_table_fed(P, 4, 2), pm = a.xl.pm != 0;
  if (pm && a.xl.nc != 16) {
    set_error("pair-major member-pair analysis needs 16 columns per member");
    return kUsage;
  }
  const size_t smem = sizeof(double) * warps *
                      (pm ? (tab ? ana_warp_doubles<4, true, true>() : ana_warp_doubles<4, false, true>())
                          : (tab ? ana_warp_doubles<4, true>() : ana_warp_doubles<4>()));
  auto kern = pm ? (tab ? ana_kernel<4, LSPLIT, 2, true, true> : ana_kernel<4, LSPLIT, 2, false, true>)
                 : (tab ? ana_kernel<4, LSPLIT, 2, true> : ana_kernel<4, LSPLIT, 2>);
  SW_TRY(set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem));
  SW_TRY(set_smem_carveout_max(reinterpret_cast<const void*>(kern)));
  StageScope sc("legendre_analysis", st);
  SW_CUDA(launch_pdl(kern, dim3(dim3(nwork, a.nmembers)), dim3(warps * 32), smem, st, P, a));
  SW_LAUNCH_CHECK();
  return kOk;
}

template <int NT, int LSPLIT>
int launch_ana_t(const PlanDev& P, const AnaArgs& a, int nwork, cudaStream_t st) {
  const int warps = LSPLIT * ana_chunks_per_cta(LSPLIT);
  if (ana_dfma()) {
    const size_t smem = sizeof(double) * warps * anad_warp_doubles<NT>();
    auto kern = ana_dfma_kernel<NT, LSPLIT>;
    SW_TRY(set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem));
    StageScope sc("legendre_analysis", st);
    SW_CUDA(launch_pdl(kern, dim3(nwork, a.nmembers), dim3(warps * 32), smem, st, P, a));
    SW_LAUNCH_CHECK();
    return kOk;
  }
  const bool tab = ana_table_fed(P, NT, 1);
  if (a.xl.pm) {
    // pair-major x (the F_E path, 7 vectors): NT = 2, recurrence-fed
    if constexpr (NT == 2) {
      const size_t smem = sizeof(double) * warps * ana_warp_doubles<NT, false, true>();
      auto kern = ana_kernel<NT, LSPLIT, 1, false, true>;
      SW_TRY(set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem));
      SW_TRY(set_smem_carveout_max(reinterpret_cast<const void*>(kern)));
      StageScope sc("legendre_analysis", st);
      SW_CUDA(launch_pdl(kern, dim3(dim3(nwork, a.nmembers)), dim3(warps * 32), smem, st, P, a));
      SW_LAUNCH_CHECK();
      return kOk;
    } else {
      set_error("pair-major analysis is built for 5..8 vectors");
      return kUsage;
    }
  }
  const size_t smem = sizeof(double) * warps * (tab ? ana_warp_doubles<NT, true>() : ana_warp_doubles<NT>());
  auto kern = tab ? ana_kernel<NT, LSPLIT, 1, true> : ana_kernel<NT, LSPLIT>;
  SW_TRY(set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem));
  SW_TRY(set_smem_carveout_max(reinterpret_cast<const void*>(kern)));
  StageScope sc("legendre_analysis", st);
  SW_CUDA(launch_pdl(kern, dim3(dim3(nwork, a.nmembers)), dim3(warps * 32), smem, st, P, a));
  SW_LAUNCH_CHECK();
  return kOk;
}

template <int NT>
int launch_ana_nt(const PlanDev& P, const AnaArgs& a, int nwork, int lsplit, cudaStream_t st) {
  switch (lsplit) {
    case 2: return launch_ana_t<NT, 2>(P, a, nwork, st);
    case 3: return launch_ana_t<NT, 3>(P, a, nwork, st);
    case 4: return launch_ana_t<NT, 4>(P, a, nwork, st);
    default: return launch_ana_t<NT, 1>(P, a, nwork, st);
  }
}

template <int NT, int LSPLIT>
int ana_ctas_per_sm_t(bool tab) {
  const int warps = LSPLIT * ana_chunks_per_cta(LSPLIT);
  const bool dfma = ana_dfma();
  const size_t smem = sizeof(double) * warps *
                      (dfma ? anad_warp_doubles<NT>()
                            : tab ? ana_warp_doubles<NT, true>() : ana_warp_doubles<NT>());
  auto kern = dfma ? ana_dfma_kernel<NT, LSPLIT>
                   : tab ? ana_kernel<NT, LSPLIT, 1, true> : ana_kernel<NT, LSPLIT>;
  if (set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem) != kOk) return 1;
  if (!dfma && set_smem_carveout_max(reinterpret_cast<const void*>(kern)) != kOk) return 1;
  int n = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, warps * 32, smem) != cudaSuccess) {
    cudaGetLastError();
    n = 1;
  }
  return n > 0 ? n : 1;
}

// ---------------------------------------------------------------------------
// Analysis, TMA-streamed variant (opt-in: SWSDC_ANA_TMA=2; measured slower than the cp.async ring of ana_kernel, which is the default).  CTA = 4 warps = 4 consecutive
// 32-degree chunks of ONE row r; the row's x tiles (32 latitudes = 8 blocks,
// contiguous in the fragment-native layout) are streamed into a 3-deep shared
// ring by one elected thread with cp.async.bulk (TMA, SASS UBLKCP) completing
// on an mbarrier, so the B fragments of every warp are conflict-free smem
// loads instead of L2 round trips; each warp regenerates its own q tile and
// runs the DMMA k-steps as before.
// ---------------------------------------------------------------------------
constexpr int kTmaBuf = 3;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes,
                                             unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

template <int NT>
__global__ void __launch_bounds__(kAnaWarps * 32)
ana_tma_kernel(PlanDev P, AnaArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) double smem[];
  const int nc = a.xl.nc;                        // layout columns (>= 8 NT)
  const int blk_doubles = 8 * 2 * nc * 4;        // one 32-latitude tile
  double* xbuf = smem;                           // [kTmaBuf][blk_doubles]
  double* wsm = xbuf + kTmaBuf * blk_doubles;    // per-warp q tile + betas
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(
      wsm + kAnaWarps * (kChunk * kQS + kChunk));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* qs = wsm + (size_t)warp * (kChunk * kQS + kChunk);
  double* bs = qs + kChunk * kQS;

  const double* x = a.x + (size_t)blockIdx.y * a.xl.mstride;
  double2* out = a.out + (size_t)blockIdx.y * a.out_mstride;
  const int4 wk = a.work[blockIdx.x];
  const int r = wk.x, c = wk.y + warp;
  const int nout = a.smax - r + 1;
  const bool active = c * kChunk < nout;

  if (a.zero_fill && wk.y == 0) ana_zero_fill(a, out, r, warp, blockDim.x >> 5, lane);
  const int jh4 = a.xl.jh4;
  const int nblk = (P.Jh + 31) >> 5;
  const double* xr = x + (size_t)r * jh4 * 2 * nc * 4;
  auto issue = [&](int jb32) {
    const int nb = min(8, jh4 - 8 * jb32);
    const unsigned bytes = (unsigned)(nb * 2 * nc * 4 * sizeof(double));
    unsigned long long* bar = &bars[jb32 % kTmaBuf];
    mbar_expect_tx(bar, bytes);
    tma_bulk_g2s(xbuf + (size_t)(jb32 % kTmaBuf) * blk_doubles, xr + (size_t)jb32 * blk_doubles,
                 bytes, bar);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTmaBuf; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < kTmaBuf - 1 && i < nblk; ++i) issue(i);

  double acc[2][2][NT][2];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int n = 0; n < NT; ++n) { acc[p][mt][n][0] = 0.0; acc[p][mt][n][1] = 0.0; }

  const int k0 = c * kChunk;
  const double2* seeds = P.ckpt + (size_t)(wk.z + (active ? c - wk.y : 0)) * P.Jh;
  if (active) bs[lane] = P.beta[(size_t)r * P.ldk + k0 + lane];
  const int ncol = 2 * a.nv;
  double2 sd_nx = make_double2(0.0, 0.0);
  double mu_nx = 0.0;
  if (active && lane < P.Jh) { sd_nx = seeds[lane]; mu_nx = P.mu_n[lane]; }

  for (int jb32 = 0; jb32 < nblk; ++jb32) {
    // refill: the slot of block jb32-1 is free once every warp passed the barrier
    __syncthreads();
    if (threadIdx.x == 0 && jb32 + kTmaBuf - 1 < nblk) issue(jb32 + kTmaBuf - 1);
    if (active) {
      const int jh = (jb32 << 5) + lane;
      const double2 sd = sd_nx;
      const double mu = mu_nx;
      {
        const int jn = ((jb32 + 1) << 5) + lane;
        if (jn < P.Jh) { sd_nx = seeds[jn]; mu_nx = P.mu_n[jn]; }
      }
      if (jh < P.Jh) {
        double qa = sd.x, qb = sd.y;
        qs[lane] = qa;
        qs[16 * kQS + lane] = qb;
#pragma unroll
        for (int kk = 2; kk < kChunk; kk += 2) {
          qa = fma(mu, qb, -bs[kk] * qa);
          qb = fma(mu, qa, -bs[kk + 1] * qb);
          qs[(kk >> 1) * kQS + lane] = qa;
          qs[(16 + (kk >> 1)) * kQS + lane] = qb;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < kChunk; ++kk) qs[((kk & 1) * 16 + (kk >> 1)) * kQS + lane] = 0.0;
      }
      __syncwarp();
      mbar_wait(&bars[jb32 % kTmaBuf], (unsigned)((jb32 / kTmaBuf) & 1));
      const double* xb = xbuf + (size_t)(jb32 % kTmaBuf) * blk_doubles;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const bool ok = ((jb32 << 5) + s * 4 + t) < P.Jh;
        double bv[2][NT];
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
          for (int n = 0; n < NT; ++n)
            bv[p][n] = (ok && (n * 8 + g) < ncol) ? xb[((s * 2 + p) * nc + n * 8) * 4 + lane] : 0.0;
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const double av = qs[(p * 16 + mt * 8 + g) * kQS + s * 4 + t];
#pragma unroll
            for (int n = 0; n < NT; ++n) dmma884(acc[p][mt][n], av, bv[p][n]);
          }
      }
      __syncwarp();
    }
  }
  if (!active) return;
  const double* gr = P.gsc + (size_t)r * P.ldk;
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int k = k0 + p + 2 * (8 * mt + g);
      if (k >= nout) continue;
      const double gs = gr[k];
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int v = n * 4 + t;
        if (v < a.nv)
          out[(size_t)v * a.out_vstride + (size_t)r * a.out_rstride + r + k] =
              make_double2(acc[p][mt][n][0] * gs, acc[p][mt][n][1] * gs);
      }
    }
}

template <int NT>
int launch_ana_tma(const PlanDev& P, const AnaArgs& a, int nwork, cudaStream_t st) {
  const size_t smem = sizeof(double) * ((size_t)kTmaBuf * 8 * 2 * a.xl.nc * 4 +
                                        kAnaWarps * (kChunk * kQS + kChunk)) +
                      sizeof(unsigned long long) * kTmaBuf + 16;
  auto kern = ana_tma_kernel<NT>;
  SW_TRY(set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem));
  StageScope sc("legendre_analysis", st);
  SW_CUDA(launch_pdl(kern, dim3(dim3(nwork, a.nmembers)), dim3(kAnaWarps * 32), smem, st, P, a));
  SW_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// Synthesis on the FP64 tensor cores (opt-in comparison, SWSDC_SYN_DMMA=1; the
// north star keeps DMMA only where it beats the vector pipe, and here it does
// not: config 1 31.3 us vs 29.1 us for syn_kernel, profiles/r02/experiments.md),
// for batches of >= 8 fields with a plan table: the DFMA kernel is bound by its per-degree coefficient
// broadcasts (one shared-memory load per 2 latitudes x 2 FMAs), so for wide
// batches the contraction F[r, j] = sum_s P[r, s, j] c[r, s] runs as DMMA
// with the product transposed, C^T = c^T P: M = 8 columns (re / im of 4
// fields), N = 8 latitudes, K = 4 degrees of one parity (even degrees -> E,
// odd -> O).  A = coefficients (staged per 32-degree chunk in shared memory,
// shared by the CTA's warps), B = Pbar from the plan's synthesis-order table
// (reference-rounded, streamed through a per-warp cp.async ring).
// CTA = one r-pair {p, R - p} of one 16-field group, one warp per 32
// latitudes; CT column tiles (8 columns each) of 2 x min(B, 16) columns.
// ---------------------------------------------------------------------------
constexpr int kSdDepth = 4;           // ring depth in k-steps (1 KB of B per k-step)
constexpr int kSdCS = 36;             // coefficient tile row stride (doubles)

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}

template <int CT>
__global__ void __launch_bounds__(256) syn_dmma_kernel(PlanDev P, SynArgs a, int nf, int ntot) {
  pdl_wait();
  pdl_trigger();
  // field group blockIdx.y: fields [y nf, min((y + 1) nf, ntot))
  nf = min(nf, ntot - (int)blockIdx.y * nf);
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nlb = (P.Jh + 31) >> 5;
  double* cs = smem;                                           // [2][32 degrees][kSdCS]
  double* ring = smem + 2 * 32 * kSdCS + (size_t)warp * kSdDepth * 128;
  const double2* src = a.src + (size_t)blockIdx.y * a.src_mstride;
  double2* eo = a.eo + (size_t)blockIdx.y * a.eo_mstride;
  const int p = blockIdx.x;
  const int rows[2] = {p, P.R - p};
  const int nrow = rows[1] > rows[0] ? 2 : 1;
  const int lb = warp;                                         // latitude block of this warp
  const bool lb_ok = lb < nlb;
  for (int ir = 0; ir < nrow; ++ir) {
    const int r = rows[ir];
    const int nst = a.smax - r + 1, nch = (nst + kChunk - 1) / kChunk;
    // coefficient staging of chunk ci into buffer ci & 1: row d = degree r + 32 ci + d,
    // columns 2 f + (re, im); zero past the input truncation / the row end
    auto stage = [&](int ci) {
      double* dst = cs + (size_t)(ci & 1) * 32 * kSdCS;
      for (int idx = threadIdx.x; idx < 32 * 8 * CT / 2; idx += blockDim.x) {
        const int d = idx / (4 * CT), f = idx - d * (4 * CT);
        const int sdeg = r + ci * kChunk + d;
        const bool valid = f < nf && r <= a.src_R && sdeg <= a.src_R && sdeg <= a.smax;
        const double2* gp = src + (size_t)f * a.src_fstride + (size_t)r * (a.src_R + 1) + (valid ? sdeg : r);
        cp_async16_zfill(dst + d * kSdCS + 2 * f, valid ? gp : src, valid);
      }
    };
    // B fragments of (chunk ci, k-step ks) for this warp's latitude block
    const double* tab = P.stab + ((size_t)P.ck_off[r] * nlb + lb) * 8 * 128;
    auto issue = [&](int i) {   // i = ci * 8 + ks
      if (lb_ok && i < nch * 8) {
        const double* s0 = tab + (size_t)(i >> 3) * nlb * 8 * 128 + (size_t)(i & 7) * 128;
        double* d0 = ring + (i % kSdDepth) * 128;
        cp_async16_ana(d0 + 2 * lane, s0 + 2 * lane);
        cp_async16_ana(d0 + 64 + 2 * lane, s0 + 64 + 2 * lane);
      }
    };
    double acc[2][CT][4][2];
#pragma unroll
    for (int pp = 0; pp < 2; ++pp)
#pragma unroll
      for (int ct = 0; ct < CT; ++ct)
#pragma unroll
        for (int lt = 0; lt < 4; ++lt) { acc[pp][ct][lt][0] = 0.0; acc[pp][ct][lt][1] = 0.0; }
    __syncthreads();                 // the previous row's last tile reads are done
    stage(0);
    cp_async_commit();
#pragma unroll
    for (int d = 0; d < kSdDepth - 1; ++d) { issue(d); cp_async_commit(); }
    for (int ci = 0; ci < nch; ++ci) {
      if (ci + 1 < nch) stage(ci + 1);
      cp_async_commit();
      const double* ct0 = cs + (size_t)(ci & 1) * 32 * kSdCS;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int i = ci * 8 + ks;
        issue(i + kSdDepth - 1);
        cp_async_commit();
        // the group of k-step i (and the chunk's coefficients) have landed
        cp_async_wait<kSdDepth - 1>();
        if (ks == 0) __syncthreads();   // every thread's coefficient copies of chunk ci
        else __syncwarp();
        const int pp = ks >> 2, q = ks & 3;
        const double* rb = ring + (i % kSdDepth) * 128;
        double bv[4], av[CT];
#pragma unroll
        for (int lt = 0; lt < 4; ++lt) bv[lt] = rb[lt * 32 + lane];
        const int drow = pp + 2 * (4 * q + t);   // degree row of this lane's A element
#pragma unroll
        for (int ct = 0; ct < CT; ++ct) av[ct] = ct0[drow * kSdCS + 8 * ct + g];
#pragma unroll
        for (int ct = 0; ct < CT; ++ct)
#pragma unroll
          for (int lt = 0; lt < 4; ++lt) dmma884(acc[pp][ct][lt], av[ct], bv[lt]);
        __syncwarp();
      }
      __syncthreads();   // the coefficient buffer of chunk ci is refilled at ci + 2
    }
    cp_async_wait<0>();
    // E / O out: lane (g, t) holds column 8 ct + g (field (8 ct + g) / 2, re for even g,
    // im for odd g) at latitudes 32 lb + 8 lt + 2 t + {0, 1}
    if (lb_ok) {
#pragma unroll
      for (int ct = 0; ct < CT; ++ct)
#pragma unroll
        for (int lt = 0; lt < 4; ++lt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double E = acc[0][ct][lt][e], O = acc[1][ct][lt][e];
            const double Ei = __shfl_down_sync(0xffffffffu, E, 4);
            const double Oi = __shfl_down_sync(0xffffffffu, O, 4);
            const int f = (8 * ct + g) >> 1;
            const int jh = 32 * lb + 8 * lt + 2 * t + e;
            if (!(g & 1) && f < nf && jh < P.Jh) {
              double2* o = eo + (size_t)f * ((size_t)(P.R + 1) * P.Jh * 2) + ((size_t)r * P.Jh + jh) * 2;
              o[0] = make_double2(E, Ei);
              o[1] = make_double2(O, Oi);
            }
          }
    }
  }
}

template <int CT>
int launch_syn_dmma_t(const PlanDev& P, const SynArgs& a, int nf, int ntot, cudaStream_t st) {
  const int npairs = P.R / 2 + 1;
  const int nlb = (P.Jh + 31) / 32;
  const int warps = nlb;
  const size_t smem = sizeof(double) * (2 * 32 * kSdCS + (size_t)warps * kSdDepth * 128);
  auto kern = syn_dmma_kernel<CT>;
  SW_TRY(set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem));
  StageScope sc("legendre_synthesis", st);
  SW_CUDA(launch_pdl(kern, dim3(npairs, a.nmembers), dim3(32 * warps), smem, st, P, a, nf, ntot));
  SW_LAUNCH_CHECK();
  return kOk;
}

}  // namespace

// Tensor-core synthesis of nf <= 16 plain fields per member (a.nmembers groups):
// needs the plan's synthesis table (P.stab) and Jh <= 256 (one warp per 32
// latitudes in a CTA of <= 8 warps).
int launch_synthesis_dmma(const PlanDev& P, const SynArgs& a, int nf, cudaStream_t st) {
  if (!P.stab || nf < 1 || nf > 16 || (P.Jh + 31) / 32 > 8 || a.pairs) {
    set_error("tensor-core synthesis needs a plan table, <= 16 fields and <= 256 latitude pairs");
    return kUsage;
  }
  // field groups of <= 8 (2 column tiles) per CTA: twice the CTAs of one 16-field group
  static const int gf = std::max(1, std::min(16, env_int("SWSDC_SYN_DMMA_GF", 8)));
  const int ng = (nf + gf - 1) / gf, per = (nf + ng - 1) / ng;
  SynArgs b = a;
  b.nmembers = ng;
  b.src_mstride = a.src_fstride * per;
  b.eo_mstride = (long long)(P.R + 1) * P.Jh * 2 * per;
  switch ((2 * per + 7) / 8) {
    case 1: return launch_syn_dmma_t<1>(P, b, per, nf, st);
    case 2: return launch_syn_dmma_t<2>(P, b, per, nf, st);
    case 3: return launch_syn_dmma_t<3>(P, b, per, nf, st);
    default: return launch_syn_dmma_t<4>(P, b, per, nf, st);
  }
}

int ana_warps_per_cta() { return kAnaWarps; }
int ana_chunks_per_cta(int lsplit) { return lsplit >= 3 ? 1 : kAnaWarps / lsplit; }

// Resident CTAs per SM of the register analysis kernel (cached per NT, LSPLIT,
// q-tile / table variant).
int ana_ctas_per_sm(int nv, int lsplit, bool tab) {
  static int cache[2][4][4] = {};
  const int nt = (2 * nv + 7) / 8;   // 1..4
  int& c = cache[tab ? 1 : 0][nt - 1][lsplit - 1];
  if (c == 0) {
    int n = 1;
#define SW_OCC(NT_)                                                   \
    switch (lsplit) {                                                 \
      case 1: n = ana_ctas_per_sm_t<NT_, 1>(tab); break;              \
      case 2: n = ana_ctas_per_sm_t<NT_, 2>(tab); break;              \
      case 3: n = ana_ctas_per_sm_t<NT_, 3>(tab); break;              \
      default: n = ana_ctas_per_sm_t<NT_, 4>(tab); break;             \
    }
    if (nt == 1) { SW_OCC(1) } else if (nt == 2) { SW_OCC(2) } else if (nt == 3) { SW_OCC(3) } else { SW_OCC(4) }
#undef SW_OCC
    c = n;
  }
  return c;
}

// TMA-streamed analysis (opt-in, SWSDC_ANA_TMA=2): measured against the
// cp.async-ring register kernel with its wave-fitted latitude split it wins only
// marginally on a single large state (config 2: 16.9 vs 17.2 us) and loses on
// config 0 (9.6 vs 8.6 us) and the 64-member ensemble (186 vs 172 us).
bool ana_uses_tma(int nv) {
  static const int knob = env_int("SWSDC_ANA_TMA", 0);   // 2: use it for <= 8 vectors
  return knob == 2 && nv <= 8;
}

// a.work must list CTAs of kAnaWarps / lsplit consecutive chunks (lsplit 1 for TMA).
int launch_analysis(const PlanDev& P, const AnaArgs& a, int nwork, int lsplit, cudaStream_t st) {
  if (a.nv <= 0) return kOk;
  if (ana_uses_tma(a.nv) && lsplit == 1) {
    if (a.nv <= 4) return launch_ana_tma<1>(P, a, nwork, st);
    if (a.nv <= 8) return launch_ana_tma<2>(P, a, nwork, st);
    if (a.nv <= 12) return launch_ana_tma<3>(P, a, nwork, st);
    if (a.nv <= 16) return launch_ana_tma<4>(P, a, nwork, st);
  }
  if (a.nv <= 4) return launch_ana_nt<1>(P, a, nwork, lsplit, st);
  if (a.nv <= 8) return launch_ana_nt<2>(P, a, nwork, lsplit, st);
  if (a.nv <= 12) return launch_ana_nt<3>(P, a, nwork, lsplit, st);
  if (a.nv <= 16) return launch_ana_nt<4>(P, a, nwork, lsplit, st);
  set_error("analysis vectors per launch must be <= 16");
  return kUsage;
}

int launch_analysis_pairs(const PlanDev& P, const AnaArgs& a, int nwork, int lsplit, cudaStream_t st) {
  if (a.nv <= 0) return kOk;
  if (a.nv > 8) {
    set_error("member-pair analysis takes <= 8 vectors per member");
    return kUsage;
  }
  switch (lsplit) {
    case 2: return launch_ana_pairs_t<2>(P, a, nwork, st);
    case 3: return launch_ana_pairs_t<3>(P, a, nwork, st);
    case 4: return launch_ana_pairs_t<4>(P, a, nwork, st);
    default: return launch_ana_pairs_t<1>(P, a, nwork, st);
  }
}

// Table-fed analysis (A fragments streamed from P.ptab) only where each A
// fragment serves >= 3 n-tiles: with 1-2 n-tiles the extra L2 -> SM traffic
// (1 KB of A per 4-16 DMMAs) costs more than the recurrence it replaces
// (config 2, 7 vectors: 1.84 -> 1.92 ms per step; config 1, 15 vectors:
// analysis 31.2 -> 29.1 us; config 4, member pairs: 6.85 -> 6.47 ms).
bool ana_table_fed(const PlanDev& P, int nt, int mp) {
  return P.ptab != nullptr && nt * mp >= 3;
}

bool ana_dfma_enabled() { return ana_dfma(); }

bool ana_pairs_ok(int nv, int nmembers) {
  static const int knob = env_int("SWSDC_ANA_PAIRS", 1);
  return knob != 0 && nv >= 1 && nv <= 8 && nmembers >= 2 && nmembers % 2 == 0 && !ana_dfma() &&
         !ana_uses_tma(nv);
}

}  // namespace swsdc

#ifdef ANA_TRACE
extern "C" int swsdc_debug_ana_trace(unsigned long long* host, int clear) {
  if (clear) {
    static unsigned long long zero[16384][8];
    return cudaMemcpyToSymbol(swsdc::g_ana_trace, zero, sizeof(zero)) == cudaSuccess ? 0 : 3;
  }
  return cudaMemcpyFromSymbol(host, swsdc::g_ana_trace, sizeof(unsigned long long) * 16384 * 8) ==
                 cudaSuccess ? 0 : 3;
}
#endif
