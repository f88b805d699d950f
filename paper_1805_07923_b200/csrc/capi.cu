// C ABI (include/swsdc_b200.h): plan construction and the host-side
// orchestration of the kernels for each reference entry point.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "fourier.cuh"
#include "legendre.cuh"
#include "spectral.cuh"
#include "../../include/swsdc_b200.h"

namespace swsdc {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

}  // namespace swsdc

using namespace swsdc;

struct swsdc_plan {
  PlanDev dev{};
  std::vector<void*> owned;
  // analysis work lists [smax = R, R + 1][lsplit = 1, 2]: CTAs of 4/lsplit chunks
  int4* work[2][kAnaSplits] = {};      // [smax = R, R + 1][latitude split - 1]
  int nwork[2][kAnaSplits] = {};
  int nchunks[2] = {0, 0};
  int ldy = 0;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  void* grid_ws = nullptr;      // large-n_lon F_E path: 5 grids per state
  size_t grid_bytes = 0;
  bool force_split = false;     // option 1: use the large-n_lon F_E path even when it fits
  // a workspace whose address a stream capture has recorded is "pinned": a
  // later larger request allocates a new buffer and retires the pinned one
  // (freed with the plan) instead of freeing memory a CUDA graph still uses
  bool ws_pinned = false, grid_pinned = false;
  std::vector<void*> retired;
  // m-sharding caches per row filter: balanced row pairs for synthesis and
  // filtered analysis work lists
  struct Shard {
    int mod = 1, rank = 0;
    int2* pairs = nullptr;
    int npairs = 0;
    int4* work[2][kAnaSplits] = {};
    int nwork[2][kAnaSplits] = {};
    int nchunks[2] = {0, 0};
  };
  std::vector<Shard> shards;
  std::vector<std::vector<int4>> host_work[2];  // host copies of the analysis lists
};

namespace swsdc {
void set_row_filter(int mod, int rank);
}

namespace {

template <typename T>
int upload(swsdc_plan* p, const std::vector<T>& h, T** d) {
  void* ptr = nullptr;
  SW_CUDA(cudaMalloc(&ptr, h.size() * sizeof(T) + 16));
  p->owned.push_back(ptr);
  SW_CUDA(cudaMemcpy(ptr, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  *d = reinterpret_cast<T*>(ptr);
  return kOk;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

size_t field_bytes(const swsdc_plan* p) {
  const PlanDev& P = p->dev;
  return (size_t)(P.R + 1) * P.Jh * 2 * sizeof(double2);
}
size_t y_bytes(const swsdc_plan* p) {
  return (size_t)(p->dev.R + 1) * p->ldy * sizeof(double2);
}

// Workspace = [eo: n_eo fields][x: x_bytes][y: n_y vectors].
size_t x_bytes_for(const swsdc_plan* p, int nv, int nmembers) {
  if (nv <= 0 || nmembers <= 0) return 0;
  return sizeof(double) * (size_t)make_xlayout(p->dev.R, p->dev.Jh, nv).mstride * nmembers + 256;
}

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

// Drop a workspace buffer before reallocation: freed if no captured graph can
// reference it, else kept alive until the plan is destroyed.
template <typename T>
int retire(swsdc_plan* p, T*& buf, size_t& bytes, bool& pinned) {
  if (buf) {
    if (pinned) {
      p->retired.push_back(buf);
    } else {
      SW_CUDA(cudaDeviceSynchronize());
      SW_CUDA(cudaFree(buf));
    }
  }
  buf = nullptr;
  bytes = 0;
  pinned = false;
  return kOk;
}

int ensure_ws(swsdc_plan* p, int n_eo, size_t x_bytes, int n_y, cudaStream_t st = 0) {
  const size_t need = (size_t)n_eo * field_bytes(p) + x_bytes + (size_t)n_y * y_bytes(p) + 256;
  if (capturing(st)) {
    // growing the workspace cannot happen during graph capture
    if (need > p->ws_bytes) {
      set_error("workspace too small during stream capture; call swsdc_plan_reserve first");
      return kUsage;
    }
    p->ws_pinned = true;
    return kOk;
  }
  if (need <= p->ws_bytes) return kOk;
  SW_TRY(retire(p, p->ws, p->ws_bytes, p->ws_pinned));
  SW_CUDA(cudaMalloc(&p->ws, need));
  p->ws_bytes = need;
  return kOk;
}

double2* ws_eo(swsdc_plan* p) { return reinterpret_cast<double2*>(p->ws); }
double* ws_x(swsdc_plan* p, int n_eo) {
  return reinterpret_cast<double*>(p->ws + (size_t)n_eo * field_bytes(p));
}
double2* ws_y(swsdc_plan* p, int n_eo, size_t x_bytes) {
  return reinterpret_cast<double2*>(p->ws + (size_t)n_eo * field_bytes(p) + x_bytes);
}

ModelConsts consts(const swsdc_params* q) {
  ModelConsts c;
  c.radius = q->radius;
  c.omega = q->omega;
  c.gravity = q->gravity;
  c.nu = q->nu;
  c.h_bar = q->h_bar;
  c.phi_bar = q->gravity * q->h_bar;
  return c;
}

int check_params(const swsdc_params* q) {
  if (!q) { set_error("params is NULL"); return kUsage; }
  if (!(q->radius > 0) || !(q->gravity > 0) || !(q->h_bar > 0)) {
    set_error("radius, gravity and h_bar must be positive");
    return kUsage;
  }
  if (q->nu < 0) { set_error("diffusion coefficient must be non-negative"); return kUsage; }
  return kOk;
}

// Plain synthesis of `batch` fields from coeffs at truncation r_in into eo.
int syn_plain(swsdc_plan* p, const double2* coeffs, int r_in, int batch, double2* eo,
              cudaStream_t st) {
  const PlanDev& P = p->dev;
  const long long cin = (long long)(r_in + 1) * (r_in + 1);
  const long long fstride = (long long)(P.R + 1) * P.Jh * 2;
  int B = 0;
  static const int fb = env_int("SWSDC_SYN_B", 0);   // tuning knob: fields per synthesis CTA
  if (fb > 0 && batch % fb == 0) B = fb;
  for (int cand = 6; cand >= 4 && !B; --cand)
    if (batch % cand == 0) { B = cand; break; }
  int done = 0;
  // wide batches on the tensor cores (opt-in, SWSDC_SYN_DMMA=1: 31.3 vs 29.1 us for the
  // DFMA kernel at config 1 -- with 16 fields per CTA only 128 CTAs, with 8 the shared
  // coefficient tiles and table stream still leave the DMMA pipe latency-bound)
  while (P.stab && batch - done >= 8) {
    const int nf = std::min(16, batch - done);
    SynArgs a{};
    a.src = coeffs + done * cin;
    a.src_fstride = cin;
    a.src_R = r_in;
    a.smax = P.R;
    a.eo = eo + done * fstride;
    a.src_mstride = cin * nf;
    a.eo_mstride = fstride * nf;
    a.nmembers = 1;
    SW_TRY(launch_synthesis_dmma(P, a, nf, st));
    done += nf;
  }
  while (done < batch) {
    int b = B;
    int groups;
    if (b == 0) {
      const int ng = (batch - done + 5) / 6;
      b = (batch - done + ng - 1) / ng;
    }
    groups = (batch - done) / b;
    if (groups == 0) { b = batch - done; groups = 1; }
    SynArgs a{};
    a.src = coeffs + done * cin;
    a.src_fstride = cin;
    a.src_R = r_in;
    a.smax = P.R;
    a.eo = eo + done * fstride;
    a.src_mstride = cin * b;
    a.eo_mstride = fstride * b;
    a.nmembers = groups;
    SW_TRY(launch_synthesis(P, a, b, kSynPlain, st));
    done += b * groups;
  }
  return kOk;
}

// Pairs / work lists for the current row filter (nullptr = all rows).
const swsdc_plan::Shard* shard_for(swsdc_plan* p) {
  const RowFilter rf = current_row_filter();
  if (rf.mod <= 1) return nullptr;
  for (auto& s : p->shards)
    if (s.mod == rf.mod && s.rank == rf.rank) return &s;
  swsdc_plan::Shard s;
  s.mod = rf.mod;
  s.rank = rf.rank;
  const int R = p->dev.R;
  std::vector<int> rows;
  for (int r = 0; r <= R; ++r)
    if (r % rf.mod == rf.rank) rows.push_back(r);
  std::vector<int2> pairs;
  const int n = (int)rows.size();
  for (int i = 0; i < (n + 1) / 2; ++i)
    pairs.push_back(make_int2(rows[i], (n - 1 - i > i) ? rows[n - 1 - i] : -1));
  s.npairs = (int)pairs.size();
  if (!pairs.empty()) {
    if (cudaMalloc(&s.pairs, sizeof(int2) * pairs.size()) != cudaSuccess) return nullptr;
    cudaMemcpy(s.pairs, pairs.data(), sizeof(int2) * pairs.size(), cudaMemcpyHostToDevice);
    p->owned.push_back(s.pairs);
  }
  for (int i = 0; i < 2; ++i) {
    for (int r : rows) s.nchunks[i] += (R + i - r + 1 + kChunk - 1) / kChunk;
    for (int j = 0; j < kAnaSplits; ++j) {
      std::vector<int4> w;
      for (const int4& it : p->host_work[i][j])
        if (it.x % rf.mod == rf.rank) w.push_back(it);
      s.nwork[i][j] = (int)w.size();
      if (!w.empty()) {
        if (cudaMalloc(&s.work[i][j], sizeof(int4) * w.size()) != cudaSuccess) return nullptr;
        cudaMemcpy(s.work[i][j], w.data(), sizeof(int4) * w.size(), cudaMemcpyHostToDevice);
        p->owned.push_back(s.work[i][j]);
      }
    }
  }
  p->shards.push_back(s);
  return &p->shards.back();
}

int upload_work(swsdc_plan* p, std::vector<int4> (&work)[2][kAnaSplits]) {
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < kAnaSplits; ++j) SW_TRY(upload(p, work[i][j], &p->work[i][j]));
  return kOk;
}

// Latitude split (1..4 warps per 32-degree chunk) of the register analysis
// kernel: the one that best fills whole waves, counting warp rounds
// ceil(items / slots) x blocks per warp ceil(nblk / split) against the
// useful work nch x nblk (tie -> fewer splits, less reduction traffic).
int pick_ana_split(int nch, int nmembers, int nv, int Jh, bool tab) {
  static const int knob = env_int("SWSDC_ANA_LSPLIT", 0);   // tuning knob: force 1..4
  if (knob >= 1 && knob <= kAnaSplits) return knob;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int nblk = (Jh + 31) / 32;
  const double useful = (double)nch * nmembers * nblk;
  // Problems spanning several waves even unsplit gain nothing from the split
  // but pay its per-item cost (seeds, split reduction, epilogue: ~1 latitude
  // block of k-steps, tools/ana_trace.py): charge it there (T1279: 19.06 ->
  // 18.33 ms per config-3 step); small problems keep the wave-fitting choice.
  const long long slots1 = (long long)sms * ana_ctas_per_sm(nv, 1, tab) * ana_chunks_per_cta(1);
  const double item_cost = (long long)nch * nmembers >= 2 * slots1 ? 1.0 : 0.0;
  // Small problems (about one wave unsplit): three latitude splits measured best
  // once the kernel runs 5 CTAs/SM (immediate barriers, max carveout): config 1
  // analysis 28.1 us vs 29.2 (two splits, the wave-fitting choice), config 2 step
  // 1.733 vs 1.764 ms; fewer latitude blocks than three cap it
  static const int small3 = env_int("SWSDC_ANA_SMALL3", 1);
  if (small3 && item_cost == 0.0 && nblk >= 3) return 3;
  int best = 1;
  double best_eff = -1.0;
  for (int ls = 1; ls <= kAnaSplits; ++ls) {
    if (ls > nblk) break;
    const int warps = ls * ana_chunks_per_cta(ls);
    const long long slots = (long long)sms * ana_ctas_per_sm(nv, ls, tab) * warps;
    const long long items = (long long)nch * nmembers * ls;
    const long long rounds = (items + slots - 1) / slots;
    const double eff = useful / ((double)slots * rounds * ((nblk + ls - 1) / ls + item_cost));
    if (eff > best_eff + 1e-9) { best_eff = eff; best = ls; }
  }
  return best;
}

// Grid workspace of the split F_E path (5 grids per state).  During stream
// capture it cannot grow: returns false so the caller can use the fused kernel.
int grow_grid_ws(swsdc_plan* p, size_t need, cudaStream_t st, bool* ok) {
  *ok = true;
  if (capturing(st)) {
    if (need > p->grid_bytes) { *ok = false; return kOk; }
    p->grid_pinned = true;
    return kOk;
  }
  if (need <= p->grid_bytes) return kOk;
  SW_TRY(retire(p, p->grid_ws, p->grid_bytes, p->grid_pinned));
  SW_CUDA(cudaMalloc(&p->grid_ws, need));
  p->grid_bytes = need;
  return kOk;
}

// F_E grid stage: fused one-pair-per-CTA kernel, or the split path (grids
// through the workspace) for n_lon too large for the fused rings, when forced,
// or for batches too small to fill the GPU (swe_split_preferred).
int fe_grid_stage(swsdc_plan* p, bool nl, const double2* eo, int batch, double* x,
                  const XLayout& xl, double omega, double radius, cudaStream_t st, int jh_begin,
                  int jh_end) {
  const PlanDev& P = p->dev;
  const long long fstride = (long long)(P.R + 1) * P.Jh * 2;
  const bool fits = swe_grid_fits(P);
  bool split = !fits || p->force_split ||
               swe_split_preferred(P, (long long)(jh_end - jh_begin) * batch);
  const long long gfield = (long long)P.I * P.J;
  const bool reg = fourier_reg_fft(P);
  // ring layout: Jh x I complex per field (>= I x J real for odd J)
  const size_t per_field = std::max<size_t>(sizeof(double2) * (size_t)P.Jh * P.I, sizeof(double) * gfield);
  if (split) {
    bool ok = true;
    SW_TRY(grow_grid_ws(p, per_field * 5 * batch, st, &ok));
    if (!ok) {
      if (!fits) {
        set_error("grid workspace too small during stream capture");
        return kUsage;
      }
      split = false;
    }
  }
  if (!split)
    return launch_swe_grid(P, nl, eo, 5 * fstride, x, xl, batch, omega, radius, st, jh_begin,
                           jh_end);
  if (reg)
    return launch_swe_split_reg(P, nl, eo, fstride, reinterpret_cast<double2*>(p->grid_ws), x, xl,
                                batch, omega, radius, st, jh_begin, jh_end);
  // smem-FFT split path: grids travel in the ring layout (coalesced rows per pair)
  double2* rg = reinterpret_cast<double2*>(p->grid_ws);
  const long long rfield = (long long)P.Jh * P.I;
  if (nl && batch <= 2) {
    // the nonlinear products never read the delta grid (its Coriolis term is
    // formed in Fourier space, swe_prod_kernel): U/a, V/a, zeta and phi' only
    for (int m = 0; m < batch; ++m) {
      SW_TRY(launch_fourier_to_rings(P, eo + (size_t)m * 5 * fstride, fstride, rg + (size_t)m * 5 * rfield,
                                     rfield, 3, st, jh_begin, jh_end));
      SW_TRY(launch_fourier_to_rings(P, eo + ((size_t)m * 5 + 4) * fstride, fstride,
                                     rg + ((size_t)m * 5 + 4) * rfield, rfield, 1, st, jh_begin, jh_end));
    }
  } else {
    SW_TRY(launch_fourier_to_rings(P, eo, fstride, rg, rfield, 5 * batch, st, jh_begin, jh_end));
  }
  return launch_swe_products(P, nl, reinterpret_cast<const double*>(rg), rfield, 5 * rfield, eo,
                             fstride, x, xl,
                             batch, omega, radius, st, jh_begin, jh_end);
}

// Legendre analysis of the nv vectors (XLayout xl) of each member into out.
// x layout of the F_E pipeline: pair-major for the nonlinear tendency on the
// fused register-FFT grid path (swe_grid5_kernel then writes whole sectors per
// latitude pair without the 4-CTA cluster exchange; measured: config 4 step
// -1.1%, config 0 -3%, config 2 -0.5%, though the analysis' ring re-ordering
// costs it ~10%); column-major elsewhere -- the large-n_lon split path (config
// 3: +0.9% with pair-major) and the DFMA / TMA comparison kernels.
XLayout fe_xlayout(const PlanDev& P, bool nl) {
  static const int knob = env_int("SWSDC_FE_PM", 1);
  const bool pm = knob && nl && !ana_dfma_enabled() && !ana_uses_tma(7) && fourier_reg_fft(P) &&
                  swe_grid_fits(P);
  return make_xlayout(P.R, P.Jh, nl ? 7 : 2, pm);
}

int ana_run(swsdc_plan* p, const double* x, const XLayout& xl, int nmembers, double2* out,
            long long out_vstride, long long out_rstride, long long out_mstride, int smax,
            bool zero_fill, cudaStream_t st) {
  const PlanDev& P = p->dev;
  const int which = (smax == P.R) ? 0 : 1;
  const swsdc_plan::Shard* sh = shard_for(p);
  const int nch = sh ? sh->nchunks[which] : p->nchunks[which];
  // TMA variant (<= 8 vectors) runs unsplit; otherwise split latitudes to fill waves
  const int nv0 = xl.nv < 16 ? xl.nv : 16;
  // ensembles: two members per CTA when each has <= 8 vectors (same q tiles, NT = 4)
  const bool pairs = xl.nv <= 8 && ana_pairs_ok(xl.nv, nmembers);
  const int lsplit = ana_uses_tma(nv0) ? 1
                     : pairs ? pick_ana_split(nch, nmembers / 2, 16, P.Jh, ana_table_fed(P, 4, 2))
                             : pick_ana_split(nch, nmembers, nv0, P.Jh,
                                              ana_table_fed(P, (2 * nv0 + 7) / 8, 1));
  const int ls = lsplit - 1;
  for (int v0 = 0; v0 < xl.nv; v0 += 16) {
    AnaArgs a{};
    a.nv = (xl.nv - v0 < 16) ? xl.nv - v0 : 16;
    a.x = x + (size_t)(v0 / 16) * xl.gstride;
    a.xl = xl;
    a.out = out + v0 * out_vstride;
    a.out_vstride = out_vstride;
    a.out_rstride = out_rstride;
    a.smax = smax;
    a.zero_fill = zero_fill ? 1 : 0;
    a.work = sh ? sh->work[which][ls] : p->work[which][ls];
    a.out_mstride = out_mstride;
    a.nmembers = nmembers;
    static const int short_tiles = env_int("SWSDC_ANA_SHORT", 1);
    a.short_tiles = short_tiles;
    const int nw = sh ? sh->nwork[which][ls] : p->nwork[which][ls];
    if (nw == 0) continue;
    if (pairs) {
      a.nmembers = nmembers / 2;
      SW_TRY(launch_analysis_pairs(P, a, nw, lsplit, st));
    } else {
      SW_TRY(launch_analysis(P, a, nw, lsplit, st));
    }
  }
  return kOk;
}

}  // namespace

extern "C" {

const char* swsdc_last_error(void) { return g_last_error.c_str(); }
const char* swsdc_version(void) { return "swsdc_b200 0.1 (sm_100a)"; }

int swsdc_plan_create(int R, int n_lon, int n_lat, const double* mu, const double* w,
                      swsdc_plan** out) {
  if (!out) { set_error("out is NULL"); return kUsage; }
  *out = nullptr;
  if (R < 0) { set_error("truncation must be non-negative"); return kUsage; }
  if (n_lon < 2 * R + 1) {
    set_error("n_lon=" + std::to_string(n_lon) + " cannot carry zonal wavenumbers up to " +
              std::to_string(R));
    return kUsage;
  }
  if (n_lat < 1) { set_error("need at least one latitude"); return kUsage; }
  if (!swfft::fft_supported(n_lon)) {
    set_error("n_lon must factor into primes <= 13");
    return kUsage;
  }
  if (!mu || !w) { set_error("mu / w are NULL"); return kUsage; }

  swsdc_plan* p = new swsdc_plan();
  PlanDev& P = p->dev;
  P.R = R;
  P.I = n_lon;
  P.J = n_lat;
  P.Jh = (n_lat + 1) / 2;
  P.ldk = ((R + 2 + kChunk + 16) + 7) / 8 * 8;
  {
    const char* mr = getenv("SWSDC_FFT_MAX_RADIX");   // tuning knob (16 default, 8)
    P.fft = swfft::make_fft_plan(n_lon, mr ? atoi(mr) : 16);
  }
  p->ldy = R + 2;
  const int ldk = P.ldk;

  std::vector<double> mu_n(P.Jh), w_n(P.Jh);
  for (int jh = 0; jh < P.Jh; ++jh) {
    const int jn = n_lat - P.Jh + jh;
    mu_n[jh] = mu[jn];
    w_n[jh] = w[jn];
  }
  // recurrence tables with the reference's expressions (spharm.py:159-169, 174-177)
  std::vector<double> a((size_t)(R + 1) * ldk, 0.0), b(a.size(), 0.0), beta(a.size(), 0.0),
      gsc(a.size(), 0.0), eps(a.size(), 0.0), sect(R + 1);
  for (int r = 0; r <= R; ++r) {
    double* ar = &a[(size_t)r * ldk];
    double* br = &b[(size_t)r * ldk];
    ar[1] = std::sqrt(2.0 * r + 3.0);
    for (int k = 2; k < ldk; ++k) {
      const long long s = r + k;
      const double s2r2 = (double)(s * s - (long long)r * r);
      ar[k] = std::sqrt((4.0 * s * s - 1.0) / s2r2);
      br[k] = std::sqrt((2.0 * s + 1.0) * (s - 1.0 - r) * (s - 1.0 + r) / ((2.0 * s - 3.0) * s2r2));
    }
    double* be = &beta[(size_t)r * ldk];
    double* g = &gsc[(size_t)r * ldk];
    for (int k = 0; k < ldk; ++k) {
      if (k >= 2) be[k] = br[k] / (ar[k] * ar[k - 1]);
      g[k] = (k % kChunk == 0) ? 1.0 : g[k - 1] * ar[k];
    }
    double* ep = &eps[(size_t)r * ldk];
    for (int s = r; s < ldk; ++s)
      ep[s] = std::sqrt(((double)s * s - (double)r * r) / (4.0 * s * s - 1.0));
    sect[r] = std::sqrt((2.0 * r + 3.0) / (2.0 * r + 2.0));
  }
  // 1 / (s (s + 1)) for the psi / chi scaling of the SWE synthesis (-a ilap[s] = 1 / (a lambda_s))
  std::vector<double> ilap(R + 66, 0.0);
  for (int s = 1; s < R + 66; ++s) ilap[s] = 1.0 / ((double)s * (s + 1.0));
  std::vector<int> ck_off(R + 1);
  int nck = 0;
  for (int r = 0; r <= R; ++r) {
    ck_off[r] = nck;
    nck += (R + 2 - r + kChunk - 1) / kChunk;
  }
  std::vector<double2> tw(n_lon);
  for (int e = 0; e < n_lon; ++e) {
    const long double ang = -2.0L * 3.141592653589793238462643383279502884L * e / n_lon;
    tw[e] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  std::vector<int> rev(n_lon);
  for (int k = 0; k < n_lon; ++k) rev[k] = swfft::pad_idx(swfft::digit_rev(P.fft, k));
  {
    int rs = swfft::padded_len(n_lon);
    rs += (9 - rs % 8) % 8;  // == 1 (mod 8) double2 slots: rings differ in bank group
    P.ring_stride = rs;
  }
  // analysis work lists: CTA items (r, first chunk c, checkpoint index of
  // chunk c); items whose first chunk is full come first and the partial last
  // chunks of the rows after them, longest first (stable, so rows stay
  // together), so the short items fill the tail of the last wave
  std::vector<int4> work[2][kAnaSplits];
  for (int which = 0; which < 2; ++which) {
    const int smax = R + which;
    for (int r = 0; r <= R; ++r) {
      const int nout = smax - r + 1;
      p->nchunks[which] += (nout + kChunk - 1) / kChunk;
      for (int ls = 0; ls < kAnaSplits; ++ls) {
        const int cpc = ana_chunks_per_cta(ls + 1);
        for (int c = 0; c * kChunk < nout; c += cpc)
          work[which][ls].push_back(make_int4(r, c, ck_off[r] + c, 0));
      }
    }
    for (int ls = 0; ls < kAnaSplits; ++ls) {
      auto len = [&](const int4& it) { return std::min(kChunk, smax - it.x + 1 - it.y * kChunk); };
      std::stable_sort(work[which][ls].begin(), work[which][ls].end(),
                       [&](const int4& u, const int4& v) { return len(u) > len(v); });
    }
  }

  int st = kOk;
  double* d_ilap = nullptr;
  double *d_mu = nullptr, *d_w = nullptr, *d_beta = nullptr, *d_gsc = nullptr, *d_eps = nullptr,
         *d_a = nullptr, *d_b = nullptr, *d_sect = nullptr;
  int* d_off = nullptr;
  int* d_rev = nullptr;
  double2* d_tw = nullptr;
  if ((st = upload(p, mu_n, &d_mu)) || (st = upload(p, w_n, &d_w)) ||
      (st = upload(p, beta, &d_beta)) || (st = upload(p, gsc, &d_gsc)) ||
      (st = upload(p, eps, &d_eps)) || (st = upload(p, ilap, &d_ilap)) || (st = upload(p, a, &d_a)) || (st = upload(p, b, &d_b)) ||
      (st = upload(p, sect, &d_sect)) || (st = upload(p, ck_off, &d_off)) ||
      (st = upload(p, tw, &d_tw)) || (st = upload(p, rev, &d_rev)) ||
      (st = upload_work(p, work))) {
    swsdc_plan_destroy(p);
    return st;
  }
  for (int i = 0; i < 2; ++i) {
    p->host_work[i].resize(kAnaSplits);
    for (int j = 0; j < kAnaSplits; ++j) {
      p->nwork[i][j] = (int)work[i][j].size();
      p->host_work[i][j] = work[i][j];
    }
  }
  void* ck = nullptr;
  if (cudaMalloc(&ck, sizeof(double2) * (size_t)nck * P.Jh) != cudaSuccess) {
    set_error("cudaMalloc of the checkpoint table failed");
    swsdc_plan_destroy(p);
    return kCuda;
  }
  p->owned.push_back(ck);
  P.mu_n = d_mu;
  P.w_n = d_w;
  P.beta = d_beta;
  P.gsc = d_gsc;
  P.eps = d_eps;
  P.ilap = d_ilap;
  P.ck_off = d_off;
  P.tw = d_tw;
  P.rev = d_rev;
  P.ckpt = reinterpret_cast<double2*>(ck);
  st = build_checkpoints(P, d_a, d_b, d_sect, reinterpret_cast<double2*>(ck), 0);
  // Table-fed analysis: a fragment-native Pbar table (reference-rounded values)
  // replaces the analysis kernel's recurrence when it is small enough to stay
  // L2-resident-ish (SWSDC_TABLES: 0 off, 1 auto; SWSDC_TABLE_MB cap, default
  // 192: T255 on 384 latitudes needs 57 MB, T639 on 960 790 MB).
  {
    static const int tables = env_int("SWSDC_TABLES", 1);
    static const int cap_mb = env_int("SWSDC_TABLE_MB", 192);
    const size_t tab_bytes = sizeof(double) * 128 * (size_t)nck * ((P.Jh + 3) / 4);
    if (st == kOk && tables && tab_bytes <= (size_t)cap_mb * 1024 * 1024) {
      void* tb = nullptr;
      if (cudaMalloc(&tb, tab_bytes) != cudaSuccess || cudaMemset(tb, 0, tab_bytes) != cudaSuccess) {
        cudaGetLastError();
        if (tb) cudaFree(tb);   // no table: the recurrence kernels run instead
      } else {
        p->owned.push_back(tb);
        P.ptab = reinterpret_cast<const double*>(tb);
        st = build_ptab(P, d_a, d_b, d_sect, reinterpret_cast<double*>(tb), 0);
      }
    }
    // the synthesis-order table of the tensor-core synthesis (wide plain batches;
    // opt-in comparison, SWSDC_SYN_DMMA=1: measured slower than the DFMA kernel)
    static const int syn_dmma = env_int("SWSDC_SYN_DMMA", 0);
    const size_t stab_bytes = sizeof(double) * 8 * 128 * (size_t)nck * ((P.Jh + 31) / 32);
    if (st == kOk && tables && syn_dmma && P.Jh <= 256 &&
        stab_bytes <= (size_t)cap_mb * 1024 * 1024) {
      void* tb = nullptr;
      if (cudaMalloc(&tb, stab_bytes) != cudaSuccess || cudaMemset(tb, 0, stab_bytes) != cudaSuccess) {
        cudaGetLastError();
        if (tb) cudaFree(tb);
      } else {
        p->owned.push_back(tb);
        P.stab = reinterpret_cast<const double*>(tb);
        st = build_ptab(P, d_a, d_b, d_sect, reinterpret_cast<double*>(tb), 0, 1);
      }
    }
  }
  if (st == kOk && cudaDeviceSynchronize() != cudaSuccess) {
    set_error("checkpoint build failed");
    st = kCuda;
  }
  if (st != kOk) {
    swsdc_plan_destroy(p);
    return st;
  }
  *out = p;
  return kOk;
}

int swsdc_plan_destroy(swsdc_plan* p) {
  if (!p) return kOk;
  cudaDeviceSynchronize();
  for (void* ptr : p->owned) cudaFree(ptr);
  if (p->ws) cudaFree(p->ws);
  if (p->grid_ws) cudaFree(p->grid_ws);
  for (void* ptr : p->retired) cudaFree(ptr);
  delete p;
  return kOk;
}

int swsdc_plan_config(swsdc_plan* p, int key, int value) {
  if (!p) { set_error("plan is NULL"); return kUsage; }
  if (key == 1) { p->force_split = value != 0; return kOk; }
  set_error("unknown plan option");
  return kUsage;
}

int swsdc_plan_reserve(swsdc_plan* p, int fields) {
  if (!p || fields < 0) { set_error("bad arguments"); return kUsage; }
  // fields ~ 5 per state: the split F_E path needs the grid workspace
  if (!swe_grid_fits(p->dev) || p->force_split ||
      swe_split_preferred(p->dev, (long long)p->dev.Jh * std::max(1, fields / 5))) {
    const size_t need = sizeof(double2) * (size_t)p->dev.I * (p->dev.Jh + 1) * fields;
    bool ok = true;
    SW_TRY(grow_grid_ws(p, need, 0, &ok));
  }
  return ensure_ws(p, 5 * fields, x_bytes_for(p, 7, fields) + x_bytes_for(p, fields, 1),
                   7 * fields);
}

// The public whole-field transforms read every row of their inputs and write every
// row of their outputs, so they refuse an active m-sharding row filter instead of
// silently leaving unowned rows unwritten (the sharded pipeline uses swsdc_fe_*).
static int reject_row_filter(const char* what) {
  if (current_row_filter().mod > 1) {
    set_error(std::string(what) + " under an m-sharding row filter: use the staged swsdc_fe_* calls");
    return kUsage;
  }
  return kOk;
}

int swsdc_synthesize(swsdc_plan* p, const double* coeffs, int r_in, int batch, double* grid,
                     void* stream) {
  if (!p) { set_error("plan is NULL"); return kUsage; }
  SW_TRY(reject_row_filter("synthesize"));
  if (r_in > p->dev.R) {
    set_error("coefficients at truncation " + std::to_string(r_in) +
              " exceed plan truncation " + std::to_string(p->dev.R));
    return kUsage;
  }
  if (r_in < 0 || batch < 0) { set_error("bad truncation or batch"); return kUsage; }
  if (batch == 0) return kOk;
  SW_TRY(ensure_ws(p, batch, 0, 0, S(stream)));
  const PlanDev& P = p->dev;
  const long long fstride = (long long)(P.R + 1) * P.Jh * 2;
  SW_TRY(syn_plain(p, reinterpret_cast<const double2*>(coeffs), r_in, batch, ws_eo(p), S(stream)));
  return launch_fourier_to_grid(P, ws_eo(p), fstride, grid, (long long)P.I * P.J, batch, S(stream));
}

int swsdc_analyze(swsdc_plan* p, const double* grid, int batch, double* coeffs, void* stream) {
  if (!p) { set_error("plan is NULL"); return kUsage; }
  SW_TRY(reject_row_filter("analyze"));
  if (batch < 0) { set_error("bad batch"); return kUsage; }
  if (batch == 0) return kOk;
  SW_TRY(ensure_ws(p, 0, x_bytes_for(p, batch, 1), 0, S(stream)));
  const PlanDev& P = p->dev;
  const XLayout xl = make_xlayout(P.R, P.Jh, batch);
  double* x = ws_x(p, 0);
  SW_TRY(launch_grid_to_fourier(P, 0, grid, nullptr, (long long)P.I * P.J, x, xl, batch,
                                S(stream)));
  const long long plane = (long long)(P.R + 1) * (P.R + 1);
  return ana_run(p, x, xl, 1, reinterpret_cast<double2*>(coeffs), plane, P.R + 1, 0, P.R, true,
                 S(stream));
}

int swsdc_synthesize_uv(swsdc_plan* p, const double* psi, const double* chi, int r_in, int batch,
                        double* u, double* v, void* stream) {
  if (!p) { set_error("plan is NULL"); return kUsage; }
  SW_TRY(reject_row_filter("synthesize_uv"));
  if (r_in > p->dev.R) {
    set_error("coefficients exceed plan truncation");
    return kUsage;
  }
  if (r_in < 0 || batch < 0) { set_error("bad truncation or batch"); return kUsage; }
  if (batch == 0) return kOk;
  SW_TRY(ensure_ws(p, 2 * batch, 0, 0, S(stream)));
  const PlanDev& P = p->dev;
  const long long fstride = (long long)(P.R + 1) * P.Jh * 2;
  const long long cin = (long long)(r_in + 1) * (r_in + 1);
  SynArgs a{};
  a.src = reinterpret_cast<const double2*>(psi);
  a.src2 = reinterpret_cast<const double2*>(chi);
  a.src_fstride = cin;
  a.src_R = r_in;
  a.smax = P.R + 1;
  a.eo = ws_eo(p);
  a.src_mstride = cin;
  a.eo_mstride = 2 * fstride;
  a.nmembers = batch;
  SW_TRY(launch_synthesis(P, a, 2, kSynUV, S(stream)));
  const long long gstride = (long long)P.I * P.J;
  SW_TRY(launch_fourier_to_grid(P, ws_eo(p), 2 * fstride, u, gstride, batch, S(stream)));
  return launch_fourier_to_grid(P, ws_eo(p) + fstride, 2 * fstride, v, gstride, batch, S(stream));
}

int swsdc_analyze_divcurl(swsdc_plan* p, const double* u, const double* v, int batch, double* div,
                          double* curl, void* stream) {
  if (!p) { set_error("plan is NULL"); return kUsage; }
  SW_TRY(reject_row_filter("analyze_divcurl"));
  if (batch < 0) { set_error("bad batch"); return kUsage; }
  if (batch == 0) return kOk;
  const size_t xb = x_bytes_for(p, 4, batch);
  SW_TRY(ensure_ws(p, 0, xb, 4 * batch, S(stream)));
  const PlanDev& P = p->dev;
  const XLayout xl = make_xlayout(P.R, P.Jh, 4);
  double* x = ws_x(p, 0);
  double2* y = ws_y(p, 0, xb);
  SW_TRY(launch_grid_to_fourier(P, 1, u, v, (long long)P.I * P.J, x, xl, batch, S(stream)));
  const long long yv = (long long)(P.R + 1) * p->ldy;
  SW_TRY(ana_run(p, x, xl, batch, y, yv, p->ldy, 4 * yv, P.R + 1, false, S(stream)));
  return launch_finalize_divcurl(P, y, 4 * yv, p->ldy, reinterpret_cast<double2*>(div),
                                 reinterpret_cast<double2*>(curl), batch, S(stream));
}

int swsdc_eval_fe(swsdc_plan* p, const swsdc_params* q, int include_nonlinear, const double* state,
                  int batch, double* out, void* stream) {
  if (!p) { set_error("plan is NULL"); return kUsage; }
  SW_TRY(check_params(q));
  if (batch < 0) { set_error("bad batch"); return kUsage; }
  if (batch == 0) return kOk;
  SW_TRY(reject_row_filter("eval_fe"));
  const bool nl = include_nonlinear != 0;
  const int nv = nl ? 7 : 2;
  const size_t xb = x_bytes_for(p, nv, batch);
  SW_TRY(ensure_ws(p, 5 * batch, xb, nv * batch, S(stream)));
  const PlanDev& P = p->dev;
  const long long fstride = (long long)(P.R + 1) * P.Jh * 2;
  const long long plane = (long long)(P.R + 1) * (P.R + 1);
  const XLayout xl = fe_xlayout(P, nl);
  double2* eo = ws_eo(p);
  double* x = ws_x(p, 5 * batch);
  double2* y = ws_y(p, 5 * batch, xb);
  SynArgs a{};
  a.src = reinterpret_cast<const double2*>(state);
  a.src_fstride = plane;
  a.src_R = P.R;
  a.smax = P.R + 1;
  a.radius = q->radius;
  a.eo = eo;
  a.src_mstride = 3 * plane;
  a.eo_mstride = 5 * fstride;
  a.nmembers = batch;
  SW_TRY(launch_synthesis(P, a, 5, kSynSWE, S(stream)));
  SW_TRY(fe_grid_stage(p, nl, eo, batch, x, xl, q->omega, q->radius, S(stream), 0, P.Jh));
  const long long yv = (long long)(P.R + 1) * p->ldy;
  SW_TRY(ana_run(p, x, xl, batch, y, yv, p->ldy, nv * yv, P.R + 1, false, S(stream)));
  return launch_finalize_swe(P, y, nv * yv, p->ldy, reinterpret_cast<double2*>(out), 3 * plane, nl,
                             q->radius, batch, S(stream));
}

int swsdc_set_row_filter(int mod, int rank) {
  if (mod < 1 || rank < 0 || rank >= mod) { set_error("bad row filter"); return kUsage; }
  set_row_filter(mod, rank);
  return kOk;
}

int swsdc_fe_layout(swsdc_plan* p, int nonlinear, int batch, long long* eo_doubles,
                    long long* x_doubles, int* x_nc, int* x_jh4) {
  if (!p || batch < 0) { set_error("bad arguments"); return kUsage; }
  const PlanDev& P = p->dev;
  const XLayout xl = fe_xlayout(P, nonlinear != 0);
  if (eo_doubles) *eo_doubles = (long long)batch * 5 * (P.R + 1) * P.Jh * 4;
  if (x_doubles) *x_doubles = (long long)batch * xl.mstride;
  if (x_nc) *x_nc = xl.nc;
  if (x_jh4) *x_jh4 = xl.jh4;
  return kOk;
}

int swsdc_fe_synthesis(swsdc_plan* p, const swsdc_params* q, const double* state, int batch,
                       double* eo, void* stream) {
  if (!p) { set_error("plan is NULL"); return kUsage; }
  SW_TRY(check_params(q));
  if (batch <= 0) return batch == 0 ? kOk : kUsage;
  const PlanDev& P = p->dev;
  const long long fstride = (long long)(P.R + 1) * P.Jh * 2;
  const long long plane = (long long)(P.R + 1) * (P.R + 1);
  const swsdc_plan::Shard* sh = shard_for(p);
  SynArgs a{};
  a.src = reinterpret_cast<const double2*>(state);
  a.src_fstride = plane;
  a.src_R = P.R;
  a.smax = P.R + 1;
  a.radius = q->radius;
  a.eo = reinterpret_cast<double2*>(eo);
  a.src_mstride = 3 * plane;
  a.eo_mstride = 5 * fstride;
  a.nmembers = batch;
  if (sh) {
    a.pairs = sh->pairs;
    a.npairs = sh->npairs;
  }
  return launch_synthesis(P, a, 5, kSynSWE, S(stream));
}

int swsdc_fe_grid(swsdc_plan* p, const swsdc_params* q, int include_nonlinear, const double* eo,
                  int batch, int jh_begin, int jh_end, double* x, void* stream) {
  if (!p) { set_error("plan is NULL"); return kUsage; }
  SW_TRY(check_params(q));
  const PlanDev& P = p->dev;
  if (jh_begin < 0 || jh_end > P.Jh || jh_begin > jh_end || batch < 0) {
    set_error("bad latitude-pair range");
    return kUsage;
  }
  if (batch == 0 || jh_begin == jh_end) return kOk;
  const bool nl = include_nonlinear != 0;
  const XLayout xl = fe_xlayout(P, nl);
  const double2* e = reinterpret_cast<const double2*>(eo);
  return fe_grid_stage(p, nl, e, batch, x, xl, q->omega, q->radius, S(stream), jh_begin, jh_end);
}

int swsdc_fe_analysis(swsdc_plan* p, const swsdc_params* q, int include_nonlinear, const double* x,
                      int batch, double* out, void* stream) {
  if (!p) { set_error("plan is NULL"); return kUsage; }
  SW_TRY(check_params(q));
  if (batch <= 0) return batch == 0 ? kOk : kUsage;
  const PlanDev& P = p->dev;
  const bool nl = include_nonlinear != 0;
  const int nv = nl ? 7 : 2;
  SW_TRY(ensure_ws(p, 0, 0, nv * batch, S(stream)));
  const XLayout xl = fe_xlayout(P, nl);
  double2* y = ws_y(p, 0, 0);
  const long long yv = (long long)(P.R + 1) * p->ldy;
  const long long plane = (long long)(P.R + 1) * (P.R + 1);
  SW_TRY(ana_run(p, x, xl, batch, y, yv, p->ldy, nv * yv, P.R + 1, false, S(stream)));
  return launch_finalize_swe(P, y, nv * yv, p->ldy, reinterpret_cast<double2*>(out), 3 * plane, nl,
                             q->radius, batch, S(stream), current_row_filter());
}

int swsdc_eval_fi(int R, const swsdc_params* q, const double* state, int batch, double* out,
                  void* stream) {
  SW_TRY(check_params(q));
  if (R < 0 || batch < 0) { set_error("bad truncation or batch"); return kUsage; }
  if (batch == 0) return kOk;
  return launch_eval_fi(R, consts(q), reinterpret_cast<const double2*>(state),
                        reinterpret_cast<double2*>(out), batch, S(stream));
}

int swsdc_solve_implicit(int R, const swsdc_params* q, double beta, const double* b, int batch,
                         double* out, void* stream) {
  SW_TRY(check_params(q));
  if (beta < 0) { set_error("implicit step must be non-negative"); return kUsage; }
  if (R < 0 || batch < 0) { set_error("bad truncation or batch"); return kUsage; }
  const ModelConsts c = consts(q);
  // implicit.py:330-333: the determinant depends on s only -- check on the host
  for (int s = 0; s <= R; ++s) {
    const double lam = (-(double)s * (s + 1.0)) / (c.radius * c.radius);
    const double d = 1.0 - beta * c.nu * lam;
    const double det = d * d - beta * beta * lam * c.phi_bar;
    if (!(det > 0.0)) {
      set_error("implicit system is singular; invalid model parameters");
      return kNumerical;
    }
  }
  if (batch == 0) return kOk;
  return launch_solve(R, c, beta, reinterpret_cast<const double2*>(b),
                      reinterpret_cast<double2*>(out), batch, S(stream));
}

int swsdc_combine(int n, const double* const* x, const double* w, long long count, double* out,
                  void* stream) {
  if (n < 0 || n > kMaxCombine || count < 0) {
    set_error("combine takes 0..32 inputs");
    return kUsage;
  }
  CombineArgs a{};
  a.n = n;
  a.out = out;
  for (int k = 0; k < n; ++k) {
    a.x[k] = x[k];
    a.w[k] = w[k];
  }
  if (count == 0) return kOk;
  return launch_combine(a, count, S(stream));
}

int swsdc_spec_combine(int n, const double* const* x, const double* w, const int* r_in, int r_out,
                       long long nmat, double* out, void* stream) {
  if (n < 0 || n > kMaxCombine || nmat < 0 || r_out < 0) {
    set_error("spec_combine takes 0..32 inputs");
    return kUsage;
  }
  SpecCombineArgs a{};
  a.n = n;
  a.rout = r_out;
  a.out = reinterpret_cast<double2*>(out);
  for (int k = 0; k < n; ++k) {
    if (r_in[k] < 0) { set_error("bad input truncation"); return kUsage; }
    a.x[k] = reinterpret_cast<const double2*>(x[k]);
    a.w[k] = w[k];
    a.rin[k] = r_in[k];
  }
  if (nmat == 0) return kOk;
  return launch_spec_combine(a, nmat, S(stream));
}

int swsdc_exchange_blocks(double* arr, long long outer, long long rows, long long cols, long long inner,
                          int nblocks, const int* row0, const int* row_step, const int* nrows,
                          const int* col0, const int* col1, double* buf, int scatter,
                          void* stream) {
  if (nblocks < 0 || nblocks > kMaxExBlocks || outer < 0 || rows < 0 || cols < 0 || inner < 1) {
    set_error("exchange_blocks: bad dimensions or more than 64 blocks");
    return kUsage;
  }
  ExchangeBlocks e{};
  e.rows = rows;
  e.cols = cols;
  e.C = inner;
  e.nb = nblocks;
  e.off[0] = 0;
  for (int b = 0; b < nblocks; ++b) {
    const long long last = row0[b] + (long long)(nrows[b] - 1) * row_step[b];
    if (nrows[b] < 0 || col0[b] < 0 || col1[b] < col0[b] || col1[b] > cols || row0[b] < 0 ||
        (nrows[b] > 0 && (last >= rows || last < 0))) {
      set_error("exchange_blocks: block outside the array");
      return kUsage;
    }
    e.row0[b] = row0[b];
    e.row_step[b] = row_step[b];
    e.nrows[b] = nrows[b];
    e.col0[b] = col0[b];
    e.col1[b] = col1[b];
    e.off[b + 1] = e.off[b] + outer * nrows[b] * (long long)(col1[b] - col0[b]) * inner;
  }
  return launch_exchange_blocks(e, arr, buf, scatter != 0, S(stream));
}

int swsdc_copy_finite(const double* src, double* dst, long long n, int* bad, void* stream) {
  if (n < 0 || !bad) { set_error("bad copy_finite arguments"); return kUsage; }
  return launch_copy_finite(src, dst, n, bad, S(stream));
}

int swsdc_spec_combine_multi(int nout, const int* nterms, const double* const* x, const double* w,
                             const int* r_in, int r_out, long long nmat, double* const* outs,
                             const int* ext, void* stream) {
  if (nout < 0 || nout > kMultiOut || nmat < 0 || r_out < 0) {
    set_error("spec_combine_multi takes 0..16 outputs");
    return kUsage;
  }
  MultiCombineArgs a{};
  a.nout = nout;
  a.rout = r_out;
  int k = 0;
  a.off[0] = 0;
  for (int o = 0; o < nout; ++o) {
    if (nterms[o] < 0 || k + nterms[o] > kMultiTerms) {
      set_error("spec_combine_multi takes at most 96 terms in total");
      return kUsage;
    }
    for (int t = 0; t < nterms[o]; ++t, ++k) {
      if (r_in[k] < 0) { set_error("bad input truncation"); return kUsage; }
      a.x[k] = reinterpret_cast<const double2*>(x[k]);
      a.w[k] = w[k];
      a.rin[k] = r_in[k];
    }
    a.off[o + 1] = k;
    a.out[o] = reinterpret_cast<double2*>(outs[o]);
    a.ext[o] = (ext && ext[o] >= 0 && ext[o] < r_out) ? ext[o] : r_out;
  }
  if (nmat == 0 || nout == 0) return kOk;
  return launch_spec_combine_multi(a, nmat, S(stream));
}

int swsdc_sweep_node(int R, const swsdc_params* q, double beta, int n, const double* const* x,
                     const double* w, int batch, double* theta, double* f_i, void* stream) {
  SW_TRY(check_params(q));
  if (beta < 0) { set_error("implicit step must be non-negative"); return kUsage; }
  if (R < 0 || batch < 0 || n < 0 || n > kMaxCombine) { set_error("bad arguments"); return kUsage; }
  const ModelConsts c = consts(q);
  for (int s = 0; s <= R; ++s) {
    const double lam = (-(double)s * (s + 1.0)) / (c.radius * c.radius);
    const double d = 1.0 - beta * c.nu * lam;
    const double det = d * d - beta * beta * lam * c.phi_bar;
    if (!(det > 0.0)) {
      set_error("implicit system is singular; invalid model parameters");
      return kNumerical;
    }
  }
  SpecCombineArgs a{};
  a.n = n;
  a.rout = R;
  for (int k = 0; k < n; ++k) {
    a.x[k] = reinterpret_cast<const double2*>(x[k]);
    a.w[k] = w[k];
    a.rin[k] = R;
  }
  if (batch == 0) return kOk;
  return launch_sweep_node(R, c, beta, a, reinterpret_cast<double2*>(theta),
                           reinterpret_cast<double2*>(f_i), batch, S(stream));
}

int swsdc_resize(const double* in, int r_in, double* out, int r_out, long long nmat, void* stream) {
  if (r_in < 0 || r_out < 0 || nmat < 0) { set_error("bad resize arguments"); return kUsage; }
  if (nmat == 0) return kOk;
  return launch_resize(reinterpret_cast<const double2*>(in), r_in, reinterpret_cast<double2*>(out),
                       r_out, nmat, S(stream));
}

int swsdc_laplacian(const double* in, double* out, int truncation, long long nmat, double radius,
                    int inverse, void* stream) {
  if (!(radius > 0)) { set_error("radius must be positive"); return kUsage; }
  if (truncation < 0 || nmat < 0) { set_error("bad laplacian arguments"); return kUsage; }
  return launch_laplacian(reinterpret_cast<const double2*>(in), reinterpret_cast<double2*>(out),
                          truncation, nmat, radius, inverse != 0, S(stream));
}

// Staircase cover of the s >= r triangle: block k holds rows [r0, r1) and
// columns [r0, R]; one 3D copy (rows x columns x matrices) per block on the copy
// engine.  kStair blocks send 1/2 + 1/(2 kStair) of the dense bytes.
static int stair_blocks() {
  static const int k = std::max(1, env_int("SWSDC_STAIR_BLOCKS", 4));
  return k;
}

static int stair_copy(const double2* src, double2* dst, int R, long long nmat, cudaMemcpyKind kind,
                      cudaStream_t st) {
  const int n = R + 1, K = std::min(stair_blocks(), n);
  const size_t pitch = sizeof(double2) * n;
  for (int k = 0; k < K; ++k) {
    const int r0 = (int)((long long)n * k / K), r1 = (int)((long long)n * (k + 1) / K);
    if (r1 <= r0) continue;
    cudaMemcpy3DParms m{};
    m.srcPtr = make_cudaPitchedPtr(const_cast<double2*>(src), pitch, pitch, n);
    m.dstPtr = make_cudaPitchedPtr(dst, pitch, pitch, n);
    m.srcPos = make_cudaPos(sizeof(double2) * r0, r0, 0);
    m.dstPos = m.srcPos;
    m.extent = make_cudaExtent(sizeof(double2) * (n - r0), r1 - r0, nmat);
    m.kind = kind;
    SW_CUDA(cudaMemcpy3DAsync(&m, st));
  }
  return kOk;
}

// Transfer engines (tuning knobs): 0 = zero-copy kernel, 1 = copy-engine staircase.
// Measured at config 1 (bench.py e2e): strided copy-engine transfers are slow
// host->device (a 5-matrix staircase upload took 130-160 us vs 55 us zero-copy),
// while SM-driven zero-copy traffic slows concurrent transforms; the best mix is
// a zero-copy upload on 32 CTAs and a 4-block staircase download.
static int upload_mode() {
  static const int m = env_int("SWSDC_UPLOAD_MODE", 0);
  return m;
}
static int packed_upload_min_bytes() {
  static const int m = env_int("SWSDC_PACK_MIN_BYTES", 1 << 20);
  return m;
}
static int download_mode() {
  static const int m = env_int("SWSDC_DOWNLOAD_MODE", 1);
  return m;
}

int swsdc_upload_coeffs(const double* host, int r, long long nmat, double* out, void* stream) {
  if (r < 0 || nmat < 0) { set_error("bad upload arguments"); return kUsage; }
  if (nmat == 0) return kOk;
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, const_cast<double*>(host), 0) != cudaSuccess) {
    cudaGetLastError();
    set_error("swsdc_upload_coeffs: source is not page-locked host memory");
    return kUsage;
  }
  if (upload_mode() == 2) {
    // packed upload (hostpack.cu) for transfers worth a copy-engine launch; not
    // capturable (stream memory operation), so a capturing stream takes the kernel
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(S(stream), &cap);
    const size_t bytes = sizeof(double2) * (size_t)nmat * (r + 1) * (r + 2) / 2;
    if (cap == cudaStreamCaptureStatusNone && bytes >= (size_t)packed_upload_min_bytes() &&
        packed_upload_available())
      return launch_upload_packed(reinterpret_cast<const double2*>(host),
                                  reinterpret_cast<double2*>(out), r, nmat, S(stream));
  }
  if (upload_mode() != 1)
    return launch_upload_triangle(reinterpret_cast<const double2*>(dptr),
                                  reinterpret_cast<double2*>(out), r, nmat, S(stream));
  SW_TRY(stair_copy(reinterpret_cast<const double2*>(host), reinterpret_cast<double2*>(out), r, nmat,
                    cudaMemcpyHostToDevice, S(stream)));
  return launch_zero_lower(reinterpret_cast<double2*>(out), r, nmat, S(stream));
}

int swsdc_pack_triangles(const double* dense, int r, long long nmat, double* packed) {
  if (r < 0 || nmat < 0 || (nmat > 0 && (!dense || !packed))) {
    set_error("bad pack arguments");
    return kUsage;
  }
  return pack_triangles_host(reinterpret_cast<const double2*>(dense), r, nmat,
                             reinterpret_cast<double2*>(packed));
}

int swsdc_download_coeffs(const double* dev, int r, long long nmat, double* host, int write_lower,
                          void* stream) {
  if (r < 0 || nmat < 0) { set_error("bad download arguments"); return kUsage; }
  if (nmat == 0) return kOk;
  void* hptr = nullptr;
  if (cudaHostGetDevicePointer(&hptr, host, 0) != cudaSuccess) {
    cudaGetLastError();
    set_error("swsdc_download_coeffs: destination is not page-locked host memory");
    return kUsage;
  }
  if (write_lower) {
    SW_CUDA(cudaMemcpyAsync(host, dev, sizeof(double2) * (size_t)nmat * (r + 1) * (r + 1),
                            cudaMemcpyDeviceToHost, S(stream)));
    return kOk;
  }
  if (download_mode() == 0)
    return launch_download_triangle(reinterpret_cast<const double2*>(dev),
                                    reinterpret_cast<double2*>(hptr), r, nmat, 0, S(stream));
  // the staircase also rewrites a few lower-triangle entries with the device's zeros
  return stair_copy(reinterpret_cast<const double2*>(dev), reinterpret_cast<double2*>(host), r, nmat,
                    cudaMemcpyDeviceToHost, S(stream));
}

}  // extern "C"
