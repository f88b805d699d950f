// Shared device-side definitions for the B200 MLSDC-SH hot path.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "fft_core.cuh"

namespace swsdc {

// Legendre recurrence chunk length (steps in total degree per checkpoint).
constexpr int kChunk = 32;

// Status codes of the C ABI (include/swsdc_b200.h).
enum Status : int { kOk = 0, kUsage = 1, kNumerical = 2, kCuda = 3 };

void set_error(const std::string& msg);

#define SW_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      ::swsdc::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));           \
      return ::swsdc::kCuda;                                                            \
    }                                                                                   \
  } while (0)

#define SW_LAUNCH_CHECK()                                                               \
  do {                                                                                  \
    cudaError_t _e = cudaGetLastError();                                                \
    if (_e != cudaSuccess) {                                                            \
      ::swsdc::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e));      \
      return ::swsdc::kCuda;                                                            \
    }                                                                                   \
  } while (0)

#define SW_TRY(expr)                      \
  do {                                    \
    int _s = (expr);                      \
    if (_s != ::swsdc::kOk) return _s;    \
  } while (0)

// Raise a kernel's dynamic shared-memory limit once per (kernel, device) and
// size growth instead of on every launch (profile.cu).
int set_max_dyn_smem(const void* kern, size_t smem);
int set_smem_carveout_max(const void* kern);
// Integer tuning knob from the environment, `dflt` when unset; callers cache it
// in a function-local static so the environment is read once per process.
int env_int(const char* name, int dflt);

// Programmatic dependent launch (PDL).  Library kernels are launched with
// launch_pdl, which lets a kernel's CTAs be scheduled while its stream
// predecessor drains; every kernel begins with pdl_wait() (returns once the
// predecessor grid has completed and its writes are visible; a no-op without
// PDL) followed by pdl_trigger() (lets our own dependents launch as soon as all
// our CTAs are resident).  SWSDC_PDL=0 disables the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Explicit early trigger (SWSDC_PDL_EARLY builds): measured to cost config 2
// ~7% (dependents land unevenly during the predecessor's tail), so by default
// dependents launch as the predecessor's CTAs exit.
__device__ __forceinline__ void pdl_trigger() {
#ifdef SWSDC_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
}
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// launch_pdl plus a 1-D thread-block cluster of `cluster_x` CTAs along x.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                      cudaStream_t st, unsigned cluster_x, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// RAII bracket of one kernel launch: counts it and, when profiling is on,
// records CUDA events around it on `st` (profile.cu).
class StageScope {
 public:
  StageScope(const char* name, cudaStream_t st);
  ~StageScope();
  StageScope(const StageScope&) = delete;
  StageScope& operator=(const StageScope&) = delete;

 private:
  int idx_;
  cudaStream_t st_;
};

// Read-only device view of one transform plan (passed by value to kernels).
//
// Latitude indexing: jh in [0, Jh), Jh = ceil(J/2).  The "north" latitude of
// half-index jh is jn = J - Jh + jh (mu >= 0), its mirror js = J - 1 - jn.
// For odd J, jh = 0 is the equator (jn == js).
struct PlanDev {
  int R;        // triangular truncation
  int I;        // n_lon
  int J;        // n_lat
  int Jh;       // ceil(J/2)
  int ldk;      // row stride of the per-(r, k) tables (>= R + 2 + kChunk + 4)
  const double* mu_n;     // [Jh] mu at the north latitude of each pair
  const double* w_n;      // [Jh] Gauss weight (symmetric)
  const double* beta;     // [(R+1) * ldk] scaled-recurrence coefficient beta[r][k], k = s - r
  const double* gsc;      // [(R+1) * ldk] scale g[r][k] relative to the chunk start
  const double* eps;      // [(R+1) * ldk] eps[r][s] = sqrt((s^2 - r^2) / (4 s^2 - 1)), index s
  const double* ilap;     // [R + 66] 1 / (s (s + 1)) (s >= 1), 0 at s = 0: -a^2 / lambda_s / a^2
  const double2* ckpt;    // [sum_r nchunk(r)][Jh] (q_{s0}, q_{s0+1}) chunk seeds
  const int* ck_off;      // [R+1] first chunk index of row r in ckpt
  const double* ptab;     // [nck][jh4][128] Pbar A fragments (table-fed analysis) or nullptr
  const double* stab;     // [nck][ceil(Jh/32)][8][128] Pbar B fragments (tensor-core synthesis) or nullptr
  const double2* tw;      // [I] exp(-2 pi i e / I)
  const int* rev;         // [I] padded ring slot of frequency k (digit-reversed DIF order)
  int ring_stride;        // double2 slots per ring in shared memory (== 1 mod 8)
  swfft::FftPlan fft;
};

// Layout of the analysis input x (written by fourier.cu, read by the DMMA
// analysis): vectors in groups of 16; per group, for each (r, block of 4
// latitudes jb, parity p in {S, D}), nc = 8*NT real columns (re/im of each
// vector) x 4 latitudes -- exactly one m8n8k4 B fragment per (jb, p, n-tile),
// so a warp loads it with one coalesced 256-byte access.
//
// pm (pair-major, the F_E path): inside each (r, jb, p) block of nc x 4
// doubles the latitude is the slow index -- [t][n] instead of [n][t] -- so
// the nc columns of one latitude pair are contiguous (whole 32-byte sectors
// written by the pair's own CTA, no cluster exchange); the analysis kernel
// re-orders them into its fragment ring (ana_item<..., PM>).
struct XLayout {
  int nv;          // vectors
  int nc;          // columns per group (8 * n-tiles of a full group)
  int jh4;         // ceil(Jh / 4)
  long long gstride;  // doubles per group of 16 vectors
  long long mstride;  // doubles per member
  int pm;          // pair-major blocks
  __host__ __device__ size_t idx(int v, int comp, int r, int jh, int p) const {
    const int g = v >> 4, n = 2 * (v & 15) + comp;
    const size_t blk = (size_t)g * gstride + (((size_t)r * jh4 + (jh >> 2)) * 2 + p) * nc * 4;
    return pm ? blk + (size_t)(jh & 3) * nc + n : blk + (size_t)n * 4 + (jh & 3);
  }
};

inline XLayout make_xlayout(int R, int Jh, int nv, bool pair_major = false) {
  XLayout L;
  L.pm = pair_major ? 1 : 0;
  L.nv = nv;
  const int nfull = nv < 16 ? nv : 16;
  L.nc = 8 * ((2 * nfull + 7) / 8);
  L.jh4 = (Jh + 3) / 4;
  L.gstride = (long long)(R + 1) * L.jh4 * 2 * L.nc * 4;
  L.mstride = L.gstride * ((nv + 15) / 16);
  return L;
}

__host__ __device__ inline int jn_of(const PlanDev& p, int jh) { return p.J - p.Jh + jh; }
__host__ __device__ inline int js_of(const PlanDev& p, int jh) { return p.J - 1 - jn_of(p, jh); }

}  // namespace swsdc
