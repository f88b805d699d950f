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
  const double2* ckpt;    // [sum_r nchunk(r)][Jh] (q_{s0}, q_{s0+1}) chunk seeds
  const int* ck_off;      // [R+1] first chunk index of row r in ckpt
  const double2* tw;      // [I] exp(-2 pi i e / I)
  swfft::FftPlan fft;
};

__host__ __device__ inline int jn_of(const PlanDev& p, int jh) { return p.J - p.Jh + jh; }
__host__ __device__ inline int js_of(const PlanDev& p, int jh) { return p.J - 1 - jn_of(p, jh); }

}  // namespace swsdc
