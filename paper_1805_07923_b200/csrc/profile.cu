// Launch accounting and optional per-stage CUDA-event timing.
//
// Every kernel launch site opens a StageScope: it always bumps the launch
// counter (bench.py reports it as gpu_launches) and, when profiling is
// enabled, brackets the launch with two events on the launching stream so
// bench.py can measure each stage's device time live inside its timed region
// (roofline "achieved").  Profiling must be off during CUDA graph capture.
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace swsdc {
namespace {

struct Rec {
  const char* name;
  cudaEvent_t a, b;
};

std::atomic<long long> g_launches{0};
std::atomic<bool> g_prof{false};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

bool pdl_enabled() {
  static const bool on = env_int("SWSDC_PDL", 1) != 0;
  return on;
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Prefer the largest shared-memory carveout (228 KB of the 256 KB L1/smem) for a
// kernel whose occupancy is smem-limited (otherwise the driver may pick 168 KB).
int set_smem_carveout_max(const void* kern) {
  static const int knob = env_int("SWSDC_CARVEOUT", 1);
  if (!knob) return kOk;
  static std::mutex mu;
  static std::map<const void*, bool> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done[kern]) return kOk;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             (int)cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute(carveout): ") + cudaGetErrorString(e));
    return kCuda;
  }
  done[kern] = true;
  return kOk;
}

int set_max_dyn_smem(const void* kern, size_t smem) {
  if (smem <= 48 * 1024) return kOk;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{kern, dev}];
  if (have >= smem) return kOk;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
  if (e != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return kCuda;
  }
  have = smem;
  return kOk;
}

StageScope::StageScope(const char* name, cudaStream_t st) : idx_(-1), st_(st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> lk(g_mu);
  Rec r{name, take_event(), take_event()};
  cudaEventRecord(r.a, st);
  g_recs.push_back(r);
  idx_ = (int)g_recs.size() - 1;
}

StageScope::~StageScope() {
  if (idx_ < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(g_recs[idx_].b, st_);
}

}  // namespace swsdc

using namespace swsdc;

extern "C" {

long long swsdc_launch_count(void) { return g_launches.load(); }

int swsdc_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& r : g_recs) {
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  g_prof.store(on != 0);
  return kOk;
}

// Waits for the recorded events and writes "name<TAB>launches<TAB>total_ms\n"
// lines (aggregated by stage name) into buf.  Returns the bytes needed.
int swsdc_profile_collect(char* buf, int buflen) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::map<std::string, std::pair<long long, double>> agg;
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& e = agg[r.name];
    e.first += 1;
    e.second += ms;
  }
  std::string out;
  for (auto& kv : agg) {
    char line[256];
    snprintf(line, sizeof(line), "%s\t%lld\t%.6f\n", kv.first.c_str(), kv.second.first,
             kv.second.second);
    out += line;
  }
  if (buf && buflen > 0) {
    const int n = (int)out.size() < buflen - 1 ? (int)out.size() : buflen - 1;
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int)out.size() + 1;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// FP64 peak probe (roofline denominator measured live on the bench box):
// 8 independent DFMA chains per thread, 148 x 8 CTAs x 128 threads.  DMMA
// reaches the same rate on sm_100a (profiles/fp64_peak_r01.txt).
// ---------------------------------------------------------------------------
namespace swsdc {
constexpr int kProbeIters = 4096;
__global__ void fp64_probe_kernel(double* sink, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < kProbeIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) sink[threadIdx.x] = s;
}
}  // namespace swsdc

extern "C" int swsdc_probe_fp64(int reps, double* tflops) {
  double* sink = nullptr;
  SW_CUDA(cudaMalloc(&sink, 1024 * sizeof(double)));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 16, threads = 128;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) fp64_probe_kernel<<<blocks, threads>>>(sink, 0.999999, 1e-7);
  cudaEventRecord(e0);
  for (int w = 0; w < reps; ++w) fp64_probe_kernel<<<blocks, threads>>>(sink, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  SW_LAUNCH_CHECK();
  const double flops = 2.0 * 8 * kProbeIters * (double)blocks * threads * reps;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return kOk;
}
