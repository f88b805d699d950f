// Packed host -> device upload of spectral matrices (SWSDC_UPLOAD_MODE=2, opt-in).
// Measured slower than the zero-copy upload on this pool's hosts: out of cache the 16
// host cores pack 7.9 MB in 240-390 us (~30 GB/s), more than the transfer it feeds
// (profiles/r02/experiments.md), so the default stays SWSDC_UPLOAD_MODE=0.
//
// The reference layout keeps (R+1)^2 dense matrices on the host of which only the
// s >= r triangle is populated (spharm.py:6-10).  PCIe only runs full duplex for
// contiguous copy-engine transfers (profiles/r02/experiments.md: SM zero-copy reads
// or pitched copy-engine reads share the link with a concurrent download at ~29 GB/s
// each way, contiguous copies reach ~47), so this path
//   1. packs the triangles into a contiguous page-locked staging buffer with a
//      persistent pool of host threads -- off the issuing thread, which only
//      enqueues work and returns (the source must stay unmodified until the stream
//      reaches the copy, the cudaMemcpyAsync contract),
//   2. gates the stream on the pack with a stream memory operation
//      (cuStreamWaitValue32 on a page-locked flag the last packing thread sets): no
//      host function on the stream, no blocked issuing thread,
//   3. moves the staging buffer with ONE contiguous copy-engine transfer, and
//   4. expands it on the device into the dense layout (lower triangle zero).
// Staging slots rotate (kSlots).  A slot is reused only after its previous pack has
// finished and the event recorded behind its previous copy has completed: the
// issuing thread waits for both, which bounds how far it can run ahead of the
// transfers (kSlots batches) and keeps CUDA calls off the packing threads.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>

#include "common.cuh"
#include "spectral.cuh"

namespace swsdc {
namespace {

constexpr int kSlots = 4;

inline int grid_1d(long long n, int threads) {
  return (int)std::min<long long>((n + threads - 1) / threads, 148LL * 16);
}

// element offset of row r inside one packed triangle of truncation R
__host__ __device__ inline long long tri_off(int R, int r) {
  return (long long)r * (2 * R + 3 - r) / 2;
}

struct PackJob {
  const double2* src = nullptr;   // dense host matrices
  double2* dst = nullptr;         // packed staging (page-locked)
  int R = 0;
  long long nmat = 0;
  volatile uint32_t* flag = nullptr;
  uint32_t seq = 0;
  int nslices = 1;
  std::atomic<int> remaining{0};
};

// Pack the packed-element range [e0, e1) of the job.
void pack_range(const PackJob& j, long long e0, long long e1) {
  const int R = j.R, n = R + 1;
  const long long T1 = (long long)n * (n + 1) / 2;
  long long e = e0;
  while (e < e1) {
    const long long m = e / T1, w = e - m * T1;
    // row holding packed offset w: largest r with tri_off(r) <= w
    int lo = 0, hi = R;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tri_off(R, mid) <= w) lo = mid; else hi = mid - 1;
    }
    int r = lo;
    long long c = w - tri_off(R, r);   // entries of row r already covered
    const double2* sm = j.src + m * (long long)n * n;
    double2* dm = j.dst + m * T1;
    long long wpos = w;
    const long long wend = std::min(T1, w + (e1 - e));
    while (wpos < wend) {
      const long long len = std::min<long long>(n - r - c, wend - wpos);
      std::memcpy(dm + wpos, sm + (long long)r * n + r + c, sizeof(double2) * (size_t)len);
      wpos += len;
      c = 0;
      ++r;
    }
    e += wend - w;
  }
}

class PackPool {
 public:
  static PackPool& get() {
    static PackPool* p = new PackPool();   // leaked: threads die with the process
    return *p;
  }
  int threads() const { return nthreads_; }
  void submit(PackJob* job) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (int s = 0; s < job->nslices; ++s) q_.push_back({job, s});
    }
    cv_.notify_all();
  }

 private:
  struct Item { PackJob* job; int slice; };
  PackPool() {
    int n = env_int("SWSDC_PACK_THREADS", 0);
    if (n <= 0) {
      const unsigned hw = std::thread::hardware_concurrency();
      n = (int)std::min(16u, std::max(2u, hw / 2));
    }
    nthreads_ = n;
    for (int i = 0; i < n; ++i) std::thread([this] { run(); }).detach();
  }
  void run() {
    for (;;) {
      Item it;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return !q_.empty(); });
        it = q_.front();
        q_.pop_front();
      }
      PackJob* j = it.job;
      const long long T1 = (long long)(j->R + 1) * (j->R + 2) / 2, total = T1 * j->nmat;
      const long long e0 = total * it.slice / j->nslices, e1 = total * (it.slice + 1) / j->nslices;
      pack_range(*j, e0, e1);
      if (j->remaining.fetch_sub(1, std::memory_order_acq_rel) == 1) {
        std::atomic_thread_fence(std::memory_order_seq_cst);
        *j->flag = j->seq;   // releases the stream (cuStreamWaitValue32 GEQ seq)
        delete j;
      }
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Item> q_;
  int nthreads_ = 0;
};

__global__ void __launch_bounds__(256) unpack_triangle_kernel(const double2* __restrict__ packed,
                                                              double2* __restrict__ out, int R,
                                                              long long total) {
  pdl_wait();
  pdl_trigger();
  const int n = R + 1;
  const long long T1 = (long long)n * (n + 1) / 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride) {
    const long long m = i / ((long long)n * n);
    const int rs = (int)(i - m * (long long)n * n);
    const int r = rs / n, s = rs - r * n;
    double2 v = make_double2(0.0, 0.0);
    if (s >= r) v = packed[m * T1 + tri_off(R, r) + (s - r)];
    out[i] = v;
  }
}

typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WaitValue32Fn wait_value_fn() {
  static WaitValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    cudaGetLastError();
    return reinterpret_cast<WaitValue32Fn>(p);
  }();
  return fn;
}

struct Slot {
  double2* host = nullptr;
  double2* dev = nullptr;
  size_t bytes = 0;
  cudaEvent_t copied = nullptr, unpacked = nullptr;
  bool used = false;
  uint32_t last_seq = 0;   // sequence number of the slot's latest pack
};

struct Uploader {
  std::mutex mu;
  Slot slots[kSlots];
  uint32_t* flags = nullptr;      // page-locked, one word per slot
  CUdeviceptr flags_dev = 0;
  uint32_t seq = 0;
  int device = -1;
};

Uploader& uploader_for(int device) {
  static std::mutex mu;
  static std::vector<Uploader*> all;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)all.size() <= device) all.resize(device + 1, nullptr);
  if (!all[device]) {
    all[device] = new Uploader();
    all[device]->device = device;
  }
  return *all[device];
}

}  // namespace

bool packed_upload_available() { return wait_value_fn() != nullptr; }

// Host-only: pack with the pool and wait (the packed layout's definition, testable
// without a device): matrix m, row r, column s >= r -> m T1 + tri_off(r) + s - r.
int pack_triangles_host(const double2* dense, int R, long long nmat, double2* packed) {
  if (nmat == 0) return kOk;
  PackPool& pool = PackPool::get();
  volatile uint32_t done = 0;
  PackJob* job = new PackJob();
  job->src = dense;
  job->dst = packed;
  job->R = R;
  job->nmat = nmat;
  job->flag = &done;
  job->seq = 1;
  const long long bytes = (long long)sizeof(double2) * nmat * (R + 1) * (R + 2) / 2;
  job->nslices = (int)std::max<long long>(1, std::min<long long>(pool.threads(), bytes >> 16));
  job->remaining.store(job->nslices);
  pool.submit(job);
  while (done == 0) std::this_thread::yield();
  std::atomic_thread_fence(std::memory_order_seq_cst);
  return kOk;
}

int launch_upload_packed(const double2* host, double2* out, int R, long long nmat, cudaStream_t st) {
  WaitValue32Fn wait_value = wait_value_fn();
  if (!wait_value) { set_error("packed upload: cuStreamWaitValue32 is unavailable"); return kCuda; }
  int device = 0;
  SW_CUDA(cudaGetDevice(&device));
  Uploader& u = uploader_for(device);
  std::lock_guard<std::mutex> lk(u.mu);
  if (!u.flags) {
    SW_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&u.flags), sizeof(uint32_t) * kSlots,
                          cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(u.flags, 0, sizeof(uint32_t) * kSlots);
    void* d = nullptr;
    SW_CUDA(cudaHostGetDevicePointer(&d, u.flags, 0));
    u.flags_dev = reinterpret_cast<CUdeviceptr>(d);
    u.seq = 0;
  }
  const long long T1 = (long long)(R + 1) * (R + 2) / 2;
  const size_t bytes = sizeof(double2) * (size_t)(T1 * nmat);
  const uint32_t seq = ++u.seq;
  const int si = (int)(seq % kSlots);
  Slot& s = u.slots[si];
  if (!s.copied) {
    SW_CUDA(cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming));
    SW_CUDA(cudaEventCreateWithFlags(&s.unpacked, cudaEventDisableTiming));
  }
  if (s.bytes < bytes) {
    // the slot's previous transfer must be over before its buffers go away
    if (s.used) SW_CUDA(cudaEventSynchronize(s.unpacked));
    if (s.host) cudaFreeHost(s.host);
    if (s.dev) cudaFree(s.dev);
    s.host = nullptr; s.dev = nullptr; s.bytes = 0;
    SW_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.host), bytes, cudaHostAllocPortable));
    SW_CUDA(cudaMalloc(reinterpret_cast<void**>(&s.dev), bytes));
    s.bytes = bytes;
  }
  if (s.used) {
    // previous pack into this slot finished, previous copy out of it complete
    volatile uint32_t* f = u.flags + si;
    while ((int32_t)(*f - s.last_seq) < 0) std::this_thread::yield();
    SW_CUDA(cudaEventSynchronize(s.copied));
  }
  PackPool& pool = PackPool::get();
  PackJob* job = new PackJob();
  job->src = host;
  job->dst = s.host;
  job->R = R;
  job->nmat = nmat;
  job->flag = u.flags + si;
  job->seq = seq;
  job->nslices = (int)std::max<long long>(1, std::min<long long>(pool.threads(), (long long)(bytes >> 16)));
  job->remaining.store(job->nslices);
  // the device staging buffer may still feed the previous unpack on another stream
  if (s.used) SW_CUDA(cudaStreamWaitEvent(st, s.unpacked, 0));
  pool.submit(job);
  {
    StageScope sc("upload", st);
    const CUresult cr = wait_value(reinterpret_cast<CUstream>(st), u.flags_dev + sizeof(uint32_t) * si,
                                   seq, CU_STREAM_WAIT_VALUE_GEQ);
    if (cr != CUDA_SUCCESS) {
      // the job still runs to completion and frees itself; nothing waits for it
      set_error("cuStreamWaitValue32 failed (" + std::to_string((int)cr) + ")");
      return kCuda;
    }
    SW_CUDA(cudaMemcpyAsync(s.dev, s.host, bytes, cudaMemcpyHostToDevice, st));
    SW_CUDA(cudaEventRecord(s.copied, st));
    const long long n = nmat * (long long)(R + 1) * (R + 1);
    SW_CUDA(launch_pdl(unpack_triangle_kernel, dim3(grid_1d(n, 256)), dim3(256), 0, st,
                       (const double2*)s.dev, out, R, n));
    SW_LAUNCH_CHECK();
    SW_CUDA(cudaEventRecord(s.unpacked, st));
  }
  s.used = true;
  s.last_seq = seq;
  return kOk;
}

}  // namespace swsdc
