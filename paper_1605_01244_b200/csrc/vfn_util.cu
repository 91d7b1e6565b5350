// Roofline denominator: sustained FP64 FMA throughput of this device,
// measured with an independent-chain DFMA kernel over all SMs (bench.py).
#include <vector>

#include "vfn_internal.cuh"

namespace vfn {

__global__ void k_dfma_peak(double* out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, c);
    }
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1234.5678) out[0] = r;
}

}  // namespace vfn

using namespace vfn;

extern "C" int vfn_bench_fp64_peak(int device, double seconds, double* tflops, double* sm_clock_mhz) {
  if (!tflops) return fail(VFN_ERR_INVALID, "null argument");
  DeviceGuard guard(device);
  int nsm = 0, clk = 0;
  VFN_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  VFN_CUDA(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device));
  double* d = nullptr;
  VFN_CUDA(cudaMalloc(&d, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = nsm * 8, iters = 2000;
  k_dfma_peak<<<blocks, threads>>>(d, iters, 0.999999);  // warm up
  cudaDeviceSynchronize();
  double flops_per_launch = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  int reps = 0;
  float total_ms = 0.f;
  cudaEventRecord(e0);
  do {
    k_dfma_peak<<<blocks, threads>>>(d, iters, 0.999999);
    ++reps;
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&total_ms, e0, e1);
  } while (total_ms < seconds * 1e3 && reps < 100000);
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (err != cudaSuccess) return fail(VFN_ERR_CUDA, cudaGetErrorString(err));
  *tflops = flops_per_launch * reps / (total_ms * 1e-3) / 1e12;
  if (sm_clock_mhz) *sm_clock_mhz = clk / 1e3;
  return VFN_OK;
}

namespace vfn {

// *dst = *src by one device thread; dst is mapped pinned host memory, so the
// host reads the word after the stream synchronises without a copy-engine D2H
// (reset: src is restored to the 0x7f.. sentinel for the next call)
__global__ void k_store_word(int64_t* __restrict__ src, volatile int64_t* dst, bool reset) {
  *dst = *src;
  if (reset) *src = 0x7f7f7f7f7f7f7f7fLL;
  __threadfence_system();
}

int store_word(int64_t* src, int64_t* dst, cudaStream_t s, bool reset) {
  k_store_word<<<1, 1, 0, s>>>(src, dst, reset);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

}  // namespace vfn

namespace vfn {

namespace {
struct PoolEntry {
  int device;
  void* ptr;
  size_t bytes;
};
std::mutex g_pool_mu;
std::vector<PoolEntry> g_pool;
constexpr int kPoolKeep = 4;  // buffers kept per device (a grid, a coefficient staging buffer, ...)
}  // namespace

void* pool_alloc(int device, size_t bytes, size_t* got) {
  {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    // the smallest cached buffer that fits without wasting more than 1/4
    int best = -1;
    for (int i = 0; i < (int)g_pool.size(); ++i) {
      const PoolEntry& e = g_pool[i];
      if (e.device == device && e.bytes >= bytes && e.bytes - bytes <= bytes / 4 &&
          (best < 0 || e.bytes < g_pool[best].bytes))
        best = i;
    }
    if (best >= 0) {
      void* p = g_pool[best].ptr;
      *got = g_pool[best].bytes;
      g_pool.erase(g_pool.begin() + best);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    vfn_pool_release(device);  // retry once without the cached buffers
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
  }
  *got = bytes;
  return p;
}

void pool_free(int device, void* ptr, size_t bytes) {
  if (!ptr) return;
  void* evict = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    int held = 0, oldest = -1;
    for (int i = 0; i < (int)g_pool.size(); ++i)
      if (g_pool[i].device == device) {
        if (oldest < 0) oldest = i;
        ++held;
      }
    if (held >= kPoolKeep) {
      evict = g_pool[oldest].ptr;
      g_pool.erase(g_pool.begin() + oldest);
    }
    g_pool.push_back({device, ptr, bytes});
  }
  if (evict) cudaFree(evict);
}

}  // namespace vfn

extern "C" int vfn_pool_release(int device) {
  std::vector<void*> drop;
  {
    std::lock_guard<std::mutex> lock(vfn::g_pool_mu);
    for (auto it = vfn::g_pool.begin(); it != vfn::g_pool.end();) {
      if (device < 0 || it->device == device) {
        drop.push_back(it->ptr);
        it = vfn::g_pool.erase(it);
      } else {
        ++it;
      }
    }
  }
  for (void* p : drop) cudaFree(p);
  return VFN_OK;
}
