// Microbenchmarks that calibrate the gather-kernel design on B200 (sm_100a):
//   1. DFMA peak (vector FP64 pipe)
//   2. DMMA peak (mma.sync m8n8k4 f64, the only FP64 tensor op on sm_100a)
//   3. shared-memory LDS.128 feeding DFMA, with 1 / 4 / 32 distinct addresses
//      per warp instruction (broadcast vs per-lane) — the K4 inner loop shape.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_fp64 microbench_fp64.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void dfma_peak(double* out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  double b = s, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 12345.678) out[0] = r;
}

__global__ void dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
      }
    }
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
  if (r == 12345.678) out[0] = r;
}

// lanes = points; each lane holds 14 weights per point; per "row" 14 complex
// grid values are loaded from smem. DIST = number of distinct addresses per
// warp instruction (1 = full broadcast, 4 = per 8-lane group, 32 = per lane).
// PPL = points per lane (each loaded value feeds 2*PPL DFMA).
template <int DIST, int PPL>
__global__ void lds_dfma(double* out, int rows) {
  extern __shared__ double2 sg[];  // 8192 double2 = 128 KB
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sg[i] = make_double2(i * 1e-3, -i * 1e-3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int grp = (DIST == 1) ? 0 : (lane / (32 / DIST));
  double w[PPL][14];
#pragma unroll
  for (int p = 0; p < PPL; ++p)
#pragma unroll
    for (int c = 0; c < 14; ++c) w[p][c] = 1.0 / (1 + c + p + lane);
  double ar[PPL], ai[PPL];
#pragma unroll
  for (int p = 0; p < PPL; ++p) { ar[p] = 0; ai[p] = 0; }
  unsigned base = (threadIdx.x >> 5) * 97;
  for (int r = 0; r < rows; ++r) {
    // distinct groups 16 double2 apart -> different bank quads
    unsigned idx = ((base + r * 29u) & 4095u) * 1u + grp;
#pragma unroll
    for (int c = 0; c < 14; ++c) {
      double2 g = sg[(idx + c) & 8191u];
#pragma unroll
      for (int p = 0; p < PPL; ++p) {
        ar[p] = fma(w[p][c], g.x, ar[p]);
        ai[p] = fma(w[p][c], g.y, ai[p]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int p = 0; p < PPL; ++p) s += ar[p] + ai[p];
  if (s == 12345.678) out[0] = s;
}

// pure LDS.128 throughput
template <int DIST>
__global__ void lds_only(double* out, int rows) {
  extern __shared__ double2 sg[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sg[i] = make_double2(i * 1e-3, -i * 1e-3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int grp = (DIST == 1) ? 0 : (lane / (32 / DIST));
  double ar = 0, ai = 0;
  unsigned base = (threadIdx.x >> 5) * 97;
  for (int r = 0; r < rows; ++r) {
    unsigned idx = ((base + r * 29u) & 4095u) + grp;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      double2 g = sg[(idx + c) & 8191u];
      ar += g.x; ai -= g.y;  // DADD on a cheap chain; issue-bound test
    }
  }
  if (ar + ai == 12345.678) out[0] = ar;
}


// DMMA with the B operand (grid values) streamed from smem: LDW = doubles per
// lane per LDS (1 -> LDS.64 per DMMA, 2 -> LDS.128 per 2 DMMAs); A (weights)
// held in registers across 4 K-chunks; NACC independent accumulators.
template <int LDW>
__global__ void dmma_lds(double* out, int rows) {
  extern __shared__ double sgd[];  // 16384 doubles = 128 KB
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sgd[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double a[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = 1.0 / (1 + k + lane);
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
  unsigned base = (threadIdx.x >> 5) * 389;
  for (int r = 0; r < rows; ++r) {
    unsigned idx = (((base + r * 131u) & 8191u) & ~1u) + lane * LDW;
    // one "row tile": 4 K-chunks x 4 accumulators = 16 DMMA
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      double b[4];
      if (LDW == 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) b[k] = sgd[(idx + (t * 4 + k) * 64) & 16383u];
      } else {
#pragma unroll
        for (int k = 0; k < 4; k += 2) {
          double2 v = *reinterpret_cast<const double2*>(&sgd[(idx + (t * 4 + k) * 64) & 16382u]);
          b[k] = v.x; b[k + 1] = v.y;
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a[k]), "d"(b[k]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}


// DMMA latency: one warp per SM, NCH independent dependent-chains
template <int NCH>
__global__ void dmma_lat(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[NCH][2];
#pragma unroll
  for (int i = 0; i < NCH; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) r += c[i][0] + c[i][1];
  if (r == 12345.678) out[0] = r;
}


// Do DMMA and DFMA share the FP64 datapath?  Warps with (warp % 2 == 0) run
// DMMA chains, the others DFMA chains; MODE 0 = both, 1 = DMMA warps only, 2 = DFMA only
template <int MODE>
__global__ void mixed_fp64(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  const bool is_mma = (warp & 1) == 0;
  double r = 0;
  if (is_mma && MODE != 2) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) { c[i][0] = i; c[i][1] = -i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) r += c[i][0] + c[i][1];
  } else if (!is_mma && MODE != 1) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    // 16 DMMA-equivalents of work per iteration = 16*256/32 = 128 FMA per lane
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999, 1e-9);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) r += a[i];
  }
  if (r == 12345.678) out[0] = r;
}

template <typename K>
float time_kernel(K kern, dim3 grid, dim3 block, size_t smem, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  kern(grid, block, smem);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) kern(grid, block, smem);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int nsm = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"smem_per_sm\": %zu, \"l2\": %d, \"clock_khz\": %d}\n",
         prop.name, nsm, prop.sharedMemPerMultiprocessor, prop.l2CacheSize, clk_khz);
  double* d; CK(cudaMalloc(&d, 64));

  // DFMA
  {
    int iters = 4000; dim3 g(nsm * 8), blk(256);
    float ms = time_kernel([&](dim3 g, dim3 b, size_t s) { dfma_peak<<<g, b, s>>>(d, iters, 0.999999); }, g, blk, 0, 5);
    double flops = 2.0 * 8 * 16 * (double)iters * g.x * blk.x;
    printf("{\"test\": \"dfma_peak\", \"ms\": %.4f, \"tflops\": %.3f, \"dfma_per_clk_per_sm_at_max\": %.2f}\n",
           ms, flops / ms / 1e9, flops / 2 / (ms * 1e-3) / nsm / (clk_khz * 1e3));
  }
  // DMMA
  {
    int iters = 2000; dim3 g(nsm * 8), blk(256);
    float ms = time_kernel([&](dim3 g, dim3 b, size_t s) { dmma_peak<<<g, b, s>>>(d, iters); }, g, blk, 0, 5);
    double flops = 2.0 * 256 * 8 * 4 * (double)iters * g.x * (blk.x / 32);
    printf("{\"test\": \"dmma_peak\", \"ms\": %.4f, \"tflops\": %.3f}\n", ms, flops / ms / 1e9);
  }
  size_t smem = 8192 * sizeof(double2);
#define RUN_LD(DIST, PPL)                                                                     \
  {                                                                                           \
    CK(cudaFuncSetAttribute(lds_dfma<DIST, PPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                            (int)smem));                                                      \
    int rows = 4000; dim3 g(nsm), blk(512);                                                   \
    float ms = time_kernel([&](dim3 g, dim3 b, size_t s) { lds_dfma<DIST, PPL><<<g, b, s>>>(d, rows); }, g, blk, smem, 5); \
    double flops = 2.0 * 2 * PPL * 14 * (double)rows * g.x * blk.x;                           \
    printf("{\"test\": \"lds_dfma\", \"distinct\": %d, \"ppl\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", DIST, PPL, ms, flops / ms / 1e9); \
  }
  RUN_LD(1, 1) RUN_LD(8, 1) RUN_LD(32, 1) RUN_LD(1, 2) RUN_LD(8, 2) RUN_LD(32, 2) RUN_LD(1, 4) RUN_LD(8, 4) RUN_LD(32, 4)
#define RUN_LO(DIST)                                                                          \
  {                                                                                           \
    CK(cudaFuncSetAttribute(lds_only<DIST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    int rows = 4000; dim3 g(nsm), blk(512);                                                   \
    float ms = time_kernel([&](dim3 g, dim3 b, size_t s) { lds_only<DIST><<<g, b, s>>>(d, rows); }, g, blk, smem, 5); \
    double ld = 16.0 * rows * g.x * (blk.x / 32);                                             \
    printf("{\"test\": \"lds_only\", \"distinct\": %d, \"ms\": %.4f, \"warp_lds_per_clk_per_sm\": %.3f}\n", DIST, ms, ld / (ms * 1e-3) / nsm / (clk_khz * 1e3)); \
  }
  RUN_LO(1) RUN_LO(2) RUN_LO(8) RUN_LO(16) RUN_LO(32)

#define RUN_DL(LDW)                                                                           \
  {                                                                                           \
    CK(cudaFuncSetAttribute(dmma_lds<LDW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    int rows = 2000; dim3 g(nsm), blk(512);                                                   \
    float ms = time_kernel([&](dim3 g, dim3 b, size_t s) { dmma_lds<LDW><<<g, b, s>>>(d, rows); }, g, blk, smem, 5); \
    double flops = 2.0 * 256 * 16 * (double)rows * g.x * (blk.x / 32);                        \
    printf("{\"test\": \"dmma_lds\", \"ldw\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", LDW, ms, flops / ms / 1e9); \
  }
  RUN_DL(1) RUN_DL(2)

#define RUN_LAT(NCH, WARPS)                                                                   \
  {                                                                                           \
    int iters = 20000; dim3 g(nsm), blk(32 * WARPS);                                          \
    float ms = time_kernel([&](dim3 g, dim3 b, size_t s) { dmma_lat<NCH><<<g, b, s>>>(d, iters); }, g, blk, 0, 3); \
    double per = ms * 1e-3 * clk_khz * 1e3 / iters;                                           \
    printf("{\"test\": \"dmma_lat\", \"chains\": %d, \"warps_per_sm\": %d, \"cycles_per_iter\": %.2f, \"cycles_per_dmma_per_warp\": %.2f}\n", NCH, WARPS, per, per / NCH); \
  }
  RUN_LAT(1, 1) RUN_LAT(2, 1) RUN_LAT(4, 1) RUN_LAT(8, 1) RUN_LAT(1, 4) RUN_LAT(2, 4) RUN_LAT(4, 4) RUN_LAT(1, 16) RUN_LAT(2, 16)

#define RUN_MIX(MODE)                                                                         \
  {                                                                                           \
    int iters = 4000; dim3 g(nsm), blk(512);                                                  \
    float ms = time_kernel([&](dim3 g, dim3 b, size_t s) { mixed_fp64<MODE><<<g, b, s>>>(d, iters); }, g, blk, 0, 3); \
    double fl_mma = (MODE != 2) ? 2.0 * 256 * 16 * (double)iters * g.x * 8 : 0;               \
    double fl_fma = (MODE != 1) ? 2.0 * 128 * 32 * (double)iters * g.x * 8 : 0;               \
    printf("{\"test\": \"mixed_fp64\", \"mode\": %d, \"ms\": %.3f, \"tflops_total\": %.2f}\n", MODE, ms, (fl_mma + fl_fma) / ms / 1e9); \
  }
  RUN_MIX(0) RUN_MIX(1) RUN_MIX(2)
  return 0;
}
