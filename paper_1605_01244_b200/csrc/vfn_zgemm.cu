// Complex double GEMM on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64),
// hand-written for the exact separable passes of the rectilinear evaluation
// (K5, rectilinear.py:59-64) and the axis-3 contraction of the NDFT (K6,
// nufft.py:141-148):
//
//   C[b][m, n] = sum_k A[b][m, k] B[b][k, n]      (complex128, FMA chains in k order)
//
// A is row-major (A[m lda + k]); B is row-major K x N (B[k ldb + n]) or, with
// bt, stored N x K (B[n ldb + k], the basis matrices E_d[m, k] used as E^T).
//
// Tiles: 64 x 64 complex outputs per CTA of 8 warps (2 x 4, each 32 x 16 =
// 4 x 2 DMMA tiles), K staged 16 at a time by cp.async into a 2-stage ring.
// Shared rows are 20 complex (320 B) long, so the 8 rows x 4 k of a fragment
// hit both bank halves evenly (conflict-free LDS.128), the same line pitch as
// the gather's tiles.  B tiles are stored n-major (transposed on the way in
// for a row-major B) so A and B fragments load alike.  One LDS.128 gives an
// element's (re, im); each complex product is 4 real DMMAs:
//   C.re += A.re B.re - A.im B.im,   C.im += A.re B.im + A.im B.re.
#include "vfn_device.cuh"

namespace vfn {

namespace zg {

constexpr int BM = 64, BN = 64, BK = 16, LD = 20;  // tile sizes (complex), smem row pitch
constexpr int kThreads = 256;
constexpr int kStageElems = (BM + BN) * LD;        // complex per stage (A then B)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 16-byte async copy global -> shared; src_bytes = 0 zero-fills
__device__ __forceinline__ void cp16(unsigned dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

template <bool BT>
__device__ __forceinline__ void load_stage(const ZGemm& g, const double2* __restrict__ A, const double2* __restrict__ B,
                                           int64_t m0, int64_t n0, int64_t k0, unsigned st) {
  const int tid = threadIdx.x;
  const unsigned as = st, bs = st + BM * LD * 16;
#pragma unroll
  for (int i = 0; i < (BM * BK) / kThreads; ++i) {
    const int idx = tid + i * kThreads;
    const int r = idx / BK, c = idx % BK;
    const bool ok = m0 + r < g.M && k0 + c < g.K;
    const double2* src = ok ? A + (m0 + r) * g.lda + (k0 + c) : A;
    cp16(as + (unsigned)(r * LD + c) * 16u, src, ok ? 16 : 0);
  }
#pragma unroll
  for (int i = 0; i < (BN * BK) / kThreads; ++i) {
    const int idx = tid + i * kThreads;
    int n, c;
    if (BT) {
      n = idx / BK;
      c = idx % BK;
    } else {
      c = idx / BN;
      n = idx % BN;
    }
    const bool ok = n0 + n < g.N && k0 + c < g.K;
    const double2* src = ok ? (BT ? B + (n0 + n) * g.ldb + (k0 + c) : B + (k0 + c) * g.ldb + (n0 + n)) : B;
    cp16(bs + (unsigned)(n * LD + c) * 16u, src, ok ? 16 : 0);
  }
}

template <bool BT>
__global__ void __launch_bounds__(kThreads, 2) k_zgemm(const ZGemm g) {
  extern __shared__ __align__(16) unsigned char zsm[];
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(zsm);
  const int64_t bz = blockIdx.z;
  const double2* __restrict__ A = g.A + bz * g.sA;
  const double2* __restrict__ B = g.B + bz * g.sB;
  double2* __restrict__ C = g.C + bz * g.sC;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int gq = lane >> 2, t = lane & 3;
  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  const int nk = (int)((g.K + BK - 1) / BK);
  const unsigned stage_bytes = kStageElems * 16u;
  load_stage<BT>(g, A, B, m0, n0, 0, sbase);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  // fragment addresses inside a stage (bytes): A row wm*32 + 8i + gq, B row wn*16 + 8j + gq, col t
  const unsigned a_off = (unsigned)(((wm * 32 + gq) * LD + t) * 16);
  const unsigned b_off = (unsigned)((BM * LD + (wn * 16 + gq) * LD + t) * 16);
  for (int kt = 0; kt < nk; ++kt) {
    if (kt + 1 < nk) {
      load_stage<BT>(g, A, B, m0, n0, (int64_t)(kt + 1) * BK, sbase + ((kt + 1) & 1) * stage_bytes);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const unsigned st = sbase + (kt & 1) * stage_bytes;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double2 af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = lds128(st + a_off + (unsigned)((i * 8 * LD + kk) * 16));
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = lds128(st + b_off + (unsigned)((j * 8 * LD + kk) * 16));
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double nai = -af[i].y;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], af[i].x, bf[j].x);
          dmma(cr[i][j][0], cr[i][j][1], nai, bf[j].y);
          dmma(ci[i][j][0], ci[i][j][1], af[i].x, bf[j].y);
          dmma(ci[i][j][0], ci[i][j][1], af[i].y, bf[j].x);
        }
      }
    }
    __syncthreads();  // the stage is refilled two iterations later
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + wm * 32 + i * 8 + gq;
    if (row >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t col = n0 + wn * 16 + j * 8 + 2 * t + e;
        if (col < g.N) C[row * g.ldc + col] = make_double2(cr[i][j][e], ci[i][j][e]);
      }
  }
}

}  // namespace zg

int zgemm(const ZGemm& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return VFN_OK;
  const size_t smem = 2 * zg::kStageElems * sizeof(double2);
  const int64_t gx = (g.N + zg::BN - 1) / zg::BN, gy = (g.M + zg::BM - 1) / zg::BM;
  if (gy > 65535 || g.batch > 65535 || gx > INT32_MAX) return fail(VFN_ERR_INVALID, "zgemm: grid too large");
  const dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)g.batch);
  if (g.bt) {
    VFN_CUDA(cudaFuncSetAttribute(zg::k_zgemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    zg::k_zgemm<true><<<grid, zg::kThreads, smem, s>>>(g);
  } else {
    VFN_CUDA(cudaFuncSetAttribute(zg::k_zgemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    zg::k_zgemm<false><<<grid, zg::kThreads, smem, s>>>(g);
  }
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

}  // namespace vfn
