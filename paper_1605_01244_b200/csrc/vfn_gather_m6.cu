// K4 v3: the m = 6 (default cutoff, nufft.py:56) specialisation of the DMMA
// box gather, fully unrolled over the 13 (or 14) x-rows of a box.
//
// Tile (4 x 4 x 4 cells) staging is two TMA loads (cp.async.bulk.tensor.3d)
// of the ghost-padded grid viewed as doubles: z-halves of 8 complex values
// (128 B lines), 16 y-rows, 16 x-rows, 128B-swizzled, completing on an
// mbarrier.  With the swizzle, a lane's B-fragment address inside a line is
// ((4 (kc & 1) + tig) ^ (y & 7)) * 16 B — conflict-free LDS.128 for the 8
// rows x 4 depths a DMMA pair reads — and every offset is a per-unit
// constant plus a compile-time x stride, so the inner body is just
// LDS.128 + 2 DMMA per k-chunk.
//
// Per unit (<= 8 points of one box): rows y are padded from YB = BXY + 12 to
// 16 (two 8-row halves); padded rows read a valid clamped row with weight 0.
//   for x in 0..XB-1, h in {0, 1}:
//     C_re/im[p, y] = sum_kc A[p, 4kc..4kc+3] . G[x, y, 4kc..4kc+3].re/im     (DMMA, axis 3)
//     s[p] += w_y[p, y] C[p, y]                                               (axis 2)
//   acc[p] += w_x[p, x] s[p]                                                  (axis 1)
// which is the reference's contraction order c -> b -> a (nufft.py:269-271).
#include <cuda.h>

#include "vfn_device.cuh"

namespace vfn {

namespace m6 {

constexpr int kUnitPts = 8;
constexpr int kWarps = 8;
constexpr int kTile = 4;             // tile = 4 x 4 x 4 cells
constexpr int kT = kTile + 12;       // staged extent per axis (16)
constexpr int kLine = 128;           // bytes per staged z-half row
constexpr int kHalf = kT * kT * kLine;  // 32 KB per z-half
constexpr int kWtO = 4;              // zero pad before j = 0 in the weights table
constexpr int kWtS = 25;             // weights-table row stride (odd: 4 + 16 + pad)

struct Args {
  const double* u;  // u = z * n per point and axis, input order (from k_map_key)
  const int32_t* perm;
  const int32_t* box_start;
  const int4* items;
  const int32_t* nitems;
  double2* out;
  const double* poly;
  int deg;
  TorusMap tm;
  BinGeom g;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s), "r"(bytes));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(s),
      "r"(parity));
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(d),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(b)
      : "memory");
}

__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

template <int BXY>
__global__ void __launch_bounds__(kWarps * 32, 2)
    k_gather_m6(const __grid_constant__ CUtensorMap tmap, const Args A) {
  constexpr int XB = BXY + 12;  // box rows per axis
  constexpr int YB = BXY + 12;
  constexpr int W = 13;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned tile for the 128B swizzle pattern
  const unsigned raw = (unsigned)__cvta_generic_to_shared(smem_raw);
  const unsigned tile_s = (raw + 1023u) & ~1023u;
  unsigned char* tile_g = smem_raw + (tile_s - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(tile_g + 2 * kHalf);  // 1024-aligned
  double* sWt = reinterpret_cast<double*>(tile_g + 2 * kHalf + 16);  // [kWarps][3][8][kWtS]
  int* sBox = reinterpret_cast<int*>(sWt + kWarps * 3 * kUnitPts * kWtS);  // [bpt + 1]
  int* sUnit = sBox + 33;                                                  // [bpt + 1]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  // window weights table: entry kWtO + j holds phi_j(delta) of point g on an
  // axis, j = 0..12; the pads j in [-kWtO, 0) and [13, 16) stay zero
  for (int i = tid; i < kWarps * 3 * kUnitPts * kWtS; i += blockDim.x) sWt[i] = 0.0;
  // B fragments of the window-polynomial DMMA: C[d][j], d = 4 kc + tig, j = 8 nb + g
  double cb[4][2];
#pragma unroll
  for (int kc = 0; kc < 4; ++kc)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      const int d = 4 * kc + tig, j = 8 * nb + g;
      cb[kc][nb] = (d <= A.deg && j < W) ? A.poly[j * (A.deg + 1) + d] : 0.0;
    }
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();

  const BinGeom& G = A.g;
  double* wt = sWt + warp * 3 * kUnitPts * kWtS;  // [3][8][kWtS]
  const int nitems = *A.nitems;
  unsigned phase = 0;

  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int4 item = A.items[it];
    const int tile = item.x;
    const int t2 = tile % G.ntile[2];
    const int t1 = (tile / G.ntile[2]) % G.ntile[1];
    const int t0 = tile / (G.ntile[2] * G.ntile[1]);
    const int ox = t0 * kTile, oy = t1 * kTile, oz = t2 * kTile;
    __syncthreads();  // everyone is done reading the previous tile
    if (tid == 0) {
      mbar_expect_tx(bar, 2 * kHalf);
      tma_load_3d(tile_g, &tmap, 2 * oz, oy, ox, bar);
      tma_load_3d(tile_g + kHalf, &tmap, 2 * oz + 16, oy, ox, bar);
    }
    if (warp == 0) {
      const int bpt = G.boxes_per_tile;
      const int32_t* bs = A.box_start + (int64_t)tile * bpt;
      int cnt = 0, start = 0;
      if (lane < bpt) {
        start = bs[lane];
        cnt = bs[lane + 1] - start;
      }
      int incl = (cnt + kUnitPts - 1) / kUnitPts;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane < bpt) {
        sBox[lane] = start;
        sUnit[lane + 1] = incl;
      }
      if (lane == 0) sUnit[0] = 0;
      if (lane == bpt - 1) sBox[bpt] = start + cnt;
    }
    __syncthreads();

    bool waited = false;
    for (int u = item.y + warp; u < item.z; u += kWarps) {
      int b = 0;
      while (sUnit[b + 1] <= u) ++b;
      const int p0 = sBox[b] + (u - sUnit[b]) * kUnitPts;
      const int cnt = min(kUnitPts, sBox[b + 1] - p0);
      constexpr int NB = kTile / BXY;  // boxes per tile along x and y (z: 1)
      const int by = b % NB, bx = b / NB;
      const int X0 = bx * BXY, Y0 = by * BXY;

      // point g of the unit: nearest cell and offset from u (nufft.py:256-257)
      const bool valid = g < cnt;
      int64_t prow = 0;
      double uu[3] = {0.0, 0.0, 0.0};
      if (valid) {
        prow = __ldg(A.perm + p0 + g);
#pragma unroll
        for (int d = 0; d < 3; ++d) uu[d] = __ldg(A.u + 3 * prow + d);
      }
      int cell[3];
      double dl[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) cell[d] = cell_from_u(uu[d], A.tm.nd[d], A.tm.n[d], dl[d]);
      // offsets inside the box; idle lanes (and out-of-domain points, whose
      // key is 0) are pinned to 0 so every table index stays in bounds
      const bool inbox = valid && cell[0] - ox - X0 >= 0 && cell[0] - ox - X0 < BXY &&
                         cell[1] - oy - Y0 >= 0 && cell[1] - oy - Y0 < BXY &&
                         cell[2] - oz >= 0 && cell[2] - oz < kTile;
      const int ci = inbox ? cell[0] - ox - X0 : 0;
      const int cj = inbox ? cell[1] - oy - Y0 : 0;
      const int ck = inbox ? cell[2] - oz : 0;
      // window weights of point g on all three axes by DMMA:
      // W[p, j] = sum_d delta_p^d C[d, j]   (A = powers of delta, B = coefficients)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double x1 = dl[d], x2 = x1 * x1, x4 = x2 * x2;
        double pw = tig == 0 ? 1.0 : (tig == 1 ? x1 : (tig == 2 ? x2 : x2 * x1));
        double w00 = 0.0, w01 = 0.0, w10 = 0.0, w11 = 0.0;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          dmma(w00, w01, pw, cb[kc][0]);
          dmma(w10, w11, pw, cb[kc][1]);
          pw *= x4;
        }
        double* row = wt + (d * kUnitPts + g) * kWtS + kWtO;
        row[2 * tig] = w00;
        row[2 * tig + 1] = w01;
        if (8 + 2 * tig < W) row[8 + 2 * tig] = w10;  // j = 13..15 stay zero
        if (9 + 2 * tig < W) row[9 + 2 * tig] = w11;
      }
      __syncwarp();
      const double* w0 = wt + (0 * kUnitPts + g) * kWtS + kWtO - ci;  // w0[x]: axis 1
      const double* w1 = wt + (1 * kUnitPts + g) * kWtS + kWtO - cj;  // w1[y]: axis 2
      const double* w2 = wt + (2 * kUnitPts + g) * kWtS + kWtO - ck;  // w2[k]: axis 3
      double a[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) a[kc] = inbox ? w2[4 * kc + tig] : 0.0;
      double wy[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int y = 8 * h + 2 * tig + e;
          wy[h][e] = y < YB ? w1[y] : 0.0;
        }
      // B-fragment row of this lane per half: y = 8h + g (clamped into the box)
      unsigned off[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int y = Y0 + min(8 * h + g, YB - 1);
        const int sw = y & 7;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc)
          off[h][kc] = tile_s + (kc >> 1) * kHalf + (X0 * kT + y) * kLine +
                       16 * (((kc & 1) * 4 + tig) ^ sw);
      }
      if (!waited) {
        mbar_wait(bar, phase);
        waited = true;
      }
      double acc_re = 0.0, acc_im = 0.0;
#pragma unroll
      for (int x = 0; x < XB; ++x) {
        double sre = 0.0, sim = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double cr0 = 0.0, cr1 = 0.0, ci0 = 0.0, ci1 = 0.0;
#pragma unroll
          for (int kc = 0; kc < 4; ++kc) {
            const double2 v = lds128(off[h][kc] + x * kT * kLine);
            dmma(cr0, cr1, a[kc], v.x);
            dmma(ci0, ci1, a[kc], v.y);
          }
          sre = fma(wy[h][0], cr0, sre);
          sre = fma(wy[h][1], cr1, sre);
          sim = fma(wy[h][0], ci0, sim);
          sim = fma(wy[h][1], ci1, sim);
        }
        const double w = w0[x];
        acc_re = fma(w, sre, acc_re);
        acc_im = fma(w, sim, acc_im);
      }
      acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 1);
      acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 1);
      acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 2);
      acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 2);
      if (valid && tig == 0) A.out[prow] = make_double2(acc_re, acc_im);
      __syncwarp();
    }
    if (!waited) mbar_wait(bar, phase);  // keep the phase bookkeeping uniform
    phase ^= 1u;
  }
}

}  // namespace m6

// Tensor map over the ghost-padded grid as doubles: (2 P2, P1, P0), box
// (16 doubles, 16, 16), 128B swizzle.
int make_grid_tmap(vfn_plan* p) {
  p->has_tmap = false;
  if (p->m != 6) return VFN_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      fn == nullptr) {
    cudaGetLastError();
    return VFN_OK;  // no TMA: generic gather
  }
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  cuuint64_t dims[3] = {(cuuint64_t)(2 * p->P[2]), (cuuint64_t)p->P[1], (cuuint64_t)p->P[0]};
  cuuint64_t strides[2] = {(cuuint64_t)(2 * p->P[2] * 8), (cuuint64_t)(2 * p->P[2] * 8 * p->P[1])};
  cuuint32_t box[3] = {16, (cuuint32_t)m6::kT, (cuuint32_t)m6::kT};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<Fn>(fn)(&p->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, p->grid, dims,
                                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(VFN_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  p->has_tmap = true;
  return VFN_OK;
}

size_t m6_smem_bytes(int deg) {
  size_t b = 1024 + 2 * m6::kHalf;
  b += 16 + sizeof(double) * m6::kWarps * 3 * m6::kUnitPts * m6::kWtS;
  b += sizeof(int) * (33 + 34);
  return b;
}

template <int BXY>
static int launch(vfn_plan* p, const m6::Args& A, cudaStream_t s) {
  const size_t smem = m6_smem_bytes(p->poly.deg);
  VFN_CUDA(cudaFuncSetAttribute(m6::k_gather_m6<BXY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  int dev = 0, nsm = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  VFN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, m6::k_gather_m6<BXY>,
                                                         m6::kWarps * 32, smem));
  if (per_sm < 1) return fail(VFN_ERR_INVALID, "m=6 gather does not fit on an SM");
  m6::k_gather_m6<BXY><<<nsm * per_sm, m6::kWarps * 32, smem, s>>>(p->tmap, A);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

bool m6_applicable(const vfn_plan* p, const BinGeom& g) {
  return p->m == 6 && p->has_tmap && p->poly.deg <= 15 && g.tile[0] == 4 && g.tile[1] == 4 && g.tile[2] == 4 &&
         g.box[2] == 4 && g.box[0] == g.box[1] && (g.box[0] == 1 || g.box[0] == 2);
}

int launch_m6(vfn_plan* p, const double* u, const int32_t* perm, const int32_t* box_start,
              const int4* items, const int32_t* nitems, double2* out, const BinGeom& g,
              cudaStream_t s) {
  m6::Args A;
  A.u = u;
  A.perm = perm;
  A.box_start = box_start;
  A.items = items;
  A.nitems = nitems;
  A.out = out;
  A.poly = p->poly.dev;
  A.deg = p->poly.deg;
  A.tm = p->map;
  A.g = g;
  return g.box[0] == 1 ? launch<1>(p, A, s) : launch<2>(p, A, s);
}

}  // namespace vfn
