// K4 v2: the general binned gather on the FP64 tensor cores (DMMA,
// mma.sync m8n8k4 f64) for the cutoffs the tensor-core gather of
// vfn_gather_tc.cu does not cover (m = 1, 8..13) and for planes without
// TMA; the box counts / offsets built here feed both.
//
// Points arrive sorted by gather box: a box is bi x bj x bk
// cells, bk = K - 2m with K = 4*KC the DMMA k-extent (16 at m = 7, so boxes
// are 2 cells deep).  A "unit" is up to 8 points of one box.  For a unit, the
// innermost contraction of the reference (axis 3, nufft.py:269) becomes a
// dense product
//     S[p, r] = sum_k  W2[p, k] * G[r, k]          p < 8 points, k < K,
// over the box's rows r = (x, y) (all (bi+2m)(bj+2m) of them), with W2[p, .]
// the point's 2m+1 axis-3 window weights placed at its offset inside the box
// (zeros elsewhere).  One m8n8k4 DMMA takes A = W2 (8 points x 4 k), B = four
// complex rows (8 real rows x 4 k) straight from the shared-memory tile, and
// accumulates C = 8 points x 8 real rows.  The remaining two contractions
// (axis 2 then axis 1, nufft.py:270-271) are applied to C in registers with
// the rows' window product w1[x] * w2[y] and reduced across the quad.
//
// CTA work item = (staging tile, range of units); the tile's grid block
// (TI+2m) x (TJ+2m) x (TK+2m) complex values is staged into shared memory with
// cp.async from the ghost-padded grid, so the periodic seam needs no modulo.
// Persistent CTAs stride over the item list built by k_tile_units/k_items.
#include <algorithm>

#include <cub/device/device_scan.cuh>

#include "vfn_device.cuh"

namespace vfn {

constexpr int kUnitPts = 8;      // points per unit (DMMA M)
constexpr int kItemUnits = 32;   // units per work item (load balance, clustered inputs)
constexpr int kWarps = 8;        // warps per CTA
constexpr int kMaxRowW = 32;     // max bi + 2m (smem weight rows per point)
constexpr int kMaxBoxes = 32;    // boxes per tile handled by one warp scan

struct GatherArgs {
  const double* pts;
  const int32_t* perm;
  const int32_t* box_start;   // nboxes + 1
  const int4* items;          // (tile, unit_begin, unit_end, -)
  const int32_t* nitems;      // device scalar
  const double2* grid;        // ghost-padded grid
  double2* out;
  const double* poly;
  int deg, m;
  int64_t P1, P2;
  TorusMap tm;
  BinGeom g;
  int X, Y, Z, SZ;            // smem tile extents (Z padded to SZ)
  int WS;                     // per-point weight row stride (odd)
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

template <int KC>
__global__ void __launch_bounds__(kWarps * 32, 2) k_gather_dmma(GatherArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sG = reinterpret_cast<double2*>(smem_raw);
  const size_t gbytes = (size_t)A.X * A.Y * A.SZ * sizeof(double2);
  double* sPoly = reinterpret_cast<double*>(smem_raw + gbytes);
  const int W = 2 * A.m + 1;
  const int npoly = W * (A.deg + 1);
  double* sW = sPoly + ((npoly + 1) & ~1);  // per warp: [2][8][WS]
  int* sBox = reinterpret_cast<int*>(sW + kWarps * 2 * kUnitPts * A.WS);
  int* sUnit = sBox + (kMaxBoxes + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  for (int i = tid; i < npoly; i += blockDim.x) sPoly[i] = A.poly[i];

  const BinGeom& G = A.g;
  const int bi = G.box[0], bj = G.box[1], bk = G.box[2];
  const int XB = bi + 2 * A.m, YB = bj + 2 * A.m;  // box row extents
  const int R = XB * YB;                           // complex rows per box
  const int NT = (R + 7) >> 3;                     // 8-row DMMA tiles
  const int WS = A.WS;                             // odd stride: conflict-free per-point rows
  double* w0 = sW + warp * 2 * kUnitPts * WS;      // [8][WS] axis-1 weights of the unit's points
  double* w1 = w0 + kUnitPts * WS;                 // [8][WS] axis-2 weights
  const int nitems = *A.nitems;
  const int XY = A.X * A.Y;

  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int4 item = A.items[it];
    const int64_t tile = item.x;
    const int t2 = (int)(tile % G.ntile[2]);
    const int t1 = (int)((tile / G.ntile[2]) % G.ntile[1]);
    const int t0 = (int)(tile / ((int64_t)G.ntile[2] * G.ntile[1]));
    const int64_t ox = (int64_t)t0 * G.tile[0], oy = (int64_t)t1 * G.tile[1],
                  oz = (int64_t)t2 * G.tile[2];
    __syncthreads();  // previous item's readers are done with sG / sBox
    // stage the tile's padded-grid block (P-index ox + x, oy + y, oz + z):
    // warp w copies rows w, w + kWarps, ...; lanes cover z
    {
      int x = warp / A.Y, y = warp % A.Y;
      const int dx = kWarps / A.Y, dy = kWarps % A.Y;
      for (int r = warp; r < XY; r += kWarps) {
        const double2* src = A.grid + ((ox + x) * A.P1 + (oy + y)) * A.P2 + oz;
        double2* dst = sG + (size_t)r * A.SZ;
        VFN_DCHECK(x < A.X && y < A.Y && oy + y < A.P1 && oz + A.Z <= A.P2);
        for (int z = lane; z < A.Z; z += 32) cp_async16(dst + z, src + z);
        x += dx;
        y += dy;
        if (y >= A.Y) { y -= A.Y; ++x; }
      }
    }
    if (warp == 0) {
      const int bpt = G.boxes_per_tile;
      const int32_t* bs = A.box_start + tile * bpt;
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
    cp_async_wait_all();
    __syncthreads();

    for (int u = item.y + warp; u < item.z; u += kWarps) {
      // unit -> box b and chunk within the box
      int b = 0;
      while (sUnit[b + 1] <= u) ++b;
      const int chunk = u - sUnit[b];
      const int p0 = sBox[b] + chunk * kUnitPts;
      const int cnt = min(kUnitPts, sBox[b + 1] - p0);
      // box origin inside the tile (cells == smem coordinates of row offset 0)
      const int bz = b % G.nbox[2];
      const int by = (b / G.nbox[2]) % G.nbox[1];
      const int bx = b / (G.nbox[2] * G.nbox[1]);
      const int X0 = bx * bi, Y0 = by * bj, Z0 = bz * bk;

      // lane quad g owns point g of the unit
      const bool valid = g < cnt;
      int cell[3] = {0, 0, 0};
      double dl[3] = {0.0, 0.0, 0.0};
      int64_t prow = 0;
      if (valid) {
        prow = A.perm[p0 + g];
#pragma unroll
        for (int d = 0; d < 3; ++d)
          cell[d] = nearest_cell(__ldg(A.pts + 3 * prow + d), A.tm.a[d], A.tm.amb[d], A.tm.nd[d],
                                 A.tm.n[d], dl[d]);
      }
      const int ci = cell[0] - (int)ox - X0;  // offsets of the point inside its box
      const int cj = cell[1] - (int)oy - Y0;
      const int ck = cell[2] - (int)oz - Z0;
      VFN_DCHECK(!valid || (ci >= 0 && ci < bi && cj >= 0 && cj < bj && ck >= 0 && ck < bk));
      // A fragment: axis-3 weights of point g at box depth k = 4 kc + tig
      double a[KC];
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int j = 4 * kc + tig - ck;
        a[kc] = (valid && j >= 0 && j < W) ? window_poly(sPoly, A.deg, j, dl[2]) : 0.0;
      }
      for (int x = tig; x < XB; x += 4) {
        const int j = x - ci;
        w0[g * WS + x] = (valid && j >= 0 && j < W) ? window_poly(sPoly, A.deg, j, dl[0]) : 0.0;
      }
      for (int y = tig; y < YB; y += 4) {
        const int j = y - cj;
        w1[g * WS + y] = (valid && j >= 0 && j < W) ? window_poly(sPoly, A.deg, j, dl[1]) : 0.0;
      }
      __syncwarp();

      // 8-row tiles.  B fragment of this lane: complex row rb = 8t + g, one
      // LDS.128 of (re, im) at depth 4 kc + tig feeds the re- and im-DMMA.
      // C fragment of this lane: point g, complex rows rc = 8t + 2 tig + {0, 1}.
      int rbx = 0, rby = g;
      while (rby >= YB) { rby -= YB; ++rbx; }
      int rcx = 0, rcy = 2 * tig;
      while (rcy >= YB) { rcy -= YB; ++rcx; }
      const double* wg0 = w0 + g * WS;
      const double* wg1 = w1 + g * WS;
      const double2* gz = sG + Z0 + tig;
      double acc_re = 0.0, acc_im = 0.0;
#pragma unroll 2
      for (int t = 0; t < NT; ++t) {
        const int rb = 8 * t + g;
        const double2* bp = gz + (rb < R ? ((X0 + rbx) * A.Y + (Y0 + rby)) * A.SZ : 0);
        VFN_DCHECK(bp >= sG && bp + 4 * (KC - 1) < sG + (size_t)A.X * A.Y * A.SZ);
        double cr0 = 0.0, cr1 = 0.0, ci0 = 0.0, ci1 = 0.0;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          const double2 v = bp[4 * kc];
          dmma(cr0, cr1, a[kc], v.x);
          dmma(ci0, ci1, a[kc], v.y);
        }
        // rows rc and rc + 1 of point g: window product w1[x] * w2[y]
        const int rc = 8 * t + 2 * tig;
        int x1 = rcx, y1 = rcy + 1;
        if (y1 >= YB) { y1 -= YB; ++x1; }
        const double wa = rc < R ? wg0[rcx] * wg1[rcy] : 0.0;
        const double wb = rc + 1 < R ? wg0[x1] * wg1[y1] : 0.0;
        acc_re = fma(wa, cr0, acc_re);
        acc_im = fma(wa, ci0, acc_im);
        acc_re = fma(wb, cr1, acc_re);
        acc_im = fma(wb, ci1, acc_im);
        // advance both row cursors by 8 rows
        rby += 8;
        while (rby >= YB) { rby -= YB; ++rbx; }
        rcy += 8;
        while (rcy >= YB) { rcy -= YB; ++rcx; }
      }
      acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 1);
      acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 1);
      acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 2);
      acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 2);
      if (valid && tig == 0) A.out[prow] = make_double2(acc_re, acc_im);
      __syncwarp();  // w0/w1 are rewritten by the next unit
    }
  }
}

// ------------------------------------------------------------------ work items

// Box offsets from the SORTED keys without atomics: the last position i of
// every run of equal boxes writes i + 1 (the number of points in boxes <= its
// own) into tails[box]; an inclusive max-scan of tails then gives
// box_start[b + 1] for every box, empty ones included (clustered inputs
// leave millions of empty boxes between a handful of runs, so nothing here
// loops over a gap).  Eight positions per thread (two 16-byte key loads).
__global__ void k_box_tails(const uint32_t* __restrict__ keys, int64_t M, uint32_t key_slots,
                            int32_t* __restrict__ tails) {
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i0 >= M) return;
  uint32_t k[9];
  if (i0 + 8 <= M) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(keys + i0));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(keys + i0) + 1);
    k[0] = a.x, k[1] = a.y, k[2] = a.z, k[3] = a.w, k[4] = b.x, k[5] = b.y, k[6] = b.z, k[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) k[j] = i0 + j < M ? keys[i0 + j] : 0u;
  }
  k[8] = i0 + 8 < M ? keys[i0 + 8] : 0u;
  uint32_t box = k[0] / key_slots;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t i = i0 + j;
    if (i >= M) break;
    const bool last = i + 1 == M;
    const uint32_t next = last ? 0u : k[j + 1] / key_slots;
    if (last || next != box) tails[box] = (int32_t)(i + 1);
    box = next;
  }
}

__global__ void k_tile_units(const int32_t* __restrict__ box_start, int64_t ntiles, int bpt,
                             int32_t* __restrict__ nitems) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  if (t == ntiles) {
    nitems[t] = 0;
    return;
  }
  const int32_t* bs = box_start + t * bpt;
  int units = 0;
  for (int b = 0; b < bpt; ++b) units += (bs[b + 1] - bs[b] + kUnitPts - 1) / kUnitPts;
  nitems[t] = (units + kItemUnits - 1) / kItemUnits;
}

__global__ void k_items(const int32_t* __restrict__ box_start, const int32_t* __restrict__ item_off,
                        int64_t ntiles, int bpt, int4* __restrict__ items) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int first = item_off[t], n = item_off[t + 1] - first;
  if (n == 0) return;
  const int32_t* bs = box_start + t * bpt;
  int units = 0;
  for (int b = 0; b < bpt; ++b) units += (bs[b + 1] - bs[b] + kUnitPts - 1) / kUnitPts;
  for (int j = 0; j < n; ++j)
    items[first + j] = make_int4((int)t, j * kItemUnits, min(units, (j + 1) * kItemUnits), 0);
}

static size_t dmma_smem_bytes(int X, int Y, int SZ, int m, int deg, int WS) {
  const int W = 2 * m + 1;
  size_t b = (size_t)X * Y * SZ * sizeof(double2);
  b += sizeof(double) * (((W * (deg + 1)) + 1) & ~1);
  b += sizeof(double) * kWarps * 2 * kUnitPts * WS;
  b += sizeof(int) * 2 * (kMaxBoxes + 1);
  return b;
}

template <int KC>
static int launch_dmma(const GatherArgs& A, size_t smem, cudaStream_t s) {
  VFN_CUDA(cudaFuncSetAttribute(k_gather_dmma<KC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                200 * 1024));
  int dev = 0, nsm = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  VFN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_dmma<KC>, kWarps * 32, smem));
  if (per_sm < 1) return fail(VFN_ERR_INVALID, "DMMA gather does not fit on an SM");
  k_gather_dmma<KC><<<nsm * per_sm, kWarps * 32, smem, s>>>(A);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

int gather_boxes(vfn_plan* p, const double* pts, int64_t M, const BinGeom& g,
                 const uint32_t* keys_sorted, const int32_t* perm, double2* out, cudaStream_t s,
                 bool* used) {
  *used = false;
  const bool tc = tc_applicable(p, g);
  const int K = 4 * ((2 * p->m + 1 + 3) / 4);
  const int KC = K / 4;
  const int X = g.tile[0] + 2 * p->m, Y = g.tile[1] + 2 * p->m, Z = g.tile[2] + 2 * p->m;
  int SZ = Z;
  while (SZ % 8 != 4) ++SZ;  // odd multiple of 4 complex: conflict-free B fragments
  const int WS = (std::max(g.box[0], g.box[1]) + 2 * p->m + 1) | 1;
  const size_t smem = dmma_smem_bytes(X, Y, SZ, p->m, p->poly.deg, WS);
  if (!tc && (smem > 200 * 1024 || g.box[0] + 2 * p->m > kMaxRowW ||
              g.box[1] + 2 * p->m > kMaxRowW || g.boxes_per_tile > kMaxBoxes || KC > 7 ||
              g.box[2] != K - 2 * p->m))
    return VFN_OK;  // not applicable: caller uses the thread-per-point gather
  if (M > INT32_MAX) return VFN_OK;

  // box offsets (nboxes + 1 entries) from the sorted keys
  const int64_t nb = g.nboxes;
  VFN_CHECK(p->box_start.ensure(sizeof(int32_t) * (2 * (nb + 1) + 2 * (g.ntiles + 1) + 4)));
  int32_t* counts = p->box_start.as<int32_t>();
  int32_t* bstart = counts + (nb + 1);
  int32_t* nitems = bstart + (nb + 1);
  int32_t* ioff = nitems + (g.ntiles + 1);
  // counts[0] = 0 (= box_start[0]), counts[1 + b] = tails[b]; box_start = the inclusive max-scan of these nb + 1 entries
  VFN_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (nb + 1), s));
  k_box_tails<<<(unsigned)(((M + 7) / 8 + 255) / 256), 256, 0, s>>>(keys_sorted, M, (uint32_t)g.key_slots, counts + 1);
  VFN_CUDA(cudaGetLastError());
  size_t tmp = 0;
  VFN_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tmp, counts, bstart, cub::Max(), (int)(nb + 1), s));
  size_t tmp2 = 0;
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, nitems, ioff, (int)(g.ntiles + 1), s));
  VFN_CHECK(p->sort_tmp.ensure(std::max(tmp, tmp2)));
  VFN_CUDA(cub::DeviceScan::InclusiveScan(p->sort_tmp.ptr, tmp, counts, bstart, cub::Max(), (int)(nb + 1), s));
  if (tc) {
    int st = launch_tc(p, p->uvals.as<double>(), perm, keys_sorted, bstart, out, g, M, s);
    if (st == VFN_OK) *used = true;
    return st;
  }
  k_tile_units<<<(unsigned)((g.ntiles + 1 + 255) / 256), 256, 0, s>>>(bstart, g.ntiles,
                                                                      g.boxes_per_tile, nitems);
  VFN_CUDA(cudaGetLastError());
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(p->sort_tmp.ptr, tmp2, nitems, ioff, (int)(g.ntiles + 1), s));
  const int64_t max_items =
      std::min<int64_t>(g.ntiles, M) * (1 + g.boxes_per_tile / kItemUnits + 1) + M / (kUnitPts * kItemUnits) + 1;
  VFN_CHECK(p->items.ensure(sizeof(int4) * max_items));
  k_items<<<(unsigned)((g.ntiles + 255) / 256), 256, 0, s>>>(bstart, ioff, g.ntiles,
                                                             g.boxes_per_tile, p->items.as<int4>());
  VFN_CUDA(cudaGetLastError());

  GatherArgs A;
  A.pts = pts;
  A.perm = perm;
  A.box_start = bstart;
  A.items = p->items.as<int4>();
  A.nitems = ioff + g.ntiles;
  A.grid = p->grid;
  A.out = out;
  A.poly = p->poly.dev;
  A.deg = p->poly.deg;
  A.m = p->m;
  A.P1 = p->P[1];
  A.P2 = p->P[2];
  A.tm = p->map;
  A.g = g;
  A.X = X;
  A.Y = Y;
  A.Z = Z;
  A.SZ = SZ;
  A.WS = WS;
  mark_event(p, 1, s);  // gather timing starts here (prep excluded)
  int st = VFN_OK;
  switch (KC) {
    case 1: st = launch_dmma<1>(A, smem, s); break;
    case 2: st = launch_dmma<2>(A, smem, s); break;
    case 3: st = launch_dmma<3>(A, smem, s); break;
    case 4: st = launch_dmma<4>(A, smem, s); break;
    case 5: st = launch_dmma<5>(A, smem, s); break;
    case 6: st = launch_dmma<6>(A, smem, s); break;
    case 7: st = launch_dmma<7>(A, smem, s); break;
  }
  if (st == VFN_OK) *used = true;
  return st;
}

}  // namespace vfn
