// K4 for the default cutoff m = 6 (nufft.py:56): binned gather on the FP64
// tensor cores (DMMA, mma.sync.m8n8k4.f64), TMA-staged, double-buffered.
//
// Geometry.  Tiles of 4 x 4 x 8 cells; their 16 x 16 x 20 complex block of
// the ghost-padded grid (80 KB) is one TMA copy (cp.async.bulk.tensor.3d) of
// the grid viewed as doubles.  z-lines are 20 complex = 320 B, so the 8 rows x
// 4 depths a DMMA pair reads hit both bank halves evenly (conflict-free
// LDS.128) without a swizzle.  Boxes are 1 x 1 x 8 (2 x 2 x 8 at low density)
// columns of a tile; inside a box the points are sorted by depth (the bin key
// numbers cells depth-major).
//
// Units.  A box's points sorted by depth are cut into chunks of 8 (the
// DMMA's M rows); a chunk spans <= 7 depths of the 8-deep box, and uses K = 16
// depths (4 k-chunks) when it spans <= 3 cells, K = 20 (5 k-chunks) otherwise.
//
// Per unit, with rows r = (x, y) of the box's (bi+12) x (bj+12) footprint in
// 8-row tiles:
//   C_re/im[p, r] = sum_k W3[p, k] G[r, k].re/im        (DMMA; axis 3, nufft.py:269)
//   acc[p] += W1[p, x(r)] W2[p, y(r)] C[p, r]           (axes 2 and 1, nufft.py:270-271)
// and the 3 x 13 window weights of the unit's points are themselves one
// DMMA each (A = powers of delta, B = the fitted polynomial coefficients).
//
// Pipeline.  One CTA of 16 warps per SM, persistent over work items (tile,
// unit range).  Two tile buffers: item k's tile is loaded while item k-1 is
// being computed; the last warp to finish an item (smem counter) issues the
// TMA for item k+2 into the freed buffer, so warps never wait for each other.
#include <cuda.h>

#include <climits>

#include <cub/device/device_scan.cuh>

#include "vfn_device.cuh"

namespace vfn {

namespace m6 {

constexpr int kUnitPts = 8;
constexpr int kWarps = 16;
constexpr int kTZ = 8;                    // tile depth in cells (x, y: 4)
constexpr int kSXY = 16;                  // staged x, y extent (4 + 12)
constexpr int kSZ = 20;                   // staged z extent (8 + 12)
constexpr int kLine = kSZ * 16;           // bytes per staged (x, y) line
constexpr int kTileBytes = kSXY * kSXY * kLine;  // 80 KB
constexpr int kItemUnits = 48;            // units per work item
// per-warp window-weight tables (doubles); entry off + j holds phi_j(delta)
constexpr int kAO = 8, kAS = 29;          // axis 3 (A fragments): j in [-8, 21)
constexpr int kXO = 1, kXS = 17;          // axes 1, 2: j in [-1, 16)
constexpr int kWarpW = kUnitPts * (kAS + 2 * kXS);

struct Args {
  const double* u;        // u = z * n per point and axis, input order (k_map_key)
  const int32_t* perm;    // sorted position -> input row
  const int4* units;      // (start, cnt | k20 << 4 | kz << 8, box, 0)
  const int4* items;      // (tile, unit_begin, unit_end, 0)
  const int32_t* nitems;  // device scalar
  double2* out;
  const double* poly;     // window polynomial table (13 x (deg+1))
  int deg;
  TorusMap tm;
  BinGeom g;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// Load item `it`'s tile into the buffer at `dst` (completes on `bar`).
__device__ __forceinline__ void issue_tile(const CUtensorMap* map, const Args& A, int it,
                                           unsigned dst, unsigned bar) {
  if (it >= *A.nitems) return;
  const int tile = A.items[it].x;
  const BinGeom& G = A.g;
  const int t2 = tile % G.ntile[2];
  const int t1 = (tile / G.ntile[2]) % G.ntile[1];
  const int t0 = tile / (G.ntile[2] * G.ntile[1]);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // prior generic reads of dst
  mbar_expect_tx(bar, kTileBytes);
  tma_load_3d(dst, map, 2 * t2 * kTZ, t1 * 4, t0 * 4, bar);
}

// One 8-row DMMA tile: C_re/im[p, n] for the lane's B row at `addr`.
template <int KC>
__device__ __forceinline__ void tile_mma(unsigned addr, const double (&a)[KC], double& cr0,
                                         double& cr1, double& ci0, double& ci1) {
  cr0 = cr1 = ci0 = ci1 = 0.0;
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    const double2 v = lds128(addr + kc * 64);
    dmma(cr0, cr1, a[kc], v.x);
    dmma(ci0, ci1, a[kc], v.y);
  }
}

// One unit: <= 8 points of one box sharing the box's rows.
// The unit's points (lane quad g owns point g): sorted-position -> input row
// and its u values.  Issued one unit ahead so the latency hides behind the
// previous unit's DMMAs.
struct UnitPoints {
  int64_t prow;
  double uu[3];
};

__device__ __forceinline__ UnitPoints load_unit_points(const Args& A, int4 desc, int g) {
  UnitPoints up;
  up.prow = 0;
  up.uu[0] = up.uu[1] = up.uu[2] = 0.0;
  if (g < (desc.y & 15)) {
    // streamed once: evict-first, so the grid's tiles keep the L2
    up.prow = __ldcs(A.perm + desc.x + g);
#pragma unroll
    for (int d = 0; d < 3; ++d) up.uu[d] = __ldcs(A.u + 3 * up.prow + d);
  }
  return up;
}

template <int BXY, int KC>
__device__ __forceinline__ void gather_unit(const Args& A, const double* __restrict__ scb, double* wt,
                                            unsigned tile_s, int tile, int ox, int oy, int oz,
                                            int4 desc, const UnitPoints& up, int lane) {
  constexpr int XB = BXY + 12, YB = BXY + 12;  // box footprint rows per axis
  constexpr int NB = 4 / BXY;                  // boxes per tile along x and y
  const int g = lane >> 2, tig = lane & 3;
  const int start = desc.x, cnt = desc.y & 15, kz = desc.y >> 8;
  const int bt = desc.z - tile * (NB * NB);
  const int X0 = (bt / NB) * BXY, Y0 = (bt % NB) * BXY;

  (void)start;
  const bool valid = g < cnt;
  const int64_t prow = up.prow;
  int cell[3];
  double dl[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) cell[d] = cell_from_u(up.uu[d], A.tm.nd[d], A.tm.n[d], dl[d]);
  // offsets inside the box; idle lanes and out-of-domain points (key 0) are
  // pinned to 0 so every table index stays in bounds
  const int ci0 = cell[0] - ox - X0, cj0 = cell[1] - oy - Y0, ck0 = cell[2] - oz;
  const bool inbox = valid && ci0 >= 0 && ci0 < BXY && cj0 >= 0 && cj0 < BXY && ck0 >= 0 && ck0 < kTZ;
  const int ci = inbox ? ci0 : 0, cj = inbox ? cj0 : 0, ck = inbox ? ck0 : 0;

  // window weights W[p, j] = sum_d delta_p^d C[d, j] on the three axes (DMMA)
  double* wA = wt;                              // [8][kAS]  axis 3
  double* wX = wt + kUnitPts * kAS;             // [8][kXS]  axis 1
  double* wY = wX + kUnitPts * kXS;             // [8][kXS]  axis 2
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double x1 = dl[d], x2 = x1 * x1, x4 = x2 * x2;
    double pw = tig == 0 ? 1.0 : (tig == 1 ? x1 : (tig == 2 ? x2 : x2 * x1));
    double w00 = 0.0, w01 = 0.0, w10 = 0.0, w11 = 0.0;
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      const double2 c = *reinterpret_cast<const double2*>(scb + 2 * kc);  // (nb 0, nb 1)
      dmma(w00, w01, pw, c.x);
      dmma(w10, w11, pw, c.y);
      pw *= x4;
    }
    double* row = d == 2 ? wA + g * kAS + kAO : (d == 0 ? wX : wY) + g * kXS + kXO;
    row[2 * tig] = w00;      // j = 2 tig, 2 tig + 1, 8 + 2 tig, 9 + 2 tig;
    row[2 * tig + 1] = w01;  // j >= 13 come out exactly 0 (zero coefficients)
    row[8 + 2 * tig] = w10;
    row[9 + 2 * tig] = w11;
  }
  __syncwarp();
  // A fragments: axis-3 weights of point g at staged depth kz + 4 kc + tig
  double a[KC];
  const double* wa = wA + g * kAS + kAO + kz + tig - ck;
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) a[kc] = inbox ? wa[4 * kc] : 0.0;
  const double* wx = wX + g * kXS + kXO - ci;  // wx[x], x in [0, XB]; zero off the stencil
  const double* wy = wY + g * kXS + kXO - cj;  // wy[y], y in [0, YB]

  // Static row schedule over the box's XB x YB rows, 8 rows per DMMA tile,
  // chosen so that every lane's B row and C rows are compile-time functions
  // of (tile, lane) — no cursors, no bounds checks in the hot loop:
  //   A: one tile per x, rows y = 0..7          (B: y = g;  C: y = 2tig + e)
  //   B: one tile per x pair, rows y = 8..11    (B: x = 2p + g/4, y = 8 + g%4)
  //   C: the rows y >= 12                       (BXY=1: x = 8q + n; BXY=2: x = 4q + n/2)
  // Rows past the box read a clamped valid row and get weight 0.
  const unsigned base = tile_s + (unsigned)((kz + tig) * 16 + (X0 * kSXY + Y0) * kLine);
  constexpr unsigned kX = kSXY * kLine;  // x stride
  // Per part, the lane's C rows have fixed y, so the x-weights are applied
  // per tile (2 FMA per row pair) and the y-weights once at the end.
  double acc_re = 0.0, acc_im = 0.0;
  {
    double t0r = 0.0, t1r = 0.0, t0i = 0.0, t1i = 0.0;
    const unsigned ba = base + g * kLine;
#pragma unroll
    for (int x = 0; x < XB; ++x) {
      double cr0, cr1, ci0, ci1;
      tile_mma<KC>(ba + x * kX, a, cr0, cr1, ci0, ci1);
      const double w = wx[x];
      t0r = fma(w, cr0, t0r);
      t1r = fma(w, cr1, t1r);
      t0i = fma(w, ci0, t0i);
      t1i = fma(w, ci1, t1i);
    }
    const double wy0 = wy[2 * tig], wy1 = wy[2 * tig + 1];
    acc_re = fma(wy0, t0r, wy1 * t1r);
    acc_im = fma(wy0, t0i, wy1 * t1i);
  }
  {
    double t0r = 0.0, t1r = 0.0, t0i = 0.0, t1i = 0.0;
    const int xb = g >> 2, xc = tig >> 1;
    const unsigned bb = base + (8 + (g & 3)) * kLine;
#pragma unroll
    for (int p = 0; p < (XB + 1) / 2; ++p) {
      double cr0, cr1, ci0, ci1;
      tile_mma<KC>(bb + min(2 * p + xb, XB - 1) * kX, a, cr0, cr1, ci0, ci1);
      const double w = wx[2 * p + xc];
      t0r = fma(w, cr0, t0r);
      t1r = fma(w, cr1, t1r);
      t0i = fma(w, ci0, t0i);
      t1i = fma(w, ci1, t1i);
    }
    const double wy0 = wy[8 + 2 * (tig & 1)], wy1 = wy[9 + 2 * (tig & 1)];
    acc_re = fma(wy0, t0r, fma(wy1, t1r, acc_re));
    acc_im = fma(wy0, t0i, fma(wy1, t1i, acc_im));
  }
  if (BXY == 1) {  // rows (x, 12), x = 0..12: two tiles
    double tr = 0.0, ti = 0.0;
    const unsigned bc = base + 12 * kLine;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      double cr0, cr1, ci0, ci1;
      tile_mma<KC>(bc + min(8 * q + g, XB - 1) * kX, a, cr0, cr1, ci0, ci1);
      const double w0 = wx[8 * q + 2 * tig], w1 = wx[8 * q + 2 * tig + 1];
      tr = fma(w0, cr0, fma(w1, cr1, tr));
      ti = fma(w0, ci0, fma(w1, ci1, ti));
    }
    const double wy0 = wy[12];
    acc_re = fma(wy0, tr, acc_re);
    acc_im = fma(wy0, ti, acc_im);
  } else {  // rows (x, 12..13), x = 0..13: four tiles
    double t0r = 0.0, t1r = 0.0, t0i = 0.0, t1i = 0.0;
    const unsigned bc = base + (12 + (g & 1)) * kLine;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double cr0, cr1, ci0, ci1;
      tile_mma<KC>(bc + min(4 * q + (g >> 1), XB - 1) * kX, a, cr0, cr1, ci0, ci1);
      const double w = wx[4 * q + tig];
      t0r = fma(w, cr0, t0r);
      t1r = fma(w, cr1, t1r);
      t0i = fma(w, ci0, t0i);
      t1i = fma(w, ci1, t1i);
    }
    const double wy0 = wy[12], wy1 = wy[13];
    acc_re = fma(wy0, t0r, fma(wy1, t1r, acc_re));
    acc_im = fma(wy0, t0i, fma(wy1, t1i, acc_im));
  }
  acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 1);
  acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 1);
  acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 2);
  acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 2);
  if (valid && tig == 0) __stcs(A.out + prow, make_double2(acc_re, acc_im));
  __syncwarp();  // the weight tables are rewritten by the next unit
}

template <int BXY>
__global__ void __launch_bounds__(kWarps * 32, 1)
    k_gather_m6(const __grid_constant__ CUtensorMap tmap, const Args A) {
  extern __shared__ unsigned char smem_raw[];
  const unsigned raw = (unsigned)__cvta_generic_to_shared(smem_raw);
  const unsigned tiles_s = (raw + 1023u) & ~1023u;          // 2 x kTileBytes
  const unsigned bar_s = tiles_s + 2 * kTileBytes;          // full[2]
  unsigned char* ctl = smem_raw + (bar_s - raw);
  int* done = reinterpret_cast<int*>(ctl + 16);              // done[2]
  int* ctr = done + 2;                                       // next CTA unit to hand out
  int* loaded = done + 4;                                    // loaded[2]: item ordinal per buffer
  double* wts = reinterpret_cast<double*>(ctl + 48);         // [kWarps][kWarpW]
  double* scb_all = wts + kWarps * kWarpW;                    // [32 lanes][8]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  for (int i = tid; i < kWarps * kWarpW; i += blockDim.x) wts[i] = 0.0;  // zero pads
  // B fragments of the weights DMMA, C[d = 4 kc + tig][j = 8 nb + g], per
  // lane in shared memory (kept out of the register budget)
  if (warp == 0) {
#pragma unroll
    for (int kc = 0; kc < 4; ++kc)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        const int d = 4 * kc + tig, j = 8 * nb + g;
        scb_all[lane * 8 + 2 * kc + nb] = (d <= A.deg && j < 13) ? A.poly[j * (A.deg + 1) + d] : 0.0;
      }
  }
  const double* scb = scb_all + lane * 8;
  // this CTA's k-th item: strided over the tile-ordered item list, so the
  // 148 CTAs work on neighbouring tiles at any moment and share the tiles'
  // halos through L2 (contiguous blocks per CTA measured 38% more DRAM reads)
  const int nitems = *A.nitems;
  auto item_of = [&](int k) {
    const long long it = (long long)blockIdx.x + (long long)k * gridDim.x;
    return it < nitems ? (int)it : INT_MAX;
  };
  if (tid == 0) {
    mbar_init(bar_s, 1);
    mbar_init(bar_s + 8, 1);
    done[0] = done[1] = 0;
    ctr[0] = 0;
    loaded[0] = 0;
    loaded[1] = 1;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    issue_tile(&tmap, A, item_of(0), tiles_s, bar_s);
    issue_tile(&tmap, A, item_of(1), tiles_s + kTileBytes, bar_s + 8);
  }
  __syncthreads();

  double* wt = wts + warp * kWarpW;
  const BinGeom& G = A.g;
  // Units are handed out from one monotonic CTA counter over the
  // concatenated units of this CTA's items (item k = items[blockIdx.x +
  // k * gridDim.x]); each warp walks the item list forward to locate the unit
  // it grabbed, reserves its next unit and prefetches its points before
  // computing the current one.  A tile buffer is refilled (item k+2) by the
  // warp that completes the last unit of item k.
  struct Cur {
    int k;      // item ordinal within this CTA (-1: none)
    int4 item;  // (tile, unit_begin, unit_end)
    int base;   // CTA unit index of the item's first unit
  };
  Cur walk;
  walk.k = 0;
  walk.item = item_of(0) < nitems ? A.items[item_of(0)] : make_int4(0, 0, 0, 0);
  walk.base = 0;
  // locate CTA unit u by walking forward (u is monotonic per warp)
  auto locate = [&](int u, int4& desc, int& kk, int4& it4) -> bool {
    while (true) {
      const int it = item_of(walk.k);
      if (it >= nitems) return false;
      const int n = walk.item.z - walk.item.y;
      if (u < walk.base + n) {
        kk = walk.k;
        it4 = walk.item;
        desc = __ldg(A.units + walk.item.y + (u - walk.base));
        return true;
      }
      walk.base += n;
      ++walk.k;
      const int itn = item_of(walk.k);
      walk.item = itn < nitems ? A.items[itn] : make_int4(0, 0, 0, 0);
    }
  };
  auto grab = [&]() {
    int v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  int4 desc, item;
  int kk = 0;
  UnitPoints up;
  bool have = locate(grab(), desc, kk, item);
  if (have) up = load_unit_points(A, desc, g);
  while (have) {
    int4 desc_n, item_n;
    int kk_n = 0;
    UnitPoints up_n;
    const bool have_n = locate(grab(), desc_n, kk_n, item_n);
    if (have_n) up_n = load_unit_points(A, desc_n, g);
    const int b = kk & 1;
    const int tile = item.x;
    const int t2 = tile % G.ntile[2];
    const int t1 = (tile / G.ntile[2]) % G.ntile[1];
    const int t0 = tile / (G.ntile[2] * G.ntile[1]);
    const unsigned tile_s = tiles_s + b * kTileBytes;
    // a warp may hold units of items far ahead (small items): the buffer's
    // mbarrier parity only distinguishes consecutive loads, so first wait
    // until the buffer's load for item kk has been issued
    while (*reinterpret_cast<volatile int*>(&loaded[b]) != kk) __nanosleep(64);
    mbar_wait(bar_s + 8 * b, (kk >> 1) & 1);
    if ((desc.y >> 4) & 1)
      gather_unit<BXY, 5>(A, scb, wt, tile_s, tile, t0 * 4, t1 * 4, t2 * kTZ, desc, up, lane);
    else
      gather_unit<BXY, 4>(A, scb, wt, tile_s, tile, t0 * 4, t1 * 4, t2 * kTZ, desc, up, lane);
    if (lane == 0) {
      if (atomicAdd(&done[b], 1) == item.z - item.y - 1) {  // last unit of item kk
        done[b] = 0;
        if (item_of(kk + 2) < nitems) {
          *reinterpret_cast<volatile int*>(&loaded[b]) = kk + 2;
          issue_tile(&tmap, A, item_of(kk + 2), tile_s, bar_s + 8 * b);
        }
      }
    }
    have = have_n;
    desc = desc_n;
    item = item_n;
    kk = kk_n;
    up = up_n;
  }
}

}  // namespace m6

// ------------------------------------------------------------------ units

// A box's points are sorted by depth and the box is 8 cells deep, so any 8
// consecutive points span <= 7 depths: units are the box's chunks of 8,
// using K = 16 depths when the chunk spans <= 3 cells and K = 20 otherwise.
__device__ __forceinline__ int box_depth(uint32_t key, int cpb, int bij) {
  return (int)(key % (uint32_t)cpb) / bij;
}

__global__ void k_unit_counts(const int32_t* __restrict__ box_start, int64_t nboxes,
                              int32_t* __restrict__ ucount) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nboxes) return;
  ucount[b] = b == nboxes ? 0 : (box_start[b + 1] - box_start[b] + m6::kUnitPts - 1) / m6::kUnitPts;
}

// One thread per sorted point; the point that opens a chunk of 8 in its box
// writes the unit (fully parallel, also for boxes holding millions of points).
__global__ void k_write_units(const uint32_t* __restrict__ keys, int64_t M,
                              const int32_t* __restrict__ box_start, int cpb, int bij,
                              const int32_t* __restrict__ uoff, int4* __restrict__ units) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const uint32_t key = keys[i];
  const int64_t b = key / (uint32_t)cpb;
  const int bs = box_start[b];
  const int r = (int)i - bs;
  if (r % m6::kUnitPts) return;
  const int be = box_start[b + 1];
  const int e = min(be, (int)i + m6::kUnitPts);
  const int k0 = box_depth(key, cpb, bij), k1 = box_depth(keys[e - 1], cpb, bij);
  const int k20 = k1 - k0 > 3 ? 1 : 0;
  const int kz = k20 ? 0 : min(k0, 4);
  units[uoff[b] + r / m6::kUnitPts] = make_int4((int)i, (e - (int)i) | (k20 << 4) | (kz << 8), (int)b, 0);
}

__global__ void k_m6_tile_items(const int32_t* __restrict__ uoff, int64_t ntiles, int bpt,
                                int32_t* __restrict__ nitems) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  if (t == ntiles) {
    nitems[t] = 0;
    return;
  }
  const int units = uoff[(t + 1) * bpt] - uoff[t * bpt];
  nitems[t] = (units + m6::kItemUnits - 1) / m6::kItemUnits;
}

__global__ void k_m6_items(const int32_t* __restrict__ uoff, const int32_t* __restrict__ ioff,
                           int64_t ntiles, int bpt, int4* __restrict__ items) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int first = ioff[t], n = ioff[t + 1] - first;
  const int u0 = uoff[t * bpt], u1 = uoff[(t + 1) * bpt];
  for (int j = 0; j < n; ++j)
    items[first + j] = make_int4((int)t, u0 + j * m6::kItemUnits, min(u1, u0 + (j + 1) * m6::kItemUnits), 0);
}

// Tensor map over the ghost-padded grid as doubles: (2 P2, P1, P0), box
// (40 doubles, 16, 16), no swizzle.
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
  cuuint32_t box[3] = {2 * m6::kSZ, (cuuint32_t)m6::kSXY, (cuuint32_t)m6::kSXY};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<Fn>(fn)(&p->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, p->grid, dims,
                                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(VFN_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  p->has_tmap = true;
  return VFN_OK;
}

static size_t m6_smem_bytes() {
  return 1024 + 2 * m6::kTileBytes + 48 + sizeof(double) * (m6::kWarps * m6::kWarpW + 32 * 8);
}

bool m6_applicable(const vfn_plan* p, const BinGeom& g) {
  return p->m == 6 && p->has_tmap && p->poly.deg <= 15 && g.tile[0] == 4 && g.tile[1] == 4 &&
         g.tile[2] == m6::kTZ && g.box[2] == m6::kTZ && g.box[0] == g.box[1] &&
         (g.box[0] == 1 || g.box[0] == 2);
}

template <int BXY>
static int launch(vfn_plan* p, const m6::Args& A, cudaStream_t s) {
  const size_t smem = m6_smem_bytes();
  VFN_CUDA(cudaFuncSetAttribute(m6::k_gather_m6<BXY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  m6::k_gather_m6<BXY><<<nsm, m6::kWarps * 32, smem, s>>>(p->tmap, A);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

// Build units and items from the box offsets, then run the m = 6 gather.
int launch_m6(vfn_plan* p, const double* u, const int32_t* perm, const uint32_t* keys_sorted,
              const int32_t* box_start, double2* out, const BinGeom& g, int64_t M,
              cudaStream_t s) {
  const int64_t nb = g.nboxes;
  const int bij = g.box[0] * g.box[1];
  // scratch: ucount/uoff (nb + 1 each), nitems/ioff (ntiles + 1 each)
  VFN_CHECK(p->uscratch.ensure(sizeof(int32_t) * (2 * (nb + 1) + 2 * (g.ntiles + 1))));
  int32_t* ucount = p->uscratch.as<int32_t>();
  int32_t* uoff = ucount + (nb + 1);
  int32_t* nitems = uoff + (nb + 1);
  int32_t* ioff = nitems + (g.ntiles + 1);
  const unsigned bb = (unsigned)((nb + 1 + 255) / 256);
  k_unit_counts<<<bb, 256, 0, s>>>(box_start, nb, ucount);
  VFN_CUDA(cudaGetLastError());
  size_t t1 = 0, t2 = 0;
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t1, ucount, uoff, (int)(nb + 1), s));
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, nitems, ioff, (int)(g.ntiles + 1), s));
  VFN_CHECK(p->sort_tmp.ensure(std::max(t1, t2)));
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(p->sort_tmp.ptr, t1, ucount, uoff, (int)(nb + 1), s));
  // units <= M (each holds >= 1 point)
  VFN_CHECK(p->units.ensure(sizeof(int4) * (M + 1)));
  k_write_units<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(keys_sorted, M, box_start,
                                                            g.cells_per_box, bij, uoff,
                                                            p->units.as<int4>());
  VFN_CUDA(cudaGetLastError());
  const unsigned tb = (unsigned)((g.ntiles + 1 + 255) / 256);
  k_m6_tile_items<<<tb, 256, 0, s>>>(uoff, g.ntiles, g.boxes_per_tile, nitems);
  VFN_CUDA(cudaGetLastError());
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(p->sort_tmp.ptr, t2, nitems, ioff, (int)(g.ntiles + 1), s));
  const int64_t max_items = std::min<int64_t>(g.ntiles, M) + M / m6::kItemUnits + 1;
  VFN_CHECK(p->items.ensure(sizeof(int4) * max_items));
  k_m6_items<<<tb, 256, 0, s>>>(uoff, ioff, g.ntiles, g.boxes_per_tile, p->items.as<int4>());
  VFN_CUDA(cudaGetLastError());

  m6::Args A;
  A.u = u;
  A.perm = perm;
  A.units = p->units.as<int4>();
  A.items = p->items.as<int4>();
  A.nitems = ioff + g.ntiles;
  A.out = out;
  A.poly = p->poly.dev;
  A.deg = p->poly.deg;
  A.tm = p->map;
  A.g = g;
  cudaEventRecord(p->ev[1], s);  // gather timing starts here (binning prep excluded)
  return g.box[0] == 1 ? launch<1>(p, A, s) : launch<2>(p, A, s);
}

}  // namespace vfn
