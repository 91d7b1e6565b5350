// K4 for cutoffs m = 2..7 (nufft.py:56 default m = 6; NufftParams.for_accuracy
// nufft.py:67-73 gives m = 2..7 for eps = 1e-4..1e-14): binned gather on the
// FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64), TMA-staged, double-buffered.
// One template over the cutoff MC and the box width BXY.
//
// Geometry.  Tiles of 4 x 4 x TZ cells (4 x 2 x 6 at m = 7) with TZ = 20 - 2m
// (8 at m = 6); their (4+2m) x (4+2m) x 20 complex block of the ghost-padded grid (80 KB at
// m = 6) is one TMA copy (cp.async.bulk.tensor.3d) of the grid viewed as
// doubles.  z-lines are always 20 complex = 320 B (= 64 B mod 128 B), so the
// 8 rows x 4 depths a DMMA pair reads hit both bank halves evenly
// (conflict-free LDS.128) without a swizzle.  Boxes are 1 x 1 x TZ (2 x 2 x
// TZ at low density) columns of a tile; inside a box the points are sorted by
// depth (the bin key numbers cells depth-major).
//
// Units.  A box's points sorted by depth are cut into chunks of 8 (the
// DMMA's M rows); a chunk spans <= TZ - 1 depths, so its stencils cover
// span + W <= 20 staged depths (W = 2m + 1).  Each unit uses the smallest
// K = 4 KC (KC = 2..5 k-chunks) with span + W <= K.
//
// Per unit, with rows r = (x, y) of the box's (BXY+2m) x (BXY+2m) footprint
// in 8-row DMMA tiles:
//   C_re/im[p, r] = sum_k W3[p, k] G[r, k].re/im        (DMMA; axis 3, nufft.py:269)
//   acc[p] += W1[p, x(r)] W2[p, y(r)] C[p, r]           (axes 2 and 1, nufft.py:270-271)
// and the 3 x W window weights of the unit's points are themselves one
// DMMA each (A = powers of delta, B = the fitted polynomial coefficients).
//
// Pipeline.  One CTA of 16 warps per SM, persistent over work items (tile,
// unit range).  Two tile buffers: item k's tile is loaded while item k-1 is
// being computed; the last warp to finish an item (smem counter) issues the
// TMA for item k+2 into the freed buffer, so warps never wait for each other.
#include <cuda.h>

#include <climits>
#include <cstdlib>

#include <cub/device/device_scan.cuh>

#include "vfn_device.cuh"

namespace vfn {

namespace tc {

constexpr int kUnitPts = 8;
// warps per CTA: 16 (128 registers each) keep the FP64 pipe fullest on
// dense tiles; sparse tiles (< ~5 points per 1x1x8 column, e.g. 1e6 points on
// 128^3) have too few units per staged tile for 16 warps and run 12
constexpr int kWarpsDense = 16, kWarpsSparse = 12;
// half-units (SPLIT) below this many points per 1x1x8 column
constexpr double kSplitDensity = 1.7, kSparseDensity = 4.8;
constexpr int kSZ = 20;                   // staged z extent (TZ + 2m)
constexpr int kLine = kSZ * 16;           // bytes per staged (x, y) line
constexpr int kItemUnits = 48;            // units per work item
constexpr int kXO = 1;                    // axes 1, 2 weight tables: entry kXO + j holds phi_j, j >= -1

template <int MC>
struct Cfg {
  static_assert(MC >= 2 && MC <= 8, "tensor-core gather covers m = 2..8");
  static constexpr int W = 2 * MC + 1;            // stencil width
  static constexpr int TZ = kSZ - 2 * MC;         // tile / box depth in cells
  // tile x, y extents in cells: 4 x 4, 4 x 2 at m = 7 and 2 x 2 at m = 8
  // (8-warp CTAs) so that two staged tiles still fit next to the weight
  // tables
  static constexpr int TX = MC == 8 ? 2 : 4, TY = MC >= 7 ? 2 : 4;
  static constexpr int SX = TX + 2 * MC, SY = TY + 2 * MC;  // staged x, y extents
  static constexpr int kTileBytes = SX * SY * kLine;
  static constexpr int KCmin = (W + 3) / 4;       // fewest k-chunks a unit can use
  // A fragments from a per-warp axis-3 table (entry kAO + j holds phi_j,
  // j in [-TZ, 21)), or at m = 7 straight from the weight DMMA's registers
  // by quad shuffles (no table: its shared memory holds the larger tiles)
  static constexpr bool kShflA = MC >= 7;
  static constexpr int kAO = TZ, kAS = kShflA ? 0 : (TZ + 21) | 1;
  static constexpr int kXS = MC == 8 ? 19 : 17;   // x / y tables: j in [-1, kXS - 1)
  // weight DMMA (even/odd split, see gather_unit): taps 0..MC, four per
  // n-block as (E, O) column pairs; two k-chunks of powers of delta^2
  static constexpr int kNB = (MC + 4) / 4;             // n-blocks in the per-lane B table
  static constexpr int kScb = 2 * kNB;                 // its doubles per lane (2 k-chunks)
  static constexpr int kWarpW = kUnitPts * (kAS + 2 * kXS);
};

size_t smem_bytes(int mc, int nw) {
  auto f = [nw](int tile, int warpw, int scb) {
    return (size_t)1024 + 2 * (size_t)tile + 48 + sizeof(double) * ((size_t)nw * warpw + 32 * (size_t)scb);
  };
  switch (mc) {
    case 2: return f(Cfg<2>::kTileBytes, Cfg<2>::kWarpW, Cfg<2>::kScb);
    case 3: return f(Cfg<3>::kTileBytes, Cfg<3>::kWarpW, Cfg<3>::kScb);
    case 4: return f(Cfg<4>::kTileBytes, Cfg<4>::kWarpW, Cfg<4>::kScb);
    case 5: return f(Cfg<5>::kTileBytes, Cfg<5>::kWarpW, Cfg<5>::kScb);
    case 7: return f(Cfg<7>::kTileBytes, Cfg<7>::kWarpW, Cfg<7>::kScb);
    case 8: return f(Cfg<8>::kTileBytes, Cfg<8>::kWarpW, Cfg<8>::kScb);
    default: return f(Cfg<6>::kTileBytes, Cfg<6>::kWarpW, Cfg<6>::kScb);
  }
}

struct Args {
  const double* u;        // u = z * n per point and axis, input order (k_map_key)
  const int32_t* perm;    // sorted position -> input row
  const int4* units;      // (start, cnt | KC << 4 | kz << 8, box, 0)
  const int4* items;      // (tile, unit_begin, unit_end, 0)
  const int32_t* nitems;  // device scalar
  double2* out;
  const double* poly;     // window polynomial table (W x (deg+1))
  int deg;
  int64_t M;              // points (bounds checks of the VFN_CHECKS build)
  int64_t nunits;         // unit-list capacity (bounds checks)
  TorusMap tm;
  BinGeom g;
  const PeerTable* peer;  // non-null: values go to their owners' buffers (sharded evaluate)
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

__device__ __forceinline__ double lds64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// Load item `it`'s tile into the buffer at `dst` (completes on `bar`).
template <int MC>
__device__ __forceinline__ void issue_tile(const CUtensorMap* map, const Args& A, int it,
                                           unsigned dst, unsigned bar) {
  if (it >= *A.nitems) return;
  const int tile = A.items[it].x;
  const BinGeom& G = A.g;
  const int t2 = tile % G.ntile[2];
  const int t1 = (tile / G.ntile[2]) % G.ntile[1];
  const int t0 = tile / (G.ntile[2] * G.ntile[1]);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // prior generic reads of dst
  mbar_expect_tx(bar, Cfg<MC>::kTileBytes);
  tma_load_3d(dst, map, 2 * t2 * Cfg<MC>::TZ, t1 * Cfg<MC>::TY, t0 * Cfg<MC>::TX, bar);
}

// One 8-row DMMA tile: C_re/im[p, n] for the lane's B row at `addr`.  SPLIT
// (half-units, see k_gather_tc): `addr` points at this warp's component (re
// or im) and only the "re" accumulators are computed.
template <int KC, bool SPLIT>
__device__ __forceinline__ void tile_mma(unsigned addr, const double (&a)[KC], double& cr0,
                                         double& cr1, double& ci0, double& ci1, unsigned lo,
                                         unsigned hi) {
  cr0 = cr1 = ci0 = ci1 = 0.0;
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    VFN_DCHECK(addr + kc * 64 >= lo && addr + kc * 64 + (SPLIT ? 8 : 16) <= hi);  // inside the staged tile
    if constexpr (SPLIT) {
      dmma(cr0, cr1, a[kc], lds64(addr + kc * 64));
    } else {
      const double2 v = lds128(addr + kc * 64);
      dmma(cr0, cr1, a[kc], v.x);
      dmma(ci0, ci1, a[kc], v.y);
    }
  }
}

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
    VFN_DCHECK(desc.x >= 0 && desc.x + g < A.M);
    // streamed once: evict-first, so the grid's tiles keep the L2
    up.prow = __ldcs(A.perm + desc.x + g);
    VFN_DCHECK(up.prow >= 0 && up.prow < A.M);
#pragma unroll
    for (int d = 0; d < 3; ++d) up.uu[d] = __ldcs(A.u + 3 * up.prow + d);
  }
  return up;
}

// What a unit waits for before it reads its staged tile: the buffer's load
// for item kk issued (loaded[b] == kk; the mbarrier parity only tells
// consecutive loads apart) and completed (mbarrier phase).  gather_unit waits
// AFTER the window weights are in place: they depend on the points only, so
// on a sparse pass (warps outnumber the runnable units) they are computed
// while the tile is still in flight.
struct TileWait {
  const int* loaded;  // &loaded[b] (shared)
  int kk;
  unsigned bar, parity;
};

// Row-schedule parts over the box footprint (XB x YB rows), each a run of
// 8-row DMMA tiles whose lane -> (x, y) maps are compile-time:
//   R8 (rows y0..y0+7, one tile per x):    B: (x, y0 + g)            C: y = y0 + 2tig + e
//   R4 (rows y0..y0+3, x pairs):           B: (2p + g/4, y0 + g%4)   C: x = 2p + tig/2
//   R2 (rows y0, y0+1, x quads):           B: (4q + g/2, y0 + g%2)   C: x = 4q + tig
//   R1 (row y0, x octets):                 B: (8q + g, y0)           C: x = 8q + 2tig + e
// Per part the lane's C rows have fixed y, so the x-weights are applied per
// tile (2 FMA per row pair) and the y-weights once at the end.  Rows past
// the box read a clamped valid row and get weight 0.
template <int MC, int BXY, int KC, bool PEER, bool SPLIT>
__device__ __forceinline__ void gather_unit(const Args& A, const double* __restrict__ scb, double* wt,
                                            unsigned tile_s, int tile, int ox, int oy, int oz,
                                            int4 desc, const UnitPoints& up, int lane, int half,
                                            const TileWait& tw) {
  using C = Cfg<MC>;
  constexpr int XB = BXY + 2 * MC, YB = BXY + 2 * MC;  // box footprint rows per axis
  constexpr int NBY = C::TY / BXY;                     // boxes per tile along y
  constexpr int kAO = C::kAO, kAS = C::kAS;
  const int g = lane >> 2, tig = lane & 3;
  const int cnt = desc.y & 15, kz = desc.y >> 8;
  const int bt = desc.z - tile * ((C::TX / BXY) * NBY);
  const int X0 = (bt / NBY) * BXY, Y0 = (bt % NBY) * BXY;

  const bool valid = g < cnt;
  const int64_t prow = up.prow;
  int cell[3];
  double dl[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) cell[d] = cell_from_u(up.uu[d], A.tm.nd[d], A.tm.n[d], dl[d]);
  // offsets inside the box; idle lanes and out-of-domain points (key 0) are
  // pinned to 0 so every table index stays in bounds
  const int ci0 = cell[0] - ox - X0, cj0 = cell[1] - oy - Y0, ck0 = cell[2] - oz;
  const bool inbox = valid && ci0 >= 0 && ci0 < BXY && cj0 >= 0 && cj0 < BXY && ck0 >= 0 && ck0 < C::TZ;
  const int ci = inbox ? ci0 : 0, cj = inbox ? cj0 : 0, ck = inbox ? ck0 : 0;

  // window weights on the three axes (DMMA).  The window is even, so tap
  // 2m - j is tap j's polynomial at -delta: with P_j(delta) = E_j(s) +
  // delta O_j(s), s = delta^2, only taps j = 0..m are evaluated,
  //   [E_j | O_j][p] = sum_k s_p^k C[k, (j, E|O)]      (K = 8 powers of s: degree <= 15),
  // and w_j = E_j + delta O_j, w_{2m-j} = E_j - delta O_j.  Columns (E_j,
  // O_j) sit side by side, four taps per n-block, so lane (g, tig) holds
  // point g's taps tig and 4 + tig (and tap 8 in lane tig = 0 at m = 8):
  // half the k-chunks and half the columns of a direct evaluation.
  constexpr int NBW = C::kNB;
  constexpr int kXS = C::kXS;
  double* wA = wt;                              // [8][kAS]  axis 3 (absent with kShflA)
  double* wX = wt + kUnitPts * kAS;             // [8][kXS]  axis 1
  double* wY = wX + kUnitPts * kXS;             // [8][kXS]  axis 2
  double zp0 = 0.0, zm0 = 0.0, zp1 = 0.0, zm1 = 0.0, z2 = 0.0;  // axis-3 weights in registers (kShflA)
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double x1 = dl[d], s1 = x1 * x1, s2 = s1 * s1, s4 = s2 * s2;
    double pw = tig == 0 ? 1.0 : (tig == 1 ? s1 : (tig == 2 ? s2 : s2 * s1));
    double e0 = 0.0, o0 = 0.0, e1 = 0.0, o1 = 0.0, e2 = 0.0, o2 = 0.0;
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) {
      if constexpr (NBW == 3) {
        const double* c = scb + 3 * kc;  // (nb 0, nb 1, nb 2)
        dmma(e0, o0, pw, c[0]);
        dmma(e1, o1, pw, c[1]);
        dmma(e2, o2, pw, c[2]);
      } else if constexpr (NBW == 2) {
        const double2 c = *reinterpret_cast<const double2*>(scb + 2 * kc);  // (nb 0, nb 1)
        dmma(e0, o0, pw, c.x);
        dmma(e1, o1, pw, c.y);
      } else {
        dmma(e0, o0, pw, scb[kc]);
      }
      pw *= s4;
    }
    const double wp0 = fma(x1, o0, e0), wm0 = fma(-x1, o0, e0);  // taps tig, 2m - tig
    const double wp1 = fma(x1, o1, e1), wm1 = fma(-x1, o1, e1);  // taps 4 + tig, 2m - 4 - tig
    if (C::kShflA && d == 2) {
      zp0 = wp0;
      zm0 = wm0;
      zp1 = wp1;
      zm1 = wm1;
      z2 = e2;
      continue;
    }
    // entries j >= W of the tables stay 0 from the start of the kernel
    double* row = d == 2 ? wA + g * kAS + kAO : (d == 0 ? wX : wY) + g * kXS + kXO;
    if (tig <= MC) {
      row[tig] = wp0;
      row[2 * MC - tig] = wm0;
    }
    if (NBW > 1 && 4 + tig <= MC) {
      row[4 + tig] = wp1;
      row[2 * MC - 4 - tig] = wm1;
    }
    if (NBW > 2 && tig == 0) row[8] = e2;  // m = 8: the centre tap (O_8 = 0)
  }
  __syncwarp();
  // A fragments: axis-3 weights of point g at staged depth kz + 4 kc + tig
  double a[KC];
  if constexpr (C::kShflA) {
    // phi_j of point g, jj = min(j, 2m - j): lane 4g + (jj mod 4), register
    // set jj / 4, the mirrored copy for j > m
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      const int j = kz + 4 * kc + tig - ck;
      const bool mir = j > MC;
      const int jj = mir ? 2 * MC - j : j;
      const int src = 4 * g + (jj & 3);
      const double vp0 = __shfl_sync(0xffffffffu, zp0, src), vm0 = __shfl_sync(0xffffffffu, zm0, src);
      const double vp1 = __shfl_sync(0xffffffffu, zp1, src), vm1 = __shfl_sync(0xffffffffu, zm1, src);
      double v = (jj & 4) ? (mir ? vm1 : vp1) : (mir ? vm0 : vp0);
      if constexpr (NBW > 2) {
        const double v2 = __shfl_sync(0xffffffffu, z2, src);
        if (jj == 8) v = v2;
      }
      a[kc] = (inbox && j >= 0 && j < C::W) ? v : 0.0;
    }
  } else {
    const double* wa = wA + g * kAS + kAO + kz + tig - ck;
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      VFN_DCHECK(kAO + kz + tig - ck + 4 * kc >= 0 && kAO + kz + tig - ck + 4 * kc < kAS);
      a[kc] = inbox ? wa[4 * kc] : 0.0;
    }
  }
  const double* wx = wX + g * kXS + kXO - ci;  // wx[x], x in [0, 16); zero off the stencil
  const double* wy = wY + g * kXS + kXO - cj;  // wy[y]
  VFN_DCHECK(kXO - ci >= 0 && kXO - ci + XB <= kXS && kXO - cj >= 0 && kXO - cj + YB <= kXS);
  // the unit's K window [kz, kz + 4 KC) of staged depths holds every point's
  // stencil (staged depths ck .. ck + W - 1) and lies inside the staged tile
#ifdef VFN_CHECKS
  if (!(kz >= 0 && kz + 4 * KC <= kSZ && (!inbox || (ck >= kz && ck + C::W <= kz + 4 * KC))))
    printf("unit window: m %d KC %d kz %d ck %d desc (%d, %d, %d) tile %d oz %d cell %d %d %d cnt %d g %d\n", MC, KC,
           kz, ck, desc.x, desc.y, desc.z, tile, oz, cell[0], cell[1], cell[2], cnt, g);
#endif
  VFN_DCHECK(kz >= 0 && kz + 4 * KC <= kSZ && (!inbox || (ck >= kz && ck + C::W <= kz + 4 * KC)));

  while (*reinterpret_cast<const volatile int*>(tw.loaded) != tw.kk) __nanosleep(64);
  mbar_wait(tw.bar, tw.parity);
  // SPLIT: this warp sums one component (half = 0: re, 1: im) of the unit's
  // values; everything named "re" below is that component, the "im" chains
  // are dead code
  const unsigned base = tile_s + (unsigned)((kz + tig) * 16 + (X0 * C::SY + Y0) * kLine + (SPLIT ? 8 * half : 0));
  constexpr unsigned kX = C::SY * kLine;  // x stride
  // parts of the YB rows: one R8 run per 8 rows, then R4 / R2 / R1 for the rest
  constexpr int Y8 = YB / 8;
  constexpr int R4 = (YB - 8 * Y8) >= 4;
  constexpr int R2 = (YB - 8 * Y8 - 4 * R4) >= 2;
  constexpr int R1 = (YB - 8 * Y8 - 4 * R4 - 2 * R2);
  static_assert(Y8 <= 2 && R1 <= 1, "row schedule");
  double acc_re = 0.0, acc_im = 0.0;
#pragma unroll
  for (int y8 = 0; y8 < Y8; ++y8) {
    double t0r = 0.0, t1r = 0.0, t0i = 0.0, t1i = 0.0;
    const unsigned ba = base + (8 * y8 + g) * kLine;
#pragma unroll
    for (int x = 0; x < XB; ++x) {
      double cr0, cr1, ci0_, ci1_;
      tile_mma<KC, SPLIT>(ba + x * kX, a, cr0, cr1, ci0_, ci1_, tile_s, tile_s + C::kTileBytes);
      const double w = wx[x];
      t0r = fma(w, cr0, t0r);
      t1r = fma(w, cr1, t1r);
      t0i = fma(w, ci0_, t0i);
      t1i = fma(w, ci1_, t1i);
    }
    const double wy0 = wy[8 * y8 + 2 * tig], wy1 = wy[8 * y8 + 2 * tig + 1];
    acc_re = fma(wy0, t0r, fma(wy1, t1r, acc_re));
    acc_im = fma(wy0, t0i, fma(wy1, t1i, acc_im));
  }
  constexpr int y4 = 8 * Y8;
  if constexpr (R4) {
    double t0r = 0.0, t1r = 0.0, t0i = 0.0, t1i = 0.0;
    const int xb = g >> 2, xc = tig >> 1;
    const unsigned bb = base + (y4 + (g & 3)) * kLine;
#pragma unroll
    for (int p = 0; p < (XB + 1) / 2; ++p) {
      double cr0, cr1, ci0_, ci1_;
      tile_mma<KC, SPLIT>(bb + min(2 * p + xb, XB - 1) * kX, a, cr0, cr1, ci0_, ci1_, tile_s, tile_s + C::kTileBytes);
      const double w = wx[2 * p + xc];
      t0r = fma(w, cr0, t0r);
      t1r = fma(w, cr1, t1r);
      t0i = fma(w, ci0_, t0i);
      t1i = fma(w, ci1_, t1i);
    }
    const double wy0 = wy[y4 + 2 * (tig & 1)], wy1 = wy[y4 + 1 + 2 * (tig & 1)];
    acc_re = fma(wy0, t0r, fma(wy1, t1r, acc_re));
    acc_im = fma(wy0, t0i, fma(wy1, t1i, acc_im));
  }
  constexpr int y2 = y4 + 4 * R4;
  if constexpr (R2) {
    double t0r = 0.0, t1r = 0.0, t0i = 0.0, t1i = 0.0;
    const unsigned bc = base + (y2 + (g & 1)) * kLine;
#pragma unroll
    for (int q = 0; q < (XB + 3) / 4; ++q) {
      double cr0, cr1, ci0_, ci1_;
      tile_mma<KC, SPLIT>(bc + min(4 * q + (g >> 1), XB - 1) * kX, a, cr0, cr1, ci0_, ci1_, tile_s, tile_s + C::kTileBytes);
      const double w = wx[4 * q + tig];
      t0r = fma(w, cr0, t0r);
      t1r = fma(w, cr1, t1r);
      t0i = fma(w, ci0_, t0i);
      t1i = fma(w, ci1_, t1i);
    }
    const double wy0 = wy[y2], wy1 = wy[y2 + 1];
    acc_re = fma(wy0, t0r, fma(wy1, t1r, acc_re));
    acc_im = fma(wy0, t0i, fma(wy1, t1i, acc_im));
  }
  constexpr int y1 = y2 + 2 * R2;
  if constexpr (R1) {
    double tr = 0.0, ti = 0.0;
    const unsigned bd = base + y1 * kLine;
#pragma unroll
    for (int q = 0; q < (XB + 7) / 8; ++q) {
      double cr0, cr1, ci0_, ci1_;
      tile_mma<KC, SPLIT>(bd + min(8 * q + g, XB - 1) * kX, a, cr0, cr1, ci0_, ci1_, tile_s, tile_s + C::kTileBytes);
      // past the footprint the x weights are 0 (m = 8: the octets reach past
      // the x table, whose rows are kXS = XB + 2 long)
      const int xa = 8 * q + 2 * tig;
      const double w0 = (8 * ((XB + 7) / 8) <= kXS - kXO || xa < XB) ? wx[xa] : 0.0;
      const double w1 = (8 * ((XB + 7) / 8) <= kXS - kXO || xa + 1 < XB) ? wx[xa + 1] : 0.0;
      tr = fma(w0, cr0, fma(w1, cr1, tr));
      ti = fma(w0, ci0_, fma(w1, ci1_, ti));
    }
    const double wy0 = wy[y1];
    acc_re = fma(wy0, tr, acc_re);
    acc_im = fma(wy0, ti, acc_im);
  }
  acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 1);
  if constexpr (!SPLIT) acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 1);
  acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 2);
  if constexpr (!SPLIT) acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 2);
  if (valid && tig == 0) {
    const double2 v = make_double2(acc_re, acc_im);
    if constexpr (PEER) {
      // fused return exchange: the value goes straight to the rank whose
      // block the point came from (IPC-mapped peer memory over NVLink)
      const PeerTable* T = A.peer;
      int o = 0;
      while (o + 1 < T->n && prow >= T->off[o + 1]) ++o;
      if constexpr (SPLIT)
        reinterpret_cast<double*>(T->out[o] + T->rows[prow])[half] = acc_re;
      else
        T->out[o][T->rows[prow]] = v;
    } else {
      if constexpr (SPLIT)
        __stcs(reinterpret_cast<double*>(A.out + prow) + half, acc_re);
      else
        __stcs(A.out + prow, v);
    }
  }
  __syncwarp();  // the weight tables are rewritten by the next unit
}

template <int MC, int BXY, bool PEER, bool SPLIT>
__device__ __forceinline__ void dispatch_unit(const Args& A, const double* scb, double* wt, unsigned tile_s,
                                              int tile, int ox, int oy, int oz, int4 desc,
                                              const UnitPoints& up, int lane, int half, const TileWait& tw) {
  const int kc = (desc.y >> 4) & 7;
  if constexpr (Cfg<MC>::KCmin <= 2) {
    if (kc == 2)
      return gather_unit<MC, BXY, 2, PEER, SPLIT>(A, scb, wt, tile_s, tile, ox, oy, oz, desc, up, lane, half, tw);
  }
  if constexpr (Cfg<MC>::KCmin <= 3) {
    if (kc == 3)
      return gather_unit<MC, BXY, 3, PEER, SPLIT>(A, scb, wt, tile_s, tile, ox, oy, oz, desc, up, lane, half, tw);
  }
  if constexpr (Cfg<MC>::KCmin <= 4) {
    if (kc == 4)
      return gather_unit<MC, BXY, 4, PEER, SPLIT>(A, scb, wt, tile_s, tile, ox, oy, oz, desc, up, lane, half, tw);
  }
  gather_unit<MC, BXY, 5, PEER, SPLIT>(A, scb, wt, tile_s, tile, ox, oy, oz, desc, up, lane, half, tw);
}

// SPLIT (low-density passes): every unit is handed out twice, once from each
// of two CTA counters — even warps take units from the first and sum the
// real parts, odd warps from the second and sum the imaginary parts.  The
// two components never mix in the contraction, so each value's bits are
// those of the unsplit kernel; a sparse tile's few units then occupy twice
// as many warps for half as long (the pass is bound by units in flight x
// unit latency, DESIGN 4).
template <int MC, int BXY, int kWarps, bool PEER, bool SPLIT>
__global__ void __launch_bounds__(kWarps * 32, 1)
    k_gather_tc(const __grid_constant__ CUtensorMap tmap, const Args A) {
  using C = Cfg<MC>;
  extern __shared__ unsigned char smem_raw[];
  const unsigned raw = (unsigned)__cvta_generic_to_shared(smem_raw);
  const unsigned tiles_s = (raw + 1023u) & ~1023u;          // 2 x kTileBytes
  const unsigned bar_s = tiles_s + 2 * C::kTileBytes;       // full[2]
  unsigned char* ctl = smem_raw + (bar_s - raw);
  int* done = reinterpret_cast<int*>(ctl + 16);              // done[2]
  int* ctr = done + 2;                                       // next CTA unit to hand out (ctr[half] with SPLIT)
  int* loaded = done + 4;                                    // loaded[2]: item ordinal per buffer
  double* wts = reinterpret_cast<double*>(ctl + 48);         // [kWarps][kWarpW]
  double* scb_all = wts + kWarps * C::kWarpW;                // [32 lanes][C::kScb]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  for (int i = tid; i < kWarps * C::kWarpW; i += blockDim.x) wts[i] = 0.0;  // zero pads
  // B fragments of the weights DMMA, per lane in shared memory (kept out of
  // the register budget): row k = 4 kc + tig is the power s^k, column 8 nb + g
  // is tap j = 4 nb + g / 2, even part (g even: coefficient of delta^2k) or
  // odd part (delta^(2k+1)); the fit's taps j and 2m - j are averaged into
  // one exactly mirror-symmetric polynomial
  if (warp == 0) {
#pragma unroll
    for (int kc = 0; kc < 2; ++kc)
#pragma unroll
      for (int nb = 0; nb < C::kNB; ++nb) {
        const int j = 4 * nb + (g >> 1), d = 2 * (4 * kc + tig) + (g & 1);
        double c = 0.0;
        if (d <= A.deg && j <= MC) {
          const double cj = A.poly[j * (A.deg + 1) + d], cm = A.poly[(2 * MC - j) * (A.deg + 1) + d];
          c = 0.5 * ((g & 1) ? cj - cm : cj + cm);
        }
        scb_all[lane * C::kScb + C::kNB * kc + nb] = c;
      }
  }
  const double* scb = scb_all + lane * C::kScb;
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
    ctr[0] = ctr[1] = 0;
    loaded[0] = 0;
    loaded[1] = 1;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    issue_tile<MC>(&tmap, A, item_of(0), tiles_s, bar_s);
    issue_tile<MC>(&tmap, A, item_of(1), tiles_s + C::kTileBytes, bar_s + 8);
  }
  __syncthreads();

  double* wt = wts + warp * C::kWarpW;
  const BinGeom& G = A.g;
  // Units are handed out from one monotonic CTA counter over the
  // concatenated units of this CTA's items (item k = items[blockIdx.x +
  // k * gridDim.x]); each warp walks the item list forward to locate the unit
  // it grabbed, reserves its next unit and prefetches its points before
  // computing the current one.  A tile buffer is refilled (item k+2) by the
  // warp that completes the last unit of item k.
  struct Cur {
    int k;      // item ordinal within this CTA
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
        VFN_DCHECK(walk.item.y + (u - walk.base) < walk.item.z && walk.item.z <= A.nunits);
        desc = __ldg(A.units + walk.item.y + (u - walk.base));
        return true;
      }
      walk.base += n;
      ++walk.k;
      const int itn = item_of(walk.k);
      walk.item = itn < nitems ? A.items[itn] : make_int4(0, 0, 0, 0);
    }
  };
  const int half = SPLIT ? (warp & 1) : 0;
  auto grab = [&]() {
    int v = 0;
    if (lane == 0) v = atomicAdd(ctr + half, 1);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  // Narrow stencils on dense tiles (m <= 5: a unit is 30-130 DMMAs, shorter
  // than or close to the DRAM round trips of its descriptor -> permutation
  // -> u loads): a three-stage software pipeline per warp, so that no load
  // is waited for in the iteration that issued it — while unit n is
  // computed, unit n+1's u values, unit n+2's permutation entries and unit
  // n+3's descriptor are in flight (c5 gathers at m = 2 / 3 / 4 / 5: 61.9 /
  // 46.2 / 72.4 / 81.5 -> 52.7 / 42.3 / 69.5 / 79.8 ms).  At m = 6 it gains
  // 0.4% on the dense gather and loses 5% end to end (the deeper reservation
  // binds the mid-density chunks' units too early); m >= 7 spills.
  if constexpr (MC <= 5 && kWarps == kWarpsDense && !SPLIT) {
    struct Pend {
      int4 desc, item;
      int kk;
      bool have;
    };
    auto fetch_desc = [&](Pend& q) {
      q.kk = 0;
      q.desc = make_int4(0, 0, 0, 0);
      q.item = make_int4(0, 0, 0, 0);
      q.have = locate(grab(), q.desc, q.kk, q.item);
    };
    auto load_perm = [&](const Pend& q) -> int {
      if (!q.have || g >= (q.desc.y & 15)) return 0;
      VFN_DCHECK(q.desc.x >= 0 && q.desc.x + g < A.M);
      return __ldcs(A.perm + q.desc.x + g);
    };
    auto load_u = [&](const Pend& q, int prow, UnitPoints& up) {
      up.prow = prow;
      up.uu[0] = up.uu[1] = up.uu[2] = 0.0;
      if (q.have && g < (q.desc.y & 15)) {
        VFN_DCHECK(prow >= 0 && prow < A.M);
#pragma unroll
        for (int d = 0; d < 3; ++d) up.uu[d] = __ldcs(A.u + 3 * (int64_t)prow + d);
      }
    };
    Pend c0, c1, c2;
    fetch_desc(c0);
    fetch_desc(c1);
    fetch_desc(c2);
    int prow1 = load_perm(c1);
    UnitPoints up;
    load_u(c0, load_perm(c0), up);
    while (c0.have) {
      Pend c3;
      fetch_desc(c3);                   // unit n + 3: descriptor
      const int prow2 = load_perm(c2);  // unit n + 2: permutation entries
      UnitPoints up_n;
      load_u(c1, prow1, up_n);          // unit n + 1: u values
      const int kk = c0.kk, b = kk & 1, tile = c0.item.x;
      const int t2 = tile % G.ntile[2];
      const int t1 = (tile / G.ntile[2]) % G.ntile[1];
      const int t0 = tile / (G.ntile[2] * G.ntile[1]);
      const unsigned tile_s = tiles_s + b * C::kTileBytes;
      const TileWait tw{&loaded[b], kk, bar_s + 8 * b, (unsigned)((kk >> 1) & 1)};
      dispatch_unit<MC, BXY, PEER, SPLIT>(A, scb, wt, tile_s, tile, t0 * C::TX, t1 * C::TY, t2 * C::TZ, c0.desc, up,
                                          lane, half, tw);
      if (lane == 0) {
        if (atomicAdd(&done[b], 1) == c0.item.z - c0.item.y - 1) {  // last unit of item kk
          done[b] = 0;
          if (item_of(kk + 2) < nitems) {
            *reinterpret_cast<volatile int*>(&loaded[b]) = kk + 2;
            issue_tile<MC>(&tmap, A, item_of(kk + 2), tile_s, bar_s + 8 * b);
          }
        }
      }
      c0 = c1;
      c1 = c2;
      c2 = c3;
      prow1 = prow2;
      up = up_n;
    }
    if constexpr (PEER) __threadfence_system();
    return;
  }
  int4 desc, item;
  int kk = 0;
  UnitPoints up;
  bool have = locate(grab(), desc, kk, item);
  if (have) up = load_unit_points(A, desc, g);
  while (have) {
    int4 desc_n, item_n;
    int kk_n = 0;
    UnitPoints up_n;
    // Dense tiles: the next unit is reserved and its points prefetched before
    // the current one is computed (its descriptor -> permutation -> u loads
    // hide behind ~16k cycles of DMMAs).  Sparse modes bind late instead: a
    // warp takes its next unit only when it is free, because a unit reserved
    // early sits behind its warp's current one while other warps idle (few
    // units per staged tile), and the load round trips overlap the wait for
    // the tile anyway (c5 chunks of 0.06 / 0.16 / 0.22: 26.3 / 36 / 39.0 ->
    // 23.3 / 32.9 / 37.8 ms, config 2 0.675 -> 0.652 ms; dense c5 would lose:
    // 127.8 -> 131.4 ms).  The wide stencils' small tiles hold few units at
    // any density (m = 8: 2 x 2 x 4 cells, ~4 units at c5), so they bind late
    // too: c5 at m = 8 365 -> 318 ms, m = 7 165.1 -> 163.8 ms
    constexpr bool kLate = (kWarps == kWarpsSparse) || SPLIT || MC >= 7;
    bool have_n = false;
    if constexpr (!kLate) {
      have_n = locate(grab(), desc_n, kk_n, item_n);
      if (have_n) up_n = load_unit_points(A, desc_n, g);
    }
    const int b = kk & 1;
    const int tile = item.x;
    const int t2 = tile % G.ntile[2];
    const int t1 = (tile / G.ntile[2]) % G.ntile[1];
    const int t0 = tile / (G.ntile[2] * G.ntile[1]);
    const unsigned tile_s = tiles_s + b * C::kTileBytes;
    // a warp may hold units of items far ahead (small items); the unit waits
    // for its tile once its weights are computed (TileWait)
    const TileWait tw{&loaded[b], kk, bar_s + 8 * b, (unsigned)((kk >> 1) & 1)};
    dispatch_unit<MC, BXY, PEER, SPLIT>(A, scb, wt, tile_s, tile, t0 * C::TX, t1 * C::TY, t2 * C::TZ, desc, up, lane,
                                        half, tw);
    if (lane == 0) {
      if (atomicAdd(&done[b], 1) == (SPLIT ? 2 : 1) * (item.z - item.y) - 1) {  // last (half-)unit of item kk
        done[b] = 0;
        if (item_of(kk + 2) < nitems) {
          *reinterpret_cast<volatile int*>(&loaded[b]) = kk + 2;
          issue_tile<MC>(&tmap, A, item_of(kk + 2), tile_s, bar_s + 8 * b);
        }
      }
    }
    if constexpr (kLate) {
      have_n = locate(grab(), desc_n, kk_n, item_n);
      if (have_n) up_n = load_unit_points(A, desc_n, g);
    }
    have = have_n;
    desc = desc_n;
    item = item_n;
    kk = kk_n;
    up = up_n;
  }
  if constexpr (PEER) __threadfence_system();  // peer stores visible before the owners read
}

}  // namespace tc

// ------------------------------------------------------------------ units

// A box's points are sorted by depth pair and the box is TZ cells deep, so
// any 8 consecutive points span <= TZ - 1 depths: units are the box's chunks
// of 8, each with the fewest k-chunks (K = 4 KC depths) covering the
// stencils of its depth-pair range.
__global__ void k_unit_counts(const int32_t* __restrict__ box_start, int64_t nboxes,
                              int32_t* __restrict__ ucount) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nboxes) return;
  ucount[b] = b == nboxes ? 0 : (box_start[b + 1] - box_start[b] + tc::kUnitPts - 1) / tc::kUnitPts;
}

// floor(x / d) for x < 2^32, d <= 256: (x * ceil(2^40 / d)) >> 40 is exact
// (the rounding error stays below x / 2^40 < 1/256 <= 1/d); the product
// needs up to 72 bits, so its high word comes from __umul64hi
struct Div {
  uint64_t inv;
  uint32_t d;
  __device__ __forceinline__ uint32_t q(uint32_t x) const {
    const uint64_t lo = (uint64_t)x * inv, hi = __umul64hi((uint64_t)x, inv);
    return (uint32_t)((hi << 24) | (lo >> 40));
  }
};
static Div make_div(uint32_t d) { return Div{((uint64_t(1) << 40) + d - 1) / d, d}; }

// Eight consecutive sorted points per thread (two 16-byte key loads); the
// point that opens a chunk of 8 in its box writes the unit (fully parallel,
// also for boxes holding millions of points — config 3).
__global__ void k_write_units(const uint32_t* __restrict__ keys, int64_t M,
                              const int32_t* __restrict__ box_start, Div cpb, int shift, int W,
                              int kcmin, const int32_t* __restrict__ uoff, int4* __restrict__ units) {
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i0 >= M) return;
  uint32_t k[8];
  if (i0 + 8 <= M) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(keys + i0));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(keys + i0) + 1);
    k[0] = a.x, k[1] = a.y, k[2] = a.z, k[3] = a.w, k[4] = b.x, k[5] = b.y, k[6] = b.z, k[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) k[j] = i0 + j < M ? keys[i0 + j] : 0u;
  }
  int64_t cur = -1;
  int bs = 0, be = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t i = i0 + j;
    if (i >= M) break;
    const int64_t b = cpb.q(k[j]);
    if (b != cur) {  // sorted: a thread's 8 points span few boxes
      cur = b;
      bs = box_start[b];
      be = box_start[b + 1];
    }
    const int r = (int)i - bs;
    if (r & (tc::kUnitPts - 1)) continue;
    const int e = min(be, (int)i + tc::kUnitPts);
    const uint32_t klast = e - 1 - i0 < 8 ? k[e - 1 - i0] : keys[e - 1];
    // the key holds depth >> shift: the unit's depths lie in [q0 << s, ((q1 + 1) << s) - 1]
    const int k0 = (int)(k[j] - cpb.q(k[j]) * cpb.d) << shift;
    const int k1 = (((int)(klast - cpb.q(klast) * cpb.d) + 1) << shift) - 1;
    const int kc = max(kcmin, (k1 - k0 + W + 3) / 4);  // span + W <= 4 kc  (<= 20 always)
    const int kz = min(k0, tc::kSZ - 4 * kc);
    units[uoff[b] + r / tc::kUnitPts] = make_int4((int)i, (e - (int)i) | (kc << 4) | (kz << 8), (int)b, 0);
  }
}

__global__ void k_tc_tile_items(const int32_t* __restrict__ uoff, int64_t ntiles, int bpt,
                                int32_t* __restrict__ nitems) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  if (t == ntiles) {
    nitems[t] = 0;
    return;
  }
  const int units = uoff[(t + 1) * bpt] - uoff[t * bpt];
  nitems[t] = (units + tc::kItemUnits - 1) / tc::kItemUnits;
}

__global__ void k_tc_items(const int32_t* __restrict__ uoff, const int32_t* __restrict__ ioff,
                           int64_t ntiles, int bpt, int4* __restrict__ items) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int first = ioff[t], n = ioff[t + 1] - first;
  const int u0 = uoff[t * bpt], u1 = uoff[(t + 1) * bpt];
  for (int j = 0; j < n; ++j)
    items[first + j] = make_int4((int)t, u0 + j * tc::kItemUnits, min(u1, u0 + (j + 1) * tc::kItemUnits), 0);
}

bool tc_supported(int m) { return m >= 2 && m <= 8; }

void tc_tile_xy(int m, int* tx, int* ty) {
  *tx = m == 8 ? 2 : 4;
  *ty = m >= 7 ? 2 : 4;
}

// box widths the tensor-core gather takes at cutoff m
int tc_max_box(int m) { return m >= 2 && m <= 8 ? 2 : 1; }

int tc_tile_depth(int m) { return tc::kSZ - 2 * m; }

// Tensor map over the ghost-padded grid as doubles: (2 P2, P1, P0), box
// (40 doubles, 4 + 2m, 4 + 2m), no swizzle.
int make_grid_tmap(vfn_plan* p) {
  p->has_tmap = false;
  if (!tc_supported(p->m)) return VFN_OK;
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
  int tx, ty;
  tc_tile_xy(p->m, &tx, &ty);
  cuuint64_t dims[3] = {(cuuint64_t)(2 * p->P[2]), (cuuint64_t)p->P[1], (cuuint64_t)p->P[0]};
  cuuint64_t strides[2] = {(cuuint64_t)(2 * p->P[2] * 8), (cuuint64_t)(2 * p->P[2] * 8 * p->P[1])};
  cuuint32_t box[3] = {2 * tc::kSZ, (cuuint32_t)(ty + 2 * p->m), (cuuint32_t)(tx + 2 * p->m)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<Fn>(fn)(&p->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, p->grid, dims,
                                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(VFN_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  p->has_tmap = true;
  return VFN_OK;
}

bool tc_applicable(const vfn_plan* p, const BinGeom& g) {
  if (!tc_supported(p->m) || !p->has_tmap || p->poly.deg > 15) return false;
  const int tz = tc_tile_depth(p->m);
  int tx, ty;
  tc_tile_xy(p->m, &tx, &ty);
  return g.tile[0] == tx && g.tile[1] == ty && g.tile[2] == tz && g.box[2] == tz && g.box[0] == g.box[1] &&
         g.box[0] >= 1 && g.box[0] <= tc_max_box(p->m);
}

template <int MC, int BXY, int NW, bool PEER, bool SPLIT>
static int launch_k(vfn_plan* p, const tc::Args& A, cudaStream_t s) {
  const size_t smem = tc::smem_bytes(MC, NW);
  VFN_CUDA(cudaFuncSetAttribute(tc::k_gather_tc<MC, BXY, NW, PEER, SPLIT>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  tc::k_gather_tc<MC, BXY, NW, PEER, SPLIT><<<nsm, NW * 32, smem, s>>>(p->tmap, A);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

// the peer-store epilogue (sharded evaluates) is its own instantiation, so
// the plain kernel carries none of its code
template <int MC, int BXY, int NW, bool SPLIT>
static int launch(vfn_plan* p, const tc::Args& A, cudaStream_t s) {
  return A.peer ? launch_k<MC, BXY, NW, true, SPLIT>(p, A, s) : launch_k<MC, BXY, NW, false, SPLIT>(p, A, s);
}

template <int MC>
static int launch_m(vfn_plan* p, const tc::Args& A, int bxy, cudaStream_t s) {
  if constexpr (MC == 8) {
    // two 18 x 18-line tiles (2 x 2 x 4 cells, up to 4 units each at c5's
    // density) and the weight tables fit next to 8 warps: every warp has a
    // unit while the other tile loads (2 x 1 tiles with 12 warps kept 4 of
    // 12 warps busy: 656 ms at c5)
    if (bxy == 1) return launch<8, 1, 8, false>(p, A, s);
    return launch<8, 2, 8, false>(p, A, s);
  } else {
    // by points per 1x1x8 column (c5: 16), measured on chunks of c5: 16-warp
    // CTAs with prefetch from 4.8 up (a 0.32 chunk at 5.1: 48.0 ms against
    // 49.1 with 12 warps), 12-warp CTAs binding late from 1.7 (config 2 at
    // 3.8; a 0.22 chunk at 3.5: 37.8 against 45.3 ms with half-units),
    // half-units on 16 warps below (a 0.06 chunk at 1.0: 23.3 against 26.5 ms).
    // Half-units only when the density saw the points: below 2^20 points it
    // is the grid-wide mean, and a small clustered set's tiles are dense
    // (half-units on dense tiles cost up to 36%, the 12-warp kernel ~5%)
    int mode = (p->col_density < tc::kSplitDensity && p->col_density_sampled)
                   ? 2
                   : (p->col_density < tc::kSparseDensity ? 1 : 0);
    if (const char* e = std::getenv("VFN_WARPS")) {  // experiments: 16, 12, or s16 (half-units)
      mode = e[0] == 's' ? 2 : (std::atoi(e) == tc::kWarpsSparse ? 1 : 0);
    }
    if (mode == 2)
      return bxy == 1 ? launch<MC, 1, tc::kWarpsDense, true>(p, A, s) : launch<MC, 2, tc::kWarpsDense, true>(p, A, s);
    if (bxy == 1)
      return mode == 1 ? launch<MC, 1, tc::kWarpsSparse, false>(p, A, s)
                       : launch<MC, 1, tc::kWarpsDense, false>(p, A, s);
    return mode == 1 ? launch<MC, 2, tc::kWarpsSparse, false>(p, A, s)
                     : launch<MC, 2, tc::kWarpsDense, false>(p, A, s);
  }
}

// Build units and items from the box offsets, then run the tensor-core gather.
int launch_tc(vfn_plan* p, const double* u, const int32_t* perm, const uint32_t* keys_sorted,
              const int32_t* box_start, double2* out, const BinGeom& g, int64_t M,
              cudaStream_t s) {
  const int64_t nb = g.nboxes;
  const int W = 2 * p->m + 1;
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
  if (g.key_slots > 256) return fail(VFN_ERR_INVALID, "box too deep for the unit builder");
  k_write_units<<<(unsigned)(((M + 7) / 8 + 255) / 256), 256, 0, s>>>(keys_sorted, M, box_start,
                                                                      make_div((uint32_t)g.key_slots), g.key_shift, W,
                                                                      (W + 3) / 4,
                                                                      uoff, p->units.as<int4>());
  VFN_CUDA(cudaGetLastError());
  const unsigned tb = (unsigned)((g.ntiles + 1 + 255) / 256);
  k_tc_tile_items<<<tb, 256, 0, s>>>(uoff, g.ntiles, g.boxes_per_tile, nitems);
  VFN_CUDA(cudaGetLastError());
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(p->sort_tmp.ptr, t2, nitems, ioff, (int)(g.ntiles + 1), s));
  const int64_t max_items = std::min<int64_t>(g.ntiles, M) + M / tc::kItemUnits + 1;
  VFN_CHECK(p->items.ensure(sizeof(int4) * max_items));
  k_tc_items<<<tb, 256, 0, s>>>(uoff, ioff, g.ntiles, g.boxes_per_tile, p->items.as<int4>());
  VFN_CUDA(cudaGetLastError());

  tc::Args A;
  A.u = u;
  A.perm = perm;
  A.units = p->units.as<int4>();
  A.items = p->items.as<int4>();
  A.nitems = ioff + g.ntiles;
  A.out = out;
  A.poly = p->poly.dev;
  A.deg = p->poly.deg;
  A.M = M;
  A.nunits = M + 1;
  A.tm = p->map;
  A.g = g;
  A.peer = p->peer_dev;
  if (p->peer_dev) p->peer_used = true;
  mark_event(p, 1, s);  // gather timing starts here (binning prep excluded)
  switch (p->m) {
    case 2: return launch_m<2>(p, A, g.box[0], s);
    case 3: return launch_m<3>(p, A, g.box[0], s);
    case 4: return launch_m<4>(p, A, g.box[0], s);
    case 5: return launch_m<5>(p, A, g.box[0], s);
    case 7: return launch_m<7>(p, A, g.box[0], s);
    case 8: return launch_m<8>(p, A, g.box[0], s);
    default: return launch_m<6>(p, A, g.box[0], s);
  }
}

}  // namespace vfn
