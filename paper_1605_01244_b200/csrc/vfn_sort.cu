// Stable LSD radix sort of (uint32 key, int32 value) pairs for the bin sort
// (perm = stable argsort of the bin keys).  8-bit digits,
// ceil(key_bits / 8) passes (the depth-pair key of c5 has 24 bits: 3 passes);
// the first pass's values are the implicit row index (no iota array read).
//
// Each pass is reduce-then-scan over a fixed segmentation of the input into
// kBlocks contiguous segments (one per CTA, in order):
//   1. k_rs_upsweep:   per-segment digit histograms       (4 B per key read)
//   2. k_rs_scan:      one CTA scans the digit-major (digit, segment) counts
//   3. k_rs_downsweep: each CTA walks its segment in tiles of 4096 keys; a
//      warp owns 512 consecutive keys, lane l holding keys l, l + 32, ...,
//      so processing item j for all lanes visits the warp's keys in input
//      order; __match_any_sync peers + warp-private digit counters give each
//      key its stable rank inside the tile, the tile is reordered by digit in
//      shared memory and written out run by run (coalesced), after the
//      segment's running offset of each digit.
// Stability: segments, tiles, warps and items are all visited in input
// order, so equal digits keep their relative order in every pass.
#include <algorithm>

#include "vfn_device.cuh"

namespace vfn {

namespace rs {

constexpr int kRadix = 256;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;                        // keys per lane per tile
constexpr int kTile = kThreads * kItems;          // 4096 keys
constexpr int kWarpKeys = 32 * kItems;            // 512 consecutive keys per warp

__global__ void __launch_bounds__(kThreads) k_rs_upsweep(const uint32_t* __restrict__ keys, int64_t M, int64_t seg,
                                                         int shift, int nseg, int32_t* __restrict__ counts) {
  __shared__ int h[kWarps][kRadix];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * seg, hi = min(M, lo + seg);
  // 16-byte loads: segments are multiples of the tile (4096 keys)
  const int64_t n4 = (hi - lo) >> 2;
  const uint4* k4 = reinterpret_cast<const uint4*>(keys + lo);
  for (int64_t i = threadIdx.x; i < n4; i += kThreads) {
    const uint4 v = __ldcs(k4 + i);
    atomicAdd(&h[warp][(v.x >> shift) & 0xff], 1);
    atomicAdd(&h[warp][(v.y >> shift) & 0xff], 1);
    atomicAdd(&h[warp][(v.z >> shift) & 0xff], 1);
    atomicAdd(&h[warp][(v.w >> shift) & 0xff], 1);
  }
  for (int64_t i = lo + 4 * n4 + threadIdx.x; i < hi; i += kThreads) atomicAdd(&h[warp][(keys[i] >> shift) & 0xff], 1);
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += kThreads) {
    int t = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) t += h[w][d];
    counts[(int64_t)d * nseg + blockIdx.x] = t;
  }
}

// Exclusive scan of n ints in place by one CTA of 1024 threads: chunks of
// 4096 (four consecutive ints per thread, coalesced), warp-shuffle scans and
// a carried chunk total.
__global__ void __launch_bounds__(1024) k_rs_scan(int32_t* __restrict__ a, int n) {
  __shared__ int wsum[32];
  __shared__ int carry_s;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) carry_s = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += 4096) {
    const int i0 = c0 + 4 * t;
    int v[4], s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = i0 + k < n ? a[i0 + k] : 0;
      s += v[k];
    }
    int incl = s;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int w = wsum[lane];
      int wi = w;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wi, off);
        if (lane >= off) wi += y;
      }
      wsum[lane] = wi - w;  // exclusive warp offsets
    }
    __syncthreads();
    int e = carry_s + wsum[warp] + incl - s;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (i0 + k < n) a[i0 + k] = e;
      e += v[k];
    }
    __syncthreads();
    if (t == 1023) carry_s = e;  // the chunk's last running value
    __syncthreads();
  }
}

template <bool IOTA>
__global__ void __launch_bounds__(kThreads, 4) k_rs_downsweep(const uint32_t* __restrict__ kin,
                                                              const int32_t* __restrict__ vin,
                                                              uint32_t* __restrict__ kout, int32_t* __restrict__ vout,
                                                              int64_t M, int64_t seg, int shift, int nseg,
                                                              const int32_t* __restrict__ offs) {
  __shared__ int wc[kWarps][kRadix];      // per-warp digit counts of the tile, then the warps' prefixes
  __shared__ int dstart[kRadix + 1];      // digit starts inside the tile
  __shared__ int run[kRadix];             // next output position of each digit (this segment)
  __shared__ uint32_t sk[kTile];          // the tile's keys, loaded once; reordered by digit in place of sv below
  __shared__ int32_t sv[kTile];
  // each key's rank among the warp's keys of its digit; aliases sv, which is
  // written only after every thread has read its ranks back
  uint16_t* rk = reinterpret_cast<uint16_t*>(sv);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int d = tid; d < kRadix; d += kThreads) run[d] = offs[(int64_t)d * nseg + blockIdx.x];
  const int64_t lo = (int64_t)blockIdx.x * seg, hi = min(M, lo + seg);
  const int wbase = warp * kWarpKeys;
  for (int64_t base = lo; base < hi; base += kTile) {
    const int n = (int)(hi - base < kTile ? hi - base : kTile);
    for (int i = tid; i < kWarps * kRadix; i += kThreads) (&wc[0][0])[i] = 0;
    __syncthreads();
    // rank: this warp's 512 keys item-major (key wbase + j * 32 + lane), so
    // the lanes of item j are in input order
    uint32_t kr[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int q = wbase + j * 32 + lane;
      kr[j] = q < n ? __ldcs(kin + base + q) : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int q = wbase + j * 32 + lane;
      const bool live = q < n;
      const int d = live ? (int)((kr[j] >> shift) & 0xff) : kRadix;  // kRadix: past the end
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int leader = __ffs(peers) - 1;
      int before = 0;
      if (lane == leader && live) {
        before = wc[warp][d];
        wc[warp][d] = before + __popc(peers);
      }
      before = __shfl_sync(0xffffffffu, before, leader);
      rk[q] = (uint16_t)(before + __popc(peers & ((1u << lane) - 1u)));
    }
    __syncthreads();
    // digit totals of the tile and each warp's prefix inside its digit
    for (int d = tid; d < kRadix; d += kThreads) {
      int s = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const int c = wc[w][d];
        wc[w][d] = s;
        s += c;
      }
      dstart[d + 1] = s;  // tile count of digit d (scanned below)
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 256 digit counts: 8 per lane
      int c[8], s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c[i] = dstart[1 + lane * 8 + i];
        s += c[i];
      }
      int incl = s;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      int e = incl - s;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        dstart[lane * 8 + i] = e;
        e += c[i];
      }
      if (lane == 31) dstart[kRadix] = e;
    }
    __syncthreads();
    // reorder the tile by digit in shared memory (tile positions first: rk
    // and sv share storage)
    int pos[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int q = wbase + j * 32 + lane;
      const int d = (int)((kr[j] >> shift) & 0xff);
      pos[j] = q < n ? dstart[d] + wc[warp][d] + rk[q] : -1;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int q = wbase + j * 32 + lane;
      if (pos[j] >= 0) {
        sk[pos[j]] = kr[j];
        sv[pos[j]] = IOTA ? (int32_t)(base + q) : __ldcs(vin + base + q);
      }
    }
    __syncthreads();
    // write the runs: position p of the tile belongs to digit d(p)
    for (int p = tid; p < n; p += kThreads) {
      const uint32_t key = sk[p];
      const int d = (int)((key >> shift) & 0xff);
      const int64_t o = (int64_t)run[d] + (p - dstart[d]);
      kout[o] = key;
      vout[o] = sv[p];
    }
    __syncthreads();
    for (int d = tid; d < kRadix; d += kThreads) run[d] += dstart[d + 1] - dstart[d];
    // run[] is read again only after the next tile's barriers
  }
}

}  // namespace rs

// keys_in is left untouched; keys_out / vals_out receive the sorted pairs.
// scratch: two key and value ping-pong buffers of M entries plus counters.
int radix_sort_pairs(DevBuf& tmp, const uint32_t* keys_in, uint32_t* keys_out, int32_t* vals_out, int64_t M,
                     int key_bits, cudaStream_t s) {
  if (M <= 0) return VFN_OK;
  if (M > INT32_MAX) return fail(VFN_ERR_INVALID, "radix sort: too many keys");
  const int passes = std::max(1, (key_bits + 7) / 8);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // segments: whole tiles, 4 per SM (the downsweep's residency)
  const int64_t tiles = (M + rs::kTile - 1) / rs::kTile;
  const int64_t per = std::max<int64_t>(1, (tiles + nsm * 4 - 1) / (nsm * 4));
  const int64_t seg = per * rs::kTile;
  const int nseg = (int)((M + seg - 1) / seg);
  const int ncnt = rs::kRadix * nseg;
  // scratch layout: counts | keys tmp | vals tmp (16-byte aligned pieces)
  const size_t cbytes = ((sizeof(int32_t) * (size_t)ncnt + 255) / 256) * 256;
  const size_t kbytes = ((sizeof(uint32_t) * (size_t)M + 255) / 256) * 256;
  VFN_CHECK(tmp.ensure(cbytes + 2 * kbytes));
  int32_t* counts = tmp.as<int32_t>();
  uint32_t* ktmp = reinterpret_cast<uint32_t*>(tmp.as<char>() + cbytes);
  int32_t* vtmp = reinterpret_cast<int32_t*>(tmp.as<char>() + cbytes + kbytes);
  // ping-pong so that the last pass lands in (keys_out, vals_out)
  const uint32_t* kin = keys_in;
  const int32_t* vin = nullptr;
  for (int pss = 0; pss < passes; ++pss) {
    const bool last_to_out = ((passes - 1 - pss) % 2) == 0;
    uint32_t* ko = last_to_out ? keys_out : ktmp;
    int32_t* vo = last_to_out ? vals_out : vtmp;
    const int shift = 8 * pss;
    rs::k_rs_upsweep<<<nseg, rs::kThreads, 0, s>>>(kin, M, seg, shift, nseg, counts);
    rs::k_rs_scan<<<1, 1024, 0, s>>>(counts, ncnt);
    if (pss == 0)
      rs::k_rs_downsweep<true><<<nseg, rs::kThreads, 0, s>>>(kin, nullptr, ko, vo, M, seg, shift, nseg, counts);
    else
      rs::k_rs_downsweep<false><<<nseg, rs::kThreads, 0, s>>>(kin, vin, ko, vo, M, seg, shift, nseg, counts);
    VFN_CUDA(cudaGetLastError());
    kin = ko;
    vin = vo;
  }
  return VFN_OK;
}

}  // namespace vfn
