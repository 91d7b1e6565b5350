// Multi-GPU key-range sharding of one point set (the reference
// allows evaluating disjoint point subsets on a shared immutable plan,
// SPEC.md:258-259).  Every rank holds a block of the input in input order;
// the ranks agree on splitters of a partition key, each rank partitions its
// block by destination (stable, so every destination receives its points in
// input order), the points move with one all-to-all (torch.distributed in
// parallel.py), every rank evaluates a spatially compact key range at full
// point density, and the values return with a second all-to-all and are put
// back in input order (vfn_gather_values).
//
// Partition key of a point: (tile << 32) | global row, where tile is the
// row-major index of the gather tile of its nearest oversampled cell (the
// tensor-core geometry's 4 x 4 x TZ tiles, independent of the box width) —
// so a key range is a run of whole tiles (x-slabs for a uniform set), and
// ties inside one tile (config 3's dense cloud) are split by row.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "vfn_device.cuh"

namespace vfn {

namespace {

constexpr int kPartMax = 256;    // destinations
constexpr int kPartThreads = 256;
constexpr int kPartRounds = 16;  // points per thread per block
constexpr int kPartChunk = kPartThreads * kPartRounds;

struct TileMap {
  TorusMap tm;
  int tile[3];
  int ntile[3];
};

__device__ __forceinline__ uint64_t tile_of(const double* __restrict__ pts, int64_t i, const TileMap& T,
                                            bool& ok) {
  int c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double x = pts[3 * i + d];
    ok = ok && inside(x, T.tm.a[d], T.tm.b[d]);
    double delta;
    c[d] = nearest_cell(x, T.tm.a[d], T.tm.amb[d], T.tm.nd[d], T.tm.n[d], delta) / T.tile[d];
  }
  return ((uint64_t)c[0] * T.ntile[1] + c[1]) * T.ntile[2] + c[2];
}

// destination = number of splitters <= key (splitters ascending)
__device__ __forceinline__ int dest_of(uint64_t key, const uint64_t* s_split, int nsplit) {
  int lo = 0, hi = nsplit;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (s_split[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_part_keys(const double* __restrict__ pts, int64_t M, int64_t stride, int64_t row0, TileMap T,
                            uint64_t* __restrict__ keys, int64_t nkeys) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nkeys) return;
  const int64_t i = j * stride;
  bool ok = true;
  const uint64_t t = tile_of(pts, i, T, ok);
  keys[j] = (t << 32) | (uint64_t)(row0 + i);
}

// Pass 1: destination of every point (one byte), the per-(destination, block)
// counts in destination-major order, and the first out-of-domain row.
__global__ void __launch_bounds__(kPartThreads) k_part_count(const double* __restrict__ pts, int64_t M, int64_t row0,
                                                             TileMap T, const uint64_t* __restrict__ split, int nsplit,
                                                             uint8_t* __restrict__ dest, int32_t* __restrict__ counts,
                                                             int nblocks, unsigned long long* __restrict__ bad) {
  __shared__ uint64_t s_split[kPartMax];
  __shared__ int s_cnt[kPartMax];
  for (int i = threadIdx.x; i < nsplit; i += blockDim.x) s_split[i] = split[i];
  for (int i = threadIdx.x; i <= nsplit; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kPartChunk;
  for (int r = 0; r < kPartRounds; ++r) {
    const int64_t i = base + r * kPartThreads + threadIdx.x;
    if (i >= M) break;
    bool ok = true;
    const uint64_t t = tile_of(pts, i, T, ok);
    if (!ok) atomicMin(bad, (unsigned long long)i);
    const int d = dest_of((t << 32) | (uint64_t)(row0 + i), s_split, nsplit);
    dest[i] = (uint8_t)d;
    atomicAdd(&s_cnt[d], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d <= nsplit; d += blockDim.x) counts[(int64_t)d * nblocks + blockIdx.x] = s_cnt[d];
}

// Pass 2: stable scatter.  Block b owns points [b C, (b+1) C) in input order,
// processed in rounds of 256; inside a round the order is warp-major, then
// lane, so ranks come from __match_any_sync within a warp plus per-warp
// per-destination prefix sums in shared memory.
// Destinations of a partition that writes straight into the receiving
// ranks' buffers (IPC-mapped over NVLink): the point at local send
// position p of destination d goes to pts[d] + 3 (base[d] + p), its row
// to rows[d][base[d] + p] (base = my offset in d's buffer - d's local start).
struct PartDst {
  double* pts[kPartMax];
  int32_t* rows[kPartMax];
  int64_t base[kPartMax];
};

template <bool REMOTE>
__global__ void __launch_bounds__(kPartThreads) k_part_scatter(const double* __restrict__ pts, int64_t M,
                                                               const uint8_t* __restrict__ dest,
                                                               const int32_t* __restrict__ offs, int nparts,
                                                               int nblocks, double* __restrict__ send,
                                                               int32_t* __restrict__ pos,
                                                               const PartDst* __restrict__ dst) {
  constexpr int kW = kPartThreads / 32;
  __shared__ int s_run[kPartMax];        // next position per destination
  __shared__ int s_wc[kW][kPartMax];     // this round's count per warp and destination
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int d = threadIdx.x; d < nparts; d += blockDim.x) s_run[d] = offs[(int64_t)d * nblocks + blockIdx.x];
  const int64_t base = (int64_t)blockIdx.x * kPartChunk;
  for (int r = 0; r < kPartRounds; ++r) {
    for (int k = threadIdx.x; k < kW * nparts; k += blockDim.x) s_wc[k / nparts][k % nparts] = 0;
    __syncthreads();
    const int64_t i = base + r * kPartThreads + threadIdx.x;
    const bool live = i < M;
    const int d = live ? dest[i] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (live && rank == 0) s_wc[warp][d] = __popc(peers);
    __syncthreads();
    if (live) {
      int p = s_run[d] + rank;
      for (int w = 0; w < warp; ++w) p += s_wc[w][d];
      const double x0 = pts[3 * i], x1 = pts[3 * i + 1], x2 = pts[3 * i + 2];
      if (REMOTE) {
        const int64_t q = dst->base[d] + p;
        double* o = dst->pts[d] + 3 * q;
        o[0] = x0;
        o[1] = x1;
        o[2] = x2;
        dst->rows[d][q] = (int32_t)i;
      } else {
        pos[i] = p;
        send[3 * (int64_t)p] = x0;
        send[3 * (int64_t)p + 1] = x1;
        send[3 * (int64_t)p + 2] = x2;
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nparts; e += blockDim.x) {
      int t = 0;
      for (int w = 0; w < kW; ++w) t += s_wc[w][e];
      s_run[e] += t;
    }
    __syncthreads();  // s_wc is zeroed by the next round
  }
  if (REMOTE) __threadfence_system();  // peer stores visible before the receivers read
}

__global__ void k_part_totals(const int32_t* __restrict__ offs, int nparts, int nblocks, int64_t* __restrict__ out) {
  const int d = threadIdx.x;
  if (d <= nparts) out[d] = offs[(int64_t)d * nblocks];
}

__global__ void k_gather_values(const double2* __restrict__ vals, const int32_t* __restrict__ pos, int64_t M,
                                double2* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) out[i] = vals[pos[i]];
}

__global__ void k_scatter_to_peers(const double2* __restrict__ vals, int64_t M, const PeerTable* __restrict__ T) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) {
    int o = 0;
    while (o + 1 < T->n && i >= T->off[o + 1]) ++o;
    T->out[o][T->rows[i]] = vals[i];
  }
  __threadfence_system();
}

TileMap tile_map(const vfn_plan* p) {
  TileMap T;
  T.tm = p->map;
  const BinGeom g = make_geometry(p, 2);
  for (int d = 0; d < 3; ++d) {
    T.tile[d] = g.tile[d];
    T.ntile[d] = g.ntile[d];
  }
  return T;
}

}  // namespace

int scatter_to_peers(const double2* values, int64_t M, const PeerTable* table_dev, cudaStream_t s) {
  if (M <= 0) return VFN_OK;
  k_scatter_to_peers<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(values, M, table_dev);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

}  // namespace vfn

using namespace vfn;

extern "C" {

int vfn_plan_part_keys(vfn_plan* p, const double* points, int64_t M, int64_t stride, int64_t row0,
                       uint64_t* keys, void* stream) {
  if (!p || (M > 0 && (!points || !keys)) || stride < 1) return fail(VFN_ERR_INVALID, "bad argument");
  if (M <= 0) return VFN_OK;
  std::lock_guard<std::mutex> plan_lock(p->mu);
  DeviceGuard guard(p->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n = (M + stride - 1) / stride;
  k_part_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(points, M, stride, row0, tile_map(p), keys, n);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

int vfn_plan_partition(vfn_plan* p, const double* points, int64_t M, int64_t row0, const uint64_t* splitters,
                       int nparts, double* send, int32_t* pos, int64_t* counts, int64_t* first_bad_row,
                       void* stream) {
  vfn::NvtxRange nvtx_range("vfn partition by key range");
  if (!p || !counts || (M > 0 && (!points || !send || !pos)) || (nparts > 1 && !splitters))
    return fail(VFN_ERR_INVALID, "null argument");
  if (nparts < 1 || nparts > kPartMax) return fail(VFN_ERR_INVALID, "destination count must be in 1..256");
  if (M < 0 || M > INT32_MAX) return fail(VFN_ERR_INVALID, "point count out of range");
  if (first_bad_row) *first_bad_row = -1;
  for (int d = 0; d < nparts; ++d) counts[d] = 0;
  if (M == 0) return VFN_OK;
  std::lock_guard<std::mutex> plan_lock(p->mu);
  DeviceGuard guard(p->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nb = (int)((M + kPartChunk - 1) / kPartChunk);
  const int64_t ncnt = (int64_t)nparts * nb + 1;
  // scratch: dest bytes, counts, offsets, totals, bad word (plan's grow-only buffers)
  VFN_CHECK(p->keys.ensure(M));  // dest (uint8)
  VFN_CHECK(p->uscratch.ensure(sizeof(int32_t) * 2 * ncnt + sizeof(int64_t) * (nparts + 2)));
  uint8_t* dest = p->keys.as<uint8_t>();
  int32_t* cnt = p->uscratch.as<int32_t>();
  int32_t* off = cnt + ncnt;
  int64_t* tot = reinterpret_cast<int64_t*>(off + ncnt);  // 8-byte aligned: 2 ncnt int32 before it
  int64_t* bad = tot + nparts + 1;
  VFN_CUDA(cudaMemsetAsync(bad, 0x7f, sizeof(int64_t), s));
  VFN_CUDA(cudaMemsetAsync(cnt + ncnt - 1, 0, sizeof(int32_t), s));
  const TileMap T = tile_map(p);
  k_part_count<<<nb, kPartThreads, 0, s>>>(points, M, row0, T, splitters, nparts - 1, dest, cnt, nb,
                                           reinterpret_cast<unsigned long long*>(bad));
  VFN_CUDA(cudaGetLastError());
  size_t tmp = 0;
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, off, (int)ncnt, s));
  VFN_CHECK(p->sort_tmp.ensure(tmp));
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(p->sort_tmp.ptr, tmp, cnt, off, (int)ncnt, s));
  k_part_scatter<false><<<nb, kPartThreads, 0, s>>>(points, M, dest, off, nparts, nb, send, pos, nullptr);
  VFN_CUDA(cudaGetLastError());
  k_part_totals<<<1, 288, 0, s>>>(off, nparts, nb, tot);
  VFN_CUDA(cudaGetLastError());
  std::vector<int64_t> h(nparts + 2);
  VFN_CUDA(cudaMemcpyAsync(h.data(), tot, sizeof(int64_t) * (nparts + 2), cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaStreamSynchronize(s));
  const int64_t b = h[nparts + 1];
  if (b != (int64_t)0x7f7f7f7f7f7f7f7fLL) {
    if (first_bad_row) *first_bad_row = b;
    return fail(VFN_ERR_OUTSIDE, "point (row " + std::to_string(b) + ") lies outside the domain");
  }
  for (int d = 0; d < nparts; ++d) counts[d] = h[d + 1] - h[d];
  return VFN_OK;
}

// Count phase of a partition whose scatter writes to the receiving ranks:
// destinations, per-destination counts (host) and the first bad row; the
// plan keeps the destination bytes and block offsets for
// vfn_plan_partition_scatter_peers with the same points.
int vfn_plan_partition_count(vfn_plan* p, const double* points, int64_t M, int64_t row0, const uint64_t* splitters,
                             int nparts, int64_t* counts, int64_t* first_bad_row, void* stream) {
  vfn::NvtxRange nvtx_range("vfn partition: count");
  if (!p || !counts || (M > 0 && !points) || (nparts > 1 && !splitters)) return fail(VFN_ERR_INVALID, "null argument");
  if (nparts < 1 || nparts > kPartMax) return fail(VFN_ERR_INVALID, "destination count must be in 1..256");
  if (M < 0 || M > INT32_MAX) return fail(VFN_ERR_INVALID, "point count out of range");
  if (first_bad_row) *first_bad_row = -1;
  for (int d = 0; d < nparts; ++d) counts[d] = 0;
  std::lock_guard<std::mutex> plan_lock(p->mu);
  p->part_M = M;
  p->part_n = nparts;
  if (M == 0) return VFN_OK;
  DeviceGuard guard(p->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nb = (int)((M + kPartChunk - 1) / kPartChunk);
  const int64_t ncnt = (int64_t)nparts * nb + 1;
  VFN_CHECK(p->keys.ensure(M));
  VFN_CHECK(p->uscratch.ensure(sizeof(int32_t) * 2 * ncnt + sizeof(int64_t) * (nparts + 2)));
  uint8_t* dest = p->keys.as<uint8_t>();
  int32_t* cnt = p->uscratch.as<int32_t>();
  int32_t* off = cnt + ncnt;
  int64_t* tot = reinterpret_cast<int64_t*>(off + ncnt);
  int64_t* bad = tot + nparts + 1;
  VFN_CUDA(cudaMemsetAsync(bad, 0x7f, sizeof(int64_t), s));
  VFN_CUDA(cudaMemsetAsync(cnt + ncnt - 1, 0, sizeof(int32_t), s));
  k_part_count<<<nb, kPartThreads, 0, s>>>(points, M, row0, tile_map(p), splitters, nparts - 1, dest, cnt, nb,
                                           reinterpret_cast<unsigned long long*>(bad));
  VFN_CUDA(cudaGetLastError());
  size_t tmp = 0;
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, off, (int)ncnt, s));
  VFN_CHECK(p->sort_tmp.ensure(tmp));
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(p->sort_tmp.ptr, tmp, cnt, off, (int)ncnt, s));
  k_part_totals<<<1, 288, 0, s>>>(off, nparts, nb, tot);
  VFN_CUDA(cudaGetLastError());
  std::vector<int64_t> h(nparts + 2);
  VFN_CUDA(cudaMemcpyAsync(h.data(), tot, sizeof(int64_t) * (nparts + 2), cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaStreamSynchronize(s));
  const int64_t b = h[nparts + 1];
  if (b != (int64_t)0x7f7f7f7f7f7f7f7fLL) {
    if (first_bad_row) *first_bad_row = b;
    return fail(VFN_ERR_OUTSIDE, "point (row " + std::to_string(b) + ") lies outside the domain");
  }
  p->part_start.assign(h.begin(), h.begin() + nparts);
  for (int d = 0; d < nparts; ++d) counts[d] = h[d + 1] - h[d];
  return VFN_OK;
}

// Scatter phase: point i of destination d (local send position q inside d)
// goes to recv_pts[d] + 3 (dst_off[d] + q) and its row i to
// recv_rows[d][dst_off[d] + q] — the receiving ranks' IPC-mapped buffers,
// written over NVLink (the all-to-all of the points fused into the split).
int vfn_plan_partition_scatter_peers(vfn_plan* p, const double* points, int64_t M, int nparts,
                                     const int64_t* dst_off, double* const* recv_pts, int32_t* const* recv_rows,
                                     void* stream) {
  vfn::NvtxRange nvtx_range("vfn partition: scatter to peers");
  if (!p || !dst_off || !recv_pts || !recv_rows || (M > 0 && !points)) return fail(VFN_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  if (M != p->part_M || nparts != p->part_n || (int)p->part_start.size() != (M ? nparts : 0))
    return fail(VFN_ERR_INVALID, "partition scatter without a matching count phase");
  if (M == 0) return VFN_OK;
  DeviceGuard guard(p->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nb = (int)((M + kPartChunk - 1) / kPartChunk);
  const int64_t ncnt = (int64_t)nparts * nb + 1;
  PartDst h;
  for (int d = 0; d < nparts; ++d) {
    h.pts[d] = recv_pts[d];
    h.rows[d] = recv_rows[d];
    h.base[d] = dst_off[d] - p->part_start[d];
  }
  VFN_CHECK(p->part_buf.ensure(sizeof(PartDst)));
  VFN_CUDA(cudaMemcpyAsync(p->part_buf.ptr, &h, sizeof(PartDst), cudaMemcpyHostToDevice, s));
  const uint8_t* dest = p->keys.as<uint8_t>();
  const int32_t* off = p->uscratch.as<int32_t>() + ncnt;
  k_part_scatter<true><<<nb, kPartThreads, 0, s>>>(points, M, dest, off, nparts, nb, nullptr, nullptr,
                                                   p->part_buf.as<PartDst>());
  VFN_CUDA(cudaGetLastError());
  VFN_CUDA(cudaStreamSynchronize(s));  // h lives on this stack frame; the receivers read after a barrier
  return VFN_OK;
}

int vfn_gather_values(int device, const double* values, const int32_t* pos, int64_t M, double* out,
                      void* stream) {
  if (M < 0 || (M > 0 && (!values || !pos || !out))) return fail(VFN_ERR_INVALID, "bad argument");
  if (M == 0) return VFN_OK;
  DeviceGuard guard(device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  k_gather_values<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(reinterpret_cast<const double2*>(values), pos, M,
                                                              reinterpret_cast<double2*>(out));
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

// ---- IPC-shared device buffers (the owners' output buffers of a sharded
// evaluate; every rank maps the others' over NVLink)
int vfn_ipc_alloc(int device, int64_t bytes, void** ptr, unsigned char handle[64]) {
  if (!ptr || !handle || bytes <= 0) return fail(VFN_ERR_INVALID, "bad argument");
  DeviceGuard guard(device);
  *ptr = nullptr;
  VFN_CUDA(cudaMalloc(ptr, (size_t)bytes));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, *ptr);
  if (e != cudaSuccess) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return fail(VFN_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle, &h, 64);
  return VFN_OK;
}

int vfn_ipc_open(int device, const unsigned char handle[64], void** ptr) {
  if (!ptr || !handle) return fail(VFN_ERR_INVALID, "bad argument");
  DeviceGuard guard(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  VFN_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return VFN_OK;
}

int vfn_ipc_close(int device, void* ptr) {
  DeviceGuard guard(device);
  VFN_CUDA(cudaIpcCloseMemHandle(ptr));
  return VFN_OK;
}

int vfn_ipc_free(int device, void* ptr) {
  DeviceGuard guard(device);
  VFN_CUDA(cudaFree(ptr));
  return VFN_OK;
}

// dst <- src, device to device on `stream`, synchronised
int vfn_copy_device(int device, void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes <= 0) return VFN_OK;
  DeviceGuard guard(device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  VFN_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, s));
  VFN_CUDA(cudaStreamSynchronize(s));
  return VFN_OK;
}

}  // extern "C"
