// Internal declarations shared by the vfnfft translation units.
#pragma once

#include <cstdint>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>
#include <cstdio>
#include <string>

#include <cuda.h>
#include <cuda_runtime.h>
#include <cufft.h>

#include "../../include/vfnfft.h"

namespace vfn {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define VFN_CUDA(expr)                                                               \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return ::vfn::fail(VFN_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define VFN_CHECK(expr)          \
  do {                           \
    int _s = (expr);             \
    if (_s != VFN_OK) return _s; \
  } while (0)

// Restores the caller's current device on scope exit.
// NVTX range for the duration of a scope (visible in Nsight Systems /
// Compute timelines; header-only NVTX3, a no-op without an attached tool)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Grow-only device buffer; owns its allocation (freed on release() or
// destruction), movable, not copyable.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), bytes(o.bytes) {
    o.ptr = nullptr;
    o.bytes = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      bytes = o.bytes;
      o.ptr = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  int ensure(size_t need) {
    if (need <= bytes) return VFN_OK;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    size_t want = need + need / 8;
    cudaError_t e = cudaMalloc(&ptr, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(VFN_ERR_NOMEM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    }
    bytes = want;
    return VFN_OK;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(ptr); }
};

// ---------------------------------------------------------------- geometry
// Everything a kernel needs to map a point to its nearest oversampled cell,
// bit-exactly as nufft.py:81-92 + :248-257 do it in numpy.
struct TorusMap {
  double a[3];
  double amb[3];  // a - b, the divisor of map_to_torus (nufft.py:92)
  double b[3];
  double nd[3];   // n_d as double
  int n[3];
};

// Box / tile geometry of the binned gather.
struct BinGeom {
  int box[3];     // gather-box size in cells
  int tile[3];    // staging-tile size in cells (multiple of box)
  int ntile[3];   // tiles per axis = ceil(n / tile)
  int nbox[3];    // boxes per tile per axis
  int boxes_per_tile;
  int cells_per_box;  // box[0] * box[1] * box[2]
  // key = (tile * boxes_per_tile + box) * key_slots + depth / 2: inside a box
  // the key keeps only the cell's depth pair (the gather's units are depth
  // runs; x, y inside the box and the low depth bit carry no information for
  // it), which keeps the key short enough for one radix pass fewer (c5: 24
  // bits, 3 passes of 8)
  int key_shift;      // 1: depth pairs; 0: single depths (odd m on the tensor-core gather,
                      // where one spare depth decides the unit's k-chunk count)
  int key_slots;      // (box[2] + 2^key_shift - 1) >> key_shift
  int64_t ntiles;
  int64_t nboxes;  // ntiles * boxes_per_tile
  // ceil(2^32 / d) for d = tile[k], box[k]: floor(x / d) = (x * inv) >> 32
  // exactly for x < 2^21 and d <= 64 (cell indices; see quot())
  uint64_t tile_inv[3], box_inv[3];
};

// Window polynomial table: w_j(delta) = sum_d coef[j*(deg+1) + d] delta^d,
// j = 0..2m (offset c = j - m), approximating phi(delta - c) (nufft.py:159-164).
struct WindowPoly {
  int m = 0;
  int deg = 0;
  double* dev = nullptr;  // (2m+1)*(deg+1) doubles
};

// Outputs of a sharded evaluate that go straight to their owners (the
// ranks whose input blocks the points came from) over NVLink: point i of
// the evaluate belongs to the owner o with off[o] <= i < off[o + 1] and its
// value is stored at out[o][rows[i]] (IPC-mapped peer memory).
constexpr int kMaxPeers = 64;
struct PeerTable {
  int n = 0;
  const int32_t* rows = nullptr;
  int64_t off[kMaxPeers + 1];
  double2* out[kMaxPeers];
};

}  // namespace vfn

struct vfn_plan {
  // Serialises every entry point that touches the plan's scratch or settings:
  // the reference allows one plan to be evaluated from several threads on
  // disjoint point subsets; calls here queue on this lock
  // (each call synchronises its stream before returning).
  mutable std::mutex mu;
  int device = 0;
  int64_t N[3] = {0, 0, 0};
  int64_t n[3] = {0, 0, 0};
  double a[3], b[3];
  double sigma = 2.0;
  int m = 6;
  double beta = 0.0;
  vfn::TorusMap map;
  vfn::WindowPoly poly;
  // ghost-padded grid: P_d = ntile_d * tile_d + 2m, element (i0,i1,i2) holds
  // g[(i0-m) mod n0, (i1-m) mod n1, (i2-m) mod n2]
  int64_t P[3] = {0, 0, 0};
  int pad_tile[3] = {8, 8, 8};  // grid padded to multiples of this
  double2* grid = nullptr;
  size_t grid_bytes = 0;      // its allocation (from the device pool, vfn_util.cu)
  cudaEvent_t bev[4] = {nullptr, nullptr, nullptr, nullptr};  // grid-build phases
  // plan-build breakdown (vfn_plan_build_timing): host total, K2, K3 (FFT),
  // halo, host setup before the grid kernels (allocations, tables)
  float build_ms[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
  int gather_variant = 0;
  int box_mode = 0;          // 0 auto, 1 or 2: gather box width in cells (vfn_plan_set_box)
  double col_density = 16.0;  // points per 1x1x8 cell column in the last call (sampled or mean)
  int64_t col_density_M = 0;  // the point count col_density refers to
  bool col_density_sampled = false;  // col_density saw the points (density sample), not only the grid-wide mean
  CUtensorMap tmap;        // TMA view of `grid` for the tensor-core gather (m = 3..6)
  bool has_tmap = false;
  vfn::DevBuf fftbuf, dfacbuf;  // grid-build scratch (fftbuf kept only if keep_fftbuf)
  bool keep_fftbuf = false;
  // evaluate scratch (grow-only)
  vfn::DevBuf pts, out, uvals, keys, keys_sorted, idx, perm, sort_tmp, box_start, items, units, uscratch, misc;
  vfn::DevBuf warp_bad;  // first-bad-row word of the warp-per-point path (never reallocated)
  vfn::DevBuf sample;    // column-density sample of choose_geometry
  // peer outputs of the current vfn_plan_eval_to_peers call (device table),
  // consumed by the tensor-core gather's epilogue (peer_used) or by a
  // scatter kernel after any other gather
  const vfn::PeerTable* peer_dev = nullptr;
  bool peer_used = false;
  vfn::DevBuf peer_buf;
  // count phase of the last vfn_plan_partition_count (for the scatter phase)
  int64_t part_M = -1;
  int part_n = 0;
  std::vector<int64_t> part_start;  // local send-buffer start of each destination
  vfn::DevBuf part_buf;
  vfn::DevBuf sample_pts;  // the density-sample rows of a host-buffer call
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t* bad_host = nullptr;  // mapped pinned word for the first-bad-row readback
  int64_t* bad_mapped = nullptr;  // its device-side address
  int64_t bad_fallback = 0;
  cudaStream_t copy_stream[2] = {nullptr, nullptr};  // H2D / D2H of the pipelined host path
  mutable float last_gather_ms = 0.f, last_total_ms = 0.f;
  mutable bool timing_pending = false;  // ev[0..3] hold the last call's unread timing
  vfn::BinGeom last_geom;
  bool has_last_geom = false;
  int64_t iota_len = 0;  // idx[0..iota_len) holds 0, 1, 2, ... (the sort's values)
  // CUDA graph of the device part of a small evaluate (vfn_api.cu
  // eval_graphed): captured on the second call with the same key, then
  // replayed on graph_stream while the key repeats
  struct GraphKey {
    const void* pts = nullptr;
    const void* out = nullptr;
    const void* bad = nullptr;
    int64_t M = -1;
    int box[3] = {0, 0, 0}, tile[3] = {0, 0, 0};
    int variant = -1;
    // the plan's scratch buffers the captured launches point into: a call
    // that grew (reallocated) any of them invalidates the graph
    const void* bufs[12] = {};
    bool valid = false;
  };
  GraphKey gkey, gseen;
  bool graphs_on = true;
  bool capturing = false;  // timing events are not recorded inside a graph
  cudaStream_t graph_stream = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaEvent_t graph_ev[2] = {nullptr, nullptr};
};

namespace vfn {

// ---------------------------------------------------------------- pageable host buffers (vfn_stage.cpp)
// Copies between pageable host memory (a fresh numpy array) and the device at
// pinned-memory speed: rings of pinned pieces, host-side copies by several
// threads, transfers on the given stream.  h2d returns once the data are in
// pinned pieces with their H2D enqueued (the caller's later work on `s`
// follows them); d2h returns once the data are in host memory.
struct HostStager;
bool is_pageable(const void* host_ptr);
HostStager* stager_create();
void stager_destroy(HostStager* st);
// process-wide stager of a device for plan-less calls (rectilinear); callers
// serialise on their own per-device locks
HostStager* device_stager(int device);
int stage_h2d(HostStager* st, void* dst_dev, const void* src_host, size_t bytes, cudaStream_t s);
int stage_d2h(HostStager* st, void* dst_host, const void* src_dev, size_t bytes, cudaStream_t s);

// ---------------------------------------------------------------- host math (vfn_host.cpp)
double kb_beta(int m, double sigma);
double bessel_i0(double x);
// phi_hat(k) for k = j - N/2, j = 0..N-1 (nufft.py:167-176)
void kb_hat_table(int64_t N, int64_t n, int m, double beta, double* out);
// fit the window polynomials; returns degree, fills coef ((2m+1)*(deg+1))
int fit_window_poly(int m, double beta, double* coef, int max_deg);

// ---------------------------------------------------------------- device pool (vfn_util.cu)
// Large device buffers (oversampled grids) are recycled per device instead of
// cudaFree'd: cudaFree synchronises the whole device, and a plan rebuilt for
// a new field (a time series of snapshots, one plan per rank) reuses the
// previous grid's memory.  At most four buffers are held per device;
// vfn_pool_release() frees them.
void* pool_alloc(int device, size_t bytes, size_t* got);
// the device's window polynomial table for (m, beta), fitted and uploaded once
int window_table(int device, int m, double beta, WindowPoly* out);
// recycled size-independent plan resources (events, mapped word, small tables)
bool shell_take(vfn_plan* p);
void shell_give(vfn_plan* p);
void pool_free(int device, void* ptr, size_t bytes);

// ---------------------------------------------------------------- complex GEMM (vfn_zgemm.cu)
// C[b][m, n] = sum_k A[b][m, k] B[b][k, n], complex128 on the FP64 tensor
// cores; A[m lda + k]; B[k ldb + n], or B[n ldb + k] with bt; C[m ldc + n];
// batch b offsets the pointers by sA / sB / sC elements.
struct ZGemm {
  int64_t M = 0, N = 0, K = 0;
  const double2* A = nullptr;
  int64_t lda = 0, sA = 0;
  const double2* B = nullptr;
  int64_t ldb = 0, sB = 0;
  bool bt = false;
  double2* C = nullptr;
  int64_t ldc = 0, sC = 0;
  int batch = 1;
};
int zgemm(const ZGemm& g, cudaStream_t s);

// ---------------------------------------------------------------- launchers
// in-place unnormalised forward Z2Z 3D FFT through a cached cuFFT plan
int fft_forward(const int64_t n[3], double2* data, cudaStream_t s);
// in-place unnormalised inverse (e^{+2 pi i k l / n}) 3D Z2Z FFT
int fft_inverse(const int64_t n[3], double2* data, cudaStream_t s);
// in-place forward transform of an n0 x n1 x n2 array embedded in a C-order
// allocation of extents embed[0..2] (the padded grid's interior)
int fft_forward_embedded(const int64_t n[3], const int64_t embed[3], double2* data, cudaStream_t s);
int build_grid(vfn_plan* p, const double* coeffs_dev, cudaStream_t s);
int map_and_key(vfn_plan* p, const double* pts_dev, int64_t M, const BinGeom& g, uint32_t* keys,
                int32_t* iota, double* u, int64_t* bad_dev, cudaStream_t s);
int sort_pairs(vfn_plan* p, const uint32_t* keys_in, uint32_t* keys_out, const int32_t* vals_in,
               int32_t* vals_out, int64_t M, int key_bits, cudaStream_t s);
// hand-written stable LSD radix sort, values = input row (vfn_sort.cu)
int radix_sort_pairs(DevBuf& tmp, const uint32_t* keys_in, uint32_t* keys_out, int32_t* vals_out, int64_t M,
                     int key_bits, cudaStream_t s);
bool use_cub_sort();  // default; VFN_SORT=radix selects radix_sort_pairs (A/B runs)
int launch_torus(const TorusMap& tm, const double* pts, int64_t M, double* zeta, cudaStream_t s);
int gather_simple(vfn_plan* p, const double* pts_dev, int64_t M, const int32_t* perm,
                  double2* out_dev, cudaStream_t s);
// warp-per-point gather of M unbinned points incl. the domain check (first
// bad row atomicMin'd into bad_dev, which must hold the 0x7f.. sentinel)
int gather_warp(vfn_plan* p, const double* pts_dev, int64_t M, double2* out_dev, int64_t* bad_dev,
                cudaStream_t s);
// *dst = *src by one device thread (dst: mapped host memory); reset: then
// *src = the 0x7f.. bad-row sentinel
int store_word(int64_t* src, int64_t* dst, cudaStream_t s, bool reset);
int gather_boxes(vfn_plan* p, const double* pts_dev, int64_t M, const BinGeom& g,
                 const uint32_t* keys_sorted, const int32_t* perm, double2* out_dev,
                 cudaStream_t s, bool* used);
// exact passes (nufft_m == 0) or 1D-NUFFT passes with cutoff nufft_m
int rect_eval(int device, const int64_t nmodes[3], const double a[3], const double b[3],
              const double* coeffs, const double* y[3], const int64_t Mv[3], double* out,
              int on_device, cudaStream_t s, int nufft_m = 0, double sigma = 2.0);
int rect_nufft_device(int device, const int64_t nm[3], const double a[3], const double b[3], double sigma, int m,
                      const double2* C, const double* y[3], const int64_t Mv[3], double2* F, cudaStream_t s);

BinGeom make_geometry(const vfn_plan* p, int bxy);
int choose_geometry(vfn_plan* p, int64_t M, const double* pts_dev, cudaStream_t s, BinGeom* g);
int make_grid_tmap(vfn_plan* p);
bool tc_supported(int m);      // tensor-core gather covers this cutoff
int tc_tile_depth(int m);     // its tile / box depth in cells (20 - 2m)
void tc_tile_xy(int m, int* tx, int* ty);  // its tile x, y extents in cells
int tc_max_box(int m);        // widest box it takes at this cutoff (1 or 2)
bool tc_applicable(const vfn_plan* p, const BinGeom& g);
// values[i] -> table.out[owner(i)][table.rows[i]] (vfn_shard.cu)
int scatter_to_peers(const double2* values, int64_t M, const PeerTable* table_dev, cudaStream_t s);
int launch_tc(vfn_plan* p, const double* u, const int32_t* perm, const uint32_t* keys_sorted,
              const int32_t* box_start, double2* out, const BinGeom& g, int64_t M,
              cudaStream_t s);

// gather-timing event (vfn_plan_last_timing); skipped while capturing a graph
inline void mark_event(vfn_plan* p, int i, cudaStream_t s) {
  if (!p->capturing) cudaEventRecord(p->ev[i], s);
}
// elapsed ms between two plan events, 0 (and the error cleared) if unavailable
inline float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    ms = 0.f;
  }
  return ms;
}

// file-format kernels (vfn_io_kernels.cu)
int launch_density(const double2* v, int64_t n, double* rho, cudaStream_t s);
int launch_vtk_pack(const double* in, const int64_t shape[3], uint32_t* out, cudaStream_t s);

}  // namespace vfn
