// extern "C" entry points of libvfnfft (see include/vfnfft.h).
#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <tuple>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "vfn_device.cuh"

namespace vfn {
const char* last_error_cstr();
int extract_grid(vfn_plan* p, double2* out_dev, cudaStream_t s);
}

using namespace vfn;

namespace {

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// oversampled size rule of nufft.py:179-187
int oversampled(int64_t N, double sigma, int64_t* n) {
  double target = sigma * (double)N;
  double r = std::nearbyint(target);
  int64_t ri = (int64_t)r;
  if (std::fabs(target - r) > 1e-9 || ri % 2 != 0 || ri < N)
    return fail(VFN_ERR_INVALID, "oversampling " + std::to_string(sigma) + " of " +
                                     std::to_string(N) + " modes gives grid size " +
                                     std::to_string(target) +
                                     "; need an even integer no smaller than the mode count");
  *n = ri;
  return VFN_OK;
}

int check_box(const double a[3], const double b[3]) {
  for (int d = 0; d < 3; ++d)
    if (!(std::isfinite(a[d]) && std::isfinite(b[d]) && a[d] < b[d]))
      return fail(VFN_ERR_INVALID, "domain bounds must be finite with a < b");
  return VFN_OK;
}

int stage_in(DevBuf& buf, const void* src, size_t bytes, int on_device, const void** dev,
             cudaStream_t s, HostStager* stager = nullptr) {
  if (on_device) {
    *dev = src;
    return VFN_OK;
  }
  VFN_CHECK(buf.ensure(bytes));
  if (stager)
    VFN_CHECK(stage_h2d(stager, buf.ptr, src, bytes, s));
  else
    VFN_CUDA(cudaMemcpyAsync(buf.ptr, src, bytes, cudaMemcpyHostToDevice, s));
  *dev = buf.ptr;
  return VFN_OK;
}

// The device's pinned stager (shared by its plans; 384 MB of pinned host
// memory per device, not per plan) when `host` is pageable and >= 1 MB.
HostStager* stager_for(vfn_plan* p, const void* host, size_t bytes) {
  if (bytes < ((size_t)1 << 20) || !is_pageable(host)) return nullptr;
  return device_stager(p->device);
}

// The sort's value input is iota (0..M-1); it never changes, so it is kept
// in the plan and K1 only (re)writes it when a call needs more entries.
int32_t* iota_for(vfn_plan* p, int64_t M, bool* write) {
  void* before = p->idx.ptr;
  if (p->idx.ensure(sizeof(int32_t) * M) != VFN_OK) return nullptr;
  if (p->idx.ptr != before) p->iota_len = 0;
  *write = p->iota_len < M;
  if (*write) p->iota_len = M;
  return p->idx.as<int32_t>();
}

// Evaluates of at most this many points take the unbinned warp-per-point
// gather (VFN_WARP_MAX_M in include/vfnfft.h; env VFN_WARP_MAX_M overrides).
int64_t warp_max_m() {
  int64_t v = VFN_WARP_MAX_M;
  if (const char* e = std::getenv("VFN_WARP_MAX_M")) v = std::atoll(e);
  return v;
}

int key_bits_for(int64_t nkeys) {
  int bits = 1;
  while (bits < 32 && ((int64_t)1 << bits) < nkeys) ++bits;
  return bits;
}

}  // namespace

namespace vfn {

// Gather geometry (K4): tiles of 4 x 4 x depth cells; boxes are
// bxy x bxy columns of a tile.  1 x 1 columns waste the fewest rows but need
// dense columns to fill 8-point units; 2 x 2 boxes fill better at low local
// density.  bxy: the plan's setting (vfn_plan_set_box), else — for large
// evaluates — from the local density measured on a sample of the points,
// else from the global density.
BinGeom make_geometry(const vfn_plan* p, int bxy) {
  BinGeom g;
  if (tc_supported(p->m) && p->has_tmap) bxy = std::min(bxy, tc_max_box(p->m));
  const int K = ((2 * p->m + 1) + 3) / 4 * 4;  // DMMA k-extent
  const int bk = K - 2 * p->m;                  // box depth in cells (2 or 4)
  const bool tc = tc_supported(p->m) && p->has_tmap;  // vfn_gather_tc.cu: 4x4xTZ tiles, depth-TZ boxes
  const int tz = tc ? tc_tile_depth(p->m) : bk;
  int tx = 4, ty = 4;
  if (tc) tc_tile_xy(p->m, &tx, &ty);
  g.box[0] = bxy;
  g.box[1] = bxy;
  g.box[2] = tz;
  g.tile[0] = tx;
  g.tile[1] = ty;
  g.tile[2] = tz;
  for (int d = 0; d < 3; ++d) {
    g.ntile[d] = (int)((p->n[d] + g.tile[d] - 1) / g.tile[d]);
    g.nbox[d] = g.tile[d] / g.box[d];
  }
  g.boxes_per_tile = g.nbox[0] * g.nbox[1] * g.nbox[2];
  g.cells_per_box = g.box[0] * g.box[1] * g.box[2];
  // depth pairs unless the tensor-core gather's K window has a single spare
  // depth for a window of W = 2m + 1 taps (odd m: W = 4 KCmin - 1), where
  // a conservative pair span would cost a whole k-chunk
  g.key_shift = (tc && (2 * p->m + 1) % 4 == 3) ? 0 : 1;
  g.key_slots = (g.box[2] + (1 << g.key_shift) - 1) >> g.key_shift;
  for (int d = 0; d < 3; ++d) {
    g.tile_inv[d] = (((uint64_t)1 << 32) + (uint64_t)g.tile[d] - 1) / (uint64_t)g.tile[d];
    g.box_inv[d] = (((uint64_t)1 << 32) + (uint64_t)g.box[d] - 1) / (uint64_t)g.box[d];
  }
  g.ntiles = (int64_t)g.ntile[0] * g.ntile[1] * g.ntile[2];
  g.nboxes = g.ntiles * g.boxes_per_tile;
  return g;
}

constexpr int kDensitySample = 16384;            // sample rows of the density estimate
constexpr int64_t kDensityMinM = (int64_t)1 << 20;  // evaluates from this size sample the density

__global__ void k_sample_columns(const double* __restrict__ pts, int64_t M, int S, TorusMap tm,
                                 uint32_t* __restrict__ cols) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= S) return;
  const int64_t i = (int64_t)j * (M / S);
  int c[3];
  for (int d = 0; d < 3; ++d) {
    double delta;
    c[d] = nearest_cell(pts[3 * i + d], tm.a[d], tm.amb[d], tm.nd[d], tm.n[d], delta);
  }
  cols[j] = (uint32_t)(((int64_t)c[0] * tm.n[1] + c[1]) * ((tm.n[2] + 7) / 8) + c[2] / 8);
}

// Expected number of OTHER points in a random point's 1 x 1 x 8 column,
// estimated from the colliding pairs of the strided sample rows j (M / S),
// j < S, of the M points.  `pts` holds all M points, or (presampled) just the
// S sample rows in order — the multi-GPU path assembles the same S rows from
// every rank's block, so the estimate, and the box width chosen from it, do
// not depend on the number of ranks.
static int local_density(vfn_plan* p, const double* pts, int64_t M, cudaStream_t s, double* rho,
                         bool presampled = false) {
  const int S = kDensitySample;
  DevBuf& buf = p->sample;  // grow-only plan scratch: no cudaMalloc/cudaFree (a device sync) per call
  VFN_CHECK(buf.ensure(sizeof(uint32_t) * 2 * S));
  uint32_t* a = buf.as<uint32_t>();
  uint32_t* b = a + S;
  k_sample_columns<<<(S + 255) / 256, 256, 0, s>>>(pts, presampled ? S : M, S, p->map, a);
  VFN_CUDA(cudaGetLastError());
  size_t tmp = 0;
  VFN_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, a, b, S, 0, 32, s));
  VFN_CHECK(p->sort_tmp.ensure(tmp));
  VFN_CUDA(cub::DeviceRadixSort::SortKeys(p->sort_tmp.ptr, tmp, a, b, S, 0, 32, s));
  std::vector<uint32_t> h(S);
  VFN_CUDA(cudaMemcpyAsync(h.data(), b, sizeof(uint32_t) * S, cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaStreamSynchronize(s));
  double pairs = 0;
  for (int i = 0, j; i < S; i = j) {
    for (j = i + 1; j < S && h[j] == h[i]; ++j) {
    }
    const double L = j - i;
    pairs += L * (L - 1) / 2;
  }
  *rho = 2.0 * pairs * (double)(M - 1) / ((double)S * (S - 1));
  return VFN_OK;
}

// Box width for an evaluate of M points (sample: the points, or their
// presampled density rows; see local_density).
static int choose_bxy(vfn_plan* p, int64_t M, const double* sample, bool presampled, cudaStream_t s, int* out) {
  int bxy = p->box_mode;
  if (bxy == 0) {
    const char* fb = std::getenv("VFN_BOX_XY");  // experiment override
    if (fb) bxy = std::atoi(fb) == 1 ? 1 : 2;
  }
  const double cells = (double)p->n[0] * (double)p->n[1] * (double)p->n[2];
  p->col_density = 8.0 * (double)M / cells;  // mean; the sample below sees clustering
  p->col_density_M = M;
  p->col_density_sampled = false;
  if (sample && tc_supported(p->m) && p->has_tmap && M >= kDensityMinM) {
    // the local density sets the CTA size (12 / 16 warps) even when the box
    // width is pinned: a key range of a sharded set covers a slab of the
    // grid at full density, eight times the whole-grid mean at P = 8
    double rho = 0.0;
    VFN_CHECK(local_density(p, sample, M, s, &rho, presampled));
    p->col_density = std::max(p->col_density, rho);
    p->col_density_sampled = true;
    // 1 x 1 columns once a column's box (TZ cells) holds >= ~32 points
    if (bxy == 0) bxy = rho * tc_tile_depth(p->m) / 8.0 >= 32.0 ? 1 : 2;
  }
  if (bxy == 0) bxy = M >= cells ? 1 : 2;
  *out = bxy;
  return VFN_OK;
}

int choose_geometry(vfn_plan* p, int64_t M, const double* pts_dev, cudaStream_t s, BinGeom* g) {
  int bxy = 2;
  VFN_CHECK(choose_bxy(p, M, pts_dev, false, s, &bxy));
  *g = make_geometry(p, bxy);
  p->last_geom = *g;
  p->has_last_geom = true;
  return VFN_OK;
}

// Window polynomial tables on the device, one per (device, m, beta), kept
// for the process (a few KB each).
int window_table(int device, int m, double beta, WindowPoly* out) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, double>, WindowPoly> tables;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(device, m, beta);
  auto it = tables.find(key);
  if (it == tables.end()) {
    const int max_deg = 26;
    std::vector<double> coef((size_t)(2 * m + 1) * (max_deg + 1));
    WindowPoly w;
    w.m = m;
    w.deg = fit_window_poly(m, beta, coef.data(), max_deg);
    const size_t bytes = sizeof(double) * (2 * m + 1) * (w.deg + 1);
    cudaError_t e = cudaMalloc(&w.dev, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(w.dev, coef.data(), bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (w.dev) cudaFree(w.dev);
      return fail(VFN_ERR_CUDA, std::string("window table: ") + cudaGetErrorString(e));
    }
    it = tables.emplace(key, w).first;
  }
  *out = it->second;
  return VFN_OK;
}

// Recycled plan shells: the size-independent per-plan resources.
namespace {
struct Shell {
  int device;
  cudaEvent_t ev[4], bev[4];
  int64_t* bad_host;
  int64_t* bad_mapped;
  DevBuf warp_bad, dfacbuf;
};
std::mutex g_shell_mu;
std::vector<Shell*> g_shells;
constexpr size_t kShellsKept = 16;
}  // namespace

bool shell_take(vfn_plan* p) {
  Shell* sh = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_shell_mu);
    for (size_t i = 0; i < g_shells.size(); ++i)
      if (g_shells[i]->device == p->device) {
        sh = g_shells[i];
        g_shells.erase(g_shells.begin() + i);
        break;
      }
  }
  if (!sh) return false;
  for (int i = 0; i < 4; ++i) {
    p->ev[i] = sh->ev[i];
    p->bev[i] = sh->bev[i];
  }
  p->bad_host = sh->bad_host;
  p->bad_mapped = sh->bad_mapped;
  p->warp_bad = std::move(sh->warp_bad);  // holds the sentinel (restored after every use)
  p->dfacbuf = std::move(sh->dfacbuf);
  delete sh;
  return true;
}

// Hand a destroyed plan's shell to the recycler; its fields are cleared so
// the caller's destroy leaves them alone.  Only complete shells are kept.
void shell_give(vfn_plan* p) {
  if (!p->bad_host || !p->warp_bad.ptr) return;
  for (int i = 0; i < 4; ++i)
    if (!p->ev[i] || !p->bev[i]) return;
  std::lock_guard<std::mutex> lock(g_shell_mu);
  if (g_shells.size() >= kShellsKept) return;
  Shell* sh = new Shell();
  sh->device = p->device;
  for (int i = 0; i < 4; ++i) {
    sh->ev[i] = p->ev[i];
    sh->bev[i] = p->bev[i];
    p->ev[i] = p->bev[i] = nullptr;
  }
  sh->bad_host = p->bad_host;
  sh->bad_mapped = p->bad_mapped;
  p->bad_host = p->bad_mapped = nullptr;
  sh->warp_bad = std::move(p->warp_bad);
  sh->dfacbuf = std::move(p->dfacbuf);
  g_shells.push_back(sh);
}

}  // namespace vfn

extern "C" {

const char* vfn_version(void) { return "vfnfft 0.1 (sm_100a)"; }

const char* vfn_last_error(void) { return last_error_cstr(); }

int vfn_plan_create(vfn_plan** out, int device, const int64_t nmodes[3], const double a[3],
                    const double b[3], double sigma, int m, const double* coeffs,
                    int coeffs_on_device, void* stream) {
  vfn::NvtxRange nvtx_range("vfn plan build");
  const auto t_start = std::chrono::steady_clock::now();
  if (!out || !nmodes || !a || !b || !coeffs) return fail(VFN_ERR_INVALID, "null argument");
  *out = nullptr;
  if (m < 1 || m > 13) return fail(VFN_ERR_INVALID, "cutoff must be in 1..13");
  if (!(sigma >= 1.0)) return fail(VFN_ERR_INVALID, "oversampling must be >= 1");
  VFN_CHECK(check_box(a, b));
  for (int d = 0; d < 3; ++d)
    if (nmodes[d] <= 0 || nmodes[d] % 2 != 0)
      return fail(VFN_ERR_INVALID, "array dimensions must be even and positive");
  DeviceGuard guard(device);
  cudaStream_t s = as_stream(stream);
  vfn_plan* p = new vfn_plan();
  p->device = device;
  p->sigma = sigma;
  p->m = m;
  for (int d = 0; d < 3; ++d) {
    p->N[d] = nmodes[d];
    p->a[d] = a[d];
    p->b[d] = b[d];
    int st = oversampled(nmodes[d], sigma, &p->n[d]);
    if (st != VFN_OK) {
      delete p;
      return st;
    }
    if (p->n[d] > (1 << 20)) {
      delete p;
      return fail(VFN_ERR_INVALID, "oversampled grid too large");
    }
    p->map.a[d] = a[d];
    p->map.b[d] = b[d];
    p->map.amb[d] = a[d] - b[d];
    p->map.nd[d] = (double)p->n[d];
    p->map.n[d] = (int)p->n[d];
    const int64_t pt = p->pad_tile[d];
    p->P[d] = (p->n[d] + pt - 1) / pt * pt + 2 * m;
  }
  p->beta = kb_beta(m, sigma);
  // window polynomial table: fitted once per (m, beta) and uploaded once per
  // device (process-wide, shared by plans)
  {
    const int st = window_table(device, m, p->beta, &p->poly);
    if (st != VFN_OK) {
      std::string msg = vfn_last_error();
      vfn_plan_destroy(p);
      return fail(st, msg);
    }
  }
  // events, the mapped bad-row word and the small tables come from a
  // recycled shell of a destroyed plan when one is available (creating them
  // costs ~1-2 ms of driver calls, more than a small plan's kernels)
  if (!shell_take(p)) {
    for (int i = 0; i < 4; ++i) cudaEventCreate(&p->ev[i]);
    for (int i = 0; i < 4; ++i) cudaEventCreate(&p->bev[i]);
    if (cudaHostAlloc(&p->bad_host, sizeof(int64_t), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&p->bad_mapped, p->bad_host, 0) != cudaSuccess) {
      cudaGetLastError();
      if (p->bad_host) cudaFreeHost(p->bad_host);
      p->bad_host = nullptr;  // pageable fallback (p->bad_fallback)
      p->bad_mapped = nullptr;
    }
    // bad-row word of the warp path, kept at the 0x7f.. sentinel between calls
    if (p->warp_bad.ensure(sizeof(int64_t)) != VFN_OK ||
        cudaMemset(p->warp_bad.ptr, 0x7f, sizeof(int64_t)) != cudaSuccess) {
      std::string msg = vfn_last_error();
      vfn_plan_destroy(p);
      return fail(VFN_ERR_CUDA, "plan scratch: " + msg);
    }
  }
  // bin keys are uint32: (tile * boxes_per_tile + box) * key_slots + depth / 2
  // must stay below 2^32 for every geometry the plan can use (n1 n2 n3 ~>
  // 4.2e9 cells); checked before the grid is allocated
  for (int tm = 0; tm < 2; ++tm)
    for (int bxy = 1; bxy <= 2; ++bxy) {
      p->has_tmap = tm == 1;
      const BinGeom g = make_geometry(p, bxy);
      p->has_tmap = false;
      if ((double)g.nboxes * (double)g.key_slots > 4294967296.0) {
        const std::string msg = "oversampled grid too large: its bin keys exceed 32 bits (" +
                                std::to_string(p->n[0]) + " x " + std::to_string(p->n[1]) + " x " +
                                std::to_string(p->n[2]) + " cells)";
        vfn_plan_destroy(p);
        return fail(VFN_ERR_INVALID, msg);
      }
    }
  // coefficients to the device
  const size_t cbytes = sizeof(double2) * nmodes[0] * nmodes[1] * nmodes[2];
  // host coefficients go through a pooled device buffer (no cudaMalloc /
  // cudaFree per plan; build_grid synchronises before it is returned)
  const void* cdev = coeffs;
  void* staging = nullptr;
  size_t staging_bytes = 0;
  int st = VFN_OK;
  if (!coeffs_on_device) {
    staging = pool_alloc(device, cbytes, &staging_bytes);
    if (!staging) st = fail(VFN_ERR_NOMEM, "coefficient staging allocation failed");
    else if (cbytes >= ((size_t)1 << 20) && is_pageable(coeffs))
      st = stage_h2d(device_stager(device), staging, coeffs, cbytes, s);
    else if (cudaMemcpyAsync(staging, coeffs, cbytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
      st = fail(VFN_ERR_CUDA, "coefficient upload failed");
    cdev = staging;
  }
  const auto t_setup = std::chrono::steady_clock::now();
  if (st == VFN_OK) st = build_grid(p, static_cast<const double*>(cdev), s);
  if (st == VFN_OK) st = make_grid_tmap(p);
  if (staging) {
    if (st != VFN_OK) cudaStreamSynchronize(s);
    pool_free(device, staging, staging_bytes);
  }
  p->build_ms[4] = std::chrono::duration<float, std::milli>(t_setup - t_start).count();
  p->build_ms[0] = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  if (st != VFN_OK) {
    std::string msg = vfn_last_error();
    vfn_plan_destroy(p);
    return fail(st, msg);
  }
  *out = p;
  return VFN_OK;
}

int vfn_plan_destroy(vfn_plan* p) {
  if (!p) return VFN_OK;
  DeviceGuard guard(p->device);
  if (p->grid) pool_free(p->device, p->grid, p->grid_bytes);
  p->poly.dev = nullptr;  // the device's shared window table
  shell_give(p);          // events, mapped word, small tables back to the recycler (if it has room)
  for (int i = 0; i < 4; ++i)
    if (p->bev[i]) cudaEventDestroy(p->bev[i]);
  DevBuf* bufs[] = {&p->pts, &p->out, &p->keys, &p->keys_sorted, &p->idx, &p->perm,
                    &p->sort_tmp, &p->box_start, &p->items, &p->units, &p->uscratch, &p->misc};
  for (DevBuf* b : bufs) b->release();
  for (int i = 0; i < 4; ++i)
    if (p->ev[i]) cudaEventDestroy(p->ev[i]);
  for (int i = 0; i < 2; ++i)
    if (p->copy_stream[i]) cudaStreamDestroy(p->copy_stream[i]);
  if (p->graph_exec) cudaGraphExecDestroy(p->graph_exec);
  for (int i = 0; i < 2; ++i)
    if (p->graph_ev[i]) cudaEventDestroy(p->graph_ev[i]);
  if (p->graph_stream) cudaStreamDestroy(p->graph_stream);
  if (p->bad_host) cudaFreeHost(p->bad_host);
  delete p;
  return VFN_OK;
}

int vfn_plan_build_timing(const vfn_plan* p, float ms_out[5]) {
  if (!p || !ms_out) return fail(VFN_ERR_INVALID, "null argument");
  for (int i = 0; i < 5; ++i) ms_out[i] = p->build_ms[i];
  return VFN_OK;
}

int vfn_plan_info(const vfn_plan* p, int64_t n_out[3], double* beta_out) {
  if (!p) return fail(VFN_ERR_INVALID, "null plan");
  if (n_out)
    for (int d = 0; d < 3; ++d) n_out[d] = p->n[d];
  if (beta_out) *beta_out = p->beta;
  return VFN_OK;
}

int vfn_plan_geometry(const vfn_plan* p, int64_t M, int box_out[3], int tile_out[3]) {
  if (!p || !box_out || !tile_out) return fail(VFN_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  // the geometry of the last evaluate/bin call, else the point-free rule for M
  const double cells = (double)p->n[0] * (double)p->n[1] * (double)p->n[2];
  BinGeom g = p->has_last_geom ? p->last_geom
                               : make_geometry(p, p->box_mode ? p->box_mode : (M >= cells ? 1 : 2));
  for (int d = 0; d < 3; ++d) {
    box_out[d] = g.box[d];
    tile_out[d] = g.tile[d];
  }
  return VFN_OK;
}

int vfn_plan_decide(vfn_plan* p, int64_t M, const double* sample, int nsample, int* variant_out,
                    int* box_out, void* stream) {
  if (!p || !variant_out || !box_out) return fail(VFN_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  DeviceGuard guard(p->device);
  const double cells = (double)p->n[0] * (double)p->n[1] * (double)p->n[2];
  const bool wants_sample = p->box_mode == 0 && !std::getenv("VFN_BOX_XY") && tc_supported(p->m) &&
                            p->has_tmap && M >= kDensityMinM;
  if (wants_sample && (!sample || nsample != kDensitySample))
    return fail(VFN_ERR_INVALID, "decide: " + std::to_string(M) + " points need the " +
                                     std::to_string(kDensitySample) + "-row density sample");
  int v = p->gather_variant;
  if (v == 0) v = M <= warp_max_m() ? 3 : 4;
  int bxy = 2;
  VFN_CHECK(choose_bxy(p, M, wants_sample ? sample : nullptr, true, reinterpret_cast<cudaStream_t>(stream), &bxy));
  (void)cells;
  *variant_out = v;
  *box_out = bxy;
  return VFN_OK;
}

int vfn_plan_key_shift(const vfn_plan* p, int64_t M, int* shift_out) {
  if (!p || !shift_out) return fail(VFN_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  const double cells = (double)p->n[0] * (double)p->n[1] * (double)p->n[2];
  const BinGeom g = p->has_last_geom ? p->last_geom
                                     : make_geometry(p, p->box_mode ? p->box_mode : (M >= cells ? 1 : 2));
  *shift_out = g.key_shift;
  return VFN_OK;
}

int vfn_plan_set_box(vfn_plan* p, int bxy) {
  if (!p || bxy < 0 || bxy > 2) return fail(VFN_ERR_INVALID, "box must be 0 (auto), 1 or 2");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  p->box_mode = bxy;
  return VFN_OK;
}

int vfn_plan_set_graphs(vfn_plan* p, int enable) {
  if (!p) return fail(VFN_ERR_INVALID, "null plan");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  p->graphs_on = enable != 0;
  p->gseen.valid = false;
  return VFN_OK;
}

int vfn_plan_set_gather(vfn_plan* p, int variant) {
  if (!p || variant < 0 || variant > 4) return fail(VFN_ERR_INVALID, "bad gather variant");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  p->gather_variant = variant;
  return VFN_OK;
}

int vfn_plan_last_timing(const vfn_plan* p, float* gather_ms, float* total_ms) {
  if (!p) return fail(VFN_ERR_INVALID, "null plan");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  if (p->timing_pending) {  // events of the last call, complete since it synchronised
    p->last_gather_ms = elapsed_ms(p->ev[1], p->ev[2]);
    p->last_total_ms = elapsed_ms(p->ev[0], p->ev[3]);
    p->timing_pending = false;
  }
  if (gather_ms) *gather_ms = p->last_gather_ms;
  if (total_ms) *total_ms = p->last_total_ms;
  return VFN_OK;
}

int vfn_plan_grid(vfn_plan* p, double* out_host) {
  if (!p || !out_host) return fail(VFN_ERR_INVALID, "null argument");
  DeviceGuard guard(p->device);
  const size_t bytes = sizeof(double2) * p->n[0] * p->n[1] * p->n[2];
  DevBuf tmp;
  VFN_CHECK(tmp.ensure(bytes));
  int st = extract_grid(p, tmp.as<double2>(), 0);
  if (st == VFN_OK) {
    cudaError_t e = cudaMemcpy(out_host, tmp.ptr, bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = fail(VFN_ERR_CUDA, std::string("grid copy: ") + cudaGetErrorString(e));
  }
  tmp.release();
  return st;
}

int vfn_map_to_torus(int device, const double a[3], const double b[3], const double* points,
                     int64_t M, double* zeta, int on_device, void* stream) {
  if (!a || !b || (M > 0 && (!points || !zeta))) return fail(VFN_ERR_INVALID, "null argument");
  if (M < 0) return fail(VFN_ERR_INVALID, "negative point count");
  VFN_CHECK(check_box(a, b));
  if (M == 0) return VFN_OK;
  DeviceGuard guard(device);
  cudaStream_t s = as_stream(stream);
  TorusMap tm;
  for (int d = 0; d < 3; ++d) {
    tm.a[d] = a[d];
    tm.b[d] = b[d];
    tm.amb[d] = a[d] - b[d];
    tm.nd[d] = 1.0;
    tm.n[d] = 1;
  }
  DevBuf in, outb;
  const size_t bytes = sizeof(double) * 3 * M;
  const void* pdev = nullptr;
  VFN_CHECK(stage_in(in, points, bytes, on_device, &pdev, s));
  double* zdev = zeta;
  if (!on_device) {
    VFN_CHECK(outb.ensure(bytes));
    zdev = outb.as<double>();
  }
  VFN_CHECK(launch_torus(tm, static_cast<const double*>(pdev), M, zdev, s));
  if (!on_device) VFN_CUDA(cudaMemcpyAsync(zeta, zdev, bytes, cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaStreamSynchronize(s));
  in.release();
  outb.release();
  return VFN_OK;
}

// Shared front half of evaluate / bin: stage points, map+validate+key, sort.
static int bin_points(vfn_plan* p, const double* points, int64_t M, int on_device,
                      BinGeom* gout, const double** pts_dev, int64_t** bad_dev,
                      cudaStream_t s) {
  const void* pdev = nullptr;
  VFN_CHECK(stage_in(p->pts, points, sizeof(double) * 3 * M, on_device, &pdev, s));
  *pts_dev = static_cast<const double*>(pdev);
  VFN_CHECK(choose_geometry(p, M, *pts_dev, s, gout));
  const BinGeom& g = *gout;
  const bool want_u = p->gather_variant != 1 && tc_applicable(p, g);
  VFN_CHECK(p->misc.ensure(64));
  *bad_dev = p->misc.as<int64_t>();
  const int64_t sentinel = INT64_MAX;
  VFN_CUDA(cudaMemcpyAsync(*bad_dev, &sentinel, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  VFN_CHECK(p->keys.ensure(sizeof(uint32_t) * M));
  VFN_CHECK(p->keys_sorted.ensure(sizeof(uint32_t) * M));
  VFN_CHECK(p->perm.ensure(sizeof(int32_t) * M));
  bool write_iota = false;
  int32_t* iota = iota_for(p, M, &write_iota);
  if (!iota) return fail(VFN_ERR_NOMEM, "iota allocation failed");
  double* u = nullptr;
  if (want_u) {
    VFN_CHECK(p->uvals.ensure(sizeof(double) * 3 * M));
    u = p->uvals.as<double>();
  }
  VFN_CHECK(map_and_key(p, *pts_dev, M, g, p->keys.as<uint32_t>(), write_iota && use_cub_sort() ? iota : nullptr, u,
                        *bad_dev, s));
  VFN_CHECK(sort_pairs(p, p->keys.as<uint32_t>(), p->keys_sorted.as<uint32_t>(),
                       p->idx.as<int32_t>(), p->perm.as<int32_t>(), M, key_bits_for(g.nboxes * g.key_slots), s));
  return VFN_OK;
}

int vfn_plan_bin(vfn_plan* p, const double* points, int64_t M, uint32_t* keys, int32_t* perm,
                 int on_device, int64_t* first_bad_row, void* stream) {
  vfn::NvtxRange nvtx_range("vfn bin");
  if (!p || (M > 0 && (!points || !keys || !perm))) return fail(VFN_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  if (M < 0 || M > INT32_MAX) return fail(VFN_ERR_INVALID, "point count out of range");
  if (first_bad_row) *first_bad_row = -1;
  if (M == 0) return VFN_OK;
  DeviceGuard guard(p->device);
  cudaStream_t s = as_stream(stream);
  BinGeom g;
  const double* pts_dev;
  int64_t* bad_dev;
  VFN_CHECK(bin_points(p, points, M, on_device, &g, &pts_dev, &bad_dev, s));
  cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  VFN_CUDA(cudaMemcpyAsync(keys, p->keys.ptr, sizeof(uint32_t) * M, k, s));
  VFN_CUDA(cudaMemcpyAsync(perm, p->perm.ptr, sizeof(int32_t) * M, k, s));
  int64_t bad = INT64_MAX;
  VFN_CUDA(cudaMemcpyAsync(&bad, bad_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaStreamSynchronize(s));
  if (bad != INT64_MAX) {
    if (first_bad_row) *first_bad_row = bad;
    return fail(VFN_ERR_OUTSIDE, "point (row " + std::to_string(bad) + ") lies outside the domain");
  }
  return VFN_OK;
}

}  // extern "C"

namespace {

constexpr unsigned char kBadByte = 0x7f;  // memset sentinel: 0x7f7f... > any row
constexpr int64_t kBadSentinel = 0x7f7f7f7f7f7f7f7fLL;

// Enqueue one evaluation of M device-resident points on stream s (no host
// synchronisation unless the geometry has to be sampled): map + key + sort,
// then the gather.  bad_dev receives the first out-of-domain row (relative).
int eval_enqueue(vfn_plan* p, const double* pts_dev, int64_t M, double2* out_dev, int64_t* bad_dev,
                 cudaStream_t s, const BinGeom* fixed) {
  vfn::NvtxRange nvtx_range("vfn evaluate batch (bin + gather)");
  BinGeom g;
  if (fixed) {
    g = *fixed;
    p->last_geom = g;
    p->has_last_geom = true;
    // later chunks / batches of one call: same point distribution, so the
    // column density (CTA size choice only; values do not depend on it)
    // scales with the chunk's point count
    if (p->col_density_M > 0) {
      p->col_density *= (double)M / (double)p->col_density_M;
      p->col_density_M = M;
    }
  } else {
    VFN_CHECK(choose_geometry(p, M, pts_dev, s, &g));
  }
  const bool want_u = p->gather_variant != 1 && tc_applicable(p, g);
  VFN_CUDA(cudaMemsetAsync(bad_dev, kBadByte, sizeof(int64_t), s));
  VFN_CHECK(p->keys.ensure(sizeof(uint32_t) * M));
  VFN_CHECK(p->keys_sorted.ensure(sizeof(uint32_t) * M));
  VFN_CHECK(p->perm.ensure(sizeof(int32_t) * M));
  bool write_iota = false;
  int32_t* iota = iota_for(p, M, &write_iota);
  if (!iota) return fail(VFN_ERR_NOMEM, "iota allocation failed");
  double* u = nullptr;
  if (want_u) {
    VFN_CHECK(p->uvals.ensure(sizeof(double) * 3 * M));
    u = p->uvals.as<double>();
  }
  VFN_CHECK(map_and_key(p, pts_dev, M, g, p->keys.as<uint32_t>(), write_iota && use_cub_sort() ? iota : nullptr, u,
                        bad_dev, s));
  VFN_CHECK(sort_pairs(p, p->keys.as<uint32_t>(), p->keys_sorted.as<uint32_t>(), p->idx.as<int32_t>(),
                       p->perm.as<int32_t>(), M, key_bits_for(g.nboxes * g.key_slots), s));
  mark_event(p, 1, s);
  bool used = false;
  if (p->gather_variant != 1)
    VFN_CHECK(gather_boxes(p, pts_dev, M, g, p->keys_sorted.as<uint32_t>(), p->perm.as<int32_t>(),
                           out_dev, s, &used));
  if (!used) {
    if (p->gather_variant == 2) return fail(VFN_ERR_INVALID, "box gather unavailable for this plan");
    VFN_CHECK(gather_simple(p, pts_dev, M, p->perm.as<int32_t>(), out_dev, s));
  }
  mark_event(p, 2, s);
  return VFN_OK;
}

// A device buffer handed to a plan must live on the plan's GPU: a pointer
// into another device's memory would be written by this device's kernels
// (a peer write or an illegal-address fault that poisons the context).
int check_on_device(const void* ptr, int device, const char* what) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return VFN_OK;  // unknown to the runtime: let the kernels report it
  }
  if ((at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) && at.device != device)
    return fail(VFN_ERR_INVALID, std::string(what) + " is on cuda:" + std::to_string(at.device) +
                                     ", the plan on cuda:" + std::to_string(device));
  return VFN_OK;
}

int outside(int64_t bad, int64_t* first_bad_row) {
  if (first_bad_row) *first_bad_row = bad;
  return fail(VFN_ERR_OUTSIDE, "point (row " + std::to_string(bad) + ") lies outside the domain");
}

// Host buffers, large M: chunks of points flow H2D (copy stream) -> evaluate
// (caller's stream) -> D2H (second copy stream), double-buffered, so the PCIe
// transfers of neighbouring chunks overlap the computation (pinned memory
// makes the copies asynchronous).
// One sort + gather handles at most max_batch() points (32-bit sort values
// and unit offsets); larger calls run as consecutive batches with the first
// batch's bin geometry, so every point's value is the one a single call
// would give it (HBM holds ~3e9 points with their scratch on a B200).

// Host-buffer evaluates of at least this many points run pipelined
// (chunked H2D / evaluate / D2H); env VFN_PIPE_MIN overrides.
int64_t pipe_min_m() {
  int64_t v = (int64_t)1 << 23;
  if (const char* e = std::getenv("VFN_PIPE_MIN")) v = std::max<int64_t>(2, std::atoll(e));
  return v;
}

int64_t max_batch() {
  int64_t b = (int64_t)1 << 30;
  if (const char* e = std::getenv("VFN_MAX_BATCH")) b = std::max<int64_t>(1 << 10, std::atoll(e));
  return b;
}

int eval_device_batches(vfn_plan* p, const double* points, int64_t M, double* out, int on_device,
                        int64_t* first_bad_row, cudaStream_t s) {
  const int64_t bsz = max_batch(), nb = (M + bsz - 1) / bsz;
  VFN_CUDA(cudaEventRecord(p->ev[0], s));
  const void* pdev = nullptr;
  VFN_CHECK(stage_in(p->pts, points, sizeof(double) * 3 * M, on_device, &pdev, s));
  double2* out_dev = reinterpret_cast<double2*>(out);
  if (!on_device) {
    VFN_CHECK(p->out.ensure(sizeof(double2) * M));
    out_dev = p->out.as<double2>();
  }
  VFN_CHECK(p->misc.ensure(sizeof(int64_t) * (nb + 8)));
  int64_t* bad_dev = p->misc.as<int64_t>();
  // one geometry for every batch, chosen from the whole call's points
  BinGeom g;
  VFN_CHECK(choose_geometry(p, M, static_cast<const double*>(pdev), s, &g));
  for (int64_t i = 0; i < nb; ++i) {
    const int64_t lo = i * bsz, n = std::min(bsz, M - lo);
    VFN_CHECK(eval_enqueue(p, static_cast<const double*>(pdev) + 3 * lo, n, out_dev + lo, bad_dev + i, s, &g));
  }
  if (!on_device)
    VFN_CUDA(cudaMemcpyAsync(out, out_dev, sizeof(double2) * M, cudaMemcpyDeviceToHost, s));
  std::vector<int64_t> bad(nb, kBadSentinel);
  VFN_CUDA(cudaMemcpyAsync(bad.data(), bad_dev, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaEventRecord(p->ev[3], s));
  VFN_CUDA(cudaStreamSynchronize(s));
  p->timing_pending = true;  // elapsed times are read lazily (vfn_plan_last_timing)
  for (int64_t i = 0; i < nb; ++i)
    if (bad[i] != kBadSentinel) return outside(i * bsz + bad[i], first_bad_row);
  return VFN_OK;
}

// Small evaluates are launch-bound (~25 kernels + scans for 1e4 points), so
// their device part runs as one CUDA graph.  A call's key is everything the
// enqueued work depends on (buffers, M, bin geometry, gather variant); the
// first call with a new key runs eagerly (and sizes every buffer), the second
// captures eval_enqueue on the plan's own stream, later ones replay it.
// Values are bitwise those of the eager path (same kernels, same order).
constexpr int64_t kGraphMaxM = ((int64_t)1 << 20) - 1;  // below the density-sampling size (2^20)

bool same_key(const vfn_plan::GraphKey& a, const vfn_plan::GraphKey& b) {
  if (!a.valid || !b.valid) return false;
  for (int d = 0; d < 3; ++d)
    if (a.box[d] != b.box[d] || a.tile[d] != b.tile[d]) return false;
  for (int i = 0; i < 12; ++i)
    if (a.bufs[i] != b.bufs[i]) return false;
  return a.pts == b.pts && a.out == b.out && a.bad == b.bad && a.M == b.M && a.variant == b.variant;
}

int eval_graphed(vfn_plan* p, const double* pts_dev, int64_t M, double2* out_dev, int64_t* bad_dev,
                 cudaStream_t s, bool* done) {
  *done = false;
  if (!p->graphs_on || M > kGraphMaxM) return VFN_OK;
  BinGeom g;
  VFN_CHECK(choose_geometry(p, M, nullptr, s, &g));  // M < 2^20: no sampling, no sync
  vfn_plan::GraphKey k;
  k.pts = pts_dev;
  k.out = out_dev;
  k.bad = bad_dev;
  k.M = M;
  for (int d = 0; d < 3; ++d) {
    k.box[d] = g.box[d];
    k.tile[d] = g.tile[d];
  }
  k.variant = p->gather_variant;
  const void* bufs[12] = {p->keys.ptr,  p->keys_sorted.ptr, p->idx.ptr,   p->perm.ptr,
                          p->sort_tmp.ptr, p->box_start.ptr, p->items.ptr, p->units.ptr,
                          p->uscratch.ptr, p->uvals.ptr, p->misc.ptr, p->pts.ptr};
  for (int i = 0; i < 12; ++i) k.bufs[i] = bufs[i];
  k.valid = true;
  if (!same_key(k, p->gkey)) {
    if (!same_key(k, p->gseen)) {
      p->gseen = k;  // first sighting: eager
      return VFN_OK;
    }
    if (!p->graph_stream) {
      VFN_CUDA(cudaStreamCreateWithFlags(&p->graph_stream, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) VFN_CUDA(cudaEventCreateWithFlags(&p->graph_ev[i], cudaEventDisableTiming));
    }
    if (p->graph_exec) {
      cudaGraphExecDestroy(p->graph_exec);
      p->graph_exec = nullptr;
      p->gkey.valid = false;
    }
    VFN_CUDA(cudaStreamBeginCapture(p->graph_stream, cudaStreamCaptureModeThreadLocal));
    p->capturing = true;
    const int st = eval_enqueue(p, pts_dev, M, out_dev, bad_dev, p->graph_stream, &g);
    p->capturing = false;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(p->graph_stream, &graph);
    if (st == VFN_OK && e == cudaSuccess) e = cudaGraphInstantiate(&p->graph_exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (st != VFN_OK || e != cudaSuccess) {
      // not capturable here: evaluate eagerly from now on (same kernels)
      if (std::getenv("VFN_DEBUG_GRAPH"))
        fprintf(stderr, "graph capture failed: st=%d (%s) end=%s\n", st, last_error_cstr(), cudaGetErrorString(e));
      cudaGetLastError();
      p->graph_exec = nullptr;
      p->graphs_on = false;
      return VFN_OK;
    }
    p->gkey = k;
  }
  // replay after the caller's earlier work on s; s continues after the graph
  VFN_CUDA(cudaEventRecord(p->graph_ev[0], s));
  VFN_CUDA(cudaStreamWaitEvent(p->graph_stream, p->graph_ev[0], 0));
  VFN_CUDA(cudaEventRecord(p->ev[1], p->graph_stream));  // last_timing: the whole graph
  VFN_CUDA(cudaGraphLaunch(p->graph_exec, p->graph_stream));
  VFN_CUDA(cudaEventRecord(p->ev[2], p->graph_stream));
  VFN_CUDA(cudaEventRecord(p->graph_ev[1], p->graph_stream));
  VFN_CUDA(cudaStreamWaitEvent(s, p->graph_ev[1], 0));
  *done = true;
  return VFN_OK;
}

// Expected number of other points in a random point's 1 x 1 x 8 cell column,
// from the colliding pairs of a strided sample of host points (cells from
// the plain scaled coordinate: a density estimate, not the bit-exact map).
double host_column_density(const vfn_plan* p, const double* pts, int64_t M) {
  const int S = (int)std::min<int64_t>(M, 2048);  // strided host reads: keep it cheap (~0.1 ms)
  if (S < 2) return 0.0;
  std::vector<uint64_t> ids(S);
  const int64_t nz = (p->n[2] + 7) / 8;
  for (int j = 0; j < S; ++j) {
    const double* x = pts + 3 * ((int64_t)j * (M / S));
    int64_t c[3];
    for (int d = 0; d < 3; ++d) {
      double t = (x[d] - p->a[d]) / (p->b[d] - p->a[d]);
      if (!(t >= 0.0 && t < 1.0)) t = 0.0;
      c[d] = std::min<int64_t>(p->n[d] - 1, (int64_t)(t * (double)p->n[d]));
    }
    ids[j] = (uint64_t)((c[0] * p->n[1] + c[1]) * nz + c[2] / 8);
  }
  std::sort(ids.begin(), ids.end());
  double pairs = 0;
  for (int i = 0, j; i < S; i = j) {
    for (j = i + 1; j < S && ids[j] == ids[i]; ++j) {
    }
    const double L = j - i;
    pairs += L * (L - 1) / 2;
  }
  return 2.0 * pairs * (double)(M - 1) / ((double)S * (S - 1));
}

// Chunk split of a pipelined host-buffer evaluate (cutoffs <= 6) from a
// timeline model: chunk i's H2D, its evaluate and its D2H run on three
// queues (copies at ~55 GB/s each way), and an evaluate of Mc points costs
// B g(Mc / B) with B the boxes that hold points and g the measured cost per
// box of the tensor-core gather + binning as a function of the points per
// box (c5 chunks on B200 at m = 6, `profiles/r02/chunk_cost_c5.json`; other
// cutoffs scaled by their dense gather time).  The per-pass part of g (every
// occupied box costs a unit, every tile a load) is what makes many chunks
// lose on sparse sets: 2^23 uniform points on a 512^3 grid take 27 ms in one
// chunk and 39 ms in two.  The candidates are the splits measured to win
// somewhere: one chunk, two, three, the four-chunk splits of c5 / c3, and
// the five- and six-chunk splits of the transfer-bound narrow stencils.
std::vector<double> model_split(const vfn_plan* p, const double* points, int64_t M) {
  static const double kX[] = {0.0, 1.9, 2.56, 3.84, 6.4, 10.2, 14.0, 20.5, 25.6, 32.0, 64.0};
  static const double kG[] = {1.3, 5.0, 5.30, 5.77, 6.85, 8.30, 9.69, 12.4, 14.6, 17.6, 33.2};  // ns per box
  static const double kDense[7] = {0, 0, 52.7, 42.3, 69.5, 79.8, 127.8};  // ms per 2^28 points, by cutoff
  const int m = std::min(std::max(p->m, 2), 6);
  auto g = [&](double x) {
    const int n = (int)(sizeof(kX) / sizeof(kX[0]));
    if (x >= kX[n - 1]) return kG[n - 1] * x / kX[n - 1];  // dense: linear in the points
    int i = 1;
    while (kX[i] < x) ++i;
    const double t = (x - kX[i - 1]) / (kX[i] - kX[i - 1]);
    return kG[i - 1] + t * (kG[i] - kG[i - 1]);
  };
  const double cells = (double)p->n[0] * (double)p->n[1] * (double)p->n[2];
  const double tz = (double)tc_tile_depth(p->m);
  // local density from colliding pairs of 2048 sampled rows; one pair is worth
  // 2 (M - 1) / (S (S - 1)) points per column, so fewer than 8 pairs say
  // nothing beyond the mean (a uniform set sees 0 or 1 by chance)
  double rho_local = host_column_density(p, points, M);
  {
    const double S = (double)std::min<int64_t>(M, 2048);
    if (rho_local < 8.0 * 2.0 * (double)(M - 1) / (S * (S - 1))) rho_local = 0.0;
  }
  const double rho = std::max(8.0 * (double)M / cells, rho_local);  // points per 8-cell column
  const double box_cols = 4.0 * tz / 8.0;                                                      // columns per 2 x 2 x TZ box
  const double b_occ = std::min(cells / (4.0 * tz), (double)M / std::max(rho * box_cols, 1e-9));  // boxes in the occupied region
  const double scale = kDense[m] / kDense[6] * 1e-6;  // ns -> ms, by cutoff
  auto eval_ms = [&](double mc) { return b_occ * g(mc / b_occ) * scale; };
  const double h2d = 24.0 / 55e6, d2h = 16.0 / 55e6;  // ms per point
  static const std::vector<std::vector<double>> cand = {
      {1.0}, {0.35, 0.65}, {0.3, 0.7}, {0.24, 0.52, 0.24}, {0.16, 0.32, 0.40, 0.12}, {0.2, 0.3, 0.3, 0.2},
      // transfer-bound calls (narrow stencils): more chunks, a short last one
      {0.25, 0.3, 0.3, 0.15}, {0.2, 0.25, 0.25, 0.2, 0.1}, {0.15, 0.2, 0.2, 0.2, 0.15, 0.1}};
  double best = 0;
  const std::vector<double>* pick = &cand[0];
  for (const auto& c : cand) {
    double t_in = 0, gpu = 0, dout = 0;
    for (double f : c) {
      const double mc = f * (double)M;
      t_in += h2d * mc;
      gpu = std::max(t_in, gpu) + eval_ms(mc);
      dout = std::max(dout, gpu) + d2h * mc;
    }
    if (pick == &cand[0] && &c == &cand[0]) best = dout;
    if (dout < best) {
      best = dout;
      pick = &c;
    }
  }
  return *pick;
}

int eval_host_pipelined(vfn_plan* p, const double* points, int64_t M, double* out,
                        int64_t* first_bad_row, cudaStream_t s) {
  vfn::NvtxRange nvtx_range("vfn evaluate pipelined (host buffers)");
  // Each chunk's gather re-reads every grid tile its points touch, so small
  // chunks cost tile traffic (c5, 2^28 points: 2 equal chunks 254 ms, 3 equal
  // 244 ms, 4 equal 270 ms, 8 equal 380 ms; unpipelined 347 ms).  From 2^26
  // points: short first and last chunks (less fill and drain) around two
  // long ones, 0.12/0.38/0.38/0.12 (238 ms); else two halves.
  // VFN_PIPE_SPLIT="f0,f1,..." sets the fractions, VFN_PIPE_CHUNK a fixed size.
  std::vector<double> frac;
  if (const char* e = std::getenv("VFN_PIPE_SPLIT")) {
    for (const char* q = e; *q;) {
      char* end = nullptr;
      const double f = std::strtod(q, &end);
      if (end == q) break;
      if (f > 0) frac.push_back(f);
      q = *end == ',' ? end + 1 : end;
    }
  }
  if (frac.empty()) {
    if (p->m >= 7)
      // wide stencils: a chunk's units fill worse at the chunk's lower point
      // density and the gather dominates the transfers, so one chunk or one
      // short lead chunk beats the m = 6 split (c5, pinned buffers: m = 8
      // 1746 ms with the m = 6 split, 1127 ms at 0.15/0.85, 855 ms one
      // chunk; m = 7 461 / 353 / 383 ms).  Having the gather store values
      // straight into pinned output instead of a D2H copy was measured too:
      // scattered 16-byte PCIe writes took c5 m = 6 from 227 to 1282 ms.
      // (m = 7 after the late-binding gather: one chunk 378 ms, 0.15/0.85 345 ms, 0.3/0.7 327 ms)
      frac = (p->m == 7 && M >= ((int64_t)1 << 27)) ? std::vector<double>{0.3, 0.7} : std::vector<double>{1.0};
    else
      frac = model_split(p, points, M);
  }
  std::vector<int64_t> lo_of{0};
  if (const char* e = std::getenv("VFN_PIPE_CHUNK")) {
    const int64_t c = std::max<int64_t>(1 << 16, std::atoll(e));
    for (int64_t x = c; x < M; x += c) lo_of.push_back(x);
  } else {
    double tot = 0;
    for (double f : frac) tot += f;
    double acc = 0;
    for (size_t i = 0; i + 1 < frac.size(); ++i) {
      acc += frac[i];
      const int64_t b = std::min<int64_t>(M, (int64_t)(acc / tot * (double)M));
      if (b > lo_of.back()) lo_of.push_back(b);
    }
  }
  // split any chunk above the batch limit
  {
    std::vector<int64_t> v{0};
    lo_of.push_back(M);
    for (size_t i = 0; i + 1 < lo_of.size(); ++i)
      for (int64_t x = lo_of[i] + max_batch(); x < lo_of[i + 1]; x += max_batch()) v.push_back(x);
    for (size_t i = 1; i + 1 < lo_of.size(); ++i) v.push_back(lo_of[i]);
    std::sort(v.begin(), v.end());
    v.push_back(M);
    lo_of = v;
  }
  const int64_t nc = (int64_t)lo_of.size() - 1;
  int64_t chunk = 0;
  for (int64_t i = 0; i < nc; ++i) chunk = std::max(chunk, lo_of[i + 1] - lo_of[i]);
  for (int i = 0; i < 2; ++i) {
    if (!p->copy_stream[i]) VFN_CUDA(cudaStreamCreateWithFlags(&p->copy_stream[i], cudaStreamNonBlocking));
  }
  cudaStream_t sin = p->copy_stream[0], sout = p->copy_stream[1];
  // pageable user buffers: chunk copies go through the device's pinned stager
  // (host threads copy one piece while the DMA engine moves the previous);
  // chunk i-1's output is staged out while chunk i computes
  HostStager* st_in = stager_for(p, points, sizeof(double) * 3 * M);
  HostStager* st_out = stager_for(p, out, sizeof(double2) * M);
  VFN_CHECK(p->pts.ensure(sizeof(double) * 3 * (nc > 1 ? 2 : 1) * chunk));
  VFN_CHECK(p->out.ensure(sizeof(double2) * (nc > 1 ? 2 : 1) * chunk));
  VFN_CHECK(p->misc.ensure(sizeof(int64_t) * (nc + 8)));
  int64_t* bad_dev = p->misc.as<int64_t>();
  std::vector<cudaEvent_t> ev(3 * nc);
  for (auto& e : ev) VFN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  auto e_in = [&](int64_t i) { return ev[3 * i]; };
  auto e_comp = [&](int64_t i) { return ev[3 * i + 1]; };
  auto e_out = [&](int64_t i) { return ev[3 * i + 2]; };
  int st = VFN_OK;
  // one geometry for every chunk, chosen from the WHOLE call's points exactly
  // as the device-resident call would (its density sample rows are copied
  // up first), so host and device inputs give bitwise the same values
  BinGeom g;
  {
    std::vector<double> hs;
    const double* sdev = nullptr;
    if (M >= kDensityMinM) {
      const int S = kDensitySample;
      hs.resize(3 * (size_t)S);
      for (int j = 0; j < S; ++j)
        for (int d = 0; d < 3; ++d) hs[3 * (size_t)j + d] = points[3 * ((int64_t)j * (M / S)) + d];
      VFN_CHECK(p->sample_pts.ensure(sizeof(double) * hs.size()));
      VFN_CUDA(cudaMemcpyAsync(p->sample_pts.ptr, hs.data(), sizeof(double) * hs.size(), cudaMemcpyHostToDevice, s));
      sdev = p->sample_pts.as<double>();
    }
    int bxy = 2;
    VFN_CHECK(choose_bxy(p, M, sdev, true, s, &bxy));
    VFN_CUDA(cudaStreamSynchronize(s));  // hs is read by the copy above
    g = make_geometry(p, bxy);
    p->last_geom = g;
    p->has_last_geom = true;
  }
  bool have_g = true;
  auto stage_out = [&](int64_t j) -> int {
    const int64_t lo = lo_of[j], n = lo_of[j + 1] - lo;
    cudaStreamWaitEvent(sout, e_comp(j), 0);
    VFN_CHECK(stage_d2h(st_out, out + 2 * lo, p->out.as<double2>() + chunk * (j & 1), sizeof(double2) * n, sout));
    cudaEventRecord(e_out(j), sout);
    return VFN_OK;
  };
  VFN_CUDA(cudaEventRecord(p->ev[0], s));
  for (int64_t i = 0; i < nc && st == VFN_OK; ++i) {
    const int64_t lo = lo_of[i], n = lo_of[i + 1] - lo;
    double* pbuf = p->pts.as<double>() + 3 * chunk * (i & 1);
    double2* obuf = p->out.as<double2>() + chunk * (i & 1);
    if (i >= 2) cudaStreamWaitEvent(sin, e_comp(i - 2), 0);
    if (st_in)
      st = stage_h2d(st_in, pbuf, points + 3 * lo, sizeof(double) * 3 * n, sin);
    else
      cudaMemcpyAsync(pbuf, points + 3 * lo, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, sin);
    if (st != VFN_OK) break;
    cudaEventRecord(e_in(i), sin);
    cudaStreamWaitEvent(s, e_in(i), 0);
    if (i >= 2) cudaStreamWaitEvent(s, e_out(i - 2), 0);
    // one geometry for all chunks (decided on the first), no mid-pipeline syncs
    st = eval_enqueue(p, pbuf, n, obuf, bad_dev + i, s, have_g ? &g : nullptr);
    if (st != VFN_OK) break;
    if (!have_g) {
      g = p->last_geom;
      have_g = true;
    }
    cudaEventRecord(e_comp(i), s);
    if (st_out) {
      if (i >= 1) st = stage_out(i - 1);
    } else {
      cudaStreamWaitEvent(sout, e_comp(i), 0);
      cudaMemcpyAsync(out + 2 * lo, obuf, sizeof(double2) * n, cudaMemcpyDeviceToHost, sout);
      cudaEventRecord(e_out(i), sout);
    }
  }
  if (st == VFN_OK && st_out) st = stage_out(nc - 1);
  std::vector<int64_t> bad(nc, kBadSentinel);
  if (st == VFN_OK) {
    cudaStreamWaitEvent(s, e_out(nc - 1), 0);
    cudaMemcpyAsync(bad.data(), bad_dev, sizeof(int64_t) * nc, cudaMemcpyDeviceToHost, s);
    cudaEventRecord(p->ev[3], s);
  }
  cudaError_t e = cudaStreamSynchronize(s);
  cudaStreamSynchronize(sin);
  cudaStreamSynchronize(sout);
  for (auto& x : ev) cudaEventDestroy(x);
  if (st != VFN_OK) return st;
  if (e != cudaSuccess) return fail(VFN_ERR_CUDA, std::string("pipelined evaluate: ") + cudaGetErrorString(e));
  p->timing_pending = true;  // elapsed times are read lazily (vfn_plan_last_timing)
  for (int64_t i = 0; i < nc; ++i)
    if (bad[i] != kBadSentinel) return outside(lo_of[i] + bad[i], first_bad_row);
  return VFN_OK;
}

// vfn_plan_eval with the plan lock held (also the body of vfn_plan_eval_to_peers)
int plan_eval_locked(vfn_plan* p, const double* points, int64_t M, double* out, int on_device,
                     int64_t* first_bad_row, void* stream) {
  if (M < 0) return fail(VFN_ERR_INVALID, "point count out of range");
  if (first_bad_row) *first_bad_row = -1;
  if (M == 0) return VFN_OK;
  DeviceGuard guard(p->device);
  cudaStream_t s = as_stream(stream);
  if (on_device) {
    VFN_CHECK(check_on_device(points, p->device, "points"));
    VFN_CHECK(check_on_device(out, p->device, "out"));
  }
  if (!on_device && M >= pipe_min_m()) return eval_host_pipelined(p, points, M, out, first_bad_row, s);
  if (M > max_batch()) return eval_device_batches(p, points, M, out, on_device, first_bad_row, s);
  VFN_CUDA(cudaEventRecord(p->ev[0], s));
  const void* pdev = nullptr;
  HostStager* st_in = on_device ? nullptr : stager_for(p, points, sizeof(double) * 3 * M);
  HostStager* st_out = on_device ? nullptr : stager_for(p, out, sizeof(double2) * M);
  VFN_CHECK(stage_in(p->pts, points, sizeof(double) * 3 * M, on_device, &pdev, s, st_in));
  double2* out_dev = reinterpret_cast<double2*>(out);
  if (!on_device) {
    VFN_CHECK(p->out.ensure(sizeof(double2) * M));
    out_dev = p->out.as<double2>();
  }
  VFN_CHECK(p->misc.ensure(64));
  int64_t* bad_dev = p->misc.as<int64_t>();
  const bool warp_path = p->gather_variant == 3 || (p->gather_variant == 0 && M <= warp_max_m());
  if (warp_path) {
    // small evaluate: one unbinned warp-per-point kernel (vfn_kernels.cu K4
    // v3); its bad-row word holds the sentinel between calls (set at plan
    // creation, restored by store_word), so no memset per call
    bad_dev = p->warp_bad.as<int64_t>();
    mark_event(p, 1, s);
    VFN_CHECK(gather_warp(p, static_cast<const double*>(pdev), M, out_dev, bad_dev, s));
    mark_event(p, 2, s);
  } else {
    bool graphed = false;
    if (!p->peer_dev)  // graphs bake in their output pointers
      VFN_CHECK(eval_graphed(p, static_cast<const double*>(pdev), M, out_dev, bad_dev, s, &graphed));
    if (!graphed) VFN_CHECK(eval_enqueue(p, static_cast<const double*>(pdev), M, out_dev, bad_dev, s, nullptr));
  }
  if (p->peer_dev && !p->peer_used)  // gathers without the fused epilogue: values out to their owners now
    VFN_CHECK(scatter_to_peers(out_dev, M, p->peer_dev, s));
  if (st_out)
    VFN_CHECK(stage_d2h(st_out, out, out_dev, sizeof(double2) * M, s));
  else if (!on_device)
    VFN_CUDA(cudaMemcpyAsync(out, out_dev, sizeof(double2) * M, cudaMemcpyDeviceToHost, s));
  // first bad row -> mapped pinned host word, stored by a one-thread kernel
  // (a copy-engine D2H of 8 bytes adds ~10-20 us of latency to every call)
  int64_t* bad_host = p->bad_host ? p->bad_host : &p->bad_fallback;
  *bad_host = kBadSentinel;
  if (p->bad_mapped) {
    VFN_CHECK(store_word(bad_dev, p->bad_mapped, s, warp_path));
  } else {
    VFN_CUDA(cudaMemcpyAsync(bad_host, bad_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (warp_path) VFN_CUDA(cudaMemsetAsync(bad_dev, kBadByte, sizeof(int64_t), s));
  }
  VFN_CUDA(cudaEventRecord(p->ev[3], s));
  VFN_CUDA(cudaStreamSynchronize(s));
  const int64_t bad = *bad_host;
  p->timing_pending = true;  // elapsed times are read lazily (vfn_plan_last_timing)
  if (bad != kBadSentinel) return outside(bad, first_bad_row);
  return VFN_OK;
}

}  // namespace

extern "C" {

int vfn_plan_eval(vfn_plan* p, const double* points, int64_t M, double* out, int on_device,
                  int64_t* first_bad_row, void* stream) {
  vfn::NvtxRange nvtx_range("vfn evaluate");
  if (!p || (M > 0 && (!points || !out))) return fail(VFN_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  return plan_eval_locked(p, points, M, out, on_device, first_bad_row, stream);
}

int vfn_plan_eval_to_peers(vfn_plan* p, const double* points, int64_t M, const int32_t* rows, int npeers,
                           const int64_t* seg_off, double* const* outs, int64_t* first_bad_row, void* stream) {
  vfn::NvtxRange nvtx_range("vfn evaluate (values to their owners)");
  if (!p || !seg_off || !outs || (M > 0 && (!points || !rows))) return fail(VFN_ERR_INVALID, "null argument");
  if (npeers < 1 || npeers > kMaxPeers) return fail(VFN_ERR_INVALID, "peer count must be in 1..64");
  if (seg_off[0] != 0 || seg_off[npeers] != M) return fail(VFN_ERR_INVALID, "peer ranges must cover the points");
  std::lock_guard<std::mutex> plan_lock(p->mu);
  if (first_bad_row) *first_bad_row = -1;
  if (M == 0) return VFN_OK;
  DeviceGuard guard(p->device);
  cudaStream_t s = as_stream(stream);
  VFN_CHECK(check_on_device(points, p->device, "points"));
  PeerTable h;
  h.n = npeers;
  h.rows = rows;
  for (int o = 0; o <= npeers; ++o) h.off[o] = seg_off[o];
  for (int o = 0; o < npeers; ++o) h.out[o] = reinterpret_cast<double2*>(outs[o]);
  VFN_CHECK(p->peer_buf.ensure(sizeof(PeerTable)));
  VFN_CUDA(cudaMemcpyAsync(p->peer_buf.ptr, &h, sizeof(PeerTable), cudaMemcpyHostToDevice, s));
  VFN_CUDA(cudaStreamSynchronize(s));  // h lives on this stack frame
  // the evaluate's own output is scratch; values land in the owners' buffers
  VFN_CHECK(p->out.ensure(sizeof(double2) * M));
  const bool fused = M <= max_batch();  // batched calls index the rows per batch: scatter afterwards
  p->peer_dev = fused ? p->peer_buf.as<PeerTable>() : nullptr;
  p->peer_used = false;
  int st = plan_eval_locked(p, points, M, p->out.as<double>(), 1, first_bad_row, stream);
  p->peer_dev = nullptr;
  if (st == VFN_OK && !fused) {
    st = scatter_to_peers(p->out.as<double2>(), M, p->peer_buf.as<PeerTable>(), s);
    if (st == VFN_OK && cudaStreamSynchronize(s) != cudaSuccess) st = fail(VFN_ERR_CUDA, "peer scatter failed");
  }
  return st;
}

int vfn_rect_eval(int device, const int64_t nmodes[3], const double a[3], const double b[3],
                  const double* coeffs, const double* y1, int64_t M1, const double* y2,
                  int64_t M2, const double* y3, int64_t M3, double* out, int on_device,
                  void* stream) {
  vfn::NvtxRange nvtx_range("vfn rectilinear");
  if (!nmodes || !a || !b || !coeffs || !out) return fail(VFN_ERR_INVALID, "null argument");
  VFN_CHECK(check_box(a, b));
  for (int d = 0; d < 3; ++d)
    if (nmodes[d] <= 0 || nmodes[d] % 2 != 0)
      return fail(VFN_ERR_INVALID, "mode counts must be positive and even");
  if (M1 < 0 || M2 < 0 || M3 < 0) return fail(VFN_ERR_INVALID, "negative coordinate count");
  if (M1 * M2 * M3 == 0) return VFN_OK;
  DeviceGuard guard(device);
  const double* y[3] = {y1, y2, y3};
  const int64_t Mv[3] = {M1, M2, M3};
  return rect_eval(device, nmodes, a, b, coeffs, y, Mv, out, on_device, as_stream(stream));
}

int vfn_rect_eval_nufft(int device, const int64_t nmodes[3], const double a[3], const double b[3],
                        const double* coeffs, const double* y1, int64_t M1, const double* y2, int64_t M2,
                        const double* y3, int64_t M3, double sigma, int m, double* out, int on_device,
                        void* stream) {
  vfn::NvtxRange nvtx_range("vfn rectilinear (NUFFT passes)");
  if (!nmodes || !a || !b || !coeffs || !out) return fail(VFN_ERR_INVALID, "null argument");
  VFN_CHECK(check_box(a, b));
  for (int d = 0; d < 3; ++d)
    if (nmodes[d] <= 0 || nmodes[d] % 2 != 0)
      return fail(VFN_ERR_INVALID, "mode counts must be positive and even");
  if (M1 < 0 || M2 < 0 || M3 < 0) return fail(VFN_ERR_INVALID, "negative coordinate count");
  if (M1 > INT32_MAX || M2 > INT32_MAX || M3 > INT32_MAX) return fail(VFN_ERR_INVALID, "coordinate count too large");
  if (m < 1) return fail(VFN_ERR_INVALID, "cutoff must be >= 1");
  if (M1 * M2 * M3 == 0) return VFN_OK;
  DeviceGuard guard(device);
  const double* y[3] = {y1, y2, y3};
  const int64_t Mv[3] = {M1, M2, M3};
  return rect_eval(device, nmodes, a, b, coeffs, y, Mv, out, on_device, as_stream(stream), m, sigma);
}

}  // extern "C"
