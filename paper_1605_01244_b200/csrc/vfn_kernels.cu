// Point mapping / binning (K0+K1), grid build (K2 deconvolve+pad, K3 cuFFT,
// K3b ghost padding) and the simple thread-per-point gather (K4 v1).
#include <algorithm>
#include <array>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "vfn_device.cuh"

namespace vfn {

// ------------------------------------------------------------ cuFFT plans
// Process-wide cache of Z2Z 3D plans keyed by (device, dims): plan creation
// (and its workspace allocation) costs milliseconds, far more than the
// transform at the sizes tube_eval / snapshot_spectral / small plans use.
// One plan's workspace is shared by its executions, so each execution waits
// on the previous one's completion event (cross-stream safe).
namespace {
struct FftEntry {
  cufftHandle h = 0;
  cudaEvent_t done = nullptr;
  uint64_t stamp = 0;
};
std::mutex g_fft_mu;
std::map<std::array<int64_t, 6>, FftEntry> g_fft;
uint64_t g_fft_clock = 0;
constexpr size_t kFftCacheMax = 6;
}  // namespace

int fft_exec(const int64_t n[3], double2* data, cudaStream_t s, int direction, const int64_t* embed = nullptr);

int fft_forward(const int64_t n[3], double2* data, cudaStream_t s) { return fft_exec(n, data, s, CUFFT_FORWARD); }

int fft_inverse(const int64_t n[3], double2* data, cudaStream_t s) { return fft_exec(n, data, s, CUFFT_INVERSE); }

// In-place transform of an (n0, n1, n2) array embedded in a (E0, E1, E2)
// C-order allocation (element (i0, i1, i2) at data[(i0 E1 + i1) E2 + i2]):
// the ghost-padded grid's interior, transformed where it lies.
int fft_forward_embedded(const int64_t n[3], const int64_t embed[3], double2* data, cudaStream_t s) {
  return fft_exec(n, data, s, CUFFT_FORWARD, embed);
}

// in-place unnormalised 3D Z2Z transform through the cached plan of its size
// (and embedding, if any)
int fft_exec(const int64_t n[3], double2* data, cudaStream_t s, int direction, const int64_t* embed) {
  int dev = 0;
  VFN_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_fft_mu);
  const std::array<int64_t, 6> key = {dev, n[0], n[1], n[2], embed ? embed[1] : 0, embed ? embed[2] : 0};
  auto it = g_fft.find(key);
  if (it == g_fft.end()) {
    if (g_fft.size() >= kFftCacheMax) {  // evict the least recently used plan
      auto lru = g_fft.begin();
      for (auto j = g_fft.begin(); j != g_fft.end(); ++j)
        if (j->second.stamp < lru->second.stamp) lru = j;
      if (lru->second.done) cudaEventSynchronize(lru->second.done);
      cufftDestroy(lru->second.h);
      if (lru->second.done) cudaEventDestroy(lru->second.done);
      g_fft.erase(lru);
    }
    FftEntry e;
    if (cufftCreate(&e.h) != CUFFT_SUCCESS) return fail(VFN_ERR_CUFFT, "cufftCreate failed");
    long long nn[3] = {n[0], n[1], n[2]};
    long long em[3] = {embed ? embed[0] : n[0], embed ? embed[1] : n[1], embed ? embed[2] : n[2]};
    const long long dist = em[0] * em[1] * em[2];
    size_t work = 0;
    const cufftResult r = cufftMakePlanMany64(e.h, 3, nn, em, 1, dist, em, 1, dist, CUFFT_Z2Z, 1, &work);
    if (r != CUFFT_SUCCESS) {
      cufftDestroy(e.h);
      return fail(VFN_ERR_CUFFT, "cufftMakePlanMany64 failed (code " + std::to_string((int)r) + ")");
    }
    if (cudaEventCreateWithFlags(&e.done, cudaEventDisableTiming) != cudaSuccess) {
      cufftDestroy(e.h);
      return fail(VFN_ERR_CUDA, "fft event creation failed");
    }
    it = g_fft.emplace(key, e).first;
  }
  FftEntry& e = it->second;
  e.stamp = ++g_fft_clock;
  VFN_CUDA(cudaStreamWaitEvent(s, e.done, 0));  // previous use of the workspace
  cufftResult r = cufftSetStream(e.h, s);
  if (r == CUFFT_SUCCESS)
    r = cufftExecZ2Z(e.h, reinterpret_cast<cufftDoubleComplex*>(data), reinterpret_cast<cufftDoubleComplex*>(data),
                     direction);
  if (r != CUFFT_SUCCESS) return fail(VFN_ERR_CUFFT, "cuFFT Z2Z failed (code " + std::to_string((int)r) + ")");
  VFN_CUDA(cudaEventRecord(e.done, s));
  return VFN_OK;
}


// ------------------------------------------------------------------ K0 + K1
// One pass over the points: domain check (first bad row by atomicMin,
// nufft.py:115-126), nearest cell per axis, and the bin key.
// u (optional) receives the reference's u = z * n per coordinate
// (nufft.py:256), from which the gather re-derives l0 and delta exactly.
__global__ void k_map_key(const double* __restrict__ pts, int64_t M, TorusMap tm, BinGeom g,
                          uint32_t* __restrict__ keys, int32_t* __restrict__ iota,
                          double* __restrict__ u, unsigned long long* __restrict__ bad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  int cell[3];
  bool ok = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double x = pts[3 * i + d];
    ok = ok && inside(x, tm.a[d], tm.b[d]);
    // one correctly rounded division per coordinate: the cell comes from u
    // exactly as nearest_cell derives it (same u, same floor)
    const double ud = torus_u(x, tm.a[d], tm.amb[d], tm.nd[d]);
    double delta;
    cell[d] = cell_from_u(ud, tm.nd[d], tm.n[d], delta);
    if (u) u[3 * i + d] = ud;
  }
  if (!ok) {
    atomicMin(bad, (unsigned long long)i);
    cell[0] = cell[1] = cell[2] = 0;  // any in-range key; the call fails anyway
  }
  // key = (tile * boxes_per_tile + box) * key_slots + (depth >> key_shift),
  // tiles and boxes row-major: a box's points come out sorted by depth pair
  // or depth (the gather's units are depth runs; BinGeom::key_shift)
  int t[3], in[3], c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    // exact quotients by multiply-shift (cells < 2^20, tile/box sizes <= 64)
    t[d] = (int)(((uint64_t)cell[d] * g.tile_inv[d]) >> 32);
    const int r = cell[d] - t[d] * g.tile[d];
    in[d] = (int)(((uint64_t)r * g.box_inv[d]) >> 32);
    c[d] = r - in[d] * g.box[d];
    VFN_DCHECK(t[d] == cell[d] / g.tile[d] && in[d] == r / g.box[d]);
  }
  int64_t tile_id = ((int64_t)t[0] * g.ntile[1] + t[1]) * g.ntile[2] + t[2];
  int box_id = (in[0] * g.nbox[1] + in[1]) * g.nbox[2] + in[2];
  const int slot = c[2] >> g.key_shift;
  VFN_DCHECK(tile_id < g.ntiles && box_id < g.boxes_per_tile && slot < g.key_slots);
  keys[i] = (uint32_t)((tile_id * g.boxes_per_tile + box_id) * g.key_slots + slot);
  if (iota) iota[i] = (int32_t)i;
}

__global__ void k_torus(const double* __restrict__ pts, int64_t M, TorusMap tm,
                        double* __restrict__ zeta) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * M) return;
  int d = (int)(i % 3);
  zeta[i] = torus_coord(pts[i], tm.a[d], tm.amb[d]);
}

int map_and_key(vfn_plan* p, const double* pts, int64_t M, const BinGeom& g, uint32_t* keys,
                int32_t* iota, double* u, int64_t* bad_dev, cudaStream_t s) {
  if (M == 0) return VFN_OK;
  int threads = 256;
  int64_t blocks = (M + threads - 1) / threads;
  k_map_key<<<(unsigned)blocks, threads, 0, s>>>(pts, M, p->map, g, keys, iota, u,
                                                  reinterpret_cast<unsigned long long*>(bad_dev));
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

int launch_torus(const TorusMap& tm, const double* pts, int64_t M, double* zeta, cudaStream_t s) {
  if (M == 0) return VFN_OK;
  int threads = 256;
  int64_t blocks = (3 * M + threads - 1) / threads;
  k_torus<<<(unsigned)blocks, threads, 0, s>>>(pts, M, tm, zeta);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

bool use_cub_sort() {
  static const bool cub = [] {
    const char* e = std::getenv("VFN_SORT");
    return !(e && std::string(e) == "radix");
  }();
  return cub;
}

// Stable sort of (key, value) pairs: CUB's onesweep with the iota values
// written by k_map_key (default), or with VFN_SORT=radix the hand-written
// LSD radix sort of vfn_sort.cu (values = the row index, implicit; bitwise
// the same permutation, measured slower at c5: 9.1 vs 7.2 ms, DESIGN 7).
int sort_pairs(vfn_plan* p, const uint32_t* keys_in, uint32_t* keys_out, const int32_t* vals_in,
               int32_t* vals_out, int64_t M, int key_bits, cudaStream_t s) {
  if (!use_cub_sort()) return radix_sort_pairs(p->sort_tmp, keys_in, keys_out, vals_out, M, key_bits, s);
  size_t tmp = 0;
  VFN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys_in, keys_out, vals_in, vals_out,
                                           (int)M, 0, key_bits, s));
  VFN_CHECK(p->sort_tmp.ensure(tmp));
  VFN_CUDA(cub::DeviceRadixSort::SortPairs(p->sort_tmp.ptr, tmp, keys_in, keys_out, vals_in,
                                           vals_out, (int)M, 0, key_bits, s));
  return VFN_OK;
}

// ------------------------------------------------------------------ K2
// Deconvolution fused with the octant zero-pad (nufft.py:219-241): every
// element of the n1 x n2 x n3 FFT input is written once; mode k lands at
// index k mod n with value coeff * sign(k) / (phihat1 phihat2 phihat3) / vol^(1/2) / prod n.
// fac_d[j] carries sign(k_d) / phihat_d(k_d) for centred index j.
__global__ void k_deconv_pad(const double2* __restrict__ coeffs, int64_t N0, int64_t N1,
                             int64_t N2, int64_t n0, int64_t n1, int64_t n2,
                             const double* __restrict__ fac0, const double* __restrict__ fac1,
                             const double* __restrict__ fac2, double scale,
                             double2* __restrict__ out) {
  const int64_t total = n0 * n1 * n2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i2 = e % n2;
    int64_t r = e / n2;
    int64_t i1 = r % n1;
    int64_t i0 = r / n1;
    // index i holds wavenumber i (i < N/2) or i - n (i >= n - N/2)
    int64_t j0 = i0 < N0 / 2 ? i0 + N0 / 2 : (i0 >= n0 - N0 / 2 ? i0 - n0 + N0 / 2 : -1);
    int64_t j1 = i1 < N1 / 2 ? i1 + N1 / 2 : (i1 >= n1 - N1 / 2 ? i1 - n1 + N1 / 2 : -1);
    int64_t j2 = i2 < N2 / 2 ? i2 + N2 / 2 : (i2 >= n2 - N2 / 2 ? i2 - n2 + N2 / 2 : -1);
    double2 v = make_double2(0.0, 0.0);
    if (j0 >= 0 && j1 >= 0 && j2 >= 0) {
      double2 c = coeffs[(j0 * N1 + j1) * N2 + j2];
      double f = fac0[j0] * fac1[j1] * fac2[j2] * scale;
      v = make_double2(c.x * f, c.y * f);
    }
    out[e] = v;
  }
}

// K2 writing straight into the ghost-padded grid's interior: row (i0, i1)
// of the n0 x n1 x n2 FFT input lives at G + (i0 P1 + i1) P2 (G = the
// interior origin), so the FFT runs in place there and only the halo faces
// are copied afterwards (no separate n^3 buffer, no full ghost-pad pass).
__global__ void k_deconv_pad_rows(const double2* __restrict__ coeffs, int64_t N0, int64_t N1,
                                  int64_t N2, int64_t n0, int64_t n1, int64_t n2,
                                  const double* __restrict__ fac0, const double* __restrict__ fac1,
                                  const double* __restrict__ fac2, double scale,
                                  double2* __restrict__ G, int64_t P1, int64_t P2) {
  const int64_t rows = n0 * n1;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t i0 = r / n1, i1 = r - i0 * n1;
    const int64_t j0 = i0 < N0 / 2 ? i0 + N0 / 2 : (i0 >= n0 - N0 / 2 ? i0 - n0 + N0 / 2 : -1);
    const int64_t j1 = i1 < N1 / 2 ? i1 + N1 / 2 : (i1 >= n1 - N1 / 2 ? i1 - n1 + N1 / 2 : -1);
    double2* row = G + (i0 * P1 + i1) * P2;
    const bool live = j0 >= 0 && j1 >= 0;
    const double f01 = live ? fac0[j0] * fac1[j1] * scale : 0.0;
    const double2* crow = coeffs + (live ? (j0 * N1 + j1) * N2 : 0);
    for (int64_t i2 = threadIdx.x; i2 < n2; i2 += blockDim.x) {
      const int64_t j2 = i2 < N2 / 2 ? i2 + N2 / 2 : (i2 >= n2 - N2 / 2 ? i2 - n2 + N2 / 2 : -1);
      double2 v = make_double2(0.0, 0.0);
      if (live && j2 >= 0) {
        const double2 c = crow[j2];
        const double f = f01 * fac2[j2];
        v = make_double2(c.x * f, c.y * f);
      }
      row[i2] = v;
    }
  }
}

// Halo faces of the ghost-padded grid from its interior: padded index i
// holds g[(i - m) mod n], i.e. interior index ((i - m) mod n) + m.  Rows with
// both (i0, i1) inside copy only their 2m (+ alignment) z-ghosts; the others
// copy the whole row from their periodic image.  Every read is interior.
__global__ void k_halo_faces(double2* __restrict__ P, int64_t P0, int64_t P1, int64_t P2, int64_t n0,
                             int64_t n1, int64_t n2, int m) {
  const int64_t rows = P0 * P1;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t r0 = r / P1, r1 = r - r0 * P1;
    const int64_t s0 = ((r0 - m) % n0 + n0) % n0 + m, s1 = ((r1 - m) % n1 + n1) % n1 + m;
    double2* dst = P + r * P2;
    const double2* src = P + (s0 * P1 + s1) * P2;
    const bool inner = s0 == r0 && s1 == r1;
    const int64_t ghosts = P2 - n2;  // z-ghosts of an interior row
    const int64_t count = inner ? ghosts : P2;
    for (int64_t t = threadIdx.x; t < count; t += blockDim.x) {
      const int64_t i2 = inner ? (t < m ? t : t - m + n2 + m) : t;
      const int64_t s2 = ((i2 - m) % n2 + n2) % n2 + m;
      dst[i2] = src[s2];
    }
  }
}

// K3b: ghost-padded copy, P[i] = g[(i - m) mod n] per axis.
__global__ void k_halo(const double2* __restrict__ g, int64_t n0, int64_t n1, int64_t n2,
                       double2* __restrict__ P, int64_t P0, int64_t P1, int64_t P2, int m) {
  const int64_t total = P0 * P1 * P2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i2 = e % P2;
    int64_t r = e / P2;
    int64_t i1 = r % P1;
    int64_t i0 = r / P1;
    int64_t s0 = ((i0 - m) % n0 + n0) % n0;
    int64_t s1 = ((i1 - m) % n1 + n1) % n1;
    int64_t s2 = ((i2 - m) % n2 + n2) % n2;
    P[e] = g[(s0 * n1 + s1) * n2 + s2];
  }
}

// interior of the padded grid back to (n0, n1, n2)
__global__ void k_unpad(const double2* __restrict__ P, int64_t P1, int64_t P2, int m,
                        int64_t n0, int64_t n1, int64_t n2, double2* __restrict__ g) {
  const int64_t total = n0 * n1 * n2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i2 = e % n2;
    int64_t r = e / n2;
    int64_t i1 = r % n1;
    int64_t i0 = r / n1;
    g[e] = P[((i0 + m) * P1 + (i1 + m)) * P2 + (i2 + m)];
  }
}

static int grid_blocks(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (int)(b < 148 * 32 ? (b < 1 ? 1 : b) : 148 * 32);
}

int build_grid(vfn_plan* p, const double* coeffs_dev, cudaStream_t s) {
  vfn::NvtxRange nvtx_range("vfn grid: deconvolve + pad + FFT + halo");
  const int64_t N0 = p->N[0], N1 = p->N[1], N2 = p->N[2];
  const int64_t n0 = p->n[0], n1 = p->n[1], n2 = p->n[2];
  const int m = p->m;
  // sign(k)/phihat tables
  std::vector<double> h(N0 + N1 + N2);
  {
    double* f = h.data();
    for (int d = 0; d < 3; ++d) {
      kb_hat_table(p->N[d], p->n[d], m, p->beta, f);
      for (int64_t j = 0; j < p->N[d]; ++j) {
        const int64_t k = j - p->N[d] / 2;
        const double sign = (k % 2 == 0) ? 1.0 : -1.0;  // 1 - 2 (|k| mod 2)  (nufft.py:101-104)
        f[j] = sign / f[j];
      }
      f += p->N[d];
    }
  }
  const double vol = (p->b[0] - p->a[0]) * (p->b[1] - p->a[1]) * (p->b[2] - p->a[2]);
  const double scale = 1.0 / std::sqrt(vol) / ((double)n0 * (double)n1 * (double)n2);
  const int64_t Ptot = p->P[0] * p->P[1] * p->P[2];
  VFN_CHECK(p->dfacbuf.ensure(sizeof(double) * (N0 + N1 + N2)));
  double* dfac = p->dfacbuf.as<double>();
  if (!p->grid) {  // a rebuild keeps the plan's grid (and its tensor map)
    p->grid = static_cast<double2*>(pool_alloc(p->device, sizeof(double2) * Ptot, &p->grid_bytes));
    if (!p->grid) return fail(VFN_ERR_NOMEM, "padded grid allocation failed");
  }
  VFN_CUDA(cudaMemcpyAsync(dfac, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, s));
  const int64_t nn[3] = {n0, n1, n2};
  const bool copy_path = std::getenv("VFN_GRID_COPY") != nullptr;  // A/B: the separate-buffer build
  cudaEventRecord(p->bev[0], s);
  if (!copy_path) {
    // K2 into the padded interior, K3 in place there, then the halo faces
    double2* G = p->grid + (m * p->P[1] + m) * p->P[2] + m;
    k_deconv_pad_rows<<<(unsigned)std::min<int64_t>(n0 * n1, 148 * 64), 256, 0, s>>>(
        reinterpret_cast<const double2*>(coeffs_dev), N0, N1, N2, n0, n1, n2, dfac, dfac + N0,
        dfac + N0 + N1, scale, G, p->P[1], p->P[2]);
    VFN_CUDA(cudaGetLastError());
    cudaEventRecord(p->bev[1], s);
    VFN_CHECK(fft_forward_embedded(nn, p->P, G, s));
    cudaEventRecord(p->bev[2], s);
    k_halo_faces<<<(unsigned)std::min<int64_t>(p->P[0] * p->P[1], 148 * 64), 128, 0, s>>>(
        p->grid, p->P[0], p->P[1], p->P[2], n0, n1, n2, m);
    VFN_CUDA(cudaGetLastError());
  } else {
    // separate n^3 FFT buffer, then a full ghost-padding copy (K3b)
    VFN_CHECK(p->fftbuf.ensure(sizeof(double2) * n0 * n1 * n2));
    double2* buf = p->fftbuf.as<double2>();
    const int64_t total = n0 * n1 * n2;
    k_deconv_pad<<<grid_blocks(total), 256, 0, s>>>(
        reinterpret_cast<const double2*>(coeffs_dev), N0, N1, N2, n0, n1, n2, dfac, dfac + N0,
        dfac + N0 + N1, scale, buf);
    VFN_CUDA(cudaGetLastError());
    cudaEventRecord(p->bev[1], s);
    VFN_CHECK(fft_forward(nn, buf, s));
    cudaEventRecord(p->bev[2], s);
    k_halo<<<grid_blocks(Ptot), 256, 0, s>>>(buf, n0, n1, n2, p->grid, p->P[0], p->P[1], p->P[2], m);
    VFN_CUDA(cudaGetLastError());
  }
  cudaEventRecord(p->bev[3], s);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (copy_path && !p->keep_fftbuf) p->fftbuf.release();
  if (e != cudaSuccess) return fail(VFN_ERR_CUDA, std::string("grid build: ") + cudaGetErrorString(e));
  for (int i = 0; i < 3; ++i) p->build_ms[1 + i] = elapsed_ms(p->bev[i], p->bev[i + 1]);
  return VFN_OK;
}

int extract_grid(vfn_plan* p, double2* out_dev, cudaStream_t s) {
  const int64_t total = p->n[0] * p->n[1] * p->n[2];
  k_unpad<<<grid_blocks(total), 256, 0, s>>>(p->grid, p->P[1], p->P[2], p->m, p->n[0], p->n[1],
                                             p->n[2], out_dev);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

// ------------------------------------------------------------------ K4 v1
// Thread per point (in binned order when a permutation is given): window
// weights from the polynomial table, then the separable (2m+1)^3 contraction
// in the reference's order, axis 3 innermost (nufft.py:264-271).
template <int MC>
__global__ void __launch_bounds__(128) k_gather_simple(const double* __restrict__ pts, int64_t M,
                                                       const int32_t* __restrict__ perm,
                                                       TorusMap tm, const double* __restrict__ poly,
                                                       int deg, const double2* __restrict__ grid,
                                                       int64_t P1, int64_t P2,
                                                       double2* __restrict__ out) {
  constexpr int W = 2 * MC + 1;
  extern __shared__ double s_poly[];
  for (int i = threadIdx.x; i < W * (deg + 1); i += blockDim.x) s_poly[i] = poly[i];
  __syncthreads();
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= M) return;
  int64_t p = perm ? (int64_t)perm[s] : s;
  double w[3][W];
  int cell[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double delta;
    cell[d] = nearest_cell(pts[3 * p + d], tm.a[d], tm.amb[d], tm.nd[d], tm.n[d], delta);
#pragma unroll
    for (int j = 0; j < W; ++j) w[d][j] = window_poly(s_poly, deg, j, delta);
  }
  // padded index of grid cell (c - m + j) is c + j
  const double2* base = grid + ((int64_t)cell[0] * P1 + cell[1]) * P2 + cell[2];
  VFN_DCHECK(cell[1] + W <= P1 && cell[2] + W <= P2 && cell[0] >= 0 && cell[1] >= 0 && cell[2] >= 0);
  double ar = 0.0, ai = 0.0;
  for (int a = 0; a < W; ++a) {
    double br = 0.0, bi = 0.0;
    for (int b = 0; b < W; ++b) {
      const double2* row = base + ((int64_t)a * P1 + b) * P2;
      double cr = 0.0, ci = 0.0;
#pragma unroll
      for (int c = 0; c < W; ++c) {
        double2 v = __ldg(row + c);
        cr = fma(w[2][c], v.x, cr);
        ci = fma(w[2][c], v.y, ci);
      }
      br = fma(w[1][b], cr, br);
      bi = fma(w[1][b], ci, bi);
    }
    ar = fma(w[0][a], br, ar);
    ai = fma(w[0][a], bi, ai);
  }
  out[p] = make_double2(ar, ai);
}

// ------------------------------------------------------------------ K4 v3
// Small evaluates (M <= VFN_WARP_MAX_M): no binning at all.  One warp per
// point, in input order: the domain check and torus map (K0/K1), the 3 W
// window weights (lanes j < W), the W x W products w1[a] w2[b] in a per-warp
// table, then lanes = (row sub-index, c): each load instruction reads
// 32 / W whole z-lines of the ghost-padded grid (coalesced), each lane sums
// its column c over its rows and applies w3[c] once; a warp reduction gives
// the value (nufft.py:244-272).  Two launches (memset + this) instead of the
// ~25 of the binned path.
template <int MC>
__global__ void __launch_bounds__(256) k_gather_warp(const double* __restrict__ pts, int64_t M, TorusMap tm,
                                                     const double* __restrict__ poly, int deg,
                                                     const double2* __restrict__ grid, int64_t P1,
                                                     int64_t P2, double2* __restrict__ out,
                                                     unsigned long long* __restrict__ bad) {
  constexpr int W = 2 * MC + 1;
  constexpr int RPI = 32 / W;  // rows per load instruction
  extern __shared__ double s_warp[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // window coefficients staged once per CTA: Horner straight from global
  // memory is a chain of dependent L2 round trips (~25 us per call)
  double* s_poly = s_warp;
  for (int i = threadIdx.x; i < W * (deg + 1); i += blockDim.x) s_poly[i] = poly[i];
  __syncthreads();
  double* w = s_warp + W * (deg + 1) + warp * (3 * W + W * W);  // w[d][j], then w12[a * W + b]
  double* w12 = w + 3 * W;
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (p >= M) return;
  int cell[3];
  double dl[3];
  bool ok = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double x = pts[3 * p + d];
    ok = ok && inside(x, tm.a[d], tm.b[d]);
    cell[d] = nearest_cell(x, tm.a[d], tm.amb[d], tm.nd[d], tm.n[d], dl[d]);
  }
  if (!ok && lane == 0) atomicMin(bad, (unsigned long long)p);
  if (lane < W) {
    double wl[3];
    window_poly3(s_poly, deg, lane, dl, wl);
#pragma unroll
    for (int d = 0; d < 3; ++d) w[d * W + lane] = wl[d];
  }
  __syncwarp();
  for (int r = lane; r < W * W; r += 32) w12[r] = w[r / W] * w[W + r % W];
  __syncwarp();
  const int c = lane % W, rs = lane / W;
  double ar = 0.0, ai = 0.0;
  if (rs < RPI) {
    // padded index of grid cell (cell - m + j) is cell + j
    const double2* base = grid + ((int64_t)cell[0] * P1 + cell[1]) * P2 + cell[2] + c;
    VFN_DCHECK(cell[1] + W <= P1 && cell[2] + W <= P2);
    // row r = a W + b sits at base + (a P1 + b) P2; walk it incrementally (a
    // single warp's call is a serial instruction stream: no 64-bit index
    // products per row)
    int b = rs % W;
    const double2* q = base + ((int64_t)(rs / W) * P1 + b) * P2;
    const int64_t step = (int64_t)RPI * P2, wrap = ((int64_t)P1 - W) * P2;
#pragma unroll 4
    for (int r = rs; r < W * W; r += RPI) {
      const double2 v = __ldg(q);
      const double f = w12[r];
      ar = fma(f, v.x, ar);
      ai = fma(f, v.y, ai);
      const int wraps = (b + RPI) / W;  // branch-free, so loads batch across rows
      b += RPI - wraps * W;
      q += step + wraps * wrap;
    }
    const double wc = w[2 * W + c];
    ar *= wc;
    ai *= wc;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ar += __shfl_xor_sync(0xffffffffu, ar, o);
    ai += __shfl_xor_sync(0xffffffffu, ai, o);
  }
  if (lane == 0) out[p] = make_double2(ar, ai);
}

template <int MC>
static void launch_warp(vfn_plan* pl, const double* pts, int64_t M, double2* out, unsigned long long* bad,
                        cudaStream_t s) {
  constexpr int W = 2 * MC + 1;
  const int warps = 8;
  const size_t smem = sizeof(double) * (W * (pl->poly.deg + 1) + warps * (3 * W + W * W));
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_gather_warp<MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_gather_warp<MC><<<(unsigned)((M + warps - 1) / warps), warps * 32, smem, s>>>(
      pts, M, pl->map, pl->poly.dev, pl->poly.deg, pl->grid, pl->P[1], pl->P[2], out, bad);
}

int gather_warp(vfn_plan* p, const double* pts, int64_t M, double2* out, int64_t* bad_dev, cudaStream_t s) {
  if (M == 0) return VFN_OK;
  auto* bad = reinterpret_cast<unsigned long long*>(bad_dev);
  switch (p->m) {
    case 1: launch_warp<1>(p, pts, M, out, bad, s); break;
    case 2: launch_warp<2>(p, pts, M, out, bad, s); break;
    case 3: launch_warp<3>(p, pts, M, out, bad, s); break;
    case 4: launch_warp<4>(p, pts, M, out, bad, s); break;
    case 5: launch_warp<5>(p, pts, M, out, bad, s); break;
    case 6: launch_warp<6>(p, pts, M, out, bad, s); break;
    case 7: launch_warp<7>(p, pts, M, out, bad, s); break;
    case 8: launch_warp<8>(p, pts, M, out, bad, s); break;
    case 9: launch_warp<9>(p, pts, M, out, bad, s); break;
    case 10: launch_warp<10>(p, pts, M, out, bad, s); break;
    case 11: launch_warp<11>(p, pts, M, out, bad, s); break;
    case 12: launch_warp<12>(p, pts, M, out, bad, s); break;
    case 13: launch_warp<13>(p, pts, M, out, bad, s); break;
    default: return fail(VFN_ERR_INVALID, "cutoff must be in 1..13");
  }
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

template <int MC>
static void launch_simple(vfn_plan* pl, const double* pts, int64_t M, const int32_t* perm,
                          double2* out, cudaStream_t s) {
  int threads = 128;
  int64_t blocks = (M + threads - 1) / threads;
  size_t smem = sizeof(double) * (2 * MC + 1) * (pl->poly.deg + 1);
  k_gather_simple<MC><<<(unsigned)blocks, threads, smem, s>>>(
      pts, M, perm, pl->map, pl->poly.dev, pl->poly.deg, pl->grid, pl->P[1], pl->P[2], out);
}

int gather_simple(vfn_plan* p, const double* pts, int64_t M, const int32_t* perm, double2* out,
                  cudaStream_t s) {
  if (M == 0) return VFN_OK;
  switch (p->m) {
    case 1: launch_simple<1>(p, pts, M, perm, out, s); break;
    case 2: launch_simple<2>(p, pts, M, perm, out, s); break;
    case 3: launch_simple<3>(p, pts, M, perm, out, s); break;
    case 4: launch_simple<4>(p, pts, M, perm, out, s); break;
    case 5: launch_simple<5>(p, pts, M, perm, out, s); break;
    case 6: launch_simple<6>(p, pts, M, perm, out, s); break;
    case 7: launch_simple<7>(p, pts, M, perm, out, s); break;
    case 8: launch_simple<8>(p, pts, M, perm, out, s); break;
    case 9: launch_simple<9>(p, pts, M, perm, out, s); break;
    case 10: launch_simple<10>(p, pts, M, perm, out, s); break;
    case 11: launch_simple<11>(p, pts, M, perm, out, s); break;
    case 12: launch_simple<12>(p, pts, M, perm, out, s); break;
    case 13: launch_simple<13>(p, pts, M, perm, out, s); break;
    default: return fail(VFN_ERR_INVALID, "cutoff must be in 1..13");
  }
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

}  // namespace vfn
