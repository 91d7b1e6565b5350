// SURVEY 8f "next" rows on the device:
//  * snapshot_spectral (gpe.py:90-113 + fourier.py:183-188): mirror
//    extension, forward 3D FFT, fftshift and scaling -> centred coefficients;
//  * tube_eval (tube.py:58-127): seed selection on the stored samples, then
//    per pass the 27-point stencils of the surviving parents on the integer
//    lattice, evaluated through ONE reused plan (vfn_plan_eval on device
//    buffers), thresholded and compacted, and finally sorted by lattice key.
// Every arithmetic step the reference's decisions depend on (|v|^2, the
// lattice coordinates) is an explicitly rounded intrinsic so that it is
// bit-identical to numpy's.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <cstring>
#include <thread>
#include <string>
#include <vector>

#include "vfn_device.cuh"

struct vfn_tube {
  int device = 0;
  int64_t count = 0;
  vfn::DevBuf points, density, level;
};

#include <chrono>
namespace vfn {
static double tube_now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define TUBE_T(tag) do { if (dbg) { cudaStreamSynchronize(s); double t_ = tube_now_ms(); fprintf(stderr, "tube %-12s %8.2f ms\n", tag, t_ - t_last); t_last = t_; } } while (0)


// ------------------------------------------------------------------ spectral

__global__ void k_mirror(const double2* __restrict__ v, int64_t N0, int64_t N1, int64_t N2,
                         int64_t E0, int64_t E1, int64_t E2, double2* __restrict__ ext) {
  const int64_t total = E0 * E1 * E2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i2 = e % E2, r = e / E2, i1 = r % E1, i0 = r / E1;
    if (i0 >= N0) i0 = 2 * N0 - 1 - i0;
    if (i1 >= N1) i1 = 2 * N1 - 1 - i1;
    if (i2 >= N2) i2 = 2 * N2 - 1 - i2;
    ext[e] = v[(i0 * N1 + i1) * N2 + i2];
  }
}

// centred[j] = F[(j + E/2) mod E] * scale   (np.fft.fftshift for even E)
__global__ void k_shift_scale(const double2* __restrict__ F, int64_t E0, int64_t E1, int64_t E2,
                              double scale, double2* __restrict__ out) {
  const int64_t total = E0 * E1 * E2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t j2 = e % E2, r = e / E2, j1 = r % E1, j0 = r / E1;
    int64_t s0 = (j0 + E0 / 2) % E0, s1 = (j1 + E1 / 2) % E1, s2 = (j2 + E2 / 2) % E2;
    double2 v = F[(s0 * E1 + s1) * E2 + s2];
    out[e] = make_double2(__dmul_rn(v.x, scale), __dmul_rn(v.y, scale));
  }
}

static int grid_blocks(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (int)(b < 148 * 32 ? (b < 1 ? 1 : b) : 148 * 32);
}

// values_dev: (N0,N1,N2) samples on the device -> coeffs_dev (E0,E1,E2).
static int spectral_device(const double2* values_dev, const int64_t N[3], const double a[3],
                           const double b[3], const int mirror[3], double2* coeffs_dev,
                           int64_t E[3], double b_ext[3], cudaStream_t s) {
  for (int d = 0; d < 3; ++d) {
    E[d] = N[d] * (mirror[d] ? 2 : 1);
    b_ext[d] = mirror[d] ? a[d] + 2.0 * (b[d] - a[d]) : b[d];  // gpe.py:81-87
  }
  const int64_t total = E[0] * E[1] * E[2];
  // scale = prod(sqrt(w_d) / E_d), left to right like np.prod (fourier.py:186)
  double scale = 1.0;
  for (int d = 0; d < 3; ++d) scale *= std::sqrt(b_ext[d] - a[d]) / (double)E[d];
  DevBuf ext;
  VFN_CHECK(ext.ensure(sizeof(double2) * total));
  k_mirror<<<grid_blocks(total), 256, 0, s>>>(values_dev, N[0], N[1], N[2], E[0], E[1], E[2],
                                              ext.as<double2>());
  VFN_CUDA(cudaGetLastError());
  VFN_CHECK(fft_forward(E, ext.as<double2>(), s));  // cached cuFFT plan
  k_shift_scale<<<grid_blocks(total), 256, 0, s>>>(ext.as<double2>(), E[0], E[1], E[2], scale,
                                                   coeffs_dev);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  ext.release();
  if (e != cudaSuccess) return fail(VFN_ERR_CUDA, std::string("spectral: ") + cudaGetErrorString(e));
  return VFN_OK;
}

// ------------------------------------------------------------------ tube

// |v|^2 as numpy computes v.real**2 + v.imag**2 (no FMA contraction)
__device__ __forceinline__ double abs2(double2 v) {
  return __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
}

struct Lattice {
  int64_t size[3];  // lattice sizes at the finest spacing (E * 3^L)
  double step[3];   // widths / size, computed on the host like numpy
  double a[3];
};

__global__ void k_seed_flags(const double2* __restrict__ v, int64_t n, double thr,
                             double* __restrict__ rho, int* __restrict__ flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r = abs2(v[i]);
  rho[i] = r;
  flag[i] = r <= thr;
}

// seeds: flat physical index -> lattice index (unravel * 3^L)
__global__ void k_seed_scatter(const int* __restrict__ flag, const int* __restrict__ pos,
                               const double* __restrict__ rho, int64_t n, int64_t N1, int64_t N2,
                               int64_t mult, longlong4* __restrict__ idx, double* __restrict__ rho_out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  const int p = pos[i];
  const int64_t i2 = i % N2, r = i / N2, i1 = r % N1, i0 = r / N1;
  idx[p] = make_longlong4(i0 * mult, i1 * mult, i2 * mult, 0);  // .w = level
  rho_out[p] = rho[i];
}

__global__ void k_keep_flags(const double* __restrict__ rho, int64_t n, double thr,
                             int* __restrict__ flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = rho[i] <= thr;
}

__global__ void k_compact(const int* __restrict__ flag, const int* __restrict__ pos, int64_t n,
                          const longlong4* __restrict__ idx, const double* __restrict__ rho,
                          longlong4* __restrict__ idx_out, double* __restrict__ rho_out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  idx_out[pos[i]] = idx[i];
  if (rho_out) rho_out[pos[i]] = rho[i];
}

// 27 children per parent (offsets in {-1,0,1}^3, first axis slowest; child
// 13 is the parent itself and keeps its level), coordinates a + idx * step
__global__ void k_children(const longlong4* __restrict__ par, int64_t P, int64_t stride, int ell,
                           Lattice L, longlong4* __restrict__ kid, double* __restrict__ coords) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= 27 * P) return;
  const int64_t p = c / 27;
  const int o = (int)(c % 27);
  const int off[3] = {o / 9 - 1, (o / 3) % 3 - 1, o % 3 - 1};
  const longlong4 q = par[p];
  int64_t id[3] = {q.x, q.y, q.z};
  for (int d = 0; d < 3; ++d) {
    int64_t v = (id[d] + off[d] * stride) % L.size[d];
    if (v < 0) v += L.size[d];
    id[d] = v;
    coords[3 * c + d] = __dadd_rn(L.a[d], __dmul_rn((double)v, L.step[d]));
  }
  kid[c] = make_longlong4(id[0], id[1], id[2], o == 13 ? q.w : (long long)ell);
}

__global__ void k_rho(const double2* __restrict__ v, int64_t n, double* __restrict__ rho) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) rho[i] = abs2(v[i]);
}

__global__ void k_keys(const longlong4* __restrict__ idx, int64_t n, Lattice L,
                       unsigned long long* __restrict__ keys, int* __restrict__ iota) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const longlong4 q = idx[i];
  keys[i] = (unsigned long long)((q.x * L.size[1] + q.y) * L.size[2] + q.z);  // tube.py:50-51
  iota[i] = (int)i;
}

__global__ void k_emit(const int* __restrict__ perm, const longlong4* __restrict__ idx,
                       const double* __restrict__ rho, int64_t n, Lattice L,
                       double* __restrict__ pts, double* __restrict__ dens,
                       int64_t* __restrict__ lev) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm[i];
  const longlong4 q = idx[j];
  const int64_t id[3] = {q.x, q.y, q.z};
  for (int d = 0; d < 3; ++d) pts[3 * i + d] = __dadd_rn(L.a[d], __dmul_rn((double)id[d], L.step[d]));
  dens[i] = rho[j];
  lev[i] = q.w;
}

static unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

// flags -> exclusive positions; returns the count (host sync)
static int scan_count(const int* flag, int* pos, int64_t n, DevBuf& tmp, int64_t* count,
                      cudaStream_t s) {
  size_t bytes = 0;
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag, pos, (int)n, s));
  VFN_CHECK(tmp.ensure(bytes));
  VFN_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, bytes, flag, pos, (int)n, s));
  int last_pos = 0, last_flag = 0;
  VFN_CUDA(cudaMemcpyAsync(&last_pos, pos + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaMemcpyAsync(&last_flag, flag + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaStreamSynchronize(s));
  *count = (int64_t)last_pos + last_flag;
  return VFN_OK;
}

}  // namespace vfn

using namespace vfn;

extern "C" {

namespace {
struct TubeScratch {
  std::mutex mu;
  vfn::DevBuf vin, coeffs, rho0, flag, pos, tmp, idxA, idxB, rhoA, rhoB, coords, vals, keys, keys2, iota, perm;
  vfn_plan* plan = nullptr;
  int64_t E[3] = {0, 0, 0};
  double a[3] = {0, 0, 0}, bx[3] = {0, 0, 0}, sigma = 0;
  int m = 0;
};
TubeScratch* tube_scratch(int device) {
  static std::mutex mu;
  static std::map<int, TubeScratch*> all;
  std::lock_guard<std::mutex> lock(mu);
  TubeScratch*& t = all[device];
  if (!t) t = new TubeScratch();
  return t;
}
}  // namespace

// synthesize_regular (fourier.py:191-196): values = ifftn(ifftshift(coeffs))
// / scale, scale = prod_d sqrt(b_d - a_d) / N_d.  One kernel writes the
// shifted, scaled coefficients (1 / (N scale): cuFFT's inverse is
// unnormalised), then an in-place inverse FFT.
__global__ void k_ishift_scale(const double2* __restrict__ c, int64_t N0, int64_t N1, int64_t N2, double f,
                               double2* __restrict__ out) {
  const int64_t total = N0 * N1 * N2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i2 = e % N2, r = e / N2, i1 = r % N1, i0 = r / N1;
    const int64_t j0 = (i0 + N0 / 2) % N0, j1 = (i1 + N1 / 2) % N1, j2 = (i2 + N2 / 2) % N2;
    const double2 v = c[(j0 * N1 + j1) * N2 + j2];
    out[e] = make_double2(v.x * f, v.y * f);
  }
}

int vfn_synthesize(int device, const double* coeffs, const int64_t shape[3], const double a[3],
                   const double b[3], double* values_out, int on_device, void* stream) {
  vfn::NvtxRange nvtx_range("vfn synthesize");
  if (!coeffs || !shape || !a || !b || !values_out) return fail(VFN_ERR_INVALID, "null argument");
  for (int d = 0; d < 3; ++d)
    if (shape[d] <= 0 || !(a[d] < b[d])) return fail(VFN_ERR_INVALID, "bad shape or domain");
  DeviceGuard guard(device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n = shape[0] * shape[1] * shape[2];
  double scale = 1.0;
  for (int d = 0; d < 3; ++d) scale *= std::sqrt(b[d] - a[d]) / (double)shape[d];
  DevBuf cin, vout;
  const double2* cdev = reinterpret_cast<const double2*>(coeffs);
  double2* vdev = reinterpret_cast<double2*>(values_out);
  if (!on_device) {
    VFN_CHECK(cin.ensure(sizeof(double2) * n));
    VFN_CUDA(cudaMemcpyAsync(cin.ptr, coeffs, sizeof(double2) * n, cudaMemcpyHostToDevice, s));
    cdev = cin.as<double2>();
    VFN_CHECK(vout.ensure(sizeof(double2) * n));
    vdev = vout.as<double2>();
  }
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
  k_ishift_scale<<<blocks, 256, 0, s>>>(cdev, shape[0], shape[1], shape[2], 1.0 / ((double)n * scale), vdev);
  VFN_CUDA(cudaGetLastError());
  VFN_CHECK(fft_inverse(shape, vdev, s));
  if (!on_device)
    VFN_CUDA(cudaMemcpy(values_out, vdev, sizeof(double2) * n, cudaMemcpyDeviceToHost));
  else
    VFN_CUDA(cudaStreamSynchronize(s));
  return VFN_OK;
}

int vfn_decompose(int device, const double* values, const int64_t shape[3], const double a[3],
                  const double b[3], const int mirror[3], double* coeffs_out, int on_device,
                  void* stream) {
  vfn::NvtxRange nvtx_range("vfn decompose");
  if (!values || !shape || !a || !b || !mirror || !coeffs_out) return fail(VFN_ERR_INVALID, "null argument");
  for (int d = 0; d < 3; ++d)
    if (shape[d] <= 0 || !(a[d] < b[d])) return fail(VFN_ERR_INVALID, "bad shape or domain");
  DeviceGuard guard(device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n = shape[0] * shape[1] * shape[2];
  int64_t E[3];
  double bx[3];
  DevBuf vin, cout;
  const double2* vdev = reinterpret_cast<const double2*>(values);
  double2* cdev = reinterpret_cast<double2*>(coeffs_out);
  if (!on_device) {
    VFN_CHECK(vin.ensure(sizeof(double2) * n));
    VFN_CUDA(cudaMemcpyAsync(vin.ptr, values, sizeof(double2) * n, cudaMemcpyHostToDevice, s));
    vdev = vin.as<double2>();
    int64_t ne = n;
    for (int d = 0; d < 3; ++d) ne *= mirror[d] ? 2 : 1;
    VFN_CHECK(cout.ensure(sizeof(double2) * ne));
    cdev = cout.as<double2>();
  }
  VFN_CHECK(spectral_device(vdev, shape, a, b, mirror, cdev, E, bx, s));
  if (!on_device) {
    VFN_CUDA(cudaMemcpy(coeffs_out, cdev, sizeof(double2) * E[0] * E[1] * E[2], cudaMemcpyDeviceToHost));
  }
  return VFN_OK;
}

int vfn_tube_eval(vfn_tube** out, int device, const double* values, const int64_t shape[3],
                  const double a[3], const double b[3], const int mirror[3],
                  const double* thresholds, int nthr, int has_filter, double final_filter,
                  double sigma, int m, int64_t* count, int* no_seeds, void* stream) {
  vfn::NvtxRange nvtx_range("vfn tube_eval");
  if (!out || !values || !shape || !a || !b || !mirror || !thresholds || !count || !no_seeds)
    return fail(VFN_ERR_INVALID, "null argument");
  if (nthr < 1) return fail(VFN_ERR_INVALID, "thresholds must be a nonempty sequence of positive values");
  for (int i = 0; i < nthr; ++i)
    if (!(thresholds[i] > 0)) return fail(VFN_ERR_INVALID, "thresholds must be a nonempty sequence of positive values");
  *out = nullptr;
  *count = 0;
  *no_seeds = 0;
  DeviceGuard guard(device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool dbg = std::getenv("VFN_DEBUG_TUBE") != nullptr;
  double t_last = tube_now_ms();
  const int64_t n = shape[0] * shape[1] * shape[2];
  // per-device scratch and plan, reused across calls (calls on one device
  // are serialised by its mutex): no allocation churn after the first call
  TubeScratch* ts = tube_scratch(device);
  std::lock_guard<std::mutex> tube_lock(ts->mu);
  DevBuf &vin = ts->vin, &coeffs = ts->coeffs, &rho0 = ts->rho0, &flag = ts->flag, &pos = ts->pos,
         &tmp = ts->tmp, &idxA = ts->idxA, &idxB = ts->idxB, &rhoA = ts->rhoA, &rhoB = ts->rhoB,
         &coords = ts->coords, &vals = ts->vals, &keys = ts->keys, &keys2 = ts->keys2, &iota = ts->iota,
         &perm = ts->perm;
  int st = VFN_OK;
  VFN_CHECK(vin.ensure(sizeof(double2) * n));
  // host or device samples (UVA): a snapshot read straight into HBM skips the host
  VFN_CUDA(cudaMemcpyAsync(vin.ptr, values, sizeof(double2) * n, cudaMemcpyDefault, s));
  int64_t ne = n;
  for (int d = 0; d < 3; ++d) ne *= mirror[d] ? 2 : 1;
  VFN_CHECK(coeffs.ensure(sizeof(double2) * ne));
  int64_t E[3];
  double bx[3];
  TUBE_T("upload");
  VFN_CHECK(spectral_device(vin.as<double2>(), shape, a, b, mirror, coeffs.as<double2>(), E, bx, s));
  TUBE_T("spectral");

  // lattice at the finest spacing h / 3^L (tube.py:82-83); step like numpy: widths / lattice
  int64_t mult = 1;
  for (int i = 0; i < nthr; ++i) mult *= 3;
  Lattice L;
  for (int d = 0; d < 3; ++d) {
    L.size[d] = E[d] * mult;
    L.a[d] = a[d];
    L.step[d] = (bx[d] - a[d]) / (double)L.size[d];
  }

  // seeds from the stored samples (tube.py:85-98)
  VFN_CHECK(rho0.ensure(sizeof(double) * n));
  VFN_CHECK(flag.ensure(sizeof(int) * n));
  VFN_CHECK(pos.ensure(sizeof(int) * n));
  k_seed_flags<<<nblk(n), 256, 0, s>>>(vin.as<double2>(), n, thresholds[0], rho0.as<double>(), flag.as<int>());
  int64_t P = 0;
  VFN_CHECK(scan_count(flag.as<int>(), pos.as<int>(), n, tmp, &P, s));
  if (P == 0) {
    *no_seeds = 1;
    *out = new vfn_tube();
    (*out)->device = device;
    return VFN_OK;
  }
  VFN_CHECK(idxA.ensure(sizeof(longlong4) * P));
  VFN_CHECK(rhoA.ensure(sizeof(double) * P));
  k_seed_scatter<<<nblk(n), 256, 0, s>>>(flag.as<int>(), pos.as<int>(), rho0.as<double>(), n, shape[1],
                                         shape[2], mult, idxA.as<longlong4>(), rhoA.as<double>());
  VFN_CUDA(cudaGetLastError());

  TUBE_T("seeds");
  // the plan of the previous call is rebuilt in place when its geometry
  // matches (grid, tensor map, evaluate scratch and FFT buffer reused)
  bool same = ts->plan && ts->sigma == sigma && ts->m == m;
  for (int d = 0; d < 3 && same; ++d) same = ts->E[d] == E[d] && ts->a[d] == a[d] && ts->bx[d] == bx[d];
  if (same) {
    VFN_CHECK(build_grid(ts->plan, coeffs.as<double>(), s));
  } else {
    if (ts->plan) vfn_plan_destroy(ts->plan);
    ts->plan = nullptr;
    VFN_CHECK(vfn_plan_create(&ts->plan, device, E, a, bx, sigma, m, coeffs.as<double>(), 1, stream));
    ts->plan->keep_fftbuf = true;
    ts->sigma = sigma;
    ts->m = m;
    for (int d = 0; d < 3; ++d) {
      ts->E[d] = E[d];
      ts->a[d] = a[d];
      ts->bx[d] = bx[d];
    }
  }
  vfn_plan* plan = ts->plan;
  TUBE_T("plan");
  int64_t cur = P;  // points of the current generation (idxA, rhoA)
  bool emptied = false;
  for (int ell = 1; ell <= nthr && st == VFN_OK; ++ell) {
    // parents: rho <= threshold (tube.py:105-108)
    if ((st = flag.ensure(sizeof(int) * cur)) != VFN_OK) break;
    if ((st = pos.ensure(sizeof(int) * cur)) != VFN_OK) break;
    k_keep_flags<<<nblk(cur), 256, 0, s>>>(rhoA.as<double>(), cur, thresholds[ell - 1], flag.as<int>());
    int64_t np_ = 0;
    if ((st = scan_count(flag.as<int>(), pos.as<int>(), cur, tmp, &np_, s)) != VFN_OK) break;
    if (np_ == 0) {
      emptied = true;
      break;
    }
    if ((st = idxB.ensure(sizeof(longlong4) * np_)) != VFN_OK) break;
    k_compact<<<nblk(cur), 256, 0, s>>>(flag.as<int>(), pos.as<int>(), cur, idxA.as<longlong4>(),
                                       nullptr, idxB.as<longlong4>(), nullptr);
    // children (tube.py:109-115) and their densities through the reused plan (:116-117)
    const int64_t nk = 27 * np_;
    int64_t stride = 1;
    for (int i = 0; i < nthr - ell; ++i) stride *= 3;
    if ((st = idxA.ensure(sizeof(longlong4) * nk)) != VFN_OK) break;
    if ((st = coords.ensure(sizeof(double) * 3 * nk)) != VFN_OK) break;
    if ((st = vals.ensure(sizeof(double2) * nk)) != VFN_OK) break;
    if ((st = rhoA.ensure(sizeof(double) * nk)) != VFN_OK) break;
    k_children<<<nblk(nk), 256, 0, s>>>(idxB.as<longlong4>(), np_, stride, ell, L,
                                        idxA.as<longlong4>(), coords.as<double>());
    int64_t bad = -1;
    st = vfn_plan_eval(plan, coords.as<double>(), nk, vals.as<double>(), 1, &bad, stream);
    if (st != VFN_OK) break;
    k_rho<<<nblk(nk), 256, 0, s>>>(vals.as<double2>(), nk, rhoA.as<double>());
    cur = nk;
    TUBE_T("pass");
  }
  TUBE_T("passes done");
  if (st != VFN_OK) return st;
  vfn_tube* t = new vfn_tube();
  t->device = device;
  if (emptied) {
    *out = t;
    return VFN_OK;
  }
  // final filter (tube.py:119-121)
  if (has_filter) {
    VFN_CHECK(flag.ensure(sizeof(int) * cur));
    VFN_CHECK(pos.ensure(sizeof(int) * cur));
    k_keep_flags<<<nblk(cur), 256, 0, s>>>(rhoA.as<double>(), cur, final_filter, flag.as<int>());
    int64_t kept = 0;
    VFN_CHECK(scan_count(flag.as<int>(), pos.as<int>(), cur, tmp, &kept, s));
    VFN_CHECK(idxB.ensure(sizeof(longlong4) * (kept + 1)));
    VFN_CHECK(rhoB.ensure(sizeof(double) * (kept + 1)));
    k_compact<<<nblk(cur), 256, 0, s>>>(flag.as<int>(), pos.as<int>(), cur, idxA.as<longlong4>(),
                                       rhoA.as<double>(), idxB.as<longlong4>(), rhoB.as<double>());
    std::swap(idxA.ptr, idxB.ptr);
    std::swap(idxA.bytes, idxB.bytes);
    std::swap(rhoA.ptr, rhoB.ptr);
    std::swap(rhoA.bytes, rhoB.bytes);
    cur = kept;
  }
  if (cur == 0) {
    *out = t;
    return VFN_OK;
  }
  // lexicographic lattice order (tube.py:125-127); keys are unique
  VFN_CHECK(keys.ensure(sizeof(unsigned long long) * cur));
  VFN_CHECK(keys2.ensure(sizeof(unsigned long long) * cur));
  VFN_CHECK(iota.ensure(sizeof(int) * cur));
  VFN_CHECK(perm.ensure(sizeof(int) * cur));
  k_keys<<<nblk(cur), 256, 0, s>>>(idxA.as<longlong4>(), cur, L, keys.as<unsigned long long>(), iota.as<int>());
  // only the bits the lattice keys can use (~31 for a 1152^3 lattice): half
  // the radix passes of a full 64-bit sort
  int key_bits = 1;
  {
    const double span = (double)L.size[0] * (double)L.size[1] * (double)L.size[2];
    while (key_bits < 64 && std::ldexp(1.0, key_bits) < span) ++key_bits;
  }
  size_t bytes = 0;
  VFN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.as<unsigned long long>(),
                                           keys2.as<unsigned long long>(), iota.as<int>(),
                                           perm.as<int>(), (int)cur, 0, key_bits, s));
  VFN_CHECK(tmp.ensure(bytes));
  VFN_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, bytes, keys.as<unsigned long long>(),
                                           keys2.as<unsigned long long>(), iota.as<int>(),
                                           perm.as<int>(), (int)cur, 0, key_bits, s));
  VFN_CHECK(t->points.ensure(sizeof(double) * 3 * cur));
  VFN_CHECK(t->density.ensure(sizeof(double) * cur));
  VFN_CHECK(t->level.ensure(sizeof(int64_t) * cur));
  k_emit<<<nblk(cur), 256, 0, s>>>(perm.as<int>(), idxA.as<longlong4>(), rhoA.as<double>(), cur, L,
                                   t->points.as<double>(), t->density.as<double>(),
                                   t->level.as<int64_t>());
  VFN_CUDA(cudaGetLastError());
  VFN_CUDA(cudaStreamSynchronize(s));
  TUBE_T("sort+emit");
  t->count = cur;
  *count = cur;
  *out = t;
  return VFN_OK;
}

int vfn_tube_copy(const vfn_tube* t, double* points, double* density, int64_t* level) {
  if (!t) return fail(VFN_ERR_INVALID, "null tube");
  if (t->count == 0) return VFN_OK;
  if (!points || !density || !level) return fail(VFN_ERR_INVALID, "null argument");
  DeviceGuard guard(t->device);
  const size_t nb[3] = {sizeof(double) * 3 * t->count, sizeof(double) * t->count, sizeof(int64_t) * t->count};
  const void* src[3] = {t->points.ptr, t->density.ptr, t->level.ptr};
  void* dst[3] = {points, density, level};
  const size_t total = nb[0] + nb[1] + nb[2];
  if (total < ((size_t)1 << 20)) {
    for (int i = 0; i < 3; ++i) VFN_CUDA(cudaMemcpy(dst[i], src[i], nb[i], cudaMemcpyDeviceToHost));
    return VFN_OK;
  }
  // Large clouds (the caller's arrays are fresh pageable numpy memory): D2H
  // at pinned speed into a per-device grow-only staging buffer, then copy
  // out with several host threads (the page faults of the fresh arrays
  // dominate a single-threaded copy)
  struct Stage {
    std::mutex mu;
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  static std::mutex smu;
  static std::map<int, Stage*> stages;
  Stage* st;
  {
    std::lock_guard<std::mutex> lock(smu);
    Stage*& slot = stages[t->device];
    if (!slot) slot = new Stage();
    st = slot;
  }
  std::lock_guard<std::mutex> lock(st->mu);
  if (st->bytes < total) {
    if (st->ptr) cudaFreeHost(st->ptr);
    st->ptr = nullptr;
    st->bytes = 0;
    if (cudaMallocHost(&st->ptr, total) != cudaSuccess) {
      cudaGetLastError();
      st->ptr = nullptr;
      for (int i = 0; i < 3; ++i) VFN_CUDA(cudaMemcpy(dst[i], src[i], nb[i], cudaMemcpyDeviceToHost));
      return VFN_OK;
    }
    st->bytes = total;
  }
  char* stg = static_cast<char*>(st->ptr);
  size_t off[3] = {0, nb[0], nb[0] + nb[1]};
  for (int i = 0; i < 3; ++i) VFN_CUDA(cudaMemcpyAsync(stg + off[i], src[i], nb[i], cudaMemcpyDeviceToHost, 0));
  VFN_CUDA(cudaStreamSynchronize(0));
  const int nt = (int)std::min<size_t>(8, std::max(1u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int k = 0; k < nt; ++k)
    th.emplace_back([&, k] {
      for (int i = 0; i < 3; ++i) {
        const size_t lo = nb[i] * k / nt, hi = nb[i] * (k + 1) / nt;
        std::memcpy(static_cast<char*>(dst[i]) + lo, stg + off[i] + lo, hi - lo);
      }
    });
  for (auto& x : th) x.join();
  return VFN_OK;
}

int vfn_tube_destroy(vfn_tube* t) {
  if (!t) return VFN_OK;
  {
    DeviceGuard guard(t->device);
    t->points.release();
    t->density.release();
    t->level.release();
  }
  delete t;
  return VFN_OK;
}

}  // extern "C"
