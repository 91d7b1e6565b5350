// K6: exact NDFT (nufft.py:129-149) on the device — the reference's
// eval_direct, O(N1 N2 N3) complex MACs per point, as dense products on the
// FP64 tensor cores.  Per chunk of P points:
//   E_d[p, j] = exp(2 pi i k_j t_d(p)),  k_j = j - N_d/2,  t = (x - a)/(b - a)
//   T[p, (k0, k1)] = sum_k2 E_2[p, k2] C[k0, k1, k2]          (DMMA ZGEMM, vfn_zgemm.cu)
//   f[p] = norm * sum_k0 E_0[p, k0] sum_k1 E_1[p, k1] T[p, (k0, k1)]   (warp per point)
// — the reference's separable basis (nufft.py:141-148) with the axis-3 sum
// for all points of the chunk done as one complex GEMM on the FP64 tensor
// cores (hand-written, vfn_zgemm.cu).

#include <algorithm>
#include <map>
#include <mutex>
#include <string>

#include "vfn_device.cuh"

namespace vfn {

// basis rows of the chunk (p < P, all three axes) and the domain check
__global__ void k_direct_basis(const double* __restrict__ pts, int64_t P, int64_t row0, TorusMap tm,
                               int N0, int N1, int N2, double2* __restrict__ E0, double2* __restrict__ E1,
                               double2* __restrict__ E2, unsigned long long* __restrict__ bad) {
  const int64_t Ns = (int64_t)N0 + N1 + N2;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P * Ns) return;
  const int64_t p = e / Ns;
  int j = (int)(e % Ns), d = 0, N = N0;
  double2* E = E0;
  if (j >= N0) {
    j -= N0;
    d = 1;
    N = N1;
    E = E1;
    if (j >= N1) {
      j -= N1;
      d = 2;
      N = N2;
      E = E2;
    }
  }
  const double x = pts[3 * p + d];
  if (j == 0 && !inside(x, tm.a[d], tm.b[d])) atomicMin(bad, (unsigned long long)(row0 + p));
  const double t = (x - tm.a[d]) / (tm.b[d] - tm.a[d]);  // nufft.py:143
  double s, c;
  sincospi(2.0 * (double)(j - N / 2) * t, &s, &c);       // exp(2 pi i k t), exact argument reduction
  E[p * N + j] = make_double2(c, s);
}

// warp per point: f = norm * sum_k0 E0[k0] sum_k1 E1[k1] T[k0, k1]
__global__ void k_direct_reduce(const double2* __restrict__ T, const double2* __restrict__ E0,
                                const double2* __restrict__ E1, int64_t P, int N0, int N1, double norm,
                                double2* __restrict__ out) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= P) return;
  const double2* t = T + p * (int64_t)N0 * N1;
  double ar = 0.0, ai = 0.0;
  for (int k0 = 0; k0 < N0; ++k0) {
    double br = 0.0, bi = 0.0;
    for (int k1 = lane; k1 < N1; k1 += 32) {
      const double2 e = E1[p * N1 + k1], v = t[(int64_t)k0 * N1 + k1];
      br = fma(e.x, v.x, fma(-e.y, v.y, br));
      bi = fma(e.x, v.y, fma(e.y, v.x, bi));
    }
    const double2 e0 = E0[p * N0 + k0];
    ar = fma(e0.x, br, fma(-e0.y, bi, ar));
    ai = fma(e0.x, bi, fma(e0.y, br, ai));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ar += __shfl_xor_sync(0xffffffffu, ar, o);
    ai += __shfl_xor_sync(0xffffffffu, ai, o);
  }
  if (lane == 0) out[p] = make_double2(ar * norm, ai * norm);
}

}  // namespace vfn

using namespace vfn;

extern "C" int vfn_direct_eval(int device, const int64_t nm[3], const double a[3],
                               const double b[3], const double* coeffs, const double* points,
                               int64_t M, double* out, int on_device, int64_t* first_bad_row,
                               void* stream) {
  if (!nm || !a || !b || !coeffs || (M > 0 && (!points || !out)))
    return fail(VFN_ERR_INVALID, "null argument");
  if (first_bad_row) *first_bad_row = -1;
  for (int d = 0; d < 3; ++d)
    if (nm[d] <= 0 || nm[d] % 2 != 0 || nm[d] > (1 << 20))
      return fail(VFN_ERR_INVALID, "direct sum needs even, positive mode counts");
  if (M < 0) return fail(VFN_ERR_INVALID, "negative point count");
  if (M == 0) return VFN_OK;
  DeviceGuard guard(device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TorusMap tm;
  double vol = 1.0;
  for (int d = 0; d < 3; ++d) {
    tm.a[d] = a[d];
    tm.b[d] = b[d];
    tm.amb[d] = a[d] - b[d];
    vol *= b[d] - a[d];
  }
  const int N0 = (int)nm[0], N1 = (int)nm[1], N2 = (int)nm[2];
  const int64_t N01 = (int64_t)N0 * N1;
  const size_t cb = sizeof(double2) * N01 * N2;
  // chunk so the intermediate T (P x N0 N1 complex) stays near 1 GB
  const int64_t P = std::max<int64_t>(1, std::min<int64_t>(M, ((int64_t)1 << 26) / N01));
  // grow-only scratch per device, reused across calls (one host thread at a
  // time, like rect_eval): a 0.5-1 GB intermediate is not reallocated per call
  struct Scratch {
    std::mutex mu;  // held for the whole call: one caller per device at a time
    DevBuf C, Pt, O, B, E, T;
  };
  static std::mutex smu;
  static std::map<int, Scratch*> scratch;
  Scratch* sc;
  {
    std::lock_guard<std::mutex> lock(smu);
    Scratch*& slot = scratch[device];
    if (!slot) slot = new Scratch();
    sc = slot;
  }
  std::lock_guard<std::mutex> call_lock(sc->mu);
  DevBuf &C = sc->C, &Pt = sc->Pt, &O = sc->O, &B = sc->B, &E = sc->E, &T = sc->T;
  const double2* cd = reinterpret_cast<const double2*>(coeffs);
  const double* pd = points;
  double2* od = reinterpret_cast<double2*>(out);
  if (!on_device) {
    VFN_CHECK(C.ensure(cb));
    VFN_CHECK(Pt.ensure(sizeof(double) * 3 * M));
    VFN_CHECK(O.ensure(sizeof(double2) * M));
    VFN_CUDA(cudaMemcpyAsync(C.ptr, coeffs, cb, cudaMemcpyHostToDevice, s));
    VFN_CUDA(cudaMemcpyAsync(Pt.ptr, points, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, s));
    cd = C.as<double2>();
    pd = Pt.as<double>();
    od = O.as<double2>();
  }
  VFN_CHECK(B.ensure(sizeof(unsigned long long)));
  VFN_CHECK(E.ensure(sizeof(double2) * P * ((int64_t)N0 + N1 + N2)));
  VFN_CHECK(T.ensure(sizeof(double2) * P * N01));
  const unsigned long long sentinel = ~0ull;
  VFN_CUDA(cudaMemcpyAsync(B.ptr, &sentinel, sizeof(sentinel), cudaMemcpyHostToDevice, s));
  const double norm = 1.0 / std::sqrt(vol);
  for (int64_t lo = 0; lo < M; lo += P) {
    const int64_t n = std::min(P, M - lo);
    double2* E0 = E.as<double2>();
    double2* E1 = E0 + n * N0;
    double2* E2 = E1 + n * N1;
    const int64_t nb = n * ((int64_t)N0 + N1 + N2);
    k_direct_basis<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(pd + 3 * lo, n, lo, tm, N0, N1, N2, E0, E1, E2,
                                                                B.as<unsigned long long>());
    VFN_CUDA(cudaGetLastError());
    // T (n x N0N1) = E2 (n x N2) C^T, C read as (N0N1 x N2) row-major
    ZGemm g;
    g.M = n, g.N = N01, g.K = N2;
    g.A = E2, g.lda = N2;
    g.B = cd, g.ldb = N2, g.bt = true;
    g.C = T.as<double2>(), g.ldc = N01;
    VFN_CHECK(zgemm(g, s));
    k_direct_reduce<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(T.as<double2>(), E0, E1, n, N0, N1, norm,
                                                                      od + lo);
    VFN_CUDA(cudaGetLastError());
  }
  if (!on_device) VFN_CUDA(cudaMemcpyAsync(out, od, sizeof(double2) * M, cudaMemcpyDeviceToHost, s));
  unsigned long long bad = sentinel;
  VFN_CUDA(cudaMemcpyAsync(&bad, B.ptr, sizeof(bad), cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaStreamSynchronize(s));
  if (bad != sentinel) {
    if (first_bad_row) *first_bad_row = (int64_t)bad;
    return fail(VFN_ERR_OUTSIDE, "point (row " + std::to_string(bad) + ") lies outside the domain");
  }
  return VFN_OK;
}
