// K6: exact NDFT (nufft.py:129-149) on the device — the reference's
// eval_direct, O(N1 N2 N3) complex MACs per point.  Thread per point; the
// per-axis exponentials e_d[k] = exp(2 pi i k t_d), k = j - N_d/2, are formed
// with sincospi in a per-thread table; the sum runs axis 3 innermost.
#include <string>

#include "vfn_device.cuh"

namespace vfn {

constexpr int kDirectMaxN = 1024;

__global__ void k_direct(const double2* __restrict__ c, int N0, int N1, int N2,
                         const double* __restrict__ pts, int64_t M, TorusMap tm, double norm,
                         double2* __restrict__ out, unsigned long long* __restrict__ bad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  double2 e[3][kDirectMaxN / 4];  // chunked below when N_d is larger
  double t[3];
  bool ok = true;
  for (int d = 0; d < 3; ++d) {
    double x = pts[3 * i + d];
    ok = ok && inside(x, tm.a[d], tm.b[d]);
    t[d] = (x - tm.a[d]) / (tm.b[d] - tm.a[d]);
  }
  if (!ok) {
    atomicMin(bad, (unsigned long long)i);
    return;
  }
  const int Nd[3] = {N0, N1, N2};
  // tables for axes 0 and 1 (<= 256 entries each in registers/local memory);
  // axis 2 phases are rebuilt per chunk
  for (int d = 0; d < 2; ++d)
    for (int j = 0; j < Nd[d] && j < kDirectMaxN / 4; ++j) {
      double s, co;
      sincospi(2.0 * (double)(j - Nd[d] / 2) * t[d], &s, &co);
      e[d][j] = make_double2(co, s);
    }
  double ar = 0.0, ai = 0.0;
  for (int j0 = 0; j0 < N0; ++j0) {
    double2 e0;
    if (j0 < kDirectMaxN / 4) e0 = e[0][j0];
    else { double s, co; sincospi(2.0 * (double)(j0 - N0 / 2) * t[0], &s, &co); e0 = make_double2(co, s); }
    double br = 0.0, bi = 0.0;
    for (int j1 = 0; j1 < N1; ++j1) {
      double2 e1;
      if (j1 < kDirectMaxN / 4) e1 = e[1][j1];
      else { double s, co; sincospi(2.0 * (double)(j1 - N1 / 2) * t[1], &s, &co); e1 = make_double2(co, s); }
      const double2* row = c + ((int64_t)j0 * N1 + j1) * N2;
      double cr = 0.0, ci = 0.0;
      for (int j2 = 0; j2 < N2; ++j2) {
        double s, co;
        sincospi(2.0 * (double)(j2 - N2 / 2) * t[2], &s, &co);
        double2 v = row[j2];
        cr += v.x * co - v.y * s;
        ci += v.x * s + v.y * co;
      }
      br += e1.x * cr - e1.y * ci;
      bi += e1.x * ci + e1.y * cr;
    }
    ar += e0.x * br - e0.y * bi;
    ai += e0.x * bi + e0.y * br;
  }
  out[i] = make_double2(ar * norm, ai * norm);
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
    if (nm[d] <= 0 || nm[d] % 2 != 0 || nm[d] > kDirectMaxN)
      return fail(VFN_ERR_INVALID, "direct sum needs even mode counts in 2..1024");
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
  const size_t cb = sizeof(double2) * nm[0] * nm[1] * nm[2];
  DevBuf C, P, O, B;
  const double2* cd = reinterpret_cast<const double2*>(coeffs);
  const double* pd = points;
  double2* od = reinterpret_cast<double2*>(out);
  if (!on_device) {
    VFN_CHECK(C.ensure(cb));
    VFN_CHECK(P.ensure(sizeof(double) * 3 * M));
    VFN_CHECK(O.ensure(sizeof(double2) * M));
    VFN_CUDA(cudaMemcpyAsync(C.ptr, coeffs, cb, cudaMemcpyHostToDevice, s));
    VFN_CUDA(cudaMemcpyAsync(P.ptr, points, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, s));
    cd = C.as<double2>();
    pd = P.as<double>();
    od = O.as<double2>();
  }
  VFN_CHECK(B.ensure(sizeof(unsigned long long)));
  const unsigned long long sentinel = ~0ull;
  VFN_CUDA(cudaMemcpyAsync(B.ptr, &sentinel, sizeof(sentinel), cudaMemcpyHostToDevice, s));
  k_direct<<<(unsigned)((M + 63) / 64), 64, 0, s>>>(cd, (int)nm[0], (int)nm[1], (int)nm[2], pd, M,
                                                   tm, 1.0 / std::sqrt(vol), od,
                                                   B.as<unsigned long long>());
  VFN_CUDA(cudaGetLastError());
  if (!on_device) VFN_CUDA(cudaMemcpyAsync(out, od, sizeof(double2) * M, cudaMemcpyDeviceToHost, s));
  unsigned long long bad = sentinel;
  VFN_CUDA(cudaMemcpyAsync(&bad, B.ptr, sizeof(bad), cudaMemcpyDeviceToHost, s));
  VFN_CUDA(cudaStreamSynchronize(s));
  C.release(); P.release(); O.release(); B.release();
  if (bad != sentinel) {
    if (first_bad_row) *first_bad_row = (int64_t)bad;
    return fail(VFN_ERR_OUTSIDE, "point (row " + std::to_string(bad) + ") lies outside the domain");
  }
  return VFN_OK;
}
