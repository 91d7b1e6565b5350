// K5: rectilinear tensor-grid evaluation (rectilinear.py:47-64) as three
// exact separable 1D non-uniform passes.  Each pass contracts one mode with
// its basis matrix E_d[m, k] = exp(2 pi i (y_m - a)(k - N/2)/(b - a))/sqrt(b - a)
// (rectilinear.py:22-44), generated on the device; the contractions are
// complex GEMMs on the FP64 tensor cores (hand-written DMMA kernel,
// vfn_zgemm.cu).

#include <algorithm>
#include <map>
#include <mutex>

#include "vfn_internal.cuh"

namespace vfn {

__global__ void k_basis(const double* __restrict__ y, int64_t M, int64_t N, double a, double width,
                        double2* __restrict__ E) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  int64_t m = e / N;
  int64_t k = e % N - N / 2;
  // phase / pi = 2 (y - a) k / (b - a); sincospi reduces the argument exactly
  double t = (y[m] - a) / width;
  double s, c;
  sincospi(2.0 * t * (double)k, &s, &c);
  double r = rsqrt(width);
  E[e] = make_double2(c * r, s * r);
}

// Host outputs: pass 3 runs in kRectSlabs slabs of output rows (m0), each
// slab's D2H on a copy stream overlapping the next slab's GEMM.
constexpr int kRectSlabs = 8;

int rect_eval(int device, const int64_t nm[3], const double a[3], const double b[3],
              const double* coeffs, const double* y[3], const int64_t Mv[3], double* out,
              int on_device, cudaStream_t s, int nufft_m, double sigma) {
  const int64_t N0 = nm[0], N1 = nm[1], N2 = nm[2];
  const int64_t M0 = Mv[0], M1 = Mv[1], M2 = Mv[2];
  const size_t cb = sizeof(double2) * N0 * N1 * N2;
  const size_t t1b = sizeof(double2) * N0 * N1 * M2;
  const size_t t2b = sizeof(double2) * N0 * M1 * M2;
  const size_t fb = sizeof(double2) * M0 * M1 * M2;
  const size_t eb[3] = {sizeof(double2) * M0 * N0, sizeof(double2) * M1 * N1,
                        sizeof(double2) * M2 * N2};
  // grow-only scratch per device, reused across calls (one host thread at a time)
  struct Scratch {
    std::mutex mu;  // held for the whole call: one caller per device at a time
    DevBuf C, T1, T2, F, E[3], Y[3];
    cudaStream_t copy = nullptr;  // D2H of result slabs (host outputs)
    cudaEvent_t ev[kRectSlabs + 1] = {};
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
  DevBuf &C = sc->C, &T1 = sc->T1, &T2 = sc->T2, &F = sc->F;
  DevBuf* E = sc->E;
  DevBuf* Y = sc->Y;
  int st = VFN_OK;
  const double2* Cd = reinterpret_cast<const double2*>(coeffs);
  double2* Fd = reinterpret_cast<double2*>(out);
  const double* yd[3];
  if (!on_device) {
    if ((st = C.ensure(cb)) != VFN_OK) goto done;
    if (cb >= ((size_t)1 << 20) && is_pageable(coeffs)) {
      if ((st = stage_h2d(device_stager(device), C.ptr, coeffs, cb, s)) != VFN_OK) goto done;
    } else if (cudaMemcpyAsync(C.ptr, coeffs, cb, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      st = fail(VFN_ERR_CUDA, "coefficient upload failed");
      goto done;
    }
    Cd = C.as<double2>();
    if ((st = F.ensure(fb)) != VFN_OK) goto done;
    Fd = F.as<double2>();
  }
  for (int d = 0; d < 3; ++d) {
    yd[d] = y[d];
    if (!on_device) {
      if ((st = Y[d].ensure(sizeof(double) * Mv[d])) != VFN_OK) goto done;
      if (cudaMemcpyAsync(Y[d].ptr, y[d], sizeof(double) * Mv[d], cudaMemcpyHostToDevice, s) !=
          cudaSuccess) {
        st = fail(VFN_ERR_CUDA, "coordinate upload failed");
        goto done;
      }
      yd[d] = Y[d].as<double>();
    }
    if (nufft_m > 0) continue;  // NUFFT passes: no basis matrices
    if ((st = E[d].ensure(eb[d])) != VFN_OK) goto done;
    {
      int64_t tot = Mv[d] * nm[d];
      k_basis<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(yd[d], Mv[d], nm[d], a[d], b[d] - a[d],
                                                           E[d].as<double2>());
    }
  }
  if (nufft_m > 0) {
    // separable 1D-NUFFT passes (vfn_rect_nufft.cu), then the whole result out
    if ((st = rect_nufft_device(device, nm, a, b, sigma, nufft_m, Cd, yd, Mv, Fd, s)) != VFN_OK) goto done;
    if (!on_device) {
      if (fb >= ((size_t)1 << 20) && is_pageable(out)) {
        if ((st = stage_d2h(device_stager(device), out, Fd, fb, s)) != VFN_OK) goto done;
      } else if (cudaMemcpyAsync(out, Fd, fb, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
        st = fail(VFN_ERR_CUDA, "result download failed");
        goto done;
      }
    }
    goto finish;
  }
  if ((st = T1.ensure(t1b)) != VFN_OK) goto done;
  if ((st = T2.ensure(t2b)) != VFN_OK) goto done;
  {
    const double2* e0 = E[0].as<double2>();
    const double2* e1 = E[1].as<double2>();
    const double2* e2 = E[2].as<double2>();
    // pass 1, mode 3 (rectilinear.py:60): T1 (N0N1 x M2) = C (N0N1 x N2) E2^T
    {
      ZGemm g;
      g.M = N0 * N1, g.N = M2, g.K = N2;
      g.A = Cd, g.lda = N2;
      g.B = e2, g.ldb = N2, g.bt = true;
      g.C = T1.as<double2>(), g.ldc = M2;
      if ((st = zgemm(g, s)) != VFN_OK) goto done;
    }
    // pass 2, mode 2 (rectilinear.py:62), batched over n0:
    // T2_n0 (M1 x M2) = E1 (M1 x N1) T1_n0 (N1 x M2)
    {
      ZGemm g;
      g.M = M1, g.N = M2, g.K = N1;
      g.A = e1, g.lda = N1, g.sA = 0;
      g.B = T1.as<double2>(), g.ldb = M2, g.sB = N1 * M2;
      g.C = T2.as<double2>(), g.ldc = M2, g.sC = M1 * M2;
      g.batch = (int)N0;
      if ((st = zgemm(g, s)) != VFN_OK) goto done;
    }
    // pass 3, mode 1: F (M0 x M1M2) = E0 (M0 x N0) T2 (N0 x M1M2); rows
    // [lo, lo + n) of F use rows [lo, lo + n) of E0
    const int nslab = on_device ? 1 : (int)std::min<int64_t>(kRectSlabs, M0);
    if (!on_device && !sc->copy) {
      if (cudaStreamCreateWithFlags(&sc->copy, cudaStreamNonBlocking) != cudaSuccess) {
        st = fail(VFN_ERR_CUDA, "copy stream creation failed");
        goto done;
      }
      for (auto& e : sc->ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    // pageable host output (a fresh numpy array): every slab's GEMM is
    // enqueued first, then the slabs are staged out through pinned pieces
    // while the later GEMMs run
    const bool staged = !on_device && fb >= ((size_t)1 << 20) && is_pageable(out);
    for (int j = 0; j < nslab; ++j) {
      const int64_t lo = M0 * j / nslab, n = M0 * (j + 1) / nslab - lo;
      if (n == 0) continue;
      {
        // pass 3, mode 1 (rectilinear.py:64): rows [lo, lo + n) of
        // F (M0 x M1M2) = E0 (M0 x N0) T2 (N0 x M1M2)
        ZGemm g;
        g.M = n, g.N = M1 * M2, g.K = N0;
        g.A = e0 + lo * N0, g.lda = N0;
        g.B = T2.as<double2>(), g.ldb = M1 * M2;
        g.C = Fd + lo * M1 * M2, g.ldc = M1 * M2;
        if ((st = zgemm(g, s)) != VFN_OK) goto done;
      }
      if (!on_device) {
        cudaEventRecord(sc->ev[j], s);
        if (staged) continue;
        cudaStreamWaitEvent(sc->copy, sc->ev[j], 0);
        if (cudaMemcpyAsync(out + 2 * lo * M1 * M2, Fd + lo * M1 * M2, sizeof(double2) * n * M1 * M2,
                            cudaMemcpyDeviceToHost, sc->copy) != cudaSuccess) {
          st = fail(VFN_ERR_CUDA, "result download failed");
          goto done;
        }
      }
    }
    if (staged) {
      for (int j = 0; j < nslab; ++j) {
        const int64_t lo = M0 * j / nslab, n = M0 * (j + 1) / nslab - lo;
        if (n == 0) continue;
        cudaStreamWaitEvent(sc->copy, sc->ev[j], 0);
        if ((st = stage_d2h(device_stager(device), out + 2 * lo * M1 * M2, Fd + lo * M1 * M2,
                            sizeof(double2) * n * M1 * M2, sc->copy)) != VFN_OK)
          goto done;
      }
    }
    if (!on_device) {
      cudaEventRecord(sc->ev[kRectSlabs], sc->copy);
      cudaStreamWaitEvent(s, sc->ev[kRectSlabs], 0);
    }
  }
finish:
  {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = fail(VFN_ERR_CUDA, std::string("rectilinear: ") + cudaGetErrorString(e));
  }
done:
  return st;
}

}  // namespace vfn
