// K5: rectilinear tensor-grid evaluation (rectilinear.py:47-64) as three
// exact separable 1D non-uniform passes.  Each pass contracts one mode with
// its basis matrix E_d[m, k] = exp(2 pi i (y_m - a)(k - N/2)/(b - a))/sqrt(b - a)
// (rectilinear.py:22-44), generated on the device; the contractions are plain
// complex GEMMs (cuBLAS ZGEMM, FP64 tensor-core DMMA on sm_100a).
#include <cublas_v2.h>

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

// One cuBLAS handle per (host thread, device): a handle carries its stream
// (cublasSetStream), so rectilinear and direct calls running concurrently on
// one device from different threads must not share it.
cublasHandle_t handle_for(int device) {
  struct Handles {
    std::map<int, cublasHandle_t> h;
    ~Handles() {
      for (auto& kv : h) cublasDestroy(kv.second);
    }
  };
  thread_local Handles handles;
  auto it = handles.h.find(device);
  if (it != handles.h.end()) return it->second;
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
  cublasSetMathMode(h, CUBLAS_DEFAULT_MATH);
  handles.h[device] = h;
  return h;
}

void* blas_handle(int device) { return handle_for(device); }

#define VFN_BLAS(expr)                                                                        \
  do {                                                                                        \
    cublasStatus_t _b = (expr);                                                               \
    if (_b != CUBLAS_STATUS_SUCCESS) {                                                        \
      st = fail(VFN_ERR_CUBLAS, std::string(#expr) + " failed (" + std::to_string((int)_b) + ")"); \
      goto done;                                                                              \
    }                                                                                         \
  } while (0)

// Host outputs: pass 3 runs in kRectSlabs slabs of output rows (m0), each
// slab's D2H on a copy stream overlapping the next slab's GEMM.
constexpr int kRectSlabs = 8;

int rect_eval(int device, const int64_t nm[3], const double a[3], const double b[3],
              const double* coeffs, const double* y[3], const int64_t Mv[3], double* out,
              int on_device, cudaStream_t s) {
  cublasHandle_t h = handle_for(device);
  if (!h) return fail(VFN_ERR_CUBLAS, "cublasCreate failed");
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
  const double2 one = make_double2(1.0, 0.0), zero = make_double2(0.0, 0.0);
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
    if ((st = E[d].ensure(eb[d])) != VFN_OK) goto done;
    {
      int64_t tot = Mv[d] * nm[d];
      k_basis<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(yd[d], Mv[d], nm[d], a[d], b[d] - a[d],
                                                           E[d].as<double2>());
    }
  }
  if ((st = T1.ensure(t1b)) != VFN_OK) goto done;
  if ((st = T2.ensure(t2b)) != VFN_OK) goto done;
  VFN_BLAS(cublasSetStream(h, s));
  {
    auto* e0 = reinterpret_cast<const cuDoubleComplex*>(E[0].ptr);
    auto* e1 = reinterpret_cast<const cuDoubleComplex*>(E[1].ptr);
    auto* e2 = reinterpret_cast<const cuDoubleComplex*>(E[2].ptr);
    auto* al = reinterpret_cast<const cuDoubleComplex*>(&one);
    auto* be = reinterpret_cast<const cuDoubleComplex*>(&zero);
    // pass 1, mode 3: T1 (N0N1 x M2) = C (N0N1 x N2) E2^T
    VFN_BLAS(cublasZgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)M2, (int)(N0 * N1), (int)N2, al, e2,
                         (int)N2, reinterpret_cast<const cuDoubleComplex*>(Cd), (int)N2, be,
                         T1.as<cuDoubleComplex>(), (int)M2));
    // pass 2, mode 2 (batched over n0): T2_n0 (M1 x M2) = E1 (M1 x N1) T1_n0 (N1 x M2)
    VFN_BLAS(cublasZgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)M2, (int)M1, (int)N1, al,
                                       T1.as<cuDoubleComplex>(), (int)M2, N1 * M2, e1, (int)N1, 0,
                                       be, T2.as<cuDoubleComplex>(), (int)M2, M1 * M2, (int)N0));
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
      VFN_BLAS(cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)(M1 * M2), (int)n, (int)N0, al,
                           T2.as<cuDoubleComplex>(), (int)(M1 * M2), e0 + lo * N0, (int)N0, be,
                           reinterpret_cast<cuDoubleComplex*>(Fd) + lo * M1 * M2, (int)(M1 * M2)));
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
  {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = fail(VFN_ERR_CUDA, std::string("rectilinear: ") + cudaGetErrorString(e));
  }
done:
  return st;
}

}  // namespace vfn
