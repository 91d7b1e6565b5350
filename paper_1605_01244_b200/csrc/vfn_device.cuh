// Device helpers shared by the kernels.
#pragma once
#include <cstdint>

#include "vfn_internal.cuh"

// Device-side bounds checks of the debug build (build.py --checks defines
// VFN_CHECKS; compute-sanitizer is unavailable on the GPU pool): a failed
// check prints its location and traps, failing the call with a CUDA error.
#ifdef VFN_CHECKS
#include <cstdio>
#define VFN_DCHECK(cond)                                                                   \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("VFN_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                           \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define VFN_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace vfn {

// zeta_d = mod((x - a) / (a - b), 1) - 1/2 with numpy's float remainder
// semantics (npy_divmod: fmod, then +b when the signs differ, +0.0 for an
// exact zero).  Every step is an explicitly rounded intrinsic so nvcc cannot
// contract it into an FMA: this must agree bit-for-bit with
// nufft.py:81-92 evaluated by numpy.
__device__ __forceinline__ double torus_coord(double x, double a, double amb) {
  double t = __ddiv_rn(__dsub_rn(x, a), amb);
  // fmod(t, 1) exactly: t - trunc(t) is exact for every finite t (the
  // fraction bits of t), NaN for +-inf like fmod; only the sign of an exact
  // zero differs, and zero is normalised to +0 below
  double r = __dsub_rn(t, trunc(t));
  if (r != 0.0) {
    if (r < 0.0) r = __dadd_rn(r, 1.0);
  } else {
    r = 0.0;
  }
  return __dsub_rn(r, 0.5);
}

// Nearest oversampled cell and fractional offset (nufft.py:249, :256-257):
//   z = zeta < 0 ? zeta + 1 : zeta;  u = z * n;  l0 = floor(u + 1/2)
// l0 may equal n; the cell index is l0 mod n and delta = u - l0 is kept
// relative to the unreduced l0, exactly like the reference's v = u - l0 - offs.
__device__ __forceinline__ int nearest_cell(double x, double a, double amb, double nd, int n,
                                            double& delta) {
  double zeta = torus_coord(x, a, amb);
  double z = zeta < 0.0 ? __dadd_rn(zeta, 1.0) : zeta;
  double u = __dmul_rn(z, nd);
  double l0 = floor(__dadd_rn(u, 0.5));
  delta = __dsub_rn(u, l0);
  if (!(l0 >= 0.0 && l0 <= nd)) {  // NaN / inf input: the call reports "outside";
    delta = 0.0;                    // keep every address in bounds meanwhile
    return 0;
  }
  int l = (int)l0;
  return l >= n ? l - n : l;
}

// u = z * n with z = zeta < 0 ? zeta + 1 : zeta (nufft.py:249, :256)
__device__ __forceinline__ double torus_u(double x, double a, double amb, double nd) {
  double zeta = torus_coord(x, a, amb);
  double z = zeta < 0.0 ? __dadd_rn(zeta, 1.0) : zeta;
  return __dmul_rn(z, nd);
}

// l0 = floor(u + 1/2) (nufft.py:257): cell = l0 mod n, delta = u - l0.
__device__ __forceinline__ int cell_from_u(double u, double nd, int n, double& delta) {
  double l0 = floor(__dadd_rn(u, 0.5));
  delta = __dsub_rn(u, l0);
  if (!(l0 >= 0.0 && l0 <= nd)) {
    delta = 0.0;
    return 0;
  }
  int l = (int)l0;
  return l >= n ? l - n : l;
}

__device__ __forceinline__ bool inside(double x, double a, double b) { return x >= a && x < b; }

// Horner evaluation of window polynomial j at delta.
__device__ __forceinline__ double window_poly(const double* __restrict__ coef, int deg, int j,
                                              double delta) {
  const double* c = coef + j * (deg + 1);
  double acc = c[deg];
  for (int i = deg - 1; i >= 0; --i) acc = fma(acc, delta, c[i]);
  return acc;
}

// window_poly of tap j at three deltas in one pass: three independent Horner
// chains per coefficient read (the same fma sequence per chain, so bitwise
// equal to three window_poly calls).
__device__ __forceinline__ void window_poly3(const double* __restrict__ coef, int deg, int j,
                                             const double dl[3], double w[3]) {
  const double* c = coef + j * (deg + 1);
  double a0 = c[deg], a1 = a0, a2 = a0;
  for (int i = deg - 1; i >= 0; --i) {
    const double ci = c[i];
    a0 = fma(a0, dl[0], ci);
    a1 = fma(a1, dl[1], ci);
    a2 = fma(a2, dl[2], ci);
  }
  w[0] = a0;
  w[1] = a1;
  w[2] = a2;
}

}  // namespace vfn
