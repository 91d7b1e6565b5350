// K5, separable NUFFT mode: the rectilinear evaluation
// (rectilinear.py:47-64) as three passes of 1D type-2 NUFFTs, one per axis,
// instead of dense basis contractions.  A pass evaluates every line of its
// input along one axis — the 1D series sum_k c_k e^{2 pi i k t(y)} / sqrt(w)
// of N coefficients at the axis' M coordinates — with the reference's own
// NFFT algorithm restricted to one dimension (the 3D plan is its tensor
// product, nufft.py:197-272):
//   deconvolve by the window transform and zero-pad to n = sigma N
//   (nufft.py:219-241), forward FFT of length n (:242), then for each
//   coordinate the 2m+1 window-weighted grid values around its nearest cell
//   (:248-271, the same torus map and window polynomial fit as the gather).
// One fused kernel per pass: a CTA stages G lines in shared memory, runs
// the padded FFTs there (radix-2, in place, bit-reversed load, XOR-swizzled
// line layout, per-stage twiddle tables) and gathers
// the line's M values, so HBM sees only each pass's input and output
// (705 MB at config 4 against 1.5e10 FMA for the exact passes).
// Accuracy: the 3D trafo's, ~10^-(2m+1) per pass (m = 6: ~1e-13).
// Coverage: n = sigma N a power of two <= 4096 (else VFN_ERR_INVALID; the
// exact mode, vfn_rect_eval, covers every size).
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "vfn_device.cuh"

namespace vfn {

namespace rn {

constexpr int kThreads = 256;
constexpr int kChunk = 128;   // targets per weight-table chunk
constexpr int kMaxGridElems = 4096;  // G lines x n complex staged per CTA

struct Pass {
  const double2* X;
  double2* Y;
  int64_t B;          // line stride (1: lines are contiguous rows)
  int64_t nlines;     // A * B
  int N, n, logn, M, m, W, G, deg;
  const double* fac;  // N: (-1)^k / phihat(k) / n / sqrt(w)
  const int* l0;      // M: nearest cell of each coordinate (mod n), coordinates sorted
  const double* wts;  // M x W: window weights of each coordinate (sorted order)
  const int* perm;    // M: sorted position -> output index along the axis
  const int2* octs;   // ceil(M/8): (window start p_lo, k-chunks) of each octet of sorted targets
  const int* delta;   // M: target's stencil start relative to its octet's window
};

// Element x of a staged line lives at x ^ ((x >> 3) & 7): the radix-8
// round over contiguous groups of 8 (h = 1) then reads 8 different 16-byte
// bank groups per 8 lanes instead of one (8-way conflicts), while the
// later rounds and the gather's runs of 4 stay conflict-free.
__device__ __forceinline__ int swz(int x) { return x ^ ((x >> 3) & 7); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ROWS: B == 1, a line is a contiguous row of X / Y.  TC: the window gather
// as DMMAs — 8 sorted targets (M) x 8 lines (N) per tile, K = the octet's
// window — with 8 lines per CTA at a pitch of n + 4 complex (lines g and
// g + 1 in opposite bank halves: conflict-free B fragments); else a scalar
// 2m+1-tap loop per output (n > 1024, where 8 lines do not fit).
template <bool ROWS, bool TC>
__global__ void __launch_bounds__(kThreads) k_nufft_pass(const Pass P) {
  extern __shared__ __align__(16) unsigned char rsm[];
  const int n = P.n, G = P.G, W = P.W, N = P.N, ld = TC ? n + 4 : n + 1;
  double2* lines = reinterpret_cast<double2*>(rsm);
  double2* tw = lines + (size_t)G * ld;                     // n - 1 twiddles, per stage (below)
  double* wts = reinterpret_cast<double*>(tw + n);          // kChunk x W window weights
  int64_t* lin = reinterpret_cast<int64_t*>(wts + (TC ? 0 : kChunk * W));  // G: line offsets into X
  int64_t* lout = lin + G;                                  // G: line offsets into Y
  int* l0s = reinterpret_cast<int*>(lout + G);              // kChunk
  const int tid = threadIdx.x;
  const int64_t L0 = (int64_t)blockIdx.x * G;
  const int gh = (int)(P.nlines - L0 < G ? P.nlines - L0 : G);
  // stage of span L = 2^l: e^{-2 pi i q / L}, q < L/2, at tw[L/2 - 1 + q], so
  // the lanes of one butterfly round read consecutive entries (a single
  // n/2 table read at stride n/L conflicts up to 8-way).  -2q/L equals the
  // -2 (q n/L)/n of that table exactly: the same twiddle values.
  for (int t = tid; t < n - 1; t += kThreads) {
    const int l = 32 - __clz(t + 1);  // L = 2^l with L/2 - 1 <= t < L - 1
    const int q = t + 1 - (1 << (l - 1));
    double s, c;
    sincospi(-2.0 * (double)q / (double)(1 << l), &s, &c);
    tw[t] = make_double2(c, s);
  }
  for (int g = tid; g < gh; g += kThreads) {
    const int64_t L = L0 + g, a = L / P.B, b = L - a * P.B;
    lin[g] = a * N * P.B + b;
    lout[g] = a * P.M * P.B + b;
  }
  for (int i = tid; i < G * ld; i += kThreads) lines[i] = make_double2(0.0, 0.0);
  __syncthreads();
  // deconvolve + zero-pad (wavenumber k - N/2 at index (k - N/2) mod n),
  // stored bit-reversed for the in-place decimation-in-time FFT
  const int shift = 32 - P.logn;
  if (ROWS) {
    // warp per line, lanes along k: coalesced rows
    for (int g = tid >> 5; g < gh; g += kThreads / 32)
      for (int k = tid & 31; k < N; k += 32) {
        const double2 c = P.X[lin[g] + k];
        const double f = P.fac[k];
        const int pos = k - N / 2 < 0 ? k - N / 2 + n : k - N / 2;
        lines[g * ld + swz((int)(__brev((unsigned)pos) >> shift))] = make_double2(c.x * f, c.y * f);
      }
  } else {
    // lanes along lines (consecutive b): coalesced columns
    const int g = tid % G, k0 = tid / G, kst = kThreads / G;
    if (g < gh && tid < kst * G)
      for (int k = k0; k < N; k += kst) {
        const double2 c = P.X[lin[g] + (int64_t)k * P.B];
        const double f = P.fac[k];
        const int pos = k - N / 2 < 0 ? k - N / 2 + n : k - N / 2;
        lines[g * ld + swz((int)(__brev((unsigned)pos) >> shift))] = make_double2(c.x * f, c.y * f);
      }
  }
  __syncthreads();
  // radix-2 decimation in time, up to three stages per shared-memory round
  // trip: a thread loads the 2^t elements base + j + i h (i < 2^t) that
  // stages s .. s+t-1 combine and runs those butterflies in registers, with
  // exactly the radix-2 arithmetic and twiddles (bitwise the same result)
  for (int s = 1; s <= P.logn; s += 3) {
    const int t = min(3, P.logn - s + 1), q = 1 << t, h = 1 << (s - 1);
    const int per_line = n >> t;  // work items per line
    for (int it = tid; it < gh * per_line; it += kThreads) {
      const int g = it / per_line, r = it - g * per_line;
      const int j = r & (h - 1), base = (r >> (s - 1)) << (s - 1 + t);
      double2* x = lines + g * ld;
      const int x0 = base + j;
      double2 e[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < q) e[i] = x[swz(x0 + i * h)];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        if (u >= t) break;
        const int step = 1 << u;
        const double2* twl = tw + (h << u) - 1;  // span L = 2^(s+u) = 2 h 2^u
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i >= q || (i & step)) continue;
          const double2 w = twl[j + (i & (step - 1)) * h];
          const double2 a = e[i], b = e[i + step];
          const double vr = fma(b.x, w.x, -b.y * w.y), vi = fma(b.x, w.y, b.y * w.x);
          e[i] = make_double2(a.x + vr, a.y + vi);
          e[i + step] = make_double2(a.x - vr, a.y - vi);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < q) x[swz(x0 + i * h)] = e[i];
    }
    __syncthreads();
  }
  if constexpr (TC) {
    // C[t, line] = sum_k A[t, k] G[line, p_lo + k] over the octet's window:
    // lane (g, tig) holds A[target g][k = 4 kc + tig], B[k][line g] and
    // C[target g][lines 2 tig, 2 tig + 1]
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tig = lane & 3;
    const int noct = (P.M + 7) >> 3;
    for (int o = warp; o < noct; o += kThreads / 32) {
      const int2 oc = P.octs[o];
      const int t = 8 * o + g;
      const bool vt = t < P.M;
      const int dlt = vt ? P.delta[t] : (1 << 30);
      const double* wt = P.wts + (int64_t)(vt ? t : 0) * W;
      const double2* xl = lines + g * ld;
      double r0 = 0.0, r1 = 0.0, i0 = 0.0, i1 = 0.0;
      for (int kc = 0; kc < oc.y; ++kc) {
        const int k = 4 * kc + tig, ow = k - dlt;
        const double a = (ow >= 0 && ow < W) ? __ldg(wt + ow) : 0.0;
        const double2 v = xl[swz((oc.x + k) & (n - 1))];
        dmma(r0, r1, a, v.x);
        dmma(i0, i1, a, v.y);
      }
      if (vt) {
        const int64_t col = ROWS ? (int64_t)P.perm[t] : (int64_t)P.perm[t] * P.B;
        if (2 * tig < gh) P.Y[lout[2 * tig] + col] = make_double2(r0, i0);
        if (2 * tig + 1 < gh) P.Y[lout[2 * tig + 1] + col] = make_double2(r1, i1);
      }
    }
    return;
  } else {
  // gather: value_j = sum_o w_o(delta_j) g[(l0_j + o - m) mod n]
  for (int j0 = 0; j0 < P.M; j0 += kChunk) {
    const int nj = min(kChunk, P.M - j0);
    for (int e = tid; e < nj * W; e += kThreads) wts[e] = P.wts[(int64_t)j0 * W + e];
    for (int j = tid; j < nj; j += kThreads) l0s[j] = ((P.l0[j0 + j] - P.m) % n + n) % n;
    __syncthreads();
    if (ROWS) {
      for (int g = tid >> 5; g < gh; g += kThreads / 32) {
        const double2* x = lines + g * ld;
        for (int j = tid & 31; j < nj; j += 32) {
          const double* w = wts + j * W;
          int p = l0s[j];
          double ar = 0.0, ai = 0.0;
          for (int o = 0; o < W; ++o) {
            const double2 v = x[swz(p)];
            ar = fma(w[o], v.x, ar);
            ai = fma(w[o], v.y, ai);
            p = p + 1 == n ? 0 : p + 1;
          }
          P.Y[lout[g] + P.perm[j0 + j]] = make_double2(ar, ai);
        }
      }
    } else {
      const int g = tid % G, jj = tid / G, jst = kThreads / G;
      if (g < gh && tid < jst * G) {
        const double2* x = lines + g * ld;
        for (int j = jj; j < nj; j += jst) {
          const double* w = wts + j * W;
          int p = l0s[j];
          double ar = 0.0, ai = 0.0;
          for (int o = 0; o < W; ++o) {
            const double2 v = x[swz(p)];
            ar = fma(w[o], v.x, ar);
            ai = fma(w[o], v.y, ai);
            p = p + 1 == n ? 0 : p + 1;
          }
          P.Y[lout[g] + (int64_t)P.perm[j0 + j] * P.B] = make_double2(ar, ai);
        }
      }
    }
    __syncthreads();
  }
  }
}

// perm = argsort(y) for M <= 4096 coordinates of one axis (one CTA, bitonic
// network in shared memory, ties by index); larger M keeps the input order
// (every order gives the same values, sorting only narrows the octets'
// windows).
constexpr int kSortMax = 4096;
__global__ void __launch_bounds__(1024) k_sort_coords(const double* __restrict__ y, int M, int* __restrict__ perm) {
  __shared__ double sy[kSortMax];
  __shared__ int si[kSortMax];
  if (M > kSortMax) {
    for (int j = threadIdx.x; j < M; j += blockDim.x) perm[j] = j;
    return;
  }
  int P2 = 1;
  while (P2 < M) P2 <<= 1;
  for (int j = threadIdx.x; j < P2; j += blockDim.x) {
    sy[j] = j < M ? y[j] : INFINITY;
    si[j] = j;
  }
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        const int l = i ^ jj;
        if (l > i) {
          const bool up = (i & k) == 0;
          const double a = sy[i], b = sy[l];
          const bool gt = a > b || (a == b && si[i] > si[l]);
          if (gt == up) {
            sy[i] = b;
            sy[l] = a;
            const int t = si[i];
            si[i] = si[l];
            si[l] = t;
          }
        }
      }
      __syncthreads();
    }
  for (int j = threadIdx.x; j < M; j += blockDim.x) perm[j] = si[j];
}

// Octets of sorted targets: the smallest circular window holding all eight
// stencils (start p_lo, K = 4 chunks) and each target's offset in it.
__global__ void k_axis_octets(const int* __restrict__ l0, int M, int n, int m, int2* __restrict__ octs,
                              int* __restrict__ delta) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (8 * o >= M) return;
  const int t0 = 8 * o, cnt = min(8, M - t0), ref = l0[t0], h = n / 2;
  int dmin = 0, dmax = 0, dd[8];
  for (int t = 0; t < cnt; ++t) {
    int d = l0[t0 + t] - ref;          // circular difference in [-n/2, n/2)
    d = ((d + h) % n + n) % n - h;
    dd[t] = d;
    dmin = min(dmin, d);
    dmax = max(dmax, d);
  }
  const int W = 2 * m + 1;
  const int p_lo = (((ref + dmin - m) % n) + n) % n;
  octs[o] = make_int2(p_lo, (dmax - dmin + W + 3) / 4);
  for (int t = 0; t < cnt; ++t) delta[t0 + t] = dd[t] - dmin;
}

// window weights of every coordinate of one axis, W per coordinate
__global__ void k_axis_weights(const double* __restrict__ dl, int M, const double* __restrict__ poly, int deg,
                               int W, double* __restrict__ wts) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * W) return;
  const int j = e / W, o = e - j * W;
  wts[e] = window_poly(poly, deg, o, dl[j]);
}

// nearest cell and offset of every coordinate of one axis (the gather's map)
__global__ void k_axis_targets(const double* __restrict__ y, const int* __restrict__ perm, int M, double a,
                               double amb, int n, int* __restrict__ l0, double* __restrict__ dl) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  double d;
  l0[j] = nearest_cell(y[perm[j]], a, amb, (double)n, n, d);
  dl[j] = d;
}

// All per-axis tables of one evaluate in ONE launch: CTA d builds axis d's
// sorted order, targets, octets and window weights, the same per-element
// arithmetic as the four kernels above (which remain for M > kSortMax
// coordinates per axis), with block barriers between the steps.
struct AxisJob {
  const double* y;
  int M, n;
  double a, amb;
  int* perm;
  int* l0;
  double* dl;
  int2* octs;
  int* delta;
  double* wts;
};
struct AxisJobs {
  AxisJob ax[3];
  const double* poly;
  int deg, W, m;
};

__global__ void __launch_bounds__(1024) k_axis_tables(const AxisJobs J) {
  __shared__ double sy[kSortMax];
  __shared__ int si[kSortMax];
  const AxisJob& q = J.ax[blockIdx.x];
  const int M = q.M, tid = threadIdx.x, nt = blockDim.x;
  // argsort(y), ties by index (k_sort_coords)
  int P2 = 1;
  while (P2 < M) P2 <<= 1;
  for (int j = tid; j < P2; j += nt) {
    sy[j] = j < M ? q.y[j] : INFINITY;
    si[j] = j;
  }
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = tid; i < P2; i += nt) {
        const int l = i ^ jj;
        if (l > i) {
          const bool up = (i & k) == 0;
          const double a = sy[i], b = sy[l];
          const bool gt = a > b || (a == b && si[i] > si[l]);
          if (gt == up) {
            sy[i] = b;
            sy[l] = a;
            const int t = si[i];
            si[i] = si[l];
            si[l] = t;
          }
        }
      }
      __syncthreads();
    }
  // targets (k_axis_targets); sy holds the sorted coordinates
  for (int j = tid; j < M; j += nt) {
    double d;
    q.perm[j] = si[j];
    q.l0[j] = nearest_cell(sy[j], q.a, q.amb, (double)q.n, q.n, d);
    q.dl[j] = d;
  }
  __syncthreads();
  // octets (k_axis_octets)
  const int W = J.W, n = q.n, h = n / 2;
  for (int o = tid; 8 * o < M; o += nt) {
    const int t0 = 8 * o, cnt = min(8, M - t0), ref = q.l0[t0];
    int dmin = 0, dmax = 0, dd[8];
    for (int t = 0; t < cnt; ++t) {
      int d = q.l0[t0 + t] - ref;
      d = ((d + h) % n + n) % n - h;
      dd[t] = d;
      dmin = min(dmin, d);
      dmax = max(dmax, d);
    }
    const int p_lo = (((ref + dmin - J.m) % n) + n) % n;
    q.octs[o] = make_int2(p_lo, (dmax - dmin + W + 3) / 4);
    for (int t = 0; t < cnt; ++t) q.delta[t0 + t] = dd[t] - dmin;
  }
  // weights (k_axis_weights)
  for (int e = tid; e < M * W; e += nt) {
    const int j = e / W, o = e - j * W;
    q.wts[e] = window_poly(J.poly, J.deg, o, q.dl[j]);
  }
}

size_t smem_bytes(int G, int n, int W, bool tc) {
  return sizeof(double2) * ((size_t)G * (tc ? n + 4 : n + 1) + n) + (tc ? 0 : sizeof(double) * kChunk * W) +
         sizeof(int64_t) * 2 * G + sizeof(int) * kChunk + 16;
}

}  // namespace rn

// The three NUFFT passes on device buffers: C (N0,N1,N2) -> F (M0,M1,M2).
int rect_nufft_device(int device, const int64_t nm[3], const double a[3], const double b[3], double sigma, int m,
                      const double2* C, const double* y[3], const int64_t Mv[3], double2* F, cudaStream_t s) {
  int64_t n[3];
  int logn[3];
  for (int d = 0; d < 3; ++d) {
    const double t = sigma * (double)nm[d];
    n[d] = (int64_t)std::llround(t);
    if (std::fabs(t - (double)n[d]) > 1e-9 || n[d] < nm[d] || (n[d] & (n[d] - 1)) || n[d] > rn::kMaxGridElems)
      return fail(VFN_ERR_INVALID, "NUFFT-mode rectilinear passes need sigma * N a power of two <= 4096 per axis "
                                   "(axis " + std::to_string(d) + ": " + std::to_string(t) + "); use the exact mode");
    logn[d] = 0;
    while ((int64_t)1 << logn[d] < n[d]) ++logn[d];
  }
  if (m < 1 || m > 13) return fail(VFN_ERR_INVALID, "cutoff must be in 1..13");
  const double beta = kb_beta(m, sigma);
  const int W = 2 * m + 1;
  std::vector<double> coef((size_t)W * 27);
  const int deg = fit_window_poly(m, beta, coef.data(), 26);
  // per-device scratch (one caller at a time per device)
  struct Scratch {
    std::mutex mu;
    DevBuf tables, T1, T2;
    // the fac / window-polynomial tables at the head of `tables` depend on
    // (modes, grid, m, sigma, box) only: kept across calls with the same key
    std::vector<double> key;
    const void* key_ptr = nullptr;
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
  // host tables: fac per axis, then the window fit
  const int64_t Ntot = nm[0] + nm[1] + nm[2], Mtot = Mv[0] + Mv[1] + Mv[2];
  const size_t hsize = (size_t)Ntot + (size_t)W * (deg + 1);
  std::vector<double> key{(double)nm[0], (double)nm[1], (double)nm[2], (double)n[0], (double)n[1], (double)n[2],
                          (double)m, sigma, a[0], a[1], a[2], b[0], b[1], b[2]};
  const int64_t noct = (Mv[0] + 7) / 8 + (Mv[1] + 7) / 8 + (Mv[2] + 7) / 8;
  const size_t tb = sizeof(double) * (hsize + Mtot + (size_t)Mtot * W) + sizeof(int) * (3 * Mtot + 4) +
                    sizeof(int2) * (noct + 4);
  VFN_CHECK(sc->tables.ensure(tb));
  if (sc->key != key || sc->key_ptr != sc->tables.ptr) {
    std::vector<double> h(hsize);
    double* f = h.data();
    for (int d = 0; d < 3; ++d) {
      kb_hat_table(nm[d], n[d], m, beta, f);
      const double nrm = 1.0 / (double)n[d] / std::sqrt(b[d] - a[d]);
      for (int64_t j = 0; j < nm[d]; ++j) {
        const int64_t k = j - nm[d] / 2;
        f[j] = ((k % 2 == 0) ? 1.0 : -1.0) / f[j] * nrm;  // (-1)^k: the torus map's half shift
      }
      f += nm[d];
    }
    std::copy(coef.begin(), coef.begin() + (size_t)W * (deg + 1), h.begin() + Ntot);
    VFN_CUDA(cudaMemcpyAsync(sc->tables.ptr, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, s));
    VFN_CUDA(cudaStreamSynchronize(s));  // h is a local
    sc->key = key;
    sc->key_ptr = sc->tables.ptr;
  }
  double* dfac = sc->tables.as<double>();
  double* dpoly = dfac + Ntot;
  double* ddl = dpoly + (size_t)W * (deg + 1);
  double* dw = ddl + Mtot;
  int2* doct = reinterpret_cast<int2*>(dw + (size_t)Mtot * W);
  int* dl0 = reinterpret_cast<int*>(doct + noct + 2);
  int* dperm = dl0 + Mtot;
  int* ddelta = dperm + Mtot;
  int64_t off_o[3];
  {
    int64_t off = 0, oo = 0;
    const bool fused = Mv[0] <= rn::kSortMax && Mv[1] <= rn::kSortMax && Mv[2] <= rn::kSortMax;
    rn::AxisJobs J;
    J.poly = dpoly;
    J.deg = deg;
    J.W = W;
    J.m = m;
    for (int d = 0; d < 3; ++d) {
      off_o[d] = oo;
      const int64_t no = (Mv[d] + 7) / 8;
      if (fused) {
        J.ax[d] = rn::AxisJob{y[d],        (int)Mv[d],  (int)n[d],    a[d],         a[d] - b[d], dperm + off,
                              dl0 + off,   ddl + off,   doct + oo,    ddelta + off, dw + off * W};
      } else {
        // the coordinates of each axis in sorted order (the DMMA gather takes 8
        // consecutive sorted targets per tile: their stencils overlap)
        rn::k_sort_coords<<<1, 1024, 0, s>>>(y[d], (int)Mv[d], dperm + off);
        VFN_CUDA(cudaGetLastError());
        rn::k_axis_targets<<<(unsigned)((Mv[d] + 255) / 256), 256, 0, s>>>(y[d], dperm + off, (int)Mv[d], a[d],
                                                                           a[d] - b[d], (int)n[d], dl0 + off, ddl + off);
        VFN_CUDA(cudaGetLastError());
        rn::k_axis_octets<<<(unsigned)((no + 127) / 128), 128, 0, s>>>(dl0 + off, (int)Mv[d], (int)n[d], m, doct + oo,
                                                                       ddelta + off);
        VFN_CUDA(cudaGetLastError());
        rn::k_axis_weights<<<(unsigned)((Mv[d] * W + 255) / 256), 256, 0, s>>>(ddl + off, (int)Mv[d], dpoly, deg, W,
                                                                                dw + off * W);
        VFN_CUDA(cudaGetLastError());
      }
      oo += no;
      off += Mv[d];
    }
    if (fused) {
      rn::k_axis_tables<<<3, 1024, 0, s>>>(J);
      VFN_CUDA(cudaGetLastError());
    }
  }
  VFN_CHECK(sc->T1.ensure(sizeof(double2) * nm[0] * nm[1] * Mv[2]));
  VFN_CHECK(sc->T2.ensure(sizeof(double2) * nm[0] * Mv[1] * Mv[2]));
  const int64_t off_f[3] = {0, nm[0], nm[0] + nm[1]};
  const int64_t off_t[3] = {0, Mv[0], Mv[0] + Mv[1]};
  // pass d: (A, N_d, B) -> (A, M_d, B)
  auto run = [&](int d, const double2* X, double2* Y, int64_t A, int64_t B) -> int {
    rn::Pass P;
    P.X = X;
    P.Y = Y;
    P.B = B;
    P.nlines = A * B;
    P.N = (int)nm[d];
    P.n = (int)n[d];
    P.logn = logn[d];
    P.M = (int)Mv[d];
    P.m = m;
    P.W = W;
    // lines per CTA: 8 for the DMMA gather (its N), which fits up to
    // n = 1024; else enough to amortise the twiddle / weight tables and few
    // enough for ~4 CTAs per SM (the FFT rounds are latency-bound)
    const bool tc = n[d] <= 1024 && !std::getenv("VFN_RECT_SCALAR");
    int64_t lpc = 8;
    if (const char* e = std::getenv("VFN_RECT_LINES")) lpc = std::max(1, std::atoi(e));
    P.G = tc ? 8 : (int)std::max<int64_t>(1, std::min<int64_t>(lpc, rn::kMaxGridElems / n[d]));
    if (B > 1 && !tc) P.G = (int)std::min<int64_t>(P.G, B);
    P.deg = deg;
    P.fac = dfac + off_f[d];
    P.l0 = dl0 + off_t[d];
    P.wts = dw + off_t[d] * W;
    P.perm = dperm + off_t[d];
    P.octs = doct + off_o[d];
    P.delta = ddelta + off_t[d];
    const size_t smem = rn::smem_bytes(P.G, P.n, W, tc);
    const int64_t blocks = (P.nlines + P.G - 1) / P.G;
    auto go = [&](auto kern) -> int {
      VFN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      // all of L1 as shared memory: the passes are occupancy-bound (3 CTAs
      // per SM under the default split at c4, 5 with the full carveout)
      VFN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      kern<<<(unsigned)blocks, rn::kThreads, smem, s>>>(P);
      VFN_CUDA(cudaGetLastError());
      return VFN_OK;
    };
    if (B == 1) return tc ? go(rn::k_nufft_pass<true, true>) : go(rn::k_nufft_pass<true, false>);
    return tc ? go(rn::k_nufft_pass<false, true>) : go(rn::k_nufft_pass<false, false>);
  };
  double2* T1 = sc->T1.as<double2>();
  double2* T2 = sc->T2.as<double2>();
  VFN_CHECK(run(2, C, T1, nm[0] * nm[1], 1));       // axis 3: rows of C
  VFN_CHECK(run(1, T1, T2, nm[0], Mv[2]));          // axis 2: (N0, N1, M2) -> (N0, M1, M2)
  VFN_CHECK(run(0, T2, F, 1, Mv[1] * Mv[2]));       // axis 1: (N0, M1 M2) -> (M0, M1 M2)
  return VFN_OK;
}

}  // namespace vfn
