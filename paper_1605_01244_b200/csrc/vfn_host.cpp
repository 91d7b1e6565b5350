// Host-side numerics of a plan: Kaiser-Bessel parameter, window transform
// table and the piecewise-polynomial window fit used by the gather kernels.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "vfn_internal.cuh"

namespace vfn {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

const char* last_error_cstr() { return g_last_error.c_str(); }

// beta = pi * sqrt((w/sigma)^2 (sigma - 1/2)^2 - 0.8), w = 2m+1  (nufft.py:152-156)
double kb_beta(int m, double sigma) {
  double w = 2.0 * m + 1.0;
  double r = (w / sigma);
  return M_PI * std::sqrt(r * r * (sigma - 0.5) * (sigma - 0.5) - 0.8);
}

// I0 by its power series in long double; all terms are positive, so the
// relative error stays at a few ulp for the arguments used here (|x| < 80).
static long double i0l(long double x) {
  long double q = x * x / 4.0L, term = 1.0L, sum = 1.0L;
  for (int k = 1; k < 500; ++k) {
    term *= q / ((long double)k * (long double)k);
    sum += term;
    if (term < sum * 1e-21L) break;
  }
  return sum;
}

double bessel_i0(double x) { return (double)i0l(x); }

// phi_hat(k) = 2 w / I0(beta) * { sinh(sqrt(beta^2 - t^2)) / sqrt(...)  (beta > |t|)
//                                { sinc branch otherwise },  t = 2 pi w k, w = (m+1/2)/n
// (nufft.py:167-176)
void kb_hat_table(int64_t N, int64_t n, int m, double beta, double* out) {
  const long double w = ((long double)m + 0.5L) / (long double)n;
  const long double i0b = i0l(beta);
  for (int64_t j = 0; j < N; ++j) {
    long double k = (long double)(j - N / 2);
    long double t = 2.0L * (long double)M_PI * w * k;
    long double d = (long double)beta * beta - t * t;
    long double r = std::sqrt(std::fabs(d));
    long double v;
    if (r == 0.0L)
      v = 1.0L;
    else if (d > 0)
      v = std::sinh(r) / r;
    else
      v = std::sin(r) / r;
    out[j] = (double)(2.0L * w * v / i0b);
  }
}

// Window value at signed cell distance v (nufft.py:159-164), long double.
static long double phi(long double v, int m, long double beta, long double i0b) {
  long double x = v / ((long double)m + 0.5L);
  long double arg = 1.0L - x * x;
  if (arg < 0) arg = 0;
  return i0l(beta * std::sqrt(arg)) / i0b;
}

// Chebyshev interpolation of phi(delta - c) on delta in [-1/2, 1/2] for
// c = j - m, converted to monomials in delta (Horner-evaluated on the GPU).
// The degree is the smallest one whose max error on a dense check grid is
// below 4e-15 (phi <= 1; a few ulp of Horner rounding), capped at max_deg.
static int fit_window_poly_uncached(int m, double beta, double* coef, int max_deg) {
  const long double i0b = i0l(beta);
  const int W = 2 * m + 1;
  int chosen = max_deg;
  std::vector<long double> best;
  for (int deg = 6; deg <= max_deg; ++deg) {
    std::vector<long double> all((size_t)W * (deg + 1));
    long double worst = 0;
    for (int j = 0; j < W; ++j) {
      const long double c = (long double)(j - m);
      const int K = deg + 1;
      // Chebyshev nodes in t in [-1, 1]; delta = t / 2
      std::vector<long double> f(K), ch(K, 0.0L);
      for (int i = 0; i < K; ++i) {
        long double t = std::cos((long double)M_PI * (i + 0.5L) / K);
        f[i] = phi(t / 2 - c, m, beta, i0b);
      }
      for (int k = 0; k < K; ++k) {
        long double s = 0;
        for (int i = 0; i < K; ++i)
          s += f[i] * std::cos((long double)M_PI * k * (i + 0.5L) / K);
        ch[k] = (k == 0 ? 1.0L : 2.0L) * s / K;
      }
      // Chebyshev -> monomial in t via the T_k recurrence
      std::vector<long double> Tkm1(K, 0), Tk(K, 0), mono(K, 0);
      Tkm1[0] = 1;        // T0
      if (K > 1) Tk[1] = 1;  // T1
      for (int i = 0; i < K; ++i) mono[i] += ch[0] * Tkm1[i];
      if (K > 1)
        for (int i = 0; i < K; ++i) mono[i] += ch[1] * Tk[i];
      for (int k = 2; k < K; ++k) {
        std::vector<long double> Tn(K, 0);
        for (int i = 0; i < K; ++i) {
          if (i > 0) Tn[i] += 2 * Tk[i - 1];
          Tn[i] -= Tkm1[i];
        }
        for (int i = 0; i < K; ++i) mono[i] += ch[k] * Tn[i];
        Tkm1 = Tk;
        Tk = Tn;
      }
      // t = 2 delta  ->  coefficient of delta^i is mono[i] * 2^i
      long double scale = 1;
      for (int i = 0; i < K; ++i) {
        all[(size_t)j * K + i] = mono[i] * scale;
        scale *= 2;
      }
      // check in double arithmetic (what the GPU does)
      for (int s = 0; s <= 400; ++s) {
        double dl = -0.5 + s / 400.0;
        double acc = (double)all[(size_t)j * K + deg];
        for (int i = deg - 1; i >= 0; --i) acc = std::fma(acc, dl, (double)all[(size_t)j * K + i]);
        long double e = std::fabs((long double)acc - phi(dl - c, m, beta, i0b));
        if (e > worst) worst = e;
      }
    }
    best = all;
    chosen = deg;
    if (std::getenv("VFN_DEBUG_FIT")) fprintf(stderr, "fit m=%d deg=%d err=%.3Le\n", m, deg, worst);
    if (worst < 4e-15L) break;
  }
  for (size_t i = 0; i < best.size(); ++i) coef[i] = (double)best[i];
  return chosen;
}

// The fit costs milliseconds of long-double work and depends only on
// (m, beta, max_deg): cached process-wide, so repeated plans (tube_eval, a
// plan per snapshot) skip it.
int fit_window_poly(int m, double beta, double* coef, int max_deg) {
  struct Fit {
    int deg;
    std::vector<double> coef;
  };
  static std::mutex mu;
  static std::map<std::tuple<int, double, int>, Fit> cache;
  const auto key = std::make_tuple(m, beta, max_deg);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      std::copy(it->second.coef.begin(), it->second.coef.end(), coef);
      return it->second.deg;
    }
  }
  Fit f;
  f.deg = fit_window_poly_uncached(m, beta, coef, max_deg);
  f.coef.assign(coef, coef + (size_t)(2 * m + 1) * (f.deg + 1));
  std::lock_guard<std::mutex> lock(mu);
  cache.emplace(key, std::move(f));
  return cache.find(key)->second.deg;
}

}  // namespace vfn
