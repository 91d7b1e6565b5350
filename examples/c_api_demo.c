/* Plain-C use of the C ABI (include/vfnfft.h), no Python or torch:
 * build a plan for a small random spectrum, evaluate scattered points,
 * compare with the exact sum (vfn_direct_eval), and show the error path.
 *
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_1605_01244_b200 -lvfnfft \
 *       -Wl,-rpath,$PWD/paper_1605_01244_b200 -lm -o c_api_demo && ./c_api_demo
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "vfnfft.h"

static double urand(unsigned long long* s) {
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return (double)(*s >> 11) / 9007199254740992.0;
}

int main(void) {
  const int64_t N[3] = {16, 24, 12};
  const double a[3] = {-1.5, 0.25, 2.0}, b[3] = {2.5, 1.25, 7.0};
  const int64_t nc = N[0] * N[1] * N[2], M = 5000;
  double* coeffs = malloc(sizeof(double) * 2 * nc);
  double* pts = malloc(sizeof(double) * 3 * M);
  double* out = malloc(sizeof(double) * 2 * M);
  double* ref = malloc(sizeof(double) * 2 * M);
  unsigned long long seed = 12345;
  for (int64_t i = 0; i < 2 * nc; ++i) coeffs[i] = urand(&seed) - 0.5;
  for (int64_t i = 0; i < M; ++i)
    for (int d = 0; d < 3; ++d) pts[3 * i + d] = a[d] + (b[d] - a[d]) * urand(&seed);

  vfn_plan* plan = NULL;
  if (vfn_plan_create(&plan, 0, N, a, b, 2.0, 6, coeffs, 0, NULL) != VFN_OK) {
    fprintf(stderr, "plan: %s\n", vfn_last_error());
    return 1;
  }
  int64_t bad = -1;
  if (vfn_plan_eval(plan, pts, M, out, 0, &bad, NULL) != VFN_OK) {
    fprintf(stderr, "eval: %s\n", vfn_last_error());
    return 1;
  }
  if (vfn_direct_eval(0, N, a, b, coeffs, pts, M, ref, 0, &bad, NULL) != VFN_OK) {
    fprintf(stderr, "direct: %s\n", vfn_last_error());
    return 1;
  }
  double err = 0, mx = 0;
  for (int64_t i = 0; i < M; ++i) {
    double dr = out[2 * i] - ref[2 * i], di = out[2 * i + 1] - ref[2 * i + 1];
    err = fmax(err, sqrt(dr * dr + di * di));
    mx = fmax(mx, sqrt(ref[2 * i] * ref[2 * i] + ref[2 * i + 1] * ref[2 * i + 1]));
  }
  printf("%s: %lld points, max |nufft - direct| / max |direct| = %.3e\n", vfn_version(),
         (long long)M, err / mx);
  pts[3 * 17 + 1] = b[1];  /* the right endpoint is outside [a, b) */
  int st = vfn_plan_eval(plan, pts, M, out, 0, &bad, NULL);
  printf("outside point: status %d, first bad row %lld (%s)\n", st, (long long)bad, vfn_last_error());
  vfn_plan_destroy(plan);
  free(coeffs);
  free(pts);
  free(out);
  free(ref);
  return (err / mx < 1e-10 && st == VFN_ERR_OUTSIDE && bad == 17) ? 0 : 2;  /* 1e-10: north-star gate */
}
