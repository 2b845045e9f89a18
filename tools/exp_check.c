#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
static double exp_nonpos(double x) {
  const double xc = x < -700.0 ? -700.0 : x;
  const double t = fma(xc, 1.4426950408889634, 6755399441055744.0);
  int64_t tb; memcpy(&tb, &t, 8);
  const int k = (int)(uint32_t)tb;
  const double kf = t - 6755399441055744.0;
  double r = fma(kf, -6.93147180369123816490e-01, xc);
  r = fma(kf, -1.90821492927058770002e-10, r);
  double p = 1.0 / 6227020800.0;
  p = fma(p, r, 1.0 / 479001600.0);
  p = fma(p, r, 1.0 / 39916800.0);
  p = fma(p, r, 1.0 / 3628800.0);
  p = fma(p, r, 1.0 / 362880.0);
  p = fma(p, r, 1.0 / 40320.0);
  p = fma(p, r, 1.0 / 5040.0);
  p = fma(p, r, 1.0 / 720.0);
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  int64_t pb; memcpy(&pb, &p, 8);
  pb += (int64_t)k << 52;
  double res; memcpy(&res, &pb, 8);
  return x != x ? x : res;
}
int main() {
  double worst = 0; double wx = 0;
  srand(1);
  for (int i = 0; i < 20000000; ++i) {
    double u = rand() / (double)RAND_MAX;
    double x = (i & 3) == 0 ? -700.0 * u : ((i & 3) == 1 ? -30.0 * u : ((i&3)==2 ? -1.0 * u : -1e-3*u));
    double a = exp_nonpos(x), b = exp(x);
    double e = fabs(a - b) / b;
    if (e > worst) { worst = e; wx = x; }
  }
  printf("max rel err %.3e at x=%.6f (ulp 1.1e-16)\n", worst, wx);
  printf("exp(0)=%.17g exp(-700)=%.6e exp(-1e4)=%.6e nan=%f\n", exp_nonpos(0.0), exp_nonpos(-700.0), exp_nonpos(-1e4), exp_nonpos(NAN));
  return 0;
}
