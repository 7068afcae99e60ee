/* TEST INFRASTRUCTURE. Pins the device glibc_hypot restatement
 * (paper_1810_03988_b200/csrc/homography.cu) to the host libm hypot that the
 * reference calls (std::hypot, homography.hpp:151): the same algorithm in C,
 * compared bit for bit on N random inputs over ordinary, tiny, huge and
 * arbitrary-bit-pattern magnitudes. Usage: hypot_check N (prints the count of
 * differing results; exit 1 if any). */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#define SCALE 0x1p-600
#define LARGE_VAL 0x1p+511
#define TINY_VAL 0x1p-511
#define EPS 0x1p-54
static double kernel(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}
static double myhypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if ((isinf(x) || isinf(y))) return INFINITY;
    return x + y;
  }
  x = fabs(x); y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  if (ax > LARGE_VAL) {
    if (ay <= ax * EPS) return ax + ay;
    return kernel(ax * SCALE, ay * SCALE) / SCALE;
  }
  if (ay < TINY_VAL) {
    if (ax >= ay / EPS) return ax + ay;
    ax = kernel(ax / SCALE, ay / SCALE) * SCALE;
    return ax;
  }
  if (ay <= ax * EPS) return ax + ay;
  return kernel(ax, ay);
}
static uint64_t s = 88172645463325252ull;
static uint64_t xr(void){ s^=s<<13; s^=s>>7; s^=s<<17; return s; }
static double rnd(void){ uint64_t b = xr(); double d; int mode = b & 3; b >>= 2;
  if (mode == 0) return ((double)(b >> 11) / 9007199254740992.0) * 10.0 - 5.0;
  if (mode == 1) return ((double)(b >> 11) / 9007199254740992.0) * 6.0;
  if (mode == 2) { uint64_t u = xr(); memcpy(&d, &u, 8); return isfinite(d) ? d : 1.0; }
  return ((double)(b >> 11) / 9007199254740992.0) * 1e-3; }
int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 1000000, bad = 0;
  for (long i = 0; i < n; ++i) {
    double x = rnd(), y = rnd();
    double a = hypot(x, y), b = myhypot(x, y);
    if (memcmp(&a, &b, 8)) { if (bad < 5) printf("diff %a %a -> %a %a\n", x, y, a, b); ++bad; }
  }
  printf("%ld / %ld differ\n", bad, n);
  return bad != 0;
}
