/* Empirical check of the RcpDiv identity the specialized search kernels rely
 * on (rpg_device.cuh rcp_div): for y = RN(1/d), q0 = RN(a*y),
 * rem = RN(a - d*q0) (fma), q = RN(q0 + y*rem) (fma) equals RN(a/d).
 * d ranges over every repetition denominator b * num_SM the plans can build
 * (b <= 4095) for several SM counts; a is random (sign, 52-bit mantissa,
 * exponent in [-900, 900]) plus integers and the model's typical values.
 * Prints the number of mismatches (0 expected) and exits non-zero on any. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t s = 0x9e3779b97f4a7c15ULL;
static uint64_t next(void) {  /* splitmix64 */
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static double rand_double(void) {
  uint64_t r = next();
  int e = (int)(next() % 1801) - 900;
  uint64_t bits = ((uint64_t)(e + 1023) << 52) | (r & 0xfffffffffffffULL);
  double a;
  memcpy(&a, &bits, 8);
  return (next() & 1) ? -a : a;
}

int main(int argc, char** argv) {
  const int per_d = argc > 1 ? atoi(argv[1]) : 2000;
  const int sms[] = {148, 132, 16, 80, 1};
  long long bad = 0, total = 0;
  for (unsigned si = 0; si < sizeof sms / sizeof sms[0]; ++si) {
    for (int b = 1; b <= 4095; ++b) {
      const double d = (double)b * (double)sms[si];
      const double y = 1.0 / d;
      for (int i = 0; i < per_d; ++i) {
        double a;
        switch (i % 4) {
          case 0: a = rand_double(); break;
          case 1: a = (double)(next() % (1ULL << 53)); break;
          case 2: a = (double)(next() % 100000000ULL) / 7.0; break;
          default: a = ldexp((double)(next() % (1ULL << 53)), (int)(next() % 120) - 60); break;
        }
        const double q0 = a * y;
        const double rem = fma(-d, q0, a);
        const double q = fma(y, rem, q0);
        const double ref = a / d;
        ++total;
        if (memcmp(&q, &ref, 8) != 0 && !(isnan(q) && isnan(ref))) {
          if (bad < 5) printf("mismatch a=%a d=%a q=%a ref=%a\n", a, d, q, ref);
          ++bad;
        }
      }
    }
  }
  printf("%lld mismatches of %lld\n", bad, total);
  return bad != 0;
}
