/* Markstein-corrected division (csrc/eval_common.cuh div_rn_rcp) against the C division on random
   (x, b): x an integer below 2^50 (log-spread), b a random positive double (1/8 of them with an
   all-zero / all-one / 1 / all-one-but-last mantissa).  gcc -O2 -mfma tools/div_check.c -lm;
   ./a.out 3000000000 -> n=3000000000 bad=0 (r02).  Replacing q2 by q (no correction) gives
   bad ~ 24%. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>
static uint64_t s = 0x9E3779B97F4A7C15ull;
static uint64_t nx(void) { uint64_t z = (s += 0x9E3779B97F4A7C15ull); z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }
int main(int argc, char **argv) {
  long n = atol(argv[1]); long bad = 0;
  for (long i = 0; i < n; i++) {
    uint64_t r1 = nx(), r2 = nx();
    double b;
    if ((i & 7) == 0) { /* mantissa edge cases */ uint64_t e = 1023 + 10 + (r1 % 40); uint64_t m = (r1 >> 8) & 3; uint64_t mant = m == 0 ? 0 : m == 1 ? 0xFFFFFFFFFFFFFull : m == 2 ? 1 : 0xFFFFFFFFFFFFEull; uint64_t bits = (e << 52) | mant; memcpy(&b, &bits, 8); }
    else { uint64_t e = 1023 + 10 + (r1 % 40); uint64_t bits = (e << 52) | (r2 & 0xFFFFFFFFFFFFFull); memcpy(&b, &bits, 8); }
    int sh = (int)(nx() % 50); uint64_t xi = nx() >> (14 + sh);  /* integers < 2^50, log-spread */
    double x = (double)xi;
    double y = 1.0 / b;
    double q = x * y;
    double r = fma(-q, b, x);
    double q2 = fma(r, y, q);
    double ref = x / b;
    if (q2 != ref) { if (bad < 10) printf("mismatch x=%.17g b=%.17g q2=%.17g ref=%.17g\n", x, b, q2, ref); bad++; }
  }
  printf("n=%ld bad=%ld\n", n, bad);
  return 0;
}
